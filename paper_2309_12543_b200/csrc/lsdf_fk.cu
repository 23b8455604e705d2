// lsdf_fk.cu — stage 1: batched forward kinematics + window alignment.
//
//   fk_align_kernel  robot.py:305-347 (FK) + placement.py:60-99 (alignment)
//   align_kernel     placement.py:60-99 alone (compute_alignment API)
//
// One thread per configuration walks the parents-first chain in fp64 with
// the reference's operation order (lsdf_math.cuh); the per-link world poses
// of the configuration live in shared memory so children can read any
// earlier link.  For the geometry links the thread also splits T into the
// window anchor and residual.  Outputs are written link-major per config,
// matching LinkPoseBatch (C, L, 3, 3).
#include <cstdlib>

#include "lsdf_device.cuh"

using namespace lsdf;

namespace {

struct FkParams {
    lsdf_link links[LSDF_MAX_LINKS];
    int32_t n_links, n_geo, D;
    int32_t link_major;  // geometry outputs (n_geo, C, .) instead of (C, n_geo, .)
    int64_t C;
    const double* q;
    const double* limits;
    lsdf_env_grid env;
    int32_t W[3];
    double rinv[3];  // RN(1 / env resolution)
    double* R_all;
    double* T_all;
    double* R_geo;
    double* dt_geo;
    int32_t* anchor_geo;
    int32_t* flags;
    int32_t* acc;        // where the kernels count (flags, or flags + 2 when self-resetting)
    uint32_t* ticket;    // self-resetting flags: CTAs done (the last one publishes and re-zeroes), or null
};

// Self-resetting flags (LSDF_FK_FLAGS_SELF_RESET): every CTA counts into
// acc = flags + 2; the last CTA to finish publishes flags[0..1] and re-zeroes
// acc and the ticket, so a captured cycle needs no memset node.
__device__ __forceinline__ void fk_epilogue(const FkParams& p, bool counted) {
    if (p.ticket == nullptr) return;
    if (counted) __threadfence();  // (only a thread that counted something needs its atomics ordered)
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(p.ticket, 1u) == gridDim.x - 1) {
        __threadfence();
        p.flags[0] = atomicExch(p.acc, 0);
        p.flags[1] = atomicExch(p.acc + 1, 0);
        *p.ticket = 0u;
    }
}

constexpr int FK_THREADS = 128;
constexpr int64_t FK_SERIAL_MIN = 6144;  // measured crossover (round 1): 12.5 vs 13.9 us at 4096, 16.7 vs 14.6 at 8192
#ifndef FK_STAGE_OUTPUTS
#define FK_STAGE_OUTPUTS 1
#endif  // configurations from which one thread per configuration wins

// Three phases per CTA of `cpb` configurations x `lp` link slots (lp = next
// power of two >= n_links):
//   1. one thread per (configuration, link): the joint-local transform
//      (sin/cos, Rodrigues, r_o @ r_motion) — independent work, in parallel;
//   2. one thread per configuration: the parents-first chain (matmuls only);
//   3. one thread per (configuration, link): outputs + window alignment.
__device__ __forceinline__ bool fk_align_body(const FkParams& p, int lp_log2) {
    bool counted = false;
    extern __shared__ double s_fk[];
    // the chain table in shared memory: lanes of a warp read different links,
    // which the constant cache would serialize
    __shared__ lsdf_link s_links[LSDF_MAX_LINKS];
    {
        const double* src = (const double*)p.links;
        double* dst = (double*)s_links;
        const int n = p.n_links * (int)(sizeof(lsdf_link) / sizeof(double));
        for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const int lp = 1 << lp_log2, cpb = FK_THREADS >> lp_log2;
    const int cl = threadIdx.x >> lp_log2, li = threadIdx.x & (lp - 1);
    const int64_t c = (int64_t)blockIdx.x * cpb + cl;
    const bool active = c < p.C && li < p.n_links;
    double* loc = s_fk + ((size_t)cl * lp + li) * 12;             // local transform of (cl, li)
    double* world = s_fk + (size_t)cpb * lp * 12;                 // [cpb][lp][12]
    const double* q = p.q + (c < p.C ? c : 0) * p.D;
    if (c < p.C && p.limits != nullptr) {  // robot.py:297-302
        int bad = 0;
        for (int j = li; j < p.D; j += lp) {
            const double v = q[j];
            bad += (v < p.limits[2 * j] || v > p.limits[2 * j + 1]);
        }
        if (bad) {
            atomicAdd(&p.acc[0], bad);
            counted = true;
        }
    }
    if (active) {
        const lsdf_link& L = s_links[li];
        if (L.kind == 1) {  // revolute: r_o @ rodrigues(q)   robot.py:331-334
            const double a = q[L.q_col];
            double M[9], rl[9];
            double sa, ca;
            sincos(a, &sa, &ca);
            rodrigues(L.skew, L.outer, ca, sa, M);
            mm33(L.joint_R, M, rl);
#pragma unroll
            for (int e = 0; e < 9; ++e) loc[e] = rl[e];
#pragma unroll
            for (int k = 0; k < 3; ++k) loc[9 + k] = L.joint_t[k];
        } else {
#pragma unroll
            for (int e = 0; e < 9; ++e) loc[e] = L.joint_R[e];
            if (L.kind == 2) {  // prismatic: t_o + q * (r_o @ axis)   robot.py:335-337
                const double a = q[L.q_col];
#pragma unroll
                for (int k = 0; k < 3; ++k) loc[9 + k] = DADD(L.joint_t[k], DMUL(a, L.R_axis[k]));
            } else {
#pragma unroll
                for (int k = 0; k < 3; ++k) loc[9 + k] = L.joint_t[k];
            }
        }
    }
    __syncthreads();
    if (li == 0 && c < p.C) {
        double* wc = world + (size_t)cl * lp * 12;
        const double* lc = s_fk + (size_t)cl * lp * 12;
        for (int k2 = 0; k2 < p.n_links; ++k2) {
            const lsdf_link& L = s_links[k2];
            double rj[9], tj[3];
            if (L.kind == 0) {
#pragma unroll
                for (int e = 0; e < 9; ++e) rj[e] = (e == 0 || e == 4 || e == 8) ? 1.0 : 0.0;
                tj[0] = tj[1] = tj[2] = 0.0;
            } else {
                double rp[9], tp[3], rl[9], tl[3], tmp[3];
                const double* wp = wc + L.parent * 12;
                const double* lk = lc + k2 * 12;
#pragma unroll
                for (int e = 0; e < 9; ++e) {
                    rp[e] = wp[e];
                    rl[e] = lk[e];
                }
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    tp[k] = wp[9 + k];
                    tl[k] = lk[9 + k];
                }
                mm33(rp, rl, rj);        // robot.py:341
                mv_einsum(rp, tl, tmp);  // robot.py:342
#pragma unroll
                for (int k = 0; k < 3; ++k) tj[k] = DADD(tp[k], tmp[k]);
            }
            double R[9], tmp[3];
            mm33(rj, L.link_R, R);         // robot.py:343
            mv_einsum(rj, L.link_t, tmp);  // robot.py:344-346
            double* w = wc + k2 * 12;
#pragma unroll
            for (int e = 0; e < 9; ++e) w[e] = R[e];
#pragma unroll
            for (int k = 0; k < 3; ++k) w[9 + k] = DADD(tj[k], tmp[k]);
        }
    }
    __syncthreads();
    if (!active) return counted;
    const double* w = world + ((size_t)cl * lp + li) * 12;
    const lsdf_link& L = s_links[li];
    if (p.R_all != nullptr) {
        double* dr = p.R_all + (c * p.n_links + li) * 9;
        double* dtt = p.T_all + (c * p.n_links + li) * 3;
#pragma unroll
        for (int e = 0; e < 9; ++e) dr[e] = w[e];
#pragma unroll
        for (int k = 0; k < 3; ++k) dtt[k] = w[9 + k];
    }
    if (L.geom_slot >= 0 && p.R_geo != nullptr) {
        const int64_t o = p.link_major ? L.geom_slot * p.C + c : c * p.n_geo + L.geom_slot;
#pragma unroll
        for (int e = 0; e < 9; ++e) p.R_geo[o * 9 + e] = w[e];
        int32_t anc[3];
        double del[3], T[3] = {w[9], w[10], w[11]};
        if (!align_one(T, p.env.extent, p.env.resolution, p.env.dims, p.W, anc, del, p.rinv)) {
                    atomicAdd(&p.acc[1], 1);
                    counted = true;
                }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            p.dt_geo[o * 3 + k] = del[k];
            p.anchor_geo[o * 3 + k] = anc[k];
        }
    }
    return counted;
}

// Large batches: one thread per configuration walks the whole chain with the
// same arithmetic as the three phases above (identical results), world poses
// in a per-thread local array (any parent order).  The joint sin/cos of all
// links are computed up front (independent, so they overlap), and the
// geometry-link outputs are staged in shared memory in their global layout
// and written by the whole CTA as contiguous, coalesced blocks.  The 3-phase
// kernel keeps small batches latency-short.
constexpr int FKS_THREADS = 64;

// FAR: some link's parent is not the link before it; those parents' poses go
// through a per-thread array (local memory).  Serial chains (every arm here)
// compile without it.
template <bool STAGE, bool LM, bool FAR = true>
__device__ __forceinline__ bool fk_serial_body(const FkParams& p) {
    bool counted = false;
    // every thread walks the same link at the same time: the chain table is
    // read straight from the kernel parameters (uniform constant-bank loads)
    const lsdf_link* s_links = p.links;
    __shared__ bool s_far_child[LSDF_MAX_LINKS];  // link k is the parent of a link other than k + 1
    extern __shared__ double s_out[];  // [FKS_THREADS * n_geo * 9] R, [.. * 3] dt, then i32 anchors
    if (FAR) {
        if (threadIdx.x < LSDF_MAX_LINKS) {
            bool f = false;
            for (int j = 0; j < p.n_links; ++j)
                f |= p.links[j].kind != 0 && p.links[j].parent == (int)threadIdx.x && j != (int)threadIdx.x + 1;
            s_far_child[threadIdx.x] = f;
        }
    }
    __syncthreads();
    const int G = p.n_geo;
    double* sR = s_out;
    double* sdt = sR + FKS_THREADS * G * 9;
    int32_t* sanc = (int32_t*)(sdt + FKS_THREADS * G * 3);
    const int64_t c0 = (int64_t)blockIdx.x * FKS_THREADS;
    const int nc = (int)(p.C - c0 < FKS_THREADS ? p.C - c0 : FKS_THREADS);
    // LM: the warp writes each link's records of its 32 configurations as one
    // contiguous run; lanes past the end walk the last configuration so the
    // warp's control flow stays uniform, and write nothing
    const int lane = threadIdx.x & 31;
    const int64_t cw = c0 + (threadIdx.x & ~31);
    if (LM && cw >= p.C) return counted;
    const int nw = (int)(p.C - cw < 32 ? p.C - cw : 32);
    const bool live = c0 + threadIdx.x < p.C;
    const int64_t c = (LM && !live) ? p.C - 1 : c0 + threadIdx.x;
    if (LM || live) {
        const double* q = p.q + c * p.D;
        if (live && p.limits != nullptr) {  // robot.py:297-302
            int bad = 0;
            for (int j = 0; j < p.D; ++j) {
                const double v = q[j];
                bad += (v < p.limits[2 * j] || v > p.limits[2 * j + 1]);
            }
            if (bad) {
            atomicAdd(&p.acc[0], bad);
            counted = true;
        }
        }
        // world pose of the previous link in registers (serial chains); poses
        // a later non-adjacent child needs go to a per-thread local array
        double prev[12];
        double world[FAR ? LSDF_MAX_LINKS : 1][12];
        // the joints' sines and cosines first: independent of the chain, so
        // they overlap instead of sitting on its dependent path
        double sn[LSDF_MAX_LINKS], cs[LSDF_MAX_LINKS];
        for (int k2 = 0; k2 < p.n_links; ++k2)
            if (s_links[k2].kind == 1) sincos(q[s_links[k2].q_col], &sn[k2], &cs[k2]);
        for (int k2 = 0; k2 < p.n_links; ++k2) {
            const lsdf_link& L = s_links[k2];
            double rl[9], tl[3];  // joint-local transform (phase 1)
            if (L.kind == 1) {    // revolute: r_o @ rodrigues(q)   robot.py:331-334
                double M[9];
                rodrigues(L.skew, L.outer, cs[k2], sn[k2], M);
                mm33(L.joint_R, M, rl);
#pragma unroll
                for (int k = 0; k < 3; ++k) tl[k] = L.joint_t[k];
            } else {
#pragma unroll
                for (int e = 0; e < 9; ++e) rl[e] = L.joint_R[e];
                if (L.kind == 2) {  // prismatic: t_o + q * (r_o @ axis)   robot.py:335-337
                    const double a = q[L.q_col];
#pragma unroll
                    for (int k = 0; k < 3; ++k) tl[k] = DADD(L.joint_t[k], DMUL(a, L.R_axis[k]));
                } else {
#pragma unroll
                    for (int k = 0; k < 3; ++k) tl[k] = L.joint_t[k];
                }
            }
            double rj[9], tj[3];  // joint frame in the world (phase 2)
            if (L.kind == 0) {
#pragma unroll
                for (int e = 0; e < 9; ++e) rj[e] = (e == 0 || e == 4 || e == 8) ? 1.0 : 0.0;
                tj[0] = tj[1] = tj[2] = 0.0;
            } else {
                double rp[9], tp[3], tmp[3];
                if (!FAR || L.parent == k2 - 1) {
#pragma unroll
                    for (int e = 0; e < 9; ++e) rp[e] = prev[e];
#pragma unroll
                    for (int k = 0; k < 3; ++k) tp[k] = prev[9 + k];
                } else {
                    const double* wp = world[FAR ? L.parent : 0];
#pragma unroll
                    for (int e = 0; e < 9; ++e) rp[e] = wp[e];
#pragma unroll
                    for (int k = 0; k < 3; ++k) tp[k] = wp[9 + k];
                }
                mm33(rp, rl, rj);        // robot.py:341
                mv_einsum(rp, tl, tmp);  // robot.py:342
#pragma unroll
                for (int k = 0; k < 3; ++k) tj[k] = DADD(tp[k], tmp[k]);
            }
            double R[9], T[3], tmp[3];
            mm33(rj, L.link_R, R);         // robot.py:343
            mv_einsum(rj, L.link_t, tmp);  // robot.py:344-346
#pragma unroll
            for (int k = 0; k < 3; ++k) T[k] = DADD(tj[k], tmp[k]);
#pragma unroll
            for (int e = 0; e < 9; ++e) prev[e] = R[e];
#pragma unroll
            for (int k = 0; k < 3; ++k) prev[9 + k] = T[k];
            if (FAR && s_far_child[k2]) {
                double* w = world[FAR ? k2 : 0];
#pragma unroll
                for (int e = 0; e < 12; ++e) w[e] = prev[e];
            }
            // outputs + window alignment (phase 3)
            if (p.R_all != nullptr && live) {
                double* dr = p.R_all + (c * p.n_links + k2) * 9;
                double* dtt = p.T_all + (c * p.n_links + k2) * 3;
#pragma unroll
                for (int e = 0; e < 9; ++e) dr[e] = R[e];
#pragma unroll
                for (int k = 0; k < 3; ++k) dtt[k] = T[k];
            }
            if constexpr (LM) if (L.geom_slot >= 0 && p.R_geo != nullptr) {
                __shared__ double s_R[FKS_THREADS / 32][32 * 9];
                __shared__ double s_dt[FKS_THREADS / 32][32 * 3];
                __shared__ int32_t s_anc[FKS_THREADS / 32][32 * 3];
                const int wi = threadIdx.x >> 5;
                int32_t anc[3];
                double del[3];
                if (!align_one(T, p.env.extent, p.env.resolution, p.env.dims, p.W, anc, del, p.rinv) && live)
                    {
                    atomicAdd(&p.acc[1], 1);
                    counted = true;
                }
#pragma unroll
                for (int e = 0; e < 9; ++e) s_R[wi][lane * 9 + e] = R[e];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    s_dt[wi][lane * 3 + k] = del[k];
                    s_anc[wi][lane * 3 + k] = anc[k];
                }
                __syncwarp();
                const int64_t run = (int64_t)L.geom_slot * p.C + cw;  // first record of the warp's run
                for (int i = lane; i < nw * 9; i += 32) p.R_geo[run * 9 + i] = s_R[wi][i];
                for (int i = lane; i < nw * 3; i += 32) {
                    p.dt_geo[run * 3 + i] = s_dt[wi][i];
                    p.anchor_geo[run * 3 + i] = s_anc[wi][i];
                }
                __syncwarp();
            }
            if (!LM && L.geom_slot >= 0 && (STAGE || p.R_geo != nullptr)) {
                const int64_t o = STAGE ? (int64_t)threadIdx.x * G + L.geom_slot : c * G + L.geom_slot;
                double* oR = STAGE ? sR : p.R_geo;
                double* odt = STAGE ? sdt : p.dt_geo;
                int32_t* oanc = STAGE ? sanc : p.anchor_geo;
#pragma unroll
                for (int e = 0; e < 9; ++e) oR[o * 9 + e] = R[e];
                int32_t anc[3];
                double del[3];
                if (!align_one(T, p.env.extent, p.env.resolution, p.env.dims, p.W, anc, del, p.rinv))
                    {
                    atomicAdd(&p.acc[1], 1);
                    counted = true;
                }
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    odt[o * 3 + k] = del[k];
                    oanc[o * 3 + k] = anc[k];
                }
            }
        }
    }
    if (!STAGE || LM) return counted;
    __syncthreads();
    if (p.R_geo == nullptr) return counted;
    // this CTA's configurations are contiguous in every output
    for (int i = threadIdx.x; i < nc * G * 9; i += FKS_THREADS) p.R_geo[c0 * G * 9 + i] = sR[i];
    for (int i = threadIdx.x; i < nc * G * 3; i += FKS_THREADS) {
        p.dt_geo[c0 * G * 3 + i] = sdt[i];
        p.anchor_geo[c0 * G * 3 + i] = sanc[i];
    }
    return counted;
}

__global__ void __launch_bounds__(FK_THREADS) fk_align_kernel(const __grid_constant__ FkParams p, int lp_log2) {
    const bool counted = fk_align_body(p, lp_log2);
    fk_epilogue(p, counted);
}

template <bool STAGE, bool LM, bool FAR = true>
__global__ void __launch_bounds__(FKS_THREADS) fk_align_serial_kernel(const __grid_constant__ FkParams p) {
    const bool counted = fk_serial_body<STAGE, LM, FAR>(p);
    fk_epilogue(p, counted);
}

__global__ void align_kernel(const double* T, int64_t n, lsdf_env_grid env, int32_t W0, int32_t W1, int32_t W2,
                             int32_t* anchor, double* dt, int32_t* flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t W[3] = {W0, W1, W2};
    int32_t a[3];
    double d[3];
    if (!align_one(T + 3 * i, env.extent, env.resolution, env.dims, W, a, d)) atomicAdd(&flags[1], 1);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        anchor[3 * i + k] = a[k];
        dt[3 * i + k] = d[k];
    }
}

}  // namespace

namespace {
int fk_align_impl(const lsdf_link* links, int32_t n_links, int32_t n_geo, const double* q_dev, int64_t C, int32_t D,
                  const double* limits_dev, const lsdf_env_grid* env, const int32_t W[3], double* R_all_dev,
                  double* T_all_dev, double* R_geo_dev, double* dt_geo_dev, int32_t* anchor_geo_dev,
                  int32_t* flags_dev, void* stream, bool link_major, bool flags_self_reset=false) {
    if (n_links < 1 || n_links > LSDF_MAX_LINKS || n_geo > LSDF_MAX_LINKS)
        return fail(LSDF_ERR_VALIDATION, "lsdf_fk_align: %d links outside 1..%d", n_links, LSDF_MAX_LINKS);
    if (C <= 0) return LSDF_OK;
    FkParams p{};
    for (int i = 0; i < n_links; ++i) p.links[i] = links[i];
    p.n_links = n_links;
    p.n_geo = n_geo;
    p.link_major = link_major;
    p.D = D;
    p.C = C;
    p.q = q_dev;
    p.limits = limits_dev;
    if (env) {
        p.env = *env;
        for (int a = 0; a < 3; ++a) p.rinv[a] = 1.0 / env->resolution[a];
    }
    if (W) {
        p.W[0] = W[0];
        p.W[1] = W[1];
        p.W[2] = W[2];
    }
    p.R_all = R_all_dev;
    p.T_all = T_all_dev;
    p.R_geo = R_geo_dev;
    p.dt_geo = dt_geo_dev;
    p.anchor_geo = anchor_geo_dev;
    p.flags = flags_dev;
    p.acc = flags_self_reset ? flags_dev + 2 : flags_dev;
    p.ticket = flags_self_reset ? (uint32_t*)(flags_dev + 4) : nullptr;
    int lp_log2 = 0;
    while ((1 << lp_log2) < n_links) ++lp_log2;
    const int cpb = FK_THREADS >> lp_log2;
    const size_t smem = (size_t)2 * FK_THREADS * 12 * sizeof(double);  // local + world, cpb * lp slots each
    if (flags_self_reset && flags_dev == nullptr) return fail(LSDF_ERR_VALIDATION, "fk: self-resetting flags need a buffer");
    if (flags_dev != nullptr && !flags_self_reset)
        LSDF_TRY(check_cuda(cudaMemsetAsync(flags_dev, 0, 2 * sizeof(int32_t), (cudaStream_t)stream), "fk flags memset"));
    static const int64_t serial_min = [] { const char* v = getenv("LSDF_TUNE_FKSERIAL"); return v && *v ? atoll(v) : FK_SERIAL_MIN; }();
    bool far = false;  // a link whose parent is not the link before it
    for (int j = 0; j < n_links; ++j) far |= links[j].kind != 0 && links[j].parent != j - 1;
    if (C >= serial_min && link_major) {
        if (far)
            fk_align_serial_kernel<true, true, true><<<grid_for(C, FKS_THREADS), FKS_THREADS, 0, (cudaStream_t)stream>>>(p);
        else
            fk_align_serial_kernel<true, true, false><<<grid_for(C, FKS_THREADS), FKS_THREADS, 0, (cudaStream_t)stream>>>(p);
        return check_launch("fk_align_serial_kernel");
    }
    if (C >= serial_min) {
        if (FK_STAGE_OUTPUTS) {
            const size_t smem_s = (size_t)FKS_THREADS * n_geo * (12 * sizeof(double) + 3 * sizeof(int32_t));
            LSDF_TRY(ensure_smem((const void*)fk_align_serial_kernel<true, false>, smem_s, "fk_align_serial_kernel"));
            fk_align_serial_kernel<true, false>
                <<<grid_for(C, FKS_THREADS), FKS_THREADS, smem_s, (cudaStream_t)stream>>>(p);
        } else {
            fk_align_serial_kernel<false, false><<<grid_for(C, FKS_THREADS), FKS_THREADS, 0, (cudaStream_t)stream>>>(p);
        }
        return check_launch("fk_align_serial_kernel");
    }
    fk_align_kernel<<<grid_for(C, cpb), FK_THREADS, smem, (cudaStream_t)stream>>>(p, lp_log2);
    return check_launch("fk_align_kernel");
}
}  // namespace

extern "C" int lsdf_fk_align(const lsdf_link* links, int32_t n_links, int32_t n_geo, const double* q_dev, int64_t C,
                             int32_t D, const double* limits_dev, const lsdf_env_grid* env, const int32_t W[3],
                             double* R_all_dev, double* T_all_dev, double* R_geo_dev, double* dt_geo_dev,
                             int32_t* anchor_geo_dev, int32_t* flags_dev, void* stream) {
    return fk_align_impl(links, n_links, n_geo, q_dev, C, D, limits_dev, env, W, R_all_dev, T_all_dev, R_geo_dev,
                         dt_geo_dev, anchor_geo_dev, flags_dev, stream, false);
}

extern "C" int lsdf_fk_align_link_major(const lsdf_link* links, int32_t n_links, int32_t n_geo, const double* q_dev,
                                        int64_t C, int32_t D, const double* limits_dev, const lsdf_env_grid* env,
                                        const int32_t W[3], double* R_all_dev, double* T_all_dev, double* R_geo_dev,
                                        double* dt_geo_dev, int32_t* anchor_geo_dev, int32_t* flags_dev,
                                        void* stream) {
    return fk_align_impl(links, n_links, n_geo, q_dev, C, D, limits_dev, env, W, R_all_dev, T_all_dev, R_geo_dev,
                         dt_geo_dev, anchor_geo_dev, flags_dev, stream, true);
}

extern "C" int lsdf_fk_align_ex(const lsdf_link* links, int32_t n_links, int32_t n_geo, const double* q_dev, int64_t C,
                                int32_t D, const double* limits_dev, const lsdf_env_grid* env, const int32_t W[3],
                                double* R_all_dev, double* T_all_dev, double* R_geo_dev, double* dt_geo_dev,
                                int32_t* anchor_geo_dev, int32_t* flags_dev, int32_t options, void* stream) {
    return fk_align_impl(links, n_links, n_geo, q_dev, C, D, limits_dev, env, W, R_all_dev, T_all_dev, R_geo_dev,
                         dt_geo_dev, anchor_geo_dev, flags_dev, stream, (options & LSDF_FK_LINK_MAJOR) != 0,
                         (options & LSDF_FK_FLAGS_SELF_RESET) != 0);
}

extern "C" int lsdf_align(const double* T_dev, int64_t n, const lsdf_env_grid* env, const int32_t W[3],
                          int32_t* anchor_dev, double* dt_dev, int32_t* flags_dev, void* stream) {
    if (n <= 0) return LSDF_OK;
    align_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(T_dev, n, *env, W[0], W[1], W[2], anchor_dev,
                                                                       dt_dev, flags_dev);
    return check_launch("align_kernel");
}
