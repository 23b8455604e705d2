// lsdf_query.cu — stages 1, 3 and 4 of the hot path on sm_100a, plus the
// obstacle voxelization and the materialized (paper) mode.
//
//   fk_align_kernel      robot.py:305-347 + placement.py:60-99   (warp per config)
//   voxel_scatter/compact query.py:106-125 + grids.py:93-113     (bitmap + rank scan)
//   query_direct_kernel  placement.py:148-169, grids.py:155-191,
//                        query.py:61-103,128-176                  (fused lookup + min/argmin)
//   place_windows_kernel placement.py:267-313
//   assemble_kernel      query.py:61-103
//   query_dense_kernel   query.py:128-150
#include <cub/block/block_scan.cuh>

#include "lsdf_common.cuh"
#include "lsdf_math.cuh"

using namespace lsdf;

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t u = __shfl_xor_sync(FULL, v, o);
        v = u < v ? u : v;
    }
    return v;
}
__device__ __forceinline__ float warp_min_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

__device__ __forceinline__ GridView view_of(const lsdf_link_grid& g) {
    GridView v;
    v.v = g.values_dev;
    v.nx = g.dims[0];
    v.ny = g.dims[1];
    v.nz = g.dims[2];
    v.d_far = g.d_far;
    v.ex = g.extent[0];
    v.ey = g.extent[1];
    v.ez = g.extent[2];
    v.rx = g.resolution[0];
    v.ry = g.resolution[1];
    v.rz = g.resolution[2];
    return v;
}

struct LdgLoad {
    const float* p;
    __device__ __forceinline__ float operator()(int64_t i) const { return __ldg(p + i); }
};

// ============================================================ stage 1: FK + align
struct FkParams {
    lsdf_link links[LSDF_MAX_LINKS];
    int32_t n_links, n_geo, D, pad_;
    int64_t C;
    const double* q;
    const double* limits;
    lsdf_env_grid env;
    int32_t W[3];
    double* R_all;
    double* T_all;
    double* R_geo;
    double* dt_geo;
    int32_t* anchor_geo;
    int32_t* flags;
};

constexpr int FK_WARPS = 4;

__global__ void __launch_bounds__(32 * FK_WARPS) fk_align_kernel(const __grid_constant__ FkParams p) {
    __shared__ double s_rl[FK_WARPS][LSDF_MAX_LINKS][9];
    __shared__ double s_tl[FK_WARPS][LSDF_MAX_LINKS][3];
    __shared__ double s_R[FK_WARPS][LSDF_MAX_LINKS][9];
    __shared__ double s_T[FK_WARPS][LSDF_MAX_LINKS][3];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c = (int64_t)blockIdx.x * FK_WARPS + w;
    if (c >= p.C) return;  // whole warp exits together
    const double* q = p.q + c * p.D;

    if (p.limits != nullptr && lane < p.D) {  // robot.py:297-302
        const double v = q[lane];
        if (v < p.limits[2 * lane] || v > p.limits[2 * lane + 1]) atomicAdd(&p.flags[0], 1);
    }
    // Joint-local transforms are independent per link: one lane each.
    if (lane < p.n_links) {
        const lsdf_link& L = p.links[lane];
        double* rl = s_rl[w][lane];
        double* tl = s_tl[w][lane];
        if (L.kind == 1) {  // revolute: r_o @ rodrigues(q)   robot.py:331-334
            const double a = q[L.q_col];
            double M[9];
            rodrigues(L.skew, L.outer, cos(a), sin(a), M);
            mm33(L.joint_R, M, rl);
            tl[0] = L.joint_t[0];
            tl[1] = L.joint_t[1];
            tl[2] = L.joint_t[2];
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
    }
    __syncwarp();
    // The chain itself is sequential (parents first): lane 0 walks it.
    if (lane == 0) {
        for (int li = 0; li < p.n_links; ++li) {
            const lsdf_link& L = p.links[li];
            double rj[9], tj[3];
            if (L.kind == 0) {
                const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
#pragma unroll
                for (int e = 0; e < 9; ++e) rj[e] = I[e];
                tj[0] = tj[1] = tj[2] = 0.0;
            } else {
                const double* rp = s_R[w][L.parent];
                const double* tp = s_T[w][L.parent];
                double tmp[3];
                mm33(rp, s_rl[w][li], rj);                // robot.py:341
                mv_einsum(rp, s_tl[w][li], tmp);          // robot.py:342
#pragma unroll
                for (int k = 0; k < 3; ++k) tj[k] = DADD(tp[k], tmp[k]);
            }
            double tmp[3];
            mm33(rj, L.link_R, s_R[w][li]);               // robot.py:343
            mv_einsum(rj, L.link_t, tmp);                 // robot.py:344-346
#pragma unroll
            for (int k = 0; k < 3; ++k) s_T[w][li][k] = DADD(tj[k], tmp[k]);
        }
    }
    __syncwarp();
    if (lane < p.n_links) {
        const lsdf_link& L = p.links[lane];
        const double* R = s_R[w][lane];
        const double* T = s_T[w][lane];
        if (p.R_all != nullptr) {
            double* dst = p.R_all + (c * p.n_links + lane) * 9;
#pragma unroll
            for (int e = 0; e < 9; ++e) dst[e] = R[e];
            double* dt = p.T_all + (c * p.n_links + lane) * 3;
            dt[0] = T[0];
            dt[1] = T[1];
            dt[2] = T[2];
        }
        if (L.geom_slot >= 0 && p.R_geo != nullptr) {
            const int64_t o = c * p.n_geo + L.geom_slot;
            double* rg = p.R_geo + o * 9;
#pragma unroll
            for (int e = 0; e < 9; ++e) rg[e] = R[e];
            int32_t anc[3];
            double del[3];
            const bool ok = align_one(T, p.env.extent, p.env.resolution, p.env.dims, p.W, anc, del);
            if (!ok) atomicAdd(&p.flags[1], 1);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                p.dt_geo[o * 3 + k] = del[k];
                p.anchor_geo[o * 3 + k] = anc[k];
            }
        }
    }
}

__global__ void align_kernel(const double* T, int64_t n, lsdf_env_grid env, int32_t W0, int32_t W1,
                             int32_t W2, int32_t* anchor, double* dt, int32_t* flags) {
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

// ============================================================ obstacles
struct Occupancy {
    uint32_t* bitmap;   // ceil(V/32) words, C-order bit index (ix*ny + iy)*nz + iz
    int32_t* posgrid;   // V entries: position of the voxel in the obstacle list
    int32_t* counters;  // [0] n_occupied, [1] n_dropped, [2..3] spare
    int64_t n_words;
};

__host__ __device__ inline int64_t n_vox(const lsdf_env_grid& e) {
    return (int64_t)e.dims[0] * e.dims[1] * e.dims[2];
}

Occupancy carve(void* base, const lsdf_env_grid& env) {
    Occupancy o;
    const int64_t V = n_vox(env);
    o.n_words = (V + 31) / 32;
    char* p = (char*)base;
    o.counters = (int32_t*)p;
    p += 64;
    o.bitmap = (uint32_t*)p;
    p += ((o.n_words * 4 + 255) / 256) * 256;
    o.posgrid = (int32_t*)p;
    return o;
}

template <typename T>
__global__ void voxel_scatter_kernel(const T* __restrict__ pts, int64_t N, lsdf_env_grid env,
                                     uint32_t* bitmap, int32_t* counters) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool dropped = false;
    if (i < N) {
        const double x = (double)pts[3 * i], y = (double)pts[3 * i + 1], z = (double)pts[3 * i + 2];
        const double ex = env.extent[0], ey = env.extent[1], ez = env.extent[2];
        // query.py:112 in-bounds test [-e, e) per axis (NaN -> dropped)
        const bool inside = (x >= -ex) && (x < ex) && (y >= -ey) && (y < ey) && (z >= -ez) && (z < ez);
        if (inside) {
            // grids.py:107-111: floor((p + e) / r), clipped to [0, dims-1]
            int64_t ix = (int64_t)floor(DDIV(DADD(x, ex), env.resolution[0]));
            int64_t iy = (int64_t)floor(DDIV(DADD(y, ey), env.resolution[1]));
            int64_t iz = (int64_t)floor(DDIV(DADD(z, ez), env.resolution[2]));
            ix = ix < 0 ? 0 : (ix > env.dims[0] - 1 ? env.dims[0] - 1 : ix);
            iy = iy < 0 ? 0 : (iy > env.dims[1] - 1 ? env.dims[1] - 1 : iy);
            iz = iz < 0 ? 0 : (iz > env.dims[2] - 1 ? env.dims[2] - 1 : iz);
            const int64_t lin = (ix * env.dims[1] + iy) * env.dims[2] + iz;
            atomicOr(bitmap + (lin >> 5), 1u << (lin & 31));
        } else {
            dropped = true;
        }
    }
    const unsigned b = __ballot_sync(FULL, dropped);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(&counters[1], __popc(b));
}

constexpr int COMPACT_THREADS = 1024;

// Rank every set bit in C-order (== np.unique(axis=0) order), write the
// position grid and the sorted index list.  One CTA; each thread owns a
// contiguous run of words.
__global__ void __launch_bounds__(COMPACT_THREADS)
voxel_compact_kernel(const uint32_t* __restrict__ bitmap, int64_t n_words, lsdf_env_grid env,
                     int32_t* posgrid, int32_t* indices, int32_t* counters) {
    using Scan = cub::BlockScan<int, COMPACT_THREADS>;
    __shared__ typename Scan::TempStorage tmp;
    const int64_t per = (n_words + COMPACT_THREADS - 1) / COMPACT_THREADS;
    const int64_t w0 = threadIdx.x * per;
    const int64_t w1 = w0 + per < n_words ? w0 + per : n_words;
    int cnt = 0;
    for (int64_t w = w0; w < w1; ++w) cnt += __popc(bitmap[w]);
    int rank, total;
    Scan(tmp).ExclusiveSum(cnt, rank, total);
    const int64_t nyz = (int64_t)env.dims[1] * env.dims[2];
    for (int64_t w = w0; w < w1; ++w) {
        uint32_t bits = bitmap[w];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int64_t lin = w * 32 + b;
            posgrid[lin] = rank;
            if (indices != nullptr) {
                indices[3 * (int64_t)rank] = (int32_t)(lin / nyz);
                indices[3 * (int64_t)rank + 1] = (int32_t)((lin / env.dims[2]) % env.dims[1]);
                indices[3 * (int64_t)rank + 2] = (int32_t)(lin % env.dims[2]);
            }
            ++rank;
        }
    }
    if (threadIdx.x == 0) counters[0] = total;
}

__global__ void occ_from_indices_kernel(const int32_t* idx, int64_t N, lsdf_env_grid env, uint32_t* bitmap,
                                        int32_t* posgrid, int mode) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int64_t lin = ((int64_t)idx[3 * i] * env.dims[1] + idx[3 * i + 1]) * env.dims[2] + idx[3 * i + 2];
    if (mode == 0) {  // sorted unique: position == list index
        posgrid[lin] = (int32_t)i;
        atomicOr(bitmap + (lin >> 5), 1u << (lin & 31));
    } else if (mode == 1) {  // general, pass 1: reset touched entries
        posgrid[lin] = 0x7fffffff;
    } else {  // general, pass 2: first occurrence wins (numpy argmin semantics)
        atomicMin(posgrid + lin, (int32_t)i);
        atomicOr(bitmap + (lin >> 5), 1u << (lin & 31));
    }
}

// ============================================================ stage 3+4: direct query
struct QueryParams {
    lsdf_link_grid grids[LSDF_MAX_LINKS];
    const double* R;
    const double* dt;
    const int32_t* anchor;
    int64_t C;
    int32_t n_geo, split;
    int32_t W[3];
    int32_t full_window;  // iterate whole window, masking per cell (d_far_l < clamp)
    double e_r;
    const double* P;
    int32_t Wmax, by_position;
    const int16_t* zrange;
    const uint32_t* mask_bits;
    int32_t dims[3];
    float clamp;
    const uint32_t* bitmap;
    const int32_t* posgrid;
    float* d_out;
    int32_t* link_out;
    int32_t* voxel_out;
    float* per_link;
};

constexpr int QCAP = 32 * 16 + 32;  // queue entries per warp: <=16 bits per lane per round

// One CTA per configuration; `split` warps per geometry link.  Each warp
// scans its share of the window's (x, y) columns against the occupancy
// bitmap, queues the occupied in-mask cells in shared memory and evaluates
// them 32 at a time (no lane idles on divergent bit counts), keeping the
// lexicographic minimum key (value, position, link).  The block reduces the
// keys and writes the finished (d, link, voxel) — no second pass, no atomics.
__global__ void __launch_bounds__(1024) query_direct_kernel(const __grid_constant__ QueryParams p) {
    extern __shared__ uint32_t s_queue[];
    __shared__ uint64_t s_key[32];
    __shared__ float s_val[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int64_t c = blockIdx.x;
    const int l = warp / p.split, sidx = warp % p.split;
    uint32_t* queue = s_queue + warp * QCAP;

    uint64_t best = ~0ull;
    float bestval = INFINITY;
    if (l < p.n_geo) {
        const lsdf_link_grid& G = p.grids[l];
        const GridView gv = view_of(G);
        const LdgLoad ld{G.values_dev};
        const int64_t o = c * p.n_geo + l;
        double R[9], dtinv[3];
#pragma unroll
        for (int e = 0; e < 9; ++e) R[e] = __ldg(p.R + o * 9 + e);
        shift_inverse(R, p.dt + o * 3, p.e_r, dtinv);
        const int ax = p.anchor[o * 3], ay = p.anchor[o * 3 + 1], az = p.anchor[o * 3 + 2];
        const int W0 = p.W[0], W1 = p.W[1], W2 = p.W[2];
        const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
        const double* Px = p.P;
        const double* Py = p.P + p.Wmax;
        const double* Pz = p.P + 2 * p.Wmax;
        const int n_cols = W0 * W1;
        int qlen = 0;

        auto evaluate = [&](uint32_t cell) {
            const int mx = cell & 0xff, my = (cell >> 8) & 0xff, mz = (cell >> 16) & 0xff;
            float v;
            bool in_mask = true;
            if (p.full_window) {
                const int bit = mx + W0 * (my + W1 * mz);
                in_mask = (__ldg(p.mask_bits + (bit >> 5)) >> (bit & 31)) & 1u;
            }
            if (in_mask) {
                double pt[3];
                window_point(__ldg(Px + mx), __ldg(Py + my), __ldg(Pz + mz), R, dtinv, p.e_r, pt);
                v = trilinear_at(gv, pt[0], pt[1], pt[2], ld);
                bestval = fminf(bestval, v);
            } else {
                v = gv.d_far;
            }
            const int64_t lin = ((int64_t)(ax + mx) * ny + (ay + my)) * nz + (az + mz);
            const uint32_t pos = p.by_position ? (uint32_t)__ldg(p.posgrid + lin) : (uint32_t)lin;
            const uint64_t key = ((uint64_t)orderable(v) << 32) | (uint64_t)(pos * (uint32_t)p.n_geo + l);
            best = key < best ? key : best;
        };

        for (int base = sidx * 32; base < n_cols; base += 32 * p.split) {
            const int col = base + lane;
            int zcur = 0, zend = 0;
            int64_t bitbase = 0;
            if (col < n_cols) {
                const int mx = col % W0, my = col / W0;
                const int x = ax + mx, y = ay + my;
                if (x >= 0 && x < nx && y >= 0 && y < ny) {
                    int zlo = 0, zhi = W2;
                    if (!p.full_window) {
                        zlo = __ldg(p.zrange + 2 * col);
                        zhi = __ldg(p.zrange + 2 * col + 1);
                    }
                    zcur = az + zlo > 0 ? az + zlo : 0;
                    zend = az + zhi < nz ? az + zhi : nz;
                    bitbase = ((int64_t)x * ny + y) * nz;
                }
            }
            // Consume the column's z-run in segments of <= 16 bits, all lanes in step.
            while (__any_sync(FULL, zcur < zend)) {
                uint32_t bits = 0;
                int zs = zcur;
                if (zcur < zend) {
                    const int64_t bp = bitbase + zcur;
                    const int off = (int)(bp & 31);
                    int n = zend - zcur;
                    n = n < 16 ? n : 16;
                    n = n < 32 - off ? n : 32 - off;
                    bits = (__ldg(p.bitmap + (bp >> 5)) >> off) & ((1u << n) - 1u);
                    zcur += n;
                }
                const int cnt = __popc(bits);
                int incl = cnt;
#pragma unroll
                for (int o2 = 1; o2 < 32; o2 <<= 1) {
                    const int t = __shfl_up_sync(FULL, incl, o2);
                    if (lane >= o2) incl += t;
                }
                const int total = __shfl_sync(FULL, incl, 31);
                if (bits) {
                    const int mx = col % W0, my = col / W0;
                    int slot = qlen + incl - cnt;
                    while (bits) {
                        const int b = __ffs(bits) - 1;
                        bits &= bits - 1;
                        const int mz = zs + b - az;
                        queue[slot++] = (uint32_t)mx | ((uint32_t)my << 8) | ((uint32_t)mz << 16);
                    }
                }
                qlen += total;
                __syncwarp();
                while (qlen >= 32) {
                    evaluate(queue[qlen - 32 + lane]);
                    qlen -= 32;
                }
                __syncwarp();
            }
        }
        if (lane < qlen) evaluate(queue[lane]);
    }
    best = warp_min_u64(best);
    bestval = warp_min_f(bestval);
    if (lane == 0) {
        s_key[warp] = best;
        s_val[warp] = bestval;
    }
    __syncthreads();
    if (warp == 0) {
        uint64_t k = lane < nwarps ? s_key[lane] : ~0ull;
        k = warp_min_u64(k);
        if (p.per_link != nullptr && lane < p.n_geo) {  // query.py:153-176
            float m = fminf(p.clamp, p.grids[lane].d_far);
            for (int s2 = 0; s2 < p.split; ++s2) m = fminf(m, s_val[lane * p.split + s2]);
            p.per_link[c * p.n_geo + lane] = m;
        }
        if (lane == 0) {
            const uint32_t hi = (uint32_t)(k >> 32);
            if (k == ~0ull || hi >= orderable(p.clamp)) {
                p.d_out[c] = p.clamp;  // nothing closer than the monitored range
                p.link_out[c] = -1;
                p.voxel_out[c] = -1;
            } else {
                const uint32_t lo = (uint32_t)k;
                const uint32_t pos = lo / (uint32_t)p.n_geo;
                p.d_out[c] = from_orderable(hi);
                p.link_out[c] = (int32_t)(lo % (uint32_t)p.n_geo);
                p.voxel_out[c] = p.by_position ? (int32_t)pos : __ldg(p.posgrid + pos);
            }
        }
    }
}

// ============================================================ materialized mode
struct PlaceParams {
    lsdf_link_grid grids[LSDF_MAX_LINKS];
    const double* R;
    const double* dt;
    int32_t n_geo;
    int32_t W[3];
    double e_r;
    const double* P;
    int32_t Wmax;
    const uint32_t* mask_bits;
    float* out;
};

__global__ void place_windows_kernel(const __grid_constant__ PlaceParams p) {
    const int64_t f = blockIdx.x;  // field = c * n_geo + l
    const int l = (int)(f % p.n_geo);
    const lsdf_link_grid& G = p.grids[l];
    const GridView gv = view_of(G);
    const LdgLoad ld{G.values_dev};
    double R[9], dtinv[3];
#pragma unroll
    for (int e = 0; e < 9; ++e) R[e] = p.R[f * 9 + e];
    shift_inverse(R, p.dt + f * 3, p.e_r, dtinv);
    const int W0 = p.W[0], W1 = p.W[1];
    const int n = W0 * W1 * p.W[2];
    float* dst = p.out + f * (int64_t)n;
    for (int cell = threadIdx.x; cell < n; cell += blockDim.x) {
        const bool keep = (__ldg(p.mask_bits + (cell >> 5)) >> (cell & 31)) & 1u;
        float v = gv.d_far;
        if (keep) {
            const int mx = cell % W0, my = (cell / W0) % W1, mz = cell / (W0 * W1);
            double pt[3];
            window_point(p.P[mx], p.P[p.Wmax + my], p.P[2 * p.Wmax + mz], R, dtinv, p.e_r, pt);
            v = trilinear_at(gv, pt[0], pt[1], pt[2], ld);
        }
        dst[cell] = v;
    }
}

__global__ void fill_kernel(float* out, int64_t n, float v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = v;
}

__device__ __forceinline__ void atomic_min_float(float* addr, float v) {
    if (v >= 0.0f)
        atomicMin((int*)addr, __float_as_int(v));
    else
        atomicMax((unsigned int*)addr, __float_as_uint(v));
}

__global__ void assemble_kernel(const float* __restrict__ windows, const int32_t* anchors, const int32_t* configs,
                                int32_t W0, int32_t W1, int32_t W2, lsdf_env_grid env, float* out) {
    const int64_t f = blockIdx.x;
    const int64_t c = configs[f];
    const int ax = anchors[3 * f], ay = anchors[3 * f + 1], az = anchors[3 * f + 2];
    const int n = W0 * W1 * W2;
    const int64_t V = n_vox(env);
    for (int cell = threadIdx.x; cell < n; cell += blockDim.x) {
        const int mx = cell % W0, my = (cell / W0) % W1, mz = cell / (W0 * W1);
        const int x = ax + mx, y = ay + my, z = az + mz;
        if (x < 0 || y < 0 || z < 0 || x >= env.dims[0] || y >= env.dims[1] || z >= env.dims[2]) continue;
        const float v = windows[f * n + cell];
        float* dst = out + c * V + ((int64_t)x * env.dims[1] + y) * env.dims[2] + z;
        if (v < *dst) atomic_min_float(dst, v);
    }
}

__global__ void query_dense_kernel(const float* __restrict__ values, int64_t V, lsdf_env_grid env,
                                   const int32_t* __restrict__ idx, int64_t N, float* d, int32_t* argmin) {
    __shared__ uint64_t s_key[32];
    const int64_t c = blockIdx.x;
    uint64_t best = ~0ull;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        const int64_t lin = ((int64_t)idx[3 * i] * env.dims[1] + idx[3 * i + 1]) * env.dims[2] + idx[3 * i + 2];
        const float v = __ldg(values + c * V + lin);
        const uint64_t key = ((uint64_t)orderable(v) << 32) | (uint64_t)i;
        best = key < best ? key : best;
    }
    best = warp_min_u64(best);
    if ((threadIdx.x & 31) == 0) s_key[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint64_t k = threadIdx.x < (blockDim.x >> 5) ? s_key[threadIdx.x] : ~0ull;
        k = warp_min_u64(k);
        if (threadIdx.x == 0) {
            d[c] = from_orderable((uint32_t)(k >> 32));
            argmin[c] = (int32_t)(uint32_t)k;
        }
    }
}

__global__ void per_link_fields_kernel(const float* __restrict__ windows, const int32_t* anchors,
                                       const int32_t* configs, const int32_t* links, const float* d_far,
                                       int32_t W0, int32_t W1, int32_t W2, int32_t n_links, lsdf_env_grid env,
                                       const uint32_t* __restrict__ bitmap, float* out) {
    __shared__ float s_min[32];
    const int64_t f = blockIdx.x;
    const int ax = anchors[3 * f], ay = anchors[3 * f + 1], az = anchors[3 * f + 2];
    const int n = W0 * W1 * W2;
    float m = d_far[f];  // query.py:171 limit starts at the field's sentinel
    for (int cell = threadIdx.x; cell < n; cell += blockDim.x) {
        const int x = ax + cell % W0, y = ay + (cell / W0) % W1, z = az + cell / (W0 * W1);
        if (x < 0 || y < 0 || z < 0 || x >= env.dims[0] || y >= env.dims[1] || z >= env.dims[2]) continue;
        const int64_t lin = ((int64_t)x * env.dims[1] + y) * env.dims[2] + z;
        if ((__ldg(bitmap + (lin >> 5)) >> (lin & 31)) & 1u) m = fminf(m, windows[f * n + cell]);
    }
    m = warp_min_f(m);
    if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? s_min[threadIdx.x] : INFINITY;
        m = warp_min_f(m);
        if (threadIdx.x == 0) atomic_min_float(out + (int64_t)configs[f] * n_links + links[f], m);
    }
}

// query.py:254-291; world centre = einsum("bsij,sj->bsi") + T, distance fp64.
__global__ void sphere_baseline_kernel(const double* __restrict__ R, const double* __restrict__ T, int32_t L,
                                       const int32_t* sl, const double* sc, const double* sr, int32_t S,
                                       const int32_t* __restrict__ idx, int64_t N, lsdf_env_grid env, double* out) {
    extern __shared__ double s_w[];  // S x 4: world centre + radius
    __shared__ double s_min[32];
    const int64_t c = blockIdx.x;
    for (int s = threadIdx.x; s < S; s += blockDim.x) {
        const double* Rc = R + (c * L + sl[s]) * 9;
        double w[3];
        mv_einsum(Rc, sc + 3 * s, w);
        for (int k = 0; k < 3; ++k) s_w[4 * s + k] = DADD(w[k], T[(c * L + sl[s]) * 3 + k]);
        s_w[4 * s + 3] = sr[s];
    }
    __syncthreads();
    double m = INFINITY;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        double x[3];
        for (int k = 0; k < 3; ++k)
            x[k] = DADD(-env.extent[k], DMUL(DADD((double)idx[3 * i + k], 0.5), env.resolution[k]));
        for (int s = 0; s < S; ++s) {
            const double d0 = DSUB(s_w[4 * s], x[0]), d1 = DSUB(s_w[4 * s + 1], x[1]),
                         d2 = DSUB(s_w[4 * s + 2], x[2]);
            const double d = DSUB(DSQRT(dot3(d0, d1, d2, d0, d1, d2)), s_w[4 * s + 3]);
            m = d < m ? d : m;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double u = __shfl_xor_sync(FULL, m, o);
        m = u < m ? u : m;
    }
    if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = INFINITY;
        for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) r = s_min[w2] < r ? s_min[w2] : r;
        out[c] = r;
    }
}

__global__ void voxel_index_kernel(const double* pts, int64_t N, lsdf_env_grid env, int32_t* out, int32_t* flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    bool bad = false;
    for (int a = 0; a < 3; ++a) {
        const double x = pts[3 * i + a];
        if (!(x >= -env.extent[a] && x < env.extent[a])) bad = true;
        int64_t j = (int64_t)floor(DDIV(DADD(x, env.extent[a]), env.resolution[a]));
        j = j < 0 ? 0 : (j > env.dims[a] - 1 ? env.dims[a] - 1 : j);
        out[3 * i + a] = (int32_t)j;
    }
    if (bad) atomicAdd(flags, 1);
}

// ============================================================ standalone pieces
__global__ void trilinear_kernel(lsdf_link_grid g, const double* pts, int64_t n, double scale, float* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = trilinear_at(view_of(g), DMUL(pts[3 * i], scale), DMUL(pts[3 * i + 1], scale),
                          DMUL(pts[3 * i + 2], scale), LdgLoad{g.values_dev});
}

__global__ void transform_exact_kernel(const double* R, const double* dt, int64_t B, const double* P, int64_t V,
                                       double e_r, double* G) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B * V) return;
    const int64_t b = i / V, v = i % V;
    double Rb[9], dtinv[3];
#pragma unroll
    for (int e = 0; e < 9; ++e) Rb[e] = R[b * 9 + e];
    shift_inverse(Rb, dt + b * 3, e_r, dtinv);
    const double px = P[3 * v], py = P[3 * v + 1], pz = P[3 * v + 2];
#pragma unroll
    for (int k = 0; k < 3; ++k)
        G[i * 3 + k] = DADD(DFMA(pz, Rb[6 + k], DFMA(py, Rb[3 + k], DMUL(px, Rb[k]))), dtinv[k]);
}

}  // namespace

// ============================================================ C ABI
extern "C" int lsdf_fk_align(const lsdf_link* links, int32_t n_links, int32_t n_geo, const double* q_dev, int64_t C,
                             int32_t D, const double* limits_dev, const lsdf_env_grid* env, const int32_t W[3],
                             double* R_all_dev, double* T_all_dev, double* R_geo_dev, double* dt_geo_dev,
                             int32_t* anchor_geo_dev, int32_t* flags_dev, void* stream) {
    if (n_links < 1 || n_links > LSDF_MAX_LINKS || D > 32 || n_geo > LSDF_MAX_LINKS)
        return fail(LSDF_ERR_VALIDATION, "lsdf_fk_align: %d links / %d dof outside supported range", n_links, D);
    if (C <= 0) return LSDF_OK;
    FkParams p{};
    for (int i = 0; i < n_links; ++i) p.links[i] = links[i];
    p.n_links = n_links;
    p.n_geo = n_geo;
    p.D = D;
    p.C = C;
    p.q = q_dev;
    p.limits = limits_dev;
    if (env) p.env = *env;
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
    fk_align_kernel<<<grid_for(C, FK_WARPS), 32 * FK_WARPS, 0, (cudaStream_t)stream>>>(p);
    return check_launch("fk_align_kernel");
}

extern "C" int lsdf_align(const double* T_dev, int64_t n, const lsdf_env_grid* env, const int32_t W[3],
                          int32_t* anchor_dev, double* dt_dev, int32_t* flags_dev, void* stream) {
    if (n <= 0) return LSDF_OK;
    align_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(T_dev, n, *env, W[0], W[1], W[2], anchor_dev,
                                                                       dt_dev, flags_dev);
    return check_launch("align_kernel");
}

extern "C" int64_t lsdf_occupancy_bytes(const lsdf_env_grid* env) {
    const int64_t V = n_vox(*env);
    const int64_t words = (V + 31) / 32;
    return 64 + ((words * 4 + 255) / 256) * 256 + V * 4;
}

extern "C" int lsdf_voxelize(const void* points_dev, int32_t points_f32, int64_t N, const lsdf_env_grid* env,
                             void* occupancy_dev, int32_t* indices_dev, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    Occupancy o = carve(occupancy_dev, *env);
    LSDF_TRY(check_cuda(cudaMemsetAsync(occupancy_dev, 0, 64 + o.n_words * 4, s), "voxelize memset"));
    if (N > 0) {
        if (points_f32)
            voxel_scatter_kernel<float><<<grid_for(N, 256), 256, 0, s>>>((const float*)points_dev, N, *env,
                                                                           o.bitmap, o.counters);
        else
            voxel_scatter_kernel<double><<<grid_for(N, 256), 256, 0, s>>>((const double*)points_dev, N, *env,
                                                                            o.bitmap, o.counters);
        LSDF_TRY(check_launch("voxel_scatter_kernel"));
    }
    voxel_compact_kernel<<<1, COMPACT_THREADS, 0, s>>>(o.bitmap, o.n_words, *env, o.posgrid, indices_dev,
                                                        o.counters);
    return check_launch("voxel_compact_kernel");
}

extern "C" int lsdf_occupancy_from_indices(const int32_t* indices_dev, int64_t N, int32_t sorted_unique,
                                           const lsdf_env_grid* env, void* occupancy_dev, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    Occupancy o = carve(occupancy_dev, *env);
    LSDF_TRY(check_cuda(cudaMemsetAsync(occupancy_dev, 0, 64 + o.n_words * 4, s), "occupancy memset"));
    if (N <= 0) return LSDF_OK;
    if (sorted_unique) {
        occ_from_indices_kernel<<<grid_for(N, 256), 256, 0, s>>>(indices_dev, N, *env, o.bitmap, o.posgrid, 0);
        return check_launch("occ_from_indices_kernel");
    }
    occ_from_indices_kernel<<<grid_for(N, 256), 256, 0, s>>>(indices_dev, N, *env, o.bitmap, o.posgrid, 1);
    LSDF_TRY(check_launch("occ_from_indices_kernel"));
    occ_from_indices_kernel<<<grid_for(N, 256), 256, 0, s>>>(indices_dev, N, *env, o.bitmap, o.posgrid, 2);
    return check_launch("occ_from_indices_kernel");
}

extern "C" int lsdf_query_direct(const double* R_geo_dev, const double* dt_geo_dev, const int32_t* anchor_geo_dev,
                                 int64_t C, int32_t n_geo, const lsdf_link_grid* grids, const lsdf_window* window,
                                 const lsdf_env_grid* env, const void* occupancy_dev, int32_t by_position,
                                 double d_far_global, float* d_dev, int32_t* link_dev, int32_t* voxel_dev,
                                 float* per_link_dev, void* stream) {
    if (n_geo < 1 || n_geo > 32) return fail(LSDF_ERR_VALIDATION, "query: %d geometry links (1..32)", n_geo);
    if (window->W[0] > LSDF_MAX_WINDOW || window->W[1] > LSDF_MAX_WINDOW || window->W[2] > LSDF_MAX_WINDOW)
        return fail(LSDF_ERR_UNSUPPORTED, "query: window wider than %d cells", LSDF_MAX_WINDOW);
    const int64_t V = n_vox(*env);
    if ((double)V * n_geo >= 4294967295.0)
        return fail(LSDF_ERR_UNSUPPORTED, "query: %lld voxels x %d links overflow the 32-bit key", (long long)V, n_geo);
    if (C <= 0) return LSDF_OK;
    QueryParams p{};
    const float clamp = (float)d_far_global;
    int full = 0;
    for (int l = 0; l < n_geo; ++l) {
        p.grids[l] = grids[l];
        if (grids[l].d_far < clamp) full = 1;  // masked cells can undercut the clamp
    }
    if (window->zrange_dev == nullptr) full = 1;
    p.R = R_geo_dev;
    p.dt = dt_geo_dev;
    p.anchor = anchor_geo_dev;
    p.C = C;
    p.n_geo = n_geo;
    // enough warps in flight for small batches, one warp per link for big ones
    int split = (int)((148LL * 48 + C * n_geo - 1) / (C * n_geo));
    split = split < 1 ? 1 : split;
    split = split > 32 / n_geo ? 32 / n_geo : split;
    split = split > 8 ? 8 : split;
    p.split = split;
    for (int a = 0; a < 3; ++a) {
        p.W[a] = window->W[a];
        p.dims[a] = env->dims[a];
    }
    p.full_window = full;
    p.e_r = window->e_r;
    p.P = window->P_dev;
    p.Wmax = window->Wmax;
    p.by_position = by_position;
    p.zrange = window->zrange_dev;
    p.mask_bits = window->mask_bits_dev;
    p.clamp = clamp;
    Occupancy o = carve(const_cast<void*>(occupancy_dev), *env);
    p.bitmap = o.bitmap;
    p.posgrid = o.posgrid;
    p.d_out = d_dev;
    p.link_out = link_dev;
    p.voxel_out = voxel_dev;
    p.per_link = per_link_dev;
    const int threads = 32 * n_geo * split;
    const size_t smem = (size_t)(threads / 32) * QCAP * sizeof(uint32_t);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(query_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    query_direct_kernel<<<(unsigned)C, threads, smem, (cudaStream_t)stream>>>(p);
    return check_launch("query_direct_kernel");
}

extern "C" int lsdf_place_windows(const double* R_geo_dev, const double* dt_geo_dev, int64_t C, int32_t n_geo,
                                  const lsdf_link_grid* grids, const lsdf_window* window, float* windows_dev,
                                  void* stream) {
    if (n_geo < 1 || n_geo > LSDF_MAX_LINKS) return fail(LSDF_ERR_VALIDATION, "place: bad link count %d", n_geo);
    if (C <= 0) return LSDF_OK;
    PlaceParams p{};
    for (int l = 0; l < n_geo; ++l) p.grids[l] = grids[l];
    p.R = R_geo_dev;
    p.dt = dt_geo_dev;
    p.n_geo = n_geo;
    for (int a = 0; a < 3; ++a) p.W[a] = window->W[a];
    p.e_r = window->e_r;
    p.P = window->P_dev;
    p.Wmax = window->Wmax;
    p.mask_bits = window->mask_bits_dev;
    p.out = windows_dev;
    place_windows_kernel<<<(unsigned)(C * n_geo), 256, 0, (cudaStream_t)stream>>>(p);
    return check_launch("place_windows_kernel");
}

extern "C" int lsdf_assemble(const float* windows_dev, const int32_t* anchors_dev, const int32_t* config_dev,
                             int64_t n_fields, const int32_t W[3], const lsdf_env_grid* env, int64_t C,
                             double d_far_global, float* values_dev, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t total = C * n_vox(*env);
    if (total > 0) {
        fill_kernel<<<148 * 8, 256, 0, s>>>(values_dev, total, (float)d_far_global);
        LSDF_TRY(check_launch("fill_kernel"));
    }
    if (n_fields <= 0) return LSDF_OK;
    assemble_kernel<<<(unsigned)n_fields, 256, 0, s>>>(windows_dev, anchors_dev, config_dev, W[0], W[1], W[2], *env,
                                                        values_dev);
    return check_launch("assemble_kernel");
}

extern "C" int lsdf_query_dense(const float* values_dev, int64_t C, const lsdf_env_grid* env,
                                const int32_t* indices_dev, int64_t N, float* d_dev, int32_t* argmin_dev,
                                void* stream) {
    if (C <= 0 || N <= 0) return LSDF_OK;
    query_dense_kernel<<<(unsigned)C, 256, 0, (cudaStream_t)stream>>>(values_dev, n_vox(*env), *env, indices_dev, N,
                                                                       d_dev, argmin_dev);
    return check_launch("query_dense_kernel");
}

extern "C" int lsdf_trilinear(const lsdf_link_grid* grid, const double* pts_dev, int64_t n, double scale,
                              float* out_dev, void* stream) {
    if (n <= 0) return LSDF_OK;
    trilinear_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(*grid, pts_dev, n, scale, out_dev);
    return check_launch("trilinear_kernel");
}

extern "C" int lsdf_grid_transform_exact(const double* R_dev, const double* dt_dev, int64_t B,
                                         const double* points_dev, int64_t V, double e_r, double* G_dev,
                                         void* stream) {
    if (B * V <= 0) return LSDF_OK;
    transform_exact_kernel<<<grid_for(B * V, 256), 256, 0, (cudaStream_t)stream>>>(R_dev, dt_dev, B, points_dev, V,
                                                                                   e_r, G_dev);
    return check_launch("transform_exact_kernel");
}

extern "C" int lsdf_voxel_index(const double* points_dev, int64_t N, const lsdf_env_grid* env, int32_t* indices_dev,
                                int32_t* flags_dev, void* stream) {
    if (N <= 0) return LSDF_OK;
    voxel_index_kernel<<<grid_for(N, 256), 256, 0, (cudaStream_t)stream>>>(points_dev, N, *env, indices_dev,
                                                                           flags_dev);
    return check_launch("voxel_index_kernel");
}

extern "C" int lsdf_fill(float* dst_dev, int64_t n, float value, void* stream) {
    if (n <= 0) return LSDF_OK;
    const int64_t blocks = (n + 255) / 256;
    fill_kernel<<<(unsigned)(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, (cudaStream_t)stream>>>(dst_dev, n, value);
    return check_launch("fill_kernel");
}

extern "C" int lsdf_per_link_fields(const float* windows_dev, const int32_t* anchors_dev, const int32_t* configs_dev,
                                    const int32_t* links_dev, const float* d_far_dev, int64_t n_fields,
                                    const int32_t W[3], int32_t n_links, const lsdf_env_grid* env,
                                    const void* occupancy_dev, float* out_dev, void* stream) {
    if (n_fields <= 0) return LSDF_OK;
    Occupancy o = carve(const_cast<void*>(occupancy_dev), *env);
    per_link_fields_kernel<<<(unsigned)n_fields, 256, 0, (cudaStream_t)stream>>>(
        windows_dev, anchors_dev, configs_dev, links_dev, d_far_dev, W[0], W[1], W[2], n_links, *env, o.bitmap,
        out_dev);
    return check_launch("per_link_fields_kernel");
}

extern "C" int lsdf_sphere_baseline(const double* R_all_dev, const double* T_all_dev, int64_t C, int32_t L,
                                    const int32_t* sphere_link_dev, const double* sphere_center_dev,
                                    const double* sphere_radius_dev, int32_t S, const int32_t* indices_dev, int64_t N,
                                    const lsdf_env_grid* env, double* out_dev, void* stream) {
    if (C <= 0) return LSDF_OK;
    if (S <= 0 || S > 4096) return fail(LSDF_ERR_VALIDATION, "sphere model with %d spheres", S);
    sphere_baseline_kernel<<<(unsigned)C, 256, (size_t)S * 4 * sizeof(double), (cudaStream_t)stream>>>(
        R_all_dev, T_all_dev, L, sphere_link_dev, sphere_center_dev, sphere_radius_dev, S, indices_dev, N, *env,
        out_dev);
    return check_launch("sphere_baseline_kernel");
}
