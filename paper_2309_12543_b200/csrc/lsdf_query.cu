// lsdf_query.cu — stages 3 + 4: the fused direct query (the hot kernel).
//
// For configuration c the reference assembles a dense robot SDF (min over
// links of each link's resampled window, clamped at d_far_global;
// placement.py:267-313, query.py:61-103) and gathers it at the occupied
// voxels (query.py:128-150).  Only the occupied voxels inside a link's
// sphere-masked window can differ from the clamp, so the query evaluates
// exactly those, recomputing for every occupied cell the reference's
// resampled value
//   g = P R + dt_inv (fp64, placement.py:164-167), point = g * e_r,
//   trilinear_sample(sdf_l, point) (grids.py:155-191),
// bit-identical to the assembled field.  Keys (value, rank, link) reduce with
// a warp shuffle and one 64-bit atomic per task into a per-configuration
// slot; finalize_kernel turns the slots into (d, link, voxel) and re-zeroes
// them (graph replays need no memset).
//
// query_shells_kernel (the hot path): one warp = one task (link l,
// configuration c, slice s), persistent CTAs with dynamic task fetch; the
// window's kept cells are visited in order of distance from the window
// centre and the scan stops as soon as no remaining cell can reach the
// running minimum (core radius of the link grid), optionally gated per cell
// by the link's segment bound.
// query_direct_kernel (fallback when a link's far value is below the clamp or
// the mask has no column intervals): walks the window's (x, y) columns over
// the kept z-interval of each, with `split` column slices per (c, l).
#include <cstddef>
#include <cstdlib>

#include "lsdf_async.cuh"
#include "lsdf_device.cuh"

using namespace lsdf;

namespace {

struct QueryParams {
    GridGeom geom;                          // shared by the links of this launch
    const float4* cells[LSDF_MAX_LINKS];    // packed-corner grid per link
    float dfar[LSDF_MAX_LINKS];             // float32 link sentinel per link
    float core[LSDF_MAX_LINKS];             // value(p) >= |p| - core  (lsdf_link_grid.core_radius)
    float4 seg_a[LSDF_MAX_LINKS];           // segment bound: (a.xyz, kappa_lo); kappa_lo < 0 disables it
    double hull;                            // ball around the link origin inside the grid's cell-centre hull
    float4 seg_u[LSDF_MAX_LINKS];           // (u.xyz, length)
    float seg_hi[LSDF_MAX_LINKS];           // kappa_hi
    int32_t seg_filter;                     // apply the segment bound (throughput-sized batches)
    int32_t round_min;                      // queued cells that trigger a lookup round (<= 32)
    const uint32_t* bricks;                 // occupancy brick columns (4^3 voxels), or null: no box test
    int32_t stage_bricks;                   // brick columns copied to shared memory (else read from global)
    int32_t dilate;                         // > 0: empty-neighbourhood test at setup, dilation radius in bricks
    int32_t pair_scan;                      // throughput scan walks two tasks per chunk loop (shell_task_pair)
    int32_t skip_empty;                     // paired scan skips chunks without occupied cells: 0 never, 1 sparse clouds, 2 always
    int32_t dual;                           // latency batches: one task per (c, l) walking two chunks per step
    const uint32_t* brick_cols;             // the occupancy brick columns (input of the dilation)
    int32_t nbx_brick, nbz_brick;           // brick grid (x columns, z bits)
    int32_t nby_brick;                      // brick columns per x row
    const uint32_t* shell_cells;            // kept window cells sorted by distance from the centre
    const float* shell_radius;              // their distance (m), rounded down
    int32_t n_shell;
    int32_t group[LSDF_MAX_LINKS];          // links handled by this launch
    const double* R;
    const double* dt;
    const int32_t* anchor;
    int64_t C;
    int64_t n_tasks;
    int32_t n_geo, split;
    int32_t split_log2;          // split is a power of two on the shell path
    uint32_t pl_mul;             // t / (C * split) as a multiply-high (Granlund-Montgomery), see fast_div
    int32_t pl_shift;
    int32_t static_sched;        // latency batches: warp w takes tasks w, w + W, ... (no task counter)
    int32_t W[3];
    int32_t full_window;  // iterate the whole window, masking per cell (d_far_l < clamp)
    double e_r, e_rinv;  // window extent and RN(1 / e_r)
    const double* P;
    int32_t Wmax, by_position;
    int64_t pose_cs, pose_ls;  // pose record of (c, l) at c * pose_cs + l * pose_ls (config- or link-major)
    const int16_t* zrange;
    const uint32_t* mask_bits;
    int32_t dims[3];
    float clamp;
    const uint32_t* bitmap;
    const int32_t* prefix;
    const int32_t* posgrid;
    uint32_t* counters;          // [LSDF_MAX_LINKS] shell-scan work counters (zero between launches)
    unsigned long long* keys;    // C: ~best key (atomicMax of the complement, zero = empty)
    uint32_t* perlink;           // C x n_geo: ~orderable(min value)
    uint32_t* link_hist;         // [LSDF_MAX_LINKS] argmin-link counts of the previous cycle (link order)
    uint32_t* exit_count;        // CTAs of the shell scan that have finished (last one resets link_hist)
    int32_t track_order;         // finalize accumulates link_hist (the shell scan consumes and resets it)
    float* d_out;
    int32_t* link_out;
    int32_t* voxel_out;
    float* per_link;
};

constexpr int WARPS = 8;
constexpr int QCAP = 32 * 16 + 32;  // queue entries per warp: <= 16 bits per lane per round

// Returns the argmin link (-1 when clamped).
__device__ __forceinline__ int finalize(const QueryParams& p, int64_t c) {
    const uint64_t k = ~(uint64_t)p.keys[c];
    p.keys[c] = 0ull;  // leave the workspace zeroed for the next launch
    if (p.per_link != nullptr) {
        for (int l = 0; l < p.n_geo; ++l) {
            const uint32_t u = ~p.perlink[c * p.n_geo + l];
            p.perlink[c * p.n_geo + l] = 0u;
            const float v = from_orderable(u);
            p.per_link[c * p.n_geo + l] = fminf(p.clamp, fminf(p.dfar[l], v));  // query.py:171-175
        }
    }
    const uint32_t hi = (uint32_t)(k >> 32);
    if (k == ~0ull || hi >= orderable(p.clamp)) {  // nothing below the monitored range
        p.d_out[c] = p.clamp;
        p.link_out[c] = -1;
        p.voxel_out[c] = -1;
        return -1;
    }
    const uint32_t lo = (uint32_t)k;
    const uint32_t pos = lo / (uint32_t)p.n_geo;
    const int link = (int)(lo % (uint32_t)p.n_geo);
    p.d_out[c] = from_orderable(hi);
    p.link_out[c] = link;
    if (p.by_position) {
        p.voxel_out[c] = (int32_t)pos;
    } else {  // rank of the winning voxel in np.unique order
        const uint32_t w = pos >> 5, b = pos & 31;
        const uint32_t below = b ? (p.bitmap[w] & ((1u << b) - 1u)) : 0u;
        p.voxel_out[c] = p.prefix[w] + __popc(below);
    }
    return link;
}

template <bool FULL, bool BY_POS>
__global__ void __launch_bounds__(32 * WARPS) query_direct_kernel(const __grid_constant__ QueryParams p,
                                                                  int64_t blocks_per_link) {
    extern __shared__ double s_dyn[];
    double* sP = s_dyn;                                       // 3 x Wmax window offsets
    uint32_t* s_queue = (uint32_t*)(s_dyn + 3 * p.Wmax);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 3 * p.Wmax; i += blockDim.x) sP[i] = p.P[i];
    __syncthreads();
    // the link is uniform over the block
    const int l = p.group[blockIdx.x / blocks_per_link];
    const int64_t t_in_link = (blockIdx.x % blocks_per_link) * WARPS + warp;
    const int64_t c = t_in_link / p.split;
    if (c >= p.C) return;
    const int sidx = (int)(t_in_link % p.split);
    uint32_t* queue = s_queue + warp * QCAP;
    const float4* __restrict__ cells = p.cells[l];
    const float far = p.dfar[l];
    const int64_t o = c * p.n_geo + l;                  // per-link slot
    const int64_t po = c * p.pose_cs + l * p.pose_ls;   // pose record
    double R[9], dtinv[3];
#pragma unroll
    for (int e = 0; e < 9; ++e) R[e] = __ldg(p.R + po * 9 + e);
    shift_inverse(R, p.dt + po * 3, p.e_r, dtinv);
    const int ax = __ldg(p.anchor + po * 3), ay = __ldg(p.anchor + po * 3 + 1), az = __ldg(p.anchor + po * 3 + 2);
    const int W0 = p.W[0], W1 = p.W[1], W2 = p.W[2];
    const int ny = p.dims[1], nz = p.dims[2];
    const int n_cols = W0 * W1;
    const int Wm = p.Wmax;
    // C-order voxel index of window cell (0, 0, 0); cell (mx, my, mz) adds (mx*ny + my)*nz + mz
    const int lin0 = (ax * ny + ay) * nz + az;

    float bestv = INFINITY;
    uint32_t bestpos = 0xffffffffu;
    int qlen = 0;
    auto consider = [&](uint32_t cell) {
        const int mx = cell & 0xff, my = (cell >> 8) & 0xff, mz = cell >> 16;
        float v = far;
        bool keep = true;
        if (FULL) {
            const int bit = mx + W0 * (my + W1 * mz);
            keep = (__ldg(p.mask_bits + (bit >> 5)) >> (bit & 31)) & 1u;
        }
        if (keep) {
            double pt[3];
            window_point(sP[mx], sP[Wm + my], sP[2 * Wm + mz], R, dtinv, p.e_r, pt);
            v = trilinear_geom(p.geom, cells, far, pt[0], pt[1], pt[2]);
        }
        const int lin = lin0 + (mx * ny + my) * nz + mz;
        const uint32_t pos = BY_POS ? (uint32_t)__ldg(p.posgrid + lin) : (uint32_t)lin;
        const bool better = (v < bestv) | ((v == bestv) & (pos < bestpos));
        bestv = better ? v : bestv;
        bestpos = better ? pos : bestpos;
    };

    for (int base = sidx * 32; base < n_cols; base += 32 * p.split) {
        const int col = base + lane;
        const int my = col / W0, mx = col - my * W0;
        int zcur = 0, zend = 0;
        int bitbase = 0;
        if (col < n_cols) {
            const int x = ax + mx, y = ay + my;
            if (x >= 0 && x < p.dims[0] && y >= 0 && y < ny) {
                int zlo = 0, zhi = W2;
                if (!FULL) {
                    const uint32_t zr = __ldg((const uint32_t*)p.zrange + col);
                    zlo = (int)(zr & 0xffff);
                    zhi = (int)(zr >> 16);
                }
                zcur = max(az + zlo, 0);
                zend = min(az + zhi, nz);
                bitbase = (x * ny + y) * nz;
            }
        }
        // consume each column's z-run in segments of <= 16 bits, all lanes in step
        while (__any_sync(FULL_MASK, zcur < zend)) {
            uint32_t bits = 0;
            const int zs = zcur - az;
            if (zcur < zend) {
                const int bp = bitbase + zcur;
                const int off = bp & 31;
                const int n = min(min(zend - zcur, 16), 32 - off);
                bits = (__ldg(p.bitmap + (bp >> 5)) >> off) & ((1u << n) - 1u);
                zcur += n;
            }
            const int cnt = __popc(bits);
            int incl = cnt;
#pragma unroll
            for (int o2 = 1; o2 < 32; o2 <<= 1) {
                const int v = __shfl_up_sync(FULL_MASK, incl, o2);
                if (lane >= o2) incl += v;
            }
            const int total = __shfl_sync(FULL_MASK, incl, 31);
            int slot = qlen + incl - cnt;
            const uint32_t colkey = (uint32_t)mx | ((uint32_t)my << 8);
            while (bits) {
                const int b = __ffs(bits) - 1;
                bits &= bits - 1;
                queue[slot++] = colkey | ((uint32_t)(zs + b) << 16);
            }
            qlen += total;
            __syncwarp();
            while (qlen >= 32) {
                consider(queue[qlen - 32 + lane]);
                qlen -= 32;
            }
            __syncwarp();
        }
    }
    if (lane < qlen) consider(queue[lane]);

    const uint32_t pos_key = bestpos == 0xffffffffu ? 0xffffffffu : bestpos * (uint32_t)p.n_geo + (uint32_t)l;
    uint64_t best = bestpos == 0xffffffffu ? ~0ull : (((uint64_t)orderable(bestv) << 32) | pos_key);
    best = warp_min_u64(best);
    const float wmin = warp_min_f(bestv);
    if (lane == 0) {
        atomicMax(p.keys + c, (unsigned long long)~best);
        if (p.per_link != nullptr) atomicMax(p.perlink + o, ~orderable(wmin));
    }
}

// ---------------------------------------------------------------- shell order
// The kept window cells are visited in order of increasing distance rho from
// the window centre (the link origin T up to the residual dt).  Every sample
// of link l at a cell obeys value >= rho - |dt| - core_l (core_radius, derived
// from the grid values), so once the next chunk's rho - |dt| - core_l exceeds
// the best value any lane of the warp has found (or, when per-link minima are
// not requested, the configuration's best over all links so far, read from
// the key slot), no remaining cell can reach or tie the minimum and the scan
// stops.  Occupied cells are compacted with a ballot and evaluated 32 at a
// time with the exact fp64 recipe, so the results are those of the full scan.
#ifndef LSDF_PAIR_N
#define LSDF_PAIR_N 2
#endif
#ifndef LSDF_DUAL_CHUNKS
#define LSDF_DUAL_CHUNKS 2
#endif
constexpr int DUAL_CHUNKS = LSDF_DUAL_CHUNKS;  // chunks per step of shell_task_dual (latency batches)
// > round_min - 1 + 32 PAIR_N (a chunk of the paired scan queues up to 32
// PAIR_N entries) and > 15 + 32 DUAL_CHUNKS (a step of the latency walk)
constexpr int QCAP_SHELL = 32 + 32 * (LSDF_PAIR_N > LSDF_DUAL_CHUNKS ? LSDF_PAIR_N : LSDF_DUAL_CHUNKS);
__host__ __device__ __forceinline__ int shell_padded(int n) { return (n + 31) & ~31; }
constexpr int SHELL_STAGE_MAX = 4096;   // kept cells staged in shared memory (W <= 20)
constexpr int BITMAP_STAGE_MAX = 8192;  // occupancy words staged in shared memory (<= 262k voxels)
constexpr int BRICK_STAGE_MAX = 4096;   // brick columns staged in shared memory (16 KB: x, y <= 256 voxels)

__device__ __forceinline__ void* align16_ptr(void* q) {
    return (void*)(((uintptr_t)q + 15) & ~(uintptr_t)15);
}
struct ShellView {
    const uint32_t* cells;   // shell-ordered kept cells (shared or global)
    const float* radius;
    const uint32_t* bits;    // occupancy bitmap (shared or global)
    const uint32_t* bricks;  // brick columns (shared), or null
    const double* P;         // window offsets (shared)
    uint32_t cells_s, radius_s, bits_s;  // shared-window addresses of the staged tables
    uint32_t P_s;                        // shared-window address of P
};

// MUFU.RSQ alone (rsqrtf adds a subnormal-input fix-up; callers pass normal values)
__device__ __forceinline__ float rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// the value of x, hidden from the optimizer (no rematerialization from its inputs)
__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
    asm volatile("mov.b32 %0, %0;" : "+r"(x));
    return x;
}
__device__ __forceinline__ int32_t lds_s32(uint32_t a) {
    int32_t v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int4 lds_i4(uint32_t a) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ double2 lds_d2(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// predicated store (no branch around it)
__device__ __forceinline__ void sts_u32_if(bool pred, uint32_t a, uint32_t v) {
    asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.shared.u32 [%0], %1;\n}" ::"r"(a), "r"(v),
                 "r"((uint32_t)pred)
                 : "memory");
}
// warp collectives of the scan's convergent loop as plain PTX
__device__ __forceinline__ uint32_t warp_redux_min(uint32_t v) {
    uint32_t r;
    asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}
__device__ __forceinline__ uint32_t warp_ballot(bool pred) {
    uint32_t r;
    asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n vote.sync.ballot.b32 %0, p, 0xffffffff;\n}"
                 : "=r"(r)
                 : "r"((uint32_t)pred));
    return r;
}

// Table reads of the scan: with STAGED, explicit ld.shared on the shared-window
// address (a generic load of a shared address costs the generic-to-shared
// resolution on every chunk's dependent chain); otherwise through the pointer.
template <bool STAGED>
__device__ __forceinline__ uint32_t sv_u32(const uint32_t* ptr, uint32_t saddr, int i) {
    if (!STAGED) return ptr[i];
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr + 4u * (uint32_t)i));
    return v;
}
template <bool STAGED>
__device__ __forceinline__ float sv_f32(const float* ptr, uint32_t saddr, int i) {
    if (!STAGED) return ptr[i];
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(saddr + 4u * (uint32_t)i));
    return v;
}

// Per-task constants, computed by one lane per task (up to GRAB_MAX tasks at a
// time) and read back from shared memory by the warp that scans the task.
#ifndef LSDF_GRAB_MAX
#define LSDF_GRAB_MAX 16
#endif
constexpr int GRAB_MAX = LSDF_GRAB_MAX;
constexpr int64_t SEG_FILTER_MIN_TASKS = 148LL * 32 * 8;  // ~8 tasks per resident warp
#ifndef LSDF_SHELL_MINB
#define LSDF_SHELL_MINB 3
#endif
struct __align__(16) ShellSetup {
    double R[9];
    double dtinv[3];
    // Segment bound in quadratic form (see seg_d2): with m' the cell index
    // relative to the window centre c, q = p - a = A m' + b (A = e_r s_a R,
    // rows orthogonal, |row a|^2 = sigma_a^2), |q|^2 = sum_a sigma_a^2 m'_a^2 +
    // m'.(2 A b) + |b|^2 and q.u = m'.(A u) + b.u
    float4 sw;   // (2 A b, |b|^2)
    float4 sv;   // (A u, b.u)
    // the paired scan's per-task state, read as two 16-B records:
    float thresh0;   // starting threshold: min(clamp, the configuration's best key at setup time)
    float slack;     // |dt| (rounded up) + core radius of the link
    float hull_lim;  // cells with shell radius <= hull_lim map inside the link grid's cell-centre hull
                     // (-inf: the segment bound is off)
    float k_lo;      // segment bound kappa_lo (+inf: off, every cell passes)
    int32_t ax, ay, az;
    int32_t lin0;    // C-order index of window cell (0, 0, 0)
    float k_hi;      // segment bound kappa_hi
    int32_t l;       // geometry link
    int32_t c;       // configuration
    int32_t sidx;    // slice of the shell list
};

static_assert(offsetof(ShellSetup, R) == 0 && offsetof(ShellSetup, dtinv) == 72 && sizeof(ShellSetup) % 16 == 0,
              "lookup_round reads R and dtinv at fixed offsets");
static_assert(offsetof(ShellSetup, thresh0) % 16 == 0 && offsetof(ShellSetup, ax) % 16 == 0 &&
                  offsetof(ShellSetup, k_lo) == offsetof(ShellSetup, thresh0) + 12 &&
                  offsetof(ShellSetup, lin0) == offsetof(ShellSetup, ax) + 12,
              "pair_task reads (thresh0, slack, hull_lim, k_lo) and (ax, ay, az, lin0) as 16-B records");

// Dilated brick occupancy (throughput batches): a (bx, by) column word whose
// bit bz is set when some occupied brick lies within `dilate` bricks of
// (bx, by, bz) in every axis.  A window [j - W/2, j + W/2) stays within
// (W/2 + 3) / 4 bricks of its centre brick j / 4, so a clear bit at the centre
// brick proves the window holds no occupied voxel.  Built per CTA in shared
// memory (separable: z by shifts, then y, then x); `tmp` is scratch.
constexpr int DILATE_MAX_COLS = 1024;  // 2 x 4 KB of shared memory (x, y <= 128 voxels)
__device__ void build_dilated(const QueryParams& p, uint32_t* dil, uint32_t* tmp) {
    const int nbx = p.nbx_brick, nby = p.nby_brick, r = p.dilate, n = nbx * nby;
    const uint32_t zmask = p.nbz_brick >= 32 ? 0xffffffffu : ((1u << p.nbz_brick) - 1u);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t w = __ldg(p.brick_cols + i);
        uint32_t d = w;
        for (int k = 1; k <= r; ++k) d |= (w << k) | (w >> k);
        dil[i] = d & zmask;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int bx = i / nby, by = i - bx * nby;
        uint32_t d = 0;
        for (int y = max(by - r, 0); y <= min(by + r, nby - 1); ++y) d |= dil[bx * nby + y];
        tmp[i] = d;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int bx = i / nby, by = i - bx * nby;
        uint32_t d = 0;
        for (int x = max(bx - r, 0); x <= min(bx + r, nbx - 1); ++x) d |= tmp[x * nby + by];
        dil[i] = d;
    }
    __syncthreads();
}

// n / d for 32-bit n and a launch-constant d: q = (hi + ((n - hi) >> 1)) >> (sh - 1),
// hi = umulhi(m, n), m = floor(2^32 (2^sh - d) / d) + 1, sh = ceil(log2 d) (d > 1);
// d == 1 is encoded as sh == 0.
__device__ __forceinline__ uint32_t fast_div(uint32_t n, uint32_t m, int sh) {
    if (sh == 0) return n;
    const uint32_t hi = __umulhi(m, n);
    return (hi + ((n - hi) >> 1)) >> (sh - 1);
}

__device__ __forceinline__ void shell_setup(const QueryParams& p, const int* order, uint32_t t, ShellSetup& s,
                                            const uint32_t* dil) {
    const uint32_t per_link = (uint32_t)(p.C * p.split);
    const uint32_t li = fast_div(t, p.pl_mul, p.pl_shift);  // rank of the task's link in the launch order
    const int l = order[li];
    const uint32_t r = t - li * per_link;
    const int64_t c = r >> p.split_log2;
    const int64_t o = c * p.pose_cs + l * p.pose_ls;  // pose record
    double R[9], dtinv[3], dt[3];
#pragma unroll
    for (int e = 0; e < 9; ++e) R[e] = __ldg(p.R + o * 9 + e);
#pragma unroll
    for (int e = 0; e < 3; ++e) dt[e] = __ldg(p.dt + o * 3 + e);
    shift_inverse(R, dt, p.e_r, dtinv, p.e_rinv);
    // |dt| rounded up (dt is the residual of T against its voxel centre): an
    // f32 square root rounded up of the fp64 square sum rounded up, plus margin
    const float dtn = __fsqrt_ru(__double2float_ru(dt[0] * dt[0] + dt[1] * dt[1] + dt[2] * dt[2])) * (1.0f + 1e-6f) +
                      1e-12f;
#pragma unroll
    for (int e = 0; e < 9; ++e) s.R[e] = R[e];
#pragma unroll
    for (int e = 0; e < 3; ++e) s.dtinv[e] = dtinv[e];
    // segment bound off unless set below: every cell passes, the threshold is never lowered by it
    s.sw = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    s.sv = s.sw;
    s.k_lo = INFINITY;
    s.hull_lim = -INFINITY;
    s.k_hi = 0.0f;
    if (p.seg_filter) {  // segment-bound constants (throughput batches only)
        const float4 sa = p.seg_a[l], su = p.seg_u[l];
        const double a3[3] = {sa.x, sa.y, sa.z}, u3[3] = {su.x, su.y, su.z};
        // the window offsets are affine in the cell index, P_a[m] = P_a[c] + (m - c) s_a
        // (c = W/2): fold them in, so the scan evaluates the bound straight from
        // the centred cell indices (no offset-table loads)
        const int Wm = p.Wmax;
        const int c0 = p.W[0] / 2, c1 = p.W[1] / 2, c2 = p.W[2] / 2;
        const double pc[3] = {__ldg(p.P + c0), __ldg(p.P + Wm + c1), __ldg(p.P + 2 * Wm + c2)};
        const double sc[3] = {__ldg(p.P + 1) - __ldg(p.P), __ldg(p.P + Wm + 1) - __ldg(p.P + Wm),
                              __ldg(p.P + 2 * Wm + 1) - __ldg(p.P + 2 * Wm)};
        double b[3], bb = 0.0, bu = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            b[k] = dtinv[k] * p.e_r - a3[k] + p.e_r * (R[k] * pc[0] + R[3 + k] * pc[1] + R[6 + k] * pc[2]);
            bb += b[k] * b[k];
            bu += b[k] * u3[k];
        }
        float w2[3], v[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double f = p.e_r * sc[a];
            w2[a] = (float)(2.0 * f * (R[3 * a] * b[0] + R[3 * a + 1] * b[1] + R[3 * a + 2] * b[2]));
            v[a] = (float)(f * (R[3 * a] * u3[0] + R[3 * a + 1] * u3[1] + R[3 * a + 2] * u3[2]));
        }
        s.sw = make_float4(w2[0], w2[1], w2[2], (float)bb);
        s.sv = make_float4(v[0], v[1], v[2], (float)bu);
        // |link-frame point| <= rho + |dt|: a cell with rho <= hull - |dt| samples
        // inside the hull of the grid's cell centres, where the segment's upper
        // bound holds (outside it the sample is the link's far value)
        s.hull_lim = (float)(p.hull - (double)dtn) * (1.0f - 0x1p-20f) - 1e-6f;
        const bool use_seg = sa.w >= 0.0f;  // (kappa_lo < 0: disabled for this link)
        s.k_lo = use_seg ? sa.w : INFINITY;
        if (!use_seg) s.hull_lim = -INFINITY;
        s.k_hi = p.seg_hi[l];
    }
    s.slack = dtn + p.core[l];
    float t0 = p.clamp;  // values >= clamp never change the answer
    if (p.per_link == nullptr) {  // best key any link of this configuration has published so far (an upper
        const uint64_t k = ~(uint64_t)__ldcg(p.keys + c);  // bound of the minimum, so an older read stays valid)
        if (k != ~0ull) t0 = fminf(t0, from_orderable((uint32_t)(k >> 32)));
    }
    s.thresh0 = t0;
    s.l = l;
    s.c = (int32_t)c;
    s.sidx = (int32_t)(r & (uint32_t)(p.split - 1));
    s.ax = __ldg(p.anchor + o * 3);
    s.ay = __ldg(p.anchor + o * 3 + 1);
    s.az = __ldg(p.anchor + o * 3 + 2);
    s.lin0 = (s.ax * p.dims[1] + s.ay) * p.dims[2] + s.az;
    if (dil != nullptr) {  // nothing occupied near the window: the task stops at its first chunk
        const unsigned bx = (unsigned)(s.ax + p.W[0] / 2) >> BRICK_LOG2, by = (unsigned)(s.ay + p.W[1] / 2) >> BRICK_LOG2;
        const unsigned bz = (unsigned)(s.az + p.W[2] / 2) >> BRICK_LOG2;
        // (a centre outside the grid -- negative coordinates wrap to large -- keeps the scan)
        if (bx < (unsigned)p.nbx_brick && by < (unsigned)p.nby_brick && bz < (unsigned)p.nbz_brick &&
            ((dil[bx * p.nby_brick + by] >> bz) & 1u) == 0u)
            s.thresh0 = -INFINITY;
    }
}

#ifdef LSDF_TIMING  // instrumented build (tools/scan_timing.py): globaltimer stamps per warp / grab / task
__device__ unsigned long long g_tim[16];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TIM(i, v) atomicAdd(g_tim + (i), (unsigned long long)(v))
#else
#define TIM(i, v) ((void)0)
#endif

#ifdef LSDF_STATS  // instrumented build (tools/scan_stats.py): per-task scan counters
__device__ unsigned long long g_stats[8];
#define STAT(i, v) (sc[i] += (v))
#else
#define STAT(i, v) ((void)0)
#endif

// One round of exact lookups over queue entries (cell | task slot << 24),
// one per lane: each lane evaluates its entry with its task's constants
// (shared memory), the entries of one task reduce together (match-any
// groups: min value, then min position) into the configuration's key slot
// and, when requested, the per-link slot.  Entries of several tasks of the
// warp's grab can share a round, so a task's leftover lookups ride with the
// next task's instead of costing a partial round each.  Returns the
// orderable minimum over the entries of task slot `cur`.
// setups_s: the shared-window address of the warp's ShellSetup array (opaque,
// so its base is not rebuilt from the shared-memory window every round)
template <bool BY_POS>
__device__ __forceinline__ uint32_t lookup_round(const QueryParams& p, const ShellView& sv,
                                                 uint32_t setups_s, uint32_t entry, bool valid, uint32_t cur,
                                                 int lane, uint32_t* ov_out = nullptr) {
    const uint32_t slot = valid ? entry >> 24 : 0xffu;
    uint32_t ov = 0xffffffffu, pk = 0xffffffffu;
    int64_t c = 0;
    int l = 0;
    if (valid) {
        const uint32_t sa = setups_s + slot * (uint32_t)sizeof(ShellSetup);
        l = lds_s32(sa + (uint32_t)offsetof(ShellSetup, l));
        c = lds_s32(sa + (uint32_t)offsetof(ShellSetup, c));
        double R[9], dtinv[3];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const double2 r2 = lds_d2(sa + 16u * e);
            R[2 * e] = r2.x;
            R[2 * e + 1] = r2.y;
        }
        R[8] = lds_f64(sa + 64u);
        dtinv[0] = lds_f64(sa + 72u);
        const double2 d2 = lds_d2(sa + 80u);
        dtinv[1] = d2.x;
        dtinv[2] = d2.y;
        const int4 an = lds_i4(sa + (uint32_t)offsetof(ShellSetup, ax));
        const int Wm = p.Wmax, ny = p.dims[1], nz = p.dims[2];
        const int mx = entry & 0xff, my = (entry >> 8) & 0xff, mz = (entry >> 16) & 0xff;
        double pt[3];
        window_point(lds_f64(sv.P_s + 8u * mx), lds_f64(sv.P_s + 8u * (Wm + my)), lds_f64(sv.P_s + 8u * (2 * Wm + mz)),
                     R, dtinv, p.e_r, pt);
        const float v = trilinear_geom(p.geom, p.cells[l], p.dfar[l], pt[0], pt[1], pt[2]);
        const int lin = ((an.x + mx) * ny + (an.y + my)) * nz + (an.z + mz);
        const uint32_t pos = BY_POS ? (uint32_t)__ldg(p.posgrid + lin) : (uint32_t)lin;
        ov = orderable(v);
        pk = pos * (uint32_t)p.n_geo + (uint32_t)l;
    }
    const unsigned grp = __match_any_sync(FULL_MASK, slot);
    const uint32_t h = __reduce_min_sync(grp, ov);
    const uint32_t lo = __reduce_min_sync(grp, ov == h ? pk : 0xffffffffu);
    if (valid && lane == __ffs(grp) - 1) {
        atomicMax(p.keys + c, ~(((unsigned long long)h << 32) | lo));
        if (p.per_link != nullptr) atomicMax(p.perlink + c * p.n_geo + l, ~h);
    }
    if (ov_out != nullptr) {  // the caller reduces per slot itself
        *ov_out = ov;
        return 0xffffffffu;
    }
    return __reduce_min_sync(FULL_MASK, slot == cur ? ov : 0xffffffffu);
}

// Centred cell coordinates m' = m - W/2 of a shell cell and sum_a sigma_a^2 m'_a^2.
struct SegCell {
    float px, py, pz, mm;
};
struct SegAxes {  // per launch: the window centre and sigma_a^2 = (e_r s_a)^2
    float cx, cy, cz, s2x, s2y, s2z;
};
__device__ __forceinline__ SegAxes seg_axes(const QueryParams& p) {
    const int Wm = p.Wmax;
    SegAxes g;
    g.cx = (float)(p.W[0] / 2);
    g.cy = (float)(p.W[1] / 2);
    g.cz = (float)(p.W[2] / 2);
    const double fx = p.e_r * (__ldg(p.P + 1) - __ldg(p.P));
    const double fy = p.e_r * (__ldg(p.P + Wm + 1) - __ldg(p.P + Wm));
    const double fz = p.e_r * (__ldg(p.P + 2 * Wm + 1) - __ldg(p.P + 2 * Wm));
    g.s2x = (float)(fx * fx);
    g.s2y = (float)(fy * fy);
    g.s2z = (float)(fz * fz);
    return g;
}
__device__ __forceinline__ SegCell seg_cell(const SegAxes& g, unsigned mx, unsigned my, unsigned mz) {
    SegCell m;
    m.px = (float)mx - g.cx;
    m.py = (float)my - g.cy;
    m.pz = (float)mz - g.cz;
    m.mm = fmaf(m.px, m.px * g.s2x, fmaf(m.py, m.py * g.s2y, m.pz * m.pz * g.s2z));
    return m;
}
// Squared distance from the cell's link-frame point to the link's axis segment,
// f32: |q|^2 - s^2 + (s - t)^2 with s = q.u and t = clamp(s, 0, L).  The
// evaluation error stays below 2^-23 m^2 on the window's range (sampled with
// fma emulation in tests/test_host.py::test_segment_bound_quadratic_form);
// callers widen by SEG_D2_ERR on both sides.
constexpr float SEG_D2_ERR = 0x1p-21f;
__device__ __forceinline__ float seg_d2(const float4 sw, const float4 sv, const SegCell& m, float len) {
    const float qq = fmaf(m.pz, sw.z, fmaf(m.py, sw.y, fmaf(m.px, sw.x, m.mm + sw.w)));
    const float sp = fmaf(m.pz, sv.z, fmaf(m.py, sv.y, fmaf(m.px, sv.x, sv.w)));
    const float dd = sp - fminf(fmaxf(sp, 0.0f), len);
    return fmaxf(fmaf(dd, dd, fmaf(-sp, sp, qq)), 0.0f);
}

// Per-task scan state of the paired scan (shell_task_pair).  A disabled
// segment bound is encoded in the constants (k_lo = +inf passes every cell,
// hull_lim = -inf never lowers the threshold), so the chunk body is the same
// branch-free code for every task.
struct PairTask {
    float thresh, slack, hull_lim, k_lo, k_hi;
    int ax, ay, az, lin0;
    bool active;
};

__device__ __forceinline__ PairTask pair_task(uint32_t sa) {  // sa: shared address of the ShellSetup
    const float4 f = lds_f4(sa + (uint32_t)offsetof(ShellSetup, thresh0));
    const int4 a = lds_i4(sa + (uint32_t)offsetof(ShellSetup, ax));
    PairTask t;
    t.thresh = f.x;
    t.slack = f.y;
    t.hull_lim = f.z;
    t.k_lo = f.w;
    t.k_hi = __int_as_float(lds_s32(sa + (uint32_t)offsetof(ShellSetup, k_hi)));
    t.ax = a.x;
    t.ay = a.y;
    t.az = a.z;
    t.lin0 = a.w;
    t.active = true;
    return t;
}

// NT tasks of a grab (slots j .. j + NT - 1; split == 1, so all walk the
// same chunk sequence) scanned together: per chunk, the cell's indices, its
// float coordinates and its C-order offset in the environment grid are
// computed once for all tasks, and every task then runs the same
// branch-free occupancy test and segment bound (a stopped task's lanes are
// masked, not skipped: both tasks are live in ~96 % of the chunks at config 4).
// The tasks' chains are independent, so the warp has NT of them in flight.
// Each task stops at its own first chunk whose bound exceeds its own
// threshold, as in shell_task; queue entries carry their slot, so lookups and
// reductions are unchanged.
constexpr int PAIR_N = LSDF_PAIR_N;
constexpr int64_t SPARSE_FRACTION = 20;  // "sparse": under 5 % of the voxels occupied (config 4's crowd: 40 %)
// SKIP (sparse clouds, chosen per CTA from the occupied fraction): a chunk in
// which neither task has an occupied cell goes straight to the next chunk
// (no bound, no ballots).  Dense clouds almost never have such a chunk and do
// without the vote.
template <bool BY_POS, bool STAGED, bool SKIP>
__device__ __forceinline__ void shell_task_pair(const QueryParams& p, const ShellView& sv, uint32_t queue,
                                                uint32_t setups_s, uint32_t j, int& qlen, int lane,
                                                const SegAxes& ga) {
    // the tasks' setup records, read through the warp's opaque shared address
    // (not rebuilt from the shared-memory window for every access)
    const uint32_t st_s = setups_s + j * (uint32_t)sizeof(ShellSetup);
    PairTask t[PAIR_N];
#pragma unroll
    for (int i = 0; i < PAIR_N; ++i) t[i] = pair_task(st_s + (uint32_t)(i * sizeof(ShellSetup)));
    const float len = p.seg_u[lds_s32(st_s + (uint32_t)offsetof(ShellSetup, l))].w;  // the paired tasks share the link
    const bool share_cfg = p.per_link == nullptr;
    // grid dimensions in registers for the whole walk (not reloaded from the
    // constant bank every chunk)
    const unsigned nx = opaque_u32((unsigned)p.dims[0]), ny = opaque_u32((unsigned)p.dims[1]),
                   nz = opaque_u32((unsigned)p.dims[2]);
    const unsigned below = (1u << lane) - 1u;
    const int n_shell = (int)opaque_u32((uint32_t)p.n_shell), round_min = (int)opaque_u32((uint32_t)p.round_min);
    int rounds = 0;
    for (int k0 = 0; k0 < n_shell; k0 += 32) {
        const float rad = sv_f32<STAGED>(sv.radius, sv.radius_s, k0);
        bool any = false;
#pragma unroll
        for (int i = 0; i < PAIR_N; ++i) {
            t[i].active = t[i].active && !(rad - t[i].slack > t[i].thresh);  // every later cell is farther
            any |= t[i].active;
        }
        if (!any) break;
        const uint32_t cell = sv_u32<STAGED>(sv.cells, sv.cells_s, k0 + lane);
        const float rad_hi = sv_f32<STAGED>(sv.radius, sv.radius_s, k0 + 31);  // the chunk's largest radius
        const unsigned mx = cell & 0xff, my = (cell >> 8) & 0xff, mz = cell >> 16;
        const int off = (int)((mx * ny + my) * nz + mz);  // C-order offset from the window's corner voxel
        const SegCell sc = seg_cell(ga, mx, my, mz);
        bool o[PAIR_N];
        bool any_occ = false;
#pragma unroll
        for (int i = 0; i < PAIR_N; ++i) {
            const bool inb = ((unsigned)t[i].ax + mx < nx) & ((unsigned)t[i].ay + my < ny) & ((unsigned)t[i].az + mz < nz);
            const int lin = inb ? t[i].lin0 + off : 0;  // cells outside the grid read word 0, masked below
            o[i] = t[i].active & inb & ((sv_u32<STAGED>(sv.bits, sv.bits_s, lin >> 5) >> (lin & 31)) & 1u);
            any_occ |= o[i];
        }
        if (SKIP && warp_ballot(any_occ) == 0u) continue;
        uint32_t mins[PAIR_N];
#pragma unroll
        for (int i = 0; i < PAIR_N; ++i) {
            bool occ = o[i];
            // segment bound (f32, conservative): d(p) - k_lo <= value(p) <= d(p) + k_hi
            const uint32_t sa = st_s + (uint32_t)(i * sizeof(ShellSetup));
            const float d2 = seg_d2(lds_f4(sa + (uint32_t)offsetof(ShellSetup, sw)),
                                    lds_f4(sa + (uint32_t)offsetof(ShellSetup, sv)), sc, len);
            // (lim < 0: only cells with d2 <= SEG_D2_ERR pass -- extra lookups, never a missed cell)
            const float lim = fmaxf(t[i].thresh + t[i].k_lo, 0.0f);
            occ = occ & (d2 <= fmaf(lim, lim, SEG_D2_ERR));
            o[i] = occ;
            mins[i] = warp_redux_min(occ ? __float_as_uint(d2) : 0x7f800000u);
        }
        // a queued cell WILL be looked up, so its upper bound lowers the
        // threshold at once -- only inside the hull of the grid's cell
        // centres, where the upper bound holds (one branch for the tasks)
        bool upd[PAIR_N], any_upd = false;
#pragma unroll
        for (int i = 0; i < PAIR_N; ++i) {
            upd[i] = (mins[i] < 0x7f800000u) & (rad_hi <= t[i].hull_lim);
            any_upd |= upd[i];
        }
        if (any_upd) {
#pragma unroll
            for (int i = 0; i < PAIR_N; ++i) {
                const float dm = __uint_as_float(mins[i]) + SEG_D2_ERR;  // (>= 2^-21: never subnormal)
                const float r = dm * rsqrt_approx(dm);  // ~2^-22 relative: rounded up below
                if (upd[i]) t[i].thresh = fminf(t[i].thresh, fmaf(r, 1.0f + 0x1p-18f, t[i].k_hi));
            }
        }
#pragma unroll
        for (int i = 0; i < PAIR_N; ++i) {
            const unsigned bl = warp_ballot(o[i]);
            sts_u32_if(o[i], queue + 4u * (uint32_t)(qlen + __popc(bl & below)), cell | ((j + i) << 24));
            qlen += __popc(bl);
        }
        __syncwarp();
        while (qlen >= round_min) {  // (NT tasks can queue up to 32 NT entries in one chunk)
            const int n = qlen < 32 ? qlen : 32;
            const uint32_t entry = lane < n ? lds_u32(queue + 4u * (uint32_t)(qlen - n + lane)) : 0u;
            uint32_t ov;
            lookup_round<BY_POS>(p, sv, setups_s, entry, lane < n, j, lane, &ov);
            const uint32_t slot = entry >> 24;  // (ov is 0xffffffff on lanes without an entry)
#pragma unroll
            for (int i = 0; i < PAIR_N; ++i) {
                const uint32_t m = __reduce_min_sync(FULL_MASK, slot == j + i ? ov : 0xffffffffu);
                if (m != 0xffffffffu) t[i].thresh = fminf(t[i].thresh, from_orderable(m));
            }
            if (share_cfg && (++rounds & 3) == 0) {
#pragma unroll
                for (int i = 0; i < PAIR_N; ++i) {
                    const int32_t ci = lds_s32(st_s + (uint32_t)(i * sizeof(ShellSetup) + offsetof(ShellSetup, c)));
                    const uint64_t k = ~(uint64_t)__ldcg(p.keys + ci);
                    if (k != ~0ull) t[i].thresh = fminf(t[i].thresh, from_orderable((uint32_t)(k >> 32)));
                }
            }
            qlen -= n;
            __syncwarp();
        }
    }
}

// One warp, one (configuration c, link l, slice sidx) task: the task in slot
// `j` of the warp's grab.  Occupied candidate cells go to the warp's queue;
// full rounds of 32 are looked up at once, a remainder stays queued for the
// next task (the kernel flushes it after the grab).
template <bool BY_POS, bool BRICKS, bool STAGED>
__device__ __forceinline__ void shell_task(const QueryParams& p, const ShellView& sv, uint32_t queue,
                                           const ShellSetup* setups, uint32_t setups_s, uint32_t j, int& qlen,
                                           int lane, const SegAxes& ga) {
    const ShellSetup& st = setups[j];
    const int l = st.l;
    const int64_t c = st.c;
    const int sidx = st.sidx;
    const float slack = st.slack;
    const int ax = st.ax, ay = st.ay, az = st.az;
    const int Wm = p.Wmax;
    // loop-invariant launch constants in registers (opaque: not reloaded per chunk)
    const int nx = (int)opaque_u32((uint32_t)p.dims[0]), ny = (int)opaque_u32((uint32_t)p.dims[1]),
              nz = (int)opaque_u32((uint32_t)p.dims[2]);
    const int n_shell = (int)opaque_u32((uint32_t)p.n_shell), stride = (int)opaque_u32(32u * (uint32_t)p.split);
    const int round_min = (int)opaque_u32((uint32_t)p.round_min);
    const int lin0 = (ax * ny + ay) * nz + az;
    const bool share_cfg = p.per_link == nullptr;

    if (BRICKS) {  // nothing occupied in the window's box: the task has nothing to look up
        const int x0 = max(ax, 0), x1 = min(ax + p.W[0], nx) - 1;
        const int y0 = max(ay, 0), y1 = min(ay + p.W[1], ny) - 1;
        const int z0 = max(az, 0), z1 = min(az + p.W[2], nz) - 1;
        bool hit = false;
        if (x0 <= x1 && y0 <= y1 && z0 <= z1) {
            const int bx0 = x0 >> BRICK_LOG2, by0 = y0 >> BRICK_LOG2, nbyr = (y1 >> BRICK_LOG2) - by0 + 1;
            const int ncol = ((x1 >> BRICK_LOG2) - bx0 + 1) * nbyr;
            const uint32_t zmask = (2u << (z1 >> BRICK_LOG2)) - (1u << (z0 >> BRICK_LOG2));
            const float rinv_y = 1.0f / (float)nbyr;
            for (int i = lane; i < ncol; i += 32) {
                const int qx = __float2int_rz(((float)i + 0.5f) * rinv_y);  // i / nbyr (small integers: exact)
                const int bx = bx0 + qx, by = by0 + (i - qx * nbyr);
                hit |= (sv.bricks[bx * p.nby_brick + by] & zmask) != 0u;
            }
        }
        if (!__any_sync(FULL_MASK, hit)) return;
    }
    float thresh = st.thresh0;  // read at setup (lane-parallel for the grab): no load latency here
    int rounds = 0;

    // Segment bound (f32, conservative): d(p) - k_lo <= value(p) <= d(p) + k_hi
    // with d the distance to the link's axis segment.  An occupied cell whose
    // lower bound exceeds the threshold can neither undercut nor tie the
    // minimum and skips the exact lookup; every cell that is queued WILL be
    // looked up, so its upper bound may lower the threshold at once.
    const float4 su = p.seg_u[l];
    const float k_lo = p.seg_a[l].w, k_hi = p.seg_hi[l];
    const bool use_seg = p.seg_filter && k_lo >= 0.0f;
    const float hull_lim = st.hull_lim;
#ifdef LSDF_STATS
    unsigned long long sc[8] = {1, 0, 0, 0, 0, 0, 0, 0};
#endif
    for (int k0 = sidx * 32; k0 < n_shell; k0 += stride) {
        if (sv_f32<STAGED>(sv.radius, sv.radius_s, k0) - slack > thresh) {  // every later cell is farther
            STAT(6, 1);
            STAT(7, k0 == sidx * 32);
            break;
        }
        STAT(1, 1);
        // the shell list is padded to whole chunks with copies of its last cell
        const uint32_t cell = sv_u32<STAGED>(sv.cells, sv.cells_s, k0 + lane);
        bool occ = false;
        {
            const int mx = cell & 0xff, my = (cell >> 8) & 0xff, mz = cell >> 16;
            // 0 <= x < nx as one unsigned compare per axis
            const unsigned x = (unsigned)(ax + mx), y = (unsigned)(ay + my), z = (unsigned)(az + mz);
            // branch-free: cells outside the grid read word 0 and are masked out
            const bool inb = (x < (unsigned)nx) & (y < (unsigned)ny) & (z < (unsigned)nz);
            const int lin = inb ? lin0 + (mx * ny + my) * nz + mz : 0;
            occ = inb & ((sv_u32<STAGED>(sv.bits, sv.bits_s, lin >> 5) >> (lin & 31)) & 1u);
        }
#ifdef LSDF_STATS
        {
            const unsigned b0 = __ballot_sync(FULL_MASK, occ);
            STAT(2, b0 != 0u);
            STAT(3, __popc(b0));
        }
#endif
        if (use_seg) {  // (dense clouds: some lane of a chunk is nearly always occupied)
            // every lane evaluates the bound (no divergent branch; most lanes are occupied)
            const SegCell sc = seg_cell(ga, cell & 0xff, (cell >> 8) & 0xff, cell >> 16);
            const float d2 = seg_d2(st.sw, st.sv, sc, su.w);
            const float lim = thresh + k_lo;
            occ = occ && lim >= 0.0f && d2 <= fmaf(lim, lim, SEG_D2_ERR);
            const float d2q = occ ? d2 : INFINITY;  // squared segment distance of a cell that stays queued
            // non-negative floats order like their bits: one integer min over the warp
            const uint32_t m = __reduce_min_sync(FULL_MASK, __float_as_uint(d2q));
            // the upper bound d + k_hi holds only for samples inside the grid's
            // cell-centre hull: chunks past the inscribed ball leave thresh alone
            if (m < 0x7f800000u && sv_f32<STAGED>(sv.radius, sv.radius_s, k0 + 31) <= hull_lim) {
                const float dm = __uint_as_float(m) + SEG_D2_ERR;
                const float r = dm * rsqrtf(dm);  // ~2^-22 relative: rounded up below
                thresh = fminf(thresh, fmaf(r, 1.0f + 0x1p-18f, k_hi));
            }
        }
        const unsigned ballot = __ballot_sync(FULL_MASK, occ);
        if (occ) sts_u32(queue + 4u * (uint32_t)(qlen + __popc(ballot & ((1u << lane) - 1u))), cell | (j << 24));
        qlen += __popc(ballot);
        STAT(4, __popc(ballot));
        __syncwarp();
        if (qlen >= round_min) {
            STAT(5, 1);
            const int n = qlen < 32 ? qlen : 32;
            const uint32_t m = lookup_round<BY_POS>(p, sv, setups_s, lane < n ? lds_u32(queue + 4u * (uint32_t)(qlen - n + lane)) : 0u, lane < n,
                                                    j, lane);
            if (m != 0xffffffffu) thresh = fminf(thresh, from_orderable(m));
            if (share_cfg && (++rounds & 3) == 0) {
                const uint64_t kk = ~(uint64_t)__ldcg(p.keys + c);
                if (kk != ~0ull) thresh = fminf(thresh, from_orderable((uint32_t)(kk >> 32)));
            }
            qlen -= n;
        }
        __syncwarp();
    }
#ifdef LSDF_STATS
    if (lane == 0)
        for (int i = 0; i < 8; ++i) atomicAdd(g_stats + i, sc[i]);
#endif
}

// Latency batches (split 1, no segment bound): one warp walks its task's
// shells two chunks per step -- the two chunks' loads, occupancy tests and
// ballots are independent, so each step costs one chunk's dependent latency,
// and one task per (configuration, link) fits the resident warps in one wave
// (split 2 gave 6,000 tasks for 3,552 warps at config 2: a second wave).  The
// second chunk of a step is tested against the threshold at the step's start.
template <bool BY_POS, bool STAGED>
__device__ __forceinline__ void shell_task_dual(const QueryParams& p, const ShellView& sv, uint32_t queue,
                                                const ShellSetup* setups, uint32_t setups_s, uint32_t j, int& qlen,
                                                int lane) {
    const ShellSetup& st = setups[j];
    const int64_t c = st.c;
    const float slack = st.slack;
    const int ax = st.ax, ay = st.ay, az = st.az;
    const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
    const int lin0 = st.lin0;
    const bool share_cfg = p.per_link == nullptr;
    {  // nothing occupied in the window's box: the task has nothing to look up (as shell_task)
        const int x0 = max(ax, 0), x1 = min(ax + p.W[0], nx) - 1;
        const int y0 = max(ay, 0), y1 = min(ay + p.W[1], ny) - 1;
        const int z0 = max(az, 0), z1 = min(az + p.W[2], nz) - 1;
        bool hit = false;
        if (x0 <= x1 && y0 <= y1 && z0 <= z1) {
            const int bx0 = x0 >> BRICK_LOG2, by0 = y0 >> BRICK_LOG2, nbyr = (y1 >> BRICK_LOG2) - by0 + 1;
            const int ncol = ((x1 >> BRICK_LOG2) - bx0 + 1) * nbyr;
            const uint32_t zmask = (2u << (z1 >> BRICK_LOG2)) - (1u << (z0 >> BRICK_LOG2));
            const float rinv_y = 1.0f / (float)nbyr;
            for (int i = lane; i < ncol; i += 32) {
                const int qx = __float2int_rz(((float)i + 0.5f) * rinv_y);  // i / nbyr (small integers: exact)
                const int bx = bx0 + qx, by = by0 + (i - qx * nbyr);
                hit |= (sv.bricks[bx * p.nby_brick + by] & zmask) != 0u;
            }
        }
        if (!__any_sync(FULL_MASK, hit)) return;
    }
    float thresh = st.thresh0;
    int rounds = 0;
    const int n_shell = p.n_shell, round_min = p.round_min;
    const unsigned below = (1u << lane) - 1u;
    auto occupied = [&](uint32_t cell) {
        const int mx = cell & 0xff, my = (cell >> 8) & 0xff, mz = cell >> 16;
        const unsigned x = (unsigned)(ax + mx), y = (unsigned)(ay + my), z = (unsigned)(az + mz);
        const bool inb = (x < (unsigned)nx) & (y < (unsigned)ny) & (z < (unsigned)nz);
        const int lin = inb ? lin0 + (mx * ny + my) * nz + mz : 0;
        return inb & ((sv_u32<STAGED>(sv.bits, sv.bits_s, lin >> 5) >> (lin & 31)) & 1u);
    };
    for (int k0 = 0; k0 < n_shell; k0 += 32 * DUAL_CHUNKS) {
        if (sv_f32<STAGED>(sv.radius, sv.radius_s, k0) - slack > thresh) break;  // every later cell is farther
        uint32_t cell[DUAL_CHUNKS];
        bool occ[DUAL_CHUNKS];
#pragma unroll
        for (int q = 0; q < DUAL_CHUNKS; ++q) {
            const bool has = k0 + 32 * q < n_shell;
            const int kq = has ? k0 + 32 * q : k0;
            const bool act = has && !(sv_f32<STAGED>(sv.radius, sv.radius_s, kq) - slack > thresh);
            cell[q] = sv_u32<STAGED>(sv.cells, sv.cells_s, kq + lane);
            occ[q] = act && occupied(cell[q]);
        }
#pragma unroll
        for (int q = 0; q < DUAL_CHUNKS; ++q) {
            const unsigned b = warp_ballot(occ[q]);
            sts_u32_if(occ[q], queue + 4u * (uint32_t)(qlen + __popc(b & below)), cell[q] | (j << 24));
            qlen += __popc(b);
        }
        __syncwarp();
        while (qlen >= round_min) {
            const int n = qlen < 32 ? qlen : 32;
            const uint32_t m = lookup_round<BY_POS>(p, sv, setups_s, lane < n ? lds_u32(queue + 4u * (uint32_t)(qlen - n + lane)) : 0u,
                                                    lane < n, j, lane);
            if (m != 0xffffffffu) thresh = fminf(thresh, from_orderable(m));
            if (share_cfg && (++rounds & 3) == 0) {
                const uint64_t kk = ~(uint64_t)__ldcg(p.keys + c);
                if (kk != ~0ull) thresh = fminf(thresh, from_orderable((uint32_t)(kk >> 32)));
            }
            qlen -= n;
            __syncwarp();
        }
    }
}

// Persistent over groups of 8 tasks (a group never mixes links).  The window
// offsets, the shell-ordered cell list and the occupancy bitmap are staged in
// shared memory once per CTA when they fit, so the per-chunk loads of the
// scan are shared-memory loads.
// STAGED: the shell list and the bitmap are both in shared memory (a
// compile-time fact, so the scan's table loads are LDS, not generic loads).
template <bool BY_POS, bool BRICKS, bool STAGED>
__global__ void __launch_bounds__(32 * WARPS, LSDF_SHELL_MINB) query_shells_kernel(const __grid_constant__ QueryParams p,
                                                                  int n_group, int launch, int grab,
                                                                  int stage_shell, int stage_bits, int64_t n_words,
                                                                  int last_launch) {
    extern __shared__ double s_dyn[];
    const int warp = threadIdx.x >> 5, lane = (int)opaque_u32(threadIdx.x & 31);
#ifdef LSDF_TIMING
    const unsigned long long t_entry = gtime();
    if (lane == 0) atomicMin(g_tim + 0, t_entry);
#endif
    double* sP = s_dyn;
    uint32_t* s_queue = (uint32_t*)(sP + 3 * p.Wmax);
    // staged tables start on 16-B boundaries (cp.async 16-B chunks)
    uint32_t* s_cells = (uint32_t*)align16_ptr(s_queue + WARPS * QCAP_SHELL);
    float* s_radius = (float*)align16_ptr(s_cells + (stage_shell ? shell_padded(p.n_shell) : 0));
    uint32_t* s_bits = (uint32_t*)align16_ptr(s_radius + (stage_shell ? shell_padded(p.n_shell) : 0));
    uint32_t* s_bricks = (uint32_t*)align16_ptr(s_bits + (stage_bits ? (n_words + 3) & ~3 : 0));
    const int n_cols = (BRICKS && p.stage_bricks) ? (int)(((p.dims[0] + 3) >> BRICK_LOG2) * p.nby_brick) : 0;
    uint32_t* s_dil = s_bricks;  // throughput variant: the dilated map (and its scratch) in place of the columns
    const bool dilate = !BRICKS && p.dilate > 0;
    __shared__ ShellSetup s_setup[WARPS][GRAB_MAX];
    // Stage the shell list and the occupancy bitmap with asynchronous copies
    // (all in flight at once), and fetch + set up the first tasks while they
    // land: the latency path pays one memory round trip here, not one per
    // loop iteration.
    // one thread issues a bulk copy per table (cp.async.bulk, completing on an
    // mbarrier); sizes round up to 16 B inside the padded source allocations
    __shared__ uint64_t s_bar;
    if (threadIdx.x == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        const uint32_t b_shell = stage_shell ? (uint32_t)shell_padded(p.n_shell) * 4u : 0u;
        const uint32_t b_bits = stage_bits ? ((uint32_t)n_words * 4u + 15u) & ~15u : 0u;
        const uint32_t b_cols = ((uint32_t)n_cols * 4u + 15u) & ~15u;
        mbar_expect_tx(&s_bar, 2u * b_shell + b_bits + b_cols);
        if (b_shell) {
            bulk_copy(s_cells, p.shell_cells, b_shell, &s_bar);
            bulk_copy(s_radius, p.shell_radius, b_shell, &s_bar);
        }
        if (b_bits) bulk_copy(s_bits, p.bitmap, b_bits, &s_bar);
        if (b_cols) bulk_copy(s_bricks, p.bricks, b_cols, &s_bar);
    }
    for (int i = threadIdx.x; i < 3 * p.Wmax; i += blockDim.x) sP[i] = p.P[i];
    if (dilate) build_dilated(p, s_dil, s_dil + p.nbx_brick * p.nby_brick);
    const uint32_t* dil = dilate ? s_dil : nullptr;
    // link processing order (lane k holds the link of rank k): decreasing
    // argmin count of the previous cycle, ties in p.group order
    int order_lane = lane < n_group ? p.group[lane] : 0;
    if (p.track_order) {
        const int k = lane;
        const uint32_t mine = k < n_group ? __ldcg(p.link_hist + p.group[k]) : 0u;
        int rank = 0;
        for (int j = 0; j < n_group; ++j) {
            const uint32_t other = __shfl_sync(FULL_MASK, mine, j);
            rank += (other > mine) | ((other == mine) & (j < k));
        }
        int inv = 0;
        for (int j = 0; j < n_group; ++j) {
            const int rj = __shfl_sync(FULL_MASK, rank, j);
            const int gj = __shfl_sync(FULL_MASK, order_lane, j);
            inv = rj == k ? gj : inv;
        }
        order_lane = inv;
    }
    // dynamic task fetch: task durations vary by orders of magnitude (early
    // stop), so each warp takes `grab` tasks at a time from a global counter
    // (reset by finalize_kernel).  Task order is link-major, so consecutive
    // tasks share the link grid.
    // The per-task constants of a grab are computed lane-parallel (lane j
    // for task base + j) into shared memory.
    const uint32_t n_tasks = (uint32_t)(p.C * p.split) * (uint32_t)n_group;
    __shared__ int s_order[WARPS][LSDF_MAX_LINKS];
    if (lane < n_group) s_order[warp][lane] = order_lane;
    __syncwarp();
    // the first grab of every warp is static (warp w takes tasks [w g, w g + g)):
    // thousands of warps starting at once would otherwise serialise on the
    // counter's L2 atomic unit; later grabs come from the counter, offset past
    // the static range
    uint32_t base = 0, g = (uint32_t)grab;
    const uint32_t static_total = gridDim.x * WARPS * g;
    base = (blockIdx.x * WARPS + warp) * g;
    if (base < n_tasks && (uint32_t)lane < min(g, n_tasks - base))
        shell_setup(p, s_order[warp], base + lane, s_setup[warp][lane], dil);
    __syncwarp();
    __syncthreads();  // (the barrier's init is visible to every thread from here)
    mbar_wait(&s_bar, 0);
#ifdef LSDF_TIMING
    const unsigned long long t_staged = gtime();
    if (lane == 0) {
        TIM(1, t_staged - t_entry);  // prologue incl. the first grab's setup
        TIM(2, 1);                   // warps
    }
#endif
    ShellView sv;
    sv.cells = (STAGED || stage_shell) ? s_cells : p.shell_cells;
    sv.radius = (STAGED || stage_shell) ? s_radius : p.shell_radius;
    sv.bits = (STAGED || stage_bits) ? s_bits : p.bitmap;
    // (opaque to the compiler: it would otherwise rematerialize these
    // shared-window addresses from the dynamic-smem base in every chunk)
    sv.cells_s = opaque_u32(smem_u32(s_cells));
    sv.radius_s = opaque_u32(smem_u32(s_radius));
    sv.bits_s = opaque_u32(smem_u32(s_bits));
    sv.P_s = opaque_u32(smem_u32(sP));
    sv.bricks = n_cols ? s_bricks : p.bricks;
    sv.P = sP;
    const uint32_t queue = opaque_u32(smem_u32(s_queue + warp * QCAP_SHELL));
    const uint32_t setups_s = opaque_u32(smem_u32(&s_setup[warp][0]));
    // paired scan (two tasks per chunk walk) for throughput batches of one slice per task
    const bool pair = p.pair_scan && p.split == 1;
    const SegAxes ga = seg_axes(p);  // (segment-bound cell constants, once per warp)
    // sparse clouds (throughput batches): the paired scan skips chunks with no
    // occupied cell when under 1/SPARSE_FRACTION of the voxels are occupied;
    // each warp estimates the fraction from 128 bitmap words spread over the
    // grid (no CTA barrier on the prologue)
    bool skip_empty = false;
    if (!BRICKS && pair && p.skip_empty) {
        const int64_t step = n_words / 128 > 1 ? n_words / 128 : 1;
        uint32_t cnt = 0, words = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t w = (int64_t)(lane + 32 * k) * step;
            if (w < n_words) {
                cnt += __popc(sv_u32<STAGED>(sv.bits, sv.bits_s, (int)w));
                ++words;
            }
        }
        cnt = __reduce_add_sync(FULL_MASK, cnt);
        words = __reduce_add_sync(FULL_MASK, words);
        skip_empty = p.skip_empty == 2 || (int64_t)cnt * SPARSE_FRACTION < (int64_t)words * 32;
    }
    // guided grab sizes: the grab shrinks as the remaining work does, so the
    // last warps to finish carry at most a small grab (shorter tail)
    const uint32_t warps_total = gridDim.x * WARPS;
    for (bool first = true;; first = false) {
        if (!first) {
            if (p.static_sched) {  // (g == 1) warp w's tasks are w, w + W, w + 2W, ...
                base += warps_total;
            } else {
                if (lane == 0) base = static_total + atomicAdd(p.counters + launch, g);
                base = __shfl_sync(FULL_MASK, base, 0);
            }
        }
        if (base >= n_tasks) break;
        const uint32_t cnt = min(g, n_tasks - base);
#ifdef LSDF_TIMING
        const unsigned long long t_g0 = gtime();
#endif
        if (!first && (uint32_t)lane < cnt)
            shell_setup(p, s_order[warp], base + lane, s_setup[warp][lane], dil);
        __syncwarp();
#ifdef LSDF_TIMING
        const unsigned long long t_g1 = gtime();
        if (lane == 0) {
            TIM(3, t_g1 - t_g0);  // setup (later grabs)
            TIM(4, 1);            // grabs
            TIM(5, cnt);          // tasks
        }
#endif
        if (grab > 1) {
            const uint32_t left = n_tasks - min(base + cnt, n_tasks);
            g = max(1u, min((uint32_t)grab, left / (2 * warps_total)));
        }
        int qlen = 0;
        uint32_t j = 0;
        if (!BRICKS && pair)
            while (j + PAIR_N <= cnt) {
                // the paired tasks share one link (a grab straddles a link boundary at most once)
                if (lds_s32(setups_s + j * (uint32_t)sizeof(ShellSetup) + (uint32_t)offsetof(ShellSetup, l)) ==
                    lds_s32(setups_s + (j + PAIR_N - 1) * (uint32_t)sizeof(ShellSetup) + (uint32_t)offsetof(ShellSetup, l))) {
                    if (skip_empty)
                        shell_task_pair<BY_POS, STAGED, true>(p, sv, queue, setups_s, j, qlen, lane, ga);
                    else
                        shell_task_pair<BY_POS, STAGED, false>(p, sv, queue, setups_s, j, qlen, lane, ga);
                    j += PAIR_N;
                } else {
                    shell_task<BY_POS, BRICKS, STAGED>(p, sv, queue, s_setup[warp], setups_s, j, qlen, lane, ga);
                    ++j;
                }
            }
        if (BRICKS && p.dual && p.split == 1)
            for (; j < cnt; ++j) shell_task_dual<BY_POS, STAGED>(p, sv, queue, s_setup[warp], setups_s, j, qlen, lane);
        for (; j < cnt; ++j) shell_task<BY_POS, BRICKS, STAGED>(p, sv, queue, s_setup[warp], setups_s, j, qlen, lane, ga);
#ifdef LSDF_TIMING
        const unsigned long long t_g2 = gtime();
        if (lane == 0) TIM(6, t_g2 - t_g1);  // scans of the grab's tasks
#endif
        if (qlen > 0)  // the grab's remaining lookups, before its setups are overwritten
            lookup_round<BY_POS>(p, sv, setups_s, lane < qlen ? lds_u32(queue + 4u * (uint32_t)lane) : 0u, lane < qlen, 0xffu, lane);
        __syncwarp();
#ifdef LSDF_TIMING
        if (lane == 0) TIM(7, gtime() - t_g2);  // flush rounds
#endif
    }
#ifdef LSDF_TIMING
    if (lane == 0) {
        const unsigned long long t_end = gtime();
        atomicMax(g_tim + 8, t_end);
        TIM(9, t_end - t_entry);  // warp lifetime
        TIM(10, t_end - t_staged);
    }
#endif
    // the last CTA of the last launch clears the counts this cycle's finalize refills
    if (p.track_order) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(p.exit_count, 1u) == gridDim.x - 1) {
                *p.exit_count = 0u;
                if (last_launch)
                    for (int k = 0; k < LSDF_MAX_LINKS; ++k) p.link_hist[k] = 0u;
            }
        }
    }
}

// (d, link, voxel) per configuration from the reduced keys; resets the slots.
// Also counts the argmin links (block histogram, then one atomic per link):
// the next shell scan processes the links most often closest first, so the
// per-configuration threshold they publish lets the other links stop early.
__global__ void finalize_kernel(const __grid_constant__ QueryParams p) {
    __shared__ uint32_t hist[LSDF_MAX_LINKS];
    if (threadIdx.x < LSDF_MAX_LINKS) hist[threadIdx.x] = 0;
    __syncthreads();
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < LSDF_MAX_LINKS) p.counters[c] = 0;  // shell-scan work counters
    const int link = c < p.C ? finalize(p, c) : -1;
    if (p.track_order) {
        if (link >= 0) atomicAdd(hist + link, 1u);
        __syncthreads();
        if (threadIdx.x < p.n_geo && hist[threadIdx.x]) atomicAdd(p.link_hist + threadIdx.x, hist[threadIdx.x]);
    }
}

inline int64_t ws_bytes(int64_t C, int32_t n_geo) {
    return align256(C * 4) + align256(C * 8) + align256(C * n_geo * 4) + 256;
}

}  // namespace

extern "C" int64_t lsdf_query_workspace_bytes(int64_t C, int32_t n_geo) { return ws_bytes(C, n_geo); }

namespace {

constexpr int STAGE_SCAN = 1, STAGE_FINALIZE = 2;

// Tuning overrides for A/B sweeps on the GPU box (tools/cycle_parts.py):
// LSDF_TUNE_<NAME>=<int>, read once per process; unset = the built-in choice.
int tune(const char* name, int dflt) {
    const char* v = getenv(name);
    return (v != nullptr && *v) ? atoi(v) : dflt;
}

int query_impl(const double* R_geo_dev, const double* dt_geo_dev, const int32_t* anchor_geo_dev, int64_t C,
               int32_t n_geo, const lsdf_link_grid* grids, const lsdf_window* window, const lsdf_env_grid* env,
               const void* occupancy_dev, int32_t by_position, double d_far_global, void* workspace_dev, float* d_dev,
               int32_t* link_dev, int32_t* voxel_dev, float* per_link_dev, void* stream, int stages) {
    if (n_geo < 1 || n_geo > LSDF_MAX_LINKS) return fail(LSDF_ERR_VALIDATION, "query: %d geometry links", n_geo);
    if (window->W[0] > LSDF_MAX_WINDOW || window->W[1] > LSDF_MAX_WINDOW || window->W[2] > LSDF_MAX_WINDOW)
        return fail(LSDF_ERR_UNSUPPORTED, "query: window wider than %d cells", LSDF_MAX_WINDOW);
    const int64_t V = n_vox(*env);
    if ((double)C * 4 * n_geo >= 4294967295.0)
        return fail(LSDF_ERR_UNSUPPORTED, "query: %lld configurations overflow the 32-bit task counter", (long long)C);
    if ((double)V * n_geo >= 4294967295.0)
        return fail(LSDF_ERR_UNSUPPORTED, "query: %lld voxels x %d links overflow the 32-bit key", (long long)V, n_geo);
    if (C <= 0) return LSDF_OK;
    QueryParams p{};
    const float clamp = (float)d_far_global;
    int full = 0;
    for (int l = 0; l < n_geo; ++l) {
        const lsdf_link_grid& g = grids[l];
        if (g.packed_dev == nullptr) return fail(LSDF_ERR_VALIDATION, "query: link %d has no packed-corner grid", l);
        p.cells[l] = (const float4*)g.packed_dev;
        p.dfar[l] = g.d_far;
        p.core[l] = g.core_radius;
        p.seg_a[l] = make_float4(g.seg_a[0], g.seg_a[1], g.seg_a[2], g.seg_kappa_lo);
        p.seg_u[l] = make_float4(g.seg_u[0], g.seg_u[1], g.seg_u[2], g.seg_len);
        p.seg_hi[l] = g.seg_kappa_hi;
        if (g.d_far < clamp) full = 1;  // masked cells can undercut the clamp
    }
    if (window->zrange_dev == nullptr) full = 1;
    p.R = R_geo_dev;
    p.dt = dt_geo_dev;
    p.anchor = anchor_geo_dev;
    p.C = C;
    p.n_geo = n_geo;
    const bool shells = !full && window->shell_cells_dev != nullptr && window->shell_radius_dev != nullptr;
    // the link order matters when links share a threshold and the batch is
    // larger than one wave of tasks (small batches run all links at once)
    p.track_order = shells && per_link_dev == nullptr && C * n_geo >= SEG_FILTER_MIN_TASKS;
    // the column scan needs enough warps in flight for small batches; the
    // shell scan stops early, so one warp per (configuration, link) is best
    const int64_t target = 148LL * 64;
    // shells: about one resident wave (148 SMs x 32 warps) in flight for small batches
    int64_t split = shells ? (148LL * 32 + C * n_geo - 1) / (C * n_geo) : (target + C * n_geo - 1) / (C * n_geo);
    split = split < 1 ? 1 : (split > (shells ? 4 : 8) ? (shells ? 4 : 8) : split);
    static const int t_split = tune("LSDF_TUNE_SPLIT", 0);
    if (t_split > 0 && shells) split = t_split;
    if (shells) split = split >= 4 ? 4 : (split >= 2 ? 2 : 1);  // a power of two: shifts in the task decode
    // latency batches walk two chunks per step with one task per (c, l) instead
    // (shell_task_dual: every task resident in one wave)
    // (dense obstacles, LSDF_QUERY_DENSE_HINT: tasks stop early, and the second
    // wave of split 2 was the latency; sparse ones keep split 2, whose two warps
    // per (c, l) share the lookups of long walks)
    static const int t_dual = tune("LSDF_TUNE_DUAL", 1);  // 0 never, 1 with the hint, 2 always
    p.dual = shells && C * n_geo < SEG_FILTER_MIN_TASKS && t_split == 0 &&
             (t_dual == 2 || (t_dual == 1 && (by_position & LSDF_QUERY_DENSE_HINT) != 0));
    if (p.dual) split = 1;
    p.split_log2 = split == 4 ? 2 : (split == 2 ? 1 : 0);
    p.split = (int32_t)split;
    p.n_tasks = C * n_geo * split;
    {  // magic numbers of t / (C * split)
        const uint64_t d = (uint64_t)C * split;
        int sh = 0;
        while ((1ull << sh) < d) ++sh;
        p.pl_shift = sh;
        p.pl_mul = sh == 0 ? 0u : (uint32_t)(((1ull << 32) * ((1ull << sh) - d)) / d + 1);
    }
    for (int a = 0; a < 3; ++a) {
        p.W[a] = window->W[a];
        p.dims[a] = env->dims[a];
    }
    p.full_window = full;
    p.e_r = window->e_r;
    p.e_rinv = 1.0 / window->e_r;
    p.shell_cells = window->shell_cells_dev;
    p.shell_radius = window->shell_radius_dev;
    p.n_shell = window->n_masked;
    // the bound saves lookups but lengthens each warp's dependent chain: a
    // win when the GPU is full of tasks, a loss on the latency path
    p.seg_filter = C * n_geo >= SEG_FILTER_MIN_TASKS;
    // latency-sized batches: a lookup round once 16 cells are queued, so the
    // task's threshold drops (and its scan stops) sooner; throughput batches
    // only run full rounds (issue-bound: a half round wastes lanes)
    static const int t_round = tune("LSDF_TUNE_ROUND_MIN", 0);
    p.round_min = t_round > 0 ? t_round : (p.seg_filter ? 32 : 16);
    p.P = window->P_dev;
    p.Wmax = window->Wmax;
    p.by_position = by_position & LSDF_QUERY_BY_POSITION;
    const bool link_major = (by_position & LSDF_QUERY_POSES_LINK_MAJOR) != 0;
    p.pose_cs = link_major ? 1 : n_geo;
    p.pose_ls = link_major ? C : 1;
    p.zrange = window->zrange_dev;
    p.mask_bits = window->mask_bits_dev;
    p.clamp = clamp;
    Occupancy o = carve_occupancy(const_cast<void*>(occupancy_dev), *env);
    p.bitmap = o.bitmap;
    // the brick box test: latency-sized batches (sparse or far obstacles leave
    // whole windows empty); dense throughput batches would only pay for it
    static const int t_bricks = tune("LSDF_TUNE_BRICKS", 1);
    p.bricks = (o.bricks_ok && !p.seg_filter && t_bricks) ? o.bricks : nullptr;
    p.nby_brick = o.nby;
    p.brick_cols = o.bricks;
    p.nbx_brick = o.nbx;
    p.nbz_brick = o.nbz;
    p.dilate = 0;
    p.prefix = o.prefix;
    p.posgrid = o.posgrid;
    char* w = (char*)workspace_dev;
    p.counters = (uint32_t*)w;
    w += align256(C * 4);
    p.keys = (unsigned long long*)w;
    w += align256(C * 8);
    p.perlink = (uint32_t*)w;
    w += align256(C * n_geo * 4);
    p.link_hist = (uint32_t*)w;                    // LSDF_MAX_LINKS counts
    p.exit_count = (uint32_t*)w + LSDF_MAX_LINKS;

    p.d_out = d_dev;
    p.link_out = link_dev;
    p.voxel_out = voxel_dev;
    p.per_link = per_link_dev;
    const size_t smem = (size_t)3 * window->Wmax * sizeof(double) + (size_t)WARPS * QCAP * sizeof(uint32_t);
    const int64_t blocks_per_link = (C * split + WARPS - 1) / WARPS;
    cudaStream_t s = (cudaStream_t)stream;
    // one launch per group of links with identical grid geometry (normally one)
    auto same_geom = [&](int a_, int b_) {
        bool same = true;
        for (int a = 0; a < 3; ++a)
            same &= grids[a_].dims[a] == grids[b_].dims[a] && grids[a_].extent[a] == grids[b_].extent[a] &&
                    grids[a_].resolution[a] == grids[b_].resolution[a];
        return same;
    };
    int n_groups_total = 0;
    for (int l = 0; l < n_geo; ++l) {
        bool first = true;
        for (int k = 0; k < l && first; ++k) first = !same_geom(k, l);
        n_groups_total += first;
    }
    bool done[LSDF_MAX_LINKS] = {false};
    int n_launch = 0;
    for (int l0 = 0; l0 < n_geo && (stages & STAGE_SCAN); ++l0) {
        if (done[l0]) continue;
        const lsdf_link_grid& g0 = grids[l0];
        int n_group = 0;
        for (int l = l0; l < n_geo; ++l) {
            const lsdf_link_grid& g = grids[l];
            bool same = true;
            for (int a = 0; a < 3; ++a)
                same &= g.dims[a] == g0.dims[a] && g.extent[a] == g0.extent[a] && g.resolution[a] == g0.resolution[a];
            if (same && !done[l]) {
                done[l] = true;
                p.group[n_group++] = l;
            }
        }
        for (int a = 0; a < 3; ++a) {
            p.geom.ext[a] = g0.extent[a];
            p.geom.res[a] = g0.resolution[a];
            p.geom.rinv[a] = 1.0 / g0.resolution[a];  // RN(1/r): the Markstein reciprocal
            p.geom.hi[a] = (double)(g0.dims[a] - 1);
            p.geom.topd[a] = (double)(g0.dims[a] - 2);
            p.geom.top[a] = g0.dims[a] - 2;
        }
        {  // inscribed ball of the cell-centre hull [-e + r/2, e - r/2]^3, less a margin for rounding
            double h = g0.extent[0] - 0.5 * g0.resolution[0];
            for (int a = 1; a < 3; ++a) h = fmin(h, g0.extent[a] - 0.5 * g0.resolution[a]);
            p.hull = h - 1e-5;
        }
        p.geom.cx = g0.dims[0] - 1;
        p.geom.cy = g0.dims[1] - 1;
        const unsigned blocks = (unsigned)(blocks_per_link * n_group);
        if (shells) {
            static const int t_stage = tune("LSDF_TUNE_STAGE", 3);  // bit 0: shell list, bit 1: bitmap
            const int stage_shell = (t_stage & 1) && p.n_shell <= SHELL_STAGE_MAX;
            const int stage_bits = (t_stage & 2) && o.n_words <= BITMAP_STAGE_MAX;
            // brick columns in shared memory when they fit the budget, else read from L2
            p.stage_bricks = p.bricks != nullptr && (int64_t)o.nbx * o.nby <= BRICK_STAGE_MAX;
            // throughput batches: the dilated brick map (one bit test per task at setup)
            p.dilate = (p.bricks == nullptr && o.bricks_ok && (int64_t)o.nbx * o.nby <= DILATE_MAX_COLS)
                           ? (window->Wmax / 2 + 3) >> BRICK_LOG2 : 0;
            const size_t smem_s = (size_t)3 * window->Wmax * sizeof(double) +
                                  (size_t)WARPS * QCAP_SHELL * 4 +
                                  (stage_shell ? (size_t)shell_padded(p.n_shell) * 8 : 0) + (stage_bits ? (size_t)o.n_words * 4 : 0) +
                                  (p.stage_bricks ? (size_t)o.nbx * o.nby * 4 : 0) +
                                  (p.dilate ? (size_t)o.nbx * o.nby * 8 : 0) +
                                  96;  // 16-B alignment and 16-B rounding of the staged tables
            using ShellsKernel = void (*)(QueryParams, int, int, int, int, int, int64_t, int);
            static const ShellsKernel kernels[8] = {
                query_shells_kernel<false, false, false>, query_shells_kernel<false, true, false>,
                query_shells_kernel<true, false, false>,  query_shells_kernel<true, true, false>,
                query_shells_kernel<false, false, true>,  query_shells_kernel<false, true, true>,
                query_shells_kernel<true, false, true>,   query_shells_kernel<true, true, true>};
            static const int t_lds = tune("LSDF_TUNE_LDS", 1);
            static const int t_pair = tune("LSDF_TUNE_PAIR", 1);
#ifdef LSDF_STATS
            p.pair_scan = 0;  // the per-task counters live in shell_task: count the same decisions one task at a time
#else
            p.pair_scan = t_pair;
#endif
            static const int t_skip = tune("LSDF_TUNE_SKIPEMPTY", 1);
            p.skip_empty = t_skip;
            const int variant = (p.by_position ? 2 : 0) + (p.bricks != nullptr ? 1 : 0) +
                                (t_lds && stage_shell && stage_bits ? 4 : 0);
            const ShellsKernel kern = kernels[variant];
            LSDF_TRY(ensure_smem((const void*)kern, smem_s, "query_shells_kernel"));
            // residency cache: (device, variant, smem bytes) -> CTAs per SM
            thread_local int c_dev = -1, c_bp = -1, c_sm = 148, c_per = 1;
            thread_local size_t c_smem = 0;
            int dev = 0;
            cudaGetDevice(&dev);
            if (dev != c_dev || variant != c_bp || smem_s != c_smem) {
                cudaDeviceGetAttribute(&c_sm, cudaDevAttrMultiProcessorCount, dev);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c_per, kern, 32 * WARPS, smem_s);
                c_dev = dev;
                c_bp = variant;
                c_smem = smem_s;
            }
            const int per_sm = c_per, n_sm = c_sm;
            const int64_t resident = (int64_t)n_sm * (per_sm < 1 ? 1 : per_sm);
            const unsigned grid = (unsigned)((int64_t)blocks < resident ? (int64_t)blocks : resident);
            const int64_t n_tasks = C * split * n_group;
            int64_t grab = n_tasks / (resident * WARPS * 8);
            grab = grab < 1 ? 1 : (grab > GRAB_MAX ? GRAB_MAX : grab);
            static const int t_grab = tune("LSDF_TUNE_GRAB", 0);
            if (t_grab > 0) grab = t_grab < GRAB_MAX ? t_grab : GRAB_MAX;
            // latency batches (one task per grab, a few tasks per warp): a static
            // round-robin schedule, no task counter for thousands of warps to
            // serialise on
            static const int t_static = tune("LSDF_TUNE_STATIC", 0);
            p.static_sched = t_static && grab == 1 && n_tasks <= 4 * resident * WARPS;
            // grids pinned in L2: an access-policy window over the span of
            // this group's packed grids (contiguous when TrajectorySdf packed
            // them into one arena), persisting within the set-aside that
            // lsdf_l2_reserve granted; the attribute is captured into graphs
            cudaLaunchAttribute attr_l2[1];
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(32 * WARPS);
            cfg.dynamicSmemBytes = smem_s;
            cfg.stream = s;
            cfg.attrs = attr_l2;
            cfg.numAttrs = 0;
            const size_t persist = l2_persist_bytes(dev);
            if (persist > 0) {
                uintptr_t lo = UINTPTR_MAX, hi = 0;
                for (int k = 0; k < n_group; ++k) {
                    const lsdf_link_grid& g = grids[p.group[k]];
                    const uintptr_t a = (uintptr_t)g.packed_dev;
                    const uintptr_t b = a + (uintptr_t)(g.dims[0] - 1) * (g.dims[1] - 1) * (g.dims[2] - 1) * 32;
                    lo = a < lo ? a : lo;
                    hi = b > hi ? b : hi;
                }
                thread_local int w_dev = -1, w_max = 0;
                if (w_dev != dev) {
                    cudaDeviceGetAttribute(&w_max, cudaDevAttrMaxAccessPolicyWindowSize, dev);
                    w_dev = dev;
                }
                const size_t span = hi - lo;
                if (span > 0 && span <= (size_t)w_max) {
                    attr_l2[0].id = cudaLaunchAttributeAccessPolicyWindow;
                    attr_l2[0].val.accessPolicyWindow.base_ptr = (void*)lo;
                    attr_l2[0].val.accessPolicyWindow.num_bytes = span;
                    attr_l2[0].val.accessPolicyWindow.hitRatio = span <= persist ? 1.0f : (float)persist / span;
                    attr_l2[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                    attr_l2[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
                    cfg.numAttrs = 1;
                }
            }
            const int ig = (int)grab;
            const int last = n_launch + 1 == n_groups_total;
            const cudaError_t le = cudaLaunchKernelEx(&cfg, kern, p, n_group, n_launch, ig, stage_shell, stage_bits,
                                                      o.n_words, last);
            if (le != cudaSuccess) return fail(LSDF_ERR_CUDA, "query_shells_kernel: %s", cudaGetErrorString(le));
            ++n_launch;
        } else if (full) {
            if (p.by_position)
                query_direct_kernel<true, true><<<blocks, 32 * WARPS, smem, s>>>(p, blocks_per_link);
            else
                query_direct_kernel<true, false><<<blocks, 32 * WARPS, smem, s>>>(p, blocks_per_link);
        } else {
            if (p.by_position)
                query_direct_kernel<false, true><<<blocks, 32 * WARPS, smem, s>>>(p, blocks_per_link);
            else
                query_direct_kernel<false, false><<<blocks, 32 * WARPS, smem, s>>>(p, blocks_per_link);
        }
        LSDF_TRY(check_launch("query_direct_kernel"));
    }
    if (!(stages & STAGE_FINALIZE)) return LSDF_OK;
    finalize_kernel<<<grid_for(C > LSDF_MAX_LINKS ? C : LSDF_MAX_LINKS, 128), 128, 0, s>>>(p);
    return check_launch("finalize_kernel");

}

}  // namespace

#define LSDF_QUERY_ARGS                                                                                            \
    const double *R_geo_dev, const double *dt_geo_dev, const int32_t *anchor_geo_dev, int64_t C, int32_t n_geo,   \
        const lsdf_link_grid *grids, const lsdf_window *window, const lsdf_env_grid *env, const void *occupancy_dev, \
        int32_t by_position, double d_far_global, void *workspace_dev, float *d_dev, int32_t *link_dev,           \
        int32_t *voxel_dev, float *per_link_dev, void *stream
#define LSDF_QUERY_FWD                                                                                   \
    R_geo_dev, dt_geo_dev, anchor_geo_dev, C, n_geo, grids, window, env, occupancy_dev, by_position,    \
        d_far_global, workspace_dev, d_dev, link_dev, voxel_dev, per_link_dev, stream

extern "C" int lsdf_query_direct(LSDF_QUERY_ARGS) { return query_impl(LSDF_QUERY_FWD, STAGE_SCAN | STAGE_FINALIZE); }
extern "C" int lsdf_query_scan(LSDF_QUERY_ARGS) { return query_impl(LSDF_QUERY_FWD, STAGE_SCAN); }
extern "C" int lsdf_query_finalize(LSDF_QUERY_ARGS) { return query_impl(LSDF_QUERY_FWD, STAGE_FINALIZE); }

#ifdef LSDF_TIMING
extern "C" int lsdf_timing_read(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, g_tim, sizeof(unsigned long long) * 16);
    if (reset) {
        unsigned long long z[16] = {0};
        z[0] = ~0ull;
        cudaMemcpyToSymbol(g_tim, z, sizeof(z));
    }
    return 0;
}
#endif

#ifdef LSDF_STATS
extern "C" int lsdf_stats_read(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, g_stats, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_stats, z, sizeof(z));
    }
    return 0;
}
#endif
