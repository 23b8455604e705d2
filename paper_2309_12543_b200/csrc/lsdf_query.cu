// lsdf_query.cu — stages 3 + 4: the fused direct query (the hot kernel).
//
// For configuration c the reference assembles a dense robot SDF (min over
// links of each link's resampled window, clamped at d_far_global;
// placement.py:267-313, query.py:61-103) and gathers it at the occupied
// voxels (query.py:128-150).  Only the occupied voxels inside a link's
// sphere-masked window can differ from the clamp, so this kernel evaluates
// exactly those: for each (c, l) it walks the window's (x, y) columns, takes
// the column's kept z-interval from the occupancy bitmap, and for every
// occupied cell recomputes the reference's resampled value
//   g = P R + dt_inv (fp64, placement.py:164-167), point = g * e_r,
//   trilinear_sample(sdf_l, point) (grids.py:155-191),
// bit-identical to the assembled field.  Keys (value, rank, link) reduce with
// a warp shuffle and one 64-bit atomic per warp; the last warp of a
// configuration finishes (d, link, voxel) and resets the workspace.
//
// Work decomposition: one warp = one task (link l, configuration c, column
// slice s).  Tasks are link-major, so the SMs sweep one link grid at a time
// (its packed-corner copy stays hot in L2/L1); warps are independent (no
// block barrier), `split` slices per (c, l) keep >= 148 x 64 warps in flight
// for small batches.
#include "lsdf_device.cuh"

using namespace lsdf;

namespace {

struct QueryParams {
    PackedGrid grids[LSDF_MAX_LINKS];
    const double* R;
    const double* dt;
    const int32_t* anchor;
    int64_t C;
    int64_t n_tasks;
    int32_t n_geo, split;
    int32_t W[3];
    int32_t full_window;  // iterate the whole window, masking per cell (d_far_l < clamp)
    double e_r;
    const double* P;
    int32_t Wmax, by_position;
    const int16_t* zrange;
    const uint32_t* mask_bits;
    int32_t dims[3];
    float clamp;
    const uint32_t* bitmap;
    const int32_t* prefix;
    const int32_t* posgrid;
    uint32_t* counters;          // C: tasks finished per configuration
    unsigned long long* keys;    // C: ~best key (atomicMax of the complement, zero = empty)
    uint32_t* perlink;           // C x n_geo: ~orderable(min value)
    float* d_out;
    int32_t* link_out;
    int32_t* voxel_out;
    float* per_link;
};

constexpr int WARPS = 8;
constexpr int QCAP = 32 * 16 + 32;  // queue entries per warp: <= 16 bits per lane per round

__device__ __forceinline__ void finalize(const QueryParams& p, int64_t c) {
    const uint64_t k = ~(uint64_t)atomicExch(p.keys + c, 0ull);
    p.counters[c] = 0;
    if (p.per_link != nullptr) {
        for (int l = 0; l < p.n_geo; ++l) {
            const uint32_t u = ~atomicExch(p.perlink + c * p.n_geo + l, 0u);
            const float v = from_orderable(u);
            p.per_link[c * p.n_geo + l] = fminf(p.clamp, fminf(p.grids[l].d_far, v));  // query.py:171-175
        }
    }
    const uint32_t hi = (uint32_t)(k >> 32);
    if (k == ~0ull || hi >= orderable(p.clamp)) {  // nothing below the monitored range
        p.d_out[c] = p.clamp;
        p.link_out[c] = -1;
        p.voxel_out[c] = -1;
        return;
    }
    const uint32_t lo = (uint32_t)k;
    const uint32_t pos = lo / (uint32_t)p.n_geo;
    p.d_out[c] = from_orderable(hi);
    p.link_out[c] = (int32_t)(lo % (uint32_t)p.n_geo);
    if (p.by_position) {
        p.voxel_out[c] = (int32_t)pos;
    } else {  // rank of the winning voxel in np.unique order
        const uint32_t w = pos >> 5, b = pos & 31;
        const uint32_t below = b ? (p.bitmap[w] & ((1u << b) - 1u)) : 0u;
        p.voxel_out[c] = p.prefix[w] + __popc(below);
    }
}

__global__ void __launch_bounds__(32 * WARPS) query_direct_kernel(const __grid_constant__ QueryParams p) {
    extern __shared__ uint32_t s_queue[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t task = (int64_t)blockIdx.x * WARPS + warp;
    if (task >= p.n_tasks) return;
    uint32_t* queue = s_queue + warp * QCAP;
    const int64_t per_link_tasks = p.C * p.split;
    const int l = (int)(task / per_link_tasks);
    const int64_t rem = task % per_link_tasks;
    const int64_t c = rem / p.split;
    const int sidx = (int)(rem % p.split);

    const PackedGrid& G = p.grids[l];
    const int64_t o = c * p.n_geo + l;
    double R[9], dtinv[3];
#pragma unroll
    for (int e = 0; e < 9; ++e) R[e] = __ldg(p.R + o * 9 + e);
    shift_inverse(R, p.dt + o * 3, p.e_r, dtinv);
    const int ax = __ldg(p.anchor + o * 3), ay = __ldg(p.anchor + o * 3 + 1), az = __ldg(p.anchor + o * 3 + 2);
    const int W0 = p.W[0], W1 = p.W[1], W2 = p.W[2];
    const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
    const double* Px = p.P;
    const double* Py = p.P + p.Wmax;
    const double* Pz = p.P + 2 * p.Wmax;
    const int n_cols = W0 * W1;
    const double e_r = p.e_r;

    uint64_t best = ~0ull;
    float bestval = INFINITY;
    int qlen = 0;

    auto evaluate = [&](uint32_t cell) {
        const int mx = cell & 0xff, my = (cell >> 8) & 0xff, mz = (cell >> 16) & 0xff;
        float v = G.d_far;
        bool in_mask = true;
        if (p.full_window) {
            const int bit = mx + W0 * (my + W1 * mz);
            in_mask = (__ldg(p.mask_bits + (bit >> 5)) >> (bit & 31)) & 1u;
        }
        if (in_mask) {
            double pt[3];
            window_point(__ldg(Px + mx), __ldg(Py + my), __ldg(Pz + mz), R, dtinv, e_r, pt);
            v = trilinear_packed(G, pt[0], pt[1], pt[2]);
            bestval = fminf(bestval, v);
        }
        const int64_t lin = ((int64_t)(ax + mx) * ny + (ay + my)) * nz + (az + mz);
        const uint32_t pos = p.by_position ? (uint32_t)__ldg(p.posgrid + lin) : (uint32_t)lin;
        const uint64_t key = ((uint64_t)orderable(v) << 32) | (uint64_t)(pos * (uint32_t)p.n_geo + l);
        best = key < best ? key : best;
    };

    for (int base = sidx * 32; base < n_cols; base += 32 * p.split) {
        const int col = base + lane;
        const int mx = col % W0, my = col / W0;
        int zcur = 0, zend = 0;
        int64_t bitbase = 0;
        if (col < n_cols) {
            const int x = ax + mx, y = ay + my;
            if (x >= 0 && x < nx && y >= 0 && y < ny) {
                int zlo = 0, zhi = W2;
                if (!p.full_window) {
                    zlo = __ldg(p.zrange + 2 * col);
                    zhi = __ldg(p.zrange + 2 * col + 1);
                }
                zcur = max(az + zlo, 0);
                zend = min(az + zhi, nz);
                bitbase = ((int64_t)x * ny + y) * nz;
            }
        }
        // consume each column's z-run in segments of <= 16 bits, all lanes in step
        while (__any_sync(FULL_MASK, zcur < zend)) {
            uint32_t bits = 0;
            const int zs = zcur;
            if (zcur < zend) {
                const int64_t bp = bitbase + zcur;
                const int off = (int)(bp & 31);
                const int n = min(min(zend - zcur, 16), 32 - off);
                bits = (__ldg(p.bitmap + (bp >> 5)) >> off) & ((1u << n) - 1u);
                zcur += n;
            }
            const int cnt = __popc(bits);
            int incl = cnt;
#pragma unroll
            for (int o2 = 1; o2 < 32; o2 <<= 1) {
                const int t = __shfl_up_sync(FULL_MASK, incl, o2);
                if (lane >= o2) incl += t;
            }
            const int total = __shfl_sync(FULL_MASK, incl, 31);
            int slot = qlen + incl - cnt;
            while (bits) {
                const int b = __ffs(bits) - 1;
                bits &= bits - 1;
                queue[slot++] = (uint32_t)mx | ((uint32_t)my << 8) | ((uint32_t)(zs + b - az) << 16);
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

    best = warp_min_u64(best);
    bestval = warp_min_f(bestval);
    if (lane == 0) {
        atomicMax(p.keys + c, (unsigned long long)~best);
        if (p.per_link != nullptr) atomicMax(p.perlink + o, ~orderable(bestval));
        __threadfence();
        const uint32_t done = atomicAdd(p.counters + c, 1u);
        if (done == (uint32_t)(p.n_geo * p.split - 1)) {
            __threadfence();
            finalize(p, c);
        }
    }
}

inline int64_t ws_bytes(int64_t C, int32_t n_geo) {
    return align256(C * 4) + align256(C * 8) + align256(C * n_geo * 4);
}

}  // namespace

extern "C" int64_t lsdf_query_workspace_bytes(int64_t C, int32_t n_geo) { return ws_bytes(C, n_geo); }

extern "C" int lsdf_query_direct(const double* R_geo_dev, const double* dt_geo_dev, const int32_t* anchor_geo_dev,
                                 int64_t C, int32_t n_geo, const lsdf_link_grid* grids, const lsdf_window* window,
                                 const lsdf_env_grid* env, const void* occupancy_dev, int32_t by_position,
                                 double d_far_global, void* workspace_dev, float* d_dev, int32_t* link_dev,
                                 int32_t* voxel_dev, float* per_link_dev, void* stream) {
    if (n_geo < 1 || n_geo > LSDF_MAX_LINKS) return fail(LSDF_ERR_VALIDATION, "query: %d geometry links", n_geo);
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
        const lsdf_link_grid& g = grids[l];
        if (g.packed_dev == nullptr) return fail(LSDF_ERR_VALIDATION, "query: link %d has no packed-corner grid", l);
        PackedGrid& q = p.grids[l];
        q.cells = (const float4*)g.packed_dev;
        for (int a = 0; a < 3; ++a) {
            q.ext[a] = g.extent[a];
            q.res[a] = g.resolution[a];
            q.rinv[a] = 1.0 / g.resolution[a];  // RN(1/r): the Markstein reciprocal
            q.hi[a] = (double)(g.dims[a] - 1);
            q.top[a] = g.dims[a] - 2;
        }
        q.cx = g.dims[0] - 1;
        q.cy = g.dims[1] - 1;
        q.d_far = g.d_far;
        if (g.d_far < clamp) full = 1;  // masked cells can undercut the clamp
    }
    if (window->zrange_dev == nullptr) full = 1;
    p.R = R_geo_dev;
    p.dt = dt_geo_dev;
    p.anchor = anchor_geo_dev;
    p.C = C;
    p.n_geo = n_geo;
    const int64_t target = 148LL * 64;  // warps for a full machine
    int64_t split = (target + C * n_geo - 1) / (C * n_geo);
    split = split < 1 ? 1 : (split > 8 ? 8 : split);
    p.split = (int32_t)split;
    p.n_tasks = C * n_geo * split;
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
    Occupancy o = carve_occupancy(const_cast<void*>(occupancy_dev), *env);
    p.bitmap = o.bitmap;
    p.prefix = o.prefix;
    p.posgrid = o.posgrid;
    char* w = (char*)workspace_dev;
    p.counters = (uint32_t*)w;
    w += align256(C * 4);
    p.keys = (unsigned long long*)w;
    w += align256(C * 8);
    p.perlink = (uint32_t*)w;
    p.d_out = d_dev;
    p.link_out = link_dev;
    p.voxel_out = voxel_dev;
    p.per_link = per_link_dev;
    const size_t smem = (size_t)WARPS * QCAP * sizeof(uint32_t);
    const int64_t blocks = (p.n_tasks + WARPS - 1) / WARPS;
    query_direct_kernel<<<(unsigned)blocks, 32 * WARPS, smem, (cudaStream_t)stream>>>(p);
    return check_launch("query_direct_kernel");
}
