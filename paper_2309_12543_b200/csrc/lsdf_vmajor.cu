// lsdf_vmajor.cu — the paper's materialized mode with a voxel-major field
// (SURVEY.md §8f rank 1): prepare the robot SDF of a fixed trajectory once,
// then answer every control cycle with one coalesced gather.
//
//   materialize_vm_kernel  placement.py:267-313 + query.py:61-103: every
//                          (c, l) window's kept cells (exact fp64 recipe, as
//                          place_windows_kernel) min-merged into
//                          field[v * C + c] (voxel-major: a voxel's C values
//                          are contiguous), initialised to f32(d_far_global)
//   query_vm_kernel        query.py:128-150: for the occupied voxels in list
//                          order, a CTA reads a voxel's C contiguous values
//                          (coalesced, up to 2 KB) and keeps the
//                          first-occurrence minimum per configuration; one
//                          64-bit atomic per (configuration, CTA) combines
//   link_vm_kernel         SURVEY Appendix B: the lowest link whose window
//                          value at the winning voxel equals d (one thread per
//                          configuration, exact lookups), and the clamp rule
//
// Identical results to assemble_robot_sdfs + query_min_distances + the
// Appendix-B argmin (tests/test_gpu_parity.py::test_voxel_major_mode).
#include "lsdf_device.cuh"

using namespace lsdf;

namespace {

struct VmParams {
    lsdf_link_grid grids[LSDF_MAX_LINKS];
    const double* R;
    const double* dt;
    const int32_t* anchor;
    int64_t C;
    int32_t n_geo;
    int32_t W[3];
    double e_r;
    const double* P;
    int32_t Wmax;
    const uint32_t* mask_bits;
    lsdf_env_grid env;
    float clamp;
    float* field;  // (V, C)
};

__device__ __forceinline__ void atomic_min_f32(float* addr, float v) {
    if (v >= 0.0f)
        atomicMin((int*)addr, __float_as_int(v));
    else
        atomicMax((unsigned int*)addr, __float_as_uint(v));
}

__global__ void fill_f32_kernel(float* out, int64_t n, float v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = v;
}

// One CTA per (c, l) window.  Kept cells carry the exact resampled value;
// masked cells carry the link's far value, which only matters when it is
// below the clamp (a caller-chosen d_far_global above a link's d_far).
__global__ void materialize_vm_kernel(const __grid_constant__ VmParams p) {
    const int64_t f = blockIdx.x;  // c * n_geo + l
    const int64_t c = f / p.n_geo;
    const int l = (int)(f % p.n_geo);
    const lsdf_link_grid& G = p.grids[l];
    const GridView gv = view_of(G);
    const LdgLoad ld{G.values_dev};
    double R[9], dtinv[3];
#pragma unroll
    for (int e = 0; e < 9; ++e) R[e] = p.R[f * 9 + e];
    shift_inverse(R, p.dt + f * 3, p.e_r, dtinv);
    const int ax = p.anchor[f * 3], ay = p.anchor[f * 3 + 1], az = p.anchor[f * 3 + 2];
    const int nx = p.env.dims[0], ny = p.env.dims[1], nz = p.env.dims[2];
    const bool masked_matter = gv.d_far < p.clamp;
    const int W0 = p.W[0], W1 = p.W[1];
    const int n = W0 * W1 * p.W[2];
    for (int cell = threadIdx.x; cell < n; cell += blockDim.x) {
        const int mx = cell % W0, my = (cell / W0) % W1, mz = cell / (W0 * W1);
        const int x = ax + mx, y = ay + my, z = az + mz;
        if (x < 0 || x >= nx || y < 0 || y >= ny || z < 0 || z >= nz) continue;  // query.py:86-99 clip
        const bool keep = (__ldg(p.mask_bits + (cell >> 5)) >> (cell & 31)) & 1u;
        float v = gv.d_far;
        if (keep) {
            double pt[3];
            window_point(p.P[mx], p.P[p.Wmax + my], p.P[2 * p.Wmax + mz], R, dtinv, p.e_r, pt);
            v = trilinear_at(gv, pt[0], pt[1], pt[2], ld);
        } else if (!masked_matter) {
            continue;
        }
        if (v < p.clamp) {
            const int64_t lin = ((int64_t)x * ny + y) * nz + z;
            float* dst = p.field + lin * p.C + c;
            if (v < *dst) atomic_min_f32(dst, v);
        }
    }
}

// Occupied voxels (list order r, indices (n, 3)) x configurations.  A CTA
// of VM_THREADS threads covers VM_THREADS consecutive configurations, so
// each voxel's row segment is one contiguous read of up to 2 KB; voxels are
// taken VM_BATCH at a time (their rows all in flight), batches interleaved
// over the CTAs along y; one 64-bit atomic per (configuration, CTA).
constexpr int VM_THREADS = 512;
constexpr int VM_BATCH = 16;
constexpr int VM_STAGE = 256;  // voxel indices staged per CTA round

__global__ void __launch_bounds__(VM_THREADS)
query_vm_kernel(const float* __restrict__ field, int64_t C, lsdf_env_grid env, const int32_t* __restrict__ indices,
                const int32_t* __restrict__ counters, int64_t n_list, unsigned long long* keys) {
    __shared__ int64_t s_lin[VM_STAGE];
    const int64_t c = (int64_t)blockIdx.x * VM_THREADS + threadIdx.x;
    const int n_occ = n_list >= 0 ? (int)n_list : counters[0];
    // each thread visits its voxels in increasing list position, so a strict
    // "<" keeps the first occurrence (and -0 == +0); the key is formed once
    float bestv = INFINITY;
    int bestr = -1;
    // this CTA's voxels: batches b0 = blockIdx.y * VM_BATCH + k * stride; their
    // indices are staged first (one round trip), then all row loads stream
    const int stride = gridDim.y * VM_BATCH;
    for (int k0 = 0;; k0 += VM_STAGE / VM_BATCH) {
        const int first = blockIdx.y * VM_BATCH + k0 * stride;
        if (first >= n_occ) break;
        __syncthreads();
        for (int i = threadIdx.x; i < VM_STAGE; i += VM_THREADS) {
            const int r = first + (i / VM_BATCH) * stride + (i % VM_BATCH);
            s_lin[i] = r < n_occ ? ((int64_t)__ldg(indices + 3 * r) * env.dims[1] + __ldg(indices + 3 * r + 1)) *
                                       env.dims[2] + __ldg(indices + 3 * r + 2)
                                 : -1;
        }
        __syncthreads();
        for (int bb = 0; bb < VM_STAGE / VM_BATCH; ++bb) {
            const int b0 = first + bb * stride;
            if (b0 >= n_occ) break;
            float v[VM_BATCH];
#pragma unroll
            for (int j = 0; j < VM_BATCH; ++j) {
                const int64_t lin = s_lin[bb * VM_BATCH + j];
                v[j] = (lin >= 0 && c < C) ? __ldcs(field + lin * C + c) : INFINITY;
            }
#pragma unroll
            for (int j = 0; j < VM_BATCH; ++j) {
                const bool better = v[j] < bestv;  // INFINITY padding never wins
                bestv = better ? v[j] : bestv;
                bestr = better ? b0 + j : bestr;
            }
        }
    }
    if (c < C && bestr >= 0)
        atomicMax(keys + c, ~(((unsigned long long)orderable(bestv) << 32) | (uint32_t)bestr));  // the workspace holds complements (zero = empty)
}

struct LinkParams {
    lsdf_link_grid grids[LSDF_MAX_LINKS];
    const double* R;
    const double* dt;
    const int32_t* anchor;
    int64_t C;
    int32_t n_geo;
    int32_t W[3];
    double e_r;
    const double* P;
    int32_t Wmax;
    const uint32_t* mask_bits;
    lsdf_env_grid env;
    float clamp;
    const int32_t* indices;
    unsigned long long* keys;
    float* d_out;
    int32_t* link_out;
    int32_t* voxel_out;
};

// CTA = 32 configurations x lp link slots (lp = pow2 >= n_geo): thread
// (l, c) evaluates link l at c's winning voxel; the lowest hitting link wins.
__global__ void link_vm_kernel(const __grid_constant__ LinkParams p, int lp_log2) {
    __shared__ unsigned int s_hit[32];
    const int cl = threadIdx.x & 31, l = threadIdx.x >> 5;
    const int64_t c = (int64_t)blockIdx.x * 32 + cl;
    if (l == 0) s_hit[cl] = 0u;
    __syncthreads();
    uint64_t k = ~0ull;
    float d = p.clamp;
    if (c < p.C) {
        k = ~(uint64_t)p.keys[c];
        if (k != ~0ull) d = from_orderable((uint32_t)(k >> 32));
    }
    const bool found = c < p.C && k != ~0ull && d < p.clamp;
    if (found && l < p.n_geo) {
        const int r = (int)(uint32_t)k;
        const int x = p.indices[3 * r], y = p.indices[3 * r + 1], z = p.indices[3 * r + 2];
        const int64_t f = c * p.n_geo + l;
        const int mx = x - p.anchor[f * 3], my = y - p.anchor[f * 3 + 1], mz = z - p.anchor[f * 3 + 2];
        if (mx >= 0 && mx < p.W[0] && my >= 0 && my < p.W[1] && mz >= 0 && mz < p.W[2]) {
            const int cell = mx + p.W[0] * (my + p.W[1] * mz);
            const GridView gv = view_of(p.grids[l]);
            float v = gv.d_far;
            if ((__ldg(p.mask_bits + (cell >> 5)) >> (cell & 31)) & 1u) {
                double R[9], dtinv[3], pt[3];
#pragma unroll
                for (int e = 0; e < 9; ++e) R[e] = p.R[f * 9 + e];
                shift_inverse(R, p.dt + f * 3, p.e_r, dtinv);
                window_point(p.P[mx], p.P[p.Wmax + my], p.P[2 * p.Wmax + mz], R, dtinv, p.e_r, pt);
                v = trilinear_at(gv, pt[0], pt[1], pt[2], LdgLoad{p.grids[l].values_dev});
            }
            if (v == d) atomicOr(&s_hit[cl], 1u << l);
        }
    }
    __syncthreads();
    if (l != 0 || c >= p.C) return;
    p.keys[c] = 0ull;  // re-zero the workspace for the next cycle
    if (!found) {  // nothing below the monitored range (query.py:142-144)
        p.d_out[c] = p.clamp;
        p.link_out[c] = -1;
        p.voxel_out[c] = -1;
        return;
    }
    p.d_out[c] = d;
    p.link_out[c] = s_hit[cl] ? __ffs(s_hit[cl]) - 1 : -1;
    p.voxel_out[c] = (int)(uint32_t)k;
}

}  // namespace

extern "C" int lsdf_materialize_vm(const double* R_geo_dev, const double* dt_geo_dev, const int32_t* anchor_geo_dev,
                                   int64_t C, int32_t n_geo, const lsdf_link_grid* grids, const lsdf_window* window,
                                   const lsdf_env_grid* env, double d_far_global, float* field_dev, void* stream) {
    if (n_geo < 1 || n_geo > LSDF_MAX_LINKS) return fail(LSDF_ERR_VALIDATION, "materialize: bad link count %d", n_geo);
    if (C <= 0) return LSDF_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t V = n_vox(*env);
    fill_f32_kernel<<<148 * 8, 256, 0, s>>>(field_dev, V * C, (float)d_far_global);
    LSDF_TRY(check_launch("fill_f32_kernel"));
    VmParams p{};
    for (int l = 0; l < n_geo; ++l) p.grids[l] = grids[l];
    p.R = R_geo_dev;
    p.dt = dt_geo_dev;
    p.anchor = anchor_geo_dev;
    p.C = C;
    p.n_geo = n_geo;
    for (int a = 0; a < 3; ++a) p.W[a] = window->W[a];
    p.e_r = window->e_r;
    p.P = window->P_dev;
    p.Wmax = window->Wmax;
    p.mask_bits = window->mask_bits_dev;
    p.env = *env;
    p.clamp = (float)d_far_global;
    p.field = field_dev;
    materialize_vm_kernel<<<(unsigned)(C * n_geo), 256, 0, s>>>(p);
    return check_launch("materialize_vm_kernel");
}

extern "C" int lsdf_query_vm(const float* field_dev, const double* R_geo_dev, const double* dt_geo_dev,
                             const int32_t* anchor_geo_dev, int64_t C, int32_t n_geo, const lsdf_link_grid* grids,
                             const lsdf_window* window, const lsdf_env_grid* env, const void* occupancy_dev,
                             const int32_t* indices_dev, int64_t n_list, double d_far_global, void* workspace_dev,
                             float* d_dev,
                             int32_t* link_dev, int32_t* voxel_dev, void* stream) {
    if (n_geo < 1 || n_geo > LSDF_MAX_LINKS) return fail(LSDF_ERR_VALIDATION, "query_vm: bad link count %d", n_geo);
    if (C <= 0) return LSDF_OK;
    cudaStream_t s = (cudaStream_t)stream;
    Occupancy o = carve_occupancy(const_cast<void*>(occupancy_dev), *env);
    unsigned long long* keys = (unsigned long long*)workspace_dev;
    const int64_t rows = n_list >= 0 ? n_list : n_vox(*env);  // device count: bound by the grid size
    if (rows >= 2147483647LL) return fail(LSDF_ERR_UNSUPPORTED, "query_vm: obstacle list too long");
    const int64_t gx = (C + VM_THREADS - 1) / VM_THREADS;
    int64_t gy = (148LL * 2 + gx - 1) / gx;  // about 2 CTAs per SM in total
    const int64_t batches = (rows + VM_BATCH - 1) / VM_BATCH;
    gy = gy < 1 ? 1 : (gy > batches ? (batches > 0 ? batches : 1) : gy);
    const dim3 grid((unsigned)gx, (unsigned)gy);
    query_vm_kernel<<<grid, VM_THREADS, 0, s>>>(field_dev, C, *env, indices_dev, o.counters, n_list, keys);
    LSDF_TRY(check_launch("query_vm_kernel"));
    LinkParams p{};
    for (int l = 0; l < n_geo; ++l) p.grids[l] = grids[l];
    p.R = R_geo_dev;
    p.dt = dt_geo_dev;
    p.anchor = anchor_geo_dev;
    p.C = C;
    p.n_geo = n_geo;
    for (int a = 0; a < 3; ++a) p.W[a] = window->W[a];
    p.e_r = window->e_r;
    p.P = window->P_dev;
    p.Wmax = window->Wmax;
    p.mask_bits = window->mask_bits_dev;
    p.env = *env;
    p.clamp = (float)d_far_global;
    p.indices = indices_dev;
    p.keys = keys;
    p.d_out = d_dev;
    p.link_out = link_dev;
    p.voxel_out = voxel_dev;
    int lp_log2 = 0;
    while ((1 << lp_log2) < n_geo) ++lp_log2;
    link_vm_kernel<<<(unsigned)((C + 31) / 32), 32 << lp_log2, 0, s>>>(p, lp_log2);
    return check_launch("link_vm_kernel");
}
