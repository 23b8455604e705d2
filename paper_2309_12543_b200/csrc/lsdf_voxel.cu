// lsdf_voxel.cu — obstacle voxelization (query.py:106-125, grids.py:93-113).
//
// voxel_scatter_kernel: one thread per point, fp64 floor((p + e) / r) exactly
//   as numpy, clipped; each CTA merges its points in a shared-memory bitmap
//   and ORs the touched words into the global one.
// prefix_only_kernel: the exclusive popcount prefix per word: rank(voxel) =
//   prefix[w] + popc(word & below) is its position in np.unique(axis=0) order.
// voxel_compact_kernel: optional, one thread per voxel, writes the sorted
//   index list (the ObstacleVoxelSet.indices the API returns) and posgrid.
#include <cub/block/block_scan.cuh>
#include <cstdlib>

#include "lsdf_device.cuh"

using namespace lsdf;

namespace {

constexpr int SCAN_THREADS = 1024;
constexpr int SCATTER_THREADS = 1024;
constexpr int64_t PRIVATE_WORDS_MAX = 12288;  // 48 KiB of shared bitmap

__device__ void prefix_scan_block(const uint32_t* bitmap, int64_t n_words, int32_t* prefix, int32_t* counters) {
    using Scan = cub::BlockScan<int, SCAN_THREADS>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    // tiles of SCAN_THREADS * 4 words; each thread owns 4 consecutive words
    for (int64_t base = 0; base < n_words; base += (int64_t)SCAN_THREADS * 4) {
        const int64_t w0 = base + threadIdx.x * 4;
        int c[4], s = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            c[k] = (w0 + k < n_words) ? __popc(__ldcg(bitmap + w0 + k)) : 0;
            s += c[k];
        }
        int excl, total;
        Scan(tmp).ExclusiveSum(s, excl, total);
        const int start = carry + excl;
        int run = start;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (w0 + k < n_words) prefix[w0 + k] = run;
            run += c[k];
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        counters[0] = carry;
        counters[2] = 0;  // reset the ticket for the next launch (graph replays)
    }
}

// floor((p + e) / r) exactly as numpy: correctly rounded quotient via
// q0 = x * RN(1/r) plus one FMA residual step (Markstein), then floor
// (q >= 0 here: the magic-number floor of floor_small, no conversion).
__device__ __forceinline__ int voxel_floor(double p, double e, double r, double rinv) {
    const double x = __dadd_rn(p, e);
    const double q0 = __dmul_rn(x, rinv);
    const double q = __fma_rn(__fma_rn(-q0, r, x), rinv, q0);
    double fl;
    return floor_small(q, fl);
}

// One thread per point.  With a small grid the CTA first merges its points
// into a shared-memory copy of the bitmap (fast shared atomics), then ORs the
// non-empty words into the global bitmap: a dense human blob costs one global
// atomic per touched word per CTA instead of one per point.
template <typename T, bool PRIVATE>
__global__ void __launch_bounds__(SCATTER_THREADS)
voxel_scatter_kernel(const T* __restrict__ pts, int64_t N, lsdf_env_grid env, double rx, double ry, double rz,
                     uint32_t* bitmap, int32_t* counters, int64_t n_words, uint32_t* bricks, int32_t nby,
                     int32_t n_cols, int32_t use_vec) {
    extern __shared__ uint32_t s_bits[];
    uint32_t* s_bricks = s_bits + n_words;  // brick columns (PRIVATE)
    if (PRIVATE) {  // (the allocation is rounded up to whole 16-B groups)
        uint4* s4 = (uint4*)s_bits;
        const int n4 = (int)((n_words + n_cols + 3) >> 2);
        for (int w = threadIdx.x; w < n4; w += blockDim.x) s4[w] = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
    }
    // grid-stride: a persistent grid of a few CTAs per SM amortises the
    // private bitmap's clear and merge over many points.  f32 clouds: each
    // thread takes VEC = 4 consecutive points per step as three 16-B loads
    // (48 B, coalesced across the warp) when the buffer is 16-B aligned.
    constexpr int VEC = sizeof(T) == 4 ? 4 : 1;
    const bool vec = VEC > 1 && use_vec;
    const int per = vec ? VEC : 1;
    int dropped_count = 0;
    for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x) * per; i0 < N; i0 += (int64_t)gridDim.x * blockDim.x * per) {
      const int64_t ib = i0 + (int64_t)threadIdx.x * per;
      float buf[12];
      if (vec && ib + VEC <= N) {
          const float4* src = (const float4*)(pts + 3 * ib);
#pragma unroll
          for (int k = 0; k < 3; ++k) {
              const float4 v = __ldcs(src + k);  // streamed once: evict-first
              buf[4 * k] = v.x;
              buf[4 * k + 1] = v.y;
              buf[4 * k + 2] = v.z;
              buf[4 * k + 3] = v.w;
          }
      }
      for (int u = 0; u < per; ++u) {
        const int64_t i = ib + u;
        bool dropped = false;
        if (i < N) {
            double x, y, z;
            if (vec && ib + VEC <= N) {
                x = (double)buf[3 * u];
                y = (double)buf[3 * u + 1];
                z = (double)buf[3 * u + 2];
            } else {
                x = (double)pts[3 * i];
                y = (double)pts[3 * i + 1];
                z = (double)pts[3 * i + 2];
            }
            const double ex = env.extent[0], ey = env.extent[1], ez = env.extent[2];
            // query.py:112: keep -e <= p < e on every axis (NaN fails the test -> dropped)
            const bool inside = (x >= -ex) && (x < ex) && (y >= -ey) && (y < ey) && (z >= -ez) && (z < ez);
            if (inside) {
                // inside => 0 <= (p + e) / r, so the exact floor fits 32 bits
                int ix = voxel_floor(x, ex, env.resolution[0], rx);
                int iy = voxel_floor(y, ey, env.resolution[1], ry);
                int iz = voxel_floor(z, ez, env.resolution[2], rz);
                ix = ix > env.dims[0] - 1 ? env.dims[0] - 1 : ix;  // grids.py:111 clip
                iy = iy > env.dims[1] - 1 ? env.dims[1] - 1 : iy;
                iz = iz > env.dims[2] - 1 ? env.dims[2] - 1 : iz;
                const uint32_t lin = ((uint32_t)ix * (uint32_t)env.dims[1] + (uint32_t)iy) * (uint32_t)env.dims[2] +
                                     (uint32_t)iz;
                const int col = (ix >> BRICK_LOG2) * nby + (iy >> BRICK_LOG2);
                const uint32_t zb = 1u << (iz >> BRICK_LOG2);
                if (PRIVATE) {
                    const uint32_t bit = 1u << (lin & 31);
                    // a voxel marks its brick once per CTA (dense clouds repeat voxels)
                    if (!(atomicOr(s_bits + (lin >> 5), bit) & bit) && n_cols) atomicOr(s_bricks + col, zb);
                } else {
                    atomicOr(bitmap + (lin >> 5), 1u << (lin & 31));
                    if (n_cols) atomicOr(bricks + col, zb);
                }
            } else {
                dropped = true;
            }
        }
        dropped_count += __popc(__ballot_sync(FULL_MASK, dropped));
      }
    }
    if ((threadIdx.x & 31) == 0 && dropped_count) atomicAdd(&counters[1], dropped_count);
    if (PRIVATE) {
        __syncthreads();
        const uint4* s4 = (const uint4*)s_bits;
        const int n4 = (int)(n_words >> 2);
        for (int w4 = threadIdx.x; w4 < n4; w4 += blockDim.x) {
            const uint4 v = s4[w4];
            uint32_t* g = bitmap + 4 * w4;
            if (v.x) atomicOr(g, v.x);
            if (v.y) atomicOr(g + 1, v.y);
            if (v.z) atomicOr(g + 2, v.z);
            if (v.w) atomicOr(g + 3, v.w);
        }
        for (int w = 4 * n4 + threadIdx.x; w < (int)n_words; w += blockDim.x) {
            const uint32_t v = s_bits[w];
            if (v) atomicOr(bitmap + w, v);
        }
        for (int w = threadIdx.x; w < n_cols; w += blockDim.x) {
            const uint32_t v = s_bricks[w];
            if (v) atomicOr(bricks + w, v);
        }
    }
}

// brick column bit of an occupied voxel (linear C-order index)
__device__ __forceinline__ void mark_brick(uint32_t* bricks, const lsdf_env_grid& env, int32_t nby, int64_t lin) {
    const int64_t nyz = (int64_t)env.dims[1] * env.dims[2];
    const int ix = (int)(lin / nyz), iy = (int)((lin / env.dims[2]) % env.dims[1]), iz = (int)(lin % env.dims[2]);
    atomicOr(bricks + (ix >> BRICK_LOG2) * nby + (iy >> BRICK_LOG2), 1u << (iz >> BRICK_LOG2));
}

// OR of n_parts partial bitmaps (n_parts, n_words) into the occupancy bitmap;
// thread 0 also sums the parts' dropped-point counters.
__global__ void merge_bitmaps_kernel(const uint32_t* __restrict__ parts, int32_t n_parts, int64_t n_words,
                                     const int32_t* __restrict__ dropped, int64_t dropped_stride, uint32_t* bitmap,
                                     int32_t* counters, lsdf_env_grid env, uint32_t* bricks, int32_t nby) {
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n_words; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = 0;
        for (int k = 0; k < n_parts; ++k) v |= __ldg(parts + k * n_words + w);
        bitmap[w] = v;
        for (uint32_t b = v; bricks != nullptr && b; b &= b - 1) mark_brick(bricks, env, nby, w * 32 + __ffs(b) - 1);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int32_t total = 0;
        for (int k = 0; k < n_parts; ++k) total += dropped[k * dropped_stride];
        counters[1] = total;
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) prefix_only_kernel(const uint32_t* bitmap, int64_t n_words,
                                                                    int32_t* prefix, int32_t* counters) {
    prefix_scan_block(bitmap, n_words, prefix, counters);
}

// one thread per voxel (bit): an occupied voxel's rank is prefix[w] +
// popc(word & below), so every write is independent (no per-word loop)
__global__ void voxel_compact_kernel(const uint32_t* __restrict__ bitmap, const int32_t* __restrict__ prefix,
                                     int64_t n_words, lsdf_env_grid env, int32_t* posgrid, int32_t* indices) {
    const int64_t lin = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (lin >= n_words * 32) return;
    const uint32_t word = __ldg(bitmap + (lin >> 5));
    const uint32_t bit = 1u << (lin & 31);
    if (!(word & bit)) return;
    const int rank = __ldg(prefix + (lin >> 5)) + __popc(word & (bit - 1u));
    posgrid[lin] = rank;
    if (indices != nullptr) {
        const int64_t nyz = (int64_t)env.dims[1] * env.dims[2];
        indices[3 * (int64_t)rank] = (int32_t)(lin / nyz);
        indices[3 * (int64_t)rank + 1] = (int32_t)((lin / env.dims[2]) % env.dims[1]);
        indices[3 * (int64_t)rank + 2] = (int32_t)(lin % env.dims[2]);
    }
}

__global__ void occ_from_indices_kernel(const int32_t* idx, int64_t N, lsdf_env_grid env, uint32_t* bitmap,
                                        int32_t* posgrid, int mode, uint32_t* bricks, int32_t nby) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int64_t lin = ((int64_t)idx[3 * i] * env.dims[1] + idx[3 * i + 1]) * env.dims[2] + idx[3 * i + 2];
    if (mode == 0) {  // sorted unique: position == list index == rank
        posgrid[lin] = (int32_t)i;
        atomicOr(bitmap + (lin >> 5), 1u << (lin & 31));
        if (bricks != nullptr) mark_brick(bricks, env, nby, lin);
    } else if (mode == 1) {  // general, pass 1: reset touched entries
        posgrid[lin] = 0x7fffffff;
    } else {  // general, pass 2: first occurrence wins (numpy argmin semantics)
        atomicMin(posgrid + lin, (int32_t)i);
        atomicOr(bitmap + (lin >> 5), 1u << (lin & 31));
        if (bricks != nullptr) mark_brick(bricks, env, nby, lin);
    }
}

__global__ void voxel_index_kernel(const double* pts, int64_t N, lsdf_env_grid env, int32_t* out, int32_t* flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    bool bad = false;
    for (int a = 0; a < 3; ++a) {
        const double x = pts[3 * i + a];
        if (!(x >= -env.extent[a] && x < env.extent[a])) bad = true;
        const double f = floor(DDIV(DADD(x, env.extent[a]), env.resolution[a]));
        int64_t j = (f == f) ? (int64_t)f : 0;
        j = j < 0 ? 0 : (j > env.dims[a] - 1 ? env.dims[a] - 1 : j);
        out[3 * i + a] = (int32_t)j;
    }
    if (bad) atomicAdd(flags, 1);
}

}  // namespace

extern "C" int64_t lsdf_occupancy_bytes(const lsdf_env_grid* env) { return occupancy_bytes(*env); }

namespace {

// memset + scatter: the bitmap (and the dropped-point counter) of a cloud
int scatter_bitmap(const void* points_dev, int32_t points_f32, int64_t N, const lsdf_env_grid* env, Occupancy& o,
                   void* occupancy_dev, cudaStream_t s) {
    LSDF_TRY(check_cuda(cudaMemsetAsync(occupancy_dev, 0, occupancy_clear_bytes(o), s), "voxelize memset"));
    if (N <= 0) return LSDF_OK;
    const int32_t n_cols = o.bricks_ok ? o.nbx * o.nby : 0;
    const double rx = 1.0 / env->resolution[0], ry = 1.0 / env->resolution[1], rz = 1.0 / env->resolution[2];
    // CTA-private shared bitmaps (a dense blob costs one global atomic per
    // touched word per CTA; measured: global atomics straight away, or
    // smaller CTAs, are slower even at 100k points), grid-stride over at most
    // two CTAs per SM so large clouds amortise the clear and merge
    const bool priv = o.n_words + n_cols <= PRIVATE_WORDS_MAX;
    // small clouds: 256-thread CTAs, so every SM issues loads (zero-copy clouds
    // come over PCIe: more SMs with reads in flight, config 2 host to host
    // 56.6 -> 50.8 us); large clouds: 1024-thread CTAs amortise the private
    // bitmap's clear and merge
    const int n_sm = sm_count();
    static const int t_threads = [] { const char* v = getenv("LSDF_TUNE_VOXTHREADS"); return v && *v ? atoi(v) : 0; }();
    const unsigned threads = t_threads > 0 ? (unsigned)t_threads
                                           : (N >= n_sm * 2LL * SCATTER_THREADS ? SCATTER_THREADS : 256u);
    // 4 points per thread (float4 loads) only when that still fills the GPU:
    // small clouds keep one point per thread (more CTAs in flight)
    static const int t_vec = [] { const char* v = getenv("LSDF_TUNE_VOXVEC"); return v && *v ? atoi(v) : -1; }();
    const bool want_vec = t_vec >= 0 ? t_vec != 0 : N >= n_sm * 2LL * SCATTER_THREADS * 2;
    const int64_t per_thread = (want_vec && points_f32 && (((uintptr_t)points_dev) & 15) == 0) ? 4 : 1;
    const unsigned want = grid_for((N + per_thread - 1) / per_thread, threads);
    static const int t_blocks = [] { const char* v = getenv("LSDF_TUNE_VOXBLOCKS"); return v && *v ? atoi(v) : 0; }();
    // 1,024-thread CTAs fit once per SM (registers): one wave, each striding
    // over more points, instead of 1.7 waves (config 4: +1.2 %)
    const unsigned cap = t_blocks > 0 ? (unsigned)t_blocks : (unsigned)(threads == SCATTER_THREADS ? n_sm : 2 * n_sm);
    const unsigned blocks = want < cap ? want : cap;  // (more CTAs: more private-bitmap merges)
    const size_t smem = priv ? (size_t)((o.n_words + n_cols + 3) & ~3LL) * 4 : 0;
    if (points_f32) {
        if (priv)
            voxel_scatter_kernel<float, true><<<blocks, threads, smem, s>>>(
                (const float*)points_dev, N, *env, rx, ry, rz, o.bitmap, o.counters, o.n_words, o.bricks, o.nby, n_cols, (int)(per_thread > 1));
        else
            voxel_scatter_kernel<float, false><<<blocks, threads, 0, s>>>(
                (const float*)points_dev, N, *env, rx, ry, rz, o.bitmap, o.counters, o.n_words, o.bricks, o.nby, n_cols, (int)(per_thread > 1));
    } else {
        if (priv)
            voxel_scatter_kernel<double, true><<<blocks, threads, smem, s>>>(
                (const double*)points_dev, N, *env, rx, ry, rz, o.bitmap, o.counters, o.n_words, o.bricks, o.nby, n_cols, (int)(per_thread > 1));
        else
            voxel_scatter_kernel<double, false><<<blocks, threads, 0, s>>>(
                (const double*)points_dev, N, *env, rx, ry, rz, o.bitmap, o.counters, o.n_words, o.bricks, o.nby, n_cols, (int)(per_thread > 1));
    }
    return check_launch("voxel_scatter_kernel");
}

}  // namespace

extern "C" int lsdf_voxelize(const void* points_dev, int32_t points_f32, int64_t N, const lsdf_env_grid* env,
                             void* occupancy_dev, int32_t* indices_dev, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    Occupancy o = carve_occupancy(occupancy_dev, *env);
    LSDF_TRY(scatter_bitmap(points_dev, points_f32, N, env, o, occupancy_dev, s));
    prefix_only_kernel<<<1, SCAN_THREADS, 0, s>>>(o.bitmap, o.n_words, o.prefix, o.counters);
    LSDF_TRY(check_launch("prefix_only_kernel"));
    if (indices_dev == nullptr) return LSDF_OK;  // hot path: the query only needs bitmap + prefix
    voxel_compact_kernel<<<grid_for(o.n_words * 32, 256), 256, 0, s>>>(o.bitmap, o.prefix, o.n_words, *env, o.posgrid,
                                                                    indices_dev);
    return check_launch("voxel_compact_kernel");
}

extern "C" int lsdf_voxelize_bitmap(const void* points_dev, int32_t points_f32, int64_t N, const lsdf_env_grid* env,
                                    void* occupancy_dev, void* stream) {
    Occupancy o = carve_occupancy(occupancy_dev, *env);
    return scatter_bitmap(points_dev, points_f32, N, env, o, occupancy_dev, (cudaStream_t)stream);
}

extern "C" int lsdf_occupancy_prefix(const lsdf_env_grid* env, void* occupancy_dev, void* stream) {
    Occupancy o = carve_occupancy(occupancy_dev, *env);
    prefix_only_kernel<<<1, SCAN_THREADS, 0, (cudaStream_t)stream>>>(o.bitmap, o.n_words, o.prefix, o.counters);
    return check_launch("prefix_only_kernel");
}

extern "C" int lsdf_occupancy_merge(const uint32_t* parts_dev, int32_t n_parts, const int32_t* dropped_dev,
                                    int64_t dropped_stride, const lsdf_env_grid* env, void* occupancy_dev,
                                    void* stream) {
    if (n_parts < 1) return fail(LSDF_ERR_VALIDATION, "occupancy merge: %d parts", n_parts);
    cudaStream_t s = (cudaStream_t)stream;
    Occupancy o = carve_occupancy(occupancy_dev, *env);
    if (o.bricks_ok)
        LSDF_TRY(check_cuda(cudaMemsetAsync(o.bricks, 0, (size_t)o.nbx * o.nby * 4, s), "brick columns memset"));
    merge_bitmaps_kernel<<<grid_for(o.n_words, 256), 256, 0, s>>>(parts_dev, n_parts, o.n_words, dropped_dev,
                                                                   dropped_stride, o.bitmap, o.counters, *env,
                                                                   o.bricks_ok ? o.bricks : nullptr, o.nby);
    LSDF_TRY(check_launch("merge_bitmaps_kernel"));
    prefix_only_kernel<<<1, SCAN_THREADS, 0, s>>>(o.bitmap, o.n_words, o.prefix, o.counters);
    return check_launch("prefix_only_kernel");
}

extern "C" int lsdf_occupancy_from_indices(const int32_t* indices_dev, int64_t N, int32_t sorted_unique,
                                           const lsdf_env_grid* env, void* occupancy_dev, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    Occupancy o = carve_occupancy(occupancy_dev, *env);
    LSDF_TRY(check_cuda(cudaMemsetAsync(occupancy_dev, 0, occupancy_clear_bytes(o), s), "occupancy memset"));
    uint32_t* bricks = o.bricks_ok ? o.bricks : nullptr;
    if (N > 0) {
        if (sorted_unique) {
            occ_from_indices_kernel<<<grid_for(N, 256), 256, 0, s>>>(indices_dev, N, *env, o.bitmap, o.posgrid, 0, bricks, o.nby);
            LSDF_TRY(check_launch("occ_from_indices_kernel"));
        } else {
            occ_from_indices_kernel<<<grid_for(N, 256), 256, 0, s>>>(indices_dev, N, *env, o.bitmap, o.posgrid, 1, bricks, o.nby);
            LSDF_TRY(check_launch("occ_from_indices_kernel"));
            occ_from_indices_kernel<<<grid_for(N, 256), 256, 0, s>>>(indices_dev, N, *env, o.bitmap, o.posgrid, 2, bricks, o.nby);
            LSDF_TRY(check_launch("occ_from_indices_kernel"));
        }
    }
    prefix_only_kernel<<<1, SCAN_THREADS, 0, s>>>(o.bitmap, o.n_words, o.prefix, o.counters);
    return check_launch("prefix_only_kernel");
}

extern "C" int lsdf_voxel_index(const double* points_dev, int64_t N, const lsdf_env_grid* env, int32_t* indices_dev,
                                int32_t* flags_dev, void* stream) {
    if (N <= 0) return LSDF_OK;
    voxel_index_kernel<<<grid_for(N, 256), 256, 0, (cudaStream_t)stream>>>(points_dev, N, *env, indices_dev,
                                                                           flags_dev);
    return check_launch("voxel_index_kernel");
}
