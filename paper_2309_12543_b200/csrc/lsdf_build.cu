// lsdf_build.cu — stage 2a: exact link-SDF precompute (meshes.py:64-82, 144-371).
//
// Primitives: one thread per cell, fp64 analytic distance, f32 store
// (fp64-issue bound: the distance with the reference's operation order is
// ~100 instructions per 4 B written).
// Meshes: exact per-(cell, triangle) tests (the spec rejects propagation
// transforms) with conservative box culling.  A CTA owns a
// compact 8 x 4 x 4 block of cells and streams the triangle list through
// shared memory in tiles, nearest tile first, skipping tiles / triangles that
// provably cannot change any of its cells' results; the per-pair
// closest-point and ray-crossing tests run in fp64 with the reference's
// operation order.
#include "lsdf_common.cuh"
#include "lsdf_math.cuh"

using namespace lsdf;

namespace {

__device__ __forceinline__ void cell_center(int64_t cell, const int32_t* dims, const double* ext, const double* res,
                                            double* p) {
    // 32-bit index arithmetic (grids stay far below 2^32 cells; 64-bit
    // division is a long instruction sequence)
    const uint32_t c = (uint32_t)cell, d0 = (uint32_t)dims[0], d1 = (uint32_t)dims[1];
    const uint32_t t = c / d0;
    const uint32_t ix = c - t * d0, iy = t % d1, iz = t / d1;
    // meshes.py:356-358: -e + (i + 0.5) * r
    p[0] = DADD(-ext[0], DMUL(DADD((double)ix, 0.5), res[0]));
    p[1] = DADD(-ext[1], DMUL(DADD((double)iy, 0.5), res[1]));
    p[2] = DADD(-ext[2], DMUL(DADD((double)iz, 0.5), res[2]));
}

struct BuildParams {
    int32_t kind;
    double prm[8];
    double ext[3], res[3];
    int32_t dims[3];
};

// grid (ceil(nx / 128), ny, nz): one x-row segment per CTA, no index division
template <int KIND>
__global__ void __launch_bounds__(128) build_primitive_kernel(const __grid_constant__ BuildParams p, float* out) {
    const int ix = blockIdx.x * 128 + threadIdx.x;
    if (ix >= p.dims[0]) return;
    const uint32_t iy = blockIdx.y, iz = blockIdx.z, row = iz * (uint32_t)p.dims[1] + iy;
    // meshes.py:356-358: -e + (i + 0.5) * r
    const double x = DADD(-p.ext[0], DMUL(DADD((double)ix, 0.5), p.res[0]));
    const double y = DADD(-p.ext[1], DMUL(DADD((double)iy, 0.5), p.res[1]));
    const double z = DADD(-p.ext[2], DMUL(DADD((double)iz, 0.5), p.res[2]));
    out[(int64_t)row * p.dims[0] + ix] = (float)primitive_at(KIND, p.prm, x, y, z);
}

__global__ void primitive_points_kernel(int32_t kind, BuildParams p, const double* pts, int64_t n, double* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = primitive_at(kind, p.prm, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
}

// meshes.py:249-256
__constant__ double c_dirs[4][3] = {
    {0.577350269, 0.577350269, 0.577350269},
    {0.267261242, 0.534522484, 0.801783726},
    {-0.455842306, 0.569802882, 0.683763459},
    {0.816496581, -0.408248290, 0.408248290},
};

// Per-(direction, triangle) ray constants, meshes.py:265-271.
__global__ void ray_setup_kernel(const double* tri, int32_t n_tri, RayTri* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 4 * n_tri) return;
    const int d = i / n_tri, t = i % n_tri;
    const double* a = tri + 9 * t;
    RayTri r;
    for (int k = 0; k < 3; ++k) {
        r.a[k] = a[k];
        r.e1[k] = DSUB(a[3 + k], a[k]);
        r.e2[k] = DSUB(a[6 + k], a[k]);
    }
    cross3(c_dirs[d], r.e2, r.h);
    const double det = dot3(r.e1[0], r.e1[1], r.e1[2], r.h[0], r.h[1], r.h[2]);
    r.parallel = fabs(det) < 1e-12;
    r.det = r.parallel ? 1.0 : det;
    out[i] = r;
}

constexpr int MESH_CELLS = 128;  // cells per CTA (one per thread)
constexpr int MESH_TILE = 128;   // triangles per shared-memory tile

struct MeshParams {
    const double* tri;
    const RayTri* ray;
    int32_t n_tri, is_signed;
    double ext[3], res[3];
    int32_t dims[3];
    const double* pts;  // explicit points instead of cell centres (or null)
    int64_t n;
    float* out_f;
    double* out_d;
};

// Per-triangle and per-tile (MESH_TILE triangles) axis-aligned bounds, fp64:
// [min x, min y, min z, max x, max y, max z].
__global__ void mesh_bounds_kernel(const double* __restrict__ tri, int32_t n_tri, double* tri_bb, double* tile_bb) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_tri) {
        const double* v = tri + 9 * (int64_t)t;
        for (int a = 0; a < 3; ++a) {
            tri_bb[6 * (int64_t)t + a] = fmin(v[a], fmin(v[3 + a], v[6 + a]));
            tri_bb[6 * (int64_t)t + 3 + a] = fmax(v[a], fmax(v[3 + a], v[6 + a]));
        }
    }
    const int n_tiles = (n_tri + MESH_TILE - 1) / MESH_TILE;
    if (t < n_tiles) {
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        const int end = (t + 1) * MESH_TILE < n_tri ? (t + 1) * MESH_TILE : n_tri;
        for (int k = t * MESH_TILE; k < end; ++k)
            for (int a = 0; a < 9; ++a) {
                const double x = tri[9 * (int64_t)k + a];
                lo[a % 3] = fmin(lo[a % 3], x);
                hi[a % 3] = fmax(hi[a % 3], x);
            }
        for (int a = 0; a < 3; ++a) {
            tile_bb[6 * t + a] = lo[a];
            tile_bb[6 * t + 3 + a] = hi[a];
        }
    }
}

// squared gap between two boxes (0 when they overlap); a lower bound of the
// squared distance between any point of one and any point of the other
__device__ __forceinline__ double box_gap2(const double* A, const double* B) {
    double g2 = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double g = fmax(0.0, fmax(B[a] - A[3 + a], A[a] - B[3 + a]));
        g2 += g * g;
    }
    return g2;
}

// no point of box B can be hit by a ray p + t dir, t > 0, from any p in box A
// (B lies behind A along an axis the direction advances on), with slack
__device__ __forceinline__ bool behind(const double* A, const double* B, const double* dir) {
    constexpr double slack = 1e-6;
    bool out = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        out |= (dir[a] > 0.0) & (B[3 + a] < A[a] - slack);
        out |= (dir[a] < 0.0) & (B[a] > A[3 + a] + slack);
    }
    return out;
}

// Exact mesh SDF with conservative culling.  A CTA owns a compact 8 x 4 x 4
// block of cells (or 128 consecutive explicit points); its box bounds every
// point.  Unsigned distance: tiles are visited nearest-box first, and a tile
// or triangle whose box gap to the cell box exceeds the largest running
// minimum of the CTA (squared, with a relative margin far above the fp64
// rounding of closest_sq) cannot be any cell's minimum and is skipped.  Ray
// parity: a triangle whose box lies behind the cell box along an axis the
// ray advances on cannot give a hit with t > 0 (ray_cross returns 0 for it,
// never "suspect").  Both leave every result identical to the full
// brute force (meshes.py:217-246, 259-305).
template <bool CELLS>
__global__ void __launch_bounds__(MESH_CELLS) mesh_kernel(const __grid_constant__ MeshParams p,
                                                          const double* __restrict__ tri_bb,
                                                          const double* __restrict__ tile_bb) {
    __shared__ double s_tri[MESH_TILE * 9];
    __shared__ RayTri s_ray[MESH_TILE];
    __shared__ unsigned char s_keep[MESH_TILE];
    __shared__ double s_blk[6];
    __shared__ double s_wbox[MESH_CELLS / 32][6];
    __shared__ unsigned long long s_key;
    __shared__ unsigned long long s_maxbest;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int64_t i;
    bool active;
    double pt[3] = {0.0, 0.0, 0.0};
    if (CELLS) {
        const int ix = blockIdx.x * 8 + (tid & 7), iy = blockIdx.y * 4 + ((tid >> 3) & 3), iz = blockIdx.z * 4 + (tid >> 5);
        active = ix < p.dims[0] && iy < p.dims[1] && iz < p.dims[2];
        i = ix + (int64_t)p.dims[0] * (iy + (int64_t)p.dims[1] * iz);
        if (active) {  // meshes.py:356-358: -e + (i + 0.5) * r
            pt[0] = DADD(-p.ext[0], DMUL(DADD((double)ix, 0.5), p.res[0]));
            pt[1] = DADD(-p.ext[1], DMUL(DADD((double)iy, 0.5), p.res[1]));
            pt[2] = DADD(-p.ext[2], DMUL(DADD((double)iz, 0.5), p.res[2]));
        }
    } else {
        i = (int64_t)blockIdx.x * MESH_CELLS + tid;
        active = i < p.n;
        if (active)
            for (int a = 0; a < 3; ++a) pt[a] = p.pts[3 * i + a];
    }
    // the CTA's point box
    {
        double lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
            lo[a] = active ? pt[a] : INFINITY;
            hi[a] = active ? pt[a] : -INFINITY;
        }
        for (int o = 16; o; o >>= 1)
            for (int a = 0; a < 3; ++a) {
                lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
                hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
            }
        if (lane == 0)
            for (int a = 0; a < 3; ++a) {
                s_wbox[warp][a] = lo[a];
                s_wbox[warp][3 + a] = hi[a];
            }
        if (tid == 0) s_key = ~0ull;
        __syncthreads();
        if (tid < 6) {
            double v = s_wbox[0][tid];
            for (int w = 1; w < MESH_CELLS / 32; ++w) v = tid < 3 ? fmin(v, s_wbox[w][tid]) : fmax(v, s_wbox[w][tid]);
            s_blk[tid] = v;
        }
        __syncthreads();
    }
    const int n_tiles = (p.n_tri + MESH_TILE - 1) / MESH_TILE;
    // nearest tile first (box gap, ties to the lower index)
    for (int t = tid; t < n_tiles; t += MESH_CELLS) {
        const float g = (float)box_gap2(s_blk, tile_bb + 6 * t);
        atomicMin(&s_key, ((unsigned long long)__float_as_uint(g) << 32) | (unsigned)t);
    }
    __syncthreads();
    const int first = (int)(s_key & 0xffffffffu);
    // exact unsigned distance: min over every triangle (meshes.py:217-246)
    double best = INFINITY;
    double maxbest = INFINITY;  // the CTA's largest running minimum (uniform)
    for (int k = 0; k < n_tiles; ++k) {
        const int tile = first + k < n_tiles ? first + k : first + k - n_tiles;
        if (box_gap2(s_blk, tile_bb + 6 * tile) > maxbest * (1.0 + 1e-9)) continue;  // uniform
        const int t0 = tile * MESH_TILE;
        const int nt = p.n_tri - t0 < MESH_TILE ? p.n_tri - t0 : MESH_TILE;
        __syncthreads();
        for (int q = tid; q < nt * 9; q += MESH_CELLS) s_tri[q] = p.tri[(int64_t)t0 * 9 + q];
        for (int q = tid; q < nt; q += MESH_CELLS)
            s_keep[q] = box_gap2(s_blk, tri_bb + 6 * (int64_t)(t0 + q)) <= maxbest * (1.0 + 1e-9);
        if (tid == 0) s_maxbest = 0ull;
        __syncthreads();
        if (active)
            for (int t = 0; t < nt; ++t) {
                if (!s_keep[t]) continue;
                const double* tr = s_tri + 9 * t;
                const double d2 = closest_sq(pt, tr, tr + 3, tr + 6);
                best = d2 < best ? d2 : best;
            }
        // non-negative doubles order like their bits
        unsigned long long mb = active ? (unsigned long long)__double_as_longlong(best) : 0ull;
        for (int o = 16; o; o >>= 1) {
            const unsigned long long u = __shfl_xor_sync(0xffffffffu, mb, o);
            mb = u > mb ? u : mb;
        }
        if (lane == 0) atomicMax(&s_maxbest, mb);
        __syncthreads();
        maxbest = __longlong_as_double((long long)s_maxbest);
    }
    double d = DSQRT(best);
    if (p.is_signed) {
        // ray parity, retried along the backup directions for suspect points
        bool inside = false, pending = active;
        for (int dir = 0; dir < 4; ++dir) {
            if (!__syncthreads_or(pending)) break;
            int count = 0;
            bool suspect = false;
            for (int tile = 0; tile < n_tiles; ++tile) {
                if (behind(s_blk, tile_bb + 6 * tile, c_dirs[dir])) continue;  // uniform
                const int t0 = tile * MESH_TILE;
                const int nt = p.n_tri - t0 < MESH_TILE ? p.n_tri - t0 : MESH_TILE;
                __syncthreads();
                for (int q = tid; q < nt; q += MESH_CELLS) {
                    s_ray[q] = p.ray[(int64_t)dir * p.n_tri + t0 + q];
                    s_keep[q] = !behind(s_blk, tri_bb + 6 * (int64_t)(t0 + q), c_dirs[dir]);
                }
                __syncthreads();
                if (pending)
                    for (int t = 0; t < nt; ++t) {
                        if (!s_keep[t]) continue;
                        const int h = ray_cross(pt, s_ray[t], c_dirs[dir]);
                        count += h != 0;
                        suspect |= h == 2;
                    }
            }
            if (pending && !suspect) {
                inside = count & 1;
                pending = false;
            }
        }
        // points suspect along all four directions stay "outside" (meshes.py:303-304)
        if (inside) d = -d;
    }
    if (active) {
        if (p.out_f) p.out_f[i] = (float)d;
        if (p.out_d) p.out_d[i] = d;
    }
}

int launch_mesh(MeshParams& p, cudaStream_t s) {
    RayTri* ray = nullptr;
    const int n_tiles = (p.n_tri + MESH_TILE - 1) / MESH_TILE;
    double* bb = nullptr;  // [n_tri * 6 | n_tiles * 6]
    LSDF_TRY(check_cuda(cudaMallocAsync((void**)&bb, sizeof(double) * 6 * ((size_t)p.n_tri + n_tiles), s),
                        "mesh bounds alloc"));
    mesh_bounds_kernel<<<grid_for(p.n_tri, 128), 128, 0, s>>>(p.tri, p.n_tri, bb, bb + 6 * (size_t)p.n_tri);
    LSDF_TRY(check_launch("mesh_bounds_kernel"));
    if (p.is_signed) {
        LSDF_TRY(check_cuda(cudaMallocAsync((void**)&ray, sizeof(RayTri) * 4 * (size_t)p.n_tri, s), "mesh ray alloc"));
        ray_setup_kernel<<<grid_for(4LL * p.n_tri, 128), 128, 0, s>>>(p.tri, p.n_tri, ray);
        LSDF_TRY(check_launch("ray_setup_kernel"));
    }
    p.ray = ray;
    if (p.pts == nullptr) {
        const dim3 grid((unsigned)((p.dims[0] + 7) / 8), (unsigned)((p.dims[1] + 3) / 4), (unsigned)((p.dims[2] + 3) / 4));
        mesh_kernel<true><<<grid, MESH_CELLS, 0, s>>>(p, bb, bb + 6 * (size_t)p.n_tri);
    } else {
        mesh_kernel<false><<<grid_for(p.n, MESH_CELLS), MESH_CELLS, 0, s>>>(p, bb, bb + 6 * (size_t)p.n_tri);
    }
    int rc = check_launch("mesh_kernel");
    if (ray) cudaFreeAsync(ray, s);
    cudaFreeAsync(bb, s);
    return rc;
}

}  // namespace

extern "C" int lsdf_build_primitive(int32_t kind, const double params[8], const double extent[3],
                                    const double resolution[3], const int32_t dims[3], float* values_dev,
                                    void* stream) {
    if (kind < 0 || kind > 2) return fail(LSDF_ERR_VALIDATION, "unknown primitive kind %d", kind);
    BuildParams p{};
    p.kind = kind;
    for (int i = 0; i < 8; ++i) p.prm[i] = params[i];
    for (int a = 0; a < 3; ++a) {
        p.ext[a] = extent[a];
        p.res[a] = resolution[a];
        p.dims[a] = dims[a];
    }
    const int64_t n = (int64_t)dims[0] * dims[1] * dims[2];
    if (n >= 4294967296LL) return fail(LSDF_ERR_UNSUPPORTED, "link grid of %lld cells (>= 2^32)", (long long)n);
    if (n <= 0) return LSDF_OK;
    if (dims[1] > 65535 || dims[2] > 65535) return fail(LSDF_ERR_UNSUPPORTED, "link grid wider than 65535 cells");
    const dim3 grid((unsigned)((dims[0] + 127) / 128), (unsigned)dims[1], (unsigned)dims[2]);
    cudaStream_t s = (cudaStream_t)stream;
    if (kind == 0)
        build_primitive_kernel<0><<<grid, 128, 0, s>>>(p, values_dev);
    else if (kind == 1)
        build_primitive_kernel<1><<<grid, 128, 0, s>>>(p, values_dev);
    else
        build_primitive_kernel<2><<<grid, 128, 0, s>>>(p, values_dev);
    return check_launch("build_primitive_kernel");
}

extern "C" int lsdf_primitive_points(int32_t kind, const double params[8], const double* pts_dev, int64_t n,
                                     double* out_dev, void* stream) {
    if (kind < 0 || kind > 2) return fail(LSDF_ERR_VALIDATION, "unknown primitive kind %d", kind);
    if (n <= 0) return LSDF_OK;
    BuildParams p{};
    for (int i = 0; i < 8; ++i) p.prm[i] = params[i];
    primitive_points_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(kind, p, pts_dev, n, out_dev);
    return check_launch("primitive_points_kernel");
}

extern "C" int lsdf_build_mesh(const double* tri_dev, int32_t n_tri, int32_t is_signed, const double extent[3],
                               const double resolution[3], const int32_t dims[3], float* values_dev, void* stream) {
    if (n_tri <= 0) return fail(LSDF_ERR_VALIDATION, "mesh has no triangles");
    MeshParams p{};
    p.tri = tri_dev;
    p.n_tri = n_tri;
    p.is_signed = is_signed;
    for (int a = 0; a < 3; ++a) {
        p.ext[a] = extent[a];
        p.res[a] = resolution[a];
        p.dims[a] = dims[a];
    }
    p.n = (int64_t)dims[0] * dims[1] * dims[2];
    if (p.n >= 4294967296LL) return fail(LSDF_ERR_UNSUPPORTED, "link grid of %lld cells (>= 2^32)", (long long)p.n);
    p.out_f = values_dev;
    if (p.n <= 0) return LSDF_OK;
    return launch_mesh(p, (cudaStream_t)stream);
}

extern "C" int lsdf_mesh_points(const double* tri_dev, int32_t n_tri, int32_t is_signed, const double* pts_dev,
                                int64_t n, double* out_dev, void* stream) {
    if (n_tri <= 0) return fail(LSDF_ERR_VALIDATION, "mesh has no triangles");
    if (n <= 0) return LSDF_OK;
    MeshParams p{};
    p.tri = tri_dev;
    p.n_tri = n_tri;
    p.is_signed = is_signed;
    p.pts = pts_dev;
    p.n = n;
    p.out_d = out_dev;
    return launch_mesh(p, (cudaStream_t)stream);
}
