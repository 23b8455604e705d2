// lsdf_device.cuh — device-side helpers shared by the kernels: warp
// reductions, workspace layouts, and the strict-parity lookup primitive.
#pragma once
#include "lsdf_common.cuh"
#include "lsdf_math.cuh"

namespace lsdf {

constexpr unsigned FULL_MASK = 0xffffffffu;

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t u = __shfl_xor_sync(FULL_MASK, v, o);
        v = u < v ? u : v;
    }
    return v;
}

// Warp minimum of the 64-bit keys (hi << 32 | lo) with two 32-bit reductions:
// the smallest hi, then the smallest lo among the lanes holding it.
__device__ __forceinline__ uint64_t warp_min_key(uint32_t hi, uint32_t lo) {
    const uint32_t h = __reduce_min_sync(FULL_MASK, hi);
    const uint32_t l = __reduce_min_sync(FULL_MASK, hi == h ? lo : 0xffffffffu);
    return ((uint64_t)h << 32) | l;
}

__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(FULL_MASK, v, o));
    return v;
}

__device__ __forceinline__ float warp_min_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(FULL_MASK, v, o));
    return v;
}

__host__ __device__ inline int64_t n_vox(const lsdf_env_grid& e) { return (int64_t)e.dims[0] * e.dims[1] * e.dims[2]; }

// ------------------------------------------------------------------ occupancy workspace
// [counters 64 B][bitmap n_words u32][prefix n_words i32][posgrid V i32], each 256-B aligned.
// Bit index = C-order linear voxel index (ix*ny + iy)*nz + iz, so the rank of
// a set bit (prefix + popcount) is its position in np.unique(axis=0) order.
struct Occupancy {
    int32_t* counters;  // [0] n_occupied, [1] n_dropped, [2] block ticket, [3] spare
    uint32_t* bitmap;
    uint32_t* bricks;   // per (bx, by) column of 4^3-voxel bricks: bit bz set when the brick is occupied
    int32_t* prefix;    // exclusive popcount prefix per word
    int32_t* posgrid;   // first position in an explicit index list (general path)
    int64_t n_words;
    int32_t nbx, nby, nbz;
    bool bricks_ok;     // nbz <= 32: every producer of the bitmap also maintains the brick columns
};

constexpr int BRICK_LOG2 = 2;  // 4^3 voxels per brick

inline int64_t align256(int64_t b) { return (b + 255) / 256 * 256; }

inline int64_t brick_columns(const lsdf_env_grid& env) {
    return (int64_t)((env.dims[0] + 3) >> BRICK_LOG2) * ((env.dims[1] + 3) >> BRICK_LOG2);
}

// [counters 256 B | bitmap | brick columns | prefix | position grid]
inline Occupancy carve_occupancy(void* base, const lsdf_env_grid& env) {
    Occupancy o;
    const int64_t V = n_vox(env);
    o.n_words = (V + 31) / 32;
    o.nbx = (env.dims[0] + 3) >> BRICK_LOG2;
    o.nby = (env.dims[1] + 3) >> BRICK_LOG2;
    o.nbz = (env.dims[2] + 3) >> BRICK_LOG2;
    o.bricks_ok = o.nbz <= 32;
    char* p = (char*)base;
    o.counters = (int32_t*)p;
    p += 256;
    o.bitmap = (uint32_t*)p;
    p += align256(o.n_words * 4);
    o.bricks = (uint32_t*)p;
    p += align256(brick_columns(env) * 4);
    o.prefix = (int32_t*)p;
    p += align256(o.n_words * 4);
    o.posgrid = (int32_t*)p;
    return o;
}

// bytes a producer clears before scattering: counters, bitmap, brick columns
inline int64_t occupancy_clear_bytes(const Occupancy& o) {
    return 256 + align256(o.n_words * 4) + (int64_t)o.nbx * o.nby * 4;
}

inline int64_t occupancy_bytes(const lsdf_env_grid& env) {
    const int64_t V = n_vox(env);
    const int64_t w = (V + 31) / 32;
    return 256 + 2 * align256(w * 4) + align256(brick_columns(env) * 4) + align256(V * 4);
}

// ------------------------------------------------------------------ link grid views
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

// Fast-path constants of one link grid for the fused query: the eight
// corners of every cell packed into 32 B (two float4) so a lookup is two
// 16-B loads from one sector instead of eight scattered 4-B loads.
struct PackedGrid {
    const float4* cells;     // (nx-1)(ny-1)(nz-1) x 2 float4, x-fastest cells
    double ext[3], res[3], rinv[3], hi[3];
    int32_t cx, cy;          // cells per axis x, y (nx-1, ny-1)
    int32_t top[3];          // dims - 2 (largest base index)
    float d_far;
};

__host__ __device__ __forceinline__ PackedGrid packed_of(const lsdf_link_grid& g) {
    PackedGrid q;
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
    return q;
}

// u = (p + e) / r - 0.5 with the division done as q0 = x*rinv, corrected by
// one FMA residual step: with rinv = RN(1/r) this yields the correctly
// rounded quotient (Markstein's theorem; also checked on 3.2e8 random
// operands in tests/test_hostcheck.py::test_division_recipe).
__device__ __forceinline__ double cell_coord(double p, double e, double r, double rinv) {
    const double x = __dadd_rn(p, e);
    const double q0 = __dmul_rn(x, rinv);
    const double rr = __fma_rn(-q0, r, x);
    return __dsub_rn(__fma_rn(rr, rinv, q0), 0.5);
}

// floor(u) for 0 <= u < 2^31 without a conversion instruction:
// u + 1.5*2^52 rounds to the nearest integer in the low word.
__device__ __forceinline__ int floor_small(double u, double& fl) {
    const double M = 6755399441055744.0;
    const double t = __dadd_rn(u, M);
    int i = __double2loint(t);
    fl = __dsub_rn(t, M);
    if (fl > u) {
        fl = __dsub_rn(fl, 1.0);
        --i;
    }
    return i;
}

// Geometry shared by every link grid of one query launch (the usual case:
// all links baked with the same extent and resolution); kept in kernel
// parameters so the compiler holds it in uniform registers.
struct GridGeom {
    double ext[3], res[3], rinv[3], hi[3], topd[3];
    int32_t top[3];
    int32_t cx, cy;
};

// grids.py:155-191 at a link-frame point, packed-corner layout, returning
// `far` outside the stored hull.  Identical arithmetic to trilinear_at.
__device__ __forceinline__ float trilinear_geom(const GridGeom& g, const float4* __restrict__ cells, float far,
                                                double px, double py, double pz) {
    const double ux = cell_coord(px, g.ext[0], g.res[0], g.rinv[0]);
    const double uy = cell_coord(py, g.ext[1], g.res[1], g.rinv[1]);
    const double uz = cell_coord(pz, g.ext[2], g.res[2], g.rinv[2]);
    const bool inside = (ux >= 0.0) & (ux <= g.hi[0]) & (uy >= 0.0) & (uy <= g.hi[1]) & (uz >= 0.0) &
                        (uz <= g.hi[2]);
    if (!inside) return far;
    double fx0, fy0, fz0;
    int ix = floor_small(ux, fx0), iy = floor_small(uy, fy0), iz = floor_small(uz, fz0);
    if (ix > g.top[0]) { ix = g.top[0]; fx0 = g.topd[0]; }
    if (iy > g.top[1]) { iy = g.top[1]; fy0 = g.topd[1]; }
    if (iz > g.top[2]) { iz = g.top[2]; fz0 = g.topd[2]; }
    const float fx = __double2float_rn(__dsub_rn(ux, fx0));
    const float fy = __double2float_rn(__dsub_rn(uy, fy0));
    const float fz = __double2float_rn(__dsub_rn(uz, fz0));
    const float gx = __fsub_rn(1.0f, fx), gy = __fsub_rn(1.0f, fy), gz = __fsub_rn(1.0f, fz);
    const uint32_t cell = (uint32_t)ix + (uint32_t)g.cx * ((uint32_t)iy + (uint32_t)g.cy * (uint32_t)iz);
    const float4 a = __ldg(cells + 2 * cell);      // v000 v100 v010 v110
    const float4 b = __ldg(cells + 2 * cell + 1);  // v001 v101 v011 v111
    const float c00 = __fadd_rn(__fmul_rn(a.x, gx), __fmul_rn(a.y, fx));
    const float c10 = __fadd_rn(__fmul_rn(a.z, gx), __fmul_rn(a.w, fx));
    const float c01 = __fadd_rn(__fmul_rn(b.x, gx), __fmul_rn(b.y, fx));
    const float c11 = __fadd_rn(__fmul_rn(b.z, gx), __fmul_rn(b.w, fx));
    const float c0 = __fadd_rn(__fmul_rn(c00, gy), __fmul_rn(c10, fy));
    const float c1 = __fadd_rn(__fmul_rn(c01, gy), __fmul_rn(c11, fy));
    return __fadd_rn(__fmul_rn(c0, gz), __fmul_rn(c1, fz));
}

// grids.py:155-191 at a link-frame point, packed-corner layout.  Identical
// arithmetic to trilinear_at (lsdf_math.cuh).
__device__ __forceinline__ float trilinear_packed(const PackedGrid& g, double px, double py, double pz) {
    const double ux = cell_coord(px, g.ext[0], g.res[0], g.rinv[0]);
    const double uy = cell_coord(py, g.ext[1], g.res[1], g.rinv[1]);
    const double uz = cell_coord(pz, g.ext[2], g.res[2], g.rinv[2]);
    const bool inside = (ux >= 0.0) && (ux <= g.hi[0]) && (uy >= 0.0) && (uy <= g.hi[1]) && (uz >= 0.0) &&
                        (uz <= g.hi[2]);
    if (!inside) return g.d_far;
    double fx0, fy0, fz0;
    int ix = floor_small(ux, fx0), iy = floor_small(uy, fy0), iz = floor_small(uz, fz0);
    if (ix > g.top[0]) { ix = g.top[0]; fx0 = (double)g.top[0]; }
    if (iy > g.top[1]) { iy = g.top[1]; fy0 = (double)g.top[1]; }
    if (iz > g.top[2]) { iz = g.top[2]; fz0 = (double)g.top[2]; }
    const float fx = __double2float_rn(__dsub_rn(ux, fx0));
    const float fy = __double2float_rn(__dsub_rn(uy, fy0));
    const float fz = __double2float_rn(__dsub_rn(uz, fz0));
    const float gx = __fsub_rn(1.0f, fx), gy = __fsub_rn(1.0f, fy), gz = __fsub_rn(1.0f, fz);
    const int64_t cell = ix + (int64_t)g.cx * (iy + (int64_t)g.cy * iz);
    const float4 a = __ldg(g.cells + 2 * cell);      // v000 v100 v010 v110
    const float4 b = __ldg(g.cells + 2 * cell + 1);  // v001 v101 v011 v111
    const float c00 = __fadd_rn(__fmul_rn(a.x, gx), __fmul_rn(a.y, fx));
    const float c10 = __fadd_rn(__fmul_rn(a.z, gx), __fmul_rn(a.w, fx));
    const float c01 = __fadd_rn(__fmul_rn(b.x, gx), __fmul_rn(b.y, fx));
    const float c11 = __fadd_rn(__fmul_rn(b.z, gx), __fmul_rn(b.w, fx));
    const float c0 = __fadd_rn(__fmul_rn(c00, gy), __fmul_rn(c10, fy));
    const float c1 = __fadd_rn(__fmul_rn(c01, gy), __fmul_rn(c11, fy));
    return __fadd_rn(__fmul_rn(c0, gz), __fmul_rn(c1, fz));
}

// dst[cell] = v for every cell of an n-cell window whose keep bit is clear
// (the masked cells carry the link sentinel, placement.py:305-308).  Threads
// take 4 cells each (one nibble of the mask) and write a float4 when all four
// are masked; i0 / stride enumerate the calling threads.
__device__ __forceinline__ void fill_masked_cells(const uint32_t* __restrict__ mask_bits, int64_t n, float* dst,
                                                  float v, int64_t i0, int64_t stride) {
    if ((n & 3) == 0 && ((uintptr_t)dst & 15) == 0) {
        const float4 v4 = make_float4(v, v, v, v);
        for (int64_t g = i0; g < (n >> 2); g += stride) {
            const int64_t cell = g << 2;
            const uint32_t nib = (__ldg(mask_bits + (cell >> 5)) >> (cell & 31)) & 0xFu;
            if (nib == 0u) {
                __stcs((float4*)(dst + cell), v4);
            } else if (nib != 0xFu) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (!((nib >> k) & 1u)) __stcs(dst + cell + k, v);
            }
        }
        return;
    }
    for (int64_t cell = i0; cell < n; cell += stride)
        if (!((__ldg(mask_bits + (cell >> 5)) >> (cell & 31)) & 1u)) dst[cell] = v;
}

// trilinear_packed in two stages, so a caller can issue several lookups'
// loads back to back (the same operations, bit-identical): packed_prep
// returns the cell (-1 outside the grid) and the f32 fractions.
__device__ __forceinline__ int64_t packed_prep(const PackedGrid& g, double px, double py, double pz, float& fx,
                                               float& fy, float& fz) {
    const double ux = cell_coord(px, g.ext[0], g.res[0], g.rinv[0]);
    const double uy = cell_coord(py, g.ext[1], g.res[1], g.rinv[1]);
    const double uz = cell_coord(pz, g.ext[2], g.res[2], g.rinv[2]);
    const bool inside = (ux >= 0.0) && (ux <= g.hi[0]) && (uy >= 0.0) && (uy <= g.hi[1]) && (uz >= 0.0) &&
                        (uz <= g.hi[2]);
    if (!inside) return -1;
    double fx0, fy0, fz0;
    int ix = floor_small(ux, fx0), iy = floor_small(uy, fy0), iz = floor_small(uz, fz0);
    if (ix > g.top[0]) { ix = g.top[0]; fx0 = (double)g.top[0]; }
    if (iy > g.top[1]) { iy = g.top[1]; fy0 = (double)g.top[1]; }
    if (iz > g.top[2]) { iz = g.top[2]; fz0 = (double)g.top[2]; }
    fx = __double2float_rn(__dsub_rn(ux, fx0));
    fy = __double2float_rn(__dsub_rn(uy, fy0));
    fz = __double2float_rn(__dsub_rn(uz, fz0));
    return ix + (int64_t)g.cx * (iy + (int64_t)g.cy * iz);
}

__device__ __forceinline__ float packed_finish(float4 a, float4 b, float fx, float fy, float fz) {
    const float gx = __fsub_rn(1.0f, fx), gy = __fsub_rn(1.0f, fy), gz = __fsub_rn(1.0f, fz);
    const float c00 = __fadd_rn(__fmul_rn(a.x, gx), __fmul_rn(a.y, fx));
    const float c10 = __fadd_rn(__fmul_rn(a.z, gx), __fmul_rn(a.w, fx));
    const float c01 = __fadd_rn(__fmul_rn(b.x, gx), __fmul_rn(b.y, fx));
    const float c11 = __fadd_rn(__fmul_rn(b.z, gx), __fmul_rn(b.w, fx));
    const float c0 = __fadd_rn(__fmul_rn(c00, gy), __fmul_rn(c10, fy));
    const float c1 = __fadd_rn(__fmul_rn(c01, gy), __fmul_rn(c11, fy));
    return __fadd_rn(__fmul_rn(c0, gz), __fmul_rn(c1, fz));
}

}  // namespace lsdf
