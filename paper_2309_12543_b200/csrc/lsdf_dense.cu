// lsdf_dense.cu — the paper's materialized mode and the standalone operators.
//
//   place_windows_kernel    placement.py:267-313 (every (c, l) window, W^3 cells)
//   place_windows_g_kernel  the same with provider coordinates G (NeuralTransformProvider,
//                           approx.py:292-306,340-355: G = f32 MLP output + fp64 shift)
//   assemble_kernel         query.py:61-103 (scatter-min into dense C x V_e)
//   query_dense_kernel      query.py:128-150 (gather + first-occurrence argmin)
//   per_link_fields_kernel  query.py:153-176
//   sphere_baseline_kernel  query.py:254-291
//   trilinear_kernel        grids.py:155-191
//   transform_exact_kernel  placement.py:148-169
//   pack_corners_kernel     layout change for the fused query (no arithmetic)
#include "lsdf_device.cuh"

using namespace lsdf;

namespace {

struct PlaceParams {
    lsdf_link_grid grids[LSDF_MAX_LINKS];
    const double* R;
    const double* dt;
    int64_t C;
    int32_t n_geo;
    int32_t W[3];
    double e_r;
    const double* P;
    int32_t Wmax;
    const uint32_t* mask_bits;
    float* out;
};

// Blocks run link-major (block b: link b / C, configuration b % C), so the
// windows of one link sample its grid back to back while it sits in L2; with
// the packed-corner grid a lookup is one 32-B sector instead of eight
// scattered 4-B loads (trilinear_packed: the same arithmetic, bit-exact).
__global__ void place_windows_kernel(const __grid_constant__ PlaceParams p) {
    const int l = (int)(blockIdx.x / p.C);
    const int64_t f = (int64_t)(blockIdx.x % p.C) * p.n_geo + l;  // field = c * n_geo + l
    const lsdf_link_grid& G = p.grids[l];
    const GridView gv = view_of(G);
    const LdgLoad ld{G.values_dev};
    const bool packed = G.packed_dev != nullptr;
    const PackedGrid pg = packed_of(G);
    double R[9], dtinv[3];
#pragma unroll
    for (int e = 0; e < 9; ++e) R[e] = p.R[f * 9 + e];
    shift_inverse(R, p.dt + f * 3, p.e_r, dtinv);
    const int W0 = p.W[0], W1 = p.W[1];
    const int n = W0 * W1 * p.W[2];
    float* dst = p.out + f * (int64_t)n;
    // warps walk the window's x rows (my, mz), lanes the cells of a row: two
    // divisions per row instead of per cell
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int row = warp; row < W1 * p.W[2]; row += nw) {
      const int my = row % W1, mz = row / W1;
      for (int mx = lane; mx < W0; mx += 32) {
        const int cell = mx + W0 * row;
        const bool keep = (__ldg(p.mask_bits + (cell >> 5)) >> (cell & 31)) & 1u;
        float v = gv.d_far;  // masked cells carry the link sentinel (placement.py:305-308)
        if (keep) {
            double pt[3];
            window_point(p.P[mx], p.P[p.Wmax + my], p.P[2 * p.Wmax + mz], R, dtinv, p.e_r, pt);
            v = packed ? trilinear_packed(pg, pt[0], pt[1], pt[2]) : trilinear_at(gv, pt[0], pt[1], pt[2], ld);
        }
        dst[cell] = v;
      }
    }
}

// Windows from provider coordinates: the kept cell k (x-fastest kept order,
// kept[k] = its cell) samples the link grid at (double(y[f, 3k..3k+2]) +
// dtinv) * e_r (approx.py:302-305 then placement.py:300-313).
__global__ void place_windows_g_kernel(const __grid_constant__ PlaceParams p, const float* __restrict__ y,
                                       int64_t ldy, const int32_t* __restrict__ kept, int32_t n_kept) {
    const int l = (int)(blockIdx.y / p.C);  // link-major, as place_windows_kernel
    const int64_t f = (int64_t)(blockIdx.y % p.C) * p.n_geo + l;  // field = c * n_geo + l
    const lsdf_link_grid& G = p.grids[l];
    const GridView gv = view_of(G);
    const LdgLoad ld{G.values_dev};
    const bool packed = G.packed_dev != nullptr;
    const PackedGrid pg = packed_of(G);
    double R[9], dtinv[3];
#pragma unroll
    for (int e = 0; e < 9; ++e) R[e] = p.R[f * 9 + e];
    shift_inverse(R, p.dt + f * 3, p.e_r, dtinv);
    const int n = p.W[0] * p.W[1] * p.W[2];
    float* dst = p.out + f * (int64_t)n;
    const int stride = gridDim.x * blockDim.x;
    const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
    fill_masked_cells(p.mask_bits, n, dst, gv.d_far, i0, stride);  // masked cells: the link sentinel
    const float* yf = y + f * ldy;
    for (int k = i0; k < n_kept; k += stride) {
        const double gx = DADD((double)__ldg(yf + 3 * k), dtinv[0]);
        const double gy = DADD((double)__ldg(yf + 3 * k + 1), dtinv[1]);
        const double gz = DADD((double)__ldg(yf + 3 * k + 2), dtinv[2]);
        const double px = DMUL(gx, p.e_r), py = DMUL(gy, p.e_r), pz = DMUL(gz, p.e_r);
        dst[__ldg(kept + k)] = packed ? trilinear_packed(pg, px, py, pz) : trilinear_at(gv, px, py, pz, ld);
    }
}

__global__ void fill_kernel(float* out, int64_t n, float v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = v;
}

// float min via integer atomics: non-negative floats order like ints, negative
// ones reverse-order like unsigned ints.
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
        const int x = ax + cell % W0, y = ay + (cell / W0) % W1, z = az + cell / (W0 * W1);
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

// SURVEY Appendix B on placed windows: the argmin link is the lowest link
// whose window value at the winning voxel equals d (d == clamp: -1 / -1).
__global__ void link_at_voxel_kernel(const float* __restrict__ windows, const int32_t* __restrict__ anchors,
                                     int64_t C, int32_t L, int32_t W0, int32_t W1, int32_t W2,
                                     const int32_t* __restrict__ idx, const int32_t* __restrict__ argmin,
                                     const float* __restrict__ d, float clamp, int32_t* link, int32_t* voxel) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    const float dc = d[c];
    if (!(dc < clamp)) {  // query.py:142-144 + the clamp rule
        link[c] = -1;
        voxel[c] = -1;
        return;
    }
    const int32_t pos = argmin[c];
    const int vx = idx[3 * pos], vy = idx[3 * pos + 1], vz = idx[3 * pos + 2];
    const int64_t n = (int64_t)W0 * W1 * W2;
    int best = -1;
    for (int l = 0; l < L && best < 0; ++l) {
        const int32_t* a = anchors + (c * L + l) * 3;
        const int rx = vx - a[0], ry = vy - a[1], rz = vz - a[2];
        if (rx < 0 || ry < 0 || rz < 0 || rx >= W0 || ry >= W1 || rz >= W2) continue;
        if (windows[(c * L + l) * n + rx + (int64_t)W0 * (ry + (int64_t)W1 * rz)] == dc) best = l;
    }
    link[c] = best;
    voxel[c] = pos;
}

__global__ void per_link_fields_kernel(const float* __restrict__ windows, const int32_t* anchors,
                                       const int32_t* configs, const int32_t* links, const float* d_far,
                                       int32_t W0, int32_t W1, int32_t W2, int32_t n_links, lsdf_env_grid env,
                                       const uint32_t* __restrict__ bitmap, float* out) {
    __shared__ float s_min[32];
    const int64_t f = blockIdx.x;
    const int ax = anchors[3 * f], ay = anchors[3 * f + 1], az = anchors[3 * f + 2];
    const int n = W0 * W1 * W2;
    float m = d_far[f];  // query.py:171: the limit starts at the field's sentinel
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
        m = threadIdx.x < (int)(blockDim.x >> 5) ? s_min[threadIdx.x] : INFINITY;
        m = warp_min_f(m);
        if (threadIdx.x == 0) atomic_min_float(out + (int64_t)configs[f] * n_links + links[f], m);
    }
}

// One CTA per configuration.  min over voxels n and spheres s of
// sqrt(|c_s - x_n|^2) - r_s equals min over s of (sqrt(min_n |c_s - x_n|^2) - r_s)
// exactly (the correctly rounded sqrt and the subtraction are monotone), so a
// thread keeps one running squared minimum per sphere (MAXS registers) and
// takes S square roots at the end instead of one per (sphere, voxel).
template <int MAXS>
__global__ void __launch_bounds__(256) sphere_baseline_kernel(const double* __restrict__ R, const double* __restrict__ T,
                                                              int32_t L, const int32_t* sl, const double* sc,
                                                              const double* sr, int32_t S,
                                                              const int32_t* __restrict__ idx, int64_t N,
                                                              lsdf_env_grid env, double* out) {
    extern __shared__ double s_w[];  // S x 4: world centre + radius
    __shared__ double s_min[32];
    const int64_t c = blockIdx.x;
    for (int s = threadIdx.x; s < S; s += blockDim.x) {
        const double* Rc = R + (c * L + sl[s]) * 9;
        double w[3];
        mv_einsum(Rc, sc + 3 * s, w);  // einsum("bsij,sj->bsi")
        for (int k = 0; k < 3; ++k) s_w[4 * s + k] = DADD(w[k], T[(c * L + sl[s]) * 3 + k]);
        s_w[4 * s + 3] = sr[s];
    }
    __syncthreads();
    double m = INFINITY;
    if (MAXS > 0) {
        double m2[MAXS > 0 ? MAXS : 1];
#pragma unroll
        for (int s = 0; s < MAXS; ++s) m2[s] = INFINITY;
        for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
            double x[3];
            for (int k = 0; k < 3; ++k)
                x[k] = DADD(-env.extent[k], DMUL(DADD((double)__ldg(idx + 3 * i + k), 0.5), env.resolution[k]));
#pragma unroll
            for (int s = 0; s < MAXS; ++s) {
                if (s < S) {
                    const double d0 = DSUB(s_w[4 * s], x[0]), d1 = DSUB(s_w[4 * s + 1], x[1]),
                                 d2 = DSUB(s_w[4 * s + 2], x[2]);
                    const double q = dot3(d0, d1, d2, d0, d1, d2);
                    m2[s] = q < m2[s] ? q : m2[s];
                }
            }
        }
#pragma unroll
        for (int s = 0; s < MAXS; ++s) {
            if (s < S) {
                const double d = DSUB(DSQRT(m2[s]), s_w[4 * s + 3]);
                m = d < m ? d : m;
            }
        }
    } else {
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
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double u = __shfl_xor_sync(FULL_MASK, m, o);
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

__global__ void trilinear_kernel(lsdf_link_grid g, const double* pts, int64_t n, double scale, float* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = trilinear_at(view_of(g), DMUL(pts[3 * i], scale), DMUL(pts[3 * i + 1], scale),
                          DMUL(pts[3 * i + 2], scale), LdgLoad{g.values_dev});
}

// One CTA per (rotation b, slice of points): R and dt_inv are computed once
// per CTA; each thread writes its points' 24-byte fp64 triples (consecutive
// threads -> consecutive points -> coalesced).
constexpr int TX_THREADS = 256, TX_PER_THREAD = 4;

__global__ void __launch_bounds__(TX_THREADS) transform_exact_kernel(const double* R, const double* dt, int64_t B,
                                                                      const double* __restrict__ P, int64_t V,
                                                                      double e_r, double* G) {
    __shared__ double s_R[9], s_dti[3];
    const int64_t b = blockIdx.y;
    if (threadIdx.x == 0) {
        double Rb[9], dti[3];
#pragma unroll
        for (int e = 0; e < 9; ++e) Rb[e] = R[b * 9 + e];
        shift_inverse(Rb, dt + b * 3, e_r, dti);
#pragma unroll
        for (int e = 0; e < 9; ++e) s_R[e] = Rb[e];
#pragma unroll
        for (int k = 0; k < 3; ++k) s_dti[k] = dti[k];
    }
    __syncthreads();
    double Rb[9], dti[3];
#pragma unroll
    for (int e = 0; e < 9; ++e) Rb[e] = s_R[e];
#pragma unroll
    for (int k = 0; k < 3; ++k) dti[k] = s_dti[k];
    // each round: TX_THREADS points -> 3 * TX_THREADS contiguous doubles of G,
    // staged in shared memory so the stores are unit-stride (full sectors)
    __shared__ double s_out[3 * TX_THREADS];
    const int64_t blk0 = (int64_t)blockIdx.x * TX_THREADS * TX_PER_THREAD;
    double* out = G + b * V * 3;
    for (int r = 0; r < TX_PER_THREAD; ++r) {
        const int64_t base = blk0 + (int64_t)r * TX_THREADS;
        if (base >= V) break;
        const int64_t v = base + threadIdx.x;
        if (v < V) {
            const double px = __ldg(P + 3 * v), py = __ldg(P + 3 * v + 1), pz = __ldg(P + 3 * v + 2);
#pragma unroll
            for (int k = 0; k < 3; ++k)
                s_out[3 * threadIdx.x + k] = DADD(DFMA(pz, Rb[6 + k], DFMA(py, Rb[3 + k], DMUL(px, Rb[k]))), dti[k]);
        }
        __syncthreads();
        const int64_t n = 3 * ((V - base) < TX_THREADS ? (V - base) : TX_THREADS);
        for (int i = threadIdx.x; i < n; i += TX_THREADS) __stcs(out + 3 * base + i, s_out[i]);
        __syncthreads();
    }
}

__global__ void pack_corners_kernel(const float* __restrict__ v, int32_t nx, int32_t ny, int32_t nz, float4* out) {
    const int64_t cx = nx - 1, cy = ny - 1, cz = nz - 1;
    const int64_t n = cx * cy * cz;
    for (int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; cell < n;
         cell += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = cell % cx, j = (cell / cx) % cy, k = cell / (cx * cy);
        const int64_t sy = nx, sz = (int64_t)nx * ny;
        const int64_t b = i + sy * j + sz * k;
        out[2 * cell] = make_float4(v[b], v[b + 1], v[b + sy], v[b + 1 + sy]);
        out[2 * cell + 1] = make_float4(v[b + sz], v[b + 1 + sz], v[b + sy + sz], v[b + 1 + sy + sz]);
    }
}

}  // namespace

extern "C" int lsdf_pack_corners(const float* values_dev, const int32_t dims[3], float* packed_dev, void* stream) {
    if (dims[0] < 2 || dims[1] < 2 || dims[2] < 2) return fail(LSDF_ERR_VALIDATION, "grid needs >= 2 cells per axis");
    pack_corners_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(values_dev, dims[0], dims[1], dims[2],
                                                                     (float4*)packed_dev);
    return check_launch("pack_corners_kernel");
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
    p.C = C;
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

extern "C" int lsdf_place_windows_g(const float* g_dev, int64_t ldg, const int32_t* kept_cells_dev, int32_t n_kept,
                                    const double* R_geo_dev, const double* dt_geo_dev, int64_t C, int32_t n_geo,
                                    const lsdf_link_grid* grids, const lsdf_window* window, float* windows_dev,
                                    void* stream) {
    if (n_geo < 1 || n_geo > LSDF_MAX_LINKS) return fail(LSDF_ERR_VALIDATION, "place_g: bad link count %d", n_geo);
    if (n_kept != window->n_masked)
        return fail(LSDF_ERR_DIMENSION_MISMATCH, "place_g: %d provider points for %d kept cells", n_kept, window->n_masked);
    if (ldg < 3 * (int64_t)n_kept) return fail(LSDF_ERR_VALIDATION, "place_g: row stride %lld too small", (long long)ldg);
    if (C <= 0) return LSDF_OK;
    if (C * n_geo > 65535) return fail(LSDF_ERR_UNSUPPORTED, "place_g: more than 65535 windows per call");
    PlaceParams p{};
    for (int l = 0; l < n_geo; ++l) p.grids[l] = grids[l];
    p.R = R_geo_dev;
    p.dt = dt_geo_dev;
    p.C = C;
    p.n_geo = n_geo;
    for (int a = 0; a < 3; ++a) p.W[a] = window->W[a];
    p.e_r = window->e_r;
    p.mask_bits = window->mask_bits_dev;
    p.out = windows_dev;
    const int n = window->W[0] * window->W[1] * window->W[2];
    const unsigned bx = (unsigned)((n + 255) / 256 < 64 ? (n + 255) / 256 : 64);
    place_windows_g_kernel<<<dim3(bx, (unsigned)(C * n_geo)), 256, 0, (cudaStream_t)stream>>>(p, g_dev, ldg,
                                                                                           kept_cells_dev, n_kept);
    return check_launch("place_windows_g_kernel");
}

extern "C" int lsdf_fill(float* dst_dev, int64_t n, float value, void* stream) {
    if (n <= 0) return LSDF_OK;
    const int64_t blocks = (n + 255) / 256;
    fill_kernel<<<(unsigned)(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, (cudaStream_t)stream>>>(dst_dev, n, value);
    return check_launch("fill_kernel");
}

extern "C" int lsdf_assemble(const float* windows_dev, const int32_t* anchors_dev, const int32_t* config_dev,
                             int64_t n_fields, const int32_t W[3], const lsdf_env_grid* env, int64_t C,
                             double d_far_global, float* values_dev, void* stream) {
    if (C > 0) LSDF_TRY(lsdf_fill(values_dev, C * n_vox(*env), (float)d_far_global, stream));
    if (n_fields <= 0) return LSDF_OK;
    assemble_kernel<<<(unsigned)n_fields, 256, 0, (cudaStream_t)stream>>>(windows_dev, anchors_dev, config_dev, W[0],
                                                                           W[1], W[2], *env, values_dev);
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

extern "C" int lsdf_link_at_voxel(const float* windows_dev, const int32_t* anchors_dev, int64_t C, int32_t n_links,
                                  const int32_t W[3], const int32_t* indices_dev, const int32_t* argmin_dev,
                                  const float* d_dev, float clamp, int32_t* link_dev, int32_t* voxel_dev,
                                  void* stream) {
    if (C <= 0) return LSDF_OK;
    link_at_voxel_kernel<<<grid_for(C, 128), 128, 0, (cudaStream_t)stream>>>(
        windows_dev, anchors_dev, C, n_links, W[0], W[1], W[2], indices_dev, argmin_dev, d_dev, clamp, link_dev,
        voxel_dev);
    return check_launch("link_at_voxel_kernel");
}

extern "C" int lsdf_per_link_fields(const float* windows_dev, const int32_t* anchors_dev, const int32_t* configs_dev,
                                    const int32_t* links_dev, const float* d_far_dev, int64_t n_fields,
                                    const int32_t W[3], int32_t n_links, const lsdf_env_grid* env,
                                    const void* occupancy_dev, float* out_dev, void* stream) {
    if (n_fields <= 0) return LSDF_OK;
    Occupancy o = carve_occupancy(const_cast<void*>(occupancy_dev), *env);
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
    const size_t smem = (size_t)S * 4 * sizeof(double);
    auto kern = S <= 8 ? sphere_baseline_kernel<8> : (S <= 24 ? sphere_baseline_kernel<24> : sphere_baseline_kernel<0>);
    LSDF_TRY(ensure_smem((const void*)kern, smem, "sphere_baseline_kernel"));
    kern<<<(unsigned)C, 256, smem, (cudaStream_t)stream>>>(R_all_dev, T_all_dev, L, sphere_link_dev, sphere_center_dev,
                                                         sphere_radius_dev, S, indices_dev, N, *env, out_dev);
    return check_launch("sphere_baseline_kernel");
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
    dim3 grid((unsigned)((V + TX_THREADS * TX_PER_THREAD - 1) / (TX_THREADS * TX_PER_THREAD)), (unsigned)B);
    transform_exact_kernel<<<grid, TX_THREADS, 0, (cudaStream_t)stream>>>(R_dev, dt_dev, B, points_dev, V, e_r, G_dev);
    return check_launch("transform_exact_kernel");
}
