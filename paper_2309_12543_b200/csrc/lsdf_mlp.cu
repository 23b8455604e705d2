// lsdf_mlp.cu — stage 2b: TinyMlp inference (approx.py:63-158, 292-306).
//
// y = relu(x W1 + b1) W2 + b2 with x the row-major rotation (B, 9) rounded to
// f32 (approx.py:125-129).  Layer 1 (K = 9) is tiny and runs on CUDA cores;
// layer 2 (K = H = 32, N = 3V up to 3.3 M) is the dense contraction.
//
// This file holds the CUDA-core path, which reproduces OpenBLAS sgemm's
// per-element FMA chain over k (bit-exact with numpy on the build host); the
// tcgen05 tensor-core path lives in lsdf_mlp_tc.cu.
#include "lsdf_common.cuh"
#include "lsdf_math.cuh"

using namespace lsdf;

namespace {

constexpr int ROWS = 32;  // rotations per CTA
constexpr int COLS = 256; // outputs per CTA (one per thread)

__global__ void __launch_bounds__(COLS) mlp_cuda_core_kernel(const float* __restrict__ w1, const float* __restrict__ b1,
                                                             const float* __restrict__ w2, const float* __restrict__ b2,
                                                             int H, int64_t n_out, const double* __restrict__ R,
                                                             int64_t B, float* __restrict__ y, int64_t ldy) {
    __shared__ float s_h[ROWS][64];
    const int64_t r0 = (int64_t)blockIdx.y * ROWS;
    // layer 1 for this CTA's rows: h[r][j] = max(fma-chain_k x[r][k] w1[k][j] + b1[j], 0)
    for (int e = threadIdx.x; e < ROWS * H; e += COLS) {
        const int r = e / H, j = e % H;
        float acc = 0.0f;
        if (r0 + r < B) {
            const double* x = R + (r0 + r) * 9;
            acc = __fmul_rn((float)x[0], w1[j]);
            for (int k = 1; k < 9; ++k) acc = __fmaf_rn((float)x[k], w1[k * H + j], acc);
            acc = __fadd_rn(acc, b1[j]);
            acc = acc > 0.0f ? acc : 0.0f;
        }
        s_h[r][j] = acc;
    }
    __syncthreads();
    const int64_t n = (int64_t)blockIdx.x * COLS + threadIdx.x;
    if (n >= n_out) return;
    float w[64];
    for (int k = 0; k < H; ++k) w[k] = w2[(int64_t)k * n_out + n];
    const float bias = b2[n];
    for (int r = 0; r < ROWS && r0 + r < B; ++r) {
        float acc = __fmul_rn(s_h[r][0], w[0]);
        for (int k = 1; k < H; ++k) acc = __fmaf_rn(s_h[r][k], w[k], acc);
        y[(r0 + r) * ldy + n] = __fadd_rn(acc, bias);
    }
}

}  // namespace

int lsdf_mlp_predict_tc(const float* w1, const float* b1, const float* w2, const float* w2_packed, const float* b2,
                        int32_t H, int64_t n_out, const double* R, int64_t B, float* y, int64_t ldy, cudaStream_t s);
int64_t lsdf_mlp_packed_bytes_tc(int32_t H, int64_t n_out);
int lsdf_mlp_pack_tc(const float* w2, int32_t H, int64_t n_out, float* packed, cudaStream_t s);

int64_t lsdf_mlp_cells_packed_bytes(int32_t H, int64_t V);
int lsdf_mlp_pack_cells(const float* w2, int32_t H, int64_t V, float* packed, cudaStream_t s);
int lsdf_mlp_place_tc(const float* w1, const float* b1, const float* w2_cells_packed, const float* b2, int32_t H,
                      int64_t V, const int32_t* kept_cells, const double* R, const double* dt, int64_t C, int32_t L,
                      const lsdf_link_grid* grids, const lsdf_window* window, float* out, cudaStream_t s);

extern "C" int64_t lsdf_mlp_place_packed_bytes(int32_t H, int64_t n_points) {
    return lsdf_mlp_cells_packed_bytes(H, n_points);
}

extern "C" int lsdf_mlp_place_pack(const float* w2_dev, int32_t H, int64_t n_points, float* packed_dev, void* stream) {
    if (H < 1 || H > 32) return fail(LSDF_ERR_UNSUPPORTED, "fused TinyMlp placement: hidden width %d outside 1..32", H);
    if (n_points <= 0) return LSDF_OK;
    return lsdf_mlp_pack_cells(w2_dev, H, n_points, packed_dev, (cudaStream_t)stream);
}

extern "C" int lsdf_mlp_place(const float* w1_dev, const float* b1_dev, const float* w2_place_packed_dev,
                              const float* b2_dev, int32_t H, int64_t n_points, const int32_t* kept_cells_dev,
                              const double* R_geo_dev, const double* dt_geo_dev, int64_t C, int32_t n_geo,
                              const lsdf_link_grid* grids, const lsdf_window* window, float* windows_dev,
                              void* stream) {
    if (H < 1 || H > 32) return fail(LSDF_ERR_UNSUPPORTED, "fused TinyMlp placement: hidden width %d outside 1..32", H);
    if (w2_place_packed_dev == nullptr) return fail(LSDF_ERR_VALIDATION, "fused placement: W2 not packed");
    if (C <= 0) return LSDF_OK;
    if (C * n_geo > 65535) return fail(LSDF_ERR_UNSUPPORTED, "fused placement: more than 65535 windows per call");
    return lsdf_mlp_place_tc(w1_dev, b1_dev, w2_place_packed_dev, b2_dev, H, n_points, kept_cells_dev, R_geo_dev,
                             dt_geo_dev, C, n_geo, grids, window, windows_dev, (cudaStream_t)stream);
}

extern "C" int64_t lsdf_mlp_packed_bytes(int32_t H, int64_t n_out) { return lsdf_mlp_packed_bytes_tc(H, n_out); }

extern "C" int lsdf_mlp_pack(const float* w2_dev, int32_t H, int64_t n_out, float* packed_dev, void* stream) {
    if (H < 1 || H > 64) return fail(LSDF_ERR_UNSUPPORTED, "TinyMlp hidden width %d outside 1..64", H);
    if (n_out <= 0) return LSDF_OK;
    return lsdf_mlp_pack_tc(w2_dev, H, n_out, packed_dev, (cudaStream_t)stream);
}

extern "C" int lsdf_mlp_predict(const float* w1_dev, const float* b1_dev, const float* w2_dev,
                                const float* w2_packed_dev, const float* b2_dev, int32_t H, int64_t n_out,
                                const double* R_dev, int64_t B, float* y_dev, int64_t ldy, int32_t use_tensor_cores,
                                void* stream) {
    if (H < 1 || H > 64) return fail(LSDF_ERR_UNSUPPORTED, "TinyMlp hidden width %d outside 1..64", H);
    if (ldy < n_out) return fail(LSDF_ERR_VALIDATION, "TinyMlp: row stride %lld < %lld outputs", (long long)ldy,
                                 (long long)n_out);
    if (B <= 0 || n_out <= 0) return LSDF_OK;
    if (use_tensor_cores)
        return lsdf_mlp_predict_tc(w1_dev, b1_dev, w2_dev, w2_packed_dev, b2_dev, H, n_out, R_dev, B, y_dev, ldy,
                                   (cudaStream_t)stream);
    dim3 grid((unsigned)((n_out + COLS - 1) / COLS), (unsigned)((B + ROWS - 1) / ROWS));
    mlp_cuda_core_kernel<<<grid, COLS, 0, (cudaStream_t)stream>>>(w1_dev, b1_dev, w2_dev, b2_dev, H, n_out, R_dev, B,
                                                                   y_dev, ldy);
    return check_launch("mlp_cuda_core_kernel");
}
