// lsdf_train.cu — TinyMlp training on the GPU (approx.py:212-289), hand-written.
//
// One optimisation step of the reference's loop, per batch of B rotations:
//   x = R (f32), pre = x W1 + b1, h = relu(pre), y = h W2 + b2,
//   t = P R (f32, the exact targets), dy = sign(y - t) / (B n_out),
//   dW2 = h^T dy, db2 = sum_b dy, dh = (dy W2^T) [pre > 0],
//   dW1 = x^T dh, db1 = sum_b dh, then Adam on every parameter with the
//   reference's f32 operation order (approx.py:262-268).
// Three launches:
//   layer1_kernel     (1 CTA)  x, pre, h for the batch; clears the dh accumulator
//   layer2_step_kernel (persistent over 256-column tiles of W2): forward,
//                     targets, dy, dW2 / db2 and their Adam update in registers
//                     (W2, m, v are read and written once per step: the step is
//                     HBM-bound on the optimiser state), then dy W2_old^T for the
//                     tile as a register-tiled shared-memory GEMM into a per-CTA
//                     dh partial (one atomic pass per CTA at the end)
//   layer1_update_kernel (1 CTA) dW1, db1 and their Adam update; step counter.
// sample_rotations_kernel draws the batch on the device (Philox, Box-Muller,
// the reference's quaternion formula approx.py:32-47) so nothing crosses PCIe
// per step.
#include <curand_kernel.h>
#include <cstdlib>

#include "lsdf_async.cuh"
#include "lsdf_common.cuh"
#include "lsdf_tc.cuh"

using namespace lsdf;

namespace {

constexpr int TJ = 128;          // W2 columns per tile (one per thread in the forward)
constexpr int THREADS = 128;
constexpr int MAXB = 128;        // batch rows
constexpr int MAXH = 32;         // hidden width handled by the fused step

struct TrainParams {
    lsdf_tmlp_train s;
    int32_t B;
    const double* R;             // (B, 3, 3) fp64 rotations
    float* x;                    // (B, 9) f32
    float* h;                    // (B, H)
    float* dh;                   // (B, H) accumulator
    double bc1, bc2;             // unused: the bias corrections come from the device step counter
};

// Adam (approx.py:262-268), f32 with the reference's numpy order (no FMA):
//   m += (1 - b1) * (g - m); v += (1 - b2) * (g * g - v);
//   p -= lr * (m / bc1) / (sqrt(v / bc2) + eps)
__device__ __forceinline__ void adam(float& p, float& m, float& v, float g, float lr, float omb1, float omb2,
                                     float bc1, float bc2, float eps) {
    m = __fadd_rn(m, __fmul_rn(omb1, __fsub_rn(g, m)));
    v = __fadd_rn(v, __fmul_rn(omb2, __fsub_rn(__fmul_rn(g, g), v)));
    const float num = __fmul_rn(lr, __fdiv_rn(m, bc1));
    const float den = __fadd_rn(__fsqrt_rn(__fdiv_rn(v, bc2)), eps);
    p = __fsub_rn(p, __fdiv_rn(num, den));
}

__device__ __forceinline__ void bias_corrections(const lsdf_tmlp_train& s, float& bc1, float& bc2) {
    const double step = (double)(*s.step + 1);  // this step's index (1-based), as the reference's loop
    bc1 = (float)(1.0 - pow((double)s.beta1, step));
    bc2 = (float)(1.0 - pow((double)s.beta2, step));
}

__global__ void layer1_kernel(const __grid_constant__ TrainParams p) {
    const int H = p.s.hidden;
    for (int i = threadIdx.x; i < p.B * 9; i += blockDim.x) p.x[i] = (float)p.R[i];
    __syncthreads();
    for (int i = threadIdx.x; i < p.B * H; i += blockDim.x) {
        const int b = i / H, k = i - b * H;
        float acc = 0.0f;
#pragma unroll
        for (int e = 0; e < 9; ++e) acc = __fmaf_rn(p.x[b * 9 + e], p.s.w1[e * H + k], acc);
        const float pre = __fadd_rn(acc, p.s.b1[k]);
        p.h[i] = pre > 0.0f ? pre : 0.0f;  // relu; dh is masked where pre <= 0 (h == 0 exactly there)
        p.dh[i] = 0.0f;
    }
}

// Persistent over column tiles.  Shared: h (B x H), x (B x 9), dy (B x TJ, row
// padded), W2_old (H x TJ, row padded), dh partial (B x H).
__global__ void __launch_bounds__(THREADS) layer2_step_kernel(const __grid_constant__ TrainParams p) {
    extern __shared__ float4 sm4[];
    const int B = p.B, H = p.s.hidden;
    const int LD = TJ + 4;  // row pitch (16-B aligned rows, bank offset between rows)
    float* s_dy = (float*)sm4;             // B x LD
    float* s_w = s_dy + B * LD;            // H x LD
    float* s_h = s_w + H * LD;             // B x H
    float* s_dh = s_h + B * H;             // B x H
    float* s_x = s_dh + B * H;             // B x 9
    for (int i = threadIdx.x; i < B * H; i += blockDim.x) {
        s_h[i] = p.h[i];
        s_dh[i] = 0.0f;
    }
    for (int i = threadIdx.x; i < B * 9; i += blockDim.x) s_x[i] = p.x[i];
    __syncthreads();
    const int64_t n_out = p.s.n_out;
    const int64_t ldw = p.s.ld_w2 > 0 ? p.s.ld_w2 : n_out;  // row pitch of W2 and its moments
    // dy = sign / float32(dy.size) (approx.py:255-256): +-RN(1 / n) exactly, as a multiply
    const float inv_n = __fdiv_rn(1.0f, (float)(B * n_out));
    float bc1, bc2;
    bias_corrections(p.s, bc1, bc2);
    const float lr = p.s.lr, omb1 = __fsub_rn(1.0f, p.s.beta1), omb2 = __fsub_rn(1.0f, p.s.beta2), eps = p.s.eps;
    const int64_t n_tiles = (n_out + TJ - 1) / TJ;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t j = tile * TJ + threadIdx.x;
        const bool live = j < n_out;
        float w[MAXH];
#pragma unroll
        for (int k = 0; k < MAXH; ++k) w[k] = (live && k < H) ? p.s.w2[(int64_t)k * ldw + j] : 0.0f;
#pragma unroll
        for (int k = 0; k < MAXH; ++k)
            if (k < H) s_w[k * LD + threadIdx.x] = w[k];
        const float bj = live ? p.s.b2[j] : 0.0f;
        // targets t[b, j] = sum_e P[v, e] R_b[e, kk] (np.matmul(points32[None], r32))
        const int64_t v = j / 3;
        const int kk = (int)(j - v * 3);
        float P0 = 0.f, P1 = 0.f, P2 = 0.f;
        if (live) {
            P0 = p.s.points[3 * v];
            P1 = p.s.points[3 * v + 1];
            P2 = p.s.points[3 * v + 2];
        }
        float gw[MAXH];
#pragma unroll
        for (int k = 0; k < MAXH; ++k) gw[k] = 0.0f;
        float gb = 0.0f;
        for (int b = 0; b < B; ++b) {
            // the batch row of h once per b (broadcast float4 loads), for the forward and the gradient
            float hb[MAXH];
#pragma unroll
            for (int k4 = 0; k4 < MAXH / 4; ++k4) {
                const float4 q = k4 * 4 < H ? *(const float4*)(s_h + b * H + 4 * k4) : make_float4(0.f, 0.f, 0.f, 0.f);
                hb[4 * k4] = q.x;
                hb[4 * k4 + 1] = q.y;
                hb[4 * k4 + 2] = q.z;
                hb[4 * k4 + 3] = q.w;
            }
            float a4[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // four interleaved partial sums (ILP)
#pragma unroll
            for (int k = 0; k < MAXH; ++k)
                if (k < H) a4[k & 3] = __fmaf_rn(hb[k], w[k], a4[k & 3]);
            const float y = __fadd_rn(__fadd_rn(__fadd_rn(a4[0], a4[1]), __fadd_rn(a4[2], a4[3])), bj);
            const float* xb = s_x + b * 9;
            const float t = __fmaf_rn(P2, xb[6 + kk], __fmaf_rn(P1, xb[3 + kk], __fmul_rn(P0, xb[kk])));
            const float sg = y > t ? 1.0f : (y < t ? -1.0f : 0.0f);
            const float dy = live ? sg * inv_n : 0.0f;
            s_dy[b * LD + threadIdx.x] = dy;
#pragma unroll
            for (int k = 0; k < MAXH; ++k)
                if (k < H) gw[k] = __fmaf_rn(hb[k], dy, gw[k]);
            gb = __fadd_rn(gb, dy);
        }
        if (live) {  // Adam on this column's W2 entries and b2[j]
#pragma unroll
            for (int k = 0; k < MAXH; ++k) {
                if (k < H) {
                    const int64_t o = (int64_t)k * ldw + j;
                    float pw = w[k], m = p.s.m_w2[o], vv = p.s.v_w2[o];
                    adam(pw, m, vv, gw[k], lr, omb1, omb2, bc1, bc2, eps);
                    p.s.w2[o] = pw;
                    p.s.m_w2[o] = m;
                    p.s.v_w2[o] = vv;
                }
            }
            float pb = bj, m = p.s.m_b2[j], vv = p.s.v_b2[j];
            adam(pb, m, vv, gb, lr, omb1, omb2, bc1, bc2, eps);
            p.s.b2[j] = pb;
            p.s.m_b2[j] = m;
            p.s.v_b2[j] = vv;
        }
        __syncthreads();
        // dh[b, k] += sum_j dy[b, j] W2_old[k, j] over the tile: thread = (b pair, k quad)
        // micro-tile, the columns in float4 steps; a warp shares its k quad (W2
        // rows broadcast) and spans 32 b pairs (rows LD apart: conflict-free)
        for (int item = threadIdx.x; item < (B / 2) * (H / 4); item += blockDim.x) {
            const int kq = item / (B / 2), bq = item - kq * (B / 2);
            const int b0 = 2 * bq, k0 = 4 * kq;
            float acc[2][4] = {};
            for (int jj = 0; jj < TJ; jj += 4) {
                const float4 a0 = *(const float4*)(s_dy + b0 * LD + jj);
                const float4 a1 = *(const float4*)(s_dy + (b0 + 1) * LD + jj);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 c = *(const float4*)(s_w + (k0 + q) * LD + jj);
                    acc[0][q] = __fmaf_rn(a0.x, c.x, __fmaf_rn(a0.y, c.y, __fmaf_rn(a0.z, c.z, __fmaf_rn(a0.w, c.w, acc[0][q]))));
                    acc[1][q] = __fmaf_rn(a1.x, c.x, __fmaf_rn(a1.y, c.y, __fmaf_rn(a1.z, c.z, __fmaf_rn(a1.w, c.w, acc[1][q]))));
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                s_dh[b0 * H + k0 + q] += acc[0][q];
                s_dh[(b0 + 1) * H + k0 + q] += acc[1][q];
            }
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < B * H; i += blockDim.x) atomicAdd(p.dh + i, s_dh[i]);
}

// ---------------------------------------------------------------- tcgen05 step
// The same layer-2 step for B = 64 and H = 32 with the forward and the W2
// gradient on the tensor cores (kind::tf32, 3xTF32 split: hi*hi + hi*lo +
// lo*hi, ~fp32 accuracy), per 128-column tile of W2:
//   GEMM1  y^T (128 x 64)   = W2^T tile (128 x 32) . h^T        -> TMEM cols [0, 64)
//   epilogue: thread t owns column j (TMEM lane t): y + b2, targets, dy, db2;
//             dy^T written as the next A operand (row t, K = batch)
//   GEMM2  dW2^T (128 x 32) = dy^T (128 x 64) . h                -> TMEM cols [64, 96)
//   epilogue: the column's Adam update (W2, m, v read and written once)
//   dh += dy . W2_old^T for the tile on the CUDA cores (register tiles from
//   shared memory), one atomic pass per CTA at the end.
// All operands are K-major, 128-byte swizzled (the layout of lsdf_mlp_tc.cu).
constexpr int TC_B = 64, TC_H = 32, TC_T = 128;
constexpr uint32_t IDESC_FWD = idesc_tf32(TC_T, TC_B);
constexpr uint32_t IDESC_GRAD = idesc_tf32(TC_T, TC_H);
constexpr int SDY_LD = TC_B + 2;       // fp32 dy rows (8-B aligned pairs)
constexpr int SW_LD = TC_T + 4;        // fp32 W2 tile rows

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}

size_t tc_step_smem() {
    return 1024 + 2 * (TC_T * 128) + 2 * (TC_B * 128) + 2 * (2 * TC_T * 128) + 2 * (2 * TC_H * 128) +
           (size_t)TC_T * SDY_LD * 4 + 3 * (size_t)TC_H * SW_LD * 4 + (size_t)TC_B * 9 * 4 + TC_T * 4 + 64;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// 256 threads: thread (half, c) with c = threadIdx % 128 owns column j (TMEM
// lane c; warps w and w + 4 read the same lane quarter) and half = threadIdx /
// 128 the batch rows [32 half, +32) of the epilogue, the hidden units
// [16 half, +16) of the Adam update and half of the dh register tiles.
constexpr int TC_THREADS = 2 * TC_T;
__global__ void __launch_bounds__(TC_THREADS, 1) layer2_tc_step_kernel(const __grid_constant__ TrainParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* A1 = sm;                         // [hi | lo] 128 rows x 128 B: W2^T tile (row c, k)
    uint8_t* B1 = A1 + 2 * TC_T * 128;        // [hi | lo] 64 rows x 128 B: h (row b, k)
    uint8_t* A2 = B1 + 2 * TC_B * 128;        // [hi | lo][2 k-blocks] 128 rows x 128 B: dy^T (row c, b)
    uint8_t* B2 = A2 + 2 * 2 * TC_T * 128;    // [hi | lo][2 k-blocks] 32 rows x 128 B: h^T (row k, b)
    float* sDY = (float*)(B2 + 2 * 2 * TC_H * 128);   // [c][SDY_LD] fp32 dy
    float* sW = sDY + TC_T * SDY_LD;                  // [k][SW_LD] fp32 W2 tile (old values)
    float* sM = sW + TC_H * SW_LD;                    // the tile's Adam moments, same layout
    float* sV = sM + TC_H * SW_LD;
    float* sX = sV + TC_H * SW_LD;                    // [b][9] f32 rotations
    float* sGB = sX + TC_B * 9;                       // [128] db2 of the upper batch half
    uint64_t* bar = (uint64_t*)(((uintptr_t)(sGB + TC_T) + 7) & ~(uintptr_t)7);
    uint32_t* tmem_slot = (uint32_t*)(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5, c = tid & (TC_T - 1), half = tid >> 7;
    const int64_t N = p.s.n_out;
    const int64_t ldw = p.s.ld_w2 > 0 ? p.s.ld_w2 : N;  // row pitch of W2 and its moments
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // h (B x H) into both operand layouts, x for the targets
    for (int i = tid; i < TC_B * TC_H; i += blockDim.x) {
        const int b = i / TC_H, k = i - b * TC_H;
        const float h = p.h[i];
        const float hh = tf32_rna(h), hl = tf32_rna(h - hh);
        const uint32_t o1 = sw128_offset((uint32_t)b, (uint32_t)k);
        *(float*)(B1 + o1) = hh;
        *(float*)(B1 + TC_B * 128 + o1) = hl;
        const uint32_t o2 = (uint32_t)(b >> 5) * (TC_H * 128) + sw128_offset((uint32_t)k, (uint32_t)(b & 31));
        *(float*)(B2 + o2) = hh;
        *(float*)(B2 + 2 * TC_H * 128 + o2) = hl;
    }
    for (int i = tid; i < TC_B * 9; i += blockDim.x) sX[i] = p.x[i];
    fence_async_smem();
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    float bc1, bc2;
    bias_corrections(p.s, bc1, bc2);
    const float lr = p.s.lr, omb1 = __fsub_rn(1.0f, p.s.beta1), omb2 = __fsub_rn(1.0f, p.s.beta2), eps = p.s.eps;
    const float inv_n = __fdiv_rn(1.0f, (float)(TC_B * N));
    // dh register tile: b pair (lane), k quad (warp)
    const int b0 = 2 * (tid & 31), k0 = 4 * warp;
    float dh[2][4] = {};
    uint32_t phase = 0;
    const int kh = 16 * half;  // this thread's hidden units in the A1 build and the Adam update
    const int bh = 32 * half;  // this thread's batch rows in the epilogue
    const int64_t n_tiles = (N + TC_T - 1) / TC_T;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t j = tile * TC_T + c;
        const bool live = j < N;
        // the tile's W2, m and v rows (k, 128 columns) land in shared memory
        // with asynchronous copies, all in flight at once: one memory round
        // trip per tile, the moments' latency hidden behind the products
        {
            const int64_t j0 = tile * TC_T;
            const int ncols = (int)(N - j0 < TC_T ? N - j0 : TC_T);
            const bool vec = ncols == TC_T && ((ldw & 3) == 0);
            for (int i = tid; i < TC_H * (TC_T / 4); i += blockDim.x) {
                const int k = i / (TC_T / 4), c4 = (i - k * (TC_T / 4)) * 4;
                const int64_t g = (int64_t)k * ldw + j0 + c4;
                if (vec) {
                    cp_async16(sW + k * SW_LD + c4, p.s.w2 + g);
                    cp_async16(sM + k * SW_LD + c4, p.s.m_w2 + g);
                    cp_async16(sV + k * SW_LD + c4, p.s.v_w2 + g);
                } else {
                    for (int e = 0; e < 4; ++e) {
                        if (c4 + e < ncols) {
                            cp_async4(sW + k * SW_LD + c4 + e, p.s.w2 + g + e);
                            cp_async4(sM + k * SW_LD + c4 + e, p.s.m_w2 + g + e);
                            cp_async4(sV + k * SW_LD + c4 + e, p.s.v_w2 + g + e);
                        } else {
                            sW[k * SW_LD + c4 + e] = 0.0f;
                        }
                    }
                }
            }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            __syncthreads();
        }
        // A1 = W2^T tile split into TF32 halves (this thread: 16 hidden units of column c)
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int k = kh + q;
            const float wv = sW[k * SW_LD + c];
            const float hi = tf32_rna(wv), lo = tf32_rna(wv - hi);
            const uint32_t o = sw128_offset((uint32_t)c, (uint32_t)k);
            *(float*)(A1 + o) = hi;
            *(float*)(A1 + TC_T * 128 + o) = lo;
        }
        const float bj = live ? p.s.b2[j] : 0.0f;
        fence_async_smem();
        tc_before();
        __syncthreads();
        if (tid == 0) {  // GEMM1: y^T = W2^T h^T, 3xTF32
            tc_after();
            const uint8_t* As[3] = {A1, A1, A1 + TC_T * 128};
            const uint8_t* Bs[3] = {B1, B1 + TC_B * 128, B1};
            uint32_t acc = 0;
#pragma unroll
            for (int term = 0; term < 3; ++term)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    mma_tf32(tmem, sdesc(smem_u32(As[term] + kk * 32)), sdesc(smem_u32(Bs[term] + kk * 32)), IDESC_FWD,
                             acc);
                    acc = 1;
                }
            tc_commit(bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1u;
        tc_after();
        float y[32];
        tmem_ld16(tmem + lane_base + (uint32_t)bh, y);
        tmem_ld16(tmem + lane_base + (uint32_t)(bh + 16), y + 16);
        // targets, dy, db2 for this thread's 32 batch rows; dy^T into the GEMM2
        // operand (k-block = half) and the fp32 copy
        const int64_t v = live ? j / 3 : 0;
        const int kk3 = live ? (int)(j - v * 3) : 0;
        const float P0 = live ? p.s.points[3 * v] : 0.f, P1 = live ? p.s.points[3 * v + 1] : 0.f,
                    P2 = live ? p.s.points[3 * v + 2] : 0.f;
        float gb = 0.0f;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            const int b = bh + q;
            const float yb = __fadd_rn(y[q], bj);
            const float* xb = sX + b * 9;
            const float tg = __fmaf_rn(P2, xb[6 + kk3], __fmaf_rn(P1, xb[3 + kk3], __fmul_rn(P0, xb[kk3])));
            const float sg = yb > tg ? 1.0f : (yb < tg ? -1.0f : 0.0f);
            const float dy = live ? sg * inv_n : 0.0f;
            gb = __fadd_rn(gb, dy);
            const float hi = tf32_rna(dy), lo = tf32_rna(dy - hi);
            const uint32_t o = (uint32_t)half * (TC_T * 128) + sw128_offset((uint32_t)c, (uint32_t)q);
            *(float*)(A2 + o) = hi;
            *(float*)(A2 + 2 * TC_T * 128 + o) = lo;
            sDY[c * SDY_LD + b] = dy;
        }
        if (half) sGB[c] = gb;
        fence_async_smem();
        tc_before();
        __syncthreads();
        if (tid == 0) {  // GEMM2: dW2^T = dy^T h, 3xTF32, K = 64 in two k-blocks
            tc_after();
            const uint8_t* As[3] = {A2, A2, A2 + 2 * TC_T * 128};
            const uint8_t* Bs[3] = {B2, B2 + 2 * TC_H * 128, B2};
            uint32_t acc = 0;
#pragma unroll
            for (int term = 0; term < 3; ++term)
#pragma unroll
                for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        mma_tf32(tmem + TC_B, sdesc(smem_u32(As[term] + kb * TC_T * 128 + kk * 32)),
                                 sdesc(smem_u32(Bs[term] + kb * TC_H * 128 + kk * 32)), IDESC_GRAD, acc);
                        acc = 1;
                    }
            tc_commit(bar);
        }
        // dh += dy . W2_old^T over the tile (CUDA cores) while GEMM2 runs
#pragma unroll 4
        for (int tt = 0; tt < TC_T; ++tt) {
            const float2 d2 = *(const float2*)(sDY + tt * SDY_LD + b0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float wv = sW[(k0 + q) * SW_LD + tt];
                dh[0][q] = __fmaf_rn(d2.x, wv, dh[0][q]);
                dh[1][q] = __fmaf_rn(d2.y, wv, dh[1][q]);
            }
        }
        mbar_wait(bar, phase);
        phase ^= 1u;
        tc_after();
        float g[16];
        tmem_ld16(tmem + lane_base + (uint32_t)(TC_B + kh), g);
        if (live) {  // Adam on this thread's 16 entries of column j (approx.py:262-268)
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int k = kh + q;
                const int64_t o = (int64_t)k * ldw + j;
                float pw = sW[k * SW_LD + c], m = sM[k * SW_LD + c], vv = sV[k * SW_LD + c];
                adam(pw, m, vv, g[q], lr, omb1, omb2, bc1, bc2, eps);
                p.s.w2[o] = pw;
                p.s.m_w2[o] = m;
                p.s.v_w2[o] = vv;
            }
            if (!half) {  // b2 with db2 summed over both batch halves (rows 0-31, then 32-63)
                float pb = bj, m = p.s.m_b2[j], vv = p.s.v_b2[j];
                adam(pb, m, vv, __fadd_rn(gb, sGB[c]), lr, omb1, omb2, bc1, bc2, eps);
                p.s.b2[j] = pb;
                p.s.m_b2[j] = m;
                p.s.v_b2[j] = vv;
            }
        }
        tc_before();
        __syncthreads();  // the next tile rewrites the operands and the staged rows
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        atomicAdd(p.dh + b0 * TC_H + k0 + q, dh[0][q]);
        atomicAdd(p.dh + (b0 + 1) * TC_H + k0 + q, dh[1][q]);
    }
    tc_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(128));
}

__global__ void layer1_update_kernel(const __grid_constant__ TrainParams p) {
    const int B = p.B, H = p.s.hidden;
    __shared__ float s_dh[MAXB * MAXH];
    for (int i = threadIdx.x; i < B * H; i += blockDim.x) s_dh[i] = p.h[i] > 0.0f ? p.dh[i] : 0.0f;  // dh[pre <= 0] = 0
    __syncthreads();
    float bc1, bc2;
    bias_corrections(p.s, bc1, bc2);
    const float lr = p.s.lr, omb1 = __fsub_rn(1.0f, p.s.beta1), omb2 = __fsub_rn(1.0f, p.s.beta2), eps = p.s.eps;
    for (int i = threadIdx.x; i < 9 * H + H; i += blockDim.x) {
        float g = 0.0f;
        if (i < 9 * H) {  // dW1 = x^T dh
            const int e = i / H, k = i - e * H;
            for (int b = 0; b < B; ++b) g = __fmaf_rn(p.x[b * 9 + e], s_dh[b * H + k], g);
            adam(p.s.w1[i], p.s.m_w1[i], p.s.v_w1[i], g, lr, omb1, omb2, bc1, bc2, eps);
        } else {  // db1 = sum_b dh
            const int k = i - 9 * H;
            for (int b = 0; b < B; ++b) g = __fadd_rn(g, s_dh[b * H + k]);
            adam(p.s.b1[k], p.s.m_b1[k], p.s.v_b1[k], g, lr, omb1, omb2, bc1, bc2, eps);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *p.s.step += 1;
}

// Uniform rotations (approx.py:32-47): q ~ N(0, I_4) normalised, then the
// quaternion-to-matrix formula, fp64.  Rotation i of the stream uses the
// Philox subsequence offset + i of `seed`.
__global__ void sample_rotations_kernel(uint64_t seed, uint64_t offset, int64_t n, double* R) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    curandStatePhilox4_32_10_t st;
    curand_init(seed, offset + (uint64_t)i, 0, &st);
    const double2 a = curand_normal2_double(&st), c = curand_normal2_double(&st);
    double q[4] = {a.x, a.y, c.x, c.y};
    const double nrm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    for (int k = 0; k < 4; ++k) q[k] /= nrm;
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    double* o = R + 9 * i;
    o[0] = 1 - 2 * (y * y + z * z);
    o[1] = 2 * (x * y - w * z);
    o[2] = 2 * (x * z + w * y);
    o[3] = 2 * (x * y + w * z);
    o[4] = 1 - 2 * (x * x + z * z);
    o[5] = 2 * (y * z - w * x);
    o[6] = 2 * (x * z - w * y);
    o[7] = 2 * (y * z + w * x);
    o[8] = 1 - 2 * (x * x + y * y);
}

size_t step_smem(int B, int H) {
    return ((size_t)B * (TJ + 4) + (size_t)H * (TJ + 4) + 2 * (size_t)B * H + (size_t)B * 9) * sizeof(float);
}

}  // namespace

extern "C" int64_t lsdf_tmlp_train_workspace_bytes(int32_t B, int32_t H) {
    return (int64_t)B * (9 + 2 * H) * (int64_t)sizeof(float) + 256;
}

extern "C" int lsdf_tmlp_train_step(const lsdf_tmlp_train* state, const double* R_dev, int32_t B, void* workspace_dev,
                                    void* stream) {
    if (B < 2 || B > MAXB || (B & 1)) return fail(LSDF_ERR_VALIDATION, "train step: batch %d (even, 2..%d)", B, MAXB);
    if (state->hidden < 4 || state->hidden > MAXH || (state->hidden & 3))
        return fail(LSDF_ERR_UNSUPPORTED, "train step: hidden %d (multiple of 4, <= %d)", state->hidden, MAXH);
    if (state->n_out <= 0 || state->n_out % 3) return fail(LSDF_ERR_VALIDATION, "train step: n_out %lld", (long long)state->n_out);
    TrainParams p{};
    p.s = *state;
    p.B = B;
    p.R = R_dev;
    float* w = (float*)workspace_dev;
    p.x = w;
    p.h = p.x + (size_t)B * 9;
    p.dh = p.h + (size_t)B * state->hidden;
    cudaStream_t s = (cudaStream_t)stream;
    layer1_kernel<<<1, 256, 0, s>>>(p);
    LSDF_TRY(check_launch("layer1_kernel"));
    static const int t_tc = [] { const char* v = getenv("LSDF_TUNE_TRAINTC"); return v && *v ? atoi(v) : 1; }();
    if (t_tc && B == TC_B && state->hidden == TC_H) {  // forward and dW2 on the tensor cores
        const size_t smem_tc = tc_step_smem();
        LSDF_TRY(ensure_smem((const void*)layer2_tc_step_kernel, smem_tc, "layer2_tc_step_kernel"));
        int dev = 0, n_sm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        const int64_t n_tiles = (state->n_out + TC_T - 1) / TC_T;
        layer2_tc_step_kernel<<<(unsigned)(n_tiles < n_sm ? n_tiles : n_sm), TC_THREADS, smem_tc, s>>>(p);
        LSDF_TRY(check_launch("layer2_tc_step_kernel"));
        layer1_update_kernel<<<1, 256, 0, s>>>(p);
        return check_launch("layer1_update_kernel");
    }
    const size_t smem = step_smem(B, state->hidden);
    LSDF_TRY(ensure_smem((const void*)layer2_step_kernel, smem, "layer2_step_kernel"));
    int dev = 0, n_sm = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, layer2_step_kernel, THREADS, smem);
    const int64_t resident = (int64_t)n_sm * (per_sm < 1 ? 1 : per_sm);
    const int64_t n_tiles = (state->n_out + TJ - 1) / TJ;
    const unsigned grid = (unsigned)(n_tiles < resident ? n_tiles : resident);
    layer2_step_kernel<<<grid, THREADS, smem, s>>>(p);
    LSDF_TRY(check_launch("layer2_step_kernel"));
    layer1_update_kernel<<<1, 256, 0, s>>>(p);
    return check_launch("layer1_update_kernel");
}

extern "C" int lsdf_sample_rotations(uint64_t seed, uint64_t offset, int64_t n, double* R_dev, void* stream) {
    if (n <= 0) return LSDF_OK;
    sample_rotations_kernel<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(seed, offset, n, R_dev);
    return check_launch("sample_rotations_kernel");
}
