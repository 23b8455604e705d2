// lsdf_mlp_tc.cu — TinyMlp layer 2 on the 5th-generation tensor cores (tcgen05).
//
// y = h W2 + b2 with h = relu(x W1 + b1) (approx.py:123-130): B rotations,
// N = 3V window coordinates (up to 3.3 M), K = hidden (32).
//
// The product is computed transposed, y^T = W2^T h^T: the MMA's M side (128
// TMEM lanes) is 128 output coordinates and its N side (256 TMEM columns) is
// 256 rotations.  tcgen05.ld 32x32b then hands each thread ONE output
// coordinate for 32 consecutive rotations, so every global store of a warp is
// 32 consecutive floats of one row of y (a coalesced 128-B segment) straight
// from registers, with the bias a per-thread constant — no shared-memory
// transpose in the epilogue.
//
// layer1_pack_kernel (CUDA cores, K = 9) writes h for every rotation, split
// into TF32 hi/lo halves, straight into the K-major 128-byte-swizzled operand
// layout; pack_w2_kernel does the same for W2^T once per weight buffer, so
// every operand tile is one contiguous cp.async.bulk (UBLKCP) on an mbarrier.
//
// mlp_tc_kernel is warp-specialized and persistent over output tiles (each W2
// tile read once, all rotation tiles streamed past it): warp 0 issues the
// copies, one thread of warp 1 issues the 3xTF32 product as tcgen05.mma
// kind::tf32 (hi*hi + hi*lo + lo*hi, K = 8 per instruction) into a
// double-buffered 128 x 256 fp32 TMEM accumulator, warps 2-9 (two per TMEM
// lane quarter, one per rotation half) drain it with tcgen05.ld and store.
// 3xTF32 keeps ~fp32 accuracy, inside the 1e-5 (normalized) contract; the
// CUDA-core kernel (lsdf_mlp.cu) stays the bit-reproducing path.
#include "lsdf_async.cuh"
#include "lsdf_device.cuh"
#include "lsdf_tc.cuh"
#include "lsdf_common.cuh"

using namespace lsdf;

namespace {

constexpr int TM = 128;   // output coordinates per tile (tcgen05 M)
constexpr int TN = 256;   // rotations per tile (tcgen05 N)
constexpr int KB_BYTES_A = TM * 128;  // one 32-wide k-block of A (W2^T): 128 rows x 128 B
constexpr int KB_BYTES_B = TN * 128;  // one 32-wide k-block of B (h): 256 rows x 128 B
constexpr uint32_t IDESC = idesc_tf32(TM, TN);


// W2 (H, N) row-major -> per output tile, per k-block: 128 rows (outputs) x
// 128 B (32 hidden units), swizzled; hi and lo TF32 halves.
__global__ void pack_w2_kernel(const float* __restrict__ w2, int H, int64_t N, int kblocks, int64_t n_tiles,
                               float* hi, float* lo) {
    const int64_t total = n_tiles * kblocks * TM * 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tile = i / ((int64_t)kblocks * TM * 32);
        const int64_t rem = i % ((int64_t)kblocks * TM * 32);
        const int kb = (int)(rem / (TM * 32));
        const int r = (int)((rem / 32) % TM);
        const int kk = (int)(rem % 32);
        const int64_t n = tile * TM + r;
        const int k = kb * 32 + kk;
        const float v = (n < N && k < H) ? w2[(int64_t)k * N + n] : 0.0f;
        const float h = tf32_rna(v);
        const float l = tf32_rna(v - h);
        const int64_t base = (tile * kblocks + kb) * (int64_t)TM * 32;  // floats
        const uint32_t off = sw128_offset((uint32_t)r, (uint32_t)kk) >> 2;
        hi[base + off] = h;
        lo[base + off] = l;
    }
}

// Layer 1 (K = 9, CUDA cores) for every rotation, split into TF32 hi/lo and
// stored in the B-operand layout: [rotation tile][k_block][256 rows x 128 B, swizzled].
__global__ void layer1_pack_kernel(const float* __restrict__ w1, const float* __restrict__ b1, int H, int kblocks,
                                   const double* __restrict__ R, int64_t B, int64_t m_tiles, float* a_hi,
                                   float* a_lo, int64_t lm_C = 0, int32_t lm_L = 0) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= m_tiles * TN) return;
    // lm_C > 0: row r is rotation (c, l) = (r % lm_C, r / lm_C) of a configuration-major (C, L, 9) R
    const int64_t src = lm_C > 0 ? (row % lm_C) * lm_L + row / lm_C : row;
    float x[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) x[k] = row < B ? (float)R[src * 9 + k] : 0.0f;
    const int64_t mt = row / TN;
    const uint32_t r = (uint32_t)(row % TN);
    for (int j = 0; j < kblocks * 32; ++j) {
        float h = 0.0f;
        if (row < B && j < H) {
            float acc = __fmul_rn(x[0], __ldg(w1 + j));
#pragma unroll
            for (int k = 1; k < 9; ++k) acc = __fmaf_rn(x[k], __ldg(w1 + k * H + j), acc);
            acc = __fadd_rn(acc, __ldg(b1 + j));
            h = acc > 0.0f ? acc : 0.0f;
        }
        const float hh = tf32_rna(h);
        const float hl = tf32_rna(h - hh);
        const int64_t base = (mt * kblocks + (j >> 5)) * (int64_t)TN * 32;
        const uint32_t off = sw128_offset(r, (uint32_t)(j & 31)) >> 2;
        a_hi[base + off] = hh;
        a_lo[base + off] = hl;
    }
}

struct MlpTcParams {
    const float* h_hi;    // [rotation tile][k-block][256 x 32] swizzled
    const float* h_lo;
    const float* w2t_hi;  // [output tile][k-block][128 x 32] swizzled
    const float* w2t_lo;
    const float* b2;
    float* y;
    int64_t ldy;  // row stride of y (elements)
    int64_t B, N, n_tiles, r_tiles;
    int32_t kblocks;
};

// Warp roles: warp 0 = bulk-copy producer, warp 1 = MMA issuer, warps 2-9 =
// epilogue (warp w drains TMEM lanes 32*(w % 4) .. +31 = 32 outputs, rotation
// half (w-2)/4).  Persistent over output tiles (each W2 tile is read once),
// looping over all rotation tiles inside; rotation tiles and TMEM
// accumulators are double-buffered so the epilogue of one tile overlaps the
// copies and MMAs of the next.
constexpr int EP_WARPS = 8;
constexpr int TC_THREADS = 64 + 32 * EP_WARPS;

__global__ void __launch_bounds__(TC_THREADS, 1) mlp_tc_kernel(const __grid_constant__ MlpTcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int kb = p.kblocks;
    const uint32_t a_bytes = (uint32_t)kb * KB_BYTES_A;  // W2 tile, one term (hi or lo)
    const uint32_t b_bytes = (uint32_t)kb * KB_BYTES_B;  // rotation tile, one term
    uint8_t* At = smem;                    // W2^T [hi | lo]
    uint8_t* Bt = At + 2 * a_bytes;        // h [stage][hi | lo]
    uint64_t* bars = (uint64_t*)(Bt + 4 * b_bytes);
    uint64_t* wfull = bars + 0;
    uint64_t* wempty = bars + 1;
    uint64_t* hfull = bars + 2;   // [2]
    uint64_t* hempty = bars + 4;  // [2]
    uint64_t* tfull = bars + 6;   // [2]
    uint64_t* tempty = bars + 8;  // [2]
    uint32_t* tmem_slot = (uint32_t*)(bars + 10);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "r"(2 * TN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (threadIdx.x == 32) {
        mbar_init(wfull, 1);
        mbar_init(wempty, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(hfull + i, 1);
            mbar_init(hempty + i, 1);
            mbar_init(tfull + i, 1);
            mbar_init(tempty + i, EP_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- producer
            uint32_t it = 0, nc = 0;
            for (int64_t nt = blockIdx.x; nt < p.n_tiles; nt += gridDim.x, ++nc) {
                if (nc > 0) mbar_wait(wempty, (nc - 1) & 1);
                mbar_expect_tx(wfull, 2 * a_bytes);
                bulk_copy(At, p.w2t_hi + nt * (int64_t)kb * TM * 32, a_bytes, wfull);
                bulk_copy(At + a_bytes, p.w2t_lo + nt * (int64_t)kb * TM * 32, a_bytes, wfull);
                for (int64_t rt = 0; rt < p.r_tiles; ++rt, ++it) {
                    const uint32_t s = it & 1, use = it >> 1;
                    if (it >= 2) mbar_wait(hempty + s, (use - 1) & 1);
                    uint8_t* dst = Bt + s * 2 * b_bytes;
                    mbar_expect_tx(hfull + s, 2 * b_bytes);
                    bulk_copy(dst, p.h_hi + rt * (int64_t)kb * TN * 32, b_bytes, hfull + s);
                    bulk_copy(dst + b_bytes, p.h_lo + rt * (int64_t)kb * TN * 32, b_bytes, hfull + s);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            uint32_t it = 0, nc = 0;
            for (int64_t nt = blockIdx.x; nt < p.n_tiles; nt += gridDim.x, ++nc) {
                mbar_wait(wfull, nc & 1);
                for (int64_t rt = 0; rt < p.r_tiles; ++rt, ++it) {
                    const uint32_t s = it & 1, acc_buf = it & 1;
                    mbar_wait(hfull + s, (it >> 1) & 1);
                    if (it >= 2) mbar_wait(tempty + acc_buf, ((it >> 1) - 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                    const uint8_t* Hh = Bt + s * 2 * b_bytes;
                    const uint8_t* As[3] = {At, At, At + a_bytes};  // W2 hi, hi, lo
                    const uint8_t* Bs[3] = {Hh, Hh + b_bytes, Hh};  // h  hi, lo, hi
                    const uint32_t d = tmem + acc_buf * TN;
                    uint32_t accumulate = 0;
#pragma unroll
                    for (int term = 0; term < 3; ++term)
                        for (int b = 0; b < kb; ++b)
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                mma_tf32(d, sdesc(smem_u32(As[term] + b * KB_BYTES_A + kk * 32)),
                                         sdesc(smem_u32(Bs[term] + b * KB_BYTES_B + kk * 32)), IDESC, accumulate);
                                accumulate = 1;
                            }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                     smem_u32(hempty + s))
                                 : "memory");
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                     smem_u32(tfull + acc_buf))
                                 : "memory");
                    if (rt == p.r_tiles - 1)
                        asm volatile(
                            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                smem_u32(wempty))
                            : "memory");
                }
            }
        }
    } else {  // ---------------- epilogue warps 2..(2 + EP_WARPS)
        const int q = warp & 3;           // TMEM lane quarter = 32 outputs
        const int half = (warp - 2) / 4;  // rotation half of the tile
        uint32_t it = 0;
        for (int64_t nt = blockIdx.x; nt < p.n_tiles; nt += gridDim.x) {
            const int64_t n = nt * TM + q * 32 + lane;  // this thread's output coordinate
            const bool col_ok = n < p.N;
            const float bias = col_ok ? __ldg(p.b2 + n) : 0.0f;
            for (int64_t rt = 0; rt < p.r_tiles; ++rt, ++it) {
                const uint32_t acc_buf = it & 1;
                mbar_wait(tfull + acc_buf, (it >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                const int64_t b0 = rt * TN + half * (TN / 2);
                float* dst = p.y + b0 * p.ldy + n;
#pragma unroll 1
                for (int c0 = 0; c0 < TN / 2; c0 += 32) {
                    float v[32];
                    const uint32_t ta =
                        tmem + acc_buf * TN + ((uint32_t)(q * 32) << 16) + (uint32_t)(half * (TN / 2) + c0);
                    tmem_ld16(ta, v);
                    tmem_ld16(ta + 16, v + 16);
                    const int64_t nb = p.B - (b0 + c0);  // rotations left from this chunk
                    if (col_ok) {
                        if (nb >= 32) {
#pragma unroll
                            for (int j = 0; j < 32; ++j) __stcs(dst + (int64_t)(c0 + j) * p.ldy, v[j] + bias);
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (j < nb) __stcs(dst + (int64_t)(c0 + j) * p.ldy, v[j] + bias);
                        }
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(tempty + acc_buf))
                                            : "memory");
            }
        }
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * TN));
}

// ---------------------------------------------------------------- fused placement
// NeuralTransformProvider placement (approx.py:292-306 -> placement.py:300-313)
// without materializing G: the MLP's layer 2 for a block of 128 kept cells and
// 128 rotations runs as three MMAs (the cells' x, y and z coordinates: W2 is
// packed so that tile (cb, k3) holds the rows 3(128 cb + i) + k3), into three
// TMEM accumulators; the epilogue adds b2 (f32), the fp64 shift -(dt/e_r) R,
// scales by e_r and samples the link's packed-corner grid, writing one window
// value per (rotation, cell) instead of three G coordinates.  Rotations are
// ordered link-major (r = l C + c) so a tile samples one or two link grids.
constexpr int PC = 128;   // cells per block (MMA M)
constexpr int PR = 128;   // rotations per tile (MMA N)
constexpr int P_THREADS = 1024;
constexpr uint32_t IDESC_PLACE = idesc_tf32(PC, PR);

// W2 (H <= 32, 3V) -> [cell block][k3][128 rows x 128 B] swizzled, hi and lo halves.
__global__ void pack_w2_cells_kernel(const float* __restrict__ w2, int H, int64_t V, int64_t n_cb, float* hi,
                                     float* lo) {
    const int64_t total = n_cb * 3 * PC * 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tile = i / (PC * 32);  // cb * 3 + k3
        const int r = (int)((i / 32) % PC), kk = (int)(i % 32);
        const int64_t cb = tile / 3;
        const int k3 = (int)(tile % 3);
        const int64_t v = cb * PC + r;
        const float x = (v < V && kk < H) ? w2[(int64_t)kk * 3 * V + 3 * v + k3] : 0.0f;
        const float h = tf32_rna(x), l = tf32_rna(x - h);
        const int64_t base = tile * (int64_t)PC * 32;
        const uint32_t off = sw128_offset((uint32_t)r, (uint32_t)kk) >> 2;
        hi[base + off] = h;
        lo[base + off] = l;
    }
}

struct PlaceTcParams {
    const float* w2c_hi;   // pack_w2_cells_kernel output
    const float* w2c_lo;
    const float* h_hi;     // layer1_pack_kernel output for the link-major rotations (256-row tiles)
    const float* h_lo;
    const float* b2;       // (3V)
    const double* R;       // (C, L, 9) configuration-major
    const double* dt;      // (C, L, 3)
    const int32_t* kept;   // V kept cells -> cell index in the W^3 window (x-fastest)
    float* out;            // (C * L, n_cells)
    int64_t C, V, n_cb, r_tiles, n_cells;
    int32_t L;
    double e_r;
    PackedGrid grids[LSDF_MAX_LINKS];  // sampler constants per link, read through the constant cache
};

// Each CTA owns whole cell blocks (its W2 tile is loaded once per block) and
// walks the rotation tiles in order, so CTAs running together sample the same
// link grid; the h tile of the next item is prefetched into the other buffer
// while the epilogue of this one samples.
__global__ void __launch_bounds__(P_THREADS, 1) mlp_place_tc_kernel(const __grid_constant__ PlaceTcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* W = sm;                                   // [hi | lo][k3] 128 x 128 B
    uint8_t* Hs = W + 2 * 3 * PC * 128;                // [buffer][hi | lo] 128 x 128 B
    double* s_dti = (double*)(Hs + 2 * 2 * PR * 128);  // [PR][3] shift of each rotation
    int64_t* s_row = (int64_t*)(s_dti + 3 * PR);       // [PR] output row offset f * n_cells (-1: past B)
    int32_t* s_link = (int32_t*)(s_row + PR);          // [PR] link of each rotation
    uint64_t* bars = (uint64_t*)(s_link + PR);         // [0,1] operand buffers, [2] MMAs
    uint32_t* tmem_slot = (uint32_t*)(bars + 3);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        mbar_init(bars, 1);
        mbar_init(bars + 1, 1);
        mbar_init(bars + 2, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const int q = warp & 3, grp = warp >> 2;  // TMEM lane quarter (cells), rotation group (16 rotations)
    const int64_t B = p.C * p.L;
    // this CTA's items: cell blocks blockIdx.x, + gridDim.x, ..., each with all rotation tiles
    const int64_t my_cb = p.n_cb > (int64_t)blockIdx.x ? (p.n_cb - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t n_my = my_cb * p.r_tiles;
    auto issue = [&](int64_t k, int buf) {  // copies of this CTA's k-th item into buffer buf
        const int64_t cb = blockIdx.x + (k / p.r_tiles) * gridDim.x, rt = k % p.r_tiles;
        const bool new_w = rt == 0;
        mbar_expect_tx(bars + buf, (new_w ? 2 * 3 * PC * 128 : 0) + 2 * PR * 128);
        if (new_w)
            for (int half = 0; half < 2; ++half)
                bulk_copy(W + half * 3 * PC * 128, (half ? p.w2c_lo : p.w2c_hi) + cb * 3 * PC * 32, 3 * PC * 128,
                          bars + buf);
        // the 128-rotation half of a 256-row layer-1 tile
        const int64_t h_off = (rt >> 1) * (int64_t)256 * 32 + (rt & 1) * (int64_t)PR * 32;
        uint8_t* Hb = Hs + buf * 2 * PR * 128;
        bulk_copy(Hb, p.h_hi + h_off, PR * 128, bars + buf);
        bulk_copy(Hb + PR * 128, p.h_lo + h_off, PR * 128, bars + buf);
    };
    if (tid == 0 && n_my > 0) issue(0, 0);
    for (int64_t k = 0; k < n_my; ++k) {
        const int buf = (int)(k & 1);
        const int64_t cb = blockIdx.x + (k / p.r_tiles) * gridDim.x, rt = k % p.r_tiles;
        if (tid < PR) {  // the fp64 shift -(dt / e_r) R of each rotation (placement.py:164-167)
            const int64_t r = rt * PR + tid;
            s_row[tid] = -1;
            s_link[tid] = 0;
            if (r < B) {
                const int64_t l = r / p.C, c = r - l * p.C, f = c * p.L + l;
                double Rr[9];
#pragma unroll
                for (int e = 0; e < 9; ++e) Rr[e] = p.R[f * 9 + e];
                shift_inverse(Rr, p.dt + f * 3, p.e_r, s_dti + 3 * tid);
                s_row[tid] = f * p.n_cells;
                s_link[tid] = (int32_t)l;
            }
        }
        __syncthreads();
        if (tid == 0) {
            mbar_wait(bars + buf, (uint32_t)((k >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint8_t* Hb = Hs + buf * 2 * PR * 128;
            for (int k3 = 0; k3 < 3; ++k3) {
                const uint8_t* Wh = W + k3 * PC * 128;
                const uint8_t* Wl = W + 3 * PC * 128 + k3 * PC * 128;
                const uint8_t* As[3] = {Wh, Wh, Wl};
                const uint8_t* Bs[3] = {Hb, Hb + PR * 128, Hb};
                uint32_t acc = 0;
#pragma unroll
                for (int term = 0; term < 3; ++term)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        mma_tf32(tmem + (uint32_t)(k3 * PR), sdesc(smem_u32(As[term] + kk * 32)),
                                 sdesc(smem_u32(Bs[term] + kk * 32)), IDESC_PLACE, acc);
                        acc = 1;
                    }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             smem_u32(bars + 2))
                         : "memory");
            mbar_wait(bars + 2, (uint32_t)(k & 1));
            // the operands of item k are consumed: prefetch item k + 1 (W only at a new cell block)
            if (k + 1 < n_my) issue(k + 1, buf ^ 1);
        }
        mbar_wait(bars + 2, (uint32_t)(k & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        // epilogue: cell v of lane quarter q, 16 rotations of group grp
        const int64_t v = cb * PC + q * 32 + lane;
        const bool cell_ok = v < p.V;
        const float bx = cell_ok ? __ldg(p.b2 + 3 * v) : 0.f, by = cell_ok ? __ldg(p.b2 + 3 * v + 1) : 0.f,
                    bz = cell_ok ? __ldg(p.b2 + 3 * v + 2) : 0.f;
        const int64_t cell = cell_ok ? __ldg(p.kept + v) : 0;
        const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
        for (int c0 = 0; c0 < 16; c0 += 8) {
            const int col = grp * 16 + c0;
            float gx[8], gy[8], gz[8];
            tmem_ld8(tl + (uint32_t)col, gx);
            tmem_ld8(tl + (uint32_t)(PR + col), gy);
            tmem_ld8(tl + (uint32_t)(2 * PR + col), gz);
#pragma unroll 2
            for (int j = 0; j < 8; ++j) {
                const int64_t row = s_row[col + j];
                if (row < 0 || !cell_ok) continue;
                const double* dti = s_dti + 3 * (col + j);
                // G = y (f32, + b2 in f32 as TinyMlp.predict) + dt_inv (fp64), point = G e_r
                const double px = DMUL(DADD((double)__fadd_rn(gx[j], bx), dti[0]), p.e_r);
                const double py = DMUL(DADD((double)__fadd_rn(gy[j], by), dti[1]), p.e_r);
                const double pz = DMUL(DADD((double)__fadd_rn(gz[j], bz), dti[2]), p.e_r);
                __stcs(p.out + row + cell, trilinear_packed(p.grids[s_link[col + j]], px, py, pz));
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();  // TMEM and the shift tables are rewritten by the next item
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

// masked window cells carry the link's sentinel (placement.py:305-308)
__global__ void fill_masked_kernel(const uint32_t* __restrict__ mask_bits, int64_t n_cells, int64_t C, int32_t L,
                                   const float* d_far, float* out) {
    const int64_t f = blockIdx.y;  // field c * L + l
    fill_masked_cells(mask_bits, n_cells, out + f * n_cells, d_far[f % L],
                      (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

}  // namespace

int64_t lsdf_mlp_cells_packed_bytes(int32_t H, int64_t V) {
    (void)H;
    const int64_t n_cb = (V + PC - 1) / PC;
    return 2 * n_cb * 3 * PC * 32 * (int64_t)sizeof(float);
}

int lsdf_mlp_pack_cells(const float* w2, int32_t H, int64_t V, float* packed, cudaStream_t s) {
    if (H > 32) return fail(LSDF_ERR_UNSUPPORTED, "fused TinyMlp placement supports hidden <= 32");
    const int64_t n_cb = (V + PC - 1) / PC;
    float* hi = packed;
    float* lo = packed + n_cb * 3 * PC * 32;
    pack_w2_cells_kernel<<<148 * 8, 256, 0, s>>>(w2, H, V, n_cb, hi, lo);
    return check_launch("pack_w2_cells_kernel");
}

int lsdf_mlp_place_tc(const float* w1, const float* b1, const float* w2_cells_packed, const float* b2, int32_t H,
                      int64_t V, const int32_t* kept_cells, const double* R, const double* dt, int64_t C, int32_t L,
                      const lsdf_link_grid* grids, const lsdf_window* window, float* out, cudaStream_t s) {
    if (H > 32) return fail(LSDF_ERR_UNSUPPORTED, "fused TinyMlp placement supports hidden <= 32");
    if (L < 1 || L > LSDF_MAX_LINKS) return fail(LSDF_ERR_VALIDATION, "fused placement: %d links", L);
    if (V != window->n_masked) return fail(LSDF_ERR_VALIDATION, "fused placement: %lld cells for a %d-cell window",
                                            (long long)V, window->n_masked);
    const int64_t B = C * L;
    if (B <= 0) return LSDF_OK;
    for (int l = 0; l < L; ++l)
        if (grids[l].packed_dev == nullptr) return fail(LSDF_ERR_VALIDATION, "fused placement: link %d unpacked", l);
    const int kblocks = 1;
    const int64_t r_tiles256 = (B + TN - 1) / TN;
    const size_t h_bytes = (size_t)r_tiles256 * kblocks * TN * 32 * sizeof(float);
    float *a_hi = nullptr, *a_lo = nullptr;
    LSDF_TRY(check_cuda(cudaMallocAsync((void**)&a_hi, h_bytes, s), "mlp place h alloc"));
    LSDF_TRY(check_cuda(cudaMallocAsync((void**)&a_lo, h_bytes, s), "mlp place h alloc"));
    layer1_pack_kernel<<<grid_for(r_tiles256 * TN, 128), 128, 0, s>>>(w1, b1, H, kblocks, R, B, r_tiles256, a_hi,
                                                                       a_lo, C, L);
    LSDF_TRY(check_launch("layer1_pack_kernel"));
    const int64_t n_cells = (int64_t)window->W[0] * window->W[1] * window->W[2];
    float dfar[LSDF_MAX_LINKS];
    for (int l = 0; l < L; ++l) dfar[l] = grids[l].d_far;
    float* dfar_dev = nullptr;
    LSDF_TRY(check_cuda(cudaMallocAsync((void**)&dfar_dev, sizeof(dfar), s), "dfar alloc"));
    LSDF_TRY(check_cuda(cudaMemcpyAsync(dfar_dev, dfar, sizeof(float) * L, cudaMemcpyHostToDevice, s), "dfar copy"));
    fill_masked_kernel<<<dim3((unsigned)((n_cells + 1023) / 1024 < 32 ? (n_cells + 1023) / 1024 : 32), (unsigned)B), 256, 0,
                         s>>>((const uint32_t*)window->mask_bits_dev, n_cells, C, L, dfar_dev, out);
    LSDF_TRY(check_launch("fill_masked_kernel"));
    PlaceTcParams p{};
    const int64_t n_cb = (V + PC - 1) / PC;
    p.w2c_hi = w2_cells_packed;
    p.w2c_lo = w2_cells_packed + n_cb * 3 * PC * 32;
    p.h_hi = a_hi;
    p.h_lo = a_lo;
    p.b2 = b2;
    p.R = R;
    p.dt = dt;
    p.kept = kept_cells;
    p.out = out;
    p.C = C;
    p.V = V;
    p.n_cb = n_cb;
    p.r_tiles = (B + PR - 1) / PR;
    p.n_cells = n_cells;
    p.L = L;
    p.e_r = window->e_r;
    for (int l = 0; l < L; ++l) p.grids[l] = packed_of(grids[l]);
    const size_t smem = 1024 + 2 * 3 * PC * 128 + 2 * 2 * PR * 128 + PR * (3 * sizeof(double) + 8 + 4) + 64;
    LSDF_TRY(ensure_smem((const void*)mlp_place_tc_kernel, smem, "mlp_place_tc_kernel"));
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    mlp_place_tc_kernel<<<(unsigned)(n_cb < n_sm ? n_cb : n_sm), P_THREADS, smem, s>>>(p);
    LSDF_TRY(check_launch("mlp_place_tc_kernel"));
    cudaFreeAsync(a_hi, s);
    cudaFreeAsync(a_lo, s);
    cudaFreeAsync(dfar_dev, s);
    return LSDF_OK;
}

// Packed W2^T (hi | lo TF32 halves, swizzled output tiles): bytes and fill.
int64_t lsdf_mlp_packed_bytes_tc(int32_t H, int64_t n_out) {
    const int kblocks = (H + 31) / 32;
    const int64_t n_tiles = (n_out + TM - 1) / TM;
    return 2 * n_tiles * kblocks * TM * 32 * (int64_t)sizeof(float);
}

int lsdf_mlp_pack_tc(const float* w2, int32_t H, int64_t n_out, float* packed, cudaStream_t s) {
    using namespace lsdf;
    const int kblocks = (H + 31) / 32;
    const int64_t n_tiles = (n_out + TM - 1) / TM;
    float* hi = packed;
    float* lo = packed + n_tiles * kblocks * TM * 32;
    pack_w2_kernel<<<148 * 8, 256, 0, s>>>(w2, H, n_out, kblocks, n_tiles, hi, lo);
    return check_launch("pack_w2_kernel");
}

// w2_packed: lsdf_mlp_pack_tc output for these weights (kept by the caller
// and re-packed whenever W2 changes), or null to pack into a temporary.
int lsdf_mlp_predict_tc(const float* w1, const float* b1, const float* w2, const float* w2_packed, const float* b2,
                        int32_t H, int64_t n_out, const double* R, int64_t B, float* y, int64_t ldy, cudaStream_t s) {
    using namespace lsdf;
    if (H > 64) return fail(LSDF_ERR_UNSUPPORTED, "tcgen05 TinyMlp supports hidden <= 64");
    const int kblocks = (H + 31) / 32;
    const int64_t n_tiles = (n_out + TM - 1) / TM;
    float* tmp = nullptr;
    if (w2_packed == nullptr) {
        LSDF_TRY(check_cuda(cudaMallocAsync((void**)&tmp, (size_t)lsdf_mlp_packed_bytes_tc(H, n_out), s),
                            "mlp pack alloc"));
        LSDF_TRY(lsdf_mlp_pack_tc(w2, H, n_out, tmp, s));
        w2_packed = tmp;
    }
    const float* w2_hi = w2_packed;
    const float* w2_lo = w2_packed + n_tiles * kblocks * TM * 32;
    const int64_t r_tiles = (B + TN - 1) / TN;
    const size_t h_bytes = (size_t)r_tiles * kblocks * TN * 32 * sizeof(float);
    float *a_hi = nullptr, *a_lo = nullptr;
    LSDF_TRY(check_cuda(cudaMallocAsync((void**)&a_hi, h_bytes, s), "mlp h alloc"));
    LSDF_TRY(check_cuda(cudaMallocAsync((void**)&a_lo, h_bytes, s), "mlp h alloc"));
    layer1_pack_kernel<<<grid_for(r_tiles * TN, 128), 128, 0, s>>>(w1, b1, H, kblocks, R, B, r_tiles, a_hi, a_lo);
    LSDF_TRY(check_launch("layer1_pack_kernel"));
    MlpTcParams p{};
    p.h_hi = a_hi;
    p.h_lo = a_lo;
    p.w2t_hi = w2_hi;
    p.w2t_lo = w2_lo;
    p.b2 = b2;
    p.y = y;
    p.ldy = ldy;
    p.B = B;
    p.N = n_out;
    p.n_tiles = n_tiles;
    p.r_tiles = r_tiles;
    p.kblocks = kblocks;
    const size_t smem = 1024 + (size_t)kblocks * (2 * KB_BYTES_A + 4 * KB_BYTES_B) + 128;
    if (smem > 227 * 1024) return fail(LSDF_ERR_UNSUPPORTED, "tcgen05 TinyMlp: hidden %d needs too much smem", H);
    LSDF_TRY(ensure_smem((const void*)mlp_tc_kernel, smem, "mlp_tc_kernel"));
    const unsigned grid = (unsigned)(n_tiles < 148 ? n_tiles : 148);
    mlp_tc_kernel<<<grid, TC_THREADS, smem, s>>>(p);
    LSDF_TRY(check_launch("mlp_tc_kernel"));
    cudaFreeAsync(a_hi, s);
    cudaFreeAsync(a_lo, s);
    if (tmp) cudaFreeAsync(tmp, s);
    return LSDF_OK;

}
