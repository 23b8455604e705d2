// lsdf_mlp_tc.cu — TinyMlp layer 2 on the 5th-generation tensor cores (tcgen05).
//
// y = h W2 + b2 with h = relu(x W1 + b1) (approx.py:123-130): M = rotations,
// N = 3V window coordinates (up to 3.3 M), K = hidden (32).  One CTA owns a
// 128-row M tile: it computes its h rows on CUDA cores (K = 9 layer), splits
// them into TF32 hi/lo halves and keeps them in shared memory (K-major,
// 128-byte swizzle).  It then streams N tiles of 256 outputs: the matching
// W2^T tile (pre-split hi/lo and pre-swizzled at model upload, so the copy is
// a single bulk async copy — cp.async.bulk, the TMA engine — completing on an
// mbarrier) lands in shared memory, one elected thread issues the 3xTF32
// product as tcgen05.mma kind::tf32 (hi*hi + hi*lo + lo*hi, K = 8 per
// instruction) into a 128 x 256 fp32 TMEM accumulator, commits to an mbarrier,
// and the four warps drain TMEM with tcgen05.ld, add b2 and store y.
// 3xTF32 keeps ~fp32 accuracy (|err| <= ~1e-6 relative), well inside the
// 1e-5 (normalized) contract; the CUDA-core kernel (lsdf_mlp.cu) stays the
// bit-reproducing path.
#include "lsdf_common.cuh"

namespace {

constexpr int TM = 128;   // rows per tile (tcgen05 M)
constexpr int TN = 256;   // outputs per tile (tcgen05 N)
constexpr int KB_BYTES_A = TM * 128;  // one 32-wide k-block of A: 128 rows x 128 B
constexpr int KB_BYTES_B = TN * 128;  // one 32-wide k-block of B: 256 rows x 128 B
constexpr int THREADS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of element (row, k) inside a K-major, 128B-swizzled k-block
__host__ __device__ __forceinline__ uint32_t sw128_offset(uint32_t row, uint32_t k) {
    return row * 128u + ((((k >> 2) ^ (row & 7u)) & 7u) << 4) + ((k & 3u) << 2);
}

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// Bounded wait: a lost arrival traps (a kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    for (uint32_t spin = 0; spin < (1u << 26); ++spin) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) return;
    }
    __trap();
}

__device__ __forceinline__ void bulk_copy(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(smem_dst)),
                 "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// tcgen05 shared-memory matrix descriptor: K-major, 128-byte swizzle,
// 8-row groups 1024 B apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = 256
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// W2 (H, N) row-major -> per N tile, per k-block: 256 rows x 128 B, swizzled; hi and lo TF32 halves.
__global__ void pack_w2_kernel(const float* __restrict__ w2, int H, int64_t N, int kblocks, int64_t n_tiles,
                               float* hi, float* lo) {
    const int64_t total = n_tiles * kblocks * TN * 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tile = i / ((int64_t)kblocks * TN * 32);
        const int64_t rem = i % ((int64_t)kblocks * TN * 32);
        const int kb = (int)(rem / (TN * 32));
        const int r = (int)((rem / 32) % TN);
        const int kk = (int)(rem % 32);
        const int64_t n = tile * TN + r;
        const int k = kb * 32 + kk;
        const float v = (n < N && k < H) ? w2[(int64_t)k * N + n] : 0.0f;
        const float h = tf32_rna(v);
        const float l = tf32_rna(v - h);
        const int64_t base = (tile * kblocks + kb) * (int64_t)TN * 32;  // floats
        const uint32_t off = sw128_offset((uint32_t)r, (uint32_t)kk) >> 2;
        hi[base + off] = h;
        lo[base + off] = l;
    }
}

struct MlpTcParams {
    const float* w1;
    const float* b1;
    const float* b2;
    const float* w2t_hi;
    const float* w2t_lo;
    const double* R;
    float* y;
    int64_t B, N, n_tiles;
    int32_t H, kblocks;
};

__global__ void __launch_bounds__(THREADS, 1) mlp_tc_kernel(const __grid_constant__ MlpTcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for the swizzled tiles
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int kb = p.kblocks;
    uint8_t* A_hi = smem;
    uint8_t* A_lo = A_hi + kb * KB_BYTES_A;
    uint8_t* B_hi = A_lo + kb * KB_BYTES_A;
    uint8_t* B_lo = B_hi + kb * KB_BYTES_B;
    uint64_t* bars = (uint64_t*)(B_lo + kb * KB_BYTES_B);  // [0] load, [1] mma
    uint32_t* tmem_slot = (uint32_t*)(bars + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t m0 = (int64_t)blockIdx.y * TM;

    // ---- layer 1 (K = 9) on CUDA cores: row tid of this tile
    {
        const int64_t row = m0 + tid;
        float x[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) x[k] = row < p.B ? (float)p.R[row * 9 + k] : 0.0f;
        for (int j = 0; j < kb * 32; ++j) {
            float h = 0.0f;
            if (row < p.B && j < p.H) {
                float acc = __fmul_rn(x[0], __ldg(p.w1 + j));
#pragma unroll
                for (int k = 1; k < 9; ++k) acc = __fmaf_rn(x[k], __ldg(p.w1 + k * p.H + j), acc);
                acc = __fadd_rn(acc, __ldg(p.b1 + j));
                h = acc > 0.0f ? acc : 0.0f;
            }
            const float hh = tf32_rna(h);
            const float hl = tf32_rna(h - hh);
            const uint32_t off = (uint32_t)(j >> 5) * KB_BYTES_A + sw128_offset((uint32_t)tid, (uint32_t)(j & 31));
            *(float*)(A_hi + off) = hh;
            *(float*)(A_lo + off) = hl;
        }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic stores -> async proxy (MMA)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "r"(TN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 32) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const uint32_t tile_bytes = (uint32_t)kb * KB_BYTES_B;
    uint32_t phase = 0;

    for (int64_t nt = blockIdx.x; nt < p.n_tiles; nt += gridDim.x) {
        if (tid == 0) {
            mbar_expect_tx(&bars[0], 2 * tile_bytes);
            bulk_copy(B_hi, p.w2t_hi + nt * (int64_t)kb * TN * 32, tile_bytes, &bars[0]);
            bulk_copy(B_lo, p.w2t_lo + nt * (int64_t)kb * TN * 32, tile_bytes, &bars[0]);
            mbar_wait(&bars[0], phase);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint8_t* As[3] = {A_hi, A_hi, A_lo};
            const uint8_t* Bs[3] = {B_hi, B_lo, B_hi};
            uint32_t acc = 0;
#pragma unroll
            for (int term = 0; term < 3; ++term)
                for (int b = 0; b < kb; ++b)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {  // K = 8 tf32 (32 B) per instruction
                        const uint64_t ad = sdesc(smem_u32(As[term] + b * KB_BYTES_A + kk * 32));
                        const uint64_t bd = sdesc(smem_u32(Bs[term] + b * KB_BYTES_B + kk * 32));
                        mma_tf32(tmem, ad, bd, acc);
                        acc = 1;
                    }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             smem_u32(&bars[1]))
                         : "memory");
        }
        __syncwarp();
        mbar_wait(&bars[1], phase);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        // ---- epilogue: warp w owns TMEM lanes [32w, 32w + 32) = rows of the tile
        const int64_t row = m0 + warp * 32 + lane;
        const int64_t n0 = nt * TN;
        for (int c0 = 0; c0 < TN; c0 += 16) {
            float v[16];
            tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
            if (row < p.B) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int64_t n = n0 + c0 + i;
                    if (n < p.N) p.y[row * p.N + n] = v[i] + __ldg(p.b2 + n);
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        phase ^= 1;
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TN));
}

struct PackCache {
    const float* w2 = nullptr;
    int64_t N = 0;
    int H = 0;
    float* hi = nullptr;
    float* lo = nullptr;
};
PackCache g_pack;

}  // namespace

// Pre-split / pre-swizzle W2 once per weight buffer (cached by pointer+shape).
int lsdf_mlp_predict_tc(const float* w1, const float* b1, const float* w2, const float* b2, int32_t H, int64_t n_out,
                        const double* R, int64_t B, float* y, cudaStream_t s) {
    using namespace lsdf;
    if (H > 64) return fail(LSDF_ERR_UNSUPPORTED, "tcgen05 TinyMlp supports hidden <= 64");
    const int kblocks = (H + 31) / 32;
    const int64_t n_tiles = (n_out + TN - 1) / TN;
    if (g_pack.w2 != w2 || g_pack.N != n_out || g_pack.H != H) {
        if (g_pack.hi) cudaFreeAsync(g_pack.hi, s);
        if (g_pack.lo) cudaFreeAsync(g_pack.lo, s);
        const size_t bytes = (size_t)n_tiles * kblocks * TN * 32 * sizeof(float);
        LSDF_TRY(check_cuda(cudaMallocAsync((void**)&g_pack.hi, bytes, s), "mlp pack alloc"));
        LSDF_TRY(check_cuda(cudaMallocAsync((void**)&g_pack.lo, bytes, s), "mlp pack alloc"));
        pack_w2_kernel<<<148 * 8, 256, 0, s>>>(w2, H, n_out, kblocks, n_tiles, g_pack.hi, g_pack.lo);
        LSDF_TRY(check_launch("pack_w2_kernel"));
        g_pack.w2 = w2;
        g_pack.N = n_out;
        g_pack.H = H;
    }
    MlpTcParams p{};
    p.w1 = w1;
    p.b1 = b1;
    p.b2 = b2;
    p.w2t_hi = g_pack.hi;
    p.w2t_lo = g_pack.lo;
    p.R = R;
    p.y = y;
    p.B = B;
    p.N = n_out;
    p.n_tiles = n_tiles;
    p.H = H;
    p.kblocks = kblocks;
    const size_t smem = 1024 + (size_t)kblocks * (2 * KB_BYTES_A + 2 * KB_BYTES_B) + 64;
    static bool attr = false;
    if (!attr) {
        LSDF_TRY(check_cuda(cudaFuncSetAttribute(mlp_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024),
                            "mlp smem attribute"));
        attr = true;
    }
    const int64_t m_tiles = (B + TM - 1) / TM;
    int64_t gx = (148 + m_tiles - 1) / m_tiles;  // enough CTAs to fill the machine
    gx = gx < 1 ? 1 : (gx > n_tiles ? n_tiles : gx);
    dim3 grid((unsigned)gx, (unsigned)m_tiles);
    mlp_tc_kernel<<<grid, THREADS, smem, s>>>(p);
    return check_launch("mlp_tc_kernel");
}
