// fold_tc.cuh — offline fold of the rotation into the weights on the 5th-generation tensor
// cores (eqs. before_merge -> after_merge; §3.2):
//   LEFT  (W_qkv, W_gate|up, adapter):  Wout[i][o] = sum_m Q[m][i] gamma[m] W[m][o]
//   RIGHT (W_o, W_down):                Wout[r][j] = sum_m W[r][m] Q[m][j]
// as C[M][N] = A[M][K] . B[N][K]^T with both operands K-major bf16 in shared memory:
//   LEFT : A = (Q diag gamma)^T split into bf16 hi + lo, B = W^T          (K = d)
//   RIGHT: A = W (already K-major),       B = Q^T split into bf16 hi + lo (K = d)
// The fp32 factor is split (hi = RNE_bf16(q), lo = RNE_bf16(q - hi)) so that the products
// keep ~16 mantissa bits (SURVEY §7 hard part 5, Z23); both halves accumulate into the same
// fp32 TMEM accumulator and Wout is rounded to bf16 (RNE) once.
//
// Kernel (one 128 x BN output tile per CTA, 6 warps):
//   warp 0 (one lane): TMA producer — cp.async.bulk.tensor 2D loads of 128B-swizzled
//                      64-element K slabs of A (and A_lo) and B (and B_lo) into a 3-stage ring,
//                      completion counted on the stage's mbarrier (expect_tx);
//   warp 1 (one lane): MMA issuer — tcgen05.mma.cta_group::1.kind::f16 (M = 128, N = BN,
//                      K = 16 per instruction), accumulator in TMEM (BN fp32 columns);
//                      tcgen05.commit releases each ring slot and finally signals the epilogue;
//   warps 2-5:         epilogue — tcgen05.ld 32x32b (warp w reads TMEM lanes 32 (w%4) ..),
//                      bf16 RNE, 16-byte global stores.
// The operand transposes / splits are small prep kernels (offline path).
#pragma once
#include <cuda.h>   // CUtensorMap (types only; the encoder comes from cudaGetDriverEntryPoint)
#include "aux.cuh"
// (ring depth: 3 stages of 64 KB for LEFT, 2 of 80 KB for RIGHT at BN = 256)

namespace larosa {

constexpr int kFoldBM = 128;
constexpr int kFoldBK = 64;          // 64 bf16 = one 128-byte swizzle row
constexpr int kFoldThreads = 192;

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 bytes apart
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* smem) {
    const uint64_t addr = smem_u32(smem);
    return ((addr >> 4) & 0x3FFFull)          // start address (16-byte units)
           | (1ull << 16)                      // leading byte offset (unused for swizzled K-major)
           | ((uint64_t)(1024 >> 4) << 32)     // stride byte offset: 8 rows x 128 B
           | (1ull << 46)                      // descriptor version (sm_100)
           | (2ull << 61);                     // SWIZZLE_128B
}

// instruction descriptor: kind::f16, A = B = BF16, D = F32, both K-major, M x N
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, bool acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"((int)acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

template <int BN, bool ASPLIT, bool BSPLIT>
__host__ __device__ constexpr int fold_stage_bytes() {
    return (ASPLIT ? 2 : 1) * kFoldBM * kFoldBK * 2 + (BSPLIT ? 2 : 1) * BN * kFoldBK * 2;
}
template <int BN, bool ASPLIT, bool BSPLIT>
__host__ __device__ constexpr int fold_stages() {   // as many ring stages as fit (<= 4)
    return (224 * 1024) / fold_stage_bytes<BN, ASPLIT, BSPLIT>() > 4 ? 4 : (224 * 1024) / fold_stage_bytes<BN, ASPLIT, BSPLIT>();
}
template <int BN, bool ASPLIT, bool BSPLIT>
__host__ __device__ constexpr int fold_smem_bytes() {
    return 1024 + fold_stages<BN, ASPLIT, BSPLIT>() * fold_stage_bytes<BN, ASPLIT, BSPLIT>() + 128;
}

// F32OUT: the epilogue stores fp32 out[m][n] = scale * acc (+ out[m][n] if accumulate) -- the
// calibration covariance X^T X (N1); else bf16 RNE (the fold).
template <int BN, bool ASPLIT, bool BSPLIT, bool F32OUT = false>
__global__ void __launch_bounds__(kFoldThreads, 1)
    fold_tc_kernel(const __grid_constant__ CUtensorMap tA0, const __grid_constant__ CUtensorMap tA1,
                   const __grid_constant__ CUtensorMap tB0, const __grid_constant__ CUtensorMap tB1,
                   void* __restrict__ out_raw, int N, int K, float scale = 1.0f, int accumulate = 0) {
    extern __shared__ __align__(1024) unsigned char fold_smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(fold_smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int A_BYTES = kFoldBM * kFoldBK * 2;
    constexpr int B_BYTES = BN * kFoldBK * 2;
    constexpr int NA = ASPLIT ? 2 : 1;
    constexpr int STAGE = fold_stage_bytes<BN, ASPLIT, BSPLIT>();
    constexpr int kFoldStages = fold_stages<BN, ASPLIT, BSPLIT>();
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kFoldStages * STAGE);
    uint64_t* empty = full + kFoldStages;
    uint64_t* accb = empty + kFoldStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accb + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * kFoldBM, n0 = blockIdx.x * BN;
    const int nk = K / kFoldBK;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kFoldStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accb, 1);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tA0)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tB0)) : "memory");
    }
    if (warp == 1) {   // TMEM accumulator: BN fp32 columns x 128 lanes
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(BN)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {   // TMA producer
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % kFoldStages;
                if (kb >= kFoldStages) mbar_wait_parity(&empty[s], ((kb / kFoldStages) & 1) ^ 1);
                unsigned char* st = smem + s * STAGE;
                mbar_arrive_expect_tx(&full[s], STAGE);
                tma_load_2d(st, &tA0, kb * kFoldBK, m0, &full[s]);
                if (ASPLIT) tma_load_2d(st + A_BYTES, &tA1, kb * kFoldBK, m0, &full[s]);
                tma_load_2d(st + NA * A_BYTES, &tB0, kb * kFoldBK, n0, &full[s]);
                if (BSPLIT) tma_load_2d(st + NA * A_BYTES + B_BYTES, &tB1, kb * kFoldBK, n0, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // MMA issuer
            constexpr uint32_t idesc = umma_idesc_bf16(kFoldBM, BN);
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % kFoldStages;
                mbar_wait_parity(&full[s], (kb / kFoldStages) & 1);
                tc_fence_after();
                unsigned char* st = smem + s * STAGE;
#pragma unroll
                for (int k = 0; k < kFoldBK / 16; ++k) {   // 16 bf16 = 32 bytes per MMA
                    const uint64_t da0 = umma_desc_sw128(st + 32 * k);
                    const uint64_t db0 = umma_desc_sw128(st + NA * A_BYTES + 32 * k);
                    umma_bf16(tmem, da0, db0, idesc, kb > 0 || k > 0);
                    if (ASPLIT) umma_bf16(tmem, umma_desc_sw128(st + A_BYTES + 32 * k), db0, idesc, true);
                    if (BSPLIT) umma_bf16(tmem, da0, umma_desc_sw128(st + NA * A_BYTES + B_BYTES + 32 * k), idesc, true);
                }
                umma_commit(&empty[s]);   // the slot is free once these MMAs have read it
            }
            umma_commit(accb);            // accumulator complete
        }
    } else {
        // epilogue: warp w reads TMEM lanes [32 (w % 4), +32) = output rows of this tile
        mbar_wait_parity(accb, 0);
        tc_fence_after();
        const int q = warp & 3;
        const int row = m0 + 32 * q + lane;
        uint16_t* orow = reinterpret_cast<uint16_t*>(out_raw) + (size_t)row * N + n0;
        float* frow = reinterpret_cast<float*>(out_raw) + (size_t)row * N + n0;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
            uint32_t v[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                  "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                  "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if constexpr (F32OUT) {
                float4* fd = reinterpret_cast<float4*>(frow + c0);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    float4 o = make_float4(scale * __uint_as_float(v[4 * j]), scale * __uint_as_float(v[4 * j + 1]),
                                           scale * __uint_as_float(v[4 * j + 2]), scale * __uint_as_float(v[4 * j + 3]));
                    if (accumulate) {
                        const float4 pv = fd[j];
                        o.x += pv.x;
                        o.y += pv.y;
                        o.z += pv.z;
                        o.w += pv.w;
                    }
                    fd[j] = o;
                }
                continue;
            }
            uint32_t p[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
                p[j] = (uint32_t)f2bf16_rne(__uint_as_float(v[2 * j])) |
                       ((uint32_t)f2bf16_rne(__uint_as_float(v[2 * j + 1])) << 16);
            uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
            for (int j = 0; j < 4; ++j) dst[j] = make_uint4(p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(BN) : "memory");
}

// ---- operand preparation (offline) -------------------------------------------------------
// dst_hi/lo[c][r] = split(src[r][c] * (scale ? scale[r] : 1)), src fp32 [R][C] row-major.
__global__ void split_transpose_kernel(const float* __restrict__ src, const float* __restrict__ scale,
                                       uint16_t* __restrict__ hi, uint16_t* __restrict__ lo, int R, int C) {
    __shared__ float t[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int r = r0 + y, c = c0 + threadIdx.x;
        t[y][threadIdx.x] = (r < R && c < C) ? src[(size_t)r * C + c] * (scale ? scale[r] : 1.f) : 0.f;
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int c = c0 + y, r = r0 + threadIdx.x;
        if (r < R && c < C) {
            const float v = t[threadIdx.x][y];
            const uint16_t h = f2bf16_rne(v);
            hi[(size_t)c * R + r] = h;
            if (lo) lo[(size_t)c * R + r] = f2bf16_rne(v - bf16f(h));
        }
    }
}
// dst[c][r] = src[r][c]  (bf16 bits)
__global__ void transpose_bf16_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst, int R, int C) {
    __shared__ uint16_t t[32][34];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int r = r0 + y, c = c0 + threadIdx.x;
        t[y][threadIdx.x] = (r < R && c < C) ? src[(size_t)r * C + c] : 0;
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int c = c0 + y, r = r0 + threadIdx.x;
        if (r < R && c < C) dst[(size_t)c * R + r] = t[threadIdx.x][y];
    }
}

}  // namespace larosa
