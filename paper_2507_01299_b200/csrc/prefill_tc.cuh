// prefill_tc.cuh — prefill with full sparsification of the prompt tokens (
// PAPER.md:77 "full activation sparsification at prefill stage", P:165 the initial tokens):
//
//   Y[t][o] = sum_{j in S_t} X[t][j] s_t W[j][o]          (S_t: token t's exact Top-K, Z10)
//
// 1. prefill_rule_mask_kernel — one CTA per token: stages x_t in shared memory, finds the k-th
//    largest key bits(|x|) by a bitwise search over the key (31 block-wide counts: the largest tk
//    with #{key >= tk} >= k is exactly the k-th key), then the index threshold ti among the keys
//    equal to tk (block prefix count in index order: lower index wins, Z10) and the RMS scale
//    s_t (fixed-order block sum); writes the masked row Xm[t][j] = bf16(x_j s_t) if kept else 0
//    (and the bf16 remainder for the split-precision mode) and one byte per 64-channel block
//    that says whether t keeps any channel of it.
// 2. prefill_tc_kernel — tcgen05 GEMM D[128 output columns][256 tokens] += W[64 rows][128 cols]^T
//    . Xm[256 tokens][64 rows]^T per 64-row block: A = the weight rows, MN-major, by TMA (two
//    64x64 boxes, 128-byte swizzle, as the batched GEMV); B = the masked activations, K-major, one
//    TMA box of 64 x 256 (and the remainder box in split mode, a second MMA into the same
//    accumulator); fp32 accumulator in TMEM (256 columns).  A 64-row block that no token of the
//    CTA's 256-token tile keeps is skipped (the tile's union of kept rows, at 64-row granularity:
//    the gathered K range).  Warp 0 TMA producer, warp 1 MMA issuer (one elected thread), warps
//    2-5 the epilogue (tcgen05.ld 32x32b: lane = output column, registers = tokens -> coalesced
//    fp32 stores of Y).
#pragma once
#include "fold_tc.cuh"
#include "gemv.cuh"

namespace larosa {

constexpr int kPfThreads = 256;
constexpr int kPfTok = 256;                       // tokens per CTA tile (UMMA N)
constexpr int kPfCols = 128;                      // output columns per CTA tile (UMMA M)
constexpr int kPfK = 64;                          // weight rows per stage
constexpr int kPfABytes = kPfCols * kPfK * 2;     // 16 KB
constexpr int kPfBBytes = kPfTok * kPfK * 2;      // 32 KB
constexpr int kPfGemmThreads = 192;

__host__ __device__ constexpr int pf_stage_bytes(bool split) { return kPfABytes + (split ? 2 : 1) * kPfBBytes; }
// bf16 mode: 2 stages of 48 KB and 2 CTAs per SM (one CTA's epilogue overlaps the other's MMAs):
// 512 tokens x 4096 x 22016 0.131 -> 0.119 ms, 2048 tokens 0.475 -> 0.406 ms vs 4 stages, 1 CTA/SM
#ifndef LAROSA_PF_STAGES
#define LAROSA_PF_STAGES 2
#endif
#ifndef LAROSA_PF_MINB
#define LAROSA_PF_MINB 2
#endif
__host__ __device__ constexpr int pf_stages(bool split) { return split ? 2 : LAROSA_PF_STAGES; }
__host__ __device__ constexpr size_t pf_smem_bytes(bool split) {
    return 1024 + (size_t)pf_stages(split) * pf_stage_bytes(split) + 128 + 2 * 512;
}

// ---- 1. per-token exact Top-K rule, RMS scale and the masked bf16 rows ---------------------------
// shared: x [d] fp32 + scratch
__global__ void __launch_bounds__(kPfThreads) prefill_rule_mask_kernel(const float* __restrict__ X, int n_tok, int d,
                                                                       int k, float eps, uint16_t* __restrict__ xm_hi,
                                                                       uint16_t* __restrict__ xm_lo,
                                                                       uint8_t* __restrict__ anyk, int n_tok_pad) {
    extern __shared__ __align__(16) float pfs[];
    float* xs = pfs;                                         // [d]
    int* red = reinterpret_cast<int*>(xs + d);               // [8] warp partials
    float* fred = reinterpret_cast<float*>(red + 8);         // [8]
    int* bcast = reinterpret_cast<int*>(fred + 8);           // [4]
    const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const float* x = X + (size_t)t * d;
    for (int i = tid; i < d; i += kPfThreads) xs[i] = x[i];
    __syncthreads();
    // block-wide count of keys >= c (fixed order not needed: integer)
    auto count_ge = [&](uint32_t c, bool strict) -> int {
        int n = 0;
        for (int i = tid; i < d; i += kPfThreads) {
            const uint32_t key = key_of(xs[i]);
            n += strict ? (key > c) : (key >= c);
        }
        n = __reduce_add_sync(0xffffffffu, n);
        if (lane == 0) red[wid] = n;
        __syncthreads();
        int tot = 0;
#pragma unroll
        for (int w = 0; w < kPfThreads / 32; ++w) tot += red[w];
        __syncthreads();
        return tot;
    };
    uint32_t tk = 0u;
    int ti = -1;                                             // keep i iff key > tk or (key == tk and i <= ti)
    if (k >= d) {
        ti = 0x7fffffff;                                     // keep all (tk = 0: key >= 0)
    } else if (k > 0) {
#pragma unroll 1
        for (int bit = 30; bit >= 0; --bit) {                // finite keys < 2^31
            const uint32_t cand = tk | (1u << bit);
            if (count_ge(cand, false) >= k) tk = cand;
        }
        // tk is the k-th largest key; need = k - #{key > tk} of the keys equal to tk, lowest indices
        const int need = k - count_ge(tk, true);
        // prefix count of (key == tk) in index order: thread tid owns indices [tid*c, tid*c + c)
        const int per = (d + kPfThreads - 1) / kPfThreads;
        const int i0 = tid * per, i1 = min(d, i0 + per);
        int mine = 0;
        for (int i = i0; i < i1; ++i) mine += key_of(xs[i]) == tk;
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) red[wid] = incl;
        __syncthreads();
        int before = incl - mine;
        for (int w = 0; w < wid; ++w) before += red[w];
        if (before < need && before + mine >= need) {        // the need-th equal key is in my range
            int c = before;
            for (int i = i0; i < i1; ++i)
                if (key_of(xs[i]) == tk && ++c == need) {
                    bcast[0] = i;
                    break;
                }
        }
        __syncthreads();
        ti = bcast[0];
    } else {
        tk = 0xffffffffu;                                    // keep none
    }
    // RMS scale (fixed-order block sum of squares)
    float s = 1.f;
    if (eps >= 0.f) {
        float q = 0.f;
        for (int i = tid; i < d; i += kPfThreads) q = fmaf(xs[i], xs[i], q);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
        if (lane == 0) fred[wid] = q;
        __syncthreads();
        float tot = 0.f;
#pragma unroll
        for (int w = 0; w < kPfThreads / 32; ++w) tot += fred[w];
        s = 1.0f / sqrtf(tot / (float)d + eps);
    }
    // masked rows and the per-64-channel-block "any kept" bytes (blocks along channels)
    uint16_t* hrow = xm_hi + (size_t)t * d;
    uint16_t* lrow = xm_lo ? xm_lo + (size_t)t * d : nullptr;
    const int nkb = (d + kPfK - 1) / kPfK;
    for (int kb = wid; kb < nkb; kb += kPfThreads / 32) {
        bool any = false;
        for (int j = lane; j < kPfK; j += 32) {
            const int i = kb * kPfK + j;
            if (i >= d) break;
            const float v = xs[i];
            const uint32_t key = key_of(v);
            const bool kp = key > tk || (key == tk && i <= ti);
            const float sv = kp ? v * s : 0.f;
            const uint16_t h = f2bf16_rne(sv);
            hrow[i] = h;
            if (lrow) lrow[i] = f2bf16_rne(sv - bf16f(h));
            any |= kp;
        }
        any = __any_sync(0xffffffffu, any);
        if (lane == 0) anyk[(size_t)kb * n_tok_pad + t] = any ? 1 : 0;
    }
}

// ---- 2. the masked GEMM on tcgen05 ---------------------------------------------------------------
template <bool SPLIT>
__global__ void __launch_bounds__(kPfGemmThreads, LAROSA_PF_MINB)
    prefill_tc_kernel(const __grid_constant__ CUtensorMap tW, const __grid_constant__ CUtensorMap tXh,
                      const __grid_constant__ CUtensorMap tXl, const uint8_t* __restrict__ anyk, int n_tok_pad,
                      int n_tok, int d_in, int d_out, float* __restrict__ Y) {
    extern __shared__ __align__(1024) unsigned char pf_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(pf_raw) + 1023) & ~uintptr_t(1023));
    constexpr int STAGE = pf_stage_bytes(SPLIT);
    constexpr int NS = pf_stages(SPLIT);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * STAGE);
    uint64_t* empty = full + NS;
    uint64_t* accb = empty + NS;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accb + 1);
    int* nact = reinterpret_cast<int*>(tmem_slot + 1);
    uint16_t* kblist = reinterpret_cast<uint16_t*>(nact + 1);          // <= 512 active blocks (d_in <= 32768)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int col0 = blockIdx.x * kPfCols, tok0 = blockIdx.y * kPfTok;
    const int nkb = (d_in + kPfK - 1) / kPfK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accb, 1);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tW)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tXh)) : "memory");
    }
    if (warp == 1) {   // TMEM accumulator: 256 fp32 columns (tokens) x 128 lanes (output columns)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    pdl_wait();
    pdl_trigger();
    // the tile's active 64-row blocks (any of its tokens keeps a row of the block), in order
    if (warp == 0) {
        int base = 0;
        for (int kb0 = 0; kb0 < nkb; kb0 += 32) {
            const int kb = kb0 + lane;
            bool act = false;
            if (kb < nkb) {
                const uint4* p = reinterpret_cast<const uint4*>(anyk + (size_t)kb * n_tok_pad + tok0);
#pragma unroll 4
                for (int q = 0; q < kPfTok / 16; ++q) {
                    const uint4 v = __ldg(p + q);
                    act |= (v.x | v.y | v.z | v.w) != 0u;
                }
            }
            const unsigned m = __ballot_sync(0xffffffffu, act);
            if (act) kblist[base + __popc(m & ((1u << lane) - 1u))] = (uint16_t)kb;
            base += __popc(m);
        }
        if (lane == 0) *nact = base;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int na = *nact;

    if (warp == 0) {
        if (lane == 0) {   // TMA producer
            for (int c = 0; c < na; ++c) {
                const int s = c % NS;
                if (c >= NS) mbar_wait_parity(&empty[s], ((c / NS) & 1) ^ 1);
                unsigned char* st = smem + s * STAGE;
                const int r0 = (int)kblist[c] * kPfK;
                mbar_arrive_expect_tx(&full[s], STAGE);
                tma_load_2d(st, &tW, col0, r0, &full[s]);
                tma_load_2d(st + kPfABytes / 2, &tW, col0 + 64, r0, &full[s]);
                tma_load_2d(st + kPfABytes, &tXh, r0, tok0, &full[s]);
                if (SPLIT) tma_load_2d(st + kPfABytes + kPfBBytes, &tXl, r0, tok0, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // MMA issuer: A MN-major (weights), B K-major (tokens), M = 128, N = 256
            constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(kPfTok >> 3) << 17) |
                                       ((uint32_t)(kPfCols >> 4) << 24);
            for (int c = 0; c < na; ++c) {
                const int s = c % NS;
                mbar_wait_parity(&full[s], (c / NS) & 1);
                tc_fence_after();
                unsigned char* st = smem + s * STAGE;
#pragma unroll
                for (int ks = 0; ks < kPfK / 16; ++ks) {
                    const uint64_t da = umma_desc_mn_sw128(st + ks * 2048, 8192, 1024);
                    const uint64_t db = umma_desc_sw128(st + kPfABytes + ks * 32);
                    umma_bf16(tmem, da, db, idesc, c > 0 || ks > 0);
                    if (SPLIT) umma_bf16(tmem, da, umma_desc_sw128(st + kPfABytes + kPfBBytes + ks * 32), idesc, true);
                }
                umma_commit(&empty[s]);
            }
            umma_commit(accb);
        }
    } else {
        // epilogue: warp w reads TMEM lanes [32 (w % 4), +32) = output columns; registers = tokens
        const int q = warp & 3;
        const int o = col0 + 32 * q + lane;
        if (na > 0) {
            mbar_wait_parity(accb, 0);
            tc_fence_after();
        }
#pragma unroll 1
        for (int c0 = 0; c0 < kPfTok; c0 += 32) {
            uint32_t v[32];
            if (na > 0) {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                    "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
                    "[%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                      "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                      "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c0));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = 0u;
            }
            if (o < d_out) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int t = tok0 + c0 + j;
                    if (t < n_tok) Y[(size_t)t * d_out + o] = __uint_as_float(v[j]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

}  // namespace larosa
