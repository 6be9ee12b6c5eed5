// gemv_tc.cuh — batched sparse GEMV on the 5th-generation tensor cores (batch 8-16; SURVEY §7
// hard part 3: at B >= 8 the fp32 CUDA-core FMA rate, not HBM, bounds the CUDA-core GEMV).
//
//   acc[b][o] += fix( sum_{r in rows} val(r, b) * W[row(r)][o] )      (same contract as gemv.cuh)
//
// As an MMA  D[M = 128 columns][N = 16 tokens] += A[M][K = kept rows] . B[K][N]:
//   A = the weight rows, MN-major (a row's 128 columns are contiguous in W): for contiguous
//       rows (DENSE, THRESH) each 64-row chunk is two TMA boxes (128-byte swizzle); for gathered
//       rows (LIST) it is copied with per-thread cp.async into the canonical 128-byte-swizzled
//       MN-major layout (atoms of 8 rows x 64 columns; next 64 columns +1 KB, next 8 rows +2 KB);
//       rows past the list are zero-filled (src-size 0);
//   B = the tokens' values, K-major, split into bf16 hi + lo (~16 mantissa bits of the fp32
//       activations), written with st.shared as the two 16-token halves of one N = 32 operand;
//   D = 32 fp32 TMEM columns x 128 lanes (hi products in 0-15, lo in 16-31, summed on read-out).
// Warps 0-3 produce (gather + values) into a kTcStages-deep ring (2 by default) whose stages complete through
// cp.async.mbarrier.arrive; one thread of warp 4 issues tcgen05.mma (M = 128, N = 32 = hi | lo, K = 16)
// and frees stages with tcgen05.commit; warps 0-3 then tcgen05.ld the accumulator (lane =
// column) and add it into the 64-bit fixed-point accumulators; the last split CTA of a slice
// finalises it (ticket), as in gemv.cuh.  Row sources: THRESH (every row of the CTA's input
// range, each token's value masked by its Top-K rule: at batch >= 8 the union of the tokens'
// kept rows is ~98% of all rows), LIST (the batch union), DENSE (adapter, LM head).
#pragma once
#include "fold_tc.cuh"
#include "gemv.cuh"

namespace larosa {

constexpr int kTcCols = 128;         // columns per CTA (UMMA M)
constexpr int kTcN = 16;             // tokens (UMMA N; batch padded to 16)
constexpr int kTcChunk = 64;         // kept rows per ring stage (UMMA K = 16 per instruction)
#ifndef LAROSA_TC_STAGES
#define LAROSA_TC_STAGES 2
#endif
// ring depth x CTAs per SM (LLaMA3-8B decode, B = 16, p = 0.4: 4 stages x 2 CTAs 7.49 ms, 3 x 3 7.25,
// 2 x 4 6.48; 6-10 stages x 1 CTA 11.1):
// per-CTA work, not bytes in flight, paces the stream, so CTAs per SM matter most
constexpr int kTcStages = LAROSA_TC_STAGES;
constexpr int kTcProdWarps = 4;
#ifndef LAROSA_TC_VPRE
#define LAROSA_TC_VPRE 1
#endif
constexpr int kTcVPre = LAROSA_TC_VPRE;   // chunks of value look-ahead per producer thread (2-8: slower)
#ifndef LAROSA_TC_PREFETCH
#define LAROSA_TC_PREFETCH 0
#endif
// 1: the first ring stages' weight tiles are requested before the dependency wait (contiguous rows)
constexpr bool kTcPrefetch = LAROSA_TC_PREFETCH != 0;
#ifndef LAROSA_TC_FUSED_HILO
#define LAROSA_TC_FUSED_HILO 1
#endif
// hi and lo as the two 16-column halves of ONE N = 32 MMA (B rows 0-15 = hi, 16-31 = lo are
// contiguous in the stage): half the MMA instructions, each reading the A tile once
constexpr bool kTcFused = LAROSA_TC_FUSED_HILO != 0;
constexpr int kTcThreads = (kTcProdWarps + 1) * 32;
// Profiling switches (1 skip MMAs, 2 skip values, 4 skip A copies, 8 skip the proxy fence, 16
// constant values) exist only in a -DLAROSA_TC_DEBUG build; the shipped library compiles them out.
#ifdef LAROSA_TC_DEBUG
__device__ __forceinline__ int tc_dbg_flags(const GemvArgs& a) { return a.tc_dbg; }
#else
__device__ __forceinline__ int tc_dbg_flags(const GemvArgs&) { return 0; }
#endif
// The input-row range [lo, lo + n) of split `split` for contiguous rows (DENSE, THRESH): whole
// 64-row chunks, so every chunk's 8-row value groups are 32-byte aligned in x.  The weight
// prefetch and the producer loop both use it, so a stage's expect_tx always matches its TMA.
__device__ __forceinline__ void tc_split_range(int d_in, int n_splits, int split, int& lo, int& n) {
    const int rng = ((d_in + n_splits - 1) / n_splits + kTcChunk - 1) / kTcChunk * kTcChunk;
    lo = min(d_in, split * rng);
    n = min(d_in, lo + rng) - lo;
}
constexpr int kTcABytes = kTcCols * kTcChunk * 2;              // 16 KB
constexpr int kTcBBytes = kTcN * kTcChunk * 2;                 // 2 KB (hi, and again lo)
constexpr int kTcStage = kTcABytes + 2 * kTcBBytes;            // 20 KB

__host__ __device__ constexpr size_t gemv_tc_smem_bytes(int list_cap) {
    return 1024 + (size_t)kTcStages * kTcStage + 128 + (size_t)list_cap * 4 + 64 * 4;
}

// UMMA descriptor of an MN-major 128B-swizzled operand: LBO = next 64 MN elements, SBO = next 8 K rows
__device__ __forceinline__ uint64_t umma_desc_mn_sw128(const void* smem, uint32_t lbo, uint32_t sbo) {
    const uint64_t addr = smem_u32(smem);
    return ((addr >> 4) & 0x3FFFull) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// kind::f16, A = B = BF16, D = F32, A MN-major, B K-major, M = 128, N = 16
__host__ __device__ constexpr uint32_t tc_idesc(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kTcCols >> 4) << 24);
}
constexpr uint32_t kTcIdesc = tc_idesc(kTcN);
constexpr uint32_t kTcIdesc2 = tc_idesc(2 * kTcN);   // fused hi|lo

__device__ __forceinline__ void cp_async16_zfill(void* smem_dst, const void* gsrc, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)), "l"(gsrc),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// {lo half = bf16(a), hi half = bf16(b)}, round to nearest even
__device__ __forceinline__ uint32_t cvt_bf16x2(float a, float b) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// DENSE / THRESH (contiguous rows): the A tile comes by TMA, two boxes of 64 rows x 64 columns
// (128-byte swizzle; box mg at +8 KB, row r at +128 r), i.e. LBO = 8 KB, SBO = 1 KB; LIST
// (gathered rows) keeps the per-thread cp.async layout (LBO = 1 KB, SBO = 2 KB).
template <int BP, int MODE>
__global__ void __launch_bounds__(kTcThreads, 1) gemv_tc_kernel(const GemvArgs a, const __grid_constant__ CUtensorMap tmw) {
    constexpr bool kTma = MODE != GEMV_LIST;
    static_assert(BP >= 2 && BP <= kTcN, "tcgen05 GEMV: batch 2..16");
    extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTcStages * kTcStage);
    uint64_t* empty = full + kTcStages;
    uint64_t* accb = empty + kTcStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accb + 1);
    int* lrow = reinterpret_cast<int*>(smem + kTcStages * kTcStage + 128);   // LIST: [cap]
    int* misc = lrow + a.list_cap;
    const int slice = blockIdx.x, split = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int col0 = slice * kTcCols;

    if (tid == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full[s], kTcProdWarps * 32);   // + the TMA bytes (expect_tx) when kTma
            mbar_init(&empty[s], 1);
        }
        mbar_init(accb, 1);
        fence_mbar_init();
    }
    if (warp == kTcProdWarps) {   // TMEM accumulator: 16 (-> 32 allocated) fp32 columns x 128 lanes
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tl_stamp(a.tl, 0);
    if constexpr (kTma && kTcPrefetch) {   // the weights do not depend on the previous kernel
        if (tid == 0 && !(tc_dbg_flags(a) & 4)) {
            int plo, pn_rows;
            tc_split_range(a.d_in, a.n_splits, split, plo, pn_rows);
            const int pch = (pn_rows + kTcChunk - 1) / kTcChunk;
            for (int c = 0; c < kTcStages && c < pch; ++c) {
                unsigned char* st = smem + c * kTcStage;
                mbar_expect_tx(&full[c], kTcABytes);
                tma_load_2d(st, &tmw, col0, plo + c * kTcChunk, &full[c]);
                tma_load_2d(st + kTcABytes / 2, &tmw, col0 + 64, plo + c * kTcChunk, &full[c]);
            }
        }
    }
    pdl_wait();
    pdl_trigger();
    tl_stamp(a.tl, 1);
    if (a.zero_hist) {   // words whose consumer has completed (the LIST path's token masks)
        const int nct = gridDim.x * gridDim.y, cta = blockIdx.y * gridDim.x + blockIdx.x;
        for (int i = cta * kTcThreads + tid; i < a.zero_words; i += nct * kTcThreads) a.zero_hist[i] = 0u;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // ---- 1. this CTA's rows: a contiguous input range (DENSE, and THRESH: at batch >= 8 the
    //         tokens' union covers nearly every row, so every row is streamed and each token's
    //         value is masked by its rule), or its share of the union list (LIST) -------------
    int n_list = 0, lo = 0;
    if constexpr (MODE == GEMV_LIST) {
        const int nrows = a.nrows_dev ? *a.nrows_dev : a.nrows;
        const int rps = (nrows + a.n_splits - 1) / a.n_splits;
        lo = min(nrows, split * rps);
        n_list = min(nrows, lo + rps) - lo;
        for (int t = tid; t < n_list; t += kTcThreads) lrow[t] = __ldg(a.rows + lo + t);
    } else {
        tc_split_range(a.d_in, a.n_splits, split, lo, n_list);
    }
    __syncthreads();
    tl_stamp(a.tl, 2);
    const int n_chunks = (n_list + kTcChunk - 1) / kTcChunk;
    // producer thread pt owns token n = pt >> 3 and rows 8 k8 .. 8 k8 + 7 of every chunk
    const int pn = tid >> 3, pk8 = tid & 7;
    ThreshOut prule;
    prule.tk = 0u;
    prule.ti = 0x7fffffff;
    prule.scale = 1.f;
    if constexpr (MODE == GEMV_THRESH)
        if (tid < kTcProdWarps * 32 && pn < a.batch) prule = a.thr[pn];
    // raw inputs of this thread's 8 values of chunk c (loaded one chunk ahead)
    // x rows 16-byte aligned: a thread's 8 consecutive values are two 16-byte loads (8 scalar
    // loads, one 32-byte sector each, made the value staging L1-wavefront bound)
    const bool xvec = MODE != GEMV_LIST && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) && (a.ldx & 3) == 0;
    auto load_raw = [&](int c, float (&r)[8]) {
        if constexpr (MODE != GEMV_LIST) {
            const int e0 = c * kTcChunk + pk8 * 8;
            if (xvec && e0 + 8 <= n_list) {
                float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f), q1 = q0;
                if (pn < a.batch && pn < BP) {
                    const float4* src = reinterpret_cast<const float4*>(a.x + (size_t)pn * a.ldx + lo + e0);
                    q0 = __ldg(src);
                    q1 = __ldg(src + 1);
                }
                r[0] = q0.x; r[1] = q0.y; r[2] = q0.z; r[3] = q0.w;
                r[4] = q1.x; r[5] = q1.y; r[6] = q1.z; r[7] = q1.w;
                return;
            }
        }
#pragma unroll
        for (int h = 0; h < 8; ++h) {
            const int e = c * kTcChunk + pk8 * 8 + h;
            float v = 0.f;
            if (pn < a.batch && pn < BP && e < n_list) {
                if constexpr (MODE == GEMV_LIST)
                    v = __ldg(a.vals + (size_t)(lo + e) * a.vs_r + (size_t)pn * a.vs_b);
                else
                    v = __ldg(a.x + (size_t)pn * a.ldx + lo + e);
            }
            r[h] = v;
        }
    };
    auto finish = [&](int c, int h, float v) -> float {   // the token's rule (THRESH)
        if constexpr (MODE == GEMV_THRESH) {
            const int i = lo + c * kTcChunk + pk8 * 8 + h;
            const uint32_t key = key_of(v);
            return (key > prule.tk || (key == prule.tk && i <= prule.ti)) ? v * prule.scale : 0.f;
        }
        return v;
    };

    if (warp < kTcProdWarps) {
        // ---- producers: gather 64 weight rows x 128 columns, and the chunk's values -------------
        const int pt = tid;                                // 0..127
        // the values are loaded kTcVPre chunks ahead (a register ring): with one chunk of
        // look-ahead their L2 latency, not HBM, paced the ring (~1.4 us per 16 KB chunk)
        float ring[kTcVPre][8];
#pragma unroll
        for (int j = 0; j < kTcVPre; ++j)
            if (j < n_chunks) load_raw(j, ring[j]);
        for (int c0 = 0; c0 < n_chunks; c0 += kTcVPre)
#pragma unroll
        for (int j = 0; j < kTcVPre; ++j) {
            const int c = c0 + j;
            if (c >= n_chunks) break;
            float (&cur)[8] = ring[j];
            const int s = c % kTcStages;
            if (c >= kTcStages) mbar_wait_parity(&empty[s], ((c / kTcStages) & 1) ^ 1);
            unsigned char* st = smem + s * kTcStage;
            // A: 64 rows x 16 chunks of 16 bytes; thread pt takes chunks pt + 128 q
            if constexpr (kTma) {
                if (pt == 0 && !(tc_dbg_flags(a) & 4) && !(kTcPrefetch && c < kTcStages)) {
                    mbar_expect_tx(&full[s], kTcABytes);
                    tma_load_2d(st, &tmw, col0, lo + c * kTcChunk, &full[s]);
                    tma_load_2d(st + kTcABytes / 2, &tmw, col0 + 64, lo + c * kTcChunk, &full[s]);
                }
            } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int u = pt + 128 * q;
                const int r = u >> 4, cc = u & 15;         // row in chunk, 16-byte chunk of the row
                const int e = c * kTcChunk + r;            // list entry
                const bool ok = e < n_list;
                const int row = !ok ? 0 : (MODE == GEMV_LIST ? lrow[e] : lo + e);
                const int mg = cc >> 3, c8 = cc & 7;       // 64-column group, chunk within it
                unsigned char* dst = st + ((r >> 3) * 2 + mg) * 1024 + (r & 7) * 128 + ((c8 ^ (r & 7)) << 4);
                const bool valid = ok && col0 + cc * 8 < a.d_out && !(tc_dbg_flags(a) & 4);
                cp_async16_zfill(dst, valid ? a.W + (size_t)row * a.ld + col0 + cc * 8 : a.W, valid);
            }
            }
            // B: token n (0..15) x 8 consecutive rows (16 bytes of hi, 16 of lo) per thread
            if (tc_dbg_flags(a) & 16) {
                const int off = (pn >> 3) * 1024 + (pn & 7) * 128 + ((pk8 ^ (pn & 7)) << 4);
                *reinterpret_cast<uint4*>(st + kTcABytes + off) = make_uint4(0u, 0u, 0u, 0u);
                *reinterpret_cast<uint4*>(st + kTcABytes + kTcBBytes + off) = make_uint4(0u, 0u, 0u, 0u);
            } else if (!(tc_dbg_flags(a) & 2)) {
                uint32_t hi[4], lw[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const float f0 = finish(c, 2 * h, cur[2 * h]), f1 = finish(c, 2 * h + 1, cur[2 * h + 1]);
                    // packed hardware RNE (cvt.rn.bf16x2: bit-identical to f2bf16_rne on finite values)
                    hi[h] = cvt_bf16x2(f0, f1);
                    lw[h] = cvt_bf16x2(f0 - __uint_as_float(hi[h] << 16), f1 - __uint_as_float(hi[h] & 0xffff0000u));
                }
                const int off = (pn >> 3) * 1024 + (pn & 7) * 128 + ((pk8 ^ (pn & 7)) << 4);
                *reinterpret_cast<uint4*>(st + kTcABytes + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<uint4*>(st + kTcABytes + kTcBBytes + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            }
            if (!(tc_dbg_flags(a) & 8)) fence_proxy_async_smem();   // the st.shared values, for the tensor core's async proxy
            if constexpr (kTma)
                mbar_arrive(&full[s]);
            else
                cp_async_mbar_arrive(&full[s]);
            // chunk c + kTcVPre's values: issued after the fence (which would wait for them)
            if (c + kTcVPre < n_chunks && !(tc_dbg_flags(a) & 2)) load_raw(c + kTcVPre, cur);
        }
    } else if (lane == 0) {
        // ---- MMA issuer ------------------------------------------------------------------------
        for (int c = 0; c < n_chunks; ++c) {
            const int s = c % kTcStages;
            mbar_wait_parity(&full[s], (c / kTcStages) & 1);
            fence_proxy_async_smem();
            tc_fence_after();
            unsigned char* st = smem + s * kTcStage;
            const int rows = min(kTcChunk, n_list - c * kTcChunk);
#pragma unroll
            for (int ks = 0; ks < kTcChunk / 16; ++ks) {
                if (16 * ks >= rows) break;
                const uint64_t da = kTma ? umma_desc_mn_sw128(st + ks * 2048, 8192, 1024)
                                         : umma_desc_mn_sw128(st + ks * 4096, 1024, 2048);
                const uint64_t dbh = umma_desc_sw128(st + kTcABytes + ks * 32);
                const uint64_t dbl = umma_desc_sw128(st + kTcABytes + kTcBBytes + ks * 32);
                if (!(tc_dbg_flags(a) & 1)) {
                    if constexpr (kTcFused) {
                        umma_bf16(tmem, da, dbh, kTcIdesc2, c > 0 || ks > 0);
                    } else {
                        umma_bf16(tmem, da, dbh, kTcIdesc, c > 0 || ks > 0);
                        umma_bf16(tmem, da, dbl, kTcIdesc, true);
                    }
                }
            }
            umma_commit(&empty[s]);
        }
        umma_commit(accb);
    }
    __syncwarp();

    // ---- accumulator -> fixed-point partial sums (warps 0-3: TMEM lane = column) ------------
    if (warp < kTcProdWarps && n_chunks > 0) {
        mbar_wait_parity(accb, 0);
        tc_fence_after();
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + ((uint32_t)(32 * warp) << 16)));
        if constexpr (kTcFused) {   // columns 16-31: the lo halves
            uint32_t w[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                "%14, %15}, [%16];"
                : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
                  "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
                : "r"(tmem + ((uint32_t)(32 * warp) << 16) + 16u));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int b = 0; b < 16; ++b) v[b] = __float_as_uint(__uint_as_float(v[b]) + __uint_as_float(w[b]));
        } else {
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        const int o = col0 + tid;
        if (o < a.d_out)
#pragma unroll
            for (int b = 0; b < BP; ++b)
                if (b < a.batch) red_fix(a.acc + (size_t)b * a.acc_ld + o, __uint_as_float(v[b]), a.err);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kTcProdWarps) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
    tl_stamp(a.tl, 3);
    if (a.epi == EPI_NONE) {
        tl_stamp(a.tl, 4);
        return;
    }

    // ---- the last split CTA of this slice finalises its 128 columns ---------------------------
    __syncthreads();
    if (tid == 0) misc[16] = atom_add_acq_rel_gpu(a.tickets + slice, 1u) == gridDim.y - 1u;
    __syncthreads();
    if (!misc[16]) {
        tl_stamp(a.tl, 4);
        return;
    }
    if (tid == 0) a.tickets[slice] = 0u;
    // (every token's sums are read before any is written: 16 independent L2 reads instead of a
    // chain of 16 round trips in the launch's tail)
    if (a.epi == EPI_SILU) {
        // the 128-column slice is one gate|up block: 64 gate, then the matching 64 up
        if (tid < kGuBlock && col0 + tid < a.d_out) {
            float g[BP], u[BP];
#pragma unroll
            for (int b = 0; b < BP; ++b)
                if (b < a.batch) {
                    const unsigned long long* acc = a.acc + (size_t)b * a.acc_ld + col0 + tid;
                    g[b] = fix_to_f(__ldcg(acc));
                    u[b] = fix_to_f(__ldcg(acc + kGuBlock));
                }
#pragma unroll
            for (int b = 0; b < BP; ++b)
                if (b < a.batch) {
                    unsigned long long* acc = a.acc + (size_t)b * a.acc_ld + col0 + tid;
                    acc[0] = 0ull;
                    acc[kGuBlock] = 0ull;
                    a.out[(size_t)b * a.out_ld + slice * kGuBlock + tid] = g[b] / (1.0f + expf(-g[b])) * u[b];
                }
        }
    } else if (tid < kTcCols && col0 + tid < a.d_out) {
        const int o = col0 + tid;
        float v[BP], r[BP];
#pragma unroll
        for (int b = 0; b < BP; ++b)
            if (b < a.batch) {
                v[b] = fix_to_f(__ldcg(a.acc + (size_t)b * a.acc_ld + o));
                r[b] = a.res ? a.res[(size_t)b * a.res_ld + o] : 0.f;
            }
        const float bias = a.bias ? bf16f(a.bias[o]) : 0.f;
#pragma unroll
        for (int b = 0; b < BP; ++b)
            if (b < a.batch) {
                a.acc[(size_t)b * a.acc_ld + o] = 0ull;
                float y = v[b];
                if (a.bias) y += bias;
                if (a.res) y = r[b] + y;
                a.out[(size_t)b * a.out_ld + o] = y;
            }
    }
    if (a.peer.n) {   // the block's outputs to every rank (thread tid wrote output column tid)
        if (a.epi == EPI_SILU)
            peer_push_cols(a.peer, a.out, a.out_ld, a.batch, slice * kGuBlock, min(kGuBlock, max(0, a.d_out - col0)));
        else
            peer_push_cols(a.peer, a.out, a.out_ld, a.batch, col0, min(kTcCols, max(0, a.d_out - col0)));
    }
    tl_stamp(a.tl, 4);
}

}  // namespace larosa
