// gemv_tc.cuh — batched sparse GEMV on the 5th-generation tensor cores (batch 8-16; SURVEY §7
// hard part 3: at B >= 8 the fp32 CUDA-core FMA rate, not HBM, bounds the CUDA-core GEMV).
//
//   acc[b][o] += fix( sum_{r in rows} val(r, b) * W[row(r)][o] )      (same contract as gemv.cuh)
//
// As an MMA  D[M = 128 columns][N = 16 tokens] += A[M][K = kept rows] . B[K][N]:
//   A = the gathered weight rows, MN-major (a row's 128 columns are contiguous in W): each
//       64-row chunk is copied with per-thread cp.async into the canonical 128-byte-swizzled
//       MN-major layout (atoms of 8 rows x 64 columns; next 64 columns +1 KB, next 8 rows +2 KB);
//       rows past the list are zero-filled (src-size 0);
//   B = the tokens' values, K-major, split into bf16 hi + lo (two MMAs into the same fp32
//       accumulator keep ~16 mantissa bits of the fp32 activations), written with st.shared;
//   D = 16 fp32 TMEM columns x 128 lanes.
// Warps 0-3 produce (gather + values) into a 4-stage ring whose stages complete through
// cp.async.mbarrier.arrive; one thread of warp 4 issues tcgen05.mma (M = 128, N = 16, K = 16)
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
constexpr int kTcStages = 4;
constexpr int kTcProdWarps = 4;
constexpr int kTcThreads = (kTcProdWarps + 1) * 32;
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
constexpr uint32_t kTcIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(kTcN >> 3) << 17) |
                              ((uint32_t)(kTcCols >> 4) << 24);

__device__ __forceinline__ void cp_async16_zfill(void* smem_dst, const void* gsrc, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)), "l"(gsrc),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int BP, int MODE>
__global__ void __launch_bounds__(kTcThreads, 1) gemv_tc_kernel(const GemvArgs a) {
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
            mbar_init(&full[s], kTcProdWarps * 32);
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
    pdl_wait();
    pdl_trigger();
    tl_stamp(a.tl, 1);
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
        const int rng = (a.d_in + a.n_splits - 1) / a.n_splits;
        lo = min(a.d_in, split * rng);
        n_list = min(a.d_in, lo + rng) - lo;
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
    auto load_raw = [&](int c, float (&r)[8]) {
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
        float nxt[8];
        if (n_chunks > 0) load_raw(0, nxt);
        for (int c = 0; c < n_chunks; ++c) {
            float cur[8];
#pragma unroll
            for (int h = 0; h < 8; ++h) cur[h] = nxt[h];
            const int s = c % kTcStages;
            if (c >= kTcStages) mbar_wait_parity(&empty[s], ((c / kTcStages) & 1) ^ 1);
            unsigned char* st = smem + s * kTcStage;
            // A: 64 rows x 16 chunks of 16 bytes; thread pt takes chunks pt + 128 q
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int u = pt + 128 * q;
                const int r = u >> 4, cc = u & 15;         // row in chunk, 16-byte chunk of the row
                const int e = c * kTcChunk + r;            // list entry
                const bool ok = e < n_list;
                const int row = !ok ? 0 : (MODE == GEMV_LIST ? lrow[e] : lo + e);
                const int mg = cc >> 3, c8 = cc & 7;       // 64-column group, chunk within it
                unsigned char* dst = st + ((r >> 3) * 2 + mg) * 1024 + (r & 7) * 128 + ((c8 ^ (r & 7)) << 4);
                const bool valid = ok && col0 + cc * 8 < a.d_out && !(a.tc_dbg & 4);
                cp_async16_zfill(dst, valid ? a.W + (size_t)row * a.ld + col0 + cc * 8 : a.W, valid);
            }
            // B: token n (0..15) x 8 consecutive rows (16 bytes of hi, 16 of lo) per thread
            if (!(a.tc_dbg & 2)) {
                uint32_t hi[4], lw[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const float f0 = finish(c, 2 * h, cur[2 * h]), f1 = finish(c, 2 * h + 1, cur[2 * h + 1]);
                    const uint16_t h0 = f2bf16_rne(f0), h1 = f2bf16_rne(f1);
                    hi[h] = (uint32_t)h0 | ((uint32_t)h1 << 16);
                    lw[h] = (uint32_t)f2bf16_rne(f0 - bf16f(h0)) | ((uint32_t)f2bf16_rne(f1 - bf16f(h1)) << 16);
                }
                const int off = (pn >> 3) * 1024 + (pn & 7) * 128 + ((pk8 ^ (pn & 7)) << 4);
                *reinterpret_cast<uint4*>(st + kTcABytes + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<uint4*>(st + kTcABytes + kTcBBytes + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            }
            fence_proxy_async_smem();   // the st.shared values, for the tensor core's async proxy
            cp_async_mbar_arrive(&full[s]);
            // the next chunk's values: issued after the fence (which would wait for them), in
            // flight during the next slot wait
            if (c + 1 < n_chunks && !(a.tc_dbg & 2)) load_raw(c + 1, nxt);
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
                const uint64_t da = umma_desc_mn_sw128(st + ks * 4096, 1024, 2048);
                const uint64_t dbh = umma_desc_sw128(st + kTcABytes + ks * 32);
                const uint64_t dbl = umma_desc_sw128(st + kTcABytes + kTcBBytes + ks * 32);
                if (!(a.tc_dbg & 1)) {
                    umma_bf16(tmem, da, dbh, kTcIdesc, c > 0 || ks > 0);
                    umma_bf16(tmem, da, dbl, kTcIdesc, true);
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
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int o = col0 + tid;
        if (o < a.d_out)
#pragma unroll
            for (int b = 0; b < BP; ++b)
                if (b < a.batch) red_add_u64(a.acc + (size_t)b * a.acc_ld + o, f_to_fix(__uint_as_float(v[b])));
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
    if (tid < kTcCols) {
        for (int b = 0; b < a.batch; ++b) {
            unsigned long long* acc = a.acc + (size_t)b * a.acc_ld;
            if (a.epi == EPI_SILU) {
                // the 128-column slice is one gate|up block: 64 gate, then the matching 64 up
                if (tid < kGuBlock && col0 + tid < a.d_out) {
                    const float g = fix_to_f(__ldcg(acc + col0 + tid));
                    const float u = fix_to_f(__ldcg(acc + col0 + tid + kGuBlock));
                    acc[col0 + tid] = 0ull;
                    acc[col0 + tid + kGuBlock] = 0ull;
                    a.out[(size_t)b * a.out_ld + slice * kGuBlock + tid] = g / (1.0f + expf(-g)) * u;
                }
            } else {
                const int o = col0 + tid;
                if (o < a.d_out) {
                    float v = fix_to_f(__ldcg(acc + o));
                    acc[o] = 0ull;
                    if (a.bias) v += bf16f(a.bias[o]);
                    if (a.res) v = a.res[(size_t)b * a.res_ld + o] + v;
                    a.out[(size_t)b * a.out_ld + o] = v;
                }
            }
        }
    }
    tl_stamp(a.tl, 4);
}

}  // namespace larosa
