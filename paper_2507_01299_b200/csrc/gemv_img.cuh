// gemv_img.cuh — batch 8-16 decode GEMV on tcgen05 with the token operand PRE-BUILT (SURVEY §8(a)
// a5 at B >= 8; the union of 16 tokens' kept rows is every row, so each row streams once and every
// token's value is 0 where its own Top-K dropped it, Z22):
//
//   acc[b][o] += fix( sum_{r in [lo, lo + n)} v_b[r] * W[r][o] )        (same contract as gemv.cuh)
//
// The token operand of a 64-row chunk -- the 16 tokens' masked, RMS-scaled values split into bf16
// hi (MMA rows 0-15) and lo (rows 16-31) -- is written ONCE per site, in the exact 128-byte-swizzled
// K-major shared-memory image the MMA reads, by the kernel that computes the tokens' Top-K rules
// (rule_image_kernel) or by dense_image_kernel (the adapter, the LM head).  Every GEMV CTA then
// moves it with one 4 KB cp.async.bulk per chunk beside the two TMA boxes of its weight tile: no
// value loads, rule checks or conversions sit on the MMA's critical path (gemv_tc.cuh does those
// per chunk in 128 producer threads and streamed at ~3.8 TB/s).
//   warp 0: producer (one lane): per chunk, expect_tx(16 KB + 4 KB), two weight boxes (TMA 2D),
//           the token image (bulk copy);  warp 1: TMEM allocation and the MMA issuer (one lane):
//           4 x tcgen05.mma (M = 128 columns, N = 32 = hi | lo, K = 16), tcgen05.commit frees the
//           stage;  warps 2-5: epilogue -- tcgen05.ld of 32 TMEM columns per lane (= output
//           column), hi + lo, one fixed-point red per token, then the slice ticket / finalise of
//           gemv_tc.cuh.
#pragma once
#include "gemv_tc.cuh"
#include "img_layout.cuh"

namespace larosa {

static_assert(kImgChunkBytes == 2 * kTcBBytes, "image chunk = 32 MMA rows (16 hi, 16 lo) x 64 K x bf16");
constexpr int kImgStageBytes = kTcABytes + kImgChunkBytes;   // 20 KB
#ifndef LAROSA_IMG_STAGES
#define LAROSA_IMG_STAGES 4
#endif
constexpr int kImgStages = LAROSA_IMG_STAGES;
constexpr int kImgThreads = 192;
__host__ __device__ constexpr size_t gemv_img_smem_bytes() { return 1024 + (size_t)kImgStages * kImgStageBytes + 128; }

__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem_dst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <int BP>
__global__ void __launch_bounds__(kImgThreads, 1) gemv_img_kernel(const GemvArgs a, const __grid_constant__ CUtensorMap tmw) {
    static_assert(BP >= 2 && BP <= kTcN, "image GEMV: batch 2..16");
    extern __shared__ __align__(1024) unsigned char img_smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(img_smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kImgStages * kImgStageBytes);
    uint64_t* empty = full + kImgStages;
    uint64_t* accb = empty + kImgStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accb + 1);
    int* flag = reinterpret_cast<int*>(tmem_slot + 1);
    const int slice = blockIdx.x, split = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int col0 = slice * kTcCols;
    int lo, n_rows;
    tc_split_range(a.d_in, a.n_splits, split, lo, n_rows);
    const int n_chunks = (n_rows + kTcChunk - 1) / kTcChunk;
    tl_stamp(a.tl, 0);

    if (tid == 0) {
        for (int s = 0; s < kImgStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accb, 1);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmw)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const unsigned char* img = reinterpret_cast<const unsigned char*>(a.img) + (size_t)(lo / kTcChunk) * kImgChunkBytes;

    if (warp == 0) {
        if (lane == 0) {
            // the weight tiles of the first stages do not depend on the previous kernel
            const int pre = min(kImgStages, n_chunks);
            for (int c = 0; c < pre; ++c) {
                unsigned char* st = smem + c * kImgStageBytes;
                mbar_arrive_expect_tx(&full[c], kImgStageBytes);
                tma_load_2d(st, &tmw, col0, lo + c * kTcChunk, &full[c]);
                tma_load_2d(st + kTcABytes / 2, &tmw, col0 + 64, lo + c * kTcChunk, &full[c]);
            }
            pdl_wait();       // the token image comes from the previous kernel
            tl_stamp_any(a.tl, 1);
            for (int c = 0; c < pre; ++c)
                bulk_g2s(smem + c * kImgStageBytes + kTcABytes, img + (size_t)c * kImgChunkBytes, kImgChunkBytes, &full[c]);
            for (int c = pre; c < n_chunks; ++c) {
                const int s = c % kImgStages;
                mbar_wait_parity(&empty[s], ((c / kImgStages) & 1) ^ 1);
                unsigned char* st = smem + s * kImgStageBytes;
                mbar_arrive_expect_tx(&full[s], kImgStageBytes);
                tma_load_2d(st, &tmw, col0, lo + c * kTcChunk, &full[s]);
                tma_load_2d(st + kTcABytes / 2, &tmw, col0 + 64, lo + c * kTcChunk, &full[s]);
                bulk_g2s(st + kTcABytes, img + (size_t)c * kImgChunkBytes, kImgChunkBytes, &full[s]);
            }
        } else {
            pdl_wait();
        }
    } else {
        pdl_wait();
    }
    pdl_trigger();
    if (warp == 1) {
        if (lane == 0) {
            for (int c = 0; c < n_chunks; ++c) {
                const int s = c % kImgStages;
                mbar_wait_parity(&full[s], (c / kImgStages) & 1);
                tc_fence_after();
                unsigned char* st = smem + s * kImgStageBytes;
                const int rows = min(kTcChunk, n_rows - c * kTcChunk);
#pragma unroll
                for (int ks = 0; ks < kTcChunk / 16; ++ks) {
                    if (16 * ks >= rows) break;
                    umma_bf16(tmem, umma_desc_mn_sw128(st + ks * 2048, 8192, 1024), umma_desc_sw128(st + kTcABytes + ks * 32),
                              kTcIdesc2, c > 0 || ks > 0);
                }
                umma_commit(&empty[s]);
            }
            umma_commit(accb);
        }
        __syncwarp();
    } else if (warp >= 2 && n_chunks > 0) {
        // epilogue warps: TMEM lanes 32 (w % 4) .. = output columns col0 + 32 (w % 4) + lane
        const int q = warp & 3;
        mbar_wait_parity(accb, 0);
        tc_fence_after();
        if (tid == 64) tl_stamp_any(a.tl, 3);   // the accumulator is complete
        uint32_t v[16], w[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + ((uint32_t)(32 * q) << 16)));
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15}, [%16];"
            : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
              "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
            : "r"(tmem + ((uint32_t)(32 * q) << 16) + 16u));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int o = col0 + 32 * q + lane;
        if (o < a.d_out)
#pragma unroll
            for (int b = 0; b < BP; ++b)
                if (b < a.batch)
                    red_fix(a.acc + (size_t)b * a.acc_ld + o, __uint_as_float(v[b]) + __uint_as_float(w[b]), a.err);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
    if (a.epi == EPI_NONE) {
        tl_stamp(a.tl, 4);
        return;
    }

    // ---- the last split CTA of this slice finalises its 128 columns (as gemv_tc.cuh) -------------
    if (tid == 0) *flag = atom_add_acq_rel_gpu(a.tickets + slice, 1u) == gridDim.y - 1u;
    tl_stamp(a.tl, 12);
    __syncthreads();
    if (!*flag) {
        tl_stamp(a.tl, 4);
        return;
    }
    tl_stamp(a.tl, 13);
    if (tid == 0) a.tickets[slice] = 0u;
    const int e = tid - 64;                       // epilogue threads 0..127 (tid 0..63 idle)
    if (e < 0) {
    } else if (a.epi == EPI_SILU) {
        if (e < kGuBlock && col0 + e < a.d_out) {
            float g[BP], u[BP];
#pragma unroll
            for (int b = 0; b < BP; ++b)
                if (b < a.batch) {
                    const unsigned long long* acc = a.acc + (size_t)b * a.acc_ld + col0 + e;
                    g[b] = fix_to_f(__ldcg(acc));
                    u[b] = fix_to_f(__ldcg(acc + kGuBlock));
                }
#pragma unroll
            for (int b = 0; b < BP; ++b)
                if (b < a.batch) {
                    unsigned long long* acc = a.acc + (size_t)b * a.acc_ld + col0 + e;
                    acc[0] = 0ull;
                    acc[kGuBlock] = 0ull;
                    a.out[(size_t)b * a.out_ld + slice * kGuBlock + e] = g[b] / (1.0f + expf(-g[b])) * u[b];
                }
        }
    } else if (col0 + e < a.d_out) {
        const int o = col0 + e;
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
    tl_stamp(a.tl, 4);
    if (a.peer.n) {   // the block's outputs to every rank (thread e wrote output column e)
        if (a.epi == EPI_SILU)
            peer_push_cols(a.peer, a.out, a.out_ld, a.batch, slice * kGuBlock, min(kGuBlock, max(0, a.d_out - col0)));
        else
            peer_push_cols(a.peer, a.out, a.out_ld, a.batch, col0, min(kTcCols, max(0, a.d_out - col0)));
    }
}

// ---- the token images --------------------------------------------------------------------------
// Rule + image (batch > 1, one CTA per token b): the exact Top-K rule of x_b (lower index on ties,
// Z10), the RMS scale (fixed-order block sum), the ThreshOut record, and the token's masked, scaled,
// hi/lo-split values in the image; img_raw (optional): the unmasked, unscaled values (the dense
// adapter on the same vector).  The rule is a 3-level radix select over the key bits(|x|) held in
// shared memory -- 4096-bin histograms (warp-aggregated shared atomics) of bits 30:19, then of
// bits 18:7 and 6:0 of the keys inside the chosen bucket, each located by a block suffix scan --
// and the index tie-break (the need-th lowest index among keys equal to the k-th) by a block
// prefix count in index order.
constexpr int kRiThreads = 512;
constexpr int kRiBins = 4096;
__host__ __device__ constexpr size_t rule_image_smem_bytes(int d) { return (size_t)d * 4 + (size_t)kRiBins * 4 + 512; }

// the bin holding the rank-th largest key (bins ascending in key), and the rank inside it
__device__ __forceinline__ void ri_find(const int* hist, int rank, int* misc, int* wsum) {
    constexpr int NW = kRiThreads / 32;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int c8[8], tot = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        c8[j] = hist[8 * tid + j];
        tot += c8[j];
    }
    int incl = tot;   // sum over lanes >= lane of this warp
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_down_sync(0xffffffffu, incl, o);
        if (lane + o < 32) incl += v;
    }
    if (lane == 0) wsum[wid] = incl;
    __syncthreads();
    int above = incl - tot;
    for (int w = wid + 1; w < NW; ++w) above += wsum[w];
    if (above < rank && above + tot >= rank) {
        int acc = above;
#pragma unroll
        for (int j = 7; j >= 0; --j) {
            if (acc + c8[j] >= rank) {
                misc[0] = 8 * tid + j;
                misc[1] = rank - acc;
                break;
            }
            acc += c8[j];
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kRiThreads) rule_image_kernel(const float* __restrict__ X, int64_t ldx, int d, int k,
                                                                float eps, ThreshOut* __restrict__ rule,
                                                                unsigned char* __restrict__ img,
                                                                unsigned char* __restrict__ img_raw) {
    extern __shared__ __align__(16) float ris[];
    float* xs = ris;                                          // [d]
    int* hist = reinterpret_cast<int*>(xs + d);               // [4096]
    int* misc = hist + kRiBins;                               // [32]
    int* wsum = misc + 32;                                    // [16]
    float* fred = reinterpret_cast<float*>(wsum + 16);        // [16]
    constexpr int NW = kRiThreads / 32;
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < kRiBins; i += kRiThreads) hist[i] = 0;
    pdl_wait();
    pdl_trigger();
    const float* x = X + (size_t)b * ldx;
    for (int i = tid; i < d; i += kRiThreads) xs[i] = x[i];
    __syncthreads();
    uint32_t tk = 0u;
    int ti = 0x7fffffff;
    if (k <= 0) {
        tk = 0xffffffffu;
        ti = -1;
    } else if (k < d) {
        uint32_t prefix = 0u, pmask = 0u;
        int rank = k;
        const int shifts[3] = {19, 7, 0};
        const uint32_t widths[3] = {0xfffu, 0xfffu, 0x7fu};
#pragma unroll 1
        for (int lv = 0; lv < 3; ++lv) {
            const int sh = shifts[lv];
            const uint32_t wm = widths[lv];
            for (int i0 = 0; i0 < d; i0 += kRiThreads) {
                const int i = i0 + tid;
                uint32_t bin = 0xffffffffu;
                if (i < d) {
                    const uint32_t key = key_of(xs[i]);
                    if ((key & pmask) == prefix) bin = (key >> sh) & wm;
                }
                const unsigned act = __ballot_sync(0xffffffffu, bin != 0xffffffffu);
                if (bin != 0xffffffffu) {
                    const unsigned peers = __match_any_sync(act, bin);
                    if (lane == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
                }
            }
            __syncthreads();
            ri_find(hist, rank, misc, wsum);
            prefix |= (uint32_t)misc[0] << sh;
            pmask |= wm << sh;
            rank = misc[1];
            for (int i = tid; i < kRiBins; i += kRiThreads) hist[i] = 0;   // (for the next level / call)
            __syncthreads();
        }
        tk = prefix;
        const int need = rank;      // keys equal to tk still to take, lowest indices first
        const int per = (d + kRiThreads - 1) / kRiThreads;
        const int i0 = tid * per, i1 = min(d, i0 + per);
        int mine = 0;
        for (int i = i0; i < i1; ++i) mine += key_of(xs[i]) == tk;
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wsum[wid] = incl;
        __syncthreads();
        int before = incl - mine;
        for (int w = 0; w < wid; ++w) before += wsum[w];
        if (before < need && before + mine >= need) {
            int c = before;
            for (int i = i0; i < i1; ++i)
                if (key_of(xs[i]) == tk && ++c == need) {
                    misc[2] = i;
                    break;
                }
        }
        __syncthreads();
        ti = misc[2];
    }
    float s = 1.f;
    if (eps >= 0.f) {
        float q = 0.f;
        for (int i = tid; i < d; i += kRiThreads) q = fmaf(xs[i], xs[i], q);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
        if (lane == 0) fred[wid] = q;
        __syncthreads();
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) t += fred[w];
        s = 1.0f / sqrtf(t / (float)d + eps);
    }
    if (tid == 0) {
        ThreshOut r;
        r.tk = tk;
        r.ti = ti;
        r.scale = s;
        r.pad = 0;
        rule[b] = r;
    }
    if (!img) return;
    // the image: one 16-byte group of 8 consecutive rows per thread and iteration (hi, lo)
    const int ngroups = (d + 7) / 8;
    for (int g = tid; g < ngroups; g += kRiThreads) {
        uint32_t hi[4], lw[4], rh[4], rl[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            float f[2], r2[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int i = g * 8 + 2 * h + u;
                const float v = i < d ? xs[i] : 0.f;
                const uint32_t key = key_of(v);
                const bool kp = i < d && (key > tk || (key == tk && i <= ti));
                f[u] = kp ? v * s : 0.f;
                r2[u] = v;
            }
            hi[h] = cvt_bf16x2(f[0], f[1]);
            lw[h] = cvt_bf16x2(f[0] - __uint_as_float(hi[h] << 16), f[1] - __uint_as_float(hi[h] & 0xffff0000u));
            rh[h] = cvt_bf16x2(r2[0], r2[1]);
            rl[h] = cvt_bf16x2(r2[0] - __uint_as_float(rh[h] << 16), r2[1] - __uint_as_float(rh[h] & 0xffff0000u));
        }
        const int i0 = g * 8;
        const size_t cb = (size_t)(i0 >> 6) * kImgChunkBytes;
        const int k8 = (i0 & 63) >> 3;
        const int oh = (b >> 3) * 1024 + (b & 7) * 128 + ((k8 ^ (b & 7)) << 4);
        const int ol = ((16 + b) >> 3) * 1024 + ((16 + b) & 7) * 128 + ((k8 ^ ((16 + b) & 7)) << 4);
        *reinterpret_cast<uint4*>(img + cb + oh) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(img + cb + ol) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        if (img_raw) {
            *reinterpret_cast<uint4*>(img_raw + cb + oh) = make_uint4(rh[0], rh[1], rh[2], rh[3]);
            *reinterpret_cast<uint4*>(img_raw + cb + ol) = make_uint4(rl[0], rl[1], rl[2], rl[3]);
        }
    }
}

// Register-resident variant (LAROSA_RULE_KERNEL=3): x_b lives in registers (EPT values per thread,
// element e * 512 + tid), so the CTA needs only the 16 KB histogram in shared memory and can become
// resident while the producer GEMV still runs (programmatic dependent launch).  Same rule: 3-level
// radix select, then the need-th lowest index among keys equal to the k-th (the equal keys are
// compacted -- usually one -- and warp 0 picks; a bitwise index search over block counts if more
// than kRiEqCap share the key).  RMS: per-thread sums in element order, fixed-order tree.  The image
// is written value by value (2-byte stores, 8 consecutive lanes fill one 16-byte group).
constexpr int kRiEqCap = 1024;
template <int EPT>
__global__ void __launch_bounds__(kRiThreads) rule_image_reg_kernel(const float* __restrict__ X, int64_t ldx, int d,
                                                                    int k, float eps, ThreshOut* __restrict__ rule,
                                                                    unsigned char* __restrict__ img,
                                                                    unsigned char* __restrict__ img_raw) {
    __shared__ int hist[kRiBins];
    __shared__ int eqi[kRiEqCap];
    __shared__ int misc[32];
    __shared__ int wsum[16];
    __shared__ float fred[16];
    constexpr int NW = kRiThreads / 32;
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < kRiBins; i += kRiThreads) hist[i] = 0;
    if (tid < 32) misc[tid] = 0;
    pdl_wait();
    pdl_trigger();
    const float* x = X + (size_t)b * ldx;
    float v[EPT];
    uint32_t key[EPT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        const int i = e * kRiThreads + tid;
        v[e] = i < d ? x[i] : 0.f;
        key[e] = i < d ? key_of(v[e]) : 0xffffffffu;   // past the end: never binned, never kept
    }
    __syncthreads();
    uint32_t tk = 0u;
    int ti = 0x7fffffff;
    if (k <= 0) {
        tk = 0xffffffffu;
        ti = -1;
    } else if (k < d) {
        uint32_t prefix = 0u, pmask = 0u;
        int rank = k;
#pragma unroll 1
        for (int lv = 0; lv < 3; ++lv) {
            const int sh = lv == 0 ? 19 : (lv == 1 ? 7 : 0);
            const uint32_t wm = lv == 2 ? 0x7fu : 0xfffu;
#pragma unroll
            for (int e = 0; e < EPT; ++e) {
                const bool ok = key[e] != 0xffffffffu && (key[e] & pmask) == prefix;
                const uint32_t bin = ok ? (key[e] >> sh) & wm : 0xffffffffu;
                const unsigned act = __ballot_sync(0xffffffffu, ok);
                if (ok) {
                    const unsigned peers = __match_any_sync(act, bin);
                    if (lane == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
                }
            }
            __syncthreads();
            ri_find(hist, rank, misc, wsum);
            prefix |= (uint32_t)misc[0] << sh;
            pmask |= wm << sh;
            rank = misc[1];
            for (int i = tid; i < kRiBins; i += kRiThreads) hist[i] = 0;
            __syncthreads();
        }
        tk = prefix;
        const int need = rank;
        // compact the indices of the keys equal to tk
#pragma unroll
        for (int e = 0; e < EPT; ++e)
            if (key[e] == tk) {
                const int slot = atomicAdd(&misc[4], 1);
                if (slot < kRiEqCap) eqi[slot] = e * kRiThreads + tid;
            }
        __syncthreads();
        const int neq = misc[4];
        if (neq <= kRiEqCap) {
            if (wid == 0) {   // the need-th smallest index: bitwise search over the index bits
                int idx = 0;
#pragma unroll 1
                for (int bit = 15; bit >= 0; --bit) {
                    const int cnd = idx | (1 << bit);
                    int n = 0;
                    for (int q = lane; q < neq; q += 32) n += eqi[q] < cnd;
                    n = __reduce_add_sync(0xffffffffu, n);
                    if (n < need) idx = cnd;
                }
                if (lane == 0) misc[5] = idx;
            }
        } else {
#pragma unroll 1
            for (int bit = 15; bit >= 0; --bit) {
                const int cnd = misc[6] | (1 << bit);
                int n = 0;
#pragma unroll
                for (int e = 0; e < EPT; ++e) n += key[e] == tk && e * kRiThreads + tid < cnd;
                n = __reduce_add_sync(0xffffffffu, n);
                if (lane == 0) wsum[wid] = n;
                __syncthreads();
                int t = 0;
#pragma unroll
                for (int w = 0; w < NW; ++w) t += wsum[w];
                if (tid == 0 && t < need) misc[6] = cnd;
                __syncthreads();
            }
            if (tid == 0) misc[5] = misc[6];
        }
        __syncthreads();
        ti = misc[5];
    }
    float s = 1.f;
    if (eps >= 0.f) {
        float q = 0.f;
#pragma unroll
        for (int e = 0; e < EPT; ++e) q = fmaf(v[e], v[e], q);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
        if (lane == 0) fred[wid] = q;
        __syncthreads();
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) t += fred[w];
        s = 1.0f / sqrtf(t / (float)d + eps);
    }
    if (tid == 0) {
        ThreshOut r;
        r.tk = tk;
        r.ti = ti;
        r.scale = s;
        r.pad = 0;
        rule[b] = r;
    }
    if (!img) return;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        const int i = e * kRiThreads + tid;
        if (i >= d) break;
        const bool kp = key[e] > tk || (key[e] == tk && i <= ti);
        const float f = kp ? v[e] * s : 0.f;
        const uint16_t h = f2bf16_rne(f);
        const uint16_t l = f2bf16_rne(f - bf16f(h));
        unsigned char* ch = img + (size_t)(i >> 6) * kImgChunkBytes;
        const int kk = i & 63;
        *reinterpret_cast<uint16_t*>(ch + img_off(b, kk)) = h;
        *reinterpret_cast<uint16_t*>(ch + img_off(16 + b, kk)) = l;
        if (img_raw) {
            const uint16_t rh = f2bf16_rne(v[e]);
            unsigned char* cr = img_raw + (size_t)(i >> 6) * kImgChunkBytes;
            *reinterpret_cast<uint16_t*>(cr + img_off(b, kk)) = rh;
            *reinterpret_cast<uint16_t*>(cr + img_off(16 + b, kk)) = f2bf16_rne(v[e] - bf16f(rh));
        }
    }
}

// Image from per-token rules computed elsewhere (the cluster Top-K kernel): token b's values, masked
// by its rule and scaled, split hi/lo; img_raw (optional): unmasked, unscaled.  grid = (groups/256, B)
__global__ void rule_apply_image_kernel(const float* __restrict__ X, int64_t ldx, int d, const ThreshOut* __restrict__ rules,
                                        unsigned char* __restrict__ img, unsigned char* __restrict__ img_raw) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.y;
    const ThreshOut r = rules[b];
    const int ngroups = (d + 7) / 8;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += gridDim.x * blockDim.x) {
        uint32_t hi[4], lw[4], rh[4], rl[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            float f[2], r2[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int i = g * 8 + 2 * h + u;
                const float v = i < d ? X[(size_t)b * ldx + i] : 0.f;
                const uint32_t key = key_of(v);
                const bool kp = i < d && (key > r.tk || (key == r.tk && i <= r.ti));
                f[u] = kp ? v * r.scale : 0.f;
                r2[u] = v;
            }
            hi[h] = cvt_bf16x2(f[0], f[1]);
            lw[h] = cvt_bf16x2(f[0] - __uint_as_float(hi[h] << 16), f[1] - __uint_as_float(hi[h] & 0xffff0000u));
            rh[h] = cvt_bf16x2(r2[0], r2[1]);
            rl[h] = cvt_bf16x2(r2[0] - __uint_as_float(rh[h] << 16), r2[1] - __uint_as_float(rh[h] & 0xffff0000u));
        }
        const int i0 = g * 8;
        const size_t cb = (size_t)(i0 >> 6) * kImgChunkBytes;
        const int k8 = (i0 & 63) >> 3;
        const int oh = (b >> 3) * 1024 + (b & 7) * 128 + ((k8 ^ (b & 7)) << 4);
        const int ol = ((16 + b) >> 3) * 1024 + ((16 + b) & 7) * 128 + ((k8 ^ ((16 + b) & 7)) << 4);
        *reinterpret_cast<uint4*>(img + cb + oh) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(img + cb + ol) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        if (img_raw) {
            *reinterpret_cast<uint4*>(img_raw + cb + oh) = make_uint4(rh[0], rh[1], rh[2], rh[3]);
            *reinterpret_cast<uint4*>(img_raw + cb + ol) = make_uint4(rl[0], rl[1], rl[2], rl[3]);
        }
    }
}

// Dense image: token b's values x_b (times scale[b] if given) split hi/lo into the image.
// grid = (groups / 256, batch)
__global__ void dense_image_kernel(const float* __restrict__ X, int64_t ldx, int d, unsigned char* __restrict__ img) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.y;
    const int ngroups = (d + 7) / 8;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += gridDim.x * blockDim.x) {
        uint32_t hi[4], lw[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const int i = g * 8 + 2 * h;
            const float f0 = i < d ? X[(size_t)b * ldx + i] : 0.f, f1 = i + 1 < d ? X[(size_t)b * ldx + i + 1] : 0.f;
            hi[h] = cvt_bf16x2(f0, f1);
            lw[h] = cvt_bf16x2(f0 - __uint_as_float(hi[h] << 16), f1 - __uint_as_float(hi[h] & 0xffff0000u));
        }
        const int i0 = g * 8;
        const size_t cb = (size_t)(i0 >> 6) * kImgChunkBytes;
        const int k8 = (i0 & 63) >> 3;
        const int oh = (b >> 3) * 1024 + (b & 7) * 128 + ((k8 ^ (b & 7)) << 4);
        const int ol = ((16 + b) >> 3) * 1024 + ((16 + b) & 7) * 128 + ((k8 ^ ((16 + b) & 7)) << 4);
        *reinterpret_cast<uint4*>(img + cb + oh) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(img + cb + ol) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

}  // namespace larosa
