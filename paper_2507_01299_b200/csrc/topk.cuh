// topk.cuh — exact per-token Top-K (S_k of eq. 2) as a block-wide radix
// select on the uint32 keys bits(|x|), with the lower-index tie-break, plus the
// RMS scale of the h1/h3 sites and stable compaction to ascending indices.
//
// One CTA (1024 threads) per token, latency-optimised (it sits between two dependent GEMVs):
//  * thread t owns the contiguous elements [t*EPT, t*EPT + EPT) and keeps their keys in
//    registers for the whole select (one coalesced float4 load per 4 elements; no shared
//    memory copy of the vector);
//  * digits: bits [30:19] (4096 bins), [18:7] (4096), [6:0] (128); a pass whose k-th-key
//    bucket is taken whole ends the select (continuous data: 2 passes); double-buffered
//    histograms so the next pass's zeroing overlaps the current one;
//  * the bucket search is a warp-level suffix scan with one shared exchange of warp totals;
//  * exact key ties straddling position k are resolved by index (lower index first);
//  * compaction is one block-wide exclusive scan of per-thread counts (contiguous
//    ownership keeps the output ascending).
#pragma once
#include "common.cuh"
#include "gemv.cuh"   // fixed-point accumulator helpers, kGuBlock

namespace larosa {

constexpr int kTopkThreads = 1024;
constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int kTopkBins = 4096;

__host__ __device__ constexpr size_t topk_smem_bytes(int d) {
    return sizeof(int) * 2 * kTopkBins + sizeof(int) * 256 + 0 * (size_t)d;
}

// elements per thread (rounded up to an instantiated size) for a vector of length d
__host__ __device__ constexpr int topk_ept(int d) {
    return ((d + 4 * kTopkThreads - 1) / (4 * kTopkThreads)) * 4;
}

// Where the site's input vector comes from (the producer GEMV leaves fixed-point
// accumulators; the Top-K kernel finalises them, see gemv.cuh):
enum TopkSrc : int {
    SRC_PLAIN = 0,      // x[i]
    SRC_RESID_ACC = 1,  // [resid[i] +] fix^-1(acc[i])                    (residual add)
    SRC_SILU_GU = 2,    // SiLU(g_i) * u_i, g/u = fix^-1 of the interleaved gate|up acc
};

struct TopkSrcArgs {
    const float* resid;          // SRC_RESID_ACC
    unsigned long long* acc;     // SRC_RESID_ACC / SRC_SILU_GU: read, then re-zeroed
    unsigned long long* zero;    // optional extra accumulator to re-zero (zero_n entries)
    int zero_n;
};

struct TopkOut {
    float* xr_out;     // [d] copy of the (rotated / finalised) input, or nullptr
    int32_t* idx;      // [k]
    float* vals;       // [k]
    uint32_t* mask;    // [ceil(d/32)] or nullptr
    float* scale_out;  // [1] the RMS scale s (1 when rms_eps < 0), or nullptr
};

// exclusive prefix over one int per thread in thread order; 1 __syncthreads.
__device__ __forceinline__ int topk_excl_scan(int v, int* sw, int* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int inc = warp_incl_scan(v);
    if (lane == 31) sw[wid] = inc;
    __syncthreads();
    const int t = sw[lane];                       // kTopkWarps == 32
    const int ti = warp_incl_scan(t);
    *total = __shfl_sync(0xffffffffu, ti, 31);
    return __shfl_sync(0xffffffffu, ti - t, wid) + inc - v;
}

template <int EPT>
__device__ void block_topk_t(const float* __restrict__ x, int d, int k, float rms_eps, TopkOut out,
                             unsigned char* smem_raw) {
    constexpr int NT = kTopkThreads;
    int* hist0 = reinterpret_cast<int*>(smem_raw);
    int* hist1 = hist0 + kTopkBins;
    int* scr = hist1 + kTopkBins;
    int* s_wtot = scr;                                   // [0, 32)   scan scratch (select)
    int* s_cnt = scr + 32;                               // [32, 160) per-round warp counts, 2 x [2][32]
    float* s_ssq = reinterpret_cast<float*>(scr + 160);  // [160, 192)
    int* s_res = scr + 192;                              // [192, 196) bucket result
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

    // 1. strided ownership: element j*NT + tid lives in xv[j] (raw fp32 bits) -- coalesced
    //    loads, and each warp-round of 32 consecutive elements is one mask word.
    //    (L2 loads: the vector may have been written by other CTAs of this kernel's cluster.)
    uint32_t xv[EPT];
    float ssq = 0.f;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
        const int i = j * NT + tid;
        const float v = i < d ? __ldcg(x + i) : 0.f;
        xv[j] = __float_as_uint(v);
        ssq = fmaf(v, v, ssq);
        if (out.xr_out && i < d) out.xr_out[i] = v;
    }
#define KEY(j) (xv[j] & 0x7fffffffu)
    ssq = warp_sum(ssq);
    if (lane == 0) s_ssq[wid] = ssq;
    for (int b = tid; b < kTopkBins; b += NT) hist0[b] = 0;
    __syncthreads();

    // 2. radix select of the k-th largest key
    uint32_t prefix = 0u, pmask = 0u;
    int rem = k;
    bool exact_ge = false;   // select key >= thr (the k-th key's bucket is taken whole)
    bool tie_mode = false;   // select key > thr, plus the first `rem` keys == thr by index
    if (k <= 0 || k >= d) {
        exact_ge = true;
        prefix = (k >= d) ? 0u : 0xffffffffu;   // keys < 2^31, so k == 0 selects nothing
    } else {
#pragma unroll 1
        for (int pass = 0; pass < 3; ++pass) {
            int* hist = (pass & 1) ? hist1 : hist0;
            int* hnext = (pass & 1) ? hist0 : hist1;
            const int sh = pass == 0 ? 19 : (pass == 1 ? 7 : 0);
            const int nb = pass == 2 ? 128 : 4096;
            const uint32_t dmask = (uint32_t)(nb - 1);
#pragma unroll
            for (int j = 0; j < EPT; ++j)
                if (j * NT + tid < d && (KEY(j) & pmask) == prefix) atomicAdd(&hist[(KEY(j) >> sh) & dmask], 1);
            if (pass < 2)
                for (int b = tid; b < kTopkBins; b += NT) hnext[b] = 0;
            __syncthreads();
            // suffix scan: warp w owns the bins [nb - (w+1)*bpw, nb - w*bpw), top bins first
            const int bpw = nb / kTopkWarps;              // 128 or 4
            const int bpl = bpw >= 32 ? bpw / 32 : 1;     // 4 or 1
            const int lhi = nb - wid * bpw - lane * bpl;  // lane's bins [lhi - bpl, lhi)
            int c = 0;
            if (lane * bpl < bpw)
                for (int b = lhi - 1; b >= lhi - bpl; --b) c += hist[b];
            const int inc = warp_incl_scan(c);
            if (lane == 31) s_wtot[wid] = inc;
            __syncthreads();
            const int t = s_wtot[lane];
            const int ti = warp_incl_scan(t);
            const int before = __shfl_sync(0xffffffffu, ti - t, wid) + inc - c;
            if (c > 0 && before < rem && rem <= before + c) {
                int acc = before;
                for (int b = lhi - 1; b >= lhi - bpl; --b) {
                    const int h = hist[b];
                    if (acc + h >= rem) {
                        s_res[0] = b;
                        s_res[1] = rem - acc;
                        s_res[2] = h;
                        break;
                    }
                    acc += h;
                }
            }
            __syncthreads();
            const int bstar = s_res[0];
            rem = s_res[1];
            const int cnt = s_res[2];
            prefix |= (uint32_t)bstar << sh;
            pmask |= dmask << sh;
            if (cnt == rem) {
                exact_ge = true;
                break;
            }
            if (pass == 2) tie_mode = true;
        }
    }
    const uint32_t thr = prefix;
    float tot_ssq = 0.f;
#pragma unroll
    for (int w = 0; w < kTopkWarps; ++w) tot_ssq += s_ssq[w];   // fixed order: deterministic
    const float scale = rms_eps >= 0.f ? 1.0f / sqrtf(tot_ssq / (float)d + rms_eps) : 1.0f;

    // 3. stable compaction, one round of NT consecutive elements at a time: warp ballots give
    //    in-warp ranks, warp counts exchanged through shared memory (double-buffered, one
    //    __syncthreads per round) give the block offsets; the stores are consecutive.
    const uint32_t lt = (1u << lane) - 1u;
    int base = 0, eq_base = 0;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
        const int i = j * NT + tid;
        const bool valid = i < d;
        const uint32_t key = KEY(j);
        bool gt, eq;
        if (exact_ge) {
            gt = valid && key >= thr;
            eq = false;
        } else {
            gt = valid && key > thr;
            eq = valid && key == thr;
        }
        const uint32_t bgt = __ballot_sync(0xffffffffu, gt);
        const uint32_t beq = __ballot_sync(0xffffffffu, eq);
        int* cnt = s_cnt + (j & 1) * 64;
        if (lane == 0) {
            cnt[wid] = __popc(bgt);
            cnt[32 + wid] = __popc(beq);
        }
        __syncthreads();
        const int cg = cnt[lane], ce = cnt[32 + lane];
        const int ig = warp_incl_scan(cg), ie = warp_incl_scan(ce);
        const int wg = __shfl_sync(0xffffffffu, ig - cg, wid);        // gt before my warp
        const int we = __shfl_sync(0xffffffffu, ie - ce, wid);        // eq before my warp
        const int tg = __shfl_sync(0xffffffffu, ig, 31), te = __shfl_sync(0xffffffffu, ie, 31);
        // eq element selected iff its index-ordered rank among eq elements is < rem
        const int erank = eq_base + we + __popc(beq & lt);
        const bool sel = gt || (eq && tie_mode && erank < rem);
        const uint32_t bsel = __ballot_sync(0xffffffffu, sel);
        // selected before me = gt before + min(eq before, rem) (eq are taken in index order)
        const int eq_before_warp = eq_base + we;
        const int sel_before_warp = base + wg + (tie_mode ? max(0, min(eq_before_warp, rem) - min(eq_base, rem)) : 0);
        const int pos = sel_before_warp + __popc(bsel & lt);
        if (sel) {
            out.idx[pos] = i;
            out.vals[pos] = __uint_as_float(xv[j]) * scale;
        }
        if (out.mask && lane == 0 && j * NT + wid * 32 < d) out.mask[(j * NT + wid * 32) >> 5] = bsel;
        base += tg + (tie_mode ? max(0, min(eq_base + te, rem) - min(eq_base, rem)) : 0);
        eq_base += te;
    }
    if (out.scale_out && tid == 0) *out.scale_out = scale;
#undef KEY
}

struct TopkKernelArgs {
    const float* x;
    int64_t ldx;
    int d, k;
    float rms_eps;
    float* xr_out;      // [batch][d]: copy of x (plain) / the finalised vector (other modes)
    int32_t* idx;       // [batch][k]
    float* vals;        // [batch][k]
    uint32_t* mask;     // [batch][ceil(d/32)] or null
    float* scale;       // [batch] or null
    int mode;           // TopkSrc
    const float* resid; int64_t resid_ld;                 // SRC_RESID_ACC
    unsigned long long* acc; int64_t acc_ld;              // SRC_RESID_ACC / SRC_SILU_GU
    unsigned long long* zero; int64_t zero_ld; int zero_n; // optional extra zeroing per token
};

// Source finalisation, spread over the CTAs of the token's cluster (coalesced): element i
// of the site's input is computed from the producer GEMV's fixed-point accumulators, written
// to xbuf (the materialised vector the layer keeps: r_mid, h4, x~) and the accumulators are
// re-zeroed.  Then a cluster barrier and CTA 0 runs the select on the whole vector.
template <int MODE>
__device__ void topk_finalize_share(int d, int rank, int cs, TopkSrcArgs src, float* xbuf) {
    const int chunk = (d + cs - 1) / cs;
    const int lo = rank * chunk, hi = min(d, lo + chunk);
#pragma unroll 1
    for (int i = lo + (int)threadIdx.x; i < hi; i += kTopkThreads) {
        float v;
        if constexpr (MODE == SRC_RESID_ACC) {
            v = (src.resid ? src.resid[i] : 0.f) + fix_to_f(src.acc[i]);
            src.acc[i] = 0ull;
        } else {
            const int gi = (i / kGuBlock) * (2 * kGuBlock) + (i % kGuBlock);
            const float g = fix_to_f(src.acc[gi]);
            const float u = fix_to_f(src.acc[gi + kGuBlock]);
            src.acc[gi] = 0ull;
            src.acc[gi + kGuBlock] = 0ull;
            v = g / (1.0f + expf(-g)) * u;
        }
        xbuf[i] = v;
    }
    if (src.zero) {
        const int zc = (src.zero_n + cs - 1) / cs;
        const int zlo = rank * zc, zhi = min(src.zero_n, zlo + zc);
        for (int i = zlo + (int)threadIdx.x; i < zhi; i += kTopkThreads) src.zero[i] = 0ull;
    }
}

__device__ __forceinline__ void topk_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// grid = (CS, batch), cluster (CS, 1, 1): one cluster per token.  One kernel per (source
// mode, elements per thread) so each launch only fetches its own (small) code: these
// latency-bound kernels stalled on instruction-cache misses when one body held every variant.
template <int MODE, int EPT>
__global__ void __launch_bounds__(kTopkThreads, 1) topk_kernel(TopkKernelArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.y, rank = blockIdx.x, cs = gridDim.x;
    const int nwords = (a.d + 31) / 32;
    TopkOut o;
    o.xr_out = nullptr;
    o.idx = a.idx + (size_t)b * a.k;
    o.vals = a.vals + (size_t)b * a.k;
    o.mask = a.mask ? a.mask + (size_t)b * nwords : nullptr;
    o.scale_out = a.scale ? a.scale + b : nullptr;
    const float* x;
    if constexpr (MODE == SRC_PLAIN) {
        x = a.x + (size_t)b * a.ldx;
        o.xr_out = a.xr_out ? a.xr_out + (size_t)b * a.d : nullptr;
    } else {
        TopkSrcArgs src;
        src.resid = a.resid ? a.resid + (size_t)b * a.resid_ld : nullptr;
        src.acc = a.acc + (size_t)b * a.acc_ld;
        src.zero = a.zero ? a.zero + (size_t)b * a.zero_ld : nullptr;
        src.zero_n = a.zero_n;
        float* xbuf = a.xr_out + (size_t)b * a.d;
        topk_finalize_share<MODE>(a.d, rank, cs, src, xbuf);
        topk_cluster_sync();
        x = xbuf;
    }
    if (rank != 0) return;
    block_topk_t<EPT>(x, a.d, a.k, a.rms_eps, o, smem);
}

}  // namespace larosa
