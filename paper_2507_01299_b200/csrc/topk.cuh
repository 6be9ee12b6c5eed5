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
    return sizeof(int) * 2 * kTopkBins + sizeof(uint32_t) * (size_t)((d + 31) / 32) + sizeof(int) * 160;
}

// elements per thread (multiple of 4) for a vector of length d
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

template <int EPT, int MODE>
__device__ void block_topk_t(const float* __restrict__ x, int d, int k, float rms_eps, TopkOut out,
                             TopkSrcArgs src, unsigned char* smem_raw) {
    constexpr int NT = kTopkThreads;
    int* hist0 = reinterpret_cast<int*>(smem_raw);
    int* hist1 = hist0 + kTopkBins;
    const int nwords = (d + 31) / 32;
    uint32_t* smask = reinterpret_cast<uint32_t*>(hist1 + kTopkBins);
    int* scr = reinterpret_cast<int*>(smask + nwords);
    int* s_wtot = scr;                                   // [0, 32)
    int* s_wtot2 = scr + 32;                             // [32, 64)
    float* s_ssq = reinterpret_cast<float*>(scr + 64);   // [64, 96)
    int* s_res = scr + 96;                               // [96, 100)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int i0 = tid * EPT;

    // 1. values (raw fp32 bits) in registers; key = bits & 0x7fffffff (-0 == +0); sum of squares
    uint32_t xv[EPT];
    float ssq = 0.f;
    if constexpr (MODE == SRC_PLAIN) {
        const bool vec = ((d & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
#pragma unroll
        for (int c = 0; c < EPT / 4; ++c) {
            const int i = i0 + 4 * c;
            float v[4];
            if (vec && i + 4 <= d) {
                const float4 f = *reinterpret_cast<const float4*>(x + i);
                v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = (i + u < d) ? x[i + u] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) xv[4 * c + u] = __float_as_uint(v[u]);
        }
    } else {
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
            const int i = i0 + e;
            float v = 0.f;
            if (i < d) {
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
            }
            xv[e] = __float_as_uint(v);
        }
    }
    if (src.zero)
        for (int i = tid; i < src.zero_n; i += NT) src.zero[i] = 0ull;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        const float v = __uint_as_float(xv[e]);
        ssq = fmaf(v, v, ssq);
        if (out.xr_out && i0 + e < d) out.xr_out[i0 + e] = v;
    }
#define KEY(e) (xv[e] & 0x7fffffffu)
    ssq = warp_sum(ssq);
    if (lane == 0) s_ssq[wid] = ssq;
    for (int b = tid; b < kTopkBins; b += NT) hist0[b] = 0;
    if (out.mask)
        for (int w = tid; w < nwords; w += NT) smask[w] = 0u;
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
            for (int e = 0; e < EPT; ++e)
                if (i0 + e < d && (KEY(e) & pmask) == prefix) atomicAdd(&hist[(KEY(e) >> sh) & dmask], 1);
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

    // 3. stable compaction over the contiguous ownership ranges
    int n_gt = 0, n_eq = 0;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        if (i0 + e >= d) continue;
        if (exact_ge) {
            n_gt += KEY(e) >= thr;
        } else {
            n_gt += KEY(e) > thr;
            n_eq += KEY(e) == thr;
        }
    }
    int take_eq = 0;
    if (tie_mode) {
        int tot;
        const int eq_before = topk_excl_scan(n_eq, s_wtot, &tot);
        take_eq = min(n_eq, max(0, rem - eq_before));
    }
    int tot_sel;
    int pos = topk_excl_scan(n_gt + take_eq, tie_mode ? s_wtot2 : s_wtot, &tot_sel);
    int eq_seen = 0;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        const int i = i0 + e;
        if (i >= d) continue;
        bool sel;
        if (exact_ge) {
            sel = KEY(e) >= thr;
        } else if (KEY(e) > thr) {
            sel = true;
        } else if (KEY(e) == thr) {
            sel = eq_seen < take_eq;
            ++eq_seen;
        } else {
            sel = false;
        }
        if (sel) {
            out.idx[pos] = i;
            out.vals[pos] = __uint_as_float(xv[e]) * scale;
            if (out.mask) atomicOr(&smask[i >> 5], 1u << (i & 31));
            ++pos;
        }
    }
    if (out.scale_out && tid == 0) *out.scale_out = scale;
    if (out.mask) {
        __syncthreads();
        for (int w = tid; w < nwords; w += NT) out.mask[w] = smask[w];
    }
}
#undef KEY

template <int MODE>
__device__ __forceinline__ void block_topk_m(const float* __restrict__ x, int d, int k, float rms_eps, TopkOut out,
                                             TopkSrcArgs src, unsigned char* smem) {
    const int ept = topk_ept(d);
    if (ept <= 4) block_topk_t<4, MODE>(x, d, k, rms_eps, out, src, smem);
    else if (ept <= 8) block_topk_t<8, MODE>(x, d, k, rms_eps, out, src, smem);
    else if (ept <= 12) block_topk_t<12, MODE>(x, d, k, rms_eps, out, src, smem);
    else if (ept <= 16) block_topk_t<16, MODE>(x, d, k, rms_eps, out, src, smem);
    else if (ept <= 24) block_topk_t<24, MODE>(x, d, k, rms_eps, out, src, smem);
    else block_topk_t<32, MODE>(x, d, k, rms_eps, out, src, smem);
}

// One CTA per token: x [batch][ldx], outputs strided per token.
struct TopkKernelArgs {
    const float* x;
    int64_t ldx;
    int d, k;
    float rms_eps;
    float* xr_out;      // [batch][d] or null
    int32_t* idx;       // [batch][k]
    float* vals;        // [batch][k]
    uint32_t* mask;     // [batch][ceil(d/32)] or null
    float* scale;       // [batch] or null
    int mode;           // TopkSrc
    const float* resid; int64_t resid_ld;                 // SRC_RESID_ACC
    unsigned long long* acc; int64_t acc_ld;              // SRC_RESID_ACC / SRC_SILU_GU
    unsigned long long* zero; int64_t zero_ld; int zero_n; // optional extra zeroing per token
};

__global__ void __launch_bounds__(kTopkThreads, 1) topk_kernel(TopkKernelArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.x;
    const int nwords = (a.d + 31) / 32;
    TopkOut o;
    o.xr_out = a.xr_out ? a.xr_out + (size_t)b * a.d : nullptr;
    o.idx = a.idx + (size_t)b * a.k;
    o.vals = a.vals + (size_t)b * a.k;
    o.mask = a.mask ? a.mask + (size_t)b * nwords : nullptr;
    o.scale_out = a.scale ? a.scale + b : nullptr;
    TopkSrcArgs src;
    src.resid = a.resid ? a.resid + (size_t)b * a.resid_ld : nullptr;
    src.acc = a.acc ? a.acc + (size_t)b * a.acc_ld : nullptr;
    src.zero = a.zero ? a.zero + (size_t)b * a.zero_ld : nullptr;
    src.zero_n = a.zero_n;
    const float* x = a.x ? a.x + (size_t)b * a.ldx : nullptr;
    if (a.mode == SRC_RESID_ACC)
        block_topk_m<SRC_RESID_ACC>(x, a.d, a.k, a.rms_eps, o, src, smem);
    else if (a.mode == SRC_SILU_GU)
        block_topk_m<SRC_SILU_GU>(x, a.d, a.k, a.rms_eps, o, src, smem);
    else
        block_topk_m<SRC_PLAIN>(x, a.d, a.k, a.rms_eps, o, src, smem);
}

}  // namespace larosa
