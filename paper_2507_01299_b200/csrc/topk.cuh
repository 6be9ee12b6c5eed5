// topk.cuh — exact per-token Top-K (S_k of eq. 2) as a block-wide radix
// select on the uint32 keys bits(|x|), with the lower-index tie-break, plus the
// RMS scale of the h1/h3 sites and stable compaction to ascending indices.
//
// One CTA per token.  Keys live in shared memory (padded one word per 32 to keep the
// contiguous-ownership compaction bank-conflict-light); the histogram passes use strided
// ownership.  Digits: bits [30:19] (4096 bins), [18:7] (4096), [6:0] (128).  A pass that
// finds the k-th key's bucket fully inside the selection stops early (typical for
// continuous data after 2 passes); an exact tie across the k-th key is resolved by index.
#pragma once
#include "common.cuh"

namespace larosa {

constexpr int kTopkThreads = 1024;
constexpr int kTopkBins = 4096;

__host__ __device__ constexpr int topk_pad(int i) { return i + (i >> 5); }

// dynamic smem bytes for a vector of length d
__host__ __device__ constexpr size_t topk_smem_bytes(int d) {
    return sizeof(uint32_t) * (size_t)(topk_pad(d) + 1)            // keys
           + sizeof(int) * kTopkBins                                // histogram
           + sizeof(uint32_t) * (size_t)((d + 31) / 32)             // mask words
           + sizeof(int) * 64;                                      // scan / broadcast scratch
}

struct TopkOut {
    float* xr_out;     // [d] copy of the (rotated) input, or nullptr
    int32_t* idx;      // [k]
    float* vals;       // [k]
    uint32_t* mask;    // [ceil(d/32)] or nullptr
    float* scale_out;  // [1] the RMS scale s (1 when rms_eps < 0), or nullptr
};

// Top-K of x[0..d) (global memory, fp32).  Must be called by all kTopkThreads threads.
__device__ void block_topk(const float* __restrict__ x, int d, int k, float rms_eps, TopkOut out,
                           unsigned char* smem_raw) {
    constexpr int NT = kTopkThreads;
    uint32_t* keys = reinterpret_cast<uint32_t*>(smem_raw);
    int* hist = reinterpret_cast<int*>(keys + topk_pad(d) + 1);
    const int nwords = (d + 31) / 32;
    uint32_t* smask = reinterpret_cast<uint32_t*>(hist + kTopkBins);
    int* scr = reinterpret_cast<int*>(smask + nwords);   // 64 ints
    float* fscr = reinterpret_cast<float*>(scr);
    const int tid = threadIdx.x;

    // 1. keys = bits(|x|) (clears the sign, so -0 == +0), sum of squares for the RMS scale
    float ssq = 0.f;
    for (int i = tid; i < d; i += NT) {
        float v = __ldg(x + i);
        keys[topk_pad(i)] = __float_as_uint(v) & 0x7fffffffu;
        ssq = fmaf(v, v, ssq);
        if (out.xr_out) out.xr_out[i] = v;
    }
    for (int w = tid; w < nwords; w += NT) smask[w] = 0u;
    float scale = 1.f;
    if (rms_eps >= 0.f) {
        float tot = block_sum<NT>(ssq, fscr);          // fixed-order, deterministic
        scale = 1.0f / sqrtf(tot / (float)d + rms_eps);
    }
    __syncthreads();

    // 2. radix select of the k-th largest key.  Selection rule afterwards:
    //    key > thr, or key == thr and (tie_mode ? among the first `rem` such indices : true)
    uint32_t prefix = 0u, pmask = 0u;
    int rem = k;              // how many still to take inside the current bucket prefix
    bool exact_ge = false;    // early exit: select key >= prefix (lower bits free)
    bool tie_mode = false;
    if (k <= 0 || k >= d) {
        exact_ge = true;
        prefix = (k >= d) ? 0u : 0xffffffffu;   // k == 0 selects nothing (keys < 2^31)
    } else {
        const int shifts[3] = {19, 7, 0};
        const int nbits[3] = {12, 12, 7};
        for (int pass = 0; pass < 3; ++pass) {
            const int sh = shifts[pass];
            const int nb = 1 << nbits[pass];
            const uint32_t dmask = (uint32_t)(nb - 1);
            for (int b = tid; b < nb; b += NT) hist[b] = 0;
            __syncthreads();
            for (int i = tid; i < d; i += NT) {
                uint32_t key = keys[topk_pad(i)];
                if ((key & pmask) == prefix) atomicAdd(&hist[(key >> sh) & dmask], 1);
            }
            __syncthreads();
            // suffix scan: thread t owns bins [nb - (t+1)*bpt, nb - t*bpt) (top bins first)
            const int bpt = (nb + NT - 1) / NT;
            const int hiB = nb - tid * bpt;
            const int loB = max(0, hiB - bpt);
            int c = 0;
            for (int b = hiB - 1; b >= loB; --b) c += hist[b];
            int tot;
            int before = block_excl_scan<NT>(c, scr, &tot);
            if (before < rem && rem <= before + c) {
                int acc = before;
                for (int b = hiB - 1; b >= loB; --b) {
                    int h = hist[b];
                    if (acc + h >= rem) {
                        scr[40] = b;
                        scr[41] = rem - acc;
                        scr[42] = h;
                        break;
                    }
                    acc += h;
                }
            }
            __syncthreads();
            const int bstar = scr[40];
            rem = scr[41];
            const int cnt = scr[42];
            prefix |= (uint32_t)bstar << sh;
            pmask |= dmask << sh;
            __syncthreads();    // scr reused by the next scan
            if (cnt == rem) {   // whole bucket selected: key >= prefix
                exact_ge = true;
                break;
            }
            if (pass == 2) tie_mode = true;   // exact key tie straddles position k
        }
    }
    const uint32_t thr = prefix;

    // 3. stable compaction, contiguous ownership: thread t owns [t*E, min(d, (t+1)*E))
    const int E = (d + NT - 1) / NT;
    const int i0 = min(d, tid * E), i1 = min(d, i0 + E);
    int n_gt = 0, n_eq = 0;
    for (int i = i0; i < i1; ++i) {
        uint32_t key = keys[topk_pad(i)];
        if (exact_ge) {
            n_gt += (key >= thr);
        } else {
            n_gt += (key > thr);
            n_eq += (key == thr);
        }
    }
    int take_eq = 0;
    if (tie_mode) {
        int tot;
        int eq_before = block_excl_scan<NT>(n_eq, scr, &tot);
        take_eq = min(n_eq, max(0, rem - eq_before));
        __syncthreads();
    }
    int tot_sel;
    int pos = block_excl_scan<NT>(n_gt + take_eq, scr, &tot_sel);
    int eq_seen = 0;
    for (int i = i0; i < i1; ++i) {
        uint32_t key = keys[topk_pad(i)];
        bool sel;
        if (exact_ge) {
            sel = key >= thr;
        } else if (key > thr) {
            sel = true;
        } else if (key == thr) {
            sel = eq_seen < take_eq;
            ++eq_seen;
        } else {
            sel = false;
        }
        if (sel) {
            out.idx[pos] = i;
            out.vals[pos] = __ldg(x + i) * scale;
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
};

__global__ void __launch_bounds__(kTopkThreads, 1) topk_kernel(TopkKernelArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    pdl_wait();
    const int b = blockIdx.x;
    const int nwords = (a.d + 31) / 32;
    TopkOut o;
    o.xr_out = a.xr_out ? a.xr_out + (size_t)b * a.d : nullptr;
    o.idx = a.idx + (size_t)b * a.k;
    o.vals = a.vals + (size_t)b * a.k;
    o.mask = a.mask ? a.mask + (size_t)b * nwords : nullptr;
    o.scale_out = a.scale ? a.scale + b : nullptr;
    block_topk(a.x + (size_t)b * a.ldx, a.d, a.k, a.rms_eps, o, smem);
    pdl_trigger();
}

}  // namespace larosa
