// attention.cuh — one-token GQA decode attention over a bf16 KV cache, split along the
// context (flash-decoding style) with a deterministic last-CTA combine.  Plumbing of the
// decoder layer (not LaRoSA content; conventions SURVEY Z27): q-head h reads kv-head
// floor(h * Hkv / Hq), scale 1/sqrt(hd), fp32 softmax.
//
// grid = (batch * Hq, n_chunks), 4 warps.  CTA (b, h, c) handles positions [c*CH, c*CH + CH)
// (CH <= 64) of query head h (one head per CTA: GQA groups of G heads share the K/V rows
// through L2, and no CTA loops over a group's heads).  Warp w owns positions c*CH + w + 4*i:
// it issues ALL its K and V row loads up front (one 16-byte or 8-byte load per lane per row,
// so the rows' DRAM latencies overlap), computes scores (lanes over head dims, the positions'
// butterfly reductions interleaved), a warp-local softmax and P.V; the 4 warps then merge in
// shared memory.  The chunk's (m, l, o[hd]) goes to the workspace and the last chunk CTA of
// the head (atomic ticket) merges the chunks in order.
#pragma once
#include "common.cuh"
#include "gemv.cuh"

namespace larosa {

constexpr int kAttnThreads = 128;
constexpr int kAttnPosPerWarp = 16;          // CH <= 4 * 16
constexpr int kAttnMaxG = 8;

struct AttnArgs {
    unsigned long long* acc;         // [batch][acc_ld] QKV GEMV fixed-point accumulators (re-zeroed)
    int64_t acc_ld;
    const uint16_t* bias;  // [(hq + 2 hkv) hd] bf16 or null
    float theta;           // RoPE base
    float* q_out;          // optional tap: [batch][hq*hd] q after bias + RoPE
    uint16_t* kc;          // [batch][hkv][max_ctx][hd]; the new k/v row is written at pos
    uint16_t* vc;
    const int32_t* pos;    // [batch]; attend to [0, pos[b]]
    int64_t max_ctx;
    int hq, hkv, hd;
    int chunk, n_chunks;
    float* part;           // [batch*hq][n_chunks][hd + 2]
    unsigned* counters;    // [batch*hq] head tickets, + kAttnGroupCounterOff: [batch*hkv] group tickets
    float* out;            // [batch][hq*hd]
    SiteSel out_sel;       // batch 1: selection data of h2 for the next GEMV (hist null = none)
    uint32_t* zero_hist;   // optional histogram to re-zero (its consumer has completed)
    int zero_words;
    unsigned long long* tl;   // debug timeline slot or null
    int keep_acc;          // 1: leave the QKV accumulators to the next kernel to re-zero (batch-1 layer)
};

constexpr int kAttnGroupCounterOff = 2048;   // counters: [0, B Hq) head tickets, then group tickets
__host__ __device__ inline size_t attn_smem_bytes(int hd) {
    // q [hd] + per-warp (m, l) [4][2] + per-warp o [4][hd] + new k/v bf16 [2][hd] + flags
    return sizeof(float) * ((size_t)hd + 8 + 4 * (size_t)hd) + 4 * (size_t)hd + 16;
}

// RoPE (HF rotate_half) of the pair (i, i + hd/2) at position p, in fp64
// (inverse frequency and angle in fp64, reduced to [-pi, pi] in fp64, then fp32 sincos:
// accurate to a few fp32 ulp at any position, without the long fp64 sincos routine)
__device__ __forceinline__ void rope_pair(float& y1, float& y2, int i, int hd, int p, float theta) {
    const double inv_freq = exp(-(2.0 * i / hd) * log((double)theta));
    double ang = (double)p * inv_freq;
    ang = fma(-6.283185307179586476925, rint(ang * 0.15915494309189533577), ang);
    float sn, cn;
    sincosf((float)ang, &sn, &cn);
    const float r1 = fmaf(y1, cn, -y2 * sn);
    const float r2 = fmaf(y2, cn, y1 * sn);
    y1 = r1;
    y2 = r2;
}

template <int DPL>   // head dims per lane: hd = 32 * DPL (2 -> 64, 4 -> 128)
__device__ void attention_body(const AttnArgs& a, float* asmem) {
    const int G = a.hq / a.hkv;
    constexpr int hd = 32 * DPL;
    float* sq = asmem;                         // [hd]
    float* sml = sq + hd;                      // [4][2]
    float* so = sml + 8;                       // [4][hd]
    uint16_t* snew = reinterpret_cast<uint16_t*>(so + 4 * hd);   // [2][hd] new k, v (bf16)
    int* sflag = reinterpret_cast<int*>(snew + 2 * hd);

    // one CTA per (token b, query head h, context chunk): kv head g = floor(h / G)
    const int bh = blockIdx.x, ch = blockIdx.y;
    const int b = bh / a.hq, h = bh % a.hq, g = h / G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ctx = a.pos[b] + 1;
    const int start = ch * a.chunk;
    const int n = max(0, min(a.chunk, ctx - start));
    const size_t kvbase = ((size_t)b * a.hkv + g) * a.max_ctx * hd;

    const int half = hd / 2;
    const int nq = a.hq * hd, nk = a.hkv * hd;
    const int pnew = ctx - 1;                                   // the position appended this step
    const bool has_new = pnew >= start && pnew < start + n;
    // every K/V row of this warp's positions except the one appended this step: issued
    // BEFORE the dependency wait (earlier steps wrote them; with programmatic dependent launch
    // these loads overlap the QKV GEMV still streaming)
    uint32_t kr[kAttnPosPerWarp][DPL / 2], vr[kAttnPosPerWarp][DPL / 2];
#pragma unroll
    for (int i = 0; i < kAttnPosPerWarp; ++i) {
        const int p = warp + 4 * i;
#pragma unroll
        for (int t = 0; t < DPL / 2; ++t) kr[i][t] = vr[i][t] = 0u;
        if (p < n && start + p != pnew) {
            const size_t off = kvbase + (size_t)(start + p) * hd + lane * DPL;
            if constexpr (DPL == 4) {
                const uint2 kk = *reinterpret_cast<const uint2*>(a.kc + off);
                const uint2 vv = *reinterpret_cast<const uint2*>(a.vc + off);
                kr[i][0] = kk.x; kr[i][1] = kk.y; vr[i][0] = vv.x; vr[i][1] = vv.y;
            } else {
                kr[i][0] = *reinterpret_cast<const uint32_t*>(a.kc + off);
                vr[i][0] = *reinterpret_cast<const uint32_t*>(a.vc + off);
            }
        }
    }
    pdl_wait();
    pdl_trigger();
    tl_stamp(a.tl, 1);
    if (a.zero_hist) {
        const int nct = gridDim.x * gridDim.y, cta = blockIdx.y * gridDim.x + blockIdx.x;
        for (int i = cta * kAttnThreads + threadIdx.x; i < a.zero_words; i += nct * kAttnThreads) a.zero_hist[i] = 0u;
    }
    const unsigned long long* accb = a.acc + (size_t)b * a.acc_ld;
    auto yval = [&](int col) -> float {
        return fix_to_f(__ldcg(accb + col)) + (a.bias ? bf16f(a.bias[col]) : 0.f);
    };
    // q of head h (bias + RoPE) and, in the chunk holding pos, the new k / v row of kv head g
    // (every query head of the group computes it; the group's first head writes it to the cache)
    for (int i = tid; i < half; i += kAttnThreads) {
        const int col = h * hd + i;
        float y1 = yval(col), y2 = yval(col + half);
        rope_pair(y1, y2, i, hd, pnew, a.theta);
        sq[i] = y1;
        sq[i + half] = y2;
        if (a.q_out && ch == 0) {
            a.q_out[(size_t)b * nq + col] = y1;
            a.q_out[(size_t)b * nq + col + half] = y2;
        }
    }
    if (has_new) {
        const bool writer = h % G == 0;
        uint16_t* kdst = a.kc + kvbase + (size_t)pnew * hd;
        uint16_t* vdst = a.vc + kvbase + (size_t)pnew * hd;
        for (int i = tid; i < half; i += kAttnThreads) {
            float y1 = yval(nq + g * hd + i), y2 = yval(nq + g * hd + i + half);
            rope_pair(y1, y2, i, hd, pnew, a.theta);
            const uint16_t k1 = f2bf16_rne(y1), k2 = f2bf16_rne(y2);
            snew[i] = k1;
            snew[i + half] = k2;
            if (writer) {
                kdst[i] = k1;
                kdst[i + half] = k2;
            }
        }
        for (int i = tid; i < hd; i += kAttnThreads) {
            const uint16_t v = f2bf16_rne(yval(nq + nk + g * hd + i));
            snew[hd + i] = v;
            if (writer) vdst[i] = v;
        }
    }
    __syncthreads();
    tl_stamp(a.tl, 2);

    // the new row (computed above into shared memory) replaces the stale cache entry
#pragma unroll
    for (int i = 0; i < kAttnPosPerWarp; ++i) {
        const int p = warp + 4 * i;
        if (p < n && start + p == pnew) {
            const uint32_t* sk = reinterpret_cast<const uint32_t*>(snew + lane * DPL);
            const uint32_t* sv = reinterpret_cast<const uint32_t*>(snew + hd + lane * DPL);
#pragma unroll
            for (int t = 0; t < DPL / 2; ++t) {
                kr[i][t] = sk[t];
                vr[i][t] = sv[t];
            }
        }
    }

    const float scale = 1.0f / sqrtf((float)hd);
    {
        float qf[DPL];
#pragma unroll
        for (int t = 0; t < DPL; ++t) qf[t] = sq[lane * DPL + t];
        float s[kAttnPosPerWarp];
        float m = -INFINITY;
#pragma unroll
        for (int i = 0; i < kAttnPosPerWarp; ++i) {
            float acc = 0.f;
#pragma unroll
            for (int t = 0; t < DPL / 2; ++t) {
                acc = fmaf(qf[2 * t], bf16lo(kr[i][t]), acc);
                acc = fmaf(qf[2 * t + 1], bf16hi(kr[i][t]), acc);
            }
            s[i] = acc;
        }
        // the positions' butterflies interleaved (independent shuffles in flight together)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int i = 0; i < kAttnPosPerWarp; ++i) s[i] += __shfl_xor_sync(0xffffffffu, s[i], o);
#pragma unroll
        for (int i = 0; i < kAttnPosPerWarp; ++i) {
            s[i] = (warp + 4 * i < n) ? s[i] * scale : -INFINITY;
            m = fmaxf(m, s[i]);
        }
        float l = 0.f, o[DPL];
#pragma unroll
        for (int t = 0; t < DPL; ++t) o[t] = 0.f;
#pragma unroll
        for (int i = 0; i < kAttnPosPerWarp; ++i) {
            if (warp + 4 * i < n) {
                const float e = expf(s[i] - m);
                l += e;
#pragma unroll
                for (int t = 0; t < DPL / 2; ++t) {
                    o[2 * t] = fmaf(e, bf16lo(vr[i][t]), o[2 * t]);
                    o[2 * t + 1] = fmaf(e, bf16hi(vr[i][t]), o[2 * t + 1]);
                }
            }
        }
        if (lane == 0) {
            sml[warp * 2 + 0] = m;
            sml[warp * 2 + 1] = l;
        }
#pragma unroll
        for (int t = 0; t < DPL; ++t) so[warp * hd + lane * DPL + t] = o[t];
    }
    __syncthreads();
    tl_stamp(a.tl, 3);

    // merge the 4 warps (fixed order) -> this chunk's (m, l, o) in the workspace
    float* myp = a.part + ((size_t)bh * a.n_chunks + ch) * (hd + 2);
    for (int dd = tid; dd < hd; dd += kAttnThreads) {
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < 4; ++w) M = fmaxf(M, sml[w * 2]);
        float L = 0.f, Ov = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const float lw = sml[w * 2 + 1];
            if (lw == 0.f) continue;
            const float e = expf(sml[w * 2] - M);
            L = fmaf(lw, e, L);
            Ov = fmaf(so[w * hd + dd], e, Ov);
        }
        myp[2 + dd] = Ov;
        if (dd == 0) {
            myp[0] = M;
            myp[1] = L;
        }
    }
    fence_acq_rel_gpu();
    __syncthreads();
    if (tid == 0) {
        const unsigned prev = atomicAdd(&a.counters[bh], 1u);
        sflag[0] = prev == (unsigned)(a.n_chunks - 1);
    }
    __syncthreads();
    if (!sflag[0]) return;
    if (tid == 0) a.counters[bh] = 0u;
    fence_acq_rel_gpu();
    tl_stamp(a.tl, 5);

    // the last chunk CTA of head h merges the chunks in order (all records loaded up front)
    const float* pb = a.part + (size_t)bh * a.n_chunks * (hd + 2);
    for (int dd = tid; dd < hd; dd += kAttnThreads) {
        float M = -INFINITY, L = 0.f, Ov = 0.f;
        for (int c0 = 0; c0 < a.n_chunks; c0 += 16) {
            float mc[16], lc[16], oc[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const bool ok = c0 + u < a.n_chunks;
                const float* r = pb + (size_t)(c0 + u) * (hd + 2);
                mc[u] = ok ? __ldcg(r) : -INFINITY;
                lc[u] = ok ? __ldcg(r + 1) : 0.f;
                oc[u] = ok ? __ldcg(r + 2 + dd) : 0.f;
            }
            float Mn = M;
#pragma unroll
            for (int u = 0; u < 16; ++u) Mn = fmaxf(Mn, lc[u] == 0.f ? -INFINITY : mc[u]);
            if (Mn == -INFINITY) continue;
            const float rescale = M == -INFINITY ? 0.f : expf(M - Mn);
            L *= rescale;
            Ov *= rescale;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                if (lc[u] == 0.f) continue;
                const float w = expf(mc[u] - Mn);
                L = fmaf(lc[u], w, L);
                Ov = fmaf(oc[u], w, Ov);
            }
            M = Mn;
        }
        const float hv = Ov / L;
        a.out[(size_t)b * a.hq * hd + (size_t)h * hd + dd] = hv;
        if (a.out_sel.hist) hist_push(a.out_sel, hv, h * hd + dd);
    }
    tl_stamp(a.tl, 6);
    if (a.keep_acc) return;   // the O GEMV re-zeroes the QKV accumulators after this kernel
    // every chunk CTA of head h has read its q accumulators: re-zero them.  The group's k / v
    // accumulators are read by all G heads: the last head merger of the group re-zeroes them.
    unsigned long long* accz = a.acc + (size_t)b * a.acc_ld;
    for (int i = tid; i < hd; i += kAttnThreads) accz[(size_t)h * hd + i] = 0ull;
    fence_acq_rel_gpu();
    __syncthreads();
    unsigned* gcnt = a.counters + kAttnGroupCounterOff + (size_t)b * a.hkv + g;
    if (tid == 0) {
        const unsigned prev = atomicAdd(gcnt, 1u);
        sflag[1] = prev == (unsigned)(G - 1);
    }
    __syncthreads();
    if (!sflag[1]) return;
    if (tid == 0) *gcnt = 0u;
    for (int i = tid; i < hd; i += kAttnThreads) {
        accz[nq + (size_t)g * hd + i] = 0ull;
        accz[nq + nk + (size_t)g * hd + i] = 0ull;
    }
}

template <int DPL>
__global__ void __launch_bounds__(kAttnThreads) attention_kernel(const AttnArgs a) {
    extern __shared__ __align__(16) float asmem[];
    tl_stamp(a.tl, 0);
    attention_body<DPL>(a, asmem);   // waits on the QKV GEMV inside, after prefetching K/V
    tl_stamp(a.tl, 4);
}

}  // namespace larosa
