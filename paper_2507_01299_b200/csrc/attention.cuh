// attention.cuh — one-token GQA decode attention over a bf16 KV cache, split along the
// context (flash-decoding style) with a deterministic last-CTA combine.  Plumbing of the
// decoder layer (not LaRoSA content; conventions SURVEY Z27): q-head h reads kv-head
// floor(h * Hkv / Hq), scale 1/sqrt(hd), fp32 softmax.
//
// grid = (batch * Hkv, n_chunks), 4 warps.  CTA (b, g, c) handles positions
// [c*CH, c*CH + CH) (CH <= 64) of the G = Hq/Hkv query heads that share kv-head g.  Warp w
// owns positions c*CH + w + 4*i: it issues ALL its K and V row loads up front (one 16-byte
// or 8-byte load per lane per row, so the rows' DRAM latencies overlap), computes scores
// (lanes over head dims + warp reduction), a warp-local softmax and P.V; the 4 warps then
// merge in shared memory.  The chunk's (m, l, o[hd]) per head goes to the workspace and
// the last chunk CTA to finish (atomic ticket) merges the chunks in order.
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
    float* part;           // [batch*hkv][n_chunks][G][hd + 2]
    unsigned* counters;    // [batch*hkv]
    float* out;            // [batch][hq*hd]
    SiteSel out_sel;       // batch 1: selection data of h2 for the next GEMV (hist null = none)
    uint32_t* zero_hist;   // optional histogram to re-zero (its consumer has completed)
    int zero_words;
    unsigned long long* tl;   // debug timeline slot or null
    int cluster;           // 1: the n_chunks CTAs of a kv group form a cluster; merge via DSMEM
};

__host__ __device__ inline size_t attn_smem_bytes(int G, int hd, int chunk) {
    (void)chunk;
    // q [G][hd] + per-warp (m, l) [4][G][2] + per-warp o [4][G][hd] + new k/v bf16 [2][hd] + flag
    // + this chunk's merged partial [G][hd + 2] (read by the cluster leader through DSMEM)
    return sizeof(float) * ((size_t)G * hd + 4 * (size_t)G * 2 + 4 * (size_t)G * hd + (size_t)G * (hd + 2)) +
           4 * (size_t)hd + 16;
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
    float* sq = asmem;                         // [G][hd]
    float* sml = sq + G * hd;                  // [4][G][2]
    float* so = sml + 4 * G * 2;               // [4][G][hd]
    int* sflag = reinterpret_cast<int*>(so + 4 * G * hd + hd);   // after the new k/v bf16 rows

    const int bg = blockIdx.x, ch = blockIdx.y;
    const int b = bg / a.hkv, g = bg % a.hkv;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ctx = a.pos[b] + 1;
    const int start = ch * a.chunk;
    const int n = max(0, min(a.chunk, ctx - start));
    const size_t kvbase = ((size_t)b * a.hkv + g) * a.max_ctx * hd;

    const int half = hd / 2;
    const int nq = a.hq * hd, nk = a.hkv * hd;
    const int pnew = ctx - 1;                                   // the position appended this step
    const bool has_new = pnew >= start && pnew < start + n;
    uint16_t* snew = reinterpret_cast<uint16_t*>(so + 4 * G * hd);   // [2][hd] new k, v (bf16)
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
        return fix_to_f(accb[col]) + (a.bias ? bf16f(a.bias[col]) : 0.f);
    };
    // q of my G heads (bias + RoPE), and, in the chunk holding pos, the new k / v row
    for (int t = tid; t < G * half; t += kAttnThreads) {
        const int j = t / half, i = t % half;
        const int col = (g * G + j) * hd + i;
        float y1 = yval(col), y2 = yval(col + half);
        rope_pair(y1, y2, i, hd, pnew, a.theta);
        sq[j * hd + i] = y1;
        sq[j * hd + i + half] = y2;
        if (a.q_out && ch == 0) {
            a.q_out[(size_t)b * nq + col] = y1;
            a.q_out[(size_t)b * nq + col + half] = y2;
        }
    }
    if (has_new) {
        uint16_t* kdst = a.kc + kvbase + (size_t)pnew * hd;
        uint16_t* vdst = a.vc + kvbase + (size_t)pnew * hd;
        for (int i = tid; i < half; i += kAttnThreads) {
            float y1 = yval(nq + g * hd + i), y2 = yval(nq + g * hd + i + half);
            rope_pair(y1, y2, i, hd, pnew, a.theta);
            const uint16_t k1 = f2bf16_rne(y1), k2 = f2bf16_rne(y2);
            snew[i] = k1;
            snew[i + half] = k2;
            kdst[i] = k1;
            kdst[i + half] = k2;
        }
        for (int i = tid; i < hd; i += kAttnThreads) {
            const uint16_t v = f2bf16_rne(yval(nq + nk + g * hd + i));
            snew[hd + i] = v;
            vdst[i] = v;
        }
    }
    __syncthreads();

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
    for (int j = 0; j < G; ++j) {
        float qf[DPL];
#pragma unroll
        for (int t = 0; t < DPL; ++t) qf[t] = sq[j * hd + lane * DPL + t];
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
            acc = warp_sum(acc) * scale;
            s[i] = (warp + 4 * i < n) ? acc : -INFINITY;
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
            sml[(warp * G + j) * 2 + 0] = m;
            sml[(warp * G + j) * 2 + 1] = l;
        }
#pragma unroll
        for (int t = 0; t < DPL; ++t) so[(warp * G + j) * hd + lane * DPL + t] = o[t];
    }
    __syncthreads();

    // merge the 4 warps (fixed order) -> this chunk's (m, l, o): in shared memory for the
    // cluster leader, else in the global workspace for the last-arriving chunk CTA
    float* spart = reinterpret_cast<float*>(sflag + 4);
    float* myp = a.cluster ? spart : a.part + ((size_t)bg * a.n_chunks + ch) * G * (hd + 2);
    for (int i = tid; i < G * hd; i += kAttnThreads) {
        const int j = i / hd, dd = i % hd;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < 4; ++w) M = fmaxf(M, sml[(w * G + j) * 2]);
        float L = 0.f, Ov = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const float lw = sml[(w * G + j) * 2 + 1];
            if (lw == 0.f) continue;
            const float e = expf(sml[(w * G + j) * 2] - M);
            L = fmaf(lw, e, L);
            Ov = fmaf(so[(w * G + j) * hd + dd], e, Ov);
        }
        myp[j * (hd + 2) + 2 + dd] = Ov;
        if (dd == 0) {
            myp[j * (hd + 2) + 0] = M;
            myp[j * (hd + 2) + 1] = L;
        }
    }
    if (a.cluster) {
        cluster_sync_all();                       // every chunk's partial is in its shared memory
        if (cluster_ctarank() != 0) {
            cluster_sync_all();                   // keep it alive until the leader has read it
            return;
        }
    } else {
        fence_acq_rel_gpu();
        __syncthreads();
        if (tid == 0) {
            const unsigned prev = atomicAdd(&a.counters[bg], 1u);
            sflag[0] = prev == (unsigned)(a.n_chunks - 1);
        }
        __syncthreads();
        if (!sflag[0]) return;
        if (tid == 0) a.counters[bg] = 0u;
        fence_acq_rel_gpu();
    }

    // merge the chunks in order (each batch of chunk records is loaded before it is used:
    // __ldcg is a volatile load, so a load->use loop would serialise the L2 round trips)
    const float* pb = a.part + (size_t)bg * a.n_chunks * G * (hd + 2);
    for (int i = tid; i < G * hd; i += kAttnThreads) {
        const int j = i / hd, dd = i % hd;
        float M = -INFINITY, L = 0.f, Ov = 0.f;
        for (int c0 = 0; c0 < a.n_chunks; c0 += 16) {
            float mc[16], lc[16], oc[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const bool ok = c0 + u < a.n_chunks;
                if (a.cluster) {   // chunk c0 + u = cluster CTA rank c0 + u (c0 == 0, n_chunks <= 8)
                    const uint32_t r = dsmem_addr(spart + (size_t)j * (hd + 2), ok ? (uint32_t)(c0 + u) : 0u);
                    mc[u] = ok ? dsmem_ld_f32(r) : -INFINITY;
                    lc[u] = ok ? dsmem_ld_f32(r + 4) : 0.f;
                    oc[u] = ok ? dsmem_ld_f32(r + 4 * (2 + dd)) : 0.f;
                } else {
                    const float* r = pb + ((size_t)(c0 + u) * G + j) * (hd + 2);
                    mc[u] = ok ? __ldcg(r) : -INFINITY;
                    lc[u] = ok ? __ldcg(r + 1) : 0.f;
                    oc[u] = ok ? __ldcg(r + 2 + dd) : 0.f;
                }
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
        a.out[(size_t)b * a.hq * hd + (size_t)(g * G + j) * hd + dd] = hv;
        if (a.out_sel.hist) hist_push(a.out_sel, hv, (g * G + j) * hd + dd);
    }
    if (a.cluster) cluster_sync_all();             // the other chunks' shared memory may go
    // every chunk CTA of this kv group has read its q / new k, v accumulators: re-zero them
    unsigned long long* accz = a.acc + (size_t)b * a.acc_ld;
    for (int i = tid; i < G * hd; i += kAttnThreads) accz[(size_t)g * G * hd + i] = 0ull;
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
