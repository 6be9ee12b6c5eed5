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

namespace larosa {

constexpr int kAttnThreads = 128;
constexpr int kAttnPosPerWarp = 16;          // CH <= 4 * 16
constexpr int kAttnMaxG = 8;

struct AttnArgs {
    const float* q;        // [batch][hq*hd]
    const uint16_t* kc;    // [batch][hkv][max_ctx][hd]
    const uint16_t* vc;
    const int32_t* pos;    // [batch]; attend to [0, pos[b]]
    int64_t max_ctx;
    int hq, hkv, hd;
    int chunk, n_chunks;
    float* part;           // [batch*hkv][n_chunks][G][hd + 2]
    unsigned* counters;    // [batch*hkv]
    float* out;            // [batch][hq*hd]
};

__host__ __device__ inline size_t attn_smem_bytes(int G, int hd, int chunk) {
    (void)chunk;
    // q [G][hd] + per-warp (m, l) [4][G][2] + per-warp o [4][G][hd] + flag
    return sizeof(float) * ((size_t)G * hd + 4 * (size_t)G * 2 + 4 * (size_t)G * hd) + 16;
}

template <int DPL>   // head dims per lane: hd = 32 * DPL (2 -> 64, 4 -> 128)
__device__ void attention_body(const AttnArgs& a, float* asmem) {
    const int G = a.hq / a.hkv;
    constexpr int hd = 32 * DPL;
    float* sq = asmem;                         // [G][hd]
    float* sml = sq + G * hd;                  // [4][G][2]
    float* so = sml + 4 * G * 2;               // [4][G][hd]
    int* sflag = reinterpret_cast<int*>(so + 4 * G * hd);

    const int bg = blockIdx.x, ch = blockIdx.y;
    const int b = bg / a.hkv, g = bg % a.hkv;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ctx = a.pos[b] + 1;
    const int start = ch * a.chunk;
    const int n = max(0, min(a.chunk, ctx - start));
    const size_t kvbase = ((size_t)b * a.hkv + g) * a.max_ctx * hd;

    // issue every K/V row load of this warp's positions before any math
    uint32_t kr[kAttnPosPerWarp][DPL / 2], vr[kAttnPosPerWarp][DPL / 2];
#pragma unroll
    for (int i = 0; i < kAttnPosPerWarp; ++i) {
        const int p = warp + 4 * i;
        if (p < n) {
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
    for (int i = tid; i < G * hd; i += kAttnThreads)
        sq[i] = a.q[(size_t)b * a.hq * hd + (size_t)g * G * hd + i];
    __syncthreads();

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

    // merge the 4 warps (fixed order) -> this chunk's (m, l, o)
    float* myp = a.part + ((size_t)bg * a.n_chunks + ch) * G * (hd + 2);
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
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned prev = atomicAdd(&a.counters[bg], 1u);
        sflag[0] = prev == (unsigned)(a.n_chunks - 1);
    }
    __syncthreads();
    if (!sflag[0]) return;
    if (tid == 0) a.counters[bg] = 0u;
    __threadfence();

    // merge the chunks in order
    const float* pb = a.part + (size_t)bg * a.n_chunks * G * (hd + 2);
    for (int i = tid; i < G * hd; i += kAttnThreads) {
        const int j = i / hd, dd = i % hd;
        float M = -INFINITY;
        for (int c = 0; c < a.n_chunks; ++c) M = fmaxf(M, __ldcg(pb + ((size_t)c * G + j) * (hd + 2)));
        float L = 0.f, Ov = 0.f;
        for (int c = 0; c < a.n_chunks; ++c) {
            const float* r = pb + ((size_t)c * G + j) * (hd + 2);
            const float l = __ldcg(r + 1);
            if (l == 0.f) continue;
            const float w = expf(__ldcg(r) - M);
            L = fmaf(l, w, L);
            Ov = fmaf(__ldcg(r + 2 + dd), w, Ov);
        }
        a.out[(size_t)b * a.hq * hd + (size_t)(g * G + j) * hd + dd] = Ov / L;
    }
}

__global__ void __launch_bounds__(kAttnThreads) attention_kernel(const AttnArgs a) {
    extern __shared__ __align__(16) float asmem[];
    pdl_wait();
    pdl_trigger();
    if (a.hd == 128)
        attention_body<4>(a, asmem);
    else
        attention_body<2>(a, asmem);
}

}  // namespace larosa
