// attention.cuh — one-token GQA decode attention over a bf16 KV cache, split along the
// context (flash-decoding style) with a deterministic last-CTA combine.  Plumbing of the
// decoder layer (not LaRoSA content; conventions SURVEY Z27): q-head h reads kv-head
// floor(h * Hkv / Hq), scale 1/sqrt(hd), fp32 softmax.
//
// grid = (batch * Hkv, n_chunks); CTA (b, g, c) handles positions [c*CH, c*CH + CH) of the
// G = Hq/Hkv query heads sharing kv-head g: scores (warp per position, lanes over head
// dims), chunk-local softmax, P.V (thread per head dim).  Its (m, l, o[hd]) per head goes
// to the workspace; the last chunk CTA to finish (atomic ticket) merges the chunks in
// order.
#pragma once
#include "common.cuh"

namespace larosa {

constexpr int kAttnThreads = 128;

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
    return sizeof(float) * ((size_t)G * hd + (size_t)G * chunk + 2 * (size_t)G) + 16;
}

__global__ void __launch_bounds__(kAttnThreads) attention_kernel(const AttnArgs a) {
    extern __shared__ __align__(16) float asmem[];
    const int G = a.hq / a.hkv;
    const int hd = a.hd;
    float* sq = asmem;                 // [G][hd]
    float* sc = sq + G * hd;           // [G][chunk]
    float* sm = sc + G * a.chunk;      // [G] max
    float* sl = sm + G;                // [G] sum
    int* sflag = reinterpret_cast<int*>(sl + G);

    const int bg = blockIdx.x, ch = blockIdx.y;
    const int b = bg / a.hkv, g = bg % a.hkv;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    pdl_wait();
    pdl_trigger();

    const int ctx = a.pos[b] + 1;
    const int start = ch * a.chunk;
    const int n = max(0, min(a.chunk, ctx - start));
    const size_t kvbase = ((size_t)b * a.hkv + g) * a.max_ctx * hd;
    const float scale = 1.0f / sqrtf((float)hd);

    for (int i = tid; i < G * hd; i += kAttnThreads) {
        const int j = i / hd, dd = i % hd;
        sq[i] = a.q[(size_t)b * a.hq * hd + (size_t)(g * G + j) * hd + dd];
    }
    __syncthreads();

    // scores: one warp per position, lanes over dims (hd/32 contiguous dims per lane)
    const int dpl = hd / 32;
    for (int p = warp; p < n; p += kAttnThreads / 32) {
        const uint16_t* kp = a.kc + kvbase + (size_t)(start + p) * hd + lane * dpl;
        float kf[4];
        if (dpl == 4) {
            const uint2 w = *reinterpret_cast<const uint2*>(kp);
            kf[0] = bf16lo(w.x); kf[1] = bf16hi(w.x); kf[2] = bf16lo(w.y); kf[3] = bf16hi(w.y);
        } else {
            for (int t = 0; t < dpl; ++t) kf[t] = bf16f(kp[t]);
        }
        for (int j = 0; j < G; ++j) {
            float s = 0.f;
            for (int t = 0; t < dpl; ++t) s = fmaf(sq[j * hd + lane * dpl + t], kf[t], s);
            s = warp_sum(s);
            if (lane == 0) sc[j * a.chunk + p] = s * scale;
        }
    }
    __syncthreads();

    // chunk-local softmax statistics, one warp per head
    for (int j = warp; j < G; j += kAttnThreads / 32) {
        float m = -INFINITY;
        for (int p = lane; p < n; p += 32) m = fmaxf(m, sc[j * a.chunk + p]);
        m = warp_max(m);
        float l = 0.f;
        for (int p = lane; p < n; p += 32) {
            const float e = (n > 0) ? expf(sc[j * a.chunk + p] - m) : 0.f;
            sc[j * a.chunk + p] = e;
            l += e;
        }
        l = warp_sum(l);
        if (lane == 0) {
            sm[j] = m;
            sl[j] = l;
        }
    }
    __syncthreads();

    // P.V: thread per head dim
    float* myp = a.part + ((size_t)bg * a.n_chunks + ch) * G * (hd + 2);
    for (int dd = tid; dd < hd; dd += kAttnThreads) {
        float o[8];
        for (int j = 0; j < G; ++j) o[j] = 0.f;
        for (int p = 0; p < n; ++p) {
            const float v = bf16f(a.vc[kvbase + (size_t)(start + p) * hd + dd]);
            for (int j = 0; j < G; ++j) o[j] = fmaf(sc[j * a.chunk + p], v, o[j]);
        }
        for (int j = 0; j < G; ++j) myp[j * (hd + 2) + 2 + dd] = o[j];
    }
    if (tid < G) {
        myp[tid * (hd + 2) + 0] = sm[tid];
        myp[tid * (hd + 2) + 1] = sl[tid];
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
        float L = 0.f, O = 0.f;
        for (int c = 0; c < a.n_chunks; ++c) {
            const float* r = pb + ((size_t)c * G + j) * (hd + 2);
            const float l = __ldcg(r + 1);
            if (l == 0.f) continue;
            const float w = expf(__ldcg(r) - M);
            L = fmaf(l, w, L);
            O = fmaf(__ldcg(r + 2 + dd), w, O);
        }
        a.out[(size_t)b * a.hq * hd + (size_t)(g * G + j) * hd + dd] = O / L;
    }
}

}  // namespace larosa
