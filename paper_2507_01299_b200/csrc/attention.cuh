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
    PeerOut peer;          // sharded phase 0: push h2 to every rank (n = 0: off)
};

constexpr int kAttnGroupCounterOff = 2048;   // counters: [0, B Hq) head tickets, then group tickets
__host__ __device__ inline size_t attn_smem_bytes(int hd) {
    // q [hd] + per-warp (m, l) [4][2] + per-warp o [4][hd] + new k/v bf16 [2][hd] + flags
    // + the chunk result (m, l, o[hd]) for a cluster merge
    return sizeof(float) * ((size_t)hd + 8 + 4 * (size_t)hd) + 4 * (size_t)hd + 16 + sizeof(float) * ((size_t)hd + 2);
}

// RoPE (HF rotate_half): cos / sin of the pair (i, i + hd/2) at position p -- the
// inverse frequency and the angle in fp64, reduced to [-pi, pi], then fp32 sincos (as rope_pair)
__device__ __forceinline__ float2 rope_cs(int i, int hd, int p, float theta) {
    const double inv_freq = exp(-(2.0 * i / hd) * log((double)theta));
    double ang = (double)p * inv_freq;
    ang = fma(-6.283185307179586476925, rint(ang * 0.15915494309189533577), ang);
    float sn, cn;
    sincosf((float)ang, &sn, &cn);
    return make_float2(cn, sn);
}
__device__ __forceinline__ void rope_apply(float& y1, float& y2, float2 cs) {
    const float r1 = fmaf(y1, cs.x, -y2 * cs.y);
    const float r2 = fmaf(y2, cs.x, y1 * cs.y);
    y1 = r1;
    y2 = r2;
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

// CL: the n_chunks CTAs of a head form one thread-block cluster (n_chunks <= 8): the chunk
// results are merged by cluster rank 0 through distributed shared memory (two cluster barriers)
// instead of the workspace partials, the head ticket and the last-CTA merge (three dependent
// global round trips).
template <int DPL, bool CL>   // head dims per lane: hd = 32 * DPL (2 -> 64, 4 -> 128)
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

    // merge the 4 warps (fixed order) -> this chunk's (m, l, o): in the workspace, or (CL) in
    // this CTA's shared memory for cluster rank 0
    float* sres = reinterpret_cast<float*>(sflag + 4);   // CL: [hd + 2]
    float* myp = CL ? sres : a.part + ((size_t)bh * a.n_chunks + ch) * (hd + 2);
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
    if constexpr (CL) {
        cluster_sync_all();                 // every chunk's (m, l, o) is in its CTA's shared memory
        tl_stamp(a.tl, 5);
        if (cluster_ctarank() == 0) {
            for (int dd = tid; dd < hd; dd += kAttnThreads) {
                float M = -INFINITY, L = 0.f, Ov = 0.f;
                for (int c = 0; c < a.n_chunks; ++c) {      // fixed (rank) order
                    const uint32_t base = dsmem_addr(sres, (uint32_t)c);
                    const float lc = dsmem_ld_f32(base + 4);
                    if (lc == 0.f) continue;
                    const float mc = dsmem_ld_f32(base), oc = dsmem_ld_f32(base + 4 * (2 + dd));
                    const float Mn = fmaxf(M, mc);
                    const float r0 = M == -INFINITY ? 0.f : expf(M - Mn), r1 = expf(mc - Mn);
                    L = fmaf(lc, r1, L * r0);
                    Ov = fmaf(oc, r1, Ov * r0);
                    M = Mn;
                }
                const float hv = Ov / L;
                a.out[(size_t)b * a.hq * hd + (size_t)h * hd + dd] = hv;
                if (a.peer.n) peer_put(a.peer, b, h * hd + dd, hv);
                if (a.out_sel.hist) hist_push(a.out_sel, hv, h * hd + dd);
            }
        }
        cluster_sync_all();                 // rank 0 has read every CTA's shared memory
        if (cluster_ctarank() != 0) return;
        peer_signal(a.peer, (unsigned)hd);
        tl_stamp(a.tl, 6);
    } else {
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
        if (a.peer.n) peer_put(a.peer, b, h * hd + dd, hv);
        if (a.out_sel.hist) hist_push(a.out_sel, hv, h * hd + dd);
    }
    peer_signal(a.peer, (unsigned)hd);
    tl_stamp(a.tl, 6);
    }
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

// ------------------------------------------------------------------------------------------
// Single-pass variant for contexts up to kAgPos * kAgWarps = 256 positions (the decode bench's
// ctx 256): one CTA per (token b, kv head g, subset of hpc of the group's G query heads), 16 warps.
// Warp w owns positions 16 w .. 16 w + 15 and loads their K and V rows into registers BEFORE the
// dependency wait (earlier steps wrote them); after it the CTA finalises q (bias + RoPE) for its
// hpc heads and the new k / v row from the QKV accumulators, then, head by head, each warp scores
// its 16 positions (lanes over head dims, butterflies interleaved), takes a warp-local softmax
// and P.V into shared memory; the 16 warps' (m, l, o) are merged in fixed order and the CTA
// writes h2 (and pushes its selection data at batch 1) itself: no chunk partials, no tickets, no
// second merge pass -- the split-KV kernel above needs both (3 dependent global round trips).
// hpc = 1 (one CTA per query head) when the batch has few heads, else hpc = G (the group's K/V
// rows are loaded once for all G heads).
constexpr int kAgWarps = 16;
constexpr int kAgThreads = kAgWarps * 32;
constexpr int kAgPos = 16;                          // positions per warp
constexpr int kAgMaxCtx = kAgWarps * kAgPos;        // 256
__host__ __device__ inline size_t attn_group_smem_bytes(int hd, int hpc) {
    // V rows bf16 [256][hd] + q [hpc][hd] + (m, l) [16][hpc][2] + o [16][hpc][hd] (fp32) + new k/v
    // bf16 [2][hd] + flags + the RoPE (cos, sin) table [hd/2]
    return 2 * (size_t)kAgMaxCtx * hd +
           sizeof(float) * ((size_t)hpc * hd + 32 * (size_t)hpc + 16 * (size_t)hpc * hd) + 4 * (size_t)hd + 16 +
           sizeof(float2) * (size_t)hd / 2;
}

template <int DPL>
__global__ void __launch_bounds__(kAgThreads, 1) attn_group_kernel(const AttnArgs a, int hpc) {
    extern __shared__ __align__(16) float agsm[];
    tl_stamp(a.tl, 0);
    constexpr int hd = 32 * DPL;
    const int G = a.hq / a.hkv, nsub = G / hpc;
    uint16_t* sv = reinterpret_cast<uint16_t*>(agsm);                   // [256][hd] V rows
    float* sq = agsm + kAgMaxCtx * hd / 2;         // [hpc][hd]
    float* sml = sq + hpc * hd;                    // [16][hpc][2]
    float* so = sml + 32 * hpc;                    // [16][hpc][hd]
    uint16_t* snew = reinterpret_cast<uint16_t*>(so + 16 * hpc * hd);   // [2][hd]
    int* sflag = reinterpret_cast<int*>(snew + 2 * hd);
    float2* scs = reinterpret_cast<float2*>(sflag + 4);                  // [hd/2] RoPE (cos, sin)
    const int u = blockIdx.x;
    const int b = u / (a.hkv * nsub), g = (u / nsub) % a.hkv, hs = u % nsub;
    const int h0 = g * G + hs * hpc;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ctx = a.pos[b] + 1;
    const int pnew = ctx - 1;
    const size_t kvbase = ((size_t)b * a.hkv + g) * a.max_ctx * hd;
    const int half = hd / 2;
    const int nq = a.hq * hd, nk = a.hkv * hd;
    // K rows in registers (lanes over head dims), V rows into shared memory by cp.async (16 bytes
    // per lane: hd * 2 / 16 lanes per row)
    uint32_t kr[kAgPos][DPL / 2];
#pragma unroll
    for (int i = 0; i < kAgPos; ++i) {
        const int p = warp * kAgPos + i;
#pragma unroll
        for (int t = 0; t < DPL / 2; ++t) kr[i][t] = 0u;
        if (p < ctx && p != pnew) {
            const size_t off = kvbase + (size_t)p * hd + lane * DPL;
            if constexpr (DPL == 4) {
                const uint2 kk = *reinterpret_cast<const uint2*>(a.kc + off);
                kr[i][0] = kk.x; kr[i][1] = kk.y;
            } else {
                kr[i][0] = *reinterpret_cast<const uint32_t*>(a.kc + off);
            }
        }
    }
    {
        constexpr int lpr = hd * 2 / 16;               // lanes per V row (16 bytes each)
        constexpr int rpi = 32 / lpr;                  // rows per warp instruction
        const int sub = lane / lpr, part = lane % lpr;
#pragma unroll
        for (int i = 0; i < kAgPos; i += rpi) {
            const int p = warp * kAgPos + i + sub;
            cp_async16(sv + (size_t)p * hd + part * 8, a.vc + kvbase + (size_t)p * hd + part * 8, p < ctx && p != pnew);
        }
        cp_async_commit();
    }
    // the rotation angles depend on the position only (not on the previous kernel)
    for (int i = tid; i < half; i += kAgThreads) scs[i] = rope_cs(i, hd, pnew, a.theta);
    pdl_wait();
    pdl_trigger();
    tl_stamp(a.tl, 1);
    __syncthreads();
    if (a.zero_hist) {
        const int nct = gridDim.x;
        for (int i = blockIdx.x * kAgThreads + tid; i < a.zero_words; i += nct * kAgThreads) a.zero_hist[i] = 0u;
    }
    const unsigned long long* accb = a.acc + (size_t)b * a.acc_ld;
    auto yval = [&](int col) -> float {
        return fix_to_f(__ldcg(accb + col)) + (a.bias ? bf16f(a.bias[col]) : 0.f);
    };
    for (int i = tid; i < hpc * half; i += kAgThreads) {          // q of the CTA's heads
        const int hh = i / half, j = i % half;
        const int col = (h0 + hh) * hd + j;
        float y1 = yval(col), y2 = yval(col + half);
        rope_apply(y1, y2, scs[j]);
        sq[hh * hd + j] = y1;
        sq[hh * hd + j + half] = y2;
        if (a.q_out) {
            a.q_out[(size_t)b * nq + col] = y1;
            a.q_out[(size_t)b * nq + col + half] = y2;
        }
    }
    {   // the new k / v row of kv head g (every CTA of the group computes it; subset 0 writes it)
        const bool writer = hs == 0;
        uint16_t* kdst = a.kc + kvbase + (size_t)pnew * hd;
        uint16_t* vdst = a.vc + kvbase + (size_t)pnew * hd;
        for (int i = tid; i < half; i += kAgThreads) {
            float y1 = yval(nq + g * hd + i), y2 = yval(nq + g * hd + i + half);
            rope_apply(y1, y2, scs[i]);
            const uint16_t k1 = f2bf16_rne(y1), k2 = f2bf16_rne(y2);
            snew[i] = k1;
            snew[i + half] = k2;
            if (writer) {
                kdst[i] = k1;
                kdst[i + half] = k2;
            }
        }
        for (int i = tid; i < hd; i += kAgThreads) {
            const uint16_t v = f2bf16_rne(yval(nq + nk + g * hd + i));
            snew[hd + i] = v;
            sv[(size_t)pnew * hd + i] = v;
            if (writer) vdst[i] = v;
        }
    }
    cp_async_wait<0>();
    __syncthreads();
    tl_stamp(a.tl, 2);
#pragma unroll
    for (int i = 0; i < kAgPos; ++i) {
        if (warp * kAgPos + i == pnew) {
            const uint32_t* sk = reinterpret_cast<const uint32_t*>(snew + lane * DPL);
#pragma unroll
            for (int t = 0; t < DPL / 2; ++t) kr[i][t] = sk[t];
        }
    }
    const float scale = 1.0f / sqrtf((float)hd);
    for (int hh = 0; hh < hpc; ++hh) {
        float qf[DPL];
#pragma unroll
        for (int t = 0; t < DPL; ++t) qf[t] = sq[hh * hd + lane * DPL + t];
        float s[kAgPos];
#pragma unroll
        for (int i = 0; i < kAgPos; ++i) {
            float acc = 0.f;
#pragma unroll
            for (int t = 0; t < DPL / 2; ++t) {
                acc = fmaf(qf[2 * t], bf16lo(kr[i][t]), acc);
                acc = fmaf(qf[2 * t + 1], bf16hi(kr[i][t]), acc);
            }
            s[i] = acc;
        }
        // transpose-reduce of the 16 partial dot products: at each butterfly level a lane keeps the
        // half of its values its partner does not, so 8 + 4 + 2 + 1 + 1 shuffles (not 5 x 16) leave
        // the full score of position pl = (lane >> 1) & 15 in lanes 2 pl and 2 pl + 1
        static_assert(kAgPos == 16, "transpose-reduce of 16 positions");
#pragma unroll
        for (int lvl = 0; lvl < 4; ++lvl) {
            const int ob = 16 >> lvl, nh = 8 >> lvl;
            const bool up = (lane & ob) != 0;
#pragma unroll
            for (int i = 0; i < nh; ++i) {
                const float send = up ? s[i] : s[i + nh];
                const float keep = up ? s[i + nh] : s[i];
                s[i] = keep + __shfl_xor_sync(0xffffffffu, send, ob);
            }
        }
        const int pl = (lane >> 1) & 15;
        const bool live = warp * kAgPos + pl < ctx;
        const float full_s = s[0] + __shfl_xor_sync(0xffffffffu, s[0], 1);   // (every lane shuffles)
        const float sc = live ? full_s * scale : -INFINITY;
        const float m = warp_max(sc);
        const float ex = live ? expf(sc - m) : 0.f;
        const float l = warp_sum((lane & 1) ? 0.f : ex);   // each position once (lanes 2 pl)
        float o[DPL];
#pragma unroll
        for (int t = 0; t < DPL; ++t) o[t] = 0.f;
#pragma unroll
        for (int i = 0; i < kAgPos; ++i) {
            const int p = warp * kAgPos + i;
            const float e = __shfl_sync(0xffffffffu, ex, 2 * i);
            if (p < ctx) {
                const uint32_t* vrow = reinterpret_cast<const uint32_t*>(sv + (size_t)p * hd + lane * DPL);
#pragma unroll
                for (int t = 0; t < DPL / 2; ++t) {
                    const uint32_t vv = vrow[t];
                    o[2 * t] = fmaf(e, bf16lo(vv), o[2 * t]);
                    o[2 * t + 1] = fmaf(e, bf16hi(vv), o[2 * t + 1]);
                }
            }
        }
        if (lane == 0) {
            sml[(warp * hpc + hh) * 2 + 0] = m;
            sml[(warp * hpc + hh) * 2 + 1] = l;
        }
#pragma unroll
        for (int t = 0; t < DPL; ++t) so[(warp * hpc + hh) * hd + lane * DPL + t] = o[t];
    }
    __syncthreads();
    tl_stamp(a.tl, 3);
    // merge the 16 warps in fixed order -> h2 of the CTA's heads
    for (int t = tid; t < hpc * hd; t += kAgThreads) {
        const int hh = t / hd, dd = t % hd;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kAgWarps; ++w)
            if (sml[(w * hpc + hh) * 2 + 1] > 0.f) M = fmaxf(M, sml[(w * hpc + hh) * 2]);
        float L = 0.f, Ov = 0.f;
#pragma unroll
        for (int w = 0; w < kAgWarps; ++w) {
            const float lw = sml[(w * hpc + hh) * 2 + 1];
            if (lw == 0.f) continue;
            const float e = expf(sml[(w * hpc + hh) * 2] - M);
            L = fmaf(lw, e, L);
            Ov = fmaf(so[(w * hpc + hh) * hd + dd], e, Ov);
        }
        const float hv = Ov / L;
        const int col = (h0 + hh) * hd + dd;
        a.out[(size_t)b * nq + col] = hv;
        if (a.peer.n) peer_put(a.peer, b, col, hv);
        if (a.out_sel.hist) hist_push(a.out_sel, hv, col);
    }
    peer_signal(a.peer, (unsigned)(hpc * hd));
    tl_stamp(a.tl, 6);
    if (a.keep_acc) {
        tl_stamp(a.tl, 4);
        return;   // the O GEMV re-zeroes the QKV accumulators after this kernel
    }
    // this CTA is the only reader of its q accumulators; the group's k / v accumulators are read
    // by its nsub CTAs: the last of them re-zeroes them
    unsigned long long* accz = a.acc + (size_t)b * a.acc_ld;
    for (int i = tid; i < hpc * hd; i += kAgThreads) accz[(size_t)h0 * hd + i] = 0ull;
    if (nsub > 1) {
        fence_acq_rel_gpu();
        __syncthreads();
        unsigned* gcnt = a.counters + kAttnGroupCounterOff + (size_t)b * a.hkv + g;
        if (tid == 0) {
            const unsigned prev = atomicAdd(gcnt, 1u);
            sflag[0] = prev == (unsigned)(nsub - 1);
        }
        __syncthreads();
        if (!sflag[0]) return;
        if (tid == 0) *gcnt = 0u;
    }
    for (int i = tid; i < hd; i += kAgThreads) {
        accz[nq + (size_t)g * hd + i] = 0ull;
        accz[nq + nk + (size_t)g * hd + i] = 0ull;
    }
    tl_stamp(a.tl, 4);
}

template <int DPL, bool CL>
__global__ void __launch_bounds__(kAttnThreads) attention_kernel(const AttnArgs a) {
    extern __shared__ __align__(16) float asmem[];
    tl_stamp(a.tl, 0);
    attention_body<DPL, CL>(a, asmem);   // waits on the QKV GEMV inside, after prefetching K/V
    tl_stamp(a.tl, 4);
}

}  // namespace larosa
