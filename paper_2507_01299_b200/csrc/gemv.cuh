// gemv.cuh — sparse GEMV over the kept rows of a column-major weight (eq. after_merge,
// PAPER.md:407-410; kernel recipe P:414: column-major storage, selective loads of the kept
// columns), with the epilogues the decoder layer fuses into it.
//
//   y[b][o] = sum_{r < nrows} val(r, b) * W[row(r)][o]      (+ epilogue)
//
// Work decomposition: the output columns are cut into tiles of TN = 256*NCW columns and
// the kept-row list into `n_splits` contiguous chunks; CTA (tile, split) streams
// rows[chunk] x [tile] of W.  Each kept row segment (TN*2 bytes, contiguous because W is
// stored [d_in][d_out]) is fetched by ONE cp.async.bulk (TMA engine) into a 6-stage shared
// memory ring guarded by mbarriers; a single producer lane issues the copies (L2
// evict-first) and NCW consumer warps do fp32 FMAs on the bf16 weights (8 columns per
// thread, 16-byte shared loads).  Splits are combined deterministically: every CTA writes
// its fp32 partial tile, and the last CTA of a tile (atomic ticket) sums the partials in
// split order and runs the epilogue.  No floating-point atomics anywhere.
#pragma once
#include "common.cuh"

namespace larosa {

enum EpKind : int { EP_STORE = 0, EP_RESID = 1, EP_SILU_GU = 2, EP_QKV_ROPE = 3 };

constexpr int kGemvStages = 6;
constexpr int kGemvStageBytes = 16384;
constexpr int kGuBlock = 64;   // == LAROSA_GU_BLOCK

struct GemvArgs {
    const uint16_t* W;
    int64_t ld;
    int d_out;
    const int32_t* rows;   // kept row indices (ascending); nullptr -> dense (row r = r)
    const float* vals;     // val(r, b) = vals[r * vs_r + b * vs_b]
    int64_t vs_r, vs_b;
    int nrows;             // row count when nrows_dev == nullptr
    const int* nrows_dev;  // device row count (batch > 1 union), or nullptr
    int batch;             // real tokens (<= template BP)
    int n_splits;
    float* partial;        // [n_splits][BP][d_out]
    unsigned* counters;    // [n_tiles], zero on entry, restored to zero on exit
    // epilogue
    int ep;
    const uint16_t* bias;  // [d_out] bf16 or nullptr
    const float* resid;    // EP_RESID: [batch][resid_ld]
    int64_t resid_ld;
    float* out;            // [batch][out_ld]
    int64_t out_ld;
    // EP_QKV_ROPE
    int hq, hkv, hd;
    float theta;
    const int32_t* pos;    // [batch]
    uint16_t* kc;          // [batch][hkv][max_ctx][hd]
    uint16_t* vc;
    int64_t max_ctx;
};

__host__ __device__ constexpr size_t gemv_smem_bytes(int bp, int ncw) {
    return 128 + (size_t)kGemvStages * kGemvStageBytes + (size_t)bp * ncw * 256 * sizeof(float);
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.0f + expf(-g)); }

template <int BP, int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32) gemv_kernel(const GemvArgs a) {
    constexpr int TN = NCW * 256;                 // columns per tile
    constexpr int G = kGemvStageBytes / (TN * 2); // rows per stage
    constexpr int NC = NCW * 32;                  // consumer threads
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kGemvStages;
    int* s_flag = reinterpret_cast<int*>(empty + kGemvStages);
    unsigned char* wbuf = smem + 128;
    float* ytile = reinterpret_cast<float*>(wbuf + kGemvStages * kGemvStageBytes);   // [BP][TN]

    const int tile = blockIdx.x, split = blockIdx.y;
    const int col0 = tile * TN;
    const int ncols = min(TN, a.d_out - col0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kGemvStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait();       // rows / vals / nrows come from the previous kernel
    pdl_trigger();    // let the next kernel's CTAs get resident as ours drain

    const int nrows = a.nrows_dev ? *a.nrows_dev : a.nrows;
    const int rps = (nrows + a.n_splits - 1) / a.n_splits;
    const int r_begin = min(nrows, split * rps);
    const int r_end = min(nrows, r_begin + rps);
    const int nstages = (r_end - r_begin + G - 1) / G;

    if (warp == NCW) {
        // ---------------- producer: one lane streams the kept row segments ----------------
        if (lane == 0) {
            const uint64_t pol = l2_policy_evict_first();
            const uint32_t seg = (uint32_t)ncols * 2u;
            for (int st = 0; st < nstages; ++st) {
                const int slot = st % kGemvStages;
                if (st >= kGemvStages) mbar_wait(&empty[slot], ((st / kGemvStages) - 1) & 1);
                const int r0 = r_begin + st * G;
                const int gc = min(G, r_end - r0);
                mbar_arrive_expect_tx(&full[slot], (uint32_t)gc * seg);
                unsigned char* dst = wbuf + slot * kGemvStageBytes;
                for (int g = 0; g < gc; ++g) {
                    const int row = a.rows ? __ldg(a.rows + r0 + g) : r0 + g;
                    bulk_g2s(dst + g * TN * 2, a.W + (size_t)row * a.ld + col0, seg, &full[slot], pol);
                }
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    const int c = threadIdx.x * 8;   // tile-local first column of this thread
    float acc[BP][8];
#pragma unroll
    for (int b = 0; b < BP; ++b)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[b][j] = 0.f;

    // token values of one row are contiguous (union layout [nrows][BP]) -> float4 loads
    const bool vec4 = (a.vs_b == 1) && (BP % 4 == 0) && (a.vs_r % 4 == 0);
    for (int st = 0; st < nstages; ++st) {
        const int slot = st % kGemvStages;
        const int r0 = r_begin + st * G;
        const int gc = min(G, r_end - r0);
        mbar_wait(&full[slot], (st / kGemvStages) & 1);
        const unsigned char* src = wbuf + slot * kGemvStageBytes + c * 2;
#pragma unroll 4
        for (int g = 0; g < gc; ++g) {
            const uint4 w = lds128(src + g * TN * 2);
            float wf[8];
            wf[0] = bf16lo(w.x); wf[1] = bf16hi(w.x);
            wf[2] = bf16lo(w.y); wf[3] = bf16hi(w.y);
            wf[4] = bf16lo(w.z); wf[5] = bf16hi(w.z);
            wf[6] = bf16lo(w.w); wf[7] = bf16hi(w.w);
            const float* vp = a.vals + (size_t)(r0 + g) * a.vs_r;
            float v[BP];
            if constexpr (BP % 4 == 0) {
                if (vec4) {
#pragma unroll
                    for (int b = 0; b < BP; b += 4) {
                        float4 t = __ldg(reinterpret_cast<const float4*>(vp) + b / 4);
                        v[b] = t.x; v[b + 1] = t.y; v[b + 2] = t.z; v[b + 3] = t.w;
                    }
                } else {
#pragma unroll
                    for (int b = 0; b < BP; ++b) v[b] = b < a.batch ? __ldg(vp + b * a.vs_b) : 0.f;
                }
            } else {
#pragma unroll
                for (int b = 0; b < BP; ++b) v[b] = b < a.batch ? __ldg(vp + b * a.vs_b) : 0.f;
            }
#pragma unroll
            for (int b = 0; b < BP; ++b)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[b][j] = fmaf(v[b], wf[j], acc[b][j]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
    }

    // ---------------- deterministic split reduction ----------------
    const bool active = c < ncols;
    if (a.n_splits == 1) {
#pragma unroll
        for (int b = 0; b < BP; ++b)
#pragma unroll
            for (int j = 0; j < 8; ++j) ytile[b * TN + c + j] = acc[b][j];
    } else {
        if (active) {
#pragma unroll
            for (int b = 0; b < BP; ++b) {
                if (b >= a.batch) break;
                float* p = a.partial + ((size_t)split * BP + b) * a.d_out + col0 + c;
                reinterpret_cast<float4*>(p)[0] = make_float4(acc[b][0], acc[b][1], acc[b][2], acc[b][3]);
                reinterpret_cast<float4*>(p)[1] = make_float4(acc[b][4], acc[b][5], acc[b][6], acc[b][7]);
            }
        }
        __threadfence();
        named_bar_sync(1, NC);
        if (threadIdx.x == 0) {
            const unsigned prev = atomicAdd(&a.counters[tile], 1u);
            s_flag[0] = (prev == (unsigned)(a.n_splits - 1));
        }
        named_bar_sync(1, NC);
        if (!s_flag[0]) return;
        if (threadIdx.x == 0) a.counters[tile] = 0u;   // self-reset for the next call
        __threadfence();
        if (active) {
            for (int b = 0; b < a.batch; ++b) {
                float y[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) y[j] = 0.f;
                const float* p = a.partial + (size_t)b * a.d_out + col0 + c;
                const size_t sstride = (size_t)BP * a.d_out;
                int s = 0;
                for (; s + 4 <= a.n_splits; s += 4) {
                    float4 t[8];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        t[2 * u] = __ldcg(reinterpret_cast<const float4*>(p + (s + u) * sstride));
                        t[2 * u + 1] = __ldcg(reinterpret_cast<const float4*>(p + (s + u) * sstride) + 1);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        y[0] += t[2 * u].x; y[1] += t[2 * u].y; y[2] += t[2 * u].z; y[3] += t[2 * u].w;
                        y[4] += t[2 * u + 1].x; y[5] += t[2 * u + 1].y; y[6] += t[2 * u + 1].z; y[7] += t[2 * u + 1].w;
                    }
                }
                for (; s < a.n_splits; ++s) {
                    float4 t0 = __ldcg(reinterpret_cast<const float4*>(p + s * sstride));
                    float4 t1 = __ldcg(reinterpret_cast<const float4*>(p + s * sstride) + 1);
                    y[0] += t0.x; y[1] += t0.y; y[2] += t0.z; y[3] += t0.w;
                    y[4] += t1.x; y[5] += t1.y; y[6] += t1.z; y[7] += t1.w;
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) ytile[b * TN + c + j] = y[j];
            }
        }
    }
    named_bar_sync(1, NC);

    // ---------------- epilogue on the complete tile (tile-local column c .. c+7) ----------------
    if (!active) return;
    const int o0 = col0 + c;
    float bias8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) bias8[j] = 0.f;
    if (a.bias && a.ep != EP_SILU_GU) {
        const uint4 bb = __ldg(reinterpret_cast<const uint4*>(a.bias + o0));
        bias8[0] = bf16lo(bb.x); bias8[1] = bf16hi(bb.x); bias8[2] = bf16lo(bb.y); bias8[3] = bf16hi(bb.y);
        bias8[4] = bf16lo(bb.z); bias8[5] = bf16hi(bb.z); bias8[6] = bf16lo(bb.w); bias8[7] = bf16hi(bb.w);
    }
    for (int b = 0; b < a.batch; ++b) {
        const float* yt = ytile + b * TN;
        if (a.ep == EP_STORE || a.ep == EP_RESID) {
            float r[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = yt[c + j] + bias8[j];
            if (a.ep == EP_RESID) {
                const float* rp = a.resid + (size_t)b * a.resid_ld + o0;
#pragma unroll
                for (int j = 0; j < 8; ++j) r[j] = rp[j] + r[j];
            }
            float* op = a.out + (size_t)b * a.out_ld + o0;
            reinterpret_cast<float4*>(op)[0] = make_float4(r[0], r[1], r[2], r[3]);
            reinterpret_cast<float4*>(op)[1] = make_float4(r[4], r[5], r[6], r[7]);
        } else if (a.ep == EP_SILU_GU) {
            // fused column o: block t = o / 128 holds gate [t*64, t*64+64) then up of the same rows
            const int within = o0 % (2 * kGuBlock);
            if (within < kGuBlock) {
                const int i0 = (o0 / (2 * kGuBlock)) * kGuBlock + within;
                float h[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float g = yt[c + j];
                    const float u = yt[c + kGuBlock + j];
                    h[j] = silu_f(g) * u;
                }
                float* op = a.out + (size_t)b * a.out_ld + i0;
                reinterpret_cast<float4*>(op)[0] = make_float4(h[0], h[1], h[2], h[3]);
                reinterpret_cast<float4*>(op)[1] = make_float4(h[4], h[5], h[6], h[7]);
            }
        } else {   // EP_QKV_ROPE
            const int hd = a.hd, half = hd >> 1;
            const int nq = a.hq * hd, nk = a.hkv * hd;
            const int p = a.pos[b];
            float r[8];
            const int head_off = o0 % hd;   // 8 consecutive columns lie in one head
            if (o0 < nq + nk) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int i = head_off + j;
                    const int fi = i < half ? i : i - half;
                    const int partner = i < half ? c + j + half : c + j - half;
                    const double inv_freq = exp(-(2.0 * fi / hd) * log((double)a.theta));
                    double sn, cs;
                    sincos((double)p * inv_freq, &sn, &cs);
                    const float x = yt[c + j] + bias8[j];
                    float xpart = yt[partner];
                    if (a.bias) xpart += bf16f(a.bias[col0 + partner]);
                    const float rot = i < half ? -xpart : xpart;
                    r[j] = (float)((double)x * cs + (double)rot * sn);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) r[j] = yt[c + j] + bias8[j];
            }
            if (o0 < nq) {
                float* op = a.out + (size_t)b * a.out_ld + o0;
                reinterpret_cast<float4*>(op)[0] = make_float4(r[0], r[1], r[2], r[3]);
                reinterpret_cast<float4*>(op)[1] = make_float4(r[4], r[5], r[6], r[7]);
            } else {
                const bool isk = o0 < nq + nk;
                const int oo = o0 - (isk ? nq : nq + nk);
                const int kvh = oo / hd;
                uint16_t* dst = (isk ? a.kc : a.vc) + (((size_t)b * a.hkv + kvh) * a.max_ctx + p) * hd + head_off;
                uint4 pk;
                pk.x = (uint32_t)f2bf16_rne(r[0]) | ((uint32_t)f2bf16_rne(r[1]) << 16);
                pk.y = (uint32_t)f2bf16_rne(r[2]) | ((uint32_t)f2bf16_rne(r[3]) << 16);
                pk.z = (uint32_t)f2bf16_rne(r[4]) | ((uint32_t)f2bf16_rne(r[5]) << 16);
                pk.w = (uint32_t)f2bf16_rne(r[6]) | ((uint32_t)f2bf16_rne(r[7]) << 16);
                *reinterpret_cast<uint4*>(dst) = pk;
            }
        }
    }
}

}  // namespace larosa
