// topk.cuh — exact per-token Top-K (S_k of eq. 2) as a radix select on
// the uint32 keys bits(|x|) with the lower-index tie-break, the RMS scale of the
// h1/h3 sites, and stable compaction to ascending indices.
//
// Latency-optimised and distributed over a thread-block CLUSTER per token (it sits between
// two dependent GEMVs on the critical path; one SM alone is issue- and bandwidth-limited):
//  * CTA r of the cluster owns the contiguous chunk [r*C, r*C + C) of the vector (C a
//    multiple of 32), element r*C + j*512 + t lives in register xv[j] of thread t
//    (coalesced loads; each warp-round of 32 consecutive elements is one mask word);
//  * fused source finalisation: the site's input is computed from the producer GEMV's
//    fixed-point accumulators (residual add, or SiLU(g)*u), written to the layer's buffer
//    and the accumulators are re-zeroed, by all CTAs of the cluster in parallel;
//  * digits: bits [30:19] (4096 bins), [18:7] (4096), [6:0] (128); each CTA histograms its
//    own candidates locally, CTA r merges bin slice r over the cluster through distributed
//    shared memory, the CTA whose slice holds the k-th key finds its bucket (block suffix
//    scan) and all CTAs read the result back through DSMEM; a pass whose bucket is taken
//    whole ends the select (continuous data: 2 passes), an exact key tie at position k is
//    resolved by index;  (remote atomics into one CTA's histogram were tried: Gaussian
//    keys crowd a few bins and the DSMEM reductions serialise);
//  * compaction: per-CTA counts and sum-of-squares partials are exchanged through DSMEM
//    (fixed order, deterministic), then per-round warp ballots give coalesced stores.
#pragma once
#include "common.cuh"
#include "gemv.cuh"   // fixed-point accumulator helpers, kGuBlock
#include "img_layout.cuh"

namespace larosa {

constexpr int kTopkThreads = 512;
constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int kTopkBins = 4096;
constexpr int kTopkMaxCluster = 8;

__host__ __device__ constexpr size_t topk_smem_bytes(int d) {
    return sizeof(int) * 3 * kTopkBins + sizeof(int) * 128 + 0 * (size_t)d;
}

// cluster size for a vector of length d: ~1024 elements per CTA, at most 8 CTAs
__host__ __device__ constexpr int topk_cluster_size(int d) {
    return d <= 1024 ? 1 : ((d + 1023) / 1024 < kTopkMaxCluster ? (d + 1023) / 1024 : kTopkMaxCluster);
}
// per-CTA chunk (multiple of 32) and elements per thread (rounded to an instantiated size)
__host__ __device__ constexpr int topk_chunk(int d, int cs) { return (((d + cs - 1) / cs) + 31) / 32 * 32; }
__host__ __device__ constexpr int topk_ept(int d) {
    return ((topk_chunk(d, topk_cluster_size(d)) + kTopkThreads - 1) / kTopkThreads + 1) / 2 * 2;
}

// Where the site's input vector comes from (the producer GEMV leaves fixed-point
// accumulators; the Top-K kernel finalises them, see gemv.cuh):
enum TopkSrc : int {
    SRC_PLAIN = 0,      // x[i]
    SRC_RESID_ACC = 1,  // [resid[i] +] fix^-1(acc[i])                    (residual add)
    SRC_SILU_GU = 2,    // SiLU(g_i) * u_i, g/u = fix^-1 of the interleaved gate|up acc
};

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
    ThreshOut* rule_out;  // [batch] if set: emit the selection rule (no idx/vals lists)
    unsigned char* img;      // rule mode, batch 2-16: also write the token image (img_layout.cuh) of
    unsigned char* img_raw;  // the masked scaled values, and optionally of the raw values
    unsigned long long* tl;  // debug timeline slot or null
};

// token b's element i = v of the image: masked and scaled (keep ? v s : 0) split bf16 hi | lo, and
// the raw value split the same way (the arithmetic of rule_apply_image_kernel)
__device__ __forceinline__ void topk_img_put(unsigned char* img, unsigned char* raw, int b, int i, float v, bool keep,
                                             float s) {
    const float f = keep ? v * s : 0.f;
    const uint16_t h = f2bf16_rne(f);
    const int kk = i & (kImgChunkK - 1);
    unsigned char* ch = img + (size_t)(i / kImgChunkK) * kImgChunkBytes;
    *reinterpret_cast<uint16_t*>(ch + img_off(b, kk)) = h;
    *reinterpret_cast<uint16_t*>(ch + img_off(16 + b, kk)) = f2bf16_rne(f - bf16f(h));
    if (raw) {
        const uint16_t rh = f2bf16_rne(v);
        unsigned char* cr = raw + (size_t)(i / kImgChunkK) * kImgChunkBytes;
        *reinterpret_cast<uint16_t*>(cr + img_off(b, kk)) = rh;
        *reinterpret_cast<uint16_t*>(cr + img_off(16 + b, kk)) = f2bf16_rne(v - bf16f(rh));
    }
}

__device__ __forceinline__ void topk_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t topk_mapa(const void* local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
    return r;
}
__device__ __forceinline__ void topk_red_remote(uint32_t addr, uint32_t v) {
    asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// (no "memory" clobber: the loads of a batch may issue back to back; the cluster barriers
// carry the ordering)
__device__ __forceinline__ uint32_t topk_ld_remote(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// grid = (CS, batch), cluster (CS, 1, 1): one cluster per token.  One kernel per (source
// mode, elements per thread) so each launch only fetches its own (small) code.
template <int MODE, int EPT>
__global__ void __launch_bounds__(kTopkThreads, 1) topk_kernel(TopkKernelArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    int* hist0 = reinterpret_cast<int*>(smem);                 // local histograms (double-buffered)
    int* hist1 = hist0 + kTopkBins;
    int* scr = hist1 + kTopkBins;
    int* s_wtot = scr;                                          // [0, 16)    scan scratch
    int* s_cnt = scr + 16;                                      // [16, 80)   per-round warp counts 2 x [2][16]
    int* s_red = scr + 80;                                      // [80, 96)   block-reduction scratch
    int* s_pub = scr + 96;                                      // [96, 100)  published: n_gt, n_eq, ssq bits
    int* s_res = scr + 100;                                     // [100, 104) bucket result (owner CTA)
    int* mh = scr + 128;                                        // merged histogram slice (<= 4096)
    tl_stamp(a.tl, 0);
    pdl_wait();
    pdl_trigger();
    tl_stamp(a.tl, 1);

    const int d = a.d, k = a.k;
    const int b = blockIdx.y, rank = blockIdx.x, cs = gridDim.x;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int C = topk_chunk(d, cs);
    const int lo = rank * C;
    constexpr int NT = kTopkThreads;
    const int nwords = (d + 31) / 32;
    int32_t* out_idx = a.idx + (size_t)b * k;
    float* out_vals = a.vals + (size_t)b * k;
    uint32_t* out_mask = a.mask ? a.mask + (size_t)b * nwords : nullptr;

    // ---- 1. this CTA's values (raw fp32 bits) in registers; finalise fused sources -------
    uint32_t xv[EPT];
    float ssq = 0.f;
    const float* x = a.x ? a.x + (size_t)b * a.ldx : nullptr;
    float* xout = a.xr_out ? a.xr_out + (size_t)b * d : nullptr;
    const float* resid = a.resid ? a.resid + (size_t)b * a.resid_ld : nullptr;
    unsigned long long* acc = a.acc ? a.acc + (size_t)b * a.acc_ld : nullptr;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
        const int i = lo + j * NT + tid;
        float v = 0.f;
        if (j * NT + tid < C && i < d) {
            if constexpr (MODE == SRC_PLAIN) {
                v = x[i];
            } else if constexpr (MODE == SRC_RESID_ACC) {
                v = (resid ? resid[i] : 0.f) + fix_to_f(acc[i]);
                acc[i] = 0ull;
            } else {
                const int gi = (i / kGuBlock) * (2 * kGuBlock) + (i % kGuBlock);
                const float g = fix_to_f(acc[gi]);
                const float u = fix_to_f(acc[gi + kGuBlock]);
                acc[gi] = 0ull;
                acc[gi + kGuBlock] = 0ull;
                v = g / (1.0f + expf(-g)) * u;
            }
            if (xout) xout[i] = v;
        }
        xv[j] = __float_as_uint(v);
        ssq = fmaf(v, v, ssq);
    }
    if (a.zero) {
        unsigned long long* z = a.zero + (size_t)b * a.zero_ld;
        const int zc = (a.zero_n + cs - 1) / cs;
        for (int i = rank * zc + tid; i < min(a.zero_n, rank * zc + zc); i += NT) z[i] = 0ull;
    }
#define KEY(j) (xv[j] & 0x7fffffffu)
#define VALID(j) ((j) * NT + tid < C && lo + (j) * NT + tid < d)
    // per-CTA sum of squares (fixed order) -> published for the cluster
    ssq = warp_sum(ssq);
    if (lane == 0) reinterpret_cast<float*>(s_red)[wid] = ssq;
    for (int i = tid; i < kTopkBins; i += NT) hist0[i] = 0;
    __syncthreads();
    if (tid == 0) {
        float t = 0.f;
        for (int w = 0; w < kTopkWarps; ++w) t += reinterpret_cast<float*>(s_red)[w];
        s_pub[2] = __float_as_int(t);
    }
    topk_cluster_sync();   // CTA 0's histograms are zero before anyone adds into them
    tl_stamp(a.tl, 2);

    // ---- 2. radix select of the k-th largest key ----------------------------------------
    // per pass: local histograms (smem atomics) -> cluster barrier -> CTA r merges bin slice
    // r over all CTAs through DSMEM and publishes the slice total -> barrier -> the CTA whose
    // slice holds the k-th key scans it and publishes (b*, rem', count) -> barrier -> read.
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
                if (VALID(j) && (KEY(j) & pmask) == prefix) atomicAdd(&hist[(KEY(j) >> sh) & dmask], 1);
            topk_cluster_sync();                                  // (A) all local histograms complete
            // merge my bin slice [s_lo, s_hi) over the cluster (fixed order) into mh
            const int spc = (nb + cs - 1) / cs;
            const int s_lo = min(nb, rank * spc), s_hi = min(nb, s_lo + spc);
            int tot = 0;
            for (int bb = s_lo + tid; bb < s_hi; bb += NT) {
                uint32_t hv[kTopkMaxCluster];          // issue all remote loads, then sum
#pragma unroll
                for (int q = 0; q < kTopkMaxCluster; ++q)
                    hv[q] = q < cs ? topk_ld_remote(topk_mapa(hist + bb, (uint32_t)q)) : 0u;
                int m = 0;
#pragma unroll
                for (int q = 0; q < kTopkMaxCluster; ++q) m += (int)hv[q];
                mh[bb - s_lo] = m;
                tot += m;
            }
            tot = warp_sum_i(tot);
            if (lane == 0) s_red[wid] = tot;
            for (int i = tid; i < kTopkBins; i += NT) hnext[i] = 0;   // next pass's local histogram
            __syncthreads();
            if (tid == 0) {
                int t = 0;
                for (int w = 0; w < kTopkWarps; ++w) t += s_red[w];
                s_pub[3] = t;
            }
            topk_cluster_sync();                                  // (B) slice totals published
            // which slice holds the rem-th key (slices cs-1 .. 0 cover bins top-down)?
            uint32_t tq[kTopkMaxCluster];
#pragma unroll
            for (int q = 0; q < kTopkMaxCluster; ++q) tq[q] = q < cs ? topk_ld_remote(topk_mapa(s_pub + 3, (uint32_t)q)) : 0u;
            int above = 0, owner = -1, rem_in = 0;
#pragma unroll
            for (int q = kTopkMaxCluster - 1; q >= 0; --q) {
                if (q < cs && owner < 0 && above + (int)tq[q] >= rem) {
                    owner = q;
                    rem_in = rem - above;
                }
                above += (int)tq[q];
            }
            if (rank == owner) {
                // block suffix scan over my merged slice (top bins first), 512 threads
                const int nsl = s_hi - s_lo;
                const int bpt = (nsl + NT - 1) / NT;
                const int thi = nsl - tid * bpt;                 // thread's bins [thi - bpt, thi) (slice-local)
                int c = 0;
                for (int bb = thi - 1; bb >= max(0, thi - bpt); --bb) c += mh[bb];
                const int inc = warp_incl_scan(c);
                if (lane == 31) s_wtot[wid] = inc;
                __syncthreads();
                const int t = lane < kTopkWarps ? s_wtot[lane] : 0;
                const int ti = warp_incl_scan(t);
                const int before = __shfl_sync(0xffffffffu, ti - t, wid) + inc - c;
                if (c > 0 && before < rem_in && rem_in <= before + c) {
                    int accu = before;
                    for (int bb = thi - 1; bb >= max(0, thi - bpt); --bb) {
                        const int h = mh[bb];
                        if (accu + h >= rem_in) {
                            s_res[0] = s_lo + bb;
                            s_res[1] = rem_in - accu;
                            s_res[2] = h;
                            break;
                        }
                        accu += h;
                    }
                }
            }
            topk_cluster_sync();                                  // (C) result published by the owner
            const uint32_t res_remote = topk_mapa(s_res, (uint32_t)owner);
            const int bstar = (int)topk_ld_remote(res_remote);
            rem = (int)topk_ld_remote(res_remote + 4);
            const int cnt = (int)topk_ld_remote(res_remote + 8);
            prefix |= (uint32_t)bstar << sh;
            pmask |= dmask << sh;
            tl_stamp(a.tl, 5 + pass);
            if (cnt == rem) {
                exact_ge = true;
                break;
            }
            if (pass == 2) tie_mode = true;
        }
    }
    const uint32_t thr = prefix;

    // ---- rule mode: publish (Tk, Ti, s) instead of the index list ------------------------
    // keep i iff key > Tk or (key == Tk and i <= Ti)  (the consumer GEMV selects its rows)
    if (a.rule_out && (exact_ge || !tie_mode)) {
        if ((rank == 0 && tid == 0) || a.img) {   // (every thread needs the scale for the image)
            float tot = 0.f;
            uint32_t psq[kTopkMaxCluster];
#pragma unroll
            for (int q = 0; q < kTopkMaxCluster; ++q)
                psq[q] = q < cs ? topk_ld_remote(topk_mapa(s_pub + 2, (uint32_t)q)) : 0u;
#pragma unroll
            for (int q = 0; q < kTopkMaxCluster; ++q)
                if (q < cs) tot += __uint_as_float(psq[q]);
            const float scale = a.rms_eps >= 0.f ? 1.0f / sqrtf(tot / (float)d + a.rms_eps) : 1.0f;
            if (rank == 0 && tid == 0) {
                ThreshOut r;
                r.tk = thr;
                r.ti = 0x7fffffff;   // key == Tk (the bucket's lower edge) is kept too
                r.scale = scale;
                r.pad = 0;
                a.rule_out[b] = r;
            }
            if (a.img) {
#pragma unroll
                for (int j = 0; j < EPT; ++j)
                    if (VALID(j)) topk_img_put(a.img, a.img_raw, b, lo + j * NT + tid, __uint_as_float(xv[j]), KEY(j) >= thr,
                                               scale);
            }
        }
        tl_stamp(a.tl, 8);
        topk_cluster_sync();   // rank 0 read the others' published partials
        tl_stamp(a.tl, 4);
        return;
    }

    // ---- 3. compaction: cluster-wide prefix of counts, then per-round ballots ------------
    int my_gt = 0, my_eq = 0;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
        if (!VALID(j)) continue;
        if (exact_ge) {
            my_gt += KEY(j) >= thr;
        } else {
            my_gt += KEY(j) > thr;
            my_eq += KEY(j) == thr;
        }
    }
    {
        int g2 = my_gt, e2 = my_eq;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            g2 += __shfl_xor_sync(0xffffffffu, g2, o);
            e2 += __shfl_xor_sync(0xffffffffu, e2, o);
        }
        __syncthreads();   // s_red reuse
        if (lane == 0) {
            s_red[wid] = g2;
            s_cnt[wid] = e2;
        }
        __syncthreads();
        if (tid == 0) {
            int tg = 0, te = 0;
            for (int w = 0; w < kTopkWarps; ++w) {
                tg += s_red[w];
                te += s_cnt[w];
            }
            s_pub[0] = tg;
            s_pub[1] = te;
        }
    }
    topk_cluster_sync();
    // counts of lower-rank CTAs (index order) and the total sum of squares (fixed order)
    int gt_before = 0, eq_before = 0;
    float tot_ssq = 0.f;
    uint32_t pg[kTopkMaxCluster], pe[kTopkMaxCluster], ps[kTopkMaxCluster];
#pragma unroll
    for (int q = 0; q < kTopkMaxCluster; ++q) {
        const uint32_t pub = topk_mapa(s_pub, (uint32_t)(q < cs ? q : 0));
        pg[q] = q < cs ? topk_ld_remote(pub) : 0u;
        pe[q] = q < cs ? topk_ld_remote(pub + 4) : 0u;
        ps[q] = q < cs ? topk_ld_remote(pub + 8) : 0u;
    }
#pragma unroll
    for (int q = 0; q < kTopkMaxCluster; ++q) {
        if (q < rank) {
            gt_before += (int)pg[q];
            eq_before += (int)pe[q];
        }
        if (q < cs) tot_ssq += __uint_as_float(ps[q]);
    }
    const float scale = a.rms_eps >= 0.f ? 1.0f / sqrtf(tot_ssq / (float)d + a.rms_eps) : 1.0f;
    // selected before this CTA = gt before + (eq taken in index order: the first rem overall)
    const int take_eq_before = tie_mode ? min(eq_before, rem) : 0;
    int base = gt_before + take_eq_before, eq_base = eq_before;
    const uint32_t lt = (1u << lane) - 1u;
    __syncthreads();   // s_cnt reuse
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
        const int off = j * NT + tid;
        const int i = lo + off;
        const bool valid = VALID(j);
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
        int* cnt = s_cnt + (j & 1) * 32;
        if (lane == 0) {
            cnt[wid] = __popc(bgt);
            cnt[16 + wid] = __popc(beq);
        }
        __syncthreads();
        const int cg = lane < kTopkWarps ? cnt[lane] : 0, ce = lane < kTopkWarps ? cnt[16 + lane] : 0;
        const int ig = warp_incl_scan(cg), ie = warp_incl_scan(ce);
        const int wg = __shfl_sync(0xffffffffu, ig - cg, wid);
        const int we = __shfl_sync(0xffffffffu, ie - ce, wid);
        const int tg = __shfl_sync(0xffffffffu, ig, 31), te = __shfl_sync(0xffffffffu, ie, 31);
        const int erank = eq_base + we + __popc(beq & lt);
        const bool sel = gt || (eq && tie_mode && erank < rem);
        const uint32_t bsel = __ballot_sync(0xffffffffu, sel);
        const int eq_sel_before_warp = tie_mode ? max(0, min(eq_base + we, rem) - min(eq_base, rem)) : 0;
        const int pos = base + wg + eq_sel_before_warp + __popc(bsel & lt);
        if (a.rule_out) {
            if (eq && tie_mode && erank == rem - 1) {   // the k-th element: Ti = its index
                ThreshOut r;
                r.tk = thr;
                r.ti = i;
                r.scale = scale;
                r.pad = 0;
                a.rule_out[b] = r;
            }
            if (a.img && valid) topk_img_put(a.img, a.img_raw, b, i, __uint_as_float(xv[j]), sel, scale);
        } else if (sel) {
            out_idx[pos] = i;
            out_vals[pos] = __uint_as_float(xv[j]) * scale;
        }
        if (out_mask && lane == 0 && j * NT + wid * 32 < C && lo + j * NT + wid * 32 < d)
            out_mask[(lo + j * NT + wid * 32) >> 5] = bsel;
        base += tg + (tie_mode ? max(0, min(eq_base + te, rem) - min(eq_base, rem)) : 0);
        eq_base += te;
    }
    if (a.scale && rank == 0 && tid == 0) a.scale[b] = scale;
#undef KEY
#undef VALID
    topk_cluster_sync();   // peers may still read this CTA's published counts
}

// ---- the per-token selection RULE at batch > 1 on one CTA per token (no cluster) -------------------
// The rule kernel of the batch 2-16 layer (rule mode, plain source): token b's exact Top-K rule
// (lower index on ties, Z10), its RMS scale and -- if img is set -- the token image, from ONE
// 1024-thread CTA (element i = thread t + 1024 j, coalesced).  The k-th key is located by at most
// three 11/11/9-bit digit histograms in shared memory; as soon as the boundary bucket holds
// <= kRsCand keys they are gathered and ranked exactly by (key desc, index asc), which yields
// (Tk, Ti) directly (usually after the first digit).  A bucket of > kRsCand identical 31-bit keys
// takes the index-ordered walk.  No cluster barriers or distributed shared memory: the cluster
// kernel's 6+ cluster-wide barriers per token were the batch-16 rule's cost.
constexpr int kRsThreads = 1024;
constexpr int kRsBins = 2048;
constexpr int kRsCand = 256;

template <int EPT>
__global__ void __launch_bounds__(kRsThreads, 1) rule_select_kernel(const TopkKernelArgs a) {
    constexpr int NT = kRsThreads;
    __shared__ int hist[kRsBins];
    __shared__ __align__(16) uint32_t ck[kRsCand];
    __shared__ __align__(16) int ci[kRsCand];
    __shared__ int sw[NT / 32 + 1];
    __shared__ float fsw[NT / 32];
    __shared__ int misc[8];
    const int b = blockIdx.x, tid = threadIdx.x;
    const int d = a.d, k = a.k;
    tl_stamp(a.tl, 0);
    for (int i = tid; i < kRsBins; i += NT) hist[i] = 0;
    pdl_wait();
    pdl_trigger();
    tl_stamp(a.tl, 1);
    const float* x = a.x + (size_t)b * a.ldx;
    uint32_t xb[EPT];
    float ssq = 0.f;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
        const int i = tid + NT * j;
        const float v = i < d ? x[i] : 0.f;
        xb[j] = __float_as_uint(v);
        ssq = fmaf(v, v, ssq);
    }
    const float tot = block_sum<NT>(ssq, fsw);   // (fixed order; contains the barrier after the zeroing)
    const float scale = a.rms_eps >= 0.f ? 1.0f / sqrtf(tot / (float)d + a.rms_eps) : 1.0f;
    tl_stamp(a.tl, 2);
#define RS_KEY(j) (xb[j] & 0x7fffffffu)
#define RS_VALID(j) (tid + NT * (j) < d)
    uint32_t tk = 0u;
    int ti = 0x7fffffff;
    if (k <= 0) {
        tk = 0xffffffffu;   // keys < 2^31: nothing is kept
        ti = -1;
    } else if (k < d) {
        uint32_t prefix = 0u, pmask = 0u;
        int rem = k;
#pragma unroll 1
        for (int L = 0; L < 3; ++L) {
            const int sh = L == 0 ? 20 : (L == 1 ? 9 : 0);
            const int nb = L == 2 ? 512 : kRsBins;
            const uint32_t dm = (uint32_t)(nb - 1);
            if (L > 0) {
                for (int i = tid; i < nb; i += NT) hist[i] = 0;
                __syncthreads();
            }
            // (plain shared atomics: warp aggregation by match.any measured slower here)
            const int lane = tid & 31;
#pragma unroll
            for (int j = 0; j < EPT; ++j)
                if (RS_VALID(j) && (RS_KEY(j) & pmask) == prefix) atomicAdd(&hist[(RS_KEY(j) >> sh) & dm], 1);
            __syncthreads();
            if (L == 0) tl_stamp(a.tl, 9);
            // thread t owns bins [nb - bpt (t + 1), nb - bpt t) (top bins first)
            const int bpt = (nb + NT - 1) / NT;
            const int hi = nb - bpt * tid;
            int c = 0;
            for (int q = hi - 1; q >= max(0, hi - bpt); --q) c += hist[q];
            int total;
            const int above = block_excl_scan<NT>(c, sw, &total);
            if (c > 0 && above < rem && rem <= above + c) {
                int acc = above;
                for (int q = hi - 1; q >= max(0, hi - bpt); --q) {
                    if (acc + hist[q] >= rem) {
                        misc[0] = q;
                        misc[1] = rem - acc;
                        misc[2] = hist[q];
                        break;
                    }
                    acc += hist[q];
                }
            }
            if (tid == 0) misc[3] = 0;
            __syncthreads();
            const int bin = misc[0], cnt = misc[2];
            if (L == 0) tl_stamp(a.tl, 10);
            rem = misc[1];
            prefix |= (uint32_t)bin << sh;
            pmask |= dm << sh;
            if (cnt == rem) {            // the bucket is taken whole: key >= prefix
                tk = prefix;
                ti = 0x7fffffff;
                break;
            }
            if (cnt <= kRsCand) {        // gather the bucket and rank it exactly
#pragma unroll
                for (int j = 0; j < EPT; ++j) {
                    const bool in = RS_VALID(j) && (RS_KEY(j) & pmask) == prefix;
                    const unsigned m = __ballot_sync(0xffffffffu, in);
                    if (m) {             // one counter atomic per warp
                        int base = 0;
                        if (lane == __ffs(m) - 1) base = atomicAdd(&misc[3], __popc(m));
                        base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
                        if (in) {
                            const int slot = base + __popc(m & ((1u << lane) - 1u));
                            ck[slot] = RS_KEY(j);
                            ci[slot] = tid + NT * j;
                        }
                    }
                }
                __syncthreads();
                tl_stamp(a.tl, 11);
                // rank: 4 threads per candidate (adjacent lanes), each over a quarter of the bucket,
                // 4 candidates per 16-byte shared load
                {
                    const int cnd = tid >> 2, part = tid & 3;
                    const int cnt4 = (cnt + 3) & ~3;
                    for (int u = cnt + tid; u < cnt4; u += NT) {   // pad to a multiple of 4 (never ranks above)
                        ck[u] = 0u;
                        ci[u] = 0x7fffffff;
                    }
                    __syncthreads();
                    int r = 0;
                    uint32_t mk = 0u;
                    int mi = 0;
                    if (cnd < cnt) {
                        mk = ck[cnd];
                        mi = ci[cnd];
                        const int q4 = cnt4 / 4;                    // 4-key groups
                        for (int g4 = part; g4 < q4; g4 += 4) {
                            const uint4 kk = reinterpret_cast<const uint4*>(ck)[g4];
                            const int4 ii = reinterpret_cast<const int4*>(ci)[g4];
                            r += (kk.x > mk || (kk.x == mk && ii.x < mi)) + (kk.y > mk || (kk.y == mk && ii.y < mi)) +
                                 (kk.z > mk || (kk.z == mk && ii.z < mi)) + (kk.w > mk || (kk.w == mk && ii.w < mi));
                        }
                    }
                    r += __shfl_xor_sync(0xffffffffu, r, 1);
                    r += __shfl_xor_sync(0xffffffffu, r, 2);
                    if (cnd < cnt && part == 0 && r == rem - 1) {
                        misc[4] = (int)mk;
                        misc[5] = mi;
                    }
                }
                __syncthreads();
                tk = (uint32_t)misc[4];
                ti = misc[5];
                break;
            }
            if (L == 2) {                // > kRsCand identical keys: the rem-th lowest index among them
                tk = prefix;
                uint32_t eqm = 0u;       // (a register bit mask: xb stays in registers)
#pragma unroll
                for (int j = 0; j < EPT; ++j)
                    if (RS_VALID(j) && RS_KEY(j) == prefix) eqm |= 1u << j;
                int base = 0;
#pragma unroll 1
                for (int j = 0; j < EPT; ++j) {
                    const bool eq = (eqm >> j) & 1u;
                    int tot_j;
                    const int pos = block_excl_scan<NT>(eq ? 1 : 0, sw, &tot_j);
                    if (eq && base + pos == rem - 1) misc[6] = tid + NT * j;
                    base += tot_j;
                    __syncthreads();
                    if (base >= rem) break;
                }
                __syncthreads();
                ti = misc[6];
            }
        }
    }
    tl_stamp(a.tl, 5);
    if (tid == 0) {
        ThreshOut r;
        r.tk = tk;
        r.ti = ti;
        r.scale = scale;
        r.pad = 0;
        a.rule_out[b] = r;
    }
    if (a.img) {
#pragma unroll
        for (int j = 0; j < EPT; ++j)
            if (RS_VALID(j)) {
                const uint32_t key = RS_KEY(j);
                const int i = tid + NT * j;
                topk_img_put(a.img, a.img_raw, b, i, __uint_as_float(xb[j]), key > tk || (key == tk && i <= ti), scale);
            }
    }
#undef RS_KEY
#undef RS_VALID
    tl_stamp(a.tl, 4);
}

}  // namespace larosa
