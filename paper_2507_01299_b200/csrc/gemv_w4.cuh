// gemv_w4.cuh — Top-K sparse GEMV over group-quantised int4 weights (W4A16; SURVEY §8(f) N3:
// the paper shows LaRoSA composes with weight quantisation).  Layout (column-major
// like the bf16 path, so a kept input channel is one contiguous run):
//   Wq uint8 [d_in][d_out / 2]: byte b of row j holds columns 2b (low nibble) and 2b + 1
//   S  fp16  [d_in][d_out / 128]: the scale of group g = o / 128 of row j
//   w[j][o] = (q[j][o] - 8) * S[j][o / 128]        (symmetric int4, q in [0, 15])
// The batch-1 SELECT prologue (select_rows: the site's exact Top-K rule, Z10) is the
// bf16 kernel's; the stream then moves a kept row's 256-column slice segment as 128 bytes: one
// warp-wide LDGSTS.128 fetches 4 rows (8 lanes x 16 B per row) into the warp's ring, and lane l
// dequantises its 8 columns (one 32-bit shared load per row) with the row's two group scales
// (staged with the list).  A quarter of the bf16 bytes and instructions per kept row.
#pragma once
#include <cuda_fp16.h>
#include "gemv.cuh"

namespace larosa {

constexpr int kW4Group = 128;                 // == LAROSA_W4_GROUP
// Slice width (columns per CTA) per launch: 512 (256 B per kept row, lane = 16 columns: twice the
// finalising CTAs, half the reds and epilogue work per CTA -- the small sites, whose tails were
// longer than their streams) or 1024 (512 B, lane = 32 columns: 16-byte loads -- the large sites)
template <int SC>
struct W4Cfg {
    static constexpr int kSliceCols = SC;
    static constexpr int kLaneCols = SC / 32;                 // columns per lane
    static constexpr int kLaneBytes = kLaneCols / 2;          // int4 bytes per lane and row (16 or 8)
    static constexpr int kGroups = SC / kW4Group;             // scale groups per slice (8 or 4)
    static constexpr int kRowBytes = SC / 2;
    static constexpr int kStages = 8192 / kRowBytes;          // rows in flight per warp: 8 KB ring per warp
    static constexpr int kCompRowBytes = SC * 2;              // a companion bf16 row segment
    static constexpr int kCompStages = kStages * kRowBytes / kCompRowBytes;
    static_assert(kLaneBytes == 16 || kLaneBytes == 8, "W4 lane width");
    static_assert(kW4Group % kLaneCols == 0, "a lane's columns lie in one scale group");
};

// cp.async of N (8 or 16) bytes; 8 bytes only exists in the L1-allocating (.ca) form
template <int N>
__device__ __forceinline__ void cp_async_n(void* smem_dst, const void* gsrc, bool pred) {
    if constexpr (N == 16) {
        cp_async16(smem_dst, gsrc, pred);
    } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
                     "@p cp.async.ca.shared.global [%0], [%1], 8;\n\t}" ::"r"(smem_u32(smem_dst)),
                     "l"(gsrc), "r"((int)pred)
                     : "memory");
    }
}

__device__ __forceinline__ float half_bits_to_f(uint16_t h) { return __half2float(__ushort_as_half(h)); }
// paired fp32 add of a constant: {w.x, w.y} += {c, c}
__device__ __forceinline__ void fadd2_const(float2& w, float c) {
    unsigned long long r, wa, ca;
    asm("mov.b64 %0, {%1, %2};" : "=l"(wa) : "f"(w.x), "f"(w.y));
    asm("mov.b64 %0, {%1, %1};" : "=l"(ca) : "f"(c));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(wa), "l"(ca));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(w.x), "=f"(w.y) : "l"(r));
}

// Shared memory: [ring 8 warps x 4 stages x 512 B | selection staging (aliased)] [row list + values]
// [misc] [row scales: 8 fp16 per kept row].  The partial sums (8 warps x 1024 fp32) alias the ring
// and the staging at the end.
static_assert((size_t)kGemvWarps * 8192 <= (size_t)kGemvWarps * kWarpRingBytes, "W4 ring size");
template <int SC>
__host__ __device__ constexpr size_t w4_region_bytes(int d_in) {
    return gemv_x_bytes(1, GEMV_SELECT, d_in) > (size_t)kGemvWarps * SC * 4 ? gemv_x_bytes(1, GEMV_SELECT, d_in)
                                                                           : (size_t)kGemvWarps * SC * 4;
}
// the whole plan: region, row list + values, misc, the fp16 scales and fp32 b = v s per kept row
template <int SC>
__host__ __device__ constexpr size_t w4_smem_bytes(int d_in, int list_cap) {
    return w4_region_bytes<SC>(d_in) + (size_t)list_cap * 8 + kGemvMisc * 4 + (size_t)list_cap * 2 * W4Cfg<SC>::kGroups +
           (size_t)list_cap * 4 * W4Cfg<SC>::kGroups + 16;
}

// (x & m) | c in one LOP3 (the compiler splits it when both are immediates)
__device__ __forceinline__ uint32_t and_or(uint32_t x, uint32_t m, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(x), "r"(m), "r"(c));
    return d;
}

// 16 + q as fp32 from a byte whose bits 3-6 hold q and bit 7 is set: bytes {0, 0, 0x80 | q << 3, 0x41}
// (2^4 has its mantissa LSB at bit 19, so q lands on weight 1)
template <int BB>
__device__ __forceinline__ float w4_f16q(uint32_t pre) {
    return __uint_as_float(__byte_perm(pre, 0x41u, 0x4055u + 0x100u * BB));
}

// Batch-1 finalisation of NV consecutive 256-column slices (vs0 .. vs0 + nv - 1) by one CTA: the
// same arithmetic and outputs as NV calls of gemv_epilogue<1>, with every accumulator load issued
// before any result is used (one L2 round trip instead of NV) and one barrier pair for the RMS
// partials.  sred: NV * 8 floats.
template <int NV>
__device__ void gemv_epilogue_b1_multi(const GemvArgs& a, int vs0, int nv, float* sred) {
    const int c = threadIdx.x, lane = c & 31, wid = c >> 5;
    float v[NV];
    int idx[NV];
    bool has[NV];
    const bool silu = a.epi == EPI_SILU;
    // pass 1: every accumulator (and bias / residual) load issued, predicated, none used yet
    unsigned long long r0[NV], r1[NV];
    float add[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int slice = vs0 + j, base = slice * kSliceCols;
        int o0;
        if (silu) {   // slice = 2 gate|up blocks of 128 columns (64 gate, then the matching 64 up)
            const int blk = c / kGuBlock, q = c % kGuBlock;
            o0 = base + blk * 2 * kGuBlock + q;
            has[j] = j < nv && c < 2 * kGuBlock && o0 < a.d_out;
            idx[j] = slice * 2 * kGuBlock + blk * kGuBlock + q;
        } else {
            o0 = base + c;
            has[j] = j < nv && o0 < a.d_out;
            idx[j] = o0;
        }
        r0[j] = has[j] ? __ldcg(a.acc + o0) : 0ull;
        r1[j] = has[j] && silu ? __ldcg(a.acc + o0 + kGuBlock) : 0ull;
        float t = 0.f;
        if (has[j] && !silu && a.bias) t = bf16f(a.bias[o0]);
        add[j] = t;
        v[j] = has[j] && !silu && a.res ? a.res[o0] : 0.f;
    }
    // pass 2: re-zero the accumulators, finalise
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        if (!has[j]) {
            v[j] = 0.f;
            continue;
        }
        const int o0 = silu ? (vs0 + j) * kSliceCols + (c / kGuBlock) * 2 * kGuBlock + c % kGuBlock : idx[j];
        a.acc[o0] = 0ull;
        if (silu) {
            a.acc[o0 + kGuBlock] = 0ull;
            const float g = fix_to_f(r0[j]), u = fix_to_f(r1[j]);
            v[j] = g / (1.0f + expf(-g)) * u;
        } else {
            float y = fix_to_f(r0[j]);
            if (a.bias) y += add[j];
            if (a.res) y = v[j] + y;
            v[j] = y;
        }
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        if (!has[j]) continue;
        a.out[idx[j]] = v[j];
        if (a.out_host) a.out_host[idx[j]] = v[j];
    }
    if (a.out_sel.hist) {   // hist_push of every value, the NV slot atomics in flight together
        uint32_t slot[NV], key[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            slot[j] = 0xffffffffu;
            key[j] = key_of(v[j]);
            if (!has[j]) continue;
            const uint32_t k16 = key[j] >> 15;
            const unsigned am = __activemask();
            const unsigned peers = __match_any_sync(am, k16 >> 8);
            if (lane == __ffs(peers) - 1) red_add_u32(a.out_sel.hist + sel_coarse_idx(k16 >> 8), __popc(peers));
            slot[j] = atomicAdd(a.out_sel.hist + sel_fine_idx(k16), 1u);
        }
#pragma unroll
        for (int j = 0; j < NV; ++j)
            if (slot[j] < (uint32_t)kPoolCap)
                a.out_sel.pool[sel_pool_idx(key[j] >> 15, slot[j])] = make_uint2(key[j], (uint32_t)idx[j]);
    }
    if (a.out_ssq) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const float w = slice_ssq_warp(v[j]);
            if (lane == 0) sred[j * 8 + wid] = w;
        }
        __syncthreads();
        if (c < nv) a.out_ssq[vs0 + c] = slice_ssq_combine(sred + c * 8);
    }
}

template <int SC>
__global__ void __launch_bounds__(kGemvThreads, 2) gemv_w4_select_kernel(const GemvArgs a, const uint8_t* __restrict__ Wq,
                                                                        const uint16_t* __restrict__ S) {
    using C = W4Cfg<SC>;
    extern __shared__ __align__(128) unsigned char smem[];
    // blockIdx.y < n_splits2: companion CTAs streaming dense bf16 rows [c_lo, c_lo + c_n) of W2
    // (ld = d_out) against x2 into the same accumulators (the residual adapter beside down)
    const int slice = blockIdx.x, split = (int)blockIdx.y - a.n_splits2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool comp = split < 0;
    int c_lo = 0, c_n = 0;
    if (comp) {
        const int rng = (a.d2 + a.n_splits2 - 1) / a.n_splits2;
        c_lo = min(a.d2, (int)blockIdx.y * rng);
        c_n = min(a.d2, c_lo + rng) - c_lo;
    }
    const size_t rb = w4_region_bytes<SC>(a.d_in);
    int* lrow = reinterpret_cast<int*>(smem + rb);                                 // [cap]
    float* lval = reinterpret_cast<float*>(lrow + a.list_cap);                     // [cap]
    int* misc = reinterpret_cast<int*>(lval + a.list_cap);                         // [kGemvMisc]
    uint16_t* lsc = reinterpret_cast<uint16_t*>(misc + kGemvMisc);                 // [cap][C::kGroups] fp16 scales
    float* lb = reinterpret_cast<float*>(lsc + (size_t)a.list_cap * C::kGroups);     // [cap][C::kGroups] b = v s
    const int ngroups = a.d_out / kW4Group;

    const int colb = slice * C::kSliceCols + C::kLaneCols * lane;
    const bool lane_on = colb < a.d_out;
    // companion ring: per warp C::kCompStages bf16 row segments (lane l: the 2 C::kLaneCols bytes of its columns)
    unsigned char* cchunk = smem + (size_t)warp * C::kStages * C::kRowBytes + 2 * C::kLaneCols * lane;
    const int c_my = c_n > warp ? (c_n - warp + kGemvWarps - 1) / kGemvWarps : 0;
    auto comp_issue = [&](int m) {
        if (m < c_my) {
            const uint16_t* src = a.W2 + (size_t)(c_lo + warp + kGemvWarps * m) * a.d_out + colb;
            unsigned char* dst = cchunk + (size_t)(m % C::kCompStages) * C::kCompRowBytes;
#pragma unroll
            for (int q = 0; q < C::kLaneCols / 8; ++q) cp_async16(dst + 16 * q, src + 8 * q, lane_on);
        }
        cp_async_commit();
    };
    if (comp) {   // the first stages do not depend on the previous kernel
#pragma unroll
        for (int m = 0; m < C::kCompStages; ++m) comp_issue(m);
    }
    int sel_guess = 0;
    if (!comp && threadIdx.x == 0) sel_guess = (int)__ldcg(a.sel.hist + kSelHistTotal);
    tl_stamp(a.tl, 0);
    pdl_wait();
    pdl_trigger();
    tl_stamp(a.tl, 1);
    if (a.zero_hist) {   // (decoder layer) a histogram / accumulators whose consumer has completed
        const int nct = gridDim.x * gridDim.y, cta = blockIdx.y * gridDim.x + blockIdx.x;
        for (int i = cta * kGemvThreads + threadIdx.x; i < a.zero_words; i += nct * kGemvThreads) a.zero_hist[i] = 0u;
    }
    if (a.zero_acc) {
        const int nct = gridDim.x * gridDim.y, cta = blockIdx.y * gridDim.x + blockIdx.x;
        for (int i = cta * kGemvThreads + threadIdx.x; i < a.zero_acc_words; i += nct * kGemvThreads) a.zero_acc[i] = 0ull;
    }
    float2 acc[C::kLaneCols / 2];
#pragma unroll
    for (int j = 0; j < C::kLaneCols / 2; ++j) acc[j] = make_float2(0.f, 0.f);
    float bsum = 0.f;
    int n_list;
    if (comp) {
        n_list = c_n;
        for (int t = threadIdx.x; t < c_n; t += kGemvThreads) lval[t] = __ldcg(a.x2 + c_lo + t);
        __syncthreads();
        tl_stamp(a.tl, 2);
        for (int m = 0; m < c_my; ++m) {
            cp_async_wait<C::kCompStages - 1>();
            const unsigned char* src = cchunk + (size_t)(m % C::kCompStages) * C::kCompRowBytes;
            const float v = lval[warp + kGemvWarps * m];
#pragma unroll
            for (int q = 0; q < C::kLaneCols / 8; ++q) {
                const uint4 w = lds128(src + 16 * q);
                ffma2(acc[4 * q + 0], bf16lo(w.x), bf16hi(w.x), v);
                ffma2(acc[4 * q + 1], bf16lo(w.y), bf16hi(w.y), v);
                ffma2(acc[4 * q + 2], bf16lo(w.z), bf16hi(w.z), v);
                ffma2(acc[4 * q + 3], bf16lo(w.w), bf16hi(w.w), v);
            }
            comp_issue(m + C::kCompStages);
        }
    } else {
    n_list = select_rows(a, smem, lrow, lval, misc, split, a.n_splits, sel_guess);
    // the kept rows' 8 group scales of this slice (16 bytes), once, before the stream
    const int g0 = slice * C::kGroups;
    const int ng = min(C::kGroups, ngroups - g0);
    for (int t = threadIdx.x; t < n_list; t += kGemvThreads) {
        const uint16_t* src = S + (size_t)lrow[t] * ngroups + g0;
        if (ng == C::kGroups && (reinterpret_cast<uintptr_t>(src) & (2 * C::kGroups - 1)) == 0) {
            cp_async_n<2 * C::kGroups>(lsc + (size_t)t * C::kGroups, src, true);
        } else {
            uint16_t* d = lsc + (size_t)t * C::kGroups;
            for (int q = 0; q < C::kGroups; ++q) d[q] = q < ng ? src[q] : (uint16_t)0;
        }
    }
    // the first stages of the stream go out with the scales (the row list is complete and the
    // staged selection data the ring aliases is dead)
    unsigned char* mychunk = smem + (size_t)warp * C::kStages * C::kRowBytes + C::kLaneBytes * lane;
    const int n_my = n_list > warp ? (n_list - warp + kGemvWarps - 1) / kGemvWarps : 0;
    const uint8_t* wl = Wq + colb / 2;
    const size_t ldq = (size_t)a.d_out / 2;
    auto issue = [&](int m) {
        if (m < n_my) cp_async_n<C::kLaneBytes>(mychunk + (size_t)(m % C::kStages) * C::kRowBytes,
                                               wl + (size_t)lrow[warp + kGemvWarps * m] * ldq, lane_on);
        cp_async_commit();
    };
    cp_async_commit();   // the scales: the group before the stream's first C::kStages groups
#pragma unroll
    for (int m = 0; m < C::kStages; ++m) issue(m);
    cp_async_wait<C::kStages>();
    __syncthreads();
    // b[t][g] = (x_j s_rms) S[j][g0 + g] for each kept row, once per CTA (the stream reads one float)
    {
        const float sel_scale = reinterpret_cast<const float*>(misc)[4];
        for (int t = threadIdx.x; t < n_list; t += kGemvThreads) {
            const float v = lval[t] * sel_scale;
#pragma unroll
            for (int q = 0; q < C::kGroups; ++q) lb[(size_t)t * C::kGroups + q] = v * half_bits_to_f(lsc[(size_t)t * C::kGroups + q]);
        }
    }
    __syncthreads();
    tl_stamp(a.tl, 2);

    // warp w takes list entries w + 8 m; lane l owns columns 32 l .. 32 l + 31 of the slice (one
    // scale group: l / 4) and copies exactly those 16 bytes of each row (no cross-lane dependency);
    // the first C::kStages rows are in flight since the prologue
    const float* lbf = lb + (C::kLaneCols * lane) / kW4Group;   // the lane's scale group
    // sum_j b_j (16 + q_j) accumulated, sum_j b_j beside it: y = acc - 24 sum_j b_j at the end
    // (16 + q is one byte permute of a pre-shifted code byte; the offset costs ~3 bits of the fp32
    // sums, far inside the 1e-5 parity bound)
    const uint32_t hibit = 0x80808080u, nmask = 0x78787878u;
    for (int m = 0; m < n_my; ++m) {
        cp_async_wait<C::kStages - 1>();
        const int pos = warp + kGemvWarps * m;
        uint32_t qw[C::kLaneBytes / 4];
        if constexpr (C::kLaneBytes == 16) {
            const uint4 q4 = lds128(mychunk + (size_t)(m % C::kStages) * C::kRowBytes);
            qw[0] = q4.x;
            qw[1] = q4.y;
            qw[2] = q4.z;
            qw[3] = q4.w;
        } else {
            const uint2 q2 = *reinterpret_cast<const uint2*>(mychunk + (size_t)(m % C::kStages) * C::kRowBytes);
            qw[0] = q2.x;
            qw[1] = q2.y;
        }
        const float b = lbf[(size_t)pos * C::kGroups];
        bsum += b;
#pragma unroll
        for (int wi = 0; wi < C::kLaneBytes / 4; ++wi) {
            const uint32_t lo = and_or(qw[wi] << 3, nmask, hibit);   // low nibbles at bits 3-6
            const uint32_t hi = and_or(qw[wi] >> 1, nmask, hibit);   // high nibbles at bits 3-6
            ffma2(acc[4 * wi + 0], w4_f16q<0>(lo), w4_f16q<0>(hi), b);
            ffma2(acc[4 * wi + 1], w4_f16q<1>(lo), w4_f16q<1>(hi), b);
            ffma2(acc[4 * wi + 2], w4_f16q<2>(lo), w4_f16q<2>(hi), b);
            ffma2(acc[4 * wi + 3], w4_f16q<3>(lo), w4_f16q<3>(hi), b);
        }
        issue(m + C::kStages);
    }
    }   // SELECT split
    cp_async_wait<0>();
    __syncthreads();
    tl_stamp(a.tl, 3);
    {
        const float corr = -24.0f * bsum;
#pragma unroll
        for (int j = 0; j < C::kLaneCols / 2; ++j) fadd2_const(acc[j], corr);
    }
    // fixed-order sum of the 8 warps' partials, one fixed-point red per column (4 per thread)
    float* part = reinterpret_cast<float*>(smem);   // [8][1024]
    {
        float* p = part + (size_t)warp * C::kSliceCols + C::kLaneCols * lane;
#pragma unroll
        for (int j = 0; j < C::kLaneCols / 4; ++j)
            reinterpret_cast<float4*>(p)[j] = make_float4(acc[2 * j].x, acc[2 * j].y, acc[2 * j + 1].x, acc[2 * j + 1].y);
    }
    __syncthreads();
    if (n_list > 0) {
        for (int c = threadIdx.x; c < C::kSliceCols; c += kGemvThreads) {
            const int o = slice * C::kSliceCols + c;
            if (o >= a.d_out) break;
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < kGemvWarps; ++w) s += part[(size_t)w * C::kSliceCols + c];
            red_fix(a.acc + o, s, a.err);
        }
    }
    if (a.epi == EPI_NONE) {   // the consumer kernel reads the accumulators (QKV -> attention)
        tl_stamp(a.tl, 4);
        return;
    }
    __syncthreads();
    if (threadIdx.x == 0) misc[0] = atom_add_acq_rel_gpu(a.tickets + slice, 1u) == gridDim.y - 1u;
    tl_stamp(a.tl, 12);
    __syncthreads();
    if (!misc[0]) {
        tl_stamp(a.tl, 4);
        return;
    }
    if (threadIdx.x == 0) a.tickets[slice] = 0u;
    tl_stamp(a.tl, 13);
    // the last split of the slice finalises its 1024 columns as four 256-column slices of the bf16
    // kernel's epilogue (bias / residual / SiLU(g) u, accumulators re-zeroed, and at batch 1 the next
    // site's histogram and RMS partials): the same output layout and selection data
    constexpr int kNv = C::kSliceCols / kSliceCols;
    const int vs0 = slice * kNv;
    const int nv = min(kNv, (a.d_out - vs0 * kSliceCols + kSliceCols - 1) / kSliceCols);
    gemv_epilogue_b1_multi<kNv>(a, vs0, nv, reinterpret_cast<float*>(misc + 16));
    tl_stamp(a.tl, 4);
}

// Quantisation (offline): per row j and group g, scale = RNE_fp16(max_o |w| / 7) (fp32 divide);
// q = clamp(rint(w / scale_fp32) + 8, 0, 15), fp32 divide; scale 0 -> q = 8.
__global__ void quantize_w4_kernel(const uint16_t* __restrict__ W, int d_in, int d_out, uint8_t* __restrict__ Wq,
                                   uint16_t* __restrict__ S) {
    const int ngroups = d_out / kW4Group;
    const int gid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);   // one warp per (row, group)
    const int lane = threadIdx.x & 31;
    if (gid >= d_in * ngroups) return;
    const int j = gid / ngroups, g = gid % ngroups;
    const uint16_t* src = W + (size_t)j * d_out + (size_t)g * kW4Group;
    float v[4];
    float amax = 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        v[t] = bf16f(src[4 * lane + t]);
        amax = fmaxf(amax, fabsf(v[t]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const uint16_t sh = __half_as_ushort(__float2half_rn(__fdiv_rn(amax, 7.0f)));
    const float s = half_bits_to_f(sh);
    uint32_t code[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        int q = 8;
        if (s > 0.f) q = max(0, min(15, (int)rintf(__fdiv_rn(v[t], s)) + 8));
        code[t] = (uint32_t)q;
    }
    uint8_t* dst = Wq + (size_t)j * (d_out / 2) + (size_t)g * (kW4Group / 2) + 2 * lane;
    dst[0] = (uint8_t)(code[0] | (code[1] << 4));
    dst[1] = (uint8_t)(code[2] | (code[3] << 4));
    if (lane == 0) S[(size_t)j * ngroups + g] = sh;
}

}  // namespace larosa
