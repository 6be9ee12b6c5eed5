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
constexpr int kW4SliceCols = 1024;            // columns per CTA: a kept row's slice segment is 512 B
constexpr int kW4Stages = 16;                 // rows in flight per warp (one 512-byte row per stage): 64 KB per CTA
constexpr int kW4RowBytes = kW4SliceCols / 2;

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
static_assert((size_t)kGemvWarps * kW4Stages * kW4RowBytes <= (size_t)kGemvWarps * kWarpRingBytes, "W4 ring size");
__host__ __device__ constexpr size_t w4_region_bytes(int d_in) {
    return gemv_x_bytes(1, GEMV_SELECT, d_in) > (size_t)kGemvWarps * kW4SliceCols * 4 ? gemv_x_bytes(1, GEMV_SELECT, d_in)
                                                                                      : (size_t)kGemvWarps * kW4SliceCols * 4;
}

__global__ void __launch_bounds__(kGemvThreads, 2) gemv_w4_select_kernel(const GemvArgs a, const uint8_t* __restrict__ Wq,
                                                                        const uint16_t* __restrict__ S) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int slice = blockIdx.x, split = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t rb = w4_region_bytes(a.d_in);
    int* lrow = reinterpret_cast<int*>(smem + rb);                                 // [cap]
    float* lval = reinterpret_cast<float*>(lrow + a.list_cap);                     // [cap]
    int* misc = reinterpret_cast<int*>(lval + a.list_cap);                         // [kGemvMisc]
    uint4* lsc = reinterpret_cast<uint4*>(misc + kGemvMisc);                       // [cap] 8 fp16 scales
    const int ngroups = a.d_out / kW4Group;

    int sel_guess = 0;
    if (threadIdx.x == 0) sel_guess = (int)__ldcg(a.sel.hist + kSelHistTotal);
    pdl_wait();
    pdl_trigger();
    if (a.zero_hist) {   // (decoder layer) a histogram / accumulators whose consumer has completed
        const int nct = gridDim.x * gridDim.y, cta = blockIdx.y * gridDim.x + blockIdx.x;
        for (int i = cta * kGemvThreads + threadIdx.x; i < a.zero_words; i += nct * kGemvThreads) a.zero_hist[i] = 0u;
    }
    if (a.zero_acc) {
        const int nct = gridDim.x * gridDim.y, cta = blockIdx.y * gridDim.x + blockIdx.x;
        for (int i = cta * kGemvThreads + threadIdx.x; i < a.zero_acc_words; i += nct * kGemvThreads) a.zero_acc[i] = 0ull;
    }
    const int n_list = select_rows(a, smem, lrow, lval, misc, split, a.n_splits, sel_guess);
    // the kept rows' 8 group scales of this slice (16 bytes), once, before the stream
    const int g0 = slice * (kW4SliceCols / kW4Group);
    const int ng = min(kW4SliceCols / kW4Group, ngroups - g0);
    for (int t = threadIdx.x; t < n_list; t += kGemvThreads) {
        const uint16_t* src = S + (size_t)lrow[t] * ngroups + g0;
        if (ng == 8 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            cp_async16(lsc + t, src, true);
        } else {
            uint16_t* d = reinterpret_cast<uint16_t*>(lsc + t);
            for (int q = 0; q < 8; ++q) d[q] = q < ng ? src[q] : (uint16_t)0;
        }
    }
    cp_async_commit();
    const float sel_scale = reinterpret_cast<const float*>(misc)[4];
    cp_async_wait<0>();
    __syncthreads();

    // warp w takes list entries w + 8 m; lane l owns columns 32 l .. 32 l + 31 of the slice and
    // copies exactly those 16 bytes of each row (no cross-lane dependency in the ring)
    const int n_my = n_list > warp ? (n_list - warp + kGemvWarps - 1) / kGemvWarps : 0;
    const int colb = slice * kW4SliceCols + 32 * lane;
    const bool lane_on = colb < a.d_out;
    unsigned char* mychunk = smem + (size_t)warp * kW4Stages * kW4RowBytes + 16 * lane;
    const uint8_t* wl = Wq + colb / 2;
    const size_t ldq = (size_t)a.d_out / 2;
    auto issue = [&](int m) {
        if (m < n_my) cp_async16(mychunk + (size_t)(m % kW4Stages) * kW4RowBytes,
                                 wl + (size_t)lrow[warp + kGemvWarps * m] * ldq, lane_on);
        cp_async_commit();
    };
#pragma unroll
    for (int m = 0; m < kW4Stages; ++m) issue(m);
    float2 acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = make_float2(0.f, 0.f);
    const int gsel = lane >> 2;   // the lane's 32 columns lie in group (32 lane) / 128 of the slice
    for (int m = 0; m < n_my; ++m) {
        cp_async_wait<kW4Stages - 1>();
        const int pos = warp + kGemvWarps * m;
        const uint4 q4 = lds128(mychunk + (size_t)(m % kW4Stages) * kW4RowBytes);
        const uint4 sc = lsc[pos];
        const int gw = gsel >> 1;
        const uint32_t sw = gw == 0 ? sc.x : (gw == 1 ? sc.y : (gw == 2 ? sc.z : sc.w));
        const float s = half_bits_to_f((uint16_t)((gsel & 1) ? (sw >> 16) : (sw & 0xffffu)));
        const float v = lval[pos] * sel_scale * s;
        const uint32_t qw[4] = {q4.x, q4.y, q4.z, q4.w};
        // nibbles -> fp32 with one byte permute each: 0x4B0000nn is 2^23 + nn, so
        // (2^23 + nn) - (2^23 + 8) = nn - 8 exactly; paired subtract + paired FMA
#pragma unroll
        for (int wi = 0; wi < 4; ++wi) {
            const uint32_t lo = qw[wi] & 0x0F0F0F0Fu, hi = (qw[wi] >> 4) & 0x0F0F0F0Fu;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                float2 w = make_float2(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7540u + b)),
                                       __uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7540u + b)));
                fadd2_const(w, -8388616.0f);
                ffma2(acc[4 * wi + b], w.x, w.y, v);
            }
        }
        issue(m + kW4Stages);
    }
    cp_async_wait<0>();
    __syncthreads();
    // fixed-order sum of the 8 warps' partials, one fixed-point red per column (4 per thread)
    float* part = reinterpret_cast<float*>(smem);   // [8][1024]
    {
        float* p = part + (size_t)warp * kW4SliceCols + 32 * lane;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            reinterpret_cast<float4*>(p)[j] = make_float4(acc[2 * j].x, acc[2 * j].y, acc[2 * j + 1].x, acc[2 * j + 1].y);
    }
    __syncthreads();
    if (n_list > 0) {
        for (int c = threadIdx.x; c < kW4SliceCols; c += kGemvThreads) {
            const int o = slice * kW4SliceCols + c;
            if (o >= a.d_out) break;
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < kGemvWarps; ++w) s += part[(size_t)w * kW4SliceCols + c];
            red_fix(a.acc + o, s, a.err);
        }
    }
    if (a.epi == EPI_NONE) return;    // the consumer kernel reads the accumulators (QKV -> attention)
    __syncthreads();
    if (threadIdx.x == 0) misc[0] = atom_add_acq_rel_gpu(a.tickets + slice, 1u) == gridDim.y - 1u;
    __syncthreads();
    if (!misc[0]) return;
    if (threadIdx.x == 0) a.tickets[slice] = 0u;
    // the last split of the slice finalises its 1024 columns as four 256-column slices of the bf16
    // kernel's epilogue (bias / residual / SiLU(g) u, accumulators re-zeroed, and at batch 1 the next
    // site's histogram and RMS partials): the same output layout and selection data
    for (int j = 0; j < kW4SliceCols / kSliceCols; ++j) {
        const int vs = slice * (kW4SliceCols / kSliceCols) + j;
        if (vs * kSliceCols >= a.d_out) break;
        gemv_epilogue<1>(a, vs, reinterpret_cast<float*>(misc + 16));
    }
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
