// gemv.cuh — sparse GEMV over the kept rows of a column-major weight (eq. after_merge,
// PAPER.md:407-410; kernel recipe P:414: column-major storage, selective loads of the kept
// columns).
//
//   acc[b][o] += fix( sum_{r in rows} val(r, b) * W[row(r)][o] )        (o in [0, d_out))
//
// The kernel only streams and accumulates; it has no tail.  Partial sums are added into
// 64-bit fixed-point accumulators (32 fractional bits) with red.global.add.u64: integer
// addition is associative, so the result is bit-identical whatever order the CTAs finish
// in (deterministic without a fixed reduction tree), and no CTA waits for another.  The
// consumer of y (the next kernel: Top-K, attention, finalize) converts acc -> fp32, applies
// the epilogue (bias / residual / RoPE / SiLU*up) and re-zeroes the accumulators.
// Fixed-point error: <= 2^-33 absolute per partial (|y| must stay < 2^31).
//
// Decomposition (B200: 148 SMs): grid = (column slices of 256, n_splits) with 8 warps per
// CTA, ~2 CTAs per SM.  CTA (slice, s) owns the s-th contiguous chunk of the kept-row list;
// warp w takes every 8th row of it.  Each kept row's 512-byte segment (contiguous in the
// [d_in][d_out] layout) is one coalesced warp-wide cp.async (LDGSTS, 16 B per lane) into the
// warp's private 4-stage ring; a lane later reads back exactly the 16 bytes it copied, so
// the pipeline needs no barrier, only the lane's own cp.async groups.  (Measured on B200:
// the TMA engine retires about one bulk copy per ~50 cycles per SM, so 0.5-2 KB gathered
// row segments cap cp.async.bulk at 15-38 GB/s per SM, below the 44 GB/s/SM that 6.5 TB/s
// needs; per-thread cp.async has no such cap.)  Math: bf16 pairs widen with one ALU op per
// value and accumulate with paired fp32 FMAs (FFMA2).  The 8 warps' partials are summed in
// shared memory in fixed order before the single red per column.
#pragma once
#include "common.cuh"

namespace larosa {

constexpr int kGuBlock = 64;          // == LAROSA_GU_BLOCK
constexpr int kSliceCols = 256;       // columns per CTA (8 per lane)
constexpr int kGemvWarps = 8;
constexpr int kStageRows = 4;         // rows per stage (one 512-byte warp copy each)
constexpr int kStages = 4;            // ring depth per warp
constexpr int kWarpRingBytes = kStages * kStageRows * kSliceCols * 2;   // 8 KB
constexpr double kFixScale = 4294967296.0;                              // 2^32

enum GemvMode : int {
    GEMV_LIST = 0,     // kept rows given as a list (rows[], vals) -- split by list position
    GEMV_THRESH = 1,   // kept rows selected in-kernel from x by the Top-K rule (thresh.cuh)
    GEMV_DENSE = 2,    // every row, value x (+ vacc) -- the residual adapter
};

// the per-token Top-K rule produced by thresh.cuh: keep row i iff
// key_i > tk or (key_i == tk and i <= ti), key = bits(|x_i|); value x_i * scale
struct ThreshOut {
    uint32_t tk;       // key threshold
    int32_t ti;        // index threshold for key == tk (inclusive)
    float scale;       // RMS scale (1 if no RMS)
    int32_t pad;
};

struct GemvArgs {
    const uint16_t* W;
    int64_t ld;
    int d_out;
    int mode;              // GemvMode
    // GEMV_LIST
    const int32_t* rows;   // kept row indices (ascending)
    int nrows;             // row count when nrows_dev == nullptr
    const int* nrows_dev;  // device row count (batch > 1 union), or nullptr
    const float* vals;     // val(r, b) = vals[r * vs_r + b * vs_b]
    int64_t vs_r, vs_b;
    // GEMV_THRESH / GEMV_DENSE: input x [batch][ldx] over rows [0, d_in)
    const float* x;
    int64_t ldx;
    int d_in;
    const ThreshOut* thr;              // THRESH: per-token rule + RMS scale
    const unsigned long long* vacc;    // DENSE (optional): val += fix^-1(vacc[b * vacc_ld + r])
    int64_t vacc_ld;
    int batch;             // real tokens (<= template BP)
    int n_splits;
    int list_cap;          // rows of the per-CTA shared list (host-checked >= rows per split)
    unsigned long long* acc;          // [batch][acc_ld] fixed-point output accumulators
    int64_t acc_ld;
};

// ring (aliased by the warp partials at the end) + the CTA's row list [cap] and values [cap][bp]
__host__ __device__ constexpr size_t gemv_ring_bytes(int bp) {
    return (size_t)kGemvWarps * kWarpRingBytes > (size_t)kGemvWarps * bp * kSliceCols * 4
               ? (size_t)kGemvWarps * kWarpRingBytes
               : (size_t)kGemvWarps * bp * kSliceCols * 4;
}
__host__ __device__ constexpr size_t gemv_smem_bytes(int bp, int list_cap) {
    return gemv_ring_bytes(bp) + (size_t)list_cap * (4 + 4 * (size_t)bp) + 128;
}

__device__ __forceinline__ float fix_to_f(unsigned long long a) {
    return (float)((double)(long long)a * (1.0 / kFixScale));
}
__device__ __forceinline__ unsigned long long f_to_fix(float v) {
    return (unsigned long long)__float2ll_rn(v * 4294967296.0f);
}
__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// cp.async (LDGSTS): 16 bytes global -> shared, L1 bypass (.cg)
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool pred) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
        "@p cp.async.cg.shared.global [%0], [%1], 16;\n\t}" ::"r"(smem_u32(smem_dst)),
        "l"(gsrc), "r"((int)pred)
        : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// paired fp32 FMA (FFMA2): {a.x, a.y} = {w0, w1} * {v, v} + {a.x, a.y}
__device__ __forceinline__ void ffma2(float2& a, float w0, float w1, float v) {
    unsigned long long r, wa, va, aa;
    asm("mov.b64 %0, {%1, %2};" : "=l"(wa) : "f"(w0), "f"(w1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(va) : "f"(v));
    asm("mov.b64 %0, {%1, %2};" : "=l"(aa) : "f"(a.x), "f"(a.y));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(wa), "l"(va), "l"(aa));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
}

template <int BP>
__global__ void __launch_bounds__(kGemvWarps * 32) gemv_kernel(const GemvArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int slice = blockIdx.x, split = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int* lrow = reinterpret_cast<int*>(smem + gemv_ring_bytes(BP));           // [cap]
    float* lval = reinterpret_cast<float*>(lrow + a.list_cap);                // [cap][BP]
    int* s_cnt = reinterpret_cast<int*>(lval + (size_t)a.list_cap * BP);      // [2][8] + [1]

    pdl_wait();       // the row source comes from the previous kernel
    pdl_trigger();

    // ---- 1. this CTA's row list in shared memory (ascending) ------------------------------
    int n_list = 0;
    if (a.mode == GEMV_LIST) {
        const int nrows = a.nrows_dev ? *a.nrows_dev : a.nrows;
        const int rps = (nrows + a.n_splits - 1) / a.n_splits;
        const int r_begin = min(nrows, split * rps);
        n_list = min(nrows, r_begin + rps) - r_begin;
        for (int t = threadIdx.x; t < n_list; t += kGemvWarps * 32) {
            const int r = r_begin + t;
            lrow[t] = __ldg(a.rows + r);
#pragma unroll
            for (int b = 0; b < BP; ++b)
                lval[t * BP + b] = b < a.batch ? __ldg(a.vals + (size_t)r * a.vs_r + (size_t)b * a.vs_b) : 0.f;
        }
    } else {
        // input range of this split; keep a row if any token keeps it (THRESH rule) or always
        const int rng = (a.d_in + a.n_splits - 1) / a.n_splits;
        const int lo = min(a.d_in, split * rng), hi = min(a.d_in, lo + rng);
        const ThreshOut* thr = a.thr;
        int base = 0;
        for (int r0 = lo, rnd = 0; r0 < hi; r0 += kGemvWarps * 32, ++rnd) {
            const int i = r0 + (int)threadIdx.x;
            float v[BP];
            bool any = false;
#pragma unroll
            for (int b = 0; b < BP; ++b) {
                float x = 0.f;
                bool keep = false;
                if (i < hi && b < a.batch) {
                    x = a.x[(size_t)b * a.ldx + i];
                    if (a.vacc) x += fix_to_f(a.vacc[(size_t)b * a.vacc_ld + i]);
                    if (a.mode == GEMV_DENSE) {
                        keep = true;
                    } else {
                        const uint32_t key = __float_as_uint(x) & 0x7fffffffu;
                        keep = key > thr[b].tk || (key == thr[b].tk && i <= thr[b].ti);
                        x *= thr[b].scale;
                    }
                }
                v[b] = keep ? x : 0.f;
                any |= keep;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, any);
            int* cnt = s_cnt + (rnd & 1) * 8;
            if (lane == 0) cnt[warp] = __popc(bal);
            __syncthreads();
            int before = 0, total = 0;
#pragma unroll
            for (int w = 0; w < kGemvWarps; ++w) {
                const int cw = cnt[w];
                before += w < warp ? cw : 0;
                total += cw;
            }
            if (any) {
                const int pos = base + before + __popc(bal & ((1u << lane) - 1u));
                lrow[pos] = i;
#pragma unroll
                for (int b = 0; b < BP; ++b) lval[pos * BP + b] = v[b];
            }
            base += total;
        }
        n_list = base;
    }
    __syncthreads();

    // my rows: list entries warp + 8*m, m in [0, n_my)
    const int n_my = n_list > warp ? (n_list - warp + kGemvWarps - 1) / kGemvWarps : 0;
    const int col0 = slice * kSliceCols + lane * 8;
    const bool lane_on = col0 < a.d_out;          // d_out % 8 == 0: a lane's chunk is all-in or all-out
    const int n_st = (n_my + kStageRows - 1) / kStageRows;
    unsigned char* mychunk = smem + (size_t)warp * kWarpRingBytes + lane * 16;
    const uint16_t* wcol = a.W + col0;

    // stage st covers my-rows [4 st, 4 st + 4)
    auto issue = [&](int st) {
        if (st < n_st) {
            unsigned char* dst = mychunk + (size_t)(st & (kStages - 1)) * (kStageRows * kSliceCols * 2);
#pragma unroll
            for (int g = 0; g < kStageRows; ++g) {
                const int m = st * kStageRows + g;
                const int row = m < n_my ? lrow[warp + kGemvWarps * m] : 0;
                cp_async16(dst + g * (kSliceCols * 2), wcol + (size_t)row * a.ld, lane_on && m < n_my);
            }
        }
        cp_async_commit();   // one (possibly empty) group per stage keeps the count uniform
    };
#pragma unroll
    for (int st = 0; st < kStages; ++st) issue(st);

    float2 acc[BP][4];
#pragma unroll
    for (int b = 0; b < BP; ++b)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[b][j] = make_float2(0.f, 0.f);

    for (int st = 0; st < n_st; ++st) {
        cp_async_wait<kStages - 1>();          // this lane's chunks of stage st have landed
        const unsigned char* src = mychunk + (size_t)(st & (kStages - 1)) * (kStageRows * kSliceCols * 2);
#pragma unroll
        for (int g = 0; g < kStageRows; ++g) {
            const int m = st * kStageRows + g;
            if (m >= n_my) break;                // short last stage (warp-uniform)
            const uint4 w = lds128(src + g * (kSliceCols * 2));
            const float w0 = bf16lo(w.x), w1 = bf16hi(w.x), w2 = bf16lo(w.y), w3 = bf16hi(w.y);
            const float w4 = bf16lo(w.z), w5 = bf16hi(w.z), w6 = bf16lo(w.w), w7 = bf16hi(w.w);
            const float* vrow = lval + (size_t)(warp + kGemvWarps * m) * BP;
#pragma unroll
            for (int b = 0; b < BP; ++b) {
                const float v = vrow[b];             // shared-memory broadcast
                ffma2(acc[b][0], w0, w1, v);
                ffma2(acc[b][1], w2, w3, v);
                ffma2(acc[b][2], w4, w5, v);
                ffma2(acc[b][3], w6, w7, v);
            }
        }
        issue(st + kStages);
    }
    cp_async_wait<0>();
    __syncthreads();   // every warp is done with its ring (the partials alias it)

    // fixed-order sum of the 8 warps' partials, then one fixed-point red per column
    float* part = reinterpret_cast<float*>(smem);   // [8][BP][256]
#pragma unroll
    for (int b = 0; b < BP; ++b) {
        float* p = part + ((size_t)warp * BP + b) * kSliceCols + lane * 8;
        reinterpret_cast<float4*>(p)[0] = make_float4(acc[b][0].x, acc[b][0].y, acc[b][1].x, acc[b][1].y);
        reinterpret_cast<float4*>(p)[1] = make_float4(acc[b][2].x, acc[b][2].y, acc[b][3].x, acc[b][3].y);
    }
    __syncthreads();
    const int c = threadIdx.x;                     // 256 threads <-> 256 columns
    const int o = slice * kSliceCols + c;
    if (o < a.d_out && n_list > 0) {
        for (int b = 0; b < a.batch; ++b) {
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < kGemvWarps; ++w) s += part[((size_t)w * BP + b) * kSliceCols + c];
            red_add_u64(a.acc + (size_t)b * a.acc_ld + o, f_to_fix(s));
        }
    }
}

}  // namespace larosa
