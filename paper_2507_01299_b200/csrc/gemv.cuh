// gemv.cuh — sparse GEMV over the kept rows of a column-major weight (eq. after_merge,
// PAPER.md:407-410; kernel recipe P:414: column-major storage, selective loads of the kept
// columns), with the site's Top-K selection fused into its prologue and the next site's
// inputs produced by its epilogue.
//
//   acc[b][o] += fix( sum_{r in rows} val(r, b) * W[row(r)][o] )        (o in [0, d_out))
//
// Streaming.  Partial sums are added into 64-bit fixed-point accumulators (32 fractional
// bits) with red.global.add.u64: integer addition is associative, so the result is
// bit-identical whatever order the CTAs finish in and no CTA waits for another.
// Fixed-point error: <= 2^-33 absolute per partial (|y| must stay < 2^31).
// Decomposition (B200: 148 SMs): grid = (column slices of 256, n_splits) with 8 warps per
// CTA, ~2 CTAs per SM.  CTA (slice, s) owns the s-th share of the kept-row list; warp w
// takes every 8th row of it.  Each kept row's 512-byte segment (contiguous in the
// [d_in][d_out] layout) is one coalesced warp-wide cp.async (LDGSTS, 16 B per lane) into the
// warp's private 4-stage ring; a lane later reads back exactly the 16 bytes it copied, so
// the pipeline needs no barrier, only the lane's own cp.async groups.  (Measured on B200:
// the TMA engine retires about one bulk copy per ~50 cycles per SM, so 0.5-2 KB gathered
// row segments cap cp.async.bulk at 15-38 GB/s per SM, below the 44 GB/s/SM that 6.5 TB/s
// needs; per-thread cp.async has no such cap.)  Math: bf16 pairs widen with one ALU op per
// value and accumulate with paired fp32 FMAs (FFMA2).  The 8 warps' partials are summed in
// shared memory in fixed order before the single red per column.
//
// Row sources (GemvMode):
//   LIST    kept rows given as (rows[], vals) — the standalone larosa_sparse_gemv;
//   THRESH  per-token selection rules (Tk, Ti, s) from the Top-K kernel (batch > 1);
//   DENSE   every input row (the residual adapter, the rotation);
//   SELECT  batch 1: every CTA derives the exact Top-K rule itself (S_k, lower
//           index wins ties) from the site's 4096-bin global histogram of the
//           key bits [30:19] (accumulated by the producer's epilogue) and the site vector x
//           staged in shared memory: the histogram suffix scan gives the bucket of the k-th
//           key; radix refinement over bits [18:7] and [6:0] of the staged x, then an index
//           tie-break, make it exact.  The CTA then takes an exactly balanced share of the
//           kept rows (block prefix count in index order).  No Top-K kernel, index list or
//           extra grid-wide dependency sits between two GEMVs.
// Epilogue (GemvEpi): the last split CTA of each column slice (ticket) converts the slice's
// accumulators to fp32, applies the site glue (bias / residual add / SiLU(g)*u), writes the
// next site's vector, re-zeroes the accumulators and, at batch 1, adds the values' key bins
// into the next site's histogram and writes the slice's sum of squares (for the RMS scale)
// — the next GEMV's SELECT prologue consumes exactly these.
#pragma once
#include "common.cuh"
#include "larosa.h"

namespace larosa {

constexpr int kGuBlock = 64;          // == LAROSA_GU_BLOCK
constexpr int kSliceCols = 256;       // columns per CTA (8 per lane)
constexpr int kGemvWarps = 8;
constexpr int kGemvThreads = kGemvWarps * 32;
constexpr int kStageRows = 4;         // rows per stage (one 512-byte warp copy each)
#ifndef LAROSA_GEMV_STAGES
#define LAROSA_GEMV_STAGES 4
#endif
constexpr int kStages = LAROSA_GEMV_STAGES;   // ring depth per warp
constexpr int kWarpRingBytes = kStages * kStageRows * kSliceCols * 2;   // 8 KB
constexpr double kFixScale = 4294967296.0;                              // 2^32
constexpr int kGemvMisc = 128;        // ints of scratch
constexpr int kPoolCap = 64;          // (key, index) entries kept per 16-bit histogram bucket

enum GemvMode : int { GEMV_LIST = 0, GEMV_THRESH = 1, GEMV_DENSE = 2, GEMV_SELECT = 3 };
enum GemvEpi : int { EPI_NONE = 0, EPI_STORE = 1, EPI_RESID = 2, EPI_SILU = 3 };

// Selection data of one batch-1 site, produced by the site's producer (GEMV epilogue,
// attention merge, or the standalone preparation kernel) and consumed by the SELECT prologue:
//   hist  [4096 fine bins of key bits 30:19][256 coarse bins of bits 30:23]   zero at rest
//   pool  [4096][kPoolCap] (key, index) of each fine bucket's first entries
//   ssq   [ceil(d / 256)] per-slice sums of squares (RMS sites)
// The site's exact Top-K rule (compute_rule, by every consuming CTA):
// keep i iff key_i > tk or (key_i == tk and i <= ti); value x_i * scale.  Consumers decide
// from the 16-bit keys; an element whose 16-bit key equals tk's top 16 bits is decided by the
// boundary table (idx, keep) -- or, if flags & kRuleExact, from its exact key in x.
constexpr int kRuleAll = 1, kRuleNone = 2, kRuleEdgeAll = 4, kRuleExact = 8;
constexpr int kRulePending = 16;   // the boundary bucket's pool lookup is still to come (select_rows)
constexpr int kRuleTable = 64;
struct __align__(16) SelRule {
    uint32_t tk;
    int32_t ti;
    float scale;
    int32_t flags;
    int32_t nb;                 // boundary table entries (the k-th key's 16-bit bucket)
    int32_t pad;
    unsigned long long keep;    // bit t: idx[t] is kept
    int32_t idx[kRuleTable];
};
struct SiteSel {
    uint32_t* hist;
    uint2* pool;
    float* ssq;
};
// histogram levels: 65536 fine bins of key bits [30:15] (the 16-bit key), then 256 coarse
// bins of bits [30:23]
constexpr int kSelFine = 65536;
constexpr int kSelCoarse = 256;
constexpr int kSelHistTotal = kSelFine + kSelCoarse;
constexpr int kSelHistAlloc = kSelHistTotal + 32;   // + the coarse-bucket guess word (not zeroed with the bins)
// fine bin of 16-bit key k16 at k16 (a coarse bucket's 256 fine bins are contiguous), coarse
// bin cb at kSelFine + cb, pool entry (k16, slot) at k16 * kPoolCap + slot
__host__ __device__ constexpr int sel_fine_idx(uint32_t k16) { return (int)k16; }
__host__ __device__ constexpr int sel_coarse_idx(uint32_t cb) { return kSelFine + (int)cb; }
__host__ __device__ constexpr size_t sel_pool_idx(uint32_t k16, uint32_t slot) { return (size_t)k16 * kPoolCap + slot; }

// the per-token Top-K rule: keep row i iff key_i > tk or (key_i == tk and i <= ti),
// key = bits(|x_i|); value x_i * scale
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
    // GEMV_THRESH / GEMV_DENSE / GEMV_SELECT: input x [batch][ldx] over rows [0, d_in)
    const float* x;
    int64_t ldx;
    int d_in;
    const ThreshOut* thr;              // THRESH: per-token rule + RMS scale
    // GEMV_SELECT (batch 1): the site's selection data; sel.ssq null unless RMS site
    SiteSel sel;
    int sel_nssq;
    int sel_k;
    float sel_eps;                     // < 0: no RMS scale
    int batch;             // real tokens (<= template BP)
    int n_splits;
    int list_cap;          // rows of the per-CTA shared list (host-checked >= rows per split)
    unsigned long long* acc;          // [batch][acc_ld] fixed-point output accumulators
    int64_t acc_ld;
    // epilogue (GemvEpi); EPI_NONE leaves the accumulators to the consumer kernel
    int epi;
    unsigned* tickets;                 // [n_slices], zero at rest
    const uint16_t* bias;              // [d_out] bf16 or null       (STORE / RESID)
    const float* res;                  // [batch][res_ld] or null    (RESID)
    int64_t res_ld;
    float* out;                        // [batch][out_ld]
    int64_t out_ld;
    float* out_host;                       // optional second copy of out (batch 1; mapped host memory)
    SiteSel out_sel;                   // batch 1: next site's selection data (hist null = none)
    float* out_ssq;                    // [batch][out_ssq_ld] per-slice sums of squares or null
    int64_t out_ssq_ld;
    uint32_t* zero_hist;               // optional: histogram words to re-zero (free by now)
    int zero_words;
    unsigned long long* zero_acc;      // optional: accumulators to re-zero (their consumer has completed)
    int zero_acc_words;
    // SELECT companion rows (batch 1): CTAs with blockIdx.y < n_splits2 stream DENSE rows of a
    // second matrix W2 [d2][ld] with values x2 [d2] into the same output columns (the residual
    // adapter folded next to the down projection: r_next = r_mid A_l + h4[S4] W_down Q_{l+1}).
    // Their rows need no selection rule, so their first stages are issued before the
    // dependency wait and they stream while the SELECT CTAs compute the rule.
    const uint16_t* W2;
    const float* x2;
    int d2;
    int n_splits2;
    unsigned long long* tl;            // debug timeline slot (5 x u64) or null
    int tc_dbg;                        // profiling (tcgen05 GEMV, -DLAROSA_TC_DEBUG builds only)
    // batch-1 split-K reduction through distributed shared memory: the gridDim.y CTAs of a
    // slice form one thread-block cluster (cluster != 0); rank 0 sums the CTAs' fp32 column
    // partials in rank order and finalises the slice itself (no global accumulators, no ticket)
    int cluster;
    int late_trigger;                  // tuning: 1 = release dependents after the main loop, not at entry
    uint32_t* err;                     // the workspace's error word (larosa_error_flags) or null
    const void* img;                   // batch >= 8, contiguous rows: the pre-built token operand (gemv_img.cuh)
    int comp_late;                     // tuning: companions issue their first stages after the dependency wait
    PeerOut peer;                      // sharded phases: push every output value to every rank (n = 0: off)
};

// error bits of a workspace's error word (larosa.h larosa_error_flags)
constexpr uint32_t kErrKeepAll = 1u;    // SELECT: inconsistent histogram -> the keep-all rule was used
constexpr uint32_t kErrFixOverflow = 2u;  // a partial sum |s| >= 2^31 does not fit the 64-bit fixed point

__host__ __device__ constexpr size_t gemv_align(size_t v, size_t a) { return (v + a - 1) / a * a; }

// shared memory: [ring | staged x (SELECT)] [hist (SELECT)] [row list + values] [misc]
__host__ __device__ constexpr size_t gemv_ring_bytes(int bp) {
    return (size_t)kGemvWarps * kWarpRingBytes > (size_t)kGemvWarps * bp * kSliceCols * 4
               ? (size_t)kGemvWarps * kWarpRingBytes
               : (size_t)kGemvWarps * bp * kSliceCols * 4;
}
__host__ __device__ constexpr size_t sel_region_bytes(int d);
// region A: the weight ring, aliased in SELECT mode by the staged selection data
__host__ __device__ constexpr size_t gemv_x_bytes(int bp, int mode, int d_in);
__host__ __device__ constexpr size_t gemv_list_off(int bp, int mode, int d_in) { return gemv_x_bytes(bp, mode, d_in); }
__host__ __device__ constexpr size_t gemv_misc_off(int bp, int mode, int d_in, int list_cap) {
    return gemv_align(gemv_list_off(bp, mode, d_in) + (size_t)list_cap * (4 + 4 * (size_t)bp), 16);
}
__host__ __device__ constexpr size_t gemv_smem_bytes(int bp, int list_cap, int mode = GEMV_LIST, int d_in = 0) {
    return gemv_misc_off(bp, mode, d_in, list_cap) + (size_t)kGemvMisc * 4;
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
// one fixed-point partial into an accumulator.  The sum of a column's gridDim.y partials stays
// inside the fixed point's +-2^31 when every partial is below 2^31 / gridDim.y: a partial at or
// above that bound is flagged (a sufficient condition; it may also flag sums that cancel).
__device__ __forceinline__ void red_fix(unsigned long long* p, float s, uint32_t* err) {
    if (err && !(fabsf(s) * (float)gridDim.y < 2147483648.0f)) atomicOr(err, kErrFixOverflow);
    red_add_u64(p, f_to_fix(s));
}
__device__ __forceinline__ void red_add_u32(uint32_t* p, uint32_t v) {
    asm volatile("red.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ uint32_t key_of(float v) { return __float_as_uint(v) & 0x7fffffffu; }
// producer side of a site: element i of value v.  Fine-bin count of its 16-bit key (the old
// value is the pool slot), coarse-bin count (warp-aggregated: a few exponents hold most
// elements) and the (key, i) pool entry.
__device__ __forceinline__ void hist_push(const SiteSel& o, float v, int i) {
    const uint32_t key = key_of(v), k16 = key >> 15;
    const unsigned am = __activemask();
    const unsigned peers = __match_any_sync(am, k16 >> 8);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) red_add_u32(o.hist + sel_coarse_idx(k16 >> 8), __popc(peers));
    const uint32_t slot = atomicAdd(o.hist + sel_fine_idx(k16), 1u);
    if (slot < (uint32_t)kPoolCap) o.pool[sel_pool_idx(k16, slot)] = make_uint2(key, (uint32_t)i);
}

// cp.async (LDGSTS): 16 bytes global -> shared, L1 bypass (.cg)
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool pred) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
        "@p cp.async.cg.shared.global [%0], [%1], 16;\n\t}" ::"r"(smem_u32(smem_dst)),
        "l"(gsrc), "r"((int)pred)
        : "memory");
}
// cp.async 4 bytes (L1-allocating .ca is the only variant below 16 bytes)
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
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

// Sum of squares of one 256-value slice (value c of the slice in thread c of 8 warps): a
// butterfly per warp, then the 8 warp sums in order.  The SELECT prologue's RMS scale sums
// these partials; the standalone prep kernel reproduces the exact same arithmetic.
__device__ __forceinline__ float slice_ssq_warp(float v) { return warp_sum(v * v); }
__device__ __forceinline__ float slice_ssq_combine(const float* w8) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += w8[w];
    return t;
}
// RMS scale from the per-slice partials (fixed order; identical in every CTA)
__device__ __forceinline__ float rms_scale_from_parts(const float* parts, int n, int d, float eps, int lane) {
    float s = 0.f;
    for (int i = lane; i < n; i += 32) s += __ldcg(parts + i);
    s = warp_sum(s);
    return 1.0f / sqrtf(s / (float)d + eps);
}

// Histograms in shared memory are padded (one word per 16 bins) so that a thread reading
// its 16 consecutive bins is bank-conflict free.
__host__ __device__ constexpr int hpad(int b) { return b + (b >> 4); }

// Suffix search over `nb` (<= 4096, multiple of 16 or < 16 per thread) padded bins
// (bins[hpad(nb-1)] = largest keys): the bin holding the rem-th largest key.  Thread t owns
// bins [nb - bpt (t+1), nb - bpt t).  Writes misc[0] = bin, misc[1] = rem within the bin,
// misc[2] = bin count (0, 0, 0 if the histogram holds fewer than rem keys).  Block-wide.
template <int NT>
__device__ void suffix_find(const int* bins, int nb, int rem, int* misc, int* scan_scratch) {
    const int tid = threadIdx.x;
    if (tid == 0) {   // defined result (keep-all, bounded work) even on an inconsistent histogram
        misc[0] = 0;
        misc[1] = 0;
        misc[2] = 0;
    }
    const int bpt = (nb + NT - 1) / NT;
    const int hi = max(0, nb - bpt * tid), lo = max(0, nb - bpt * (tid + 1));
    int c = 0;
    for (int bb = hi - 1; bb >= lo; --bb) c += bins[hpad(bb)];
    int total;
    const int before = block_excl_scan<NT>(c, scan_scratch, &total);
    if (c > 0 && before < rem && rem <= before + c) {
        int accu = before;
        for (int bb = hi - 1; bb >= lo; --bb) {
            const int h = bins[hpad(bb)];
            if (accu + h >= rem) {
                misc[0] = bb;
                misc[1] = rem - accu;
                misc[2] = h;
                break;
            }
            accu += h;
        }
    }
    __syncthreads();
}

// ---- the exact rule of a site (one CTA, NT threads, after every producer has pushed) ------
// Fast path, one warp, no block barrier:
//  1. coarse suffix search (256 bins of key bits 30:23, 8 per lane) -> coarse bucket; the
//     same over its 256 fine bins (bits 30:15) -> the 16-bit bucket b16 of the k-th key and
//     rem = how many of it to keep;
//  2. if b16 is not taken whole and holds <= kPoolCap elements: lane l ranks pool entries
//     l and l + 32 exactly (key desc, index asc) -> the rem-th one is (tk, ti); the bucket's
//     entries with their keep bits form the consumers' boundary table;
//  3. otherwise (rare: more than kPoolCap elements share the 16-bit key, e.g. constant
//     vectors): block-wide radix refinement over bits [14:7], [6:0] of x, then an index walk.
// The RMS scale (fixed-order sum of the slice partials) comes from another warp.
__host__ __device__ constexpr size_t rule_scratch_bytes() { return (size_t)(16 + 272 + 16) * 4 + 64; }

// warp-wide suffix search over 256 contiguous bins (bin 255 = largest keys; two 16-byte loads
// per lane through L1, so the CTAs sharing an SM hit): the bin holding the rem-th largest
// element.  Returns true and (bin, rem in bin, count) on every lane; false if the bins hold
// fewer than rem elements.
__device__ __forceinline__ void load256(const uint32_t* bins, uint4& a, uint4& b) {
    const int lane = threadIdx.x & 31;
    const uint4* p = reinterpret_cast<const uint4*>(bins + 256 - 8 * (lane + 1));
    a = __ldca(p);        // (L1-allocating: the SM's other CTA reads the same lines; .cg measured ~0.2 us slower)
    b = __ldca(p + 1);
}
__device__ __forceinline__ bool suffix256(const uint4& a, const uint4& b, int rem, int& bin, int& rem_in, int& cnt) {
    const int lane = threadIdx.x & 31;
    const int j0 = 256 - 8 * (lane + 1);
    const int c[8] = {(int)a.x, (int)a.y, (int)a.z, (int)a.w, (int)b.x, (int)b.y, (int)b.z, (int)b.w};
    int sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) sum += c[j];
    const int incl = warp_incl_scan(sum);
    const int before = incl - sum;
    int mb = 0, mr = 0, mc = 0;
    const bool mine = sum > 0 && before < rem && rem <= incl;
    if (mine) {
        int accu = before;
#pragma unroll
        for (int j = 7; j >= 0; --j) {
            if (accu >= 0 && accu + c[j] >= rem) {
                mb = j0 + j;
                mr = rem - accu;
                mc = c[j];
                accu = -(1 << 30);
            }
            accu += c[j];
        }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, mine);
    if (!bal) return false;
    const int src = __ffs(bal) - 1;
    bin = __shfl_sync(0xffffffffu, mb, src);
    rem_in = __shfl_sync(0xffffffffu, mr, src);
    cnt = __shfl_sync(0xffffffffu, mc, src);
    return true;
}
__device__ __forceinline__ bool warp_suffix256(const uint32_t* bins, int rem, int& bin, int& rem_in, int& cnt) {
    uint4 a, b;
    load256(bins, a, b);
    return suffix256(a, b, rem, bin, rem_in, cnt);
}

// warp-wide: the exact rule inside the k-th key's 16-bit bucket b16 (cnt entries, rem of them kept)
// from the bucket's pool of (key, index) entries: Tk, Ti and the keep table of the entries' indices
__device__ __forceinline__ void rule_pool(const SiteSel& sel, int b16, int rem, int cnt, SelRule* R, uint32_t& tk,
                                          int& ti, int& nb, unsigned long long& keep) {
    const int lane = threadIdx.x & 31;
    const uint2 e0 = lane < cnt ? __ldca(sel.pool + sel_pool_idx(b16, lane)) : make_uint2(0u, 0x7fffffffu);
    const uint2 e1 = lane + 32 < cnt ? __ldca(sel.pool + sel_pool_idx(b16, lane + 32)) : make_uint2(0u, 0x7fffffffu);
    int r0 = 0, r1b = 0;
    for (int q = 0; q < cnt; ++q) {
        const uint32_t kq = __shfl_sync(0xffffffffu, q < 32 ? e0.x : e1.x, q & 31);
        const uint32_t iq = __shfl_sync(0xffffffffu, q < 32 ? e0.y : e1.y, q & 31);
        r0 += kq > e0.x || (kq == e0.x && iq < e0.y);
        r1b += kq > e1.x || (kq == e1.x && iq < e1.y);
    }
    const bool h0 = lane < cnt && r0 == rem - 1, h1 = lane + 32 < cnt && r1b == rem - 1;
    const unsigned b0 = __ballot_sync(0xffffffffu, h0), b1 = __ballot_sync(0xffffffffu, h1);
    const int s0 = __ffs(b0 ? b0 : b1) - 1;
    const uint32_t hk0 = __shfl_sync(0xffffffffu, e0.x, s0), hi0 = __shfl_sync(0xffffffffu, e0.y, s0);
    const uint32_t hk1 = __shfl_sync(0xffffffffu, e1.x, s0), hi1 = __shfl_sync(0xffffffffu, e1.y, s0);
    tk = b0 ? hk0 : hk1;
    ti = (int)(b0 ? hi0 : hi1);
    nb = cnt;
    const unsigned k0 = __ballot_sync(0xffffffffu, lane < cnt && r0 < rem);
    const unsigned k1 = __ballot_sync(0xffffffffu, lane + 32 < cnt && r1b < rem);
    keep = (unsigned long long)k0 | ((unsigned long long)k1 << 32);
    if (lane < cnt) R->idx[lane] = (int)e0.y;
    if (lane + 32 < cnt) R->idx[lane + 32] = (int)e1.y;
}

// defer_pool: when the boundary bucket needs its pool, return with kRulePending (tk = the bucket's
// lower edge, misc[1..3] = b16 / rem / cnt) and let the caller's warp 0 resolve it (rule_pool)
// while the other warps compute the definite keep masks
// (zero job: words whose consumer has completed, cleared by warps 2.. while warp 0 looks the rule up and
// warp 1 sums the squares -- not ahead of warp 0's loads in program order)
struct ZeroJob {
    uint32_t* w32;
    int n32;
    unsigned long long* w64;
    int n64;
};
// this CTA's share of a zero job: nz threads per CTA (t < nz), the same partition in every CTA of the grid
__device__ __forceinline__ void zero_share(const ZeroJob& zj, int t, int nz) {
    const int nct = gridDim.x * gridDim.y, cta = blockIdx.y * gridDim.x + blockIdx.x;
    for (int i = cta * nz + t; i < zj.n32; i += nct * nz) zj.w32[i] = 0u;
    for (int i = cta * nz + t; i < zj.n64; i += nct * nz) zj.w64[i] = 0ull;
}
template <int NT>
__device__ void compute_rule(const SiteSel& sel, const float* x, int d, int k, float eps, int nssq,
                             unsigned char* scratch, SelRule* R, unsigned long long* tl = nullptr, int guess = 0,
                             uint32_t* err = nullptr, bool defer_pool = false, const ZeroJob* zj = nullptr) {
    static_assert(NT >= 64, "two warps");
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int* misc = reinterpret_cast<int*>(scratch);           // [0] status, [1..3] b16/rem/cnt, [4] scale
    int* shist = misc + 16;                                 // fallback: <= 256 padded bins
    int* scan = shist + 272;
    float* fmisc = reinterpret_cast<float*>(misc);
    if (zj && wid >= 2) zero_share(*zj, tid - 64, NT - 64);
    if (wid == 1) {
        const float sc = eps >= 0.f ? rms_scale_from_parts(sel.ssq, nssq, d, eps, lane) : 1.0f;
        if (lane == 0) fmisc[4] = sc;
        if (tl && lane == 0 && blockIdx.x + blockIdx.y * gridDim.x < 1024)
            tl[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + 10] = gtime();
    }
    if (wid == 0) {
        uint32_t tk = 0u;
        int ti = 0x7fffffff, flags = 0, nb = 0, status = 0;
        unsigned long long keep = 0ull;
        int b16 = 0, rem = 0, cnt = 0;
        if (k <= 0) {
            flags = kRuleNone;
            tk = 0xffffffffu;
            ti = -1;
        } else if (k >= d) {
            flags = kRuleAll;
        } else {
            // lookup 1 reads the coarse bins together with the fine bins of the coarse buckets
            // around the previous call's (guess = cb + 1 of this site's last consumer): when the
            // k-th key's bucket is among them, lookup 2 costs no extra round trip
            int cb = 0, r1 = 0, cc = 0, fb = 0;
            const int g = __shfl_sync(0xffffffffu, guess, 0) - 1;
            uint4 ca, cbv, f0a, f0b, f1a, f1b, f2a, f2b;
            const uint4 z = make_uint4(0u, 0u, 0u, 0u);
            load256(sel.hist + kSelFine, ca, cbv);
            f0a = f0b = f1a = f1b = f2a = f2b = z;
            if (g >= 0 && g < 256) load256(sel.hist + 256 * g, f0a, f0b);
            if (g >= 1 && g < 257) load256(sel.hist + 256 * (g - 1), f1a, f1b);
            if (g >= -1 && g < 255) load256(sel.hist + 256 * (g + 1), f2a, f2b);
            if (tl) {   // (timeline only) the coarse bins have arrived
                uint32_t dep;
                asm volatile("mov.b32 %0, %1;" : "=r"(dep) : "r"(ca.x ^ cbv.w ^ f0a.x ^ f2b.w));
                if (dep == 0x5eed5eedu) tl_stamp(tl, 15);
                tl_stamp(tl, 14);
            }
            const bool ok1 = suffix256(ca, cbv, k, cb, r1, cc);
            tl_stamp(tl, 6);
            bool ok2 = false;
            if (ok1) {
                if (cb == g) {
                    ok2 = suffix256(f0a, f0b, r1, fb, rem, cnt);
                } else if (cb == g - 1) {
                    ok2 = suffix256(f1a, f1b, r1, fb, rem, cnt);
                } else if (cb == g + 1) {
                    ok2 = suffix256(f2a, f2b, r1, fb, rem, cnt);
                } else {
                    ok2 = warp_suffix256(sel.hist + 256 * cb, r1, fb, rem, cnt);
                }
                if (lane == 0 && blockIdx.x == 0 && blockIdx.y == 0 && cb + 1 != guess)
                    sel.hist[kSelHistTotal] = (uint32_t)(cb + 1);   // next call's guess (not zeroed with the bins)
            }
            tl_stamp(tl, 8);
            if (!ok1 || !ok2) {
                flags = kRuleAll;   // inconsistent histogram: keep-all (bounded, never faults), flagged
                if (err && lane == 0) atomicOr(err, kErrKeepAll);
            } else {
                b16 = 256 * cb + fb;
                if (cnt == rem) {
                    tk = (uint32_t)b16 << 15;   // the 16-bit bucket is taken whole: key >= tk
                    flags = kRuleEdgeAll;
                } else if (cnt <= kPoolCap && defer_pool) {
                    tk = (uint32_t)b16 << 15;   // only the 16-bit bucket is known yet
                    flags = kRulePending;
                } else if (cnt <= kPoolCap) {
                    rule_pool(sel, b16, rem, cnt, R, tk, ti, nb, keep);
                    tl_stamp(tl, 9);
                } else {
                    status = 1;      // overflow: block-wide fallback below
                }
            }
        }
        if (lane == 0) {
            misc[0] = status;
            misc[1] = b16;
            misc[2] = rem;
            misc[3] = cnt;
            if (!status) {
                R->tk = tk;
                R->ti = ti;
                R->flags = flags;
                R->nb = nb;
                R->keep = keep;
            }
        }
    }
    __syncthreads();
    if (misc[0]) {
        // fallback: radix refinement of the 16-bit bucket over x, then the index walk
        uint32_t prefix = (uint32_t)misc[1] << 15, pmask = 0xffffu << 15;
        int rem = misc[2], cnt = misc[3];
#pragma unroll 1
        for (int pass = 0; pass < 2 && cnt != rem; ++pass) {
            const int sh = pass == 0 ? 7 : 0;
            const int nbins = pass == 0 ? 256 : 128;
            const uint32_t dm = (uint32_t)(nbins - 1);
            for (int i = tid; i < hpad(nbins - 1) + 1; i += NT) shist[i] = 0;
            __syncthreads();
            for (int i = tid; i < d; i += NT) {
                const uint32_t key = key_of(__ldcg(x + i));
                if ((key & pmask) == prefix) atomicAdd(&shist[hpad((key >> sh) & dm)], 1);
            }
            __syncthreads();
            suffix_find<NT>(shist, nbins, rem, misc + 8, scan);
            prefix |= (uint32_t)misc[8] << sh;
            pmask |= dm << sh;
            rem = misc[9];
            cnt = misc[10];
            __syncthreads();
        }
        int ti = 0x7fffffff;
        if (cnt != rem) {
            if (wid == 0) {
                int seen = 0, at = -1;
                for (int i0 = 0; i0 < d; i0 += 32) {
                    const int i = i0 + lane;
                    const uint32_t bal = __ballot_sync(0xffffffffu, i < d && key_of(__ldcg(x + i)) == prefix);
                    if (seen + __popc(bal) >= rem) {
                        uint32_t m = bal;
                        for (int q = 1; q < min(rem - seen, 32); ++q) m &= m - 1;
                        at = i0 + __ffs(m) - 1;
                        break;
                    }
                    seen += __popc(bal);
                }
                if (lane == 0) misc[11] = at;
            }
            __syncthreads();
            ti = misc[11];
        }
        if (tid == 0) {
            R->tk = prefix;
            R->ti = ti;
            R->flags = kRuleExact;
            R->nb = 0;
            R->keep = 0ull;
        }
    }
    if (tid == 0) R->scale = fmisc[4];
    __syncthreads();
}

// ---- SELECT prologue (batch 1): this CTA's rows of the site's kept set -------------------
// Shared memory (region A, aliased later by the weight ring): the 16-bit keys of the CTA's
// words and their keep masks / counts.  The CTA's words: w_j = split + n_splits j (32-index
// words round-robin over the splits: balanced in expectation, robust to index-correlated
// keep rates such as PCA-ordered channels).
constexpr int kSelMaxWords = 256;
__host__ __device__ constexpr size_t sel_mask_off(int d) { return (size_t)kSelMaxWords * 128; }
__host__ __device__ constexpr size_t sel_region_bytes(int d) {
    return gemv_align(sel_mask_off(d) + (size_t)kSelMaxWords * 12 + rule_scratch_bytes(), 128);
}
__host__ __device__ constexpr size_t gemv_x_bytes(int bp, int mode, int d_in) {
    return mode == GEMV_SELECT && sel_region_bytes(d_in) > gemv_ring_bytes(bp) ? sel_region_bytes(d_in)
                                                                               : gemv_ring_bytes(bp);
}

// Returns the number of rows placed in lrow (ascending); misc[4] receives the RMS scale.
__device__ __forceinline__ int select_rows(const GemvArgs& a, unsigned char* region, int* lrow, float* lval, int* misc,
                                           int split, int n_splits, int guess, const ZeroJob* zj = nullptr) {
    constexpr int NT = kGemvThreads, NW = kGemvWarps;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int d = a.d_in;
    float* xs = reinterpret_cast<float*>(region);   // the CTA's words of x (keys and values)
    uint32_t* wmk = reinterpret_cast<uint32_t*>(region + sel_mask_off(d));
    int* wcnt = reinterpret_cast<int*>(wmk + kSelMaxWords);
    int* scan = misc + 8;
    const uint32_t lt = (1u << lane) - 1u;
    const int nwords = (d + 31) / 32;
    const int nj = nwords > split ? (nwords - 1 - split) / n_splits + 1 : 0;
    for (int c = tid; c < 8 * nj; c += NT) {
        const int j = c >> 3, w = split + n_splits * j;
        const int i0 = 32 * w + 4 * (c & 7);
        cp_async16(xs + 32 * j + 4 * (c & 7), a.x + i0, i0 < d);
    }
    cp_async_commit();
    // the exact rule, computed by warps 0 (selection) and 1 (RMS scale) while the CTA's words land
    SelRule* R = reinterpret_cast<SelRule*>(misc + 48);
    unsigned char* rscratch = region + sel_mask_off(d) + kSelMaxWords * 8;
    compute_rule<NT>(a.sel, a.x, d, a.sel_k, a.sel_eps, a.sel_nssq, rscratch, R, a.tl, guess, a.err, true, zj);
    const int* rmisc = reinterpret_cast<const int*>(rscratch);
    const int flags0 = R->flags;
    if (tid == 0) reinterpret_cast<float*>(misc)[4] = R->scale;
    cp_async_wait<0>();
    __syncthreads();
    tl_stamp(a.tl, 5);
    uint32_t* bmk = reinterpret_cast<uint32_t*>(rscratch + rule_scratch_bytes());   // pending: boundary lanes per word
    int total;
    if (flags0 & kRulePending) {
        // warp 0 resolves the boundary bucket from its pool while warps 1.. mark the definite rows
        // (16-bit key above the bucket) and the boundary elements of every word
        const uint32_t t16 = R->tk >> 15;
        if (wid == 0) {
            uint32_t tk;
            int ti, nb;
            unsigned long long keep;
            rule_pool(a.sel, rmisc[1], rmisc[2], rmisc[3], R, tk, ti, nb, keep);
            if (lane == 0) {
                R->tk = tk;
                R->ti = ti;
                R->nb = nb;
                R->keep = keep;
                R->flags = 0;
            }
            tl_stamp(a.tl, 9);
        } else {
            for (int j = wid - 1; j < nj; j += NW - 1) {
                const int i = 32 * (split + n_splits * j) + lane;
                const uint32_t k16 = i < d ? key_of(xs[32 * j + lane]) >> 15 : 0u;
                const uint32_t m = __ballot_sync(0xffffffffu, i < d && k16 > t16);
                const uint32_t bm = __ballot_sync(0xffffffffu, i < d && k16 == t16);
                if (lane == 0) {
                    wmk[j] = m;
                    wcnt[j] = __popc(m);
                    bmk[j] = bm;
                }
            }
        }
        __syncthreads();
        // the boundary elements by the pool's keep table
        const int nbt = R->nb;
        const unsigned long long keepm = R->keep;
        for (int j = wid; j < nj; j += NW) {
            const uint32_t bm = bmk[j];
            if (!bm) continue;
            const int i = 32 * (split + n_splits * j) + lane;
            bool kp = false;
            if ((bm >> lane) & 1u)
                for (int q = 0; q < nbt; ++q)
                    if (R->idx[q] == i) kp = (keepm >> q) & 1ull;
            const uint32_t m = __ballot_sync(0xffffffffu, kp);
            if (lane == 0) {
                wmk[j] |= m;
                wcnt[j] += __popc(m);
            }
        }
        __syncthreads();
    } else {
    const uint32_t tk = R->tk;
    const int ti = R->ti;
    const int flags = R->flags;
    const int nbt = R->nb;
    const unsigned long long keepm = R->keep;
    const int* tab = R->idx;
    const uint32_t t16 = tk >> 15;
    auto keep16 = [&](uint32_t key, int i) -> bool {
        const uint32_t k16 = key >> 15;
        if (k16 != t16) return k16 > t16;
        if (flags & kRuleEdgeAll) return true;
        if (!(flags & kRuleExact)) {
            for (int q = 0; q < nbt; ++q)
                if (tab[q] == i) return (keepm >> q) & 1ull;
            return false;
        }
        return key > tk || (key == tk && i <= ti);
    };
    const bool all = flags & kRuleAll, none = flags & kRuleNone;
        for (int j = wid; j < nj; j += NW) {
            const int i = 32 * (split + n_splits * j) + lane;
            bool kp = false;
            if (i < d) kp = all ? true : (none ? false : keep16(key_of(xs[32 * j + lane]), i));
            const uint32_t m = __ballot_sync(0xffffffffu, kp);
            if (lane == 0) {
                wmk[j] = m;
                wcnt[j] = __popc(m);
            }
        }
        __syncthreads();
    }
    {
        tl_stamp(a.tl, 7);
        const int cj = tid < nj ? wcnt[tid] : 0;
        const int before = block_excl_scan<NT>(cj, scan, &total);
        __syncthreads();
        if (tid < nj) wcnt[tid] = before;
        __syncthreads();
        for (int j = wid; j < nj; j += NW) {
            const uint32_t m = wmk[j];
            if ((m >> lane) & 1u) {   // the row index and its activation (the value rides with the list)
                const int pos = wcnt[j] + __popc(m & lt);
                lrow[pos] = 32 * (split + n_splits * j) + lane;
                lval[pos] = xs[32 * j + lane];
            }
        }
        __syncthreads();   // list complete; the staged region (aliased by the ring) is dead
        tl_stamp(a.tl, 11);
    }
    return total;
}

// ---- epilogue: the last split CTA of a slice finalises its columns ------------------------
// tot == nullptr: the slice's sums are in the global fixed-point accumulators (re-zeroed here);
// else tot[256] (shared memory, batch 1) holds them in fp32 (cluster reduction).
template <int BP>
__device__ void gemv_epilogue(const GemvArgs& a, int slice, float* sred, const float* tot = nullptr) {
    const int c = threadIdx.x, lane = c & 31, wid = c >> 5;
    const int base = slice * kSliceCols;
    for (int b = 0; b < a.batch; ++b) {
        unsigned long long* acc = a.acc + (size_t)b * a.acc_ld;
        float v = 0.f;
        bool has = false;
        if (a.epi == EPI_SILU) {
            // slice = 2 gate|up blocks of 128 columns (64 gate, then the matching 64 up)
            if (c < 2 * kGuBlock) {
                const int blk = c / kGuBlock, q = c % kGuBlock;
                const int og = base + blk * 2 * kGuBlock + q;
                if (og < a.d_out) {
                    float g, u;
                    if (tot) {
                        g = tot[og - base];
                        u = tot[og - base + kGuBlock];
                    } else {
                        g = fix_to_f(__ldcg(acc + og));
                        u = fix_to_f(__ldcg(acc + og + kGuBlock));
                        acc[og] = 0ull;
                        acc[og + kGuBlock] = 0ull;
                    }
                    v = g / (1.0f + expf(-g)) * u;
                    a.out[(size_t)b * a.out_ld + slice * 2 * kGuBlock + blk * kGuBlock + q] = v;
                    has = true;
                }
            }
        } else {
            const int o = base + c;
            if (o < a.d_out) {
                float y;
                if (tot) {
                    y = tot[c];
                } else {
                    y = fix_to_f(__ldcg(acc + o));
                    acc[o] = 0ull;
                }
                v = y;
                if (a.bias) v += bf16f(a.bias[o]);
                if (a.res) v = a.res[(size_t)b * a.res_ld + o] + v;
                a.out[(size_t)b * a.out_ld + o] = v;
                if (a.out_host) a.out_host[(size_t)b * a.out_ld + o] = v;
                has = true;
            }
        }
        if (has && a.out_sel.hist && a.batch == 1) {
            const int idx = a.epi == EPI_SILU ? slice * 2 * kGuBlock + (c / kGuBlock) * kGuBlock + c % kGuBlock
                                              : base + c;
            hist_push(a.out_sel, v, idx);
        }
        if (a.out_ssq) {
            const float w = slice_ssq_warp(v);
            if (lane == 0) sred[wid] = w;
            __syncthreads();
            if (c == 0) a.out_ssq[(size_t)b * a.out_ssq_ld + slice] = slice_ssq_combine(sred);
            __syncthreads();
        }
    }
    if (a.peer.n) {   // the slice's outputs (thread c wrote output column c of the block) to every rank
        if (a.epi == EPI_SILU)
            peer_push_cols(a.peer, a.out, a.out_ld, a.batch, slice * 2 * kGuBlock,
                           kGuBlock * min(2, max(0, (a.d_out - base + 2 * kGuBlock - 1) / (2 * kGuBlock))));
        else
            peer_push_cols(a.peer, a.out, a.out_ld, a.batch, base, min(kSliceCols, max(0, a.d_out - base)));
    }
}

// One instantiation per (padded batch, row source) keeps each kernel's code small: these
// launches are latency-bound and start on a cold instruction cache.
template <int BP, int MODE>
__global__ void __launch_bounds__(kGemvThreads) gemv_kernel(const GemvArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int slice = blockIdx.x;
    // SELECT with companions: blockIdx.y < n_splits2 are the companion CTAs (dispatched first,
    // so they take the slots that free up early), the rest are the SELECT splits
    const int split = (int)blockIdx.y - (MODE == GEMV_SELECT ? a.n_splits2 : 0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int mode = MODE;
    int* lrow = reinterpret_cast<int*>(smem + gemv_list_off(BP, mode, a.d_in));       // [cap]
    float* lval = reinterpret_cast<float*>(lrow + a.list_cap);                        // [cap][BP]
    int* misc = reinterpret_cast<int*>(smem + gemv_misc_off(BP, mode, a.d_in, a.list_cap));

    // companion CTA (SELECT mode, blockIdx.y < n_splits2): dense rows [c_lo, c_lo + n) of W2
    bool comp = false;
    int c_lo = 0, c_n = 0;
    if constexpr (MODE == GEMV_SELECT) {
        if (split < 0) {
            comp = true;
            const int rng = (a.d2 + a.n_splits2 - 1) / a.n_splits2;
            c_lo = min(a.d2, (int)blockIdx.y * rng);
            c_n = min(a.d2, c_lo + rng) - c_lo;
        }
    }
    const uint16_t* Wb = comp ? a.W2 : a.W;
    const int col0 = slice * kSliceCols + lane * 8;
    const bool lane_on = col0 < a.d_out;          // d_out % 8 == 0: a lane's chunk is all-in or all-out
    unsigned char* mychunk = smem + (size_t)warp * kWarpRingBytes + lane * 16;
    const uint16_t* wcol = Wb + col0;
    // companion: the weights of the first kStages stages do not depend on the previous kernel
    const int c_my = c_n > warp ? (c_n - warp + kGemvWarps - 1) / kGemvWarps : 0;
    auto comp_prefetch = [&]() {
#pragma unroll
        for (int st = 0; st < kStages; ++st) {
            unsigned char* dst = mychunk + (size_t)st * (kStageRows * kSliceCols * 2);
#pragma unroll
            for (int g = 0; g < kStageRows; ++g) {
                const int m = st * kStageRows + g;
                const int row = m < c_my ? c_lo + warp + kGemvWarps * m : 0;
                cp_async16(dst + g * (kSliceCols * 2), wcol + (size_t)row * a.ld, lane_on && m < c_my);
            }
            cp_async_commit();
        }
    };
    if (comp && !a.comp_late) comp_prefetch();

    // SELECT: the coarse-bucket guess left by this site's previous consumer (written by a kernel
    // that completed before the previous one; any value is safe, a wrong one costs a round trip)
    int sel_guess = 0;
    if constexpr (MODE == GEMV_SELECT)
        if (!comp && threadIdx.x == 0) sel_guess = (int)__ldcg(a.sel.hist + kSelHistTotal);

    tl_stamp(a.tl, 0);
    pdl_wait();       // the row source comes from the previous kernel
    if (!a.late_trigger) pdl_trigger();
    tl_stamp(a.tl, 1);
    if (comp && a.comp_late) comp_prefetch();   // (tuning: not while the previous kernel's prologue runs)
    // words whose consumer has completed (kernel-boundary ordered): a histogram, accumulators.  A
    // SELECT CTA clears them inside the rule lookup with its otherwise idle warps (every CTA of the
    // grid takes a share; the companions' shares too); the other modes clear them here
    ZeroJob zj;
    zj.w32 = a.zero_hist;
    zj.n32 = a.zero_hist ? a.zero_words : 0;
    zj.w64 = a.zero_acc;
    zj.n64 = a.zero_acc ? a.zero_acc_words : 0;
    // (one partition for the whole grid: kGemvThreads - 64 threads per CTA in SELECT launches, whose
    // companion CTAs clear their share here with the same partition)
    const bool zero_in_rule = MODE == GEMV_SELECT && !comp;
    if (!zero_in_rule && (zj.n32 || zj.n64)) {
        const int nz = MODE == GEMV_SELECT ? kGemvThreads - 64 : kGemvThreads;
        if ((int)threadIdx.x < nz) zero_share(zj, threadIdx.x, nz);
    }

    // ---- 1. this CTA's row list in shared memory (ascending) ------------------------------
    int n_list = 0;
    if constexpr (MODE == GEMV_SELECT) {
        static_assert(BP == 1, "SELECT is the batch-1 path");
        if (comp) {
            n_list = c_n;
            // every value of the CTA's dense rows, once (list position t = row c_lo + t)
            for (int t = threadIdx.x; t < c_n; t += kGemvThreads) lval[t] = __ldcg(a.x2 + c_lo + t);
            __syncthreads();
        } else {
            n_list = select_rows(a, smem, lrow, lval, misc, split, a.n_splits, sel_guess, &zj);
        }
    } else if constexpr (MODE == GEMV_LIST) {
        const int nrows = a.nrows_dev ? *a.nrows_dev : a.nrows;
        const int rps = (nrows + a.n_splits - 1) / a.n_splits;
        const int r_begin = min(nrows, split * rps);
        n_list = min(nrows, r_begin + rps) - r_begin;
        for (int t = threadIdx.x; t < n_list; t += kGemvThreads) {
            const int r = r_begin + t;
            lrow[t] = __ldg(a.rows + r);
#pragma unroll
            for (int b = 0; b < BP; ++b)
                lval[t * BP + b] = b < a.batch ? __ldg(a.vals + (size_t)r * a.vs_r + (size_t)b * a.vs_b) : 0.f;
        }
        __syncthreads();
    } else {
        // input range of this split; keep a row if any token keeps it (THRESH rule) or always
        const int rng = (a.d_in + a.n_splits - 1) / a.n_splits;
        const int lo = min(a.d_in, split * rng), hi = min(a.d_in, lo + rng);
        const ThreshOut* thr = a.thr;
        int base = 0;
        for (int r0 = lo, rnd = 0; r0 < hi; r0 += kGemvThreads, ++rnd) {
            const int i = r0 + (int)threadIdx.x;
            float v[BP];
            bool any = false;
#pragma unroll
            for (int b = 0; b < BP; ++b) {
                float x = 0.f;
                bool keep = false;
                if (i < hi && b < a.batch) {
                    x = a.x[(size_t)b * a.ldx + i];
                    if constexpr (MODE == GEMV_DENSE) {
                        keep = true;
                    } else {
                        const uint32_t key = key_of(x);
                        keep = key > thr[b].tk || (key == thr[b].tk && i <= thr[b].ti);
                        x *= thr[b].scale;
                    }
                }
                v[b] = keep ? x : 0.f;
                any |= keep;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, any);
            int* cnt = misc + 32 + (rnd & 1) * 8;
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
        __syncthreads();
    }

    tl_stamp(a.tl, 2);
    float sel_scale = 1.f;
    if constexpr (MODE == GEMV_SELECT) sel_scale = comp ? 1.f : reinterpret_cast<const float*>(misc)[4];
    // my rows: list entries warp + 8*m, m in [0, n_my)
    const int n_my = n_list > warp ? (n_list - warp + kGemvWarps - 1) / kGemvWarps : 0;
    const int n_st = (n_my + kStageRows - 1) / kStageRows;

    // stage st covers my-rows [4 st, 4 st + 4)
    auto issue = [&](int st) {
        if (st < n_st) {
            unsigned char* dst = mychunk + (size_t)(st % kStages) * (kStageRows * kSliceCols * 2);
#pragma unroll
            for (int g = 0; g < kStageRows; ++g) {
                const int m = st * kStageRows + g;
                const int lpos = warp + kGemvWarps * m;
                const int row = m < n_my ? (comp ? c_lo + lpos : lrow[lpos]) : 0;
                cp_async16(dst + g * (kSliceCols * 2), wcol + (size_t)row * a.ld, lane_on && m < n_my);

            }
        }
        cp_async_commit();   // one (possibly empty) group per stage keeps the count uniform
    };
    if (!comp) {
#pragma unroll
        for (int st = 0; st < kStages; ++st) issue(st);
    }

    float2 acc[BP][4];
#pragma unroll
    for (int b = 0; b < BP; ++b)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[b][j] = make_float2(0.f, 0.f);

    for (int st = 0; st < n_st; ++st) {
        cp_async_wait<kStages - 1>();          // this lane's chunks of stage st have landed
        const unsigned char* src = mychunk + (size_t)(st % kStages) * (kStageRows * kSliceCols * 2);
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
                const float v = MODE == GEMV_SELECT ? vrow[b] * sel_scale : vrow[b];   // smem broadcast
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
    if (a.late_trigger) pdl_trigger();
    tl_stamp(a.tl, 3);

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
    if constexpr (BP == 1) {
        if (a.cluster) {
            // cluster split-K: every CTA's column partials in its own shared memory, rank 0 sums
            // them in rank order (deterministic) and finalises; the others wait until it has read
            float* cpart = part + kGemvWarps * kSliceCols;   // [256]
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < kGemvWarps; ++w) s += part[(size_t)w * kSliceCols + c];
            cpart[c] = n_list > 0 ? s : 0.f;
            cluster_sync_all();
            const uint32_t rank = cluster_ctarank();
            if (rank != 0) {
                cluster_sync_all();
                tl_stamp(a.tl, 4);
                return;
            }
            tl_stamp(a.tl, 12);
            float t = 0.f;
            const uint32_t my = smem_u32(cpart + c);
            for (int r = 0; r < a.cluster; ++r) {
                uint32_t addr;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(my), "r"(r));
                t += dsmem_ld_f32(addr);
            }
            cluster_sync_all();                              // the peers may exit now
            float* tot = cpart + kSliceCols;                  // [256]
            tot[c] = t;
            if (a.epi == EPI_NONE) {                         // the consumer kernel reads the accumulators
                if (o < a.d_out) a.acc[o] = f_to_fix(t);
                tl_stamp(a.tl, 4);
                return;
            }
            __syncthreads();
            tl_stamp(a.tl, 13);
            gemv_epilogue<BP>(a, slice, reinterpret_cast<float*>(misc + 16), tot);
            tl_stamp(a.tl, 4);
            return;
        }
    }
    if (o < a.d_out && n_list > 0) {
        for (int b = 0; b < a.batch; ++b) {
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < kGemvWarps; ++w) s += part[((size_t)w * BP + b) * kSliceCols + c];
            red_fix(a.acc + (size_t)b * a.acc_ld + o, s, a.err);
        }
    }
    if (a.epi == EPI_NONE) {
        tl_stamp(a.tl, 4);
        return;
    }

    // ---- epilogue: the last split of this slice finalises it ------------------------------
    // (bar.sync orders the CTA's reds before thread 0's release; its acquire plus the next
    // bar.sync order the other splits' reds before this CTA's accumulator reads)
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
    gemv_epilogue<BP>(a, slice, reinterpret_cast<float*>(misc + 16));
    tl_stamp(a.tl, 4);
}

// ---- standalone SELECT preparation: histogram + per-slice sums of squares of x ------------
// (batch 1, when the site vector was not produced by a GEMV epilogue).  One 256-thread CTA per
// 256-element slice: the CTAs zero the bins, meet at a grid barrier (all CTAs are co-resident:
// d <= 32768 -> <= 128 small CTAs), then each pushes its slice's elements and writes the slice's
// sum of squares with the exact arithmetic of gemv_epilogue.  bar: 2 zero-at-rest words.
constexpr int kPrepThreads = kSliceCols;
__global__ void __launch_bounds__(kPrepThreads) select_prep_kernel(const float* __restrict__ x, int d, SiteSel o,
                                                                   unsigned* bar, float* __restrict__ copy_out) {
    __shared__ float sred[kPrepThreads / 32];
    pdl_wait();
    pdl_trigger();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nct = gridDim.x, cta = blockIdx.x;
    for (int i = cta * kPrepThreads + tid; i < kSelHistTotal / 4; i += nct * kPrepThreads)
        reinterpret_cast<uint4*>(o.hist)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        atomicAdd(&bar[0], 1u);
        unsigned seen;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
            if (seen < (unsigned)nct) __nanosleep(64);
        } while (seen < (unsigned)nct);
    }
    __syncthreads();
    const int i = cta * kPrepThreads + tid;
    // copy_out != null: x is mapped host memory -- read it uncached (.cv: fetched over the bus
    // every call, never an L2 hit on an earlier step's line) and store it to the device copy
    const float v = i < d ? (copy_out ? __ldcv(x + i) : x[i]) : 0.f;
    if (copy_out && i < d) copy_out[i] = v;
    if (i < d) hist_push(o, v, i);
    if (o.ssq) {
        const float w = slice_ssq_warp(v);
        if (lane == 0) sred[wid] = w;
        __syncthreads();
        if (tid == 0) o.ssq[cta] = slice_ssq_combine(sred);
    }
    if (tid == 0 && atomicAdd(&bar[1], 1u) == (unsigned)nct - 1u) {   // every CTA is past the barrier
        bar[0] = 0u;
        bar[1] = 0u;
    }
}

}  // namespace larosa
