// gemv.cuh — sparse GEMV over the kept rows of a column-major weight (eq. after_merge,
// PAPER.md:407-410; kernel recipe P:414: column-major storage, selective loads of the kept
// columns), with the epilogues the decoder layer fuses into it.
//
//   y[b][o] = sum_{r < nrows} val(r, b) * W[row(r)][o]      (+ epilogue)
//
// Decomposition (B200: 148 SMs, 227 KB smem, thread-block clusters with DSMEM):
//  * output columns are cut into tiles of TN (a multiple of 256); the kept-row list into CS
//    contiguous chunks; the CS CTAs of one tile form a thread-block CLUSTER (CS <= 16), one
//    CTA per SM with a ~200 KB shared-memory staging ring;
//  * inside a CTA, warp (cs, rg) owns the 256-column slice cs of the tile and every RG-th
//    kept row of the CTA's chunk.  Each kept row's 512-byte segment (contiguous in the
//    [d_in][d_out] layout) is one coalesced warp-wide cp.async (LDGSTS, 16 B per lane) into
//    the warp's private ring of 4-row stages, up to 16 stages deep.  A lane later reads back
//    exactly the 16 bytes it copied, so the pipeline needs no barrier, only the lane's own
//    cp.async groups.  (Measured on B200: the TMA engine retires about one bulk copy per
//    ~50 cycles per SM, so 0.5-2 KB gathered row segments cap cp.async.bulk at 15-38 GB/s
//    per SM, below the 44 GB/s/SM that 6.5 TB/s needs; per-thread cp.async has no such cap.)
//  * fp32 FMAs on the bf16 weights (8 columns per lane); the kept rows' token values come
//    from a 32-row register window broadcast with shfl;
//  * the split-K reduction is deterministic and never touches global memory: each CTA
//    reduces its RG row groups in shared memory, a cluster barrier, then CTA q sums its
//    share of column PAIRS over the CS CTAs in fixed order through distributed shared
//    memory (ld.shared::cluster) and runs the epilogue on complete values (pairs
//    (c, c + po) keep RoPE halves and gate/up blocks together).
#pragma once
#include "common.cuh"

namespace larosa {

enum EpKind : int { EP_STORE = 0, EP_RESID = 1, EP_SILU_GU = 2, EP_QKV_ROPE = 3 };

constexpr int kGuBlock = 64;         // == LAROSA_GU_BLOCK
constexpr int kWarpCols = 256;       // columns per warp slice (8 per lane)
constexpr int kStageRows = 4;        // rows per stage per warp (one 512-byte copy each)
constexpr int kStageBytes = kStageRows * kWarpCols * 2;
constexpr int kGemvMaxWarps = 16;

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
    int tn, rg, stages;    // tile width, row groups, ring depth (stages per warp)
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

__host__ __device__ constexpr size_t gemv_ring_bytes(int nwarps, int stages) {
    return (size_t)nwarps * stages * kStageBytes;
}
// tail scratch (aliases the ring): part [RG][BP][TN] + pred [BP][TN] + fin [TN][BP]
__host__ __device__ constexpr size_t gemv_tail_bytes(int rg, int bp, int tn) {
    return ((size_t)rg * bp * tn + 2 * (size_t)bp * tn) * 4;
}
__host__ __device__ constexpr size_t gemv_smem_bytes(int nwarps, int stages, int rg, int bp, int tn) {
    return 1024 + (gemv_ring_bytes(nwarps, stages) > gemv_tail_bytes(rg, bp, tn) ? gemv_ring_bytes(nwarps, stages)
                                                                                   : gemv_tail_bytes(rg, bp, tn));
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.0f + expf(-g)); }

// cp.async (LDGSTS): 16 bytes global -> shared, bypassing L1 (.cg)
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
constexpr int kMaxStagesM1 = 15;   // ring depth <= 16
// wait until at most n of this thread's most recent groups are pending (n runtime <= MAXN)
template <int MAXN>
__device__ __forceinline__ void cp_async_wait(int n) {
    if constexpr (MAXN <= 0) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    } else {
        if (n >= MAXN) asm volatile("cp.async.wait_group %0;" ::"n"(MAXN) : "memory");
        else cp_async_wait<MAXN - 1>(n);
    }
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_map(uint32_t local_smem_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem_addr), "r"(rank));
    return r;
}
__device__ __forceinline__ float ld_dsmem(uint32_t addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}

template <int BP>
__global__ void __launch_bounds__(BP >= 8 ? 256 : kGemvMaxWarps * 32, 1) gemv_kernel(const GemvArgs a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int CS = gridDim.x;                 // cluster spans x: blockIdx.x == rank
    const int split = blockIdx.x, tile = blockIdx.y;
    const int TN = a.tn, RG = a.rg, ST = a.stages;
    const int slices = TN / kWarpCols;
    const int nwarps = slices * RG;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cs = warp % slices, rg = warp / slices;
    unsigned char* ring = smem + 1024;                           // [nwarps][ST][kStageBytes]
    float* part = reinterpret_cast<float*>(ring);                // reused: [RG][BP][TN]

    pdl_wait();       // rows / vals / nrows come from the previous kernel
    pdl_trigger();

    const int nrows = a.nrows_dev ? *a.nrows_dev : a.nrows;
    const int rps = (nrows + CS - 1) / CS;
    const int r_begin = min(nrows, split * rps);
    const int r_end = min(nrows, r_begin + rps);
    const int n_my = r_end - r_begin > rg ? (r_end - r_begin - rg + RG - 1) / RG : 0;   // my rows: r_begin + rg + RG*m
    const int col0 = tile * TN + cs * kWarpCols;
    const bool lane_on = col0 + lane * 8 < a.d_out;     // this lane's 16-byte chunk exists
    const int n_st = (n_my + kStageRows - 1) / kStageRows;
    // each lane copies, and later reads back, only its own 16-byte chunk of every row: the
    // staging needs no cross-lane synchronisation, only the lane's own cp.async groups
    unsigned char* mychunk = ring + (size_t)warp * ST * kStageBytes + lane * 16;
    const uint16_t* wcol = a.W + col0 + lane * 8;

    // Row indices / token values are read in 32-row windows (lane j holds my-row base + j),
    // double-buffered: the next window's loads are in flight while the current one is used,
    // so the steady state never waits on them.
    auto load_row = [&](int m) -> int {
        const int r = r_begin + rg + RG * m;
        return m < n_my ? (a.rows ? __ldg(a.rows + r) : r) : 0;
    };
    int iw_base = 0;
    int iw_row = load_row(lane);
    int iw_next = load_row(32 + lane);
    auto issue = [&](int st) {
        if (st < n_st) {
            const int m0 = st * kStageRows;
            if (m0 >= iw_base + 32) {        // advance one window (kStageRows divides 32)
                iw_base += 32;
                iw_row = iw_next;
                iw_next = load_row(iw_base + 32 + lane);
            }
            const int gc = min(kStageRows, n_my - m0);
            unsigned char* dst = mychunk + (size_t)(st % ST) * kStageBytes;
#pragma unroll
            for (int g = 0; g < kStageRows; ++g) {
                const int row = __shfl_sync(0xffffffffu, iw_row, (m0 - iw_base + g) & 31);
                if (g < gc && lane_on) cp_async16(dst + g * (kWarpCols * 2), wcol + (size_t)row * a.ld);
            }
        }
        cp_async_commit();   // (possibly empty) group per stage keeps the group count uniform
    };
    for (int st = 0; st < ST; ++st) issue(st);

    float acc[BP][8];
#pragma unroll
    for (int b = 0; b < BP; ++b)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[b][j] = 0.f;

    auto load_vals = [&](int m, float* v) {
        const size_t r = (size_t)(r_begin + rg + RG * m);
#pragma unroll
        for (int b = 0; b < BP; ++b)
            v[b] = (m < n_my && b < a.batch) ? __ldg(a.vals + r * a.vs_r + (size_t)b * a.vs_b) : 0.f;
    };
    int vw_base = 0;
    float vwin[BP], vnext[BP];
    load_vals(lane, vwin);
    load_vals(32 + lane, vnext);
    for (int st = 0; st < n_st; ++st) {
        const int m0 = st * kStageRows;
        if (m0 >= vw_base + 32) {
            vw_base += 32;
#pragma unroll
            for (int b = 0; b < BP; ++b) vwin[b] = vnext[b];
            load_vals(vw_base + 32 + lane, vnext);
        }
        const int gc = min(kStageRows, n_my - m0);
        cp_async_wait<kMaxStagesM1>(ST - 1);    // this lane's chunks of stage st have landed
        const unsigned char* src = mychunk + (size_t)(st % ST) * kStageBytes;
#pragma unroll
        for (int g = 0; g < kStageRows; ++g) {
            if (g < gc) {
                const uint4 w = lds128(src + g * (kWarpCols * 2));
                float wf[8];
                wf[0] = bf16lo(w.x); wf[1] = bf16hi(w.x);
                wf[2] = bf16lo(w.y); wf[3] = bf16hi(w.y);
                wf[4] = bf16lo(w.z); wf[5] = bf16hi(w.z);
                wf[6] = bf16lo(w.w); wf[7] = bf16hi(w.w);
                const int src_lane = (m0 - vw_base + g) & 31;
#pragma unroll
                for (int b = 0; b < BP; ++b) {
                    const float v = __shfl_sync(0xffffffffu, vwin[b], src_lane);
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[b][j] = fmaf(v, wf[j], acc[b][j]);
                }
            }
        }
        issue(st + ST);
    }
    cp_async_wait<kMaxStagesM1>(0);
    if (!lane_on) {
#pragma unroll
        for (int b = 0; b < BP; ++b)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[b][j] = 0.f;
    }

    // ---------------- publish this CTA's partial tile: part[rg][b][cs*256 + lane*8 + j] --------
    __syncthreads();   // every warp is done reading its ring (part aliases it)
#pragma unroll
    for (int b = 0; b < BP; ++b) {
        float* p = part + ((size_t)rg * BP + b) * TN + cs * kWarpCols + lane * 8;
        reinterpret_cast<float4*>(p)[0] = make_float4(acc[b][0], acc[b][1], acc[b][2], acc[b][3]);
        reinterpret_cast<float4*>(p)[1] = make_float4(acc[b][4], acc[b][5], acc[b][6], acc[b][7]);
    }
    __syncthreads();
    // local row-group reduction (fixed order): pred[b][c] = sum_g part[g][b][c]
    const int nthreads = nwarps * 32;
    float* pred = part + (size_t)RG * BP * TN;             // [BP][TN]
    float* fin = pred + (size_t)BP * TN;                    // [2 * pairs-per-CTA][BP]
    for (int t = threadIdx.x; t < a.batch * TN; t += nthreads) {
        const int b = t / TN, c = t % TN;
        float v = 0.f;
        for (int g = 0; g < RG; ++g) v += part[((size_t)g * BP + b) * TN + c];
        pred[(size_t)b * TN + c] = v;
    }
    cluster_sync_all();

    // ---------------- cluster reduction over the CS CTAs (fixed order, DSMEM) ----------------
    const int po = (a.ep == EP_QKV_ROPE) ? (a.hd >> 1) : kGuBlock;   // pair offset
    const int npairs = TN >> 1;
    const int ppc = (npairs + CS - 1) / CS;                            // pairs per CTA
    const int p_begin = min(npairs, split * ppc), p_end = min(npairs, p_begin + ppc);
    const int nmine = p_end - p_begin;
    const uint32_t pred_local = smem_u32(pred);
    for (int t = threadIdx.x; t < nmine * 2 * a.batch; t += nthreads) {
        const int b = t % a.batch;
        const int pi = (t / a.batch) >> 1, half = (t / a.batch) & 1;
        const int pj = p_begin + pi;
        const int c = (pj / po) * (2 * po) + (pj % po) + half * po;
        const uint32_t off = (uint32_t)(((size_t)b * TN + c) * 4);
        float v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = q < CS ? ld_dsmem(cluster_map(pred_local + off, (uint32_t)q)) : 0.f;
        float y = 0.f;
#pragma unroll
        for (int q = 0; q < 16; ++q) y += v[q];
        fin[(size_t)(pi * 2 + half) * BP + b] = y;
    }
    __syncthreads();

    // ---------------- epilogue on complete column pairs (c1, c1 + po) ----------------
    for (int t = threadIdx.x; t < nmine * a.batch; t += nthreads) {
        const int b = t % a.batch, pi = t / a.batch;
        const int pj = p_begin + pi;
        const int c1 = (pj / po) * (2 * po) + (pj % po);
        const int c2 = c1 + po;
        const int o1 = tile * TN + c1, o2 = tile * TN + c2;
        float y1 = fin[(size_t)(pi * 2) * BP + b];
        float y2 = fin[(size_t)(pi * 2 + 1) * BP + b];
        const bool in1 = o1 < a.d_out, in2 = o2 < a.d_out;
        if (a.bias && a.ep != EP_SILU_GU) {
            if (in1) y1 += bf16f(a.bias[o1]);
            if (in2) y2 += bf16f(a.bias[o2]);
        }
        if (a.ep == EP_STORE || a.ep == EP_RESID) {
            float* op = a.out + (size_t)b * a.out_ld;
            if (a.ep == EP_RESID) {
                const float* rp = a.resid + (size_t)b * a.resid_ld;
                if (in1) y1 = rp[o1] + y1;
                if (in2) y2 = rp[o2] + y2;
            }
            if (in1) op[o1] = y1;
            if (in2) op[o2] = y2;
        } else if (a.ep == EP_SILU_GU) {
            // fused block t = o1 / 128: gate [t*64, t*64+64) then up of the same rows
            const int i = (o1 / (2 * kGuBlock)) * kGuBlock + (o1 % (2 * kGuBlock));
            a.out[(size_t)b * a.out_ld + i] = silu_f(y1) * y2;
        } else {   // EP_QKV_ROPE: (o1, o2) = head dims (i, i + hd/2) of one head
            const int hd = a.hd;
            const int nq = a.hq * hd, nk = a.hkv * hd;
            const int p = a.pos[b];
            float r1 = y1, r2 = y2;
            if (o1 < nq + nk) {
                const int i = o1 % hd;
                const double inv_freq = exp(-(2.0 * i / hd) * log((double)a.theta));
                double sn, cn;
                sincos((double)p * inv_freq, &sn, &cn);
                r1 = (float)((double)y1 * cn - (double)y2 * sn);
                r2 = (float)((double)y2 * cn + (double)y1 * sn);
            }
            if (o1 < nq) {
                float* op = a.out + (size_t)b * a.out_ld;
                op[o1] = r1;
                op[o2] = r2;
            } else {
                const bool isk = o1 < nq + nk;
                const int oo = o1 - (isk ? nq : nq + nk);
                const int kvh = oo / hd, i = oo % hd;
                uint16_t* dst = (isk ? a.kc : a.vc) + (((size_t)b * a.hkv + kvh) * a.max_ctx + p) * hd;
                dst[i] = f2bf16_rne(r1);
                dst[i + (hd >> 1)] = f2bf16_rne(r2);
            }
        }
    }
    cluster_sync_all();   // keep every CTA's partial alive until all peers finished reading
}

}  // namespace larosa
