// larosa.cu — host side of the C ABI declared in include/larosa.h: argument validation,
// workspace carving, launch configuration (grids sized to the 148-SM B200), programmatic
// dependent launch, thread-local error strings.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "larosa.h"
#include "common.cuh"
#include "topk.cuh"
#include "gemv.cuh"
#include "attention.cuh"
#include "aux.cuh"
#include "thresh.cuh"
#include "fold_tc.cuh"

using namespace larosa;

static_assert(LAROSA_GU_BLOCK == kGuBlock, "gate|up interleave block mismatch");

// ============================================================================== errors
namespace {
thread_local std::string g_err;

larosa_status fail(larosa_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

larosa_status cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) return fail(LAROSA_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return LAROSA_OK;
}

#define LAROSA_TRY(expr)                          \
    do {                                          \
        larosa_status _s = (expr);                \
        if (_s != LAROSA_OK) return _s;           \
    } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (cached[dev] == 0) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cached[dev] = n;
    }
    return cached[dev];
}

bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("LAROSA_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Opt a kernel in to > 48 KB dynamic shared memory once per process (per function).
template <typename K>
cudaError_t allow_smem(K kern, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// ============================================================================== workspace
// Every workspace starts with a fixed header of self-resetting counters, followed by the
// call's fixed-point GEMV accumulators; both are zero at rest (kernels restore the zeros),
// so the caller zero-fills a workspace once.  A workspace must be reused only for calls of
// the same kind and shapes (other layouts would place live data where accumulators were).
constexpr size_t kCounterHeaderWords = 8192;   // attention tickets
constexpr size_t kAttnCounterBase = 0;

struct Carver {
    char* base;      // nullptr -> size query
    size_t off = kCounterHeaderWords * sizeof(unsigned);
    explicit Carver(void* b) : base(static_cast<char*>(b)) {}
    unsigned* counters(size_t first) const {
        return base ? reinterpret_cast<unsigned*>(base) + first : nullptr;
    }
    template <typename T>
    T* take(size_t n) {
        off = (off + 255) & ~size_t(255);
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += n * sizeof(T);
        return p;
    }
    size_t size() const { return (off + 255) & ~size_t(255); }
};

int pad_batch(int b) { return b <= 1 ? 1 : b <= 2 ? 2 : b <= 4 ? 4 : b <= 8 ? 8 : 16; }

// ============================================================================== GEMV plan
struct GemvPlan {
    int n_slices, n_splits, list_cap;
    size_t smem;
};

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}

int gemv_list_max(int bp) { return bp <= 2 ? 2048 : 1024; }

// 256-column slices x row splits, about `per_sm` 256-thread CTAs per SM in one wave.
// rows_per_split_src: the number of candidate rows a split may hold (list length for
// GEMV_LIST, input length for GEMV_THRESH / GEMV_DENSE), bounded by the shared list.
GemvPlan plan_gemv(int64_t d_out, int64_t rows_src, int bp) {
    static const int per_sm_env = env_int("LAROSA_GEMV_CTAS_PER_SM", 0);   // tuning knob (0 = auto)
    GemvPlan p;
    p.n_slices = (int)((d_out + kSliceCols - 1) / kSliceCols);
    const int per_sm = per_sm_env > 0 ? per_sm_env : (bp <= 4 ? 2 : 1);
    const int target = sm_count() * per_sm;
    const int by_target = std::max(1, (target + p.n_slices / 2) / p.n_slices);
    const int by_rows = (int)std::max<int64_t>(1, rows_src / 16);
    const int lmax = gemv_list_max(bp);
    const int by_cap = (int)std::max<int64_t>(1, (rows_src + lmax - 1) / lmax);
    p.n_splits = std::max(by_cap, std::min(by_target, by_rows));
    p.list_cap = (int)std::max<int64_t>(32, (rows_src + p.n_splits - 1) / p.n_splits);
    p.smem = gemv_smem_bytes(bp, p.list_cap);
    return p;
}

template <int BP>
larosa_status launch_gemv_bp(const GemvArgs& a, const GemvPlan& p, cudaStream_t st) {
    auto kern = gemv_kernel<BP>;
    static bool attr_done = false;
    if (!attr_done) {
        LAROSA_TRY(cuda_check(allow_smem(kern, gemv_smem_bytes(BP, gemv_list_max(BP))), "cudaFuncSetAttribute(gemv)"));
        attr_done = true;
    }
    GemvArgs aa = a;
    aa.n_splits = p.n_splits;
    aa.list_cap = p.list_cap;
    return cuda_check(launch(kern, dim3(p.n_slices, p.n_splits), dim3(kGemvWarps * 32), p.smem, st, aa), "gemv launch");
}

larosa_status launch_gemv(const GemvArgs& a, const GemvPlan& p, int bp, cudaStream_t st) {
    switch (bp) {
        case 1: return launch_gemv_bp<1>(a, p, st);
        case 2: return launch_gemv_bp<2>(a, p, st);
        case 4: return launch_gemv_bp<4>(a, p, st);
        case 8: return launch_gemv_bp<8>(a, p, st);
        default: return launch_gemv_bp<16>(a, p, st);
    }
}

GemvArgs gemv_args_base() {
    GemvArgs a;
    memset(&a, 0, sizeof(a));
    return a;
}

// ============================================================================== small launches
template <int MODE, int EPT>
larosa_status launch_topk_t(const TopkKernelArgs& a, int batch, cudaStream_t st) {
    auto kern = topk_kernel<MODE, EPT>;
    static bool attr_done = false;
    if (!attr_done) {
        LAROSA_TRY(cuda_check(allow_smem(kern, topk_smem_bytes(LAROSA_MAX_DIM)), "cudaFuncSetAttribute(topk)"));
        attr_done = true;
    }
    const int cs = topk_cluster_size(a.d);   // one cluster of cs CTAs per token
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs, batch);
    cfg.blockDim = dim3(kTopkThreads);
    cfg.dynamicSmemBytes = topk_smem_bytes(a.d);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (!pdl_enabled()) {
        at[0] = at[0];
        cfg.numAttrs = 1;
    }
    return cuda_check(cudaLaunchKernelEx(&cfg, kern, a), "topk launch");
}

template <int MODE>
larosa_status launch_topk_m(const TopkKernelArgs& a, int batch, cudaStream_t st) {
    const int ept = topk_ept(a.d);
    if (ept <= 2) return launch_topk_t<MODE, 2>(a, batch, st);
    if (ept <= 4) return launch_topk_t<MODE, 4>(a, batch, st);
    if (ept <= 6) return launch_topk_t<MODE, 6>(a, batch, st);
    return launch_topk_t<MODE, 8>(a, batch, st);
}

larosa_status launch_topk(const TopkKernelArgs& a, int batch, cudaStream_t st) {
    if (a.mode == SRC_RESID_ACC) return launch_topk_m<SRC_RESID_ACC>(a, batch, st);
    if (a.mode == SRC_SILU_GU) return launch_topk_m<SRC_SILU_GU>(a, batch, st);
    return launch_topk_m<SRC_PLAIN>(a, batch, st);
}

TopkKernelArgs topk_args_base() {
    TopkKernelArgs t;
    memset(&t, 0, sizeof(t));
    t.mode = SRC_PLAIN;
    return t;
}

larosa_status launch_union(const uint32_t* mask, int nwords, int batch, int bp, const float* vals, int64_t k, int d,
                           int32_t* rows, float* V, int* nrows, cudaStream_t st) {
    const int grid = (nwords + 31) / 32;
    return cuda_check(launch(union_kernel, dim3(grid), dim3(kUnionThreads), 0, st, mask, nwords, batch, bp, vals, k, d,
                             rows, V, nrows),
                      "union launch");
}

larosa_status launch_finalize(const FinalizeArgs& f, cudaStream_t st) {
    const int64_t total = (int64_t)f.batch * std::max(f.n, f.zero3_n);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 2 * sm_count()));
    return cuda_check(launch(finalize_kernel, dim3(grid), dim3(256), 0, st, f), "finalize launch");
}

FinalizeArgs finalize_args_base() {
    FinalizeArgs f;
    memset(&f, 0, sizeof(f));
    return f;
}

}  // namespace

// ============================================================================== basics
extern "C" int larosa_abi_version(void) { return LAROSA_ABI_VERSION; }

extern "C" const char* larosa_status_string(int s) {
    switch (s) {
        case LAROSA_OK: return "LAROSA_OK";
        case LAROSA_EINVAL: return "LAROSA_EINVAL: invalid argument";
        case LAROSA_ESHAPE: return "LAROSA_ESHAPE: inconsistent shapes";
        case LAROSA_EUNSUPPORTED: return "LAROSA_EUNSUPPORTED: unsupported configuration";
        case LAROSA_ECUDA: return "LAROSA_ECUDA: CUDA error";
        case LAROSA_ENCCL: return "LAROSA_ENCCL: collective error";
        case LAROSA_EWORKSPACE: return "LAROSA_EWORKSPACE: workspace too small";
        default: return "LAROSA_?: unknown status";
    }
}

extern "C" const char* larosa_last_error(void) { return g_err.c_str(); }

extern "C" larosa_status larosa_compute_k(double alpha, double p, int64_t d_in, int64_t* k_out) {
    if (!k_out) return fail(LAROSA_EINVAL, "compute_k: k_out is NULL");
    if (d_in <= 0) return fail(LAROSA_EINVAL, "compute_k: d_in must be > 0");
    if (!(p >= 0.0 && p <= 1.0)) return fail(LAROSA_EINVAL, "compute_k: p outside [0, 1]");
    if (!(alpha >= 0.0)) return fail(LAROSA_EINVAL, "compute_k: alpha < 0");
    if (p == 0.0) {            // dense "0%" configuration (Z16)
        *k_out = d_in;
        return LAROSA_OK;
    }
    const double v = alpha * (1.0 - p) * (double)d_in;
    int64_t k = (int64_t)std::floor(v + 0.5);              // half away from zero (v >= 0)
    if (k < 0) k = 0;
    if (k > d_in) k = d_in;
    *k_out = k;
    return LAROSA_OK;
}

extern "C" larosa_status larosa_solve_alpha(double a1, double a3, double m, double* a2, double* a4) {
    if (!a2 || !a4) return fail(LAROSA_EINVAL, "solve_alpha: NULL output");
    if (!(m > 0.0)) return fail(LAROSA_EINVAL, "solve_alpha: M must be > 0");
    const double x2 = 4.0 - 3.0 * a1;             // 3 a1 + a2 = 4
    const double x4 = (2.0 + m - 2.0 * a3) / m;   // 2 a3 + M a4 = 2 + M
    if (!(x2 > 0.0) || !(x4 > 0.0)) return fail(LAROSA_EINVAL, "solve_alpha: infeasible coefficients");
    *a2 = x2;
    *a4 = x4;
    return LAROSA_OK;
}

// ============================================================================== sparse GEMV
static void carve_sparse_gemv(Carver& c, int32_t batch, int64_t d_in, int64_t d_out, unsigned long long** acc,
                              uint32_t** mask, int32_t** rows, float** V, int** nrows) {
    const int bp = pad_batch(batch);
    unsigned long long* a = c.take<unsigned long long>((size_t)batch * d_out);
    if (acc) *acc = a;
    if (batch > 1) {
        const int64_t nw = (d_in + 31) / 32;
        uint32_t* m = c.take<uint32_t>((size_t)batch * nw);
        int32_t* r = c.take<int32_t>((size_t)d_in);
        float* v = c.take<float>((size_t)d_in * bp + 16);
        int* n = c.take<int>(4);
        if (mask) *mask = m;
        if (rows) *rows = r;
        if (V) *V = v;
        if (nrows) *nrows = n;
    }
}

extern "C" size_t larosa_sparse_gemv_workspace_size(int32_t batch, int64_t d_in, int64_t k, int64_t d_out) {
    if (batch < 1 || d_in <= 0 || d_out <= 0 || k < 0) return 0;
    Carver c(nullptr);
    carve_sparse_gemv(c, batch, d_in, d_out, nullptr, nullptr, nullptr, nullptr, nullptr);
    return c.size();
}

extern "C" larosa_status larosa_sparse_gemv(const uint16_t* W, int64_t d_in, int64_t d_out, int64_t ld,
                                            const int32_t* idx, const float* vals, int32_t batch, int64_t k,
                                            const uint16_t* bias, float* y, void* ws, size_t ws_bytes,
                                            larosa_stream_t stream) {
    if (!W || !y) return fail(LAROSA_EINVAL, "sparse_gemv: W or y is NULL");
    if (k > 0 && (!idx || !vals)) return fail(LAROSA_EINVAL, "sparse_gemv: idx/vals NULL with k > 0");
    if (d_in <= 0 || d_out <= 0) return fail(LAROSA_EINVAL, "sparse_gemv: d_in, d_out must be > 0");
    if (batch < 1) return fail(LAROSA_EINVAL, "sparse_gemv: batch < 1");
    if (batch > LAROSA_MAX_BATCH) return fail(LAROSA_EUNSUPPORTED, "sparse_gemv: batch > %d", LAROSA_MAX_BATCH);
    if (k < 0 || k > d_in) return fail(LAROSA_EINVAL, "sparse_gemv: k=%lld outside [0, d_in=%lld]", (long long)k, (long long)d_in);
    if (ld < d_out) return fail(LAROSA_ESHAPE, "sparse_gemv: ld < d_out");
    if (ld % 8 || d_out % 8) return fail(LAROSA_EUNSUPPORTED, "sparse_gemv: ld and d_out must be multiples of 8");
    if (!aligned16(W)) return fail(LAROSA_EINVAL, "sparse_gemv: W must be 16-byte aligned");
    if (!aligned16(y) || (bias && !aligned16(bias)))
        return fail(LAROSA_EINVAL, "sparse_gemv: W, y, bias must be 16-byte aligned");
    if (d_in > INT32_MAX || d_out > INT32_MAX) return fail(LAROSA_EUNSUPPORTED, "sparse_gemv: dims too large");
    const size_t need = larosa_sparse_gemv_workspace_size(batch, d_in, k, d_out);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "sparse_gemv: workspace %zu < %zu", ws_bytes, need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);

    Carver c(ws);
    unsigned long long* acc = nullptr;
    uint32_t* mask = nullptr;
    int32_t* rows = nullptr;
    float* V = nullptr;
    int* nrows = nullptr;
    carve_sparse_gemv(c, batch, d_in, d_out, &acc, &mask, &rows, &V, &nrows);
    const int bp = pad_batch(batch);
    const int64_t nrows_max = batch == 1 ? k : std::min<int64_t>(d_in, (int64_t)batch * k);
    const GemvPlan p = plan_gemv(d_out, nrows_max, bp);

    GemvArgs a = gemv_args_base();
    a.W = W;
    a.ld = ld;
    a.d_out = (int)d_out;
    a.mode = GEMV_LIST;
    a.batch = batch;
    a.acc = acc;
    a.acc_ld = d_out;
    if (batch == 1) {
        a.rows = idx;
        a.vals = vals;
        a.vs_r = 1;
        a.vs_b = k;
        a.nrows = (int)k;
    } else {
        const int nw = (int)((d_in + 31) / 32);
        LAROSA_TRY(cuda_check(cudaMemsetAsync(mask, 0, sizeof(uint32_t) * (size_t)batch * nw, st), "memset mask"));
        if (k > 0) {
            const int64_t n = (int64_t)batch * k;
            const int grid = (int)std::min<int64_t>((n + 255) / 256, 4096);
            LAROSA_TRY(cuda_check(launch(idx_to_mask_kernel, dim3(grid), dim3(256), 0, st, idx, k, (int)batch, nw, mask),
                                  "idx_to_mask launch"));
        }
        LAROSA_TRY(launch_union(mask, nw, batch, bp, vals, k, (int)d_in, rows, V, nrows, st));
        a.rows = rows;
        a.vals = V;
        a.vs_r = bp;
        a.vs_b = 1;
        a.nrows_dev = nrows;
    }
    LAROSA_TRY(launch_gemv(a, p, bp, st));
    FinalizeArgs f = finalize_args_base();
    f.n = (int)d_out;
    f.batch = batch;
    f.acc1 = acc;
    f.acc1_ld = d_out;
    f.bias1 = bias;
    f.out1 = y;
    f.out1_ld = d_out;
    return launch_finalize(f, st);
}

extern "C" larosa_status larosa_gemv_plan_info(int64_t d_out, int64_t nrows_max, int32_t batch, int32_t* info) {
    if (!info || d_out <= 0 || nrows_max < 0 || batch < 1 || batch > LAROSA_MAX_BATCH)
        return fail(LAROSA_EINVAL, "gemv_plan_info: bad arguments");
    const GemvPlan p = plan_gemv(d_out, nrows_max, pad_batch(batch));
    info[0] = kSliceCols;
    info[1] = p.n_slices;
    info[2] = p.n_splits;
    info[3] = kGemvWarps;
    info[4] = kStages;
    info[5] = kStageRows;
    info[6] = (int32_t)p.smem;
    info[7] = p.n_slices * p.n_splits;
    return LAROSA_OK;
}

// ============================================================================== rotate + Top-K
static void carve_rotate_topk(Carver& c, int32_t batch, int64_t d, unsigned long long** acc, float** xbuf) {
    unsigned long long* a = c.take<unsigned long long>((size_t)batch * d);
    float* x = c.take<float>((size_t)batch * d);
    if (acc) *acc = a;
    if (xbuf) *xbuf = x;
}

extern "C" size_t larosa_rotate_topk_workspace_size(int32_t batch, int64_t d) {
    if (batch < 1 || d <= 0) return 0;
    Carver c(nullptr);
    carve_rotate_topk(c, batch, d, nullptr, nullptr);
    return c.size();
}

extern "C" larosa_status larosa_rotate_topk(const float* x, const uint16_t* R, int32_t batch, int64_t d, int64_t k,
                                            float rms_eps, float* xr_out, int32_t* idx, float* vals, uint32_t* mask,
                                            void* ws, size_t ws_bytes, larosa_stream_t stream) {
    if (!x) return fail(LAROSA_EINVAL, "rotate_topk: x is NULL");
    if (k > 0 && (!idx || !vals)) return fail(LAROSA_EINVAL, "rotate_topk: idx/vals NULL with k > 0");
    if (batch < 1) return fail(LAROSA_EINVAL, "rotate_topk: batch < 1");
    if (batch > LAROSA_MAX_BATCH) return fail(LAROSA_EUNSUPPORTED, "rotate_topk: batch > %d", LAROSA_MAX_BATCH);
    if (d <= 0) return fail(LAROSA_EINVAL, "rotate_topk: d must be > 0");
    if (d > LAROSA_MAX_DIM) return fail(LAROSA_EUNSUPPORTED, "rotate_topk: d > %d", LAROSA_MAX_DIM);
    if (k < 0 || k > d) return fail(LAROSA_EINVAL, "rotate_topk: k outside [0, d]");
    if (R && d % 8) return fail(LAROSA_EUNSUPPORTED, "rotate_topk: d must be a multiple of 8 when R != NULL");
    if (R && !aligned16(R)) return fail(LAROSA_EINVAL, "rotate_topk: R must be 16-byte aligned");
    if (R && xr_out == x) return fail(LAROSA_EINVAL, "rotate_topk: xr_out aliases x with R != NULL");
    const size_t need = larosa_rotate_topk_workspace_size(batch, d);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "rotate_topk: workspace %zu < %zu", ws_bytes, need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Carver c(ws);
    unsigned long long* acc;
    float* xbuf;
    carve_rotate_topk(c, batch, d, &acc, &xbuf);

    TopkKernelArgs t = topk_args_base();
    t.ldx = d;
    t.d = (int)d;
    t.k = (int)k;
    t.rms_eps = rms_eps;
    t.xr_out = xr_out;
    t.idx = idx;
    t.vals = vals;
    t.mask = mask;
    if (R) {
        // dense rotation GEMV x . R over all d rows (token-major values), then the Top-K
        // kernel finalises the fixed-point accumulators into x~
        const int bp = pad_batch(batch);
        const GemvPlan p = plan_gemv(d, d, bp);
        GemvArgs a = gemv_args_base();
        a.W = R;
        a.ld = d;
        a.d_out = (int)d;
        a.mode = GEMV_DENSE;
        a.x = x;
        a.ldx = d;
        a.d_in = (int)d;
        a.batch = batch;
        a.acc = acc;
        a.acc_ld = d;
        LAROSA_TRY(launch_gemv(a, p, bp, st));
        t.mode = SRC_RESID_ACC;
        t.acc = acc;
        t.acc_ld = d;
        if (!xr_out) t.xr_out = xbuf;   // the finalised x~ must be materialised for the select
    } else {
        t.x = x;
    }
    return launch_topk(t, batch, st);
}

// ============================================================================== fold
extern "C" size_t larosa_fold_workspace_size(int64_t rows, int64_t cols, int side) {
    if (rows <= 0 || cols <= 0) return 0;
    return fold_tc_workspace_bytes(rows, cols, side == LAROSA_LEFT_QT);
}

extern "C" larosa_status larosa_fold_rotation(const float* Q, const float* gamma, const uint16_t* W, uint16_t* Wout,
                                              int64_t rows, int64_t cols, int side, void* ws, size_t ws_bytes,
                                              larosa_stream_t stream) {
    if (!Q || !W || !Wout) return fail(LAROSA_EINVAL, "fold: NULL pointer");
    if (side != LAROSA_LEFT_QT && side != LAROSA_RIGHT_Q) return fail(LAROSA_EINVAL, "fold: bad side");
    if (rows <= 0 || cols <= 0) return fail(LAROSA_EINVAL, "fold: rows, cols must be > 0");
    if (side == LAROSA_RIGHT_Q && gamma) return fail(LAROSA_EINVAL, "fold: gamma must be NULL for RIGHT_Q");
    if ((const void*)W == (const void*)Wout) return fail(LAROSA_EINVAL, "fold: Wout aliases W");
    if (rows % 64 || cols % 64) return fail(LAROSA_EUNSUPPORTED, "fold: rows and cols must be multiples of 64");
    if (rows > INT32_MAX / 2 || cols > INT32_MAX / 2) return fail(LAROSA_EUNSUPPORTED, "fold: dims too large");
    const size_t need = larosa_fold_workspace_size(rows, cols, side);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "fold: workspace %zu < %zu", ws_bytes, need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const char* simt = getenv("LAROSA_FOLD_SIMT");
    if (simt && simt[0] == '1') {
        const bool left = side == LAROSA_LEFT_QT;
        const int M = (int)rows, N = (int)cols, K = left ? (int)rows : (int)cols;
        dim3 grid((N + 63) / 64, (M + 63) / 64);
        if (left)
            return cuda_check(launch(fold_simt_kernel<true>, grid, dim3(256), 0, st, Q, gamma, W, Wout, M, N, K), "fold");
        return cuda_check(launch(fold_simt_kernel<false>, grid, dim3(256), 0, st, Q, gamma, W, Wout, M, N, K), "fold");
    }
    return cuda_check(fold_tc_run(Q, gamma, W, Wout, rows, cols, side == LAROSA_LEFT_QT, ws, st), "fold (tcgen05)");
}

extern "C" larosa_status larosa_pack_gate_up(const uint16_t* Wg, const uint16_t* Wu, uint16_t* Wgu, int64_t d,
                                             int64_t inter, larosa_stream_t stream) {
    if (!Wg || !Wu || !Wgu) return fail(LAROSA_EINVAL, "pack_gate_up: NULL pointer");
    if (d <= 0 || inter <= 0) return fail(LAROSA_EINVAL, "pack_gate_up: dims must be > 0");
    if (inter % LAROSA_GU_BLOCK) return fail(LAROSA_EUNSUPPORTED, "pack_gate_up: inter %% %d != 0", LAROSA_GU_BLOCK);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t n = d * 2 * inter;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 64);
    return cuda_check(launch(pack_gate_up_kernel, dim3(grid), dim3(256), 0, st, Wg, Wu, Wgu, d, inter), "pack_gate_up");
}

// ============================================================================== decoder layer
namespace {
struct SiteWs {
    uint32_t* ghist;      // [B][4096]  zero at rest
    unsigned* ticket;     // [B]        zero at rest
    float* ssq;           // [B][NB]
    ThreshOut* thr;       // [B]
};

struct LayerWs {
    unsigned long long *acc_qkv, *acc_o, *acc_gu, *acc_down, *acc_adp;
    SiteWs site[4];
    float* h2;
    float* rmid;
    float* h4;
    float* attn_part;
    unsigned* attn_cnt;
};

struct LayerDims {
    int64_t d, inter, hq, hkv, hd, nq, nqkv, dgu;
    int G;
};

LayerDims layer_dims(const larosa_layer_weights* w) {
    LayerDims L;
    L.d = w->d;
    L.inter = w->inter;
    L.hq = w->n_q_heads;
    L.hkv = w->n_kv_heads;
    L.hd = w->head_dim;
    L.nq = L.hq * L.hd;
    L.nqkv = (L.hq + 2 * L.hkv) * L.hd;
    L.dgu = 2 * L.inter;
    L.G = (int)(L.hkv > 0 ? L.hq / L.hkv : 1);
    return L;
}

int attn_chunk(int64_t max_ctx, int units) {
    // enough CTAs to cover the SMs: units * n_chunks >= sm_count
    int ch = 4 * kAttnPosPerWarp;
    while (ch > 16 && units * ((max_ctx + ch - 1) / ch) < sm_count()) ch >>= 1;
    return ch;
}

void carve_layer(Carver& c, const LayerDims& L, int batch, int64_t max_ctx, LayerWs* ws) {
    const int64_t din[4] = {L.d, L.nq, L.d, L.inter};
    LayerWs tmp;
    LayerWs* o = ws ? ws : &tmp;
    // zero-at-rest state first: GEMV accumulators, threshold histograms and tickets
    o->acc_qkv = c.take<unsigned long long>((size_t)batch * L.nqkv);
    o->acc_o = c.take<unsigned long long>((size_t)batch * L.d);
    o->acc_gu = c.take<unsigned long long>((size_t)batch * L.dgu);
    o->acc_down = c.take<unsigned long long>((size_t)batch * L.d);
    o->acc_adp = c.take<unsigned long long>((size_t)batch * L.d);
    for (int s = 0; s < 4; ++s) {
        o->site[s].ghist = c.take<uint32_t>((size_t)batch * kThrBins);
        o->site[s].ticket = c.take<unsigned>((size_t)batch);
    }
    for (int s = 0; s < 4; ++s) {
        o->site[s].ssq = c.take<float>((size_t)batch * thresh_nb((int)din[s]));
        o->site[s].thr = c.take<ThreshOut>((size_t)batch);
    }
    o->h2 = c.take<float>((size_t)batch * L.nq);
    o->rmid = c.take<float>((size_t)batch * L.d);
    o->h4 = c.take<float>((size_t)batch * L.inter);
    const int ch = attn_chunk(max_ctx, batch * (int)L.hkv);
    const int nch = (int)((max_ctx + ch - 1) / ch);
    o->attn_part = c.take<float>((size_t)batch * L.hkv * nch * L.G * (L.hd + 2));
    o->attn_cnt = c.counters(kAttnCounterBase);
}

larosa_status validate_layer(const larosa_layer_weights* w, const larosa_layer_plan* p, const larosa_layer_state* s) {
    if (!w || !p || !s) return fail(LAROSA_EINVAL, "sparse_layer: NULL struct");
    if (!w->w_qkv || !w->w_o || !w->w_gu || !w->w_down) return fail(LAROSA_EINVAL, "sparse_layer: NULL weight");
    if (!s->resid || !s->k_cache || !s->v_cache || !s->pos) return fail(LAROSA_EINVAL, "sparse_layer: NULL state");
    if (s->batch < 1) return fail(LAROSA_EINVAL, "sparse_layer: batch < 1");
    if (s->batch > LAROSA_MAX_BATCH) return fail(LAROSA_EUNSUPPORTED, "sparse_layer: batch > 16");
    if (w->d <= 0 || w->inter <= 0 || w->n_q_heads <= 0 || w->n_kv_heads <= 0 || w->head_dim <= 0)
        return fail(LAROSA_EINVAL, "sparse_layer: dims must be > 0");
    if (w->n_q_heads % w->n_kv_heads) return fail(LAROSA_ESHAPE, "sparse_layer: Hq %% Hkv != 0");
    if (w->n_q_heads / w->n_kv_heads > kAttnMaxG) return fail(LAROSA_EUNSUPPORTED, "sparse_layer: GQA group > 8");
    if (w->head_dim != 64 && w->head_dim != 128) return fail(LAROSA_EUNSUPPORTED, "sparse_layer: head_dim must be 64 or 128");
    if (w->d % 8 || w->inter % LAROSA_GU_BLOCK) return fail(LAROSA_EUNSUPPORTED, "sparse_layer: d %% 8 or inter %% 64");
    if (w->d > LAROSA_MAX_DIM || w->inter > LAROSA_MAX_DIM || w->n_q_heads * w->head_dim > LAROSA_MAX_DIM)
        return fail(LAROSA_EUNSUPPORTED, "sparse_layer: dimension > %d", LAROSA_MAX_DIM);
    if (s->max_ctx <= 0) return fail(LAROSA_EINVAL, "sparse_layer: max_ctx must be > 0");
    if ((int64_t)s->batch * w->n_kv_heads > (int64_t)kCounterHeaderWords)
        return fail(LAROSA_EUNSUPPORTED, "sparse_layer: batch * Hkv too large");
    const int64_t nq = w->n_q_heads * w->head_dim;
    if (p->k_h1 < 0 || p->k_h1 > w->d || p->k_h2 < 0 || p->k_h2 > nq || p->k_h3 < 0 || p->k_h3 > w->d || p->k_h4 < 0 ||
        p->k_h4 > w->inter)
        return fail(LAROSA_EINVAL, "sparse_layer: a k is outside [0, D_in of its site]");
    const void* ptrs[] = {w->w_qkv, w->w_o, w->w_gu, w->w_down, w->adapter, w->b_qkv, s->resid, s->k_cache, s->v_cache};
    for (const void* q : ptrs)
        if (q && !aligned16(q)) return fail(LAROSA_EINVAL, "sparse_layer: pointers must be 16-byte aligned");
    return LAROSA_OK;
}

larosa_status tap_copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (!dst) return LAROSA_OK;
    return cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st), "tap copy");
}

template <int MODE>
larosa_status launch_thresh_m(const ThreshArgs& t, int batch, cudaStream_t st) {
    return cuda_check(launch(thresh_kernel<MODE>, dim3(thresh_nb(t.d), batch), dim3(kThrThreads), 0, st, t),
                      "thresh launch");
}
larosa_status launch_thresh(const ThreshArgs& t, int batch, cudaStream_t st) {
    if (t.mode == THR_RESID_ACC) return launch_thresh_m<THR_RESID_ACC>(t, batch, st);
    if (t.mode == THR_SILU_GU) return launch_thresh_m<THR_SILU_GU>(t, batch, st);
    return launch_thresh_m<THR_PLAIN>(t, batch, st);
}

static_assert((int)THR_PLAIN == (int)SRC_PLAIN && (int)THR_RESID_ACC == (int)SRC_RESID_ACC &&
                  (int)THR_SILU_GU == (int)SRC_SILU_GU,
              "source enums must agree");
// the single-wave ticket threshold kernel (thresh.cuh) instead of the cluster Top-K
bool use_ticket_thresh() {
    static const int v = env_int("LAROSA_THRESH_KERNEL", 0);
    return v != 0;
}

// profiling aid: bitmask of the layer's kernels that are launched (default: all)
int g_phase_mask = -2;
unsigned long long* g_thr_dbg = nullptr;   // device buffer [4][16] of threshold-kernel stamps
int layer_phase_mask() {
    if (g_phase_mask == -2) g_phase_mask = env_int("LAROSA_LAYER_PHASES", -1);
    return g_phase_mask;
}
}  // namespace

extern "C" void larosa_debug_set_layer_phases(int mask) { g_phase_mask = mask; }
extern "C" void larosa_debug_set_thresh_stamps(void* dev_buf) { g_thr_dbg = static_cast<unsigned long long*>(dev_buf); }

extern "C" size_t larosa_layer_workspace_size(const larosa_layer_weights* w, int32_t batch, int64_t max_ctx) {
    if (!w || batch < 1 || max_ctx <= 0) return 0;
    Carver c(nullptr);
    carve_layer(c, layer_dims(w), batch, max_ctx, nullptr);
    return c.size();
}

// Kernel sequence (one decode step of one layer; every kernel is launched with PDL):
//   thresh(h1 = r, RMS)                       -> rule T1, s1
//   gemv(W_qkv, THRESH: rows kept by T1)      -> acc_qkv
//   attention <- acc_qkv (+bias, RoPE, KV append)          -> h2
//   thresh(h2)                                -> T2
//   gemv(W_o, THRESH)                         -> acc_o
//   thresh(h3 = r + acc_o, RMS; zero acc_o)   -> r_mid, T3, s3
//   gemv(W_gate|up, THRESH)                   -> acc_gu
//   thresh(h4 = SiLU(g) * u; zero acc_gu)     -> h4, T4
//   gemv(W_down, THRESH)                      -> acc_down
//   gemv(adapter, DENSE; values r_mid + acc_down)          -> acc_adp          (if adapter)
//   finalize: r <- acc_adp  (or r_mid + acc_down); zero acc_down, acc_adp, acc_qkv
// Taps (parity checks) add exact index-list Top-K launches on the materialised inputs.
extern "C" larosa_status larosa_sparse_layer(const larosa_layer_weights* w, const larosa_layer_plan* plan,
                                             const larosa_layer_state* s, const larosa_layer_taps* taps, void* ws,
                                             size_t ws_bytes, larosa_stream_t stream) {
    LAROSA_TRY(validate_layer(w, plan, s));
    const int phases = layer_phase_mask();
    auto on = [&](int bit) { return (phases >> bit) & 1; };
    const size_t need = larosa_layer_workspace_size(w, s->batch, s->max_ctx);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "sparse_layer: workspace %zu < %zu", ws_bytes, need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const LayerDims L = layer_dims(w);
    const int B = s->batch, bp = pad_batch(B);
    Carver c(ws);
    LayerWs W;
    carve_layer(c, L, B, s->max_ctx, &W);
    larosa_layer_taps T;
    if (taps)
        T = *taps;
    else
        memset(&T, 0, sizeof(T));

    // one site: threshold kernel, optional exact index-list tap, THRESH GEMV
    auto site = [&](int si, ThreshArgs t, int64_t din, int64_t k, const float* xmat, int32_t* tap_idx,
                    float* tap_vals, const uint16_t* Wt, int64_t dout, unsigned long long* acc) -> larosa_status {
        t.d = (int)din;
        t.k = (int)k;
        t.ghist = W.site[si].ghist;
        t.ticket = W.site[si].ticket;
        t.ssq_part = W.site[si].ssq;
        t.out = W.site[si].thr;
        t.dbg = g_thr_dbg ? g_thr_dbg + 32 * si : nullptr;
        if (!on(si == 0 ? 0 : 2 * si + 1)) {
        } else if (use_ticket_thresh()) {
            LAROSA_TRY(launch_thresh(t, B, st));
        } else {
            // cluster Top-K in rule mode: finalises the fused source, emits (Tk, Ti, s)
            TopkKernelArgs r = topk_args_base();
            r.mode = t.mode;   // ThrSrc and TopkSrc share their numbering
            r.x = t.x;
            r.ldx = t.ldx;
            r.d = (int)din;
            r.k = (int)k;
            r.rms_eps = t.rms_eps;
            r.xr_out = t.xout;
            r.resid = t.resid;
            r.resid_ld = t.resid_ld;
            r.acc = t.acc;
            r.acc_ld = t.acc_ld;
            r.rule_out = W.site[si].thr;
            LAROSA_TRY(launch_topk(r, B, st));
        }
        if (tap_idx || tap_vals) {
            // exact ascending index list + values (same rule) for parity checks
            TopkKernelArgs tk = topk_args_base();
            tk.x = xmat;
            tk.ldx = din;
            tk.d = (int)din;
            tk.k = (int)k;
            tk.rms_eps = t.rms_eps;
            tk.idx = tap_idx;
            tk.vals = tap_vals;
            if (tap_idx && tap_vals) LAROSA_TRY(launch_topk(tk, B, st));
        }
        const int bit = si == 0 ? 1 : (si == 1 ? 4 : (si == 2 ? 6 : 8));
        if (!on(bit)) return LAROSA_OK;
        const GemvPlan p = plan_gemv(dout, din, bp);
        GemvArgs a = gemv_args_base();
        a.W = Wt;
        a.ld = dout;
        a.d_out = (int)dout;
        a.mode = GEMV_THRESH;
        a.x = xmat;
        a.ldx = din;
        a.d_in = (int)din;
        a.thr = W.site[si].thr;
        a.batch = B;
        a.acc = acc;
        a.acc_ld = dout;
        return launch_gemv(a, p, bp, st);
    };

    // ---- h1: r (RMS scale) -> QKV -------------------------------------------------------------
    {
        ThreshArgs t;
        memset(&t, 0, sizeof(t));
        t.mode = THR_PLAIN;
        t.x = s->resid;
        t.ldx = L.d;
        t.rms_eps = w->rms_eps;
        LAROSA_TRY(site(0, t, L.d, plan->k_h1, s->resid, T.idx_h1, T.vals_h1, w->w_qkv, L.nqkv, W.acc_qkv));
    }
    // ---- attention (finalises q / new k, v from acc_qkv) -------------------------------------
    {
        AttnArgs aa;
        memset(&aa, 0, sizeof(aa));
        aa.acc = W.acc_qkv;
        aa.acc_ld = L.nqkv;
        aa.bias = w->b_qkv;
        aa.theta = w->rope_theta;
        aa.q_out = T.q;
        aa.kc = s->k_cache;
        aa.vc = s->v_cache;
        aa.pos = s->pos;
        aa.max_ctx = s->max_ctx;
        aa.hq = (int)L.hq;
        aa.hkv = (int)L.hkv;
        aa.hd = (int)L.hd;
        aa.chunk = attn_chunk(s->max_ctx, B * (int)L.hkv);
        aa.n_chunks = (int)((s->max_ctx + aa.chunk - 1) / aa.chunk);
        aa.part = W.attn_part;
        aa.counters = W.attn_cnt;
        aa.out = W.h2;
        const size_t smem = attn_smem_bytes(L.G, (int)L.hd, aa.chunk);
        const dim3 grid(B * (int)L.hkv, aa.n_chunks);
        if (!on(2)) {
        } else if (L.hd == 128)
            LAROSA_TRY(cuda_check(launch(attention_kernel<4>, grid, dim3(kAttnThreads), smem, st, aa), "attention launch"));
        else
            LAROSA_TRY(cuda_check(launch(attention_kernel<2>, grid, dim3(kAttnThreads), smem, st, aa), "attention launch"));
        LAROSA_TRY(tap_copy(T.h2, W.h2, sizeof(float) * B * L.nq, st));
    }
    // ---- h2: attention output -> O -------------------------------------------------------------
    {
        ThreshArgs t;
        memset(&t, 0, sizeof(t));
        t.mode = THR_PLAIN;
        t.x = W.h2;
        t.ldx = L.nq;
        t.rms_eps = -1.0f;
        LAROSA_TRY(site(1, t, L.nq, plan->k_h2, W.h2, T.idx_h2, T.vals_h2, w->w_o, L.d, W.acc_o));
    }
    // ---- h3: r_mid = r + y_o (RMS scale) -> gate|up --------------------------------------------
    {
        ThreshArgs t;
        memset(&t, 0, sizeof(t));
        t.mode = THR_RESID_ACC;
        t.resid = s->resid;
        t.resid_ld = L.d;
        t.acc = W.acc_o;
        t.acc_ld = L.d;
        t.xout = W.rmid;
        t.rms_eps = w->rms_eps;
        LAROSA_TRY(site(2, t, L.d, plan->k_h3, W.rmid, T.idx_h3, T.vals_h3, w->w_gu, L.dgu, W.acc_gu));
        LAROSA_TRY(tap_copy(T.r_mid, W.rmid, sizeof(float) * B * L.d, st));
    }
    // ---- h4 = SiLU(g) * u -> down --------------------------------------------------------------
    {
        ThreshArgs t;
        memset(&t, 0, sizeof(t));
        t.mode = THR_SILU_GU;
        t.acc = W.acc_gu;
        t.acc_ld = L.dgu;
        t.xout = W.h4;
        t.rms_eps = -1.0f;
        LAROSA_TRY(site(3, t, L.inter, plan->k_h4, W.h4, T.idx_h4, T.vals_h4, w->w_down, L.d, W.acc_down));
        LAROSA_TRY(tap_copy(T.h4, W.h4, sizeof(float) * B * L.inter, st));
    }
    // ---- residual adapter r <- (r_mid + y_down) . A_l (dense GEMV), finalize ------------
    FinalizeArgs f = finalize_args_base();
    f.n = (int)L.d;
    f.batch = B;
    f.zero3 = W.acc_qkv;          // attention read it; zero it for the next step
    f.zero3_ld = L.nqkv;
    f.zero3_n = (int)L.nqkv;
    if (w->adapter) {
        if (on(9)) {
            const GemvPlan p = plan_gemv(L.d, L.d, bp);
            GemvArgs a = gemv_args_base();
            a.W = w->adapter;
            a.ld = L.d;
            a.d_out = (int)L.d;
            a.mode = GEMV_DENSE;
            a.x = W.rmid;
            a.ldx = L.d;
            a.d_in = (int)L.d;
            a.vacc = W.acc_down;
            a.vacc_ld = L.d;
            a.batch = B;
            a.acc = W.acc_adp;
            a.acc_ld = L.d;
            LAROSA_TRY(launch_gemv(a, p, bp, st));
        }
        f.acc1 = W.acc_adp;
        f.acc1_ld = L.d;
        f.out1 = s->resid;
        f.out1_ld = L.d;
        f.acc2 = W.acc_down;          // r_out = r_mid + y_down (tap), then zero
        f.acc2_ld = L.d;
        f.res2 = W.rmid;
        f.res2_ld = L.d;
        f.out2 = T.r_out;
        f.out2_ld = L.d;
        if (on(10)) LAROSA_TRY(launch_finalize(f, st));
    } else {
        f.acc1 = W.acc_down;
        f.acc1_ld = L.d;
        f.res1 = W.rmid;
        f.res1_ld = L.d;
        f.out1 = s->resid;
        f.out1_ld = L.d;
        if (on(10)) LAROSA_TRY(launch_finalize(f, st));
        LAROSA_TRY(tap_copy(T.r_out, s->resid, sizeof(float) * B * L.d, st));
    }
    return LAROSA_OK;
}
