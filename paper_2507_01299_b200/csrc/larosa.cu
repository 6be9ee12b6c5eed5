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
// Every workspace starts with a fixed header of self-resetting counters (zero on entry and
// on exit of every call).  All other regions come after it, so calls with different
// shapes can share one workspace without ever clobbering the counters' zero state.
constexpr size_t kCounterHeaderWords = 8192;   // GEMV tile tickets [0, 4096), attention [4096, 8192)
constexpr size_t kGemvCounterBase = 0;
constexpr size_t kAttnCounterBase = 4096;

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
    int tn, cs, rg, nwarps, stages, n_tiles;
    size_t smem;
};

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}

constexpr size_t kGemvSmemBudget = 200 * 1024;

// Tile width TN (multiple of 256) x cluster size CS so that n_tiles * CS CTAs fill the SMs
// once (one CTA per SM, ~200 KB ring); prefer the portable cluster size 8.
GemvPlan plan_gemv(int64_t d_out, int64_t nrows_max, int bp) {
    static const int force_cs = env_int("LAROSA_GEMV_CS", 0);     // tuning knobs (0 = auto)
    static const int force_tn = env_int("LAROSA_GEMV_TN", 0);
    static const int force_rg = env_int("LAROSA_GEMV_RG", 0);
    const int sms = sm_count();
    const int64_t max_cs_rows = std::max<int64_t>(1, nrows_max / 8);
    GemvPlan best = {256, 1, 1, 1, 2, (int)((d_out + 255) / 256), 0};
    int best_ctas = 0;
    const int max_warps = bp >= 8 ? 8 : kGemvMaxWarps;   // matches the kernel's launch bounds
    const int cs_order[5] = {8, 16, 4, 2, 1};
    for (int ci = 0; ci < 5; ++ci) {
        const int cs = cs_order[ci];
        if (force_cs && cs != force_cs) continue;
        if (cs > max_cs_rows && cs > 1) continue;
        for (int tn = 256; tn <= 4096; tn += 256) {
            if (force_tn && tn != force_tn) continue;
            const int slices = tn / 256;
            if (tn - 256 >= d_out) break;
            const int tiles = (int)((d_out + tn - 1) / tn);
            const int ctas = tiles * cs;
            if (ctas > sms) continue;
            if (slices > max_warps) break;
            int rg = std::max(1, std::min(8, 8 / slices));
            if (force_rg) rg = force_rg;
            rg = std::min(rg, max_warps / slices);
            if (rg < 1 || rg * slices > max_warps) continue;
            if (gemv_tail_bytes(rg, bp, tn) > kGemvSmemBudget) continue;
            if (ctas > best_ctas) {
                best_ctas = ctas;
                best.tn = tn;
                best.cs = cs;
                best.rg = rg;
                best.n_tiles = tiles;
            }
        }
    }
    best.nwarps = (best.tn / 256) * best.rg;
    int st = (int)((kGemvSmemBudget - 1024) / ((size_t)best.nwarps * kStageBytes));
    st = std::max(2, std::min(st, std::min(16, 128 / best.nwarps)));
    best.stages = st;
    best.smem = gemv_smem_bytes(best.nwarps, st, best.rg, bp, best.tn);
    return best;
}

template <int BP>
larosa_status launch_gemv_bp(GemvArgs a, const GemvPlan& p, cudaStream_t st) {
    auto kern = gemv_kernel<BP>;
    static bool attr_done = false;
    if (!attr_done) {
        LAROSA_TRY(cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024),
                              "cudaFuncSetAttribute(gemv smem)"));
        LAROSA_TRY(cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                              "cudaFuncSetAttribute(gemv cluster)"));
        attr_done = true;
    }
    a.tn = p.tn;
    a.rg = p.rg;
    a.stages = p.stages;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.cs, p.n_tiles);
    cfg.blockDim = dim3(p.nwarps * 32);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p.cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cuda_check(cudaLaunchKernelEx(&cfg, kern, a), "gemv launch");
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
    a.ep = EP_STORE;
    return a;
}

// ============================================================================== Top-K launch
larosa_status launch_topk(const TopkKernelArgs& a, int batch, cudaStream_t st) {
    const size_t smem = topk_smem_bytes(a.d);
    static bool attr_done = false;
    if (!attr_done) {
        LAROSA_TRY(cuda_check(allow_smem(topk_kernel, topk_smem_bytes(LAROSA_MAX_DIM)), "cudaFuncSetAttribute(topk)"));
        attr_done = true;
    }
    return cuda_check(launch(topk_kernel, dim3(batch), dim3(kTopkThreads), smem, st, a), "topk launch");
}

larosa_status launch_union(const uint32_t* mask, int nwords, int batch, int bp, const float* vals, int64_t k, int d,
                           int32_t* rows, float* V, int* nrows, cudaStream_t st) {
    const int grid = (nwords + 31) / 32;
    return cuda_check(launch(union_kernel, dim3(grid), dim3(kUnionThreads), 0, st, mask, nwords, batch, bp, vals, k, d,
                             rows, V, nrows),
                      "union launch");
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
static void carve_sparse_gemv(Carver& c, int32_t batch, int64_t d_in, int64_t k, uint32_t** mask, int32_t** rows,
                              float** V, int** nrows) {
    const int bp = pad_batch(batch);
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
    (void)d_out;
    carve_sparse_gemv(c, batch, d_in, k, nullptr, nullptr, nullptr, nullptr);
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
    if (!aligned16(W) || !aligned16(y) || (bias && !aligned16(bias)))
        return fail(LAROSA_EINVAL, "sparse_gemv: W, y, bias must be 16-byte aligned");
    if (d_in > INT32_MAX || d_out > INT32_MAX) return fail(LAROSA_EUNSUPPORTED, "sparse_gemv: dims too large");
    const size_t need = larosa_sparse_gemv_workspace_size(batch, d_in, k, d_out);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "sparse_gemv: workspace %zu < %zu", ws_bytes, need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);

    Carver c(ws);
    uint32_t* mask = nullptr;
    int32_t* rows = nullptr;
    float* V = nullptr;
    int* nrows = nullptr;
    carve_sparse_gemv(c, batch, d_in, k, &mask, &rows, &V, &nrows);
    const int bp = pad_batch(batch);
    const int64_t nrows_max = batch == 1 ? k : std::min<int64_t>(d_in, (int64_t)batch * k);
    GemvPlan p = plan_gemv(d_out, nrows_max, bp);

    GemvArgs a = gemv_args_base();
    a.W = W;
    a.ld = ld;
    a.d_out = (int)d_out;
    a.batch = batch;
    a.bias = bias;
    a.out = y;
    a.out_ld = d_out;
    a.ep = EP_STORE;
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
    return launch_gemv(a, p, bp, st);
}

extern "C" larosa_status larosa_gemv_plan_info(int64_t d_out, int64_t nrows_max, int32_t batch, int32_t* info) {
    if (!info || d_out <= 0 || nrows_max < 0 || batch < 1 || batch > LAROSA_MAX_BATCH)
        return fail(LAROSA_EINVAL, "gemv_plan_info: bad arguments");
    const int bp = pad_batch(batch);
    const GemvPlan p = plan_gemv(d_out, nrows_max, bp);
    info[0] = p.tn;
    info[1] = p.cs;
    info[2] = p.rg;
    info[3] = p.nwarps;
    info[4] = p.stages;
    info[5] = p.n_tiles;
    info[6] = (int32_t)p.smem;
    info[7] = 0;
    int dev = -1;
    if (cudaGetDevice(&dev) == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(p.cs, p.n_tiles);
        cfg.blockDim = dim3(p.nwarps * 32);
        cfg.dynamicSmemBytes = p.smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = p.cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        cudaError_t e;
        switch (bp) {
            case 1: e = cudaOccupancyMaxActiveClusters(&n, gemv_kernel<1>, &cfg); break;
            case 2: e = cudaOccupancyMaxActiveClusters(&n, gemv_kernel<2>, &cfg); break;
            case 4: e = cudaOccupancyMaxActiveClusters(&n, gemv_kernel<4>, &cfg); break;
            case 8: e = cudaOccupancyMaxActiveClusters(&n, gemv_kernel<8>, &cfg); break;
            default: e = cudaOccupancyMaxActiveClusters(&n, gemv_kernel<16>, &cfg); break;
        }
        if (e == cudaSuccess) info[7] = n;
        cudaGetLastError();
    }
    return LAROSA_OK;
}

// ============================================================================== rotate + Top-K
static void carve_rotate_topk(Carver& c, int32_t batch, int64_t d, float** xr) {
    float* x = c.take<float>((size_t)batch * d);
    if (xr) *xr = x;
}

extern "C" size_t larosa_rotate_topk_workspace_size(int32_t batch, int64_t d) {
    if (batch < 1 || d <= 0) return 0;
    Carver c(nullptr);
    carve_rotate_topk(c, batch, d, nullptr);
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
    if (R && (!aligned16(R) || !aligned16(x))) return fail(LAROSA_EINVAL, "rotate_topk: R, x must be 16-byte aligned");
    if (R && xr_out == x) return fail(LAROSA_EINVAL, "rotate_topk: xr_out aliases x with R != NULL");
    const size_t need = larosa_rotate_topk_workspace_size(batch, d);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "rotate_topk: workspace %zu < %zu", ws_bytes, need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Carver c(ws);
    float* xr_ws;
    carve_rotate_topk(c, batch, d, &xr_ws);

    const float* src = x;
    if (R) {
        // dense rotation GEMV x . R (all d rows, token-major values)
        float* xr = (xr_out && aligned16(xr_out)) ? xr_out : xr_ws;
        const int bp = pad_batch(batch);
        GemvPlan p = plan_gemv(d, d, bp);
        GemvArgs a = gemv_args_base();
        a.W = R;
        a.ld = d;
        a.d_out = (int)d;
        a.rows = nullptr;
        a.vals = x;
        a.vs_r = 1;
        a.vs_b = d;
        a.nrows = (int)d;
        a.batch = batch;
        a.out = xr;
        a.out_ld = d;
        a.ep = EP_STORE;
        LAROSA_TRY(launch_gemv(a, p, bp, st));
        src = xr;
    }
    TopkKernelArgs t;
    t.x = src;
    t.ldx = d;
    t.d = (int)d;
    t.k = (int)k;
    t.rms_eps = rms_eps;
    t.xr_out = (xr_out && src != xr_out) ? xr_out : nullptr;
    t.idx = idx;
    t.vals = vals;
    t.mask = mask;
    t.scale = nullptr;
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
struct LayerWs {
    int32_t* idx[4];
    float* vals[4];
    uint32_t* mask[4];
    float* q;
    float* h2;
    float* rmid;
    float* h4;
    float* rout;
    int32_t* urows;
    float* uV;
    int* unrows;
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
    const int bp = pad_batch(batch);
    const int64_t din[4] = {L.d, L.nq, L.d, L.inter};
    LayerWs tmp;
    LayerWs* o = ws ? ws : &tmp;
    for (int s = 0; s < 4; ++s) {
        o->idx[s] = c.take<int32_t>((size_t)batch * din[s]);
        o->vals[s] = c.take<float>((size_t)batch * din[s]);
        o->mask[s] = c.take<uint32_t>((size_t)batch * ((din[s] + 31) / 32));
    }
    o->q = c.take<float>((size_t)batch * L.nq);
    o->h2 = c.take<float>((size_t)batch * L.nq);
    o->rmid = c.take<float>((size_t)batch * L.d);
    o->h4 = c.take<float>((size_t)batch * L.inter);
    o->rout = c.take<float>((size_t)batch * L.d);
    const int64_t dmax = std::max(std::max(L.d, L.nq), L.inter);
    o->urows = c.take<int32_t>((size_t)dmax);
    o->uV = c.take<float>((size_t)dmax * bp + 16);
    o->unrows = c.take<int>(4);
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
    if (w->n_q_heads / w->n_kv_heads > 8) return fail(LAROSA_EUNSUPPORTED, "sparse_layer: GQA group > 8");
    if (w->head_dim != 64 && w->head_dim != 128) return fail(LAROSA_EUNSUPPORTED, "sparse_layer: head_dim must be 64 or 128");
    if (w->d % 8 || w->inter % LAROSA_GU_BLOCK) return fail(LAROSA_EUNSUPPORTED, "sparse_layer: d %% 8 or inter %% 64");
    if (w->d > LAROSA_MAX_DIM || w->inter > LAROSA_MAX_DIM || w->n_q_heads * w->head_dim > LAROSA_MAX_DIM)
        return fail(LAROSA_EUNSUPPORTED, "sparse_layer: dimension > %d", LAROSA_MAX_DIM);
    if (s->max_ctx <= 0) return fail(LAROSA_EINVAL, "sparse_layer: max_ctx must be > 0");
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

// Top-K of one site (+ union for batch > 1), then the GEMV over its kept rows.
struct SiteGemv {
    const float* x;        // [batch][din]
    int64_t din;
    int64_t k;
    float rms_eps;         // < 0: no RMS scale
    int site;
};
}  // namespace

extern "C" size_t larosa_layer_workspace_size(const larosa_layer_weights* w, int32_t batch, int64_t max_ctx) {
    if (!w || batch < 1 || max_ctx <= 0) return 0;
    Carver c(nullptr);
    carve_layer(c, layer_dims(w), batch, max_ctx, nullptr);
    return c.size();
}

extern "C" larosa_status larosa_sparse_layer(const larosa_layer_weights* w, const larosa_layer_plan* plan,
                                             const larosa_layer_state* s, const larosa_layer_taps* taps, void* ws,
                                             size_t ws_bytes, larosa_stream_t stream) {
    LAROSA_TRY(validate_layer(w, plan, s));
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

    // Top-K at a site; fills the GEMV row source (idx list, or union for batch > 1)
    auto site = [&](const SiteGemv& sg, GemvArgs& a) -> larosa_status {
        TopkKernelArgs t;
        t.x = sg.x;
        t.ldx = sg.din;
        t.d = (int)sg.din;
        t.k = (int)sg.k;
        t.rms_eps = sg.rms_eps;
        t.xr_out = nullptr;
        t.idx = W.idx[sg.site];
        t.vals = W.vals[sg.site];
        t.mask = B > 1 ? W.mask[sg.site] : nullptr;
        t.scale = nullptr;
        LAROSA_TRY(launch_topk(t, B, st));
        if (B == 1) {
            a.rows = W.idx[sg.site];
            a.vals = W.vals[sg.site];
            a.vs_r = 1;
            a.vs_b = sg.k;
            a.nrows = (int)sg.k;
            a.nrows_dev = nullptr;
        } else {
            const int nw = (int)((sg.din + 31) / 32);
            LAROSA_TRY(launch_union(W.mask[sg.site], nw, B, bp, W.vals[sg.site], sg.k, (int)sg.din, W.urows, W.uV,
                                    W.unrows, st));
            a.rows = W.urows;
            a.vals = W.uV;
            a.vs_r = bp;
            a.vs_b = 1;
            a.nrows = 0;
            a.nrows_dev = W.unrows;
        }
        a.batch = B;
        return LAROSA_OK;
    };
    auto nrows_max = [&](int64_t din, int64_t k) { return B == 1 ? k : std::min<int64_t>(din, (int64_t)B * k); };

    // ---- h1: Top-K of r (RMS scale), QKV GEMV + bias + RoPE + KV append --------------------
    {
        GemvArgs a = gemv_args_base();
        LAROSA_TRY(site({s->resid, L.d, plan->k_h1, w->rms_eps, 0}, a));
        GemvPlan p = plan_gemv(L.nqkv, nrows_max(L.d, plan->k_h1), bp);
        a.W = w->w_qkv;
        a.ld = L.nqkv;
        a.d_out = (int)L.nqkv;
        a.ep = EP_QKV_ROPE;
        a.bias = w->b_qkv;
        a.out = W.q;
        a.out_ld = L.nq;
        a.hq = (int)L.hq;
        a.hkv = (int)L.hkv;
        a.hd = (int)L.hd;
        a.theta = w->rope_theta;
        a.pos = s->pos;
        a.kc = s->k_cache;
        a.vc = s->v_cache;
        a.max_ctx = s->max_ctx;
        LAROSA_TRY(launch_gemv(a, p, bp, st));
        LAROSA_TRY(tap_copy(T.idx_h1, W.idx[0], sizeof(int32_t) * B * plan->k_h1, st));
        LAROSA_TRY(tap_copy(T.vals_h1, W.vals[0], sizeof(float) * B * plan->k_h1, st));
        LAROSA_TRY(tap_copy(T.q, W.q, sizeof(float) * B * L.nq, st));
    }
    // ---- attention ---------------------------------------------------------------------------
    {
        AttnArgs aa;
        aa.q = W.q;
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
        LAROSA_TRY(cuda_check(launch(attention_kernel, dim3(B * (int)L.hkv, aa.n_chunks), dim3(kAttnThreads), smem, st, aa),
                              "attention launch"));
        LAROSA_TRY(tap_copy(T.h2, W.h2, sizeof(float) * B * L.nq, st));
    }
    // ---- h2: Top-K of the attention output, O GEMV, r_mid = r + y ----------------------------
    {
        GemvArgs a = gemv_args_base();
        LAROSA_TRY(site({W.h2, L.nq, plan->k_h2, -1.0f, 1}, a));
        GemvPlan p = plan_gemv(L.d, nrows_max(L.nq, plan->k_h2), bp);
        a.W = w->w_o;
        a.ld = L.d;
        a.d_out = (int)L.d;
        a.ep = EP_RESID;
        a.resid = s->resid;
        a.resid_ld = L.d;
        a.out = W.rmid;
        a.out_ld = L.d;
        LAROSA_TRY(launch_gemv(a, p, bp, st));
        LAROSA_TRY(tap_copy(T.idx_h2, W.idx[1], sizeof(int32_t) * B * plan->k_h2, st));
        LAROSA_TRY(tap_copy(T.vals_h2, W.vals[1], sizeof(float) * B * plan->k_h2, st));
        LAROSA_TRY(tap_copy(T.r_mid, W.rmid, sizeof(float) * B * L.d, st));
    }
    // ---- h3: Top-K of r_mid (RMS scale), gate|up GEMV, h4 = SiLU(g) * u ----------------------
    {
        GemvArgs a = gemv_args_base();
        LAROSA_TRY(site({W.rmid, L.d, plan->k_h3, w->rms_eps, 2}, a));
        GemvPlan p = plan_gemv(L.dgu, nrows_max(L.d, plan->k_h3), bp);
        a.W = w->w_gu;
        a.ld = L.dgu;
        a.d_out = (int)L.dgu;
        a.ep = EP_SILU_GU;
        a.out = W.h4;
        a.out_ld = L.inter;
        LAROSA_TRY(launch_gemv(a, p, bp, st));
        LAROSA_TRY(tap_copy(T.idx_h3, W.idx[2], sizeof(int32_t) * B * plan->k_h3, st));
        LAROSA_TRY(tap_copy(T.vals_h3, W.vals[2], sizeof(float) * B * plan->k_h3, st));
        LAROSA_TRY(tap_copy(T.h4, W.h4, sizeof(float) * B * L.inter, st));
    }
    // ---- h4: Top-K of h4, down GEMV, r_out = r_mid + y ---------------------------------------
    float* r_out = w->adapter ? W.rout : s->resid;
    {
        GemvArgs a = gemv_args_base();
        LAROSA_TRY(site({W.h4, L.inter, plan->k_h4, -1.0f, 3}, a));
        GemvPlan p = plan_gemv(L.d, nrows_max(L.inter, plan->k_h4), bp);
        a.W = w->w_down;
        a.ld = L.d;
        a.d_out = (int)L.d;
        a.ep = EP_RESID;
        a.resid = W.rmid;
        a.resid_ld = L.d;
        a.out = r_out;
        a.out_ld = L.d;
        LAROSA_TRY(launch_gemv(a, p, bp, st));
        LAROSA_TRY(tap_copy(T.idx_h4, W.idx[3], sizeof(int32_t) * B * plan->k_h4, st));
        LAROSA_TRY(tap_copy(T.vals_h4, W.vals[3], sizeof(float) * B * plan->k_h4, st));
        LAROSA_TRY(tap_copy(T.r_out, r_out, sizeof(float) * B * L.d, st));
    }
    // ---- residual adapter r <- r_out . A_l (dense GEMV) -------------------------------
    if (w->adapter) {
        GemvPlan p = plan_gemv(L.d, L.d, bp);
        GemvArgs a = gemv_args_base();
        a.W = w->adapter;
        a.ld = L.d;
        a.d_out = (int)L.d;
        a.rows = nullptr;
        a.vals = W.rout;
        a.vs_r = 1;
        a.vs_b = L.d;
        a.nrows = (int)L.d;
        a.batch = B;
        a.ep = EP_STORE;
        a.out = s->resid;
        a.out_ld = L.d;
        LAROSA_TRY(launch_gemv(a, p, bp, st));
    }
    return LAROSA_OK;
}
