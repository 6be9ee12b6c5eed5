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
#include "gemv_tc.cuh"
#include "calib.cuh"
#include "gemv_w4.cuh"
#include "prefill_tc.cuh"
#include "gemv_img.cuh"

#include <map>
#include <mutex>
#include <set>
#include <tuple>

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

// Function attributes are per device context: track the value of each (kernel, device, attribute)
// under a lock (calls are re-entrant and a process may drive several GPUs) and call the driver only
// when it changes; the dynamic shared memory limit only ever grows (a launch needing less than the
// current limit is valid, and lowering it would break a later larger launch).
cudaError_t set_func_attr_once(const void* kern, cudaFuncAttribute attr, int value) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, int>, int> cur;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const auto key = std::make_tuple(kern, dev, (int)attr);
    std::lock_guard<std::mutex> lk(mu);
    const auto it = cur.find(key);
    if (it != cur.end()) {
        if (it->second == value) return cudaSuccess;
        if (attr == cudaFuncAttributeMaxDynamicSharedMemorySize && it->second > value) return cudaSuccess;
    }
    e = cudaFuncSetAttribute(kern, attr, value);
    if (e == cudaSuccess) cur[key] = value;
    return e;
}

// Opt a kernel in to > 48 KB dynamic shared memory (once per kernel and device).
template <typename K>
cudaError_t allow_smem(K kern, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    return set_func_attr_once(reinterpret_cast<const void*>(kern), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)bytes);
}

// ============================================================================== workspace
// Every workspace starts with a fixed header of self-resetting counters, followed by the
// call's fixed-point GEMV accumulators; both are zero at rest (kernels restore the zeros),
// so the caller zero-fills a workspace once.  A workspace must be reused only for calls of
// the same kind and shapes (other layouts would place live data where accumulators were).
constexpr size_t kCounterHeaderWords = 8192;   // attention tickets
constexpr size_t kAttnCounterBase = 0;        // [0, 4096): attention group tickets
constexpr size_t kGemvTicketBase = 4096;      // + 256 j: slice tickets of the j-th epilogue GEMV
constexpr size_t kPrepBarrier = 6000;         // 2 words: grid barrier of select_prep_kernel
constexpr size_t kErrWord = kCounterHeaderWords - 1;   // error bits (kErrKeepAll, kErrFixOverflow)

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

int n_slices_of(int64_t n) { return (int)((n + kSliceCols - 1) / kSliceCols); }
int pad_batch(int b) { return b <= 1 ? 1 : b <= 2 ? 2 : b <= 4 ? 4 : b <= 8 ? 8 : 16; }

// ============================================================================== GEMV plan
struct GemvPlan {
    int n_slices, n_splits, list_cap;
    size_t smem;
    int n_splits2 = 0;   // SELECT companion CTAs per slice (dense rows of W2)
};

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}

int gemv_list_max(int bp) { return bp <= 2 ? 2048 : 1024; }

// Opt-in (LAROSA_GEMV_CLUSTER=1): batch-1 SELECT GEMVs reduce split-K through a thread-block
// cluster of the slice's CTAs (<= 16, non-portable above 8) instead of global fixed-point reds
// and a slice ticket.  Measured on the LLaMA2-7B block: 88.7 us vs 83.2 us with the reds (the
// cluster's CTAs are co-scheduled in one GPC and the tail waits on the slowest of them).
constexpr int kMaxGemvCluster = 16;
bool gemv_cluster_enabled() {
    static const int v = env_int("LAROSA_GEMV_CLUSTER", 0);
    return v != 0;
}

// 256-column slices x row splits, as many 256-thread CTAs per SM as fit (at most 2), one
// wave.  rows_src: candidate rows (list length for LIST, k for SELECT, input length for
// THRESH / DENSE).  LIST/THRESH/DENSE lists are bounded by gemv_list_max.
GemvPlan plan_gemv(int64_t d_out, int64_t rows_src, int bp, int mode = GEMV_LIST, int64_t d_in = 0) {
    static const int per_sm_env = env_int("LAROSA_GEMV_CTAS_PER_SM", 0);   // tuning knob (0 = auto)
    GemvPlan p;
    p.n_slices = (int)((d_out + kSliceCols - 1) / kSliceCols);
    int per_sm = per_sm_env > 0 ? per_sm_env : (bp <= 4 ? 2 : 1);
    const int by_rows = (int)std::max<int64_t>(1, rows_src / 16);
    int by_cap = 1;
    const int64_t nwords = (d_in + 31) / 32;
    if (mode != GEMV_SELECT) {
        const int lmax = gemv_list_max(bp);
        by_cap = (int)std::max<int64_t>(1, (rows_src + lmax - 1) / lmax);
    } else {
        by_cap = (int)std::max<int64_t>(1, (nwords + kSelMaxWords - 1) / kSelMaxWords);   // words per CTA
    }
    for (int it = 0; it < 2; ++it) {
        static const int sel_wave_pct = env_int("LAROSA_SEL_WAVE_PCT", 100);   // SELECT: waves of CTAs (tuning)
        const int target = mode == GEMV_SELECT ? sm_count() * per_sm * sel_wave_pct / 100 : sm_count() * per_sm;
        int by_target = std::max(1, target / p.n_slices);   // one wave: slices x splits <= target
        // SELECT: cap the splits at the cluster size when that keeps >= 85% of the wave's slots
        if (mode == GEMV_SELECT && gemv_cluster_enabled() && by_target > kMaxGemvCluster &&
            p.n_slices * kMaxGemvCluster * 100 >= target * 85)
            by_target = kMaxGemvCluster;
        p.n_splits = std::max(by_cap, std::min(by_target, by_rows));
        if (mode == GEMV_DENSE && p.n_slices >= target) {
            // more slices than slots (the LM head): choose the splits that fill the last wave best
            double best = 0.0;
            for (int sp = std::max(1, by_cap); sp <= 8 && rows_src / sp >= 256; ++sp) {
                const double ctas = (double)p.n_slices * sp, waves = std::ceil(ctas / target);
                const double eff = ctas / (waves * target);
                if (eff > best + 0.02) {
                    best = eff;
                    p.n_splits = sp;
                }
            }
        }
        p.list_cap = mode == GEMV_SELECT ? (int)(32 * ((nwords + p.n_splits - 1) / p.n_splits))   // interleaved words
                                         : (int)std::max<int64_t>(32, (rows_src + p.n_splits - 1) / p.n_splits + 1);
        p.smem = gemv_smem_bytes(bp, p.list_cap, mode, (int)d_in);
        // B200: 228 KB of shared memory per SM, 1 KB reserved per CTA
        const int fit = (int)(233472 / (p.smem + 1024));
        if (fit >= per_sm || per_sm == 1) break;
        per_sm = std::max(1, fit);
    }
    return p;
}

// SELECT site (k kept rows of d_in) plus d2 dense companion rows into the same d_out columns:
// one wave of 2 CTAs per SM split between the two row sources in proportion to their bytes
// (LAROSA_COMP_PCT overrides the companion share, in percent of the splits).
GemvPlan plan_gemv_comp(int64_t d_out, int64_t k, int64_t d_in, int64_t d2) {
    static const int pct_env = env_int("LAROSA_COMP_PCT", 0);
    GemvPlan p = plan_gemv(d_out, k, 1, GEMV_SELECT, d_in);
    // ~1.3 waves of 2 CTAs per SM, one third companions (measured on the LLaMA2-7B block: the
    // companions finish early and free their slots; more, shorter SELECT CTAs shorten the tail)
    static const int wave_pct = env_int("LAROSA_COMP_WAVE_PCT", 130);
    int total = std::max(2, (sm_count() * 2 * wave_pct / 100 + p.n_slices - 1) / p.n_slices);
    if (gemv_cluster_enabled() && total > kMaxGemvCluster && p.n_slices * kMaxGemvCluster * 100 >= sm_count() * 2 * 85)
        total = kMaxGemvCluster;
    const int64_t nwords = (d_in + 31) / 32;
    const int min_sel = (int)std::max<int64_t>(1, (nwords + kSelMaxWords - 1) / kSelMaxWords);
    int n2 = pct_env > 0 ? (total * pct_env + 50) / 100 : (total + 1) / 3;
    n2 = std::max(1, std::min(n2, total - min_sel));
    p.n_splits = std::max(min_sel, total - n2);
    p.list_cap = (int)(32 * ((nwords + p.n_splits - 1) / p.n_splits));
    n2 = std::max<int>(n2, (int)((d2 + p.list_cap - 1) / p.list_cap));
    static const int sel_env = env_int("LAROSA_COMP_SEL", 0), n2_env = env_int("LAROSA_COMP_N", 0);   // tuning
    if (sel_env > 0) {
        p.n_splits = std::max(min_sel, sel_env);
        p.list_cap = (int)(32 * ((nwords + p.n_splits - 1) / p.n_splits));
    }
    if (n2_env > 0) n2 = std::max<int>(n2_env, (int)((d2 + p.list_cap - 1) / p.list_cap));
    p.n_splits2 = n2;
    p.smem = gemv_smem_bytes(1, p.list_cap, GEMV_SELECT, (int)d_in);
    return p;
}

template <int BP, int MODE>
larosa_status launch_gemv_bm(const GemvArgs& a, const GemvPlan& p, cudaStream_t st) {
    auto kern = gemv_kernel<BP, MODE>;
    LAROSA_TRY(cuda_check(allow_smem(kern, 227 * 1024), "cudaFuncSetAttribute(gemv)"));
    if (p.smem > 227 * 1024) return fail(LAROSA_EUNSUPPORTED, "gemv: shared memory plan %zu B too large", p.smem);
    GemvArgs aa = a;
    static const int late = env_int("LAROSA_PDL_LATE", 0);    // tuning
    aa.late_trigger = late;
    static const int comp_late = env_int("LAROSA_COMP_LATE", 0);   // tuning
    aa.comp_late = comp_late;
    aa.n_splits = p.n_splits;
    aa.n_splits2 = p.n_splits2;
    aa.list_cap = p.list_cap;
    if (p.n_splits2 > 0 && (MODE != GEMV_SELECT || !a.W2 || !a.x2 || a.d2 <= 0 ||
                            (a.d2 + p.n_splits2 - 1) / p.n_splits2 > p.list_cap))
        return fail(LAROSA_EUNSUPPORTED, "gemv: bad companion plan");
    const int ny = p.n_splits + p.n_splits2;
    aa.cluster = 0;
    if (MODE == GEMV_SELECT && BP == 1 && gemv_cluster_enabled() && ny >= 2 && ny <= kMaxGemvCluster &&
        a.batch == 1) {
        LAROSA_TRY(cuda_check(set_func_attr_once(reinterpret_cast<const void*>(kern),
                                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                              "cudaFuncSetAttribute(non-portable cluster)"));
        aa.cluster = ny;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(p.n_slices, ny);
        cfg.blockDim = dim3(kGemvThreads);
        cfg.dynamicSmemBytes = p.smem;
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1;
        at[0].val.clusterDim.y = ny;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl_enabled() ? 2 : 1;
        return cuda_check(cudaLaunchKernelEx(&cfg, kern, aa), "gemv cluster launch");
    }
    return cuda_check(launch(kern, dim3(p.n_slices, ny), dim3(kGemvThreads), p.smem, st, aa), "gemv launch");
}

template <int BP>
larosa_status launch_gemv_bp(const GemvArgs& a, const GemvPlan& p, cudaStream_t st) {
    switch (a.mode) {
        case GEMV_LIST: return launch_gemv_bm<BP, GEMV_LIST>(a, p, st);
        case GEMV_DENSE: return launch_gemv_bm<BP, GEMV_DENSE>(a, p, st);
        case GEMV_THRESH:
            if constexpr (BP > 1) return launch_gemv_bm<BP, GEMV_THRESH>(a, p, st);
            return fail(LAROSA_EUNSUPPORTED, "gemv: THRESH needs batch > 1");
        case GEMV_SELECT:
            if constexpr (BP == 1) return launch_gemv_bm<1, GEMV_SELECT>(a, p, st);
            return fail(LAROSA_EUNSUPPORTED, "gemv: SELECT is batch 1 only");
        default: return fail(LAROSA_EINVAL, "gemv: bad mode");
    }
}

// ---- batch >= 8: the tcgen05 GEMV (gemv_tc.cuh), 128-column slices -------------------------
bool use_tc_gemv(int bp) {
    static const int v = env_int("LAROSA_GEMV_TC", 1);
    return v != 0 && bp >= 8;
}
GemvPlan plan_gemv_tc(int64_t d_out, int64_t rows_src) {
    GemvPlan p;
    p.n_slices = (int)((d_out + kTcCols - 1) / kTcCols);
    static const int tc_target_pct = env_int("LAROSA_TC_TARGET_PCT", 400);   // CTAs per SM x 100
    const int target = sm_count() * tc_target_pct / 100;
    const int by_target = std::max(1, target / p.n_slices);
    const int by_rows = (int)std::max<int64_t>(1, rows_src / 64);
    const int by_cap = (int)std::max<int64_t>(1, (rows_src + 8191) / 8192);   // <= 8192 rows per CTA
    p.n_splits = std::max(by_cap, std::min(by_target, by_rows));
    p.list_cap = (int)std::max<int64_t>(64, (rows_src + p.n_splits - 1) / p.n_splits + 1);
    p.smem = gemv_tc_smem_bytes(p.list_cap);
    return p;
}
bool make_w_mn_map(CUtensorMap* m, const void* W, int64_t d_in, int64_t d_out, int64_t ld);   // (fold section)
template <int BP, int MODE>
larosa_status launch_gemv_tc_bm(const GemvArgs& a, cudaStream_t st) {
    const int64_t rows_src = MODE == GEMV_LIST ? (a.nrows_dev ? a.d_in : a.nrows) : a.d_in;
    GemvPlan p = plan_gemv_tc(a.d_out, rows_src);
    if (MODE != GEMV_LIST) {   // contiguous rows: no row list in shared memory
        p.list_cap = 0;
        p.smem = gemv_tc_smem_bytes(p.list_cap);
    }
    auto kern = gemv_tc_kernel<BP, MODE>;
    LAROSA_TRY(cuda_check(allow_smem(kern, 227 * 1024), "cudaFuncSetAttribute(gemv_tc)"));
    if (p.smem > 227 * 1024) return fail(LAROSA_EUNSUPPORTED, "gemv_tc: shared memory plan %zu B too large", p.smem);
    GemvArgs aa = a;
    aa.n_splits = p.n_splits;
    aa.list_cap = p.list_cap;
#ifdef LAROSA_TC_DEBUG
    static const int tc_dbg = env_int("LAROSA_TC_DBG", 0);   // profiling builds only
    aa.tc_dbg = tc_dbg;
#endif
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    if (MODE != GEMV_LIST && !make_w_mn_map(&tm, a.W, a.d_in, a.d_out, a.ld))
        return fail(LAROSA_ECUDA, "gemv_tc: cuTensorMapEncodeTiled failed for the weight matrix");
    return cuda_check(launch(kern, dim3(p.n_slices, p.n_splits), dim3(kTcThreads), p.smem, st, aa, tm), "gemv_tc launch");
}
// batch >= 8 with a pre-built token image (gemv_img.cuh): weight tiles by TMA, the image by bulk copy
GemvPlan plan_gemv_img(int64_t d_out, int64_t d_in) {
    GemvPlan p;
    p.n_slices = (int)((d_out + kTcCols - 1) / kTcCols);
    static const int target_pct = env_int("LAROSA_IMG_TARGET_PCT", 200);   // CTAs per SM x 100
    const int target = sm_count() * target_pct / 100;
    const int by_rows = (int)std::max<int64_t>(1, d_in / 64);
    p.n_splits = std::max(1, std::min(target / p.n_slices, by_rows));
    p.list_cap = 0;
    p.smem = gemv_img_smem_bytes();
    return p;
}
template <int BP>
larosa_status launch_gemv_img(const GemvArgs& a, cudaStream_t st) {
    const GemvPlan p = plan_gemv_img(a.d_out, a.d_in);
    auto kern = gemv_img_kernel<BP>;
    LAROSA_TRY(cuda_check(allow_smem(kern, p.smem), "cudaFuncSetAttribute(gemv_img)"));
    GemvArgs aa = a;
    aa.n_splits = p.n_splits;
    CUtensorMap tm;
    if (!make_w_mn_map(&tm, a.W, a.d_in, a.d_out, a.ld))
        return fail(LAROSA_ECUDA, "gemv_img: cuTensorMapEncodeTiled failed for the weight matrix");
    return cuda_check(launch(kern, dim3(p.n_slices, p.n_splits), dim3(kImgThreads), p.smem, st, aa, tm), "gemv_img launch");
}
size_t img_bytes(int64_t d) { return (size_t)((d + kTcChunk - 1) / kTcChunk) * kImgChunkBytes; }
larosa_status launch_rule_image(const float* x, int64_t ldx, int64_t d, int64_t k, float eps, int batch, ThreshOut* rule,
                                void* img, void* img_raw, cudaStream_t st) {
    const size_t smem = rule_image_smem_bytes((int)d);
    LAROSA_TRY(cuda_check(allow_smem(rule_image_kernel, smem), "cudaFuncSetAttribute(rule_image)"));
    return cuda_check(launch(rule_image_kernel, dim3(batch), dim3(kRiThreads), smem, st, x, ldx, (int)d, (int)k, eps, rule,
                             static_cast<unsigned char*>(img), static_cast<unsigned char*>(img_raw)),
                      "rule_image launch");
}
larosa_status launch_rule_image_reg(const float* x, int64_t ldx, int64_t d, int64_t k, float eps, int batch,
                                    ThreshOut* rule, void* img, void* img_raw, cudaStream_t st) {
    unsigned char* im = static_cast<unsigned char*>(img);
    unsigned char* ir = static_cast<unsigned char*>(img_raw);
    const dim3 g(batch), blk(kRiThreads);
    if (d <= 8 * kRiThreads)
        return cuda_check(launch(rule_image_reg_kernel<8>, g, blk, 0, st, x, ldx, (int)d, (int)k, eps, rule, im, ir), "rule_image_reg");
    if (d <= 16 * kRiThreads)
        return cuda_check(launch(rule_image_reg_kernel<16>, g, blk, 0, st, x, ldx, (int)d, (int)k, eps, rule, im, ir), "rule_image_reg");
    if (d <= 32 * kRiThreads)
        return cuda_check(launch(rule_image_reg_kernel<32>, g, blk, 0, st, x, ldx, (int)d, (int)k, eps, rule, im, ir), "rule_image_reg");
    return cuda_check(launch(rule_image_reg_kernel<64>, g, blk, 0, st, x, ldx, (int)d, (int)k, eps, rule, im, ir), "rule_image_reg");
}
larosa_status launch_dense_image(const float* x, int64_t ldx, int64_t d, int batch, void* img, cudaStream_t st) {
    const int groups = (int)((d + 7) / 8);
    return cuda_check(launch(dense_image_kernel, dim3((unsigned)((groups + 255) / 256), batch), dim3(256), 0, st, x, ldx,
                             (int)d, static_cast<unsigned char*>(img)),
                      "dense_image launch");
}

template <int BP>
larosa_status launch_gemv_tc(const GemvArgs& a, cudaStream_t st) {
    switch (a.mode) {
        case GEMV_LIST: return launch_gemv_tc_bm<BP, GEMV_LIST>(a, st);
        case GEMV_DENSE: return launch_gemv_tc_bm<BP, GEMV_DENSE>(a, st);
        case GEMV_THRESH: return launch_gemv_tc_bm<BP, GEMV_THRESH>(a, st);
        default: return fail(LAROSA_EUNSUPPORTED, "gemv_tc: bad mode");
    }
}

larosa_status launch_gemv(const GemvArgs& a, const GemvPlan& p, int bp, cudaStream_t st) {
    if (use_tc_gemv(bp) && a.img && (a.mode == GEMV_THRESH || a.mode == GEMV_DENSE)) {
        if (bp == 8) return launch_gemv_img<8>(a, st);
        return launch_gemv_img<16>(a, st);
    }
    if (use_tc_gemv(bp) && a.mode != GEMV_SELECT) {
        if (bp == 8) return launch_gemv_tc<8>(a, st);
        return launch_gemv_tc<16>(a, st);
    }
    switch (bp) {
        case 1: return launch_gemv_bp<1>(a, p, st);
        case 2: return launch_gemv_bp<2>(a, p, st);
        case 4: return launch_gemv_bp<4>(a, p, st);
        case 8: return launch_gemv_bp<8>(a, p, st);
        default: return launch_gemv_bp<16>(a, p, st);
    }
}

// the error word of the workspace the current API call carved (one call at a time per host thread)
thread_local uint32_t* t_err_word = nullptr;
struct ErrScope {
    uint32_t* prev;
    explicit ErrScope(const Carver& c) : prev(t_err_word) { t_err_word = c.counters(kErrWord); }
    ~ErrScope() { t_err_word = prev; }
};
GemvArgs gemv_args_base() {
    GemvArgs a;
    memset(&a, 0, sizeof(a));
    a.err = t_err_word;
    return a;
}

// W4A16 SELECT GEMV (gemv_w4.cuh) with the layer's epilogue: SC-column slices, one wave of 2 CTAs
// per SM
template <int SC>
larosa_status launch_gemv_w4_t(GemvArgs a, const uint8_t* Wq, const uint16_t* S, cudaStream_t st) {
    using C = W4Cfg<SC>;
    const int64_t d_in = a.d_in, d_out = a.d_out, k = a.sel_k;
    const int n_sl = (int)((d_out + SC - 1) / SC);
    const int64_t nwords = (d_in + 31) / 32;
    const int by_cap = (int)std::max<int64_t>(1, (nwords + kSelMaxWords - 1) / kSelMaxWords);
    a.n_splits = std::max(by_cap, std::min(std::max(1, sm_count() * 2 / n_sl), (int)std::max<int64_t>(1, k / 16)));
    a.n_splits2 = 0;
    if (a.W2) {   // companions (dense bf16 rows of W2): one wave split between the two row sets by bytes,
                  // an int4 byte weighted 3x (the SELECT CTAs' prologue and dequantisation; measured on
                  // the LLaMA3-8B down site: 40% companions, layer 84.2 -> 82.4 us)
        static const int pct_env = env_int("LAROSA_W4_COMP_PCT", 0);   // tuning
        const int total = std::max(2, sm_count() * 2 / n_sl);
        const double main_b = (double)k * (C::kRowBytes + 2 * C::kGroups);
        const double comp_b = (double)a.d2 * C::kCompRowBytes;
        int n2 = pct_env > 0 ? (total * pct_env + 50) / 100 : (int)(total * comp_b / (3.0 * main_b + comp_b) + 0.5);
        n2 = std::max(1, std::min(n2, total - by_cap));
        a.n_splits = std::max(by_cap, total - n2);
        a.n_splits2 = n2;
    }
    a.list_cap = (int)(32 * ((nwords + a.n_splits - 1) / a.n_splits));
    if (a.W2) {   // a companion's values live in the list: c_n <= list_cap
        a.n_splits2 = std::max<int>(a.n_splits2, (int)((a.d2 + a.list_cap - 1) / a.list_cap));
        if (a.n_splits + a.n_splits2 > 65535) return fail(LAROSA_EUNSUPPORTED, "W4 site: too many CTAs");
    }
    const size_t smem = w4_smem_bytes<SC>((int)d_in, a.list_cap);
    if (smem > 227 * 1024) return fail(LAROSA_EUNSUPPORTED, "W4 site: shared memory plan too large");
    LAROSA_TRY(cuda_check(allow_smem(gemv_w4_select_kernel<SC>, smem), "cudaFuncSetAttribute(gemv_w4)"));
    return cuda_check(launch(gemv_w4_select_kernel<SC>, dim3(n_sl, a.n_splits + a.n_splits2), dim3(kGemvThreads), smem,
                             st, a, Wq, S),
                      "gemv_w4 launch");
}

// slice width: 512 for a site of <= 4096 outputs without companions (the O projection: its tail was
// longer than its stream at 1024), 1024 otherwise (16-byte loads stream the large sites faster).
// Measured on the LLaMA3-8B W4 layer: O 16.4 -> 13.4 us at 512; gate|up 23.1 vs 26.0, down 19.5 vs
// 22.3 us in favour of 1024.
larosa_status launch_gemv_w4(GemvArgs a, const uint8_t* Wq, const uint16_t* S, cudaStream_t st) {
    if (a.d_out % kSliceCols || a.d_out > 65536)
        return fail(LAROSA_EUNSUPPORTED, "W4 site: d_out must be a multiple of 256 (<= 65536)");
    static const int forced = env_int("LAROSA_W4_SLICE", 0);   // tuning: 512 or 1024
    const int sc = forced == 512 || forced == 1024 ? forced : (a.d_out <= 4096 && !a.W2 ? 512 : 1024);
    return sc == 512 ? launch_gemv_w4_t<512>(a, Wq, S, st) : launch_gemv_w4_t<1024>(a, Wq, S, st);
}

// ============================================================================== small launches
template <int MODE, int EPT>
larosa_status launch_topk_t(const TopkKernelArgs& a, int batch, cudaStream_t st) {
    auto kern = topk_kernel<MODE, EPT>;
    LAROSA_TRY(cuda_check(allow_smem(kern, topk_smem_bytes(LAROSA_MAX_DIM)), "cudaFuncSetAttribute(topk)"));
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

template <int EPT>
larosa_status launch_rule_select_t(const TopkKernelArgs& a, int batch, cudaStream_t st) {
    return cuda_check(launch(rule_select_kernel<EPT>, dim3(batch), dim3(kRsThreads), 0, st, a), "rule_select launch");
}

larosa_status launch_topk(const TopkKernelArgs& a, int batch, cudaStream_t st) {
    // the per-token rule from a plain source (the batch 2-16 layer and shard phases): one CTA per
    // token (tuning: LAROSA_RULE_CTA=0 = the cluster kernel)
    static const int rule_cta = env_int("LAROSA_RULE_CTA", 1);
    if (rule_cta && a.rule_out && a.mode == SRC_PLAIN && !a.idx && !a.vals && !a.mask && !a.xr_out && !a.zero &&
        !a.scale && a.d <= kRsThreads * 32) {
        const int ept = (a.d + kRsThreads - 1) / kRsThreads;
        if (ept <= 4) return launch_rule_select_t<4>(a, batch, st);
        if (ept <= 8) return launch_rule_select_t<8>(a, batch, st);
        if (ept <= 16) return launch_rule_select_t<16>(a, batch, st);
        return launch_rule_select_t<32>(a, batch, st);
    }
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

// attention: the n_chunks CTAs of a kv group form one thread-block cluster when n_chunks <= 8
// (split-KV merge through distributed shared memory), else the ticket merge
// Attention kernel choice (LAROSA_ATTN: 0 auto, 1 split-KV + ticket merge, 2 split-KV with the
// cluster merge, 3 single-pass per head / group).  Auto: max_ctx <= 256 -> single pass, else the
// ticket merge.  Measured (LLaMA3-8B decode step, ctx 256, p = 0.4): B = 1 2.942 / 2.943 / 2.919 ms,
// B = 16 6.158 / 6.361 / 5.901 ms for modes 1 / 2 / 3 (the cluster merge waits on the slowest chunk
// CTA and rank 0's DSMEM merge; it stays selectable).
int attn_mode(int64_t max_ctx, int n_chunks) {
    static const int forced = env_int("LAROSA_ATTN", 0);
    if (forced == 2 && n_chunks >= 1 && n_chunks <= 8) return 2;
    if (forced == 1) return 1;
    return max_ctx <= kAgMaxCtx ? 3 : 1;
}

larosa_status launch_attention(AttnArgs aa, int units, int hd, int G, cudaStream_t st) {
    const int mode = attn_mode(aa.max_ctx, aa.n_chunks);
    if (mode == 3) {
        // units = batch * Hq query heads: one CTA per head when they fit one wave, else one per group
        static const int hpc_env = env_int("LAROSA_ATTN_HPC", 0);   // tuning
        int hpc = units <= sm_count() ? 1 : G;
        if (hpc_env > 0 && G % hpc_env == 0) hpc = hpc_env;
        const size_t smem = attn_group_smem_bytes(hd, hpc);
        auto kern = hd == 128 ? attn_group_kernel<4> : attn_group_kernel<2>;
        LAROSA_TRY(cuda_check(allow_smem(kern, smem), "cudaFuncSetAttribute(attention)"));
        return cuda_check(launch(kern, dim3(units / hpc), dim3(kAgThreads), smem, st, aa, hpc), "attention launch");
    }
    const size_t smem = attn_smem_bytes(hd);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(units, aa.n_chunks);
    cfg.blockDim = dim3(kAttnThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (mode == 2) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = 1;
        at[na].val.clusterDim.y = aa.n_chunks;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    if (mode == 2)
        return cuda_check(cudaLaunchKernelEx(&cfg, hd == 128 ? attention_kernel<4, true> : attention_kernel<2, true>, aa),
                          "attention launch");
    return cuda_check(cudaLaunchKernelEx(&cfg, hd == 128 ? attention_kernel<4, false> : attention_kernel<2, false>, aa),
                      "attention launch");
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

extern "C" larosa_status larosa_error_flags(void* ws, int32_t clear, uint32_t* flags, larosa_stream_t stream) {
    if (!ws || !flags) return fail(LAROSA_EINVAL, "error_flags: NULL pointer");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    uint32_t* w = static_cast<uint32_t*>(ws) + kErrWord;
    LAROSA_TRY(cuda_check(cudaMemcpyAsync(flags, w, sizeof(uint32_t), cudaMemcpyDeviceToHost, st), "error_flags: read"));
    if (clear) LAROSA_TRY(cuda_check(cudaMemsetAsync(w, 0, sizeof(uint32_t), st), "error_flags: clear"));
    return cuda_check(cudaStreamSynchronize(st), "error_flags: synchronize");
}

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
    ErrScope err_scope(c);
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
    a.d_in = (int)d_in;                  // bounds the union's row count (tcgen05 plan)
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
        // the token masks are zero at rest: the GEMV below re-zeroes them once the union kernel
        // has consumed them (no memset on the path)
        const int nw = (int)((d_in + 31) / 32);
        a.zero_hist = mask;
        a.zero_words = batch * nw;
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
    a.epi = EPI_STORE;
    a.tickets = c.counters(kGemvTicketBase);
    a.bias = bias;
    a.out = y;
    a.out_ld = d_out;
    return launch_gemv(a, p, bp, st);
}

// ============================================================================== fused Top-K + GEMV
static void carve_topk_gemv(Carver& c, int64_t d_in, int64_t d_out, unsigned long long** acc, SiteSel* sel) {
    unsigned long long* a = c.take<unsigned long long>((size_t)d_out);
    SiteSel q;
    q.hist = c.take<uint32_t>(kSelHistAlloc);
    q.pool = c.take<uint2>((size_t)kSelFine * kPoolCap);
    q.ssq = c.take<float>((size_t)(d_in + kSliceCols - 1) / kSliceCols);
    if (acc) *acc = a;
    if (sel) *sel = q;
}

extern "C" size_t larosa_topk_sparse_gemv_workspace_size(int64_t d_in, int64_t d_out) {
    if (d_in <= 0 || d_out <= 0) return 0;
    Carver c(nullptr);
    carve_topk_gemv(c, d_in, d_out, nullptr, nullptr);
    return c.size();
}

static larosa_status topk_sparse_gemv_impl(const float* x, int64_t d_in, int64_t k, float rms_eps, const uint16_t* W,
                                           int64_t d_out, int64_t ld, const uint16_t* bias, const float* x2,
                                           const uint16_t* W2, int64_t d2, float* y, int32_t prepared, void* ws,
                                           size_t ws_bytes, cudaStream_t st) {
    if (!x || !W || !y) return fail(LAROSA_EINVAL, "topk_sparse_gemv: NULL pointer");
    if (W2 || x2) {
        if (!W2 || !x2) return fail(LAROSA_EINVAL, "topk_sparse_gemv_dense2: NULL pointer");
        if (d2 <= 0 || d2 > LAROSA_MAX_DIM) return fail(LAROSA_EINVAL, "topk_sparse_gemv_dense2: d2 outside [1, %d]",
                                                        LAROSA_MAX_DIM);
        if (!aligned16(W2)) return fail(LAROSA_EINVAL, "topk_sparse_gemv_dense2: W2 must be 16-byte aligned");
    }
    if (d_in <= 0 || d_out <= 0) return fail(LAROSA_EINVAL, "topk_sparse_gemv: d_in, d_out must be > 0");
    if (k < 0 || k > d_in) return fail(LAROSA_EINVAL, "topk_sparse_gemv: k outside [0, d_in]");
    if (d_in > LAROSA_MAX_DIM) return fail(LAROSA_EUNSUPPORTED, "topk_sparse_gemv: d_in > %d", LAROSA_MAX_DIM);
    if (d_in % 8) return fail(LAROSA_EUNSUPPORTED, "topk_sparse_gemv: d_in %% 8 != 0");
    if (ld < d_out) return fail(LAROSA_ESHAPE, "topk_sparse_gemv: ld < d_out");
    if (ld % 8 || d_out % 8) return fail(LAROSA_EUNSUPPORTED, "topk_sparse_gemv: ld and d_out must be multiples of 8");
    if (d_out > (int64_t)256 * kSliceCols) return fail(LAROSA_EUNSUPPORTED, "topk_sparse_gemv: d_out > 65536");
    if (!aligned16(W) || !aligned16(x) || !aligned16(y) || (bias && !aligned16(bias)))
        return fail(LAROSA_EINVAL, "topk_sparse_gemv: pointers must be 16-byte aligned");
    const size_t need = larosa_topk_sparse_gemv_workspace_size(d_in, d_out);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "topk_sparse_gemv: workspace %zu < %zu", ws_bytes, need);
    Carver c(ws);
    ErrScope err_scope(c);
    unsigned long long* acc;
    SiteSel sel;
    carve_topk_gemv(c, d_in, d_out, &acc, &sel);
    if (rms_eps < 0.f) sel.ssq = nullptr;
    if (!prepared)
        LAROSA_TRY(cuda_check(launch(select_prep_kernel, dim3(n_slices_of(d_in)), dim3(kPrepThreads), 0, st, x, (int)d_in,
                                     sel, c.counters(kPrepBarrier), (float*)nullptr),
                              "select prep launch"));
    const GemvPlan p = W2 ? plan_gemv_comp(d_out, k, d_in, d2) : plan_gemv(d_out, k, 1, GEMV_SELECT, d_in);
    GemvArgs a = gemv_args_base();
    a.W = W;
    a.ld = ld;
    a.d_out = (int)d_out;
    a.mode = GEMV_SELECT;
    a.x = x;
    a.ldx = d_in;
    a.d_in = (int)d_in;
    a.sel = sel;
    a.sel_nssq = (int)((d_in + kSliceCols - 1) / kSliceCols);
    a.sel_k = (int)k;
    a.sel_eps = rms_eps;
    a.batch = 1;
    a.acc = acc;
    a.acc_ld = d_out;
    a.epi = EPI_STORE;
    a.tickets = c.counters(kGemvTicketBase);
    a.bias = bias;
    a.out = y;
    a.out_ld = d_out;
    a.W2 = W2;
    a.x2 = x2;
    a.d2 = (int)d2;
    return launch_gemv(a, p, 1, st);
}

extern "C" larosa_status larosa_topk_sparse_gemv(const float* x, int64_t d_in, int64_t k, float rms_eps,
                                                 const uint16_t* W, int64_t d_out, int64_t ld, const uint16_t* bias,
                                                 float* y, int32_t prepared, void* ws, size_t ws_bytes,
                                                 larosa_stream_t stream) {
    return topk_sparse_gemv_impl(x, d_in, k, rms_eps, W, d_out, ld, bias, nullptr, nullptr, 0, y, prepared, ws,
                                 ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" larosa_status larosa_topk_sparse_gemv_dense2(const float* x, int64_t d_in, int64_t k, float rms_eps,
                                                        const uint16_t* W, int64_t d_out, int64_t ld,
                                                        const float* x2, const uint16_t* W2, int64_t d2, float* y,
                                                        int32_t prepared, void* ws, size_t ws_bytes,
                                                        larosa_stream_t stream) {
    if (!x2 || !W2) return fail(LAROSA_EINVAL, "topk_sparse_gemv_dense2: NULL pointer");
    return topk_sparse_gemv_impl(x, d_in, k, rms_eps, W, d_out, ld, nullptr, x2, W2, d2, y, prepared, ws, ws_bytes,
                                 reinterpret_cast<cudaStream_t>(stream));
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
    ErrScope err_scope(c);
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
namespace {
using PFN_encodeTiled_t = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled_t tensor_map_encoder() {
    static const PFN_encodeTiled_t fn = [] {   // thread-safe one-time initialisation
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_encodeTiled_t>(p);
        return (PFN_encodeTiled_t) nullptr;
    }();
    return fn;
}
// K-major bf16 matrix [rows][K]: boxes of 64 (K) x box_rows, 128-byte swizzle
bool make_kmajor_map(CUtensorMap* m, const void* base, int64_t rows, int64_t K, int box_rows) {
    PFN_encodeTiled_t enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {(cuuint32_t)kFoldBK, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// row-major bf16 weights [d_in][ld] (d_out columns used): boxes of 64 columns x 64 rows, 128-byte
// swizzle; rows >= d_in and columns >= d_out read as zero (gemv_tc DENSE / THRESH)
bool make_w_mn_map(CUtensorMap* m, const void* W, int64_t d_in, int64_t d_out, int64_t ld) {
    PFN_encodeTiled_t enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)d_out, (cuuint64_t)d_in};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(W), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
int fold_bn(int64_t n) { return n % 256 == 0 ? 256 : (n % 128 == 0 ? 128 : 0); }
// output [rows][cols] = M x N; K = d (rows for LEFT, cols for RIGHT)
bool fold_tc_supported(int64_t rows, int64_t cols, bool left) {
    const int64_t K = left ? rows : cols;
    return rows % kFoldBM == 0 && fold_bn(cols) != 0 && K % kFoldBK == 0 && env_int("LAROSA_FOLD_SIMT", 0) == 0;
}
size_t fold_ws_bytes(int64_t rows, int64_t cols, bool left) {
    if (!fold_tc_supported(rows, cols, left)) return 256;
    const int64_t d = left ? rows : cols;
    return (size_t)2 * d * d * 2 + (left ? (size_t)cols * rows * 2 : 0) + 1024;
}

template <int BN, bool AS, bool BS, bool F32OUT = false>
cudaError_t launch_fold_tc(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0, const CUtensorMap& b1,
                           void* out, int M, int N, int K, cudaStream_t st, float scale = 1.0f, int accumulate = 0) {
    auto kern = fold_tc_kernel<BN, AS, BS, F32OUT>;
    constexpr int smem = fold_smem_bytes<BN, AS, BS>();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<dim3(N / BN, M / kFoldBM), kFoldThreads, smem, st>>>(a0, a1, b0, b1, out, N, K, scale, accumulate);
    return cudaGetLastError();
}

// LEFT : out[d][cols]  = (Q diag gamma)^T W      A = split((Q diag gamma)^T) [d][d], B = W^T [cols][d]
// RIGHT: out[rows][d]  = W Q                     A = W [rows][d],                B = split(Q^T) [d][d]
cudaError_t fold_tc_run(const float* Q, const float* gamma, const uint16_t* W, uint16_t* out, int64_t rows,
                        int64_t cols, bool left, void* ws, cudaStream_t st) {
    const int64_t d = left ? rows : cols;
    uint16_t* s_hi = static_cast<uint16_t*>(ws);
    uint16_t* s_lo = s_hi + (size_t)d * d;
    const dim3 tb(32, 8), tg((unsigned)((d + 31) / 32), (unsigned)((d + 31) / 32));
    split_transpose_kernel<<<tg, tb, 0, st>>>(Q, left ? gamma : nullptr, s_hi, s_lo, (int)d, (int)d);
    CUtensorMap a0, a1, b0, b1;
    const int M = (int)rows, N = (int)cols, K = (int)d;
    const int bn = fold_bn(N);
    if (left) {
        uint16_t* wt = s_lo + (size_t)d * d;
        transpose_bf16_kernel<<<dim3((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32)), tb, 0, st>>>(
            W, wt, (int)rows, (int)cols);
        if (!make_kmajor_map(&a0, s_hi, M, K, kFoldBM) || !make_kmajor_map(&a1, s_lo, M, K, kFoldBM) ||
            !make_kmajor_map(&b0, wt, N, K, bn))
            return cudaErrorInvalidValue;
        b1 = b0;
        return bn == 256 ? launch_fold_tc<256, true, false>(a0, a1, b0, b1, out, M, N, K, st)
                         : launch_fold_tc<128, true, false>(a0, a1, b0, b1, out, M, N, K, st);
    }
    if (!make_kmajor_map(&a0, W, M, K, kFoldBM) || !make_kmajor_map(&b0, s_hi, N, K, bn) ||
        !make_kmajor_map(&b1, s_lo, N, K, bn))
        return cudaErrorInvalidValue;
    a1 = a0;
    return bn == 256 ? launch_fold_tc<256, false, true>(a0, a1, b0, b1, out, M, N, K, st)
                     : launch_fold_tc<128, false, true>(a0, a1, b0, b1, out, M, N, K, st);
}
}  // namespace

extern "C" size_t larosa_fold_workspace_size(int64_t rows, int64_t cols, int side) {
    if (rows <= 0 || cols <= 0) return 0;
    return fold_ws_bytes(rows, cols, side == LAROSA_LEFT_QT);
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
    if (!aligned16(W) || !aligned16(Wout)) return fail(LAROSA_EINVAL, "fold: W, Wout must be 16-byte aligned");
    const bool left = side == LAROSA_LEFT_QT;
    const size_t need = larosa_fold_workspace_size(rows, cols, side);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "fold: workspace %zu < %zu", ws_bytes, need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (fold_tc_supported(rows, cols, left))
        return cuda_check(fold_tc_run(Q, gamma, W, Wout, rows, cols, left, ws, st), "fold (tcgen05)");
    // CUDA-core fp32 kernel: shapes without full 128 x 128 tiles (toy layers), or LAROSA_FOLD_SIMT=1
    const int M = (int)rows, N = (int)cols, K = left ? (int)rows : (int)cols;
    dim3 grid((N + 63) / 64, (M + 63) / 64);
    if (left)
        return cuda_check(launch(fold_simt_kernel<true>, grid, dim3(256), 0, st, Q, gamma, W, Wout, M, N, K,
                                 (const float*)nullptr), "fold");
    return cuda_check(launch(fold_simt_kernel<false>, grid, dim3(256), 0, st, Q, gamma, W, Wout, M, N, K,
                             (const float*)nullptr), "fold");
}

// ============================================================================== residual adapter
// A = Q_l^T Q_next with both factors split into bf16 hi + lo: the LEFT fold's tcgen05 kernel with
// ASPLIT (Q_l^T) and BSPLIT (Q_next^T as the K-major B operand): hi.hi + lo.hi + hi.lo in fp32.
extern "C" size_t larosa_residual_adapter_workspace_size(int64_t d) {
    if (d <= 0) return 0;
    return (size_t)4 * d * d * 2 + 1024;
}

extern "C" larosa_status larosa_residual_adapter(const float* Q_l, const float* Q_next, uint16_t* A, int64_t d,
                                                 void* ws, size_t ws_bytes, larosa_stream_t stream) {
    if (!Q_l || !Q_next || !A) return fail(LAROSA_EINVAL, "residual_adapter: NULL pointer");
    if (d <= 0) return fail(LAROSA_EINVAL, "residual_adapter: d must be > 0");
    if (d % 64) return fail(LAROSA_EUNSUPPORTED, "residual_adapter: d must be a multiple of 64");
    if (d > 32768) return fail(LAROSA_EUNSUPPORTED, "residual_adapter: d too large");
    if ((const void*)A == (const void*)Q_l || (const void*)A == (const void*)Q_next)
        return fail(LAROSA_EINVAL, "residual_adapter: A aliases a factor");
    if (!aligned16(A)) return fail(LAROSA_EINVAL, "residual_adapter: A must be 16-byte aligned");
    const size_t need = larosa_residual_adapter_workspace_size(d);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "residual_adapter: workspace %zu < %zu", ws_bytes, need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int M = (int)d;
    if (!fold_tc_supported(d, d, true)) {
        dim3 grid((M + 63) / 64, (M + 63) / 64);
        return cuda_check(launch(fold_simt_kernel<true>, grid, dim3(256), 0, st, Q_l, (const float*)nullptr,
                                 (const uint16_t*)nullptr, A, M, M, M, Q_next), "residual_adapter");
    }
    uint16_t* a_hi = static_cast<uint16_t*>(ws);
    uint16_t* a_lo = a_hi + (size_t)d * d;
    uint16_t* b_hi = a_lo + (size_t)d * d;
    uint16_t* b_lo = b_hi + (size_t)d * d;
    const dim3 tb(32, 8), tg((unsigned)((d + 31) / 32), (unsigned)((d + 31) / 32));
    split_transpose_kernel<<<tg, tb, 0, st>>>(Q_l, nullptr, a_hi, a_lo, M, M);      // A op [i][m] = Q_l[m][i]
    split_transpose_kernel<<<tg, tb, 0, st>>>(Q_next, nullptr, b_hi, b_lo, M, M);   // B op [j][m] = Q_next[m][j]
    LAROSA_TRY(cuda_check(cudaGetLastError(), "residual_adapter split"));
    CUtensorMap a0, a1, b0, b1;
    const int bn = fold_bn(M);
    if (!make_kmajor_map(&a0, a_hi, M, M, kFoldBM) || !make_kmajor_map(&a1, a_lo, M, M, kFoldBM) ||
        !make_kmajor_map(&b0, b_hi, M, M, bn) || !make_kmajor_map(&b1, b_lo, M, M, bn))
        return fail(LAROSA_ECUDA, "residual_adapter: tensor map");
    return cuda_check(bn == 256 ? launch_fold_tc<256, true, true>(a0, a1, b0, b1, A, M, M, M, st)
                                : launch_fold_tc<128, true, true>(a0, a1, b0, b1, A, M, M, M, st),
                      "residual_adapter (tcgen05)");
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

// ============================================================================== decode-step ends
extern "C" larosa_status larosa_embed(const uint16_t* E, int64_t vocab, int64_t d, const int32_t* tokens,
                                      int32_t batch, float* resid, larosa_stream_t stream) {
    if (!E || !tokens || !resid) return fail(LAROSA_EINVAL, "embed: NULL pointer");
    if (vocab <= 0 || d <= 0 || batch < 1) return fail(LAROSA_EINVAL, "embed: bad sizes");
    if (batch > LAROSA_MAX_BATCH) return fail(LAROSA_EUNSUPPORTED, "embed: batch > %d", LAROSA_MAX_BATCH);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    return cuda_check(launch(embed_kernel, dim3((unsigned)((d + 1023) / 1024), batch), dim3(1024), 0, st, E, tokens,
                             (int)d, resid),
                      "embed launch");
}

static void carve_lm_head(Carver& c, int32_t batch, int64_t d, int64_t vocab, unsigned long long** acc, float** xs,
                          float** logits, unsigned char** img = nullptr) {
    unsigned long long* a = c.take<unsigned long long>((size_t)batch * vocab);
    float* x = c.take<float>((size_t)batch * d);
    float* l = c.take<float>((size_t)batch * vocab);
    unsigned char* im = batch >= 8 ? c.take<unsigned char>(img_bytes(d)) : nullptr;
    if (acc) *acc = a;
    if (xs) *xs = x;
    if (logits) *logits = l;
    if (img) *img = im;
}

extern "C" size_t larosa_lm_head_workspace_size(int32_t batch, int64_t d, int64_t vocab) {
    if (batch < 1 || d <= 0 || vocab <= 0) return 0;
    Carver c(nullptr);
    carve_lm_head(c, batch, d, vocab, nullptr, nullptr, nullptr);
    return c.size();
}

extern "C" larosa_status larosa_lm_head(const float* resid, int32_t batch, int64_t d, const uint16_t* H, int64_t vocab,
                                        float rms_eps, float* logits, int32_t* next_token, void* ws, size_t ws_bytes,
                                        larosa_stream_t stream) {
    if (!resid || !H || !next_token) return fail(LAROSA_EINVAL, "lm_head: NULL pointer");
    if (batch < 1 || d <= 0 || vocab <= 0) return fail(LAROSA_EINVAL, "lm_head: bad sizes");
    if (batch > LAROSA_MAX_BATCH) return fail(LAROSA_EUNSUPPORTED, "lm_head: batch > %d", LAROSA_MAX_BATCH);
    if (vocab % 8 || d % 8) return fail(LAROSA_EUNSUPPORTED, "lm_head: vocab and d must be multiples of 8");
    // one slice ticket per column slice: 128-column slices on the tcgen05 path (batch >= 8), 256 otherwise;
    // size the check by the narrower one so either path fits the counter header
    if ((vocab + kTcCols - 1) / kTcCols > (int64_t)(kPrepBarrier - kGemvTicketBase))
        return fail(LAROSA_EUNSUPPORTED, "lm_head: vocab too large");
    if (!aligned16(H) || (logits && !aligned16(logits))) return fail(LAROSA_EINVAL, "lm_head: H, logits must be 16-byte aligned");
    const size_t need = larosa_lm_head_workspace_size(batch, d, vocab);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "lm_head: workspace %zu < %zu", ws_bytes, need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Carver c(ws);
    ErrScope err_scope(c);
    unsigned long long* acc;
    float *xs, *lg;
    unsigned char* img;
    carve_lm_head(c, batch, d, vocab, &acc, &xs, &lg, &img);
    if (!logits) logits = lg;
    LAROSA_TRY(cuda_check(launch(rms_rows_kernel, dim3(batch), dim3(kRowThreads), 0, st, resid, (int)d, rms_eps, xs),
                          "rms launch"));
    const int bp = pad_batch(batch);
    const GemvPlan p = plan_gemv(vocab, d, bp, GEMV_DENSE, d);
    GemvArgs a = gemv_args_base();
    if (use_tc_gemv(bp) && img) {   // the scaled rows as the tensor-core GEMV's token image
        LAROSA_TRY(launch_dense_image(xs, d, d, batch, img, st));
        a.img = img;
    }
    a.W = H;
    a.ld = vocab;
    a.d_out = (int)vocab;
    a.mode = GEMV_DENSE;
    a.x = xs;
    a.ldx = d;
    a.d_in = (int)d;
    a.batch = batch;
    a.acc = acc;
    a.acc_ld = vocab;
    a.epi = EPI_STORE;
    a.tickets = c.counters(kGemvTicketBase);
    a.out = logits;
    a.out_ld = vocab;
    LAROSA_TRY(launch_gemv(a, p, bp, st));
    return cuda_check(launch(argmax_kernel, dim3(batch), dim3(kRowThreads), 0, st, (const float*)logits, vocab,
                             (int)vocab, next_token),
                      "argmax launch");
}

// ============================================================================== decoder layer
namespace {
struct LayerWs {
    unsigned long long *acc_qkv, *acc_o, *acc_gu, *acc_down, *acc_adp;
    SiteSel sel[4];       // batch 1: selection data of the site inputs h1..h4 (gemv.cuh)
    ThreshOut* thr[4];    // batch > 1: per-token Top-K rules
    float* h2;
    float* rmid;
    float* h4;
    float* radp;          // r_mid + y_down, the adapter's input
    float* attn_part;
    unsigned* attn_cnt;
    unsigned* tickets[4]; // slice tickets of the O, gate|up, down, adapter GEMV epilogues
    unsigned char* img[4];   // batch >= 8: the sites' token operand images (gemv_img.cuh)
    unsigned char* img_raw[2];   // batch >= 8: unmasked images of h1 (A_mid) and h3 (the adapter)
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
    static const int forced = env_int("LAROSA_ATTN_CHUNK", 0);   // tuning: 16, 32 or 64 positions
    if (forced == 16 || forced == 32 || forced == 64) return forced;
    // enough CTAs to cover the SMs: units * n_chunks >= sm_count
    int ch = 4 * kAttnPosPerWarp;
    while (ch > 16 && units * ((max_ctx + ch - 1) / ch) < sm_count()) ch >>= 1;
    return ch;
}

int n_slices(int64_t n) { return (int)((n + kSliceCols - 1) / kSliceCols); }

void carve_layer(Carver& c, const LayerDims& L, int batch, int64_t max_ctx, LayerWs* ws) {
    LayerWs tmp;
    LayerWs* o = ws ? ws : &tmp;
    // zero-at-rest state first: GEMV accumulators and histograms
    o->acc_qkv = c.take<unsigned long long>((size_t)batch * L.nqkv);
    o->acc_o = c.take<unsigned long long>((size_t)batch * L.d);
    o->acc_gu = c.take<unsigned long long>((size_t)batch * L.dgu);
    o->acc_down = c.take<unsigned long long>((size_t)batch * L.d);
    o->acc_adp = c.take<unsigned long long>((size_t)batch * L.d);
    for (int s = 0; s < 4; ++s) {
        SiteSel& q = o->sel[s];
        q.hist = c.take<uint32_t>(kSelHistAlloc);
        q.pool = batch == 1 ? c.take<uint2>((size_t)kSelFine * kPoolCap) : nullptr;
        q.ssq = (s == 0 || s == 2) ? c.take<float>((size_t)batch * n_slices(L.d)) : nullptr;
    }
    for (int s = 0; s < 4; ++s) o->thr[s] = c.take<ThreshOut>((size_t)batch);
    o->h2 = c.take<float>((size_t)batch * L.nq);
    o->rmid = c.take<float>((size_t)batch * L.d);
    o->h4 = c.take<float>((size_t)batch * L.inter);
    o->radp = c.take<float>((size_t)batch * L.d);
    const int ch = attn_chunk(max_ctx, batch * (int)L.hq);
    const int nch = (int)((max_ctx + ch - 1) / ch);
    o->attn_part = c.take<float>((size_t)batch * L.hq * nch * (L.hd + 2));
    o->attn_cnt = c.counters(kAttnCounterBase);
    for (int j = 0; j < 4; ++j) o->tickets[j] = c.counters(kGemvTicketBase + 256 * j);
    if (batch >= 8) {
        const int64_t din[4] = {L.d, L.nq, L.d, L.inter};
        for (int j = 0; j < 4; ++j) o->img[j] = c.take<unsigned char>(img_bytes(din[j]));
        for (int j = 0; j < 2; ++j) o->img_raw[j] = c.take<unsigned char>(img_bytes(L.d));
    } else {
        for (int j = 0; j < 4; ++j) o->img[j] = nullptr;
        o->img_raw[0] = o->img_raw[1] = nullptr;
    }
}

larosa_status validate_layer(const larosa_layer_weights* w, const larosa_layer_plan* p, const larosa_layer_state* s) {
    if (!w || !p || !s) return fail(LAROSA_EINVAL, "sparse_layer: NULL struct");
    if ((!w->w_qkv && !w->w4_codes[0]) || (!w->w_o && !w->w4_codes[1]) || (!w->w_gu && !w->w4_codes[2]) ||
        (!w->w_down && !w->w4_codes[3]))
        return fail(LAROSA_EINVAL, "sparse_layer: NULL weight");
    if (!s->resid || !s->k_cache || !s->v_cache || !s->pos) return fail(LAROSA_EINVAL, "sparse_layer: NULL state");
    if (s->batch < 1) return fail(LAROSA_EINVAL, "sparse_layer: batch < 1");
    if (s->batch > LAROSA_MAX_BATCH) return fail(LAROSA_EUNSUPPORTED, "sparse_layer: batch > 16");
    if (w->d <= 0 || w->inter <= 0 || w->n_q_heads <= 0 || w->n_kv_heads <= 0 || w->head_dim <= 0)
        return fail(LAROSA_EINVAL, "sparse_layer: dims must be > 0");
    if (w->n_q_heads % w->n_kv_heads) return fail(LAROSA_ESHAPE, "sparse_layer: Hq %% Hkv != 0");
    if (w->adapter_in_down && !w->adapter) return fail(LAROSA_EINVAL, "sparse_layer: adapter_in_down needs the adapter");
    for (int j = 0; j < 4; ++j) {
        if (!w->w4_codes[j] != !w->w4_scales[j]) return fail(LAROSA_EINVAL, "sparse_layer: W4 site %d needs codes and scales", j);
        if (w->w4_codes[j] && s->batch != 1) return fail(LAROSA_EUNSUPPORTED, "sparse_layer: W4 sites need batch 1");
        if (w->w4_codes[j] && (!aligned16(w->w4_codes[j]) || (reinterpret_cast<uintptr_t>(w->w4_scales[j]) & 3)))
            return fail(LAROSA_EINVAL, "sparse_layer: W4 codes 16-byte, scales 4-byte aligned");
    }
    {
        const int64_t douts[4] = {(w->n_q_heads + 2 * w->n_kv_heads) * w->head_dim, w->d, 2 * w->inter, w->d};
        for (int j = 0; j < 4; ++j)
            if (w->w4_codes[j] && douts[j] % 256)
                return fail(LAROSA_EUNSUPPORTED, "sparse_layer: W4 site %d needs D_out %% 256 == 0", j);
    }
    if (w->w4_codes[1] && w->adapter_mid) return fail(LAROSA_EUNSUPPORTED, "sparse_layer: a W4 O site with adapter_mid");
    if ((s->host_in || s->host_out) && s->batch != 1) return fail(LAROSA_EINVAL, "sparse_layer: host_in/out need batch 1");
    if (w->n_q_heads / w->n_kv_heads > kAttnMaxG) return fail(LAROSA_EUNSUPPORTED, "sparse_layer: GQA group > 8");
    if (w->head_dim != 64 && w->head_dim != 128) return fail(LAROSA_EUNSUPPORTED, "sparse_layer: head_dim must be 64 or 128");
    if (w->d % 8 || w->inter % LAROSA_GU_BLOCK) return fail(LAROSA_EUNSUPPORTED, "sparse_layer: d %% 8 or inter %% 64");
    if (w->d > LAROSA_MAX_DIM || w->inter > LAROSA_MAX_DIM || w->n_q_heads * w->head_dim > LAROSA_MAX_DIM)
        return fail(LAROSA_EUNSUPPORTED, "sparse_layer: dimension > %d", LAROSA_MAX_DIM);
    if (s->max_ctx <= 0) return fail(LAROSA_EINVAL, "sparse_layer: max_ctx must be > 0");
    if ((int64_t)s->batch * w->n_q_heads > (int64_t)kAttnGroupCounterOff)
        return fail(LAROSA_EUNSUPPORTED, "sparse_layer: batch * Hq too large");
    const int64_t nq = w->n_q_heads * w->head_dim;
    if (p->k_h1 < 0 || p->k_h1 > w->d || p->k_h2 < 0 || p->k_h2 > nq || p->k_h3 < 0 || p->k_h3 > w->d || p->k_h4 < 0 ||
        p->k_h4 > w->inter || p->k_next_h1 > w->d)
        return fail(LAROSA_EINVAL, "sparse_layer: a k is outside [0, D_in of its site]");
    const void* ptrs[] = {w->w_qkv, w->w_o, w->w_gu, w->w_down, w->adapter, w->b_qkv, s->resid, s->k_cache, s->v_cache,
                          w->adapter_mid};
    for (const void* q : ptrs)
        if (q && !aligned16(q)) return fail(LAROSA_EINVAL, "sparse_layer: pointers must be 16-byte aligned");
    return LAROSA_OK;
}

larosa_status tap_copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (!dst) return LAROSA_OK;
    return cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st), "tap copy");
}

// profiling aid: bitmask of the layer's kernels that are launched (default: all)
int g_phase_mask = -2;
unsigned long long* g_tl = nullptr;   // debug timeline: [n][1024 CTAs][8] u64, one block per layer kernel
int g_tl_n = 0;
int layer_phase_mask() {
    if (g_phase_mask == -2) g_phase_mask = env_int("LAROSA_LAYER_PHASES", -1);
    return g_phase_mask;
}
}  // namespace

extern "C" void larosa_debug_set_layer_phases(int mask) { g_phase_mask = mask; }
extern "C" void larosa_debug_set_timeline(void* dev_buf, int n_slots) {
    g_tl = static_cast<unsigned long long*>(dev_buf);
    g_tl_n = n_slots;
}

extern "C" size_t larosa_layer_workspace_size(const larosa_layer_weights* w, int32_t batch, int64_t max_ctx) {
    if (!w || batch < 1 || max_ctx <= 0) return 0;
    Carver c(nullptr);
    carve_layer(c, layer_dims(w), batch, max_ctx, nullptr);
    return c.size();
}

// Kernel sequence of one decode step of one layer (every kernel launched with PDL).
// Batch 1 (the Top-K selection of each site is fused into the consuming GEMV, SELECT):
//   [prep(h1 = r): histogram + RMS partials]          unless state->chained
//   gemv W_qkv   SELECT(h1, k1, RMS)  -> acc_qkv                 (EPI_NONE)
//   attention    <- acc_qkv (+bias, RoPE, KV append) -> h2, hist(h2); re-zero acc_qkv
// (each histogram is re-zeroed by a later kernel once its consumer has completed)
//   gemv W_o     SELECT(h2, k2)       -> r_mid = r + y, hist(h3), RMS partials(h3)
//   gemv W_gu    SELECT(h3, k3, RMS)  -> h4 = SiLU(g) u, hist(h4)
//   gemv W_down  SELECT(h4, k4)       -> r_adp = r_mid + y          [no adapter: -> r, hist(h1)]
//   gemv A_l     DENSE(r_adp)         -> r = y, hist(h1'), RMS partials(h1')  (next layer's h1)
// Batch > 1: the same GEMVs in THRESH mode, each preceded by the cluster Top-K kernel that
// publishes every token's rule (Tk, Ti, s) from the materialised site vector.
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
    const bool fused = B == 1;
    Carver c(ws);
    ErrScope err_scope(c);
    LayerWs W;
    carve_layer(c, L, B, s->max_ctx, &W);
    larosa_layer_taps T;
    if (taps)
        T = *taps;
    else
        memset(&T, 0, sizeof(T));
    const int nsl_d = n_slices(L.d);
    auto tl_slot = [&](int i) -> unsigned long long* { return g_tl && i < g_tl_n ? g_tl + 16384 * i : nullptr; };

    // exact index-list Top-K of a materialised site vector (parity taps only)
    auto tap_topk = [&](const float* x, int64_t din, int64_t k, float eps, int32_t* idx, float* vals) -> larosa_status {
        if (!idx || !vals) return LAROSA_OK;
        TopkKernelArgs tk = topk_args_base();
        tk.x = x;
        tk.ldx = din;
        tk.d = (int)din;
        tk.k = (int)k;
        tk.rms_eps = eps;
        tk.idx = idx;
        tk.vals = vals;
        return launch_topk(tk, B, st);
    };
    // batch > 1: every token's selection rule (and at batch >= 8 the site's token image; for h1 / h3
    // also the unmasked image the dense A_mid / adapter GEMV reads) from one CTA per token
    // tuning (B = 16 LLaMA3-8B layer, in graph: 0 180 us, 1 233 us, 2 172 us): 1 = rule_image_kernel
    // (rule + image in one CTA per token, large shared memory: no early residency), 2 = the cluster Top-K rule +
    // rule_apply_image_kernel, 0 = the cluster Top-K rule and gemv_tc (no image)
    static const int rule_kernel = env_int("LAROSA_RULE_KERNEL", 2);
    const bool img_path = !fused && use_tc_gemv(bp) && W.img[0] != nullptr && rule_kernel != 0;
    auto rule_topk = [&](int si, const float* x, int64_t din, int64_t k, float eps) -> larosa_status {
        void* raw = nullptr;
        if (img_path && si == 0 && w->adapter_mid) raw = W.img_raw[0];
        if (img_path && si == 2 && w->adapter && w->adapter_in_down) raw = W.img_raw[1];
        if (rule_kernel == 3) return launch_rule_image_reg(x, din, din, k, eps, B, W.thr[si], img_path ? W.img[si] : nullptr,
                                                           raw, st);
        if (rule_kernel != 1) {   // the cluster Top-K rule (+ the image from it, mode 2)
            TopkKernelArgs r = topk_args_base();
            r.x = x;
            r.ldx = din;
            r.d = (int)din;
            r.k = (int)k;
            r.rms_eps = eps;
            r.rule_out = W.thr[si];
            r.tl = tl_slot(6 + si);
            // (tuning: 0 = the image from a separate rule_apply_image launch)
            static const int topk_image = env_int("LAROSA_TOPK_IMAGE", 1);
            if (img_path && topk_image) {   // the cluster Top-K kernel writes the image too
                r.img = W.img[si];
                r.img_raw = (unsigned char*)raw;
                return launch_topk(r, B, st);
            }
            LAROSA_TRY(launch_topk(r, B, st));
            if (!img_path) return LAROSA_OK;
            const int groups = (int)((din + 7) / 8);
            return cuda_check(launch(rule_apply_image_kernel, dim3((unsigned)((groups + 255) / 256), B), dim3(256), 0, st,
                                     x, din, (int)din, (const ThreshOut*)W.thr[si], W.img[si], (unsigned char*)raw),
                              "rule_apply_image launch");
        }
        return launch_rule_image(x, din, din, k, eps, B, W.thr[si], img_path ? W.img[si] : nullptr, raw, st);
    };
    // the GEMV of site si on the site vector x (SELECT at batch 1, THRESH otherwise)
    auto site_gemv = [&](int si, const float* x, int64_t din, int64_t k, float eps, const uint16_t* Wt, int64_t dout,
                         unsigned long long* acc) {
        GemvArgs a = gemv_args_base();
        a.W = Wt;
        a.ld = dout;
        a.d_out = (int)dout;
        a.x = x;
        a.ldx = din;
        a.d_in = (int)din;
        a.batch = B;
        a.acc = acc;
        a.acc_ld = dout;
        if (fused) {
            a.mode = GEMV_SELECT;
            a.sel = W.sel[si];
            if (eps < 0.f) a.sel.ssq = nullptr;
            a.sel_nssq = nsl_d;
            a.sel_k = (int)k;
            a.sel_eps = eps;
        } else {
            a.mode = GEMV_THRESH;
            a.thr = W.thr[si];
            if (img_path) a.img = W.img[si];
        }
        return a;
    };
    auto plan_site = [&](int64_t dout, int64_t din, int64_t k) {
        return fused ? plan_gemv(dout, k, 1, GEMV_SELECT, din) : plan_gemv(dout, din, bp, GEMV_THRESH, din);
    };
    // site si's GEMV: the W4A16 kernel when the site has int4 weights (batch 1), else the bf16 one
    auto site_launch = [&](const GemvArgs& a, int si, const GemvPlan& p, int bpl) -> larosa_status {
        if (w->w4_codes[si]) return launch_gemv_w4(a, w->w4_codes[si], w->w4_scales[si], st);
        return launch_gemv(a, p, bpl, st);
    };
    // epilogue of a site GEMV; `next` = the site whose selection data it produces (-1: none)
    auto epi = [&](GemvArgs& a, int j, int mode, const float* res, float* out, int next) {
        a.epi = mode;
        a.tickets = W.tickets[j];
        a.res = res;
        a.res_ld = L.d;
        a.out = out;
        a.out_ld = mode == EPI_SILU ? L.inter : L.d;
        if (fused && next >= 0) {
            a.out_sel = W.sel[next];
            a.out_ssq = W.sel[next].ssq;   // RMS partials for h1 / h3
            a.out_ssq_ld = nsl_d;
        }
    };

    // ---- h1: r (RMS) -> QKV ---------------------------------------------------------------------
    if (fused) {
        if (!s->chained && on(0))
            LAROSA_TRY(cuda_check(launch(select_prep_kernel, dim3(n_slices_of(L.d)), dim3(kPrepThreads), 0, st,
                                         s->host_in ? s->host_in : (const float*)s->resid, (int)L.d, W.sel[0],
                                         c.counters(kPrepBarrier), s->host_in ? s->resid : (float*)nullptr),
                                  "select prep launch"));
    } else if (on(0)) {
        LAROSA_TRY(rule_topk(0, s->resid, L.d, plan->k_h1, w->rms_eps));
    }
    LAROSA_TRY(tap_topk(s->resid, L.d, plan->k_h1, w->rms_eps, T.idx_h1, T.vals_h1));
    if (on(1)) {
        GemvArgs a = site_gemv(0, s->resid, L.d, plan->k_h1, w->rms_eps, w->w_qkv, L.nqkv, W.acc_qkv);
        a.zero_hist = fused ? W.sel[3].hist : nullptr;   // h4's consumer (previous layer's down GEMV) is done
        a.tl = tl_slot(0);
        a.zero_words = kSelHistTotal;
        LAROSA_TRY(site_launch(a, 0, plan_site(L.nqkv, L.d, plan->k_h1), fused ? 1 : bp));
    }
    // ---- attention (finalises q / new k, v from acc_qkv, re-zeroes it) -> h2 ---------------------
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
        aa.chunk = attn_chunk(s->max_ctx, B * (int)L.hq);
        aa.n_chunks = (int)((s->max_ctx + aa.chunk - 1) / aa.chunk);
        aa.part = W.attn_part;
        aa.counters = W.attn_cnt;
        aa.out = W.h2;
        if (fused) aa.out_sel = W.sel[1];
        aa.keep_acc = fused && on(4);   // batch 1: the O GEMV re-zeroes acc_qkv
        aa.tl = tl_slot(1);

        if (on(2)) LAROSA_TRY(launch_attention(aa, B * (int)L.hq, (int)L.hd, L.G, st));
        LAROSA_TRY(tap_copy(T.h2, W.h2, sizeof(float) * B * L.nq, st));
    }
    // ---- h2 -> O; epilogue r_mid = r + y_o (h3) -------------------------------------------------
    if (!fused && on(3)) LAROSA_TRY(rule_topk(1, W.h2, L.nq, plan->k_h2, -1.0f));
    LAROSA_TRY(tap_topk(W.h2, L.nq, plan->k_h2, -1.0f, T.idx_h2, T.vals_h2));
    if (on(4)) {
        GemvArgs a = site_gemv(1, W.h2, L.nq, plan->k_h2, -1.0f, w->w_o, L.d, W.acc_o);
        const bool qb = w->adapter_mid != nullptr;   // r_mid = r A_mid + y_o (block-wise rotation)
        epi(a, 0, EPI_RESID, qb ? nullptr : s->resid, W.rmid, 2);
        if (fused) {   // attention (complete by now) left the QKV accumulators to be re-zeroed here
            a.zero_acc = W.acc_qkv;
            a.zero_acc_words = (int)L.nqkv;
        }
        a.tl = tl_slot(2);
        a.zero_hist = fused ? W.sel[0].hist : nullptr;   // h1's consumer (QKV) is done
        a.zero_words = kSelHistTotal;
        if (qb && fused) {   // the dense r rows of A_mid as companion CTAs of the O launch
            a.W2 = w->adapter_mid;
            a.x2 = s->resid;
            a.d2 = (int)L.d;
            LAROSA_TRY(launch_gemv(a, plan_gemv_comp(L.d, plan->k_h2, L.nq, L.d), 1, st));
        } else if (qb) {     // batch > 1: the O GEMV leaves its sums, the dense A_mid GEMV finalises
            const int epi_mode = a.epi;
            a.epi = EPI_NONE;
            LAROSA_TRY(launch_gemv(a, plan_site(L.d, L.nq, plan->k_h2), bp, st));
            GemvArgs b = gemv_args_base();
            b.W = w->adapter_mid;
            b.ld = L.d;
            b.d_out = (int)L.d;
            b.mode = GEMV_DENSE;
            b.x = s->resid;
            b.ldx = L.d;
            b.d_in = (int)L.d;
            b.batch = B;
            b.acc = W.acc_o;
            b.acc_ld = L.d;
            if (img_path) b.img = W.img_raw[0];
            epi(b, 0, epi_mode, nullptr, W.rmid, 2);
            LAROSA_TRY(launch_gemv(b, plan_gemv(L.d, L.d, bp, GEMV_DENSE, L.d), bp, st));
        } else {
            LAROSA_TRY(site_launch(a, 1, plan_site(L.d, L.nq, plan->k_h2), fused ? 1 : bp));
        }
    }
    LAROSA_TRY(tap_copy(T.r_mid, W.rmid, sizeof(float) * B * L.d, st));
    // ---- h3 (RMS) -> gate|up; epilogue h4 = SiLU(g) u ----------------------------------------------
    if (!fused && on(5)) LAROSA_TRY(rule_topk(2, W.rmid, L.d, plan->k_h3, w->rms_eps));
    LAROSA_TRY(tap_topk(W.rmid, L.d, plan->k_h3, w->rms_eps, T.idx_h3, T.vals_h3));
    if (on(6)) {
        GemvArgs a = site_gemv(2, W.rmid, L.d, plan->k_h3, w->rms_eps, w->w_gu, L.dgu, W.acc_gu);
        epi(a, 1, EPI_SILU, nullptr, W.h4, 3);
        a.tl = tl_slot(3);
        a.zero_hist = fused ? W.sel[1].hist : nullptr;   // h2's consumer (O) is done
        a.zero_words = kSelHistTotal;
        LAROSA_TRY(site_launch(a, 2, plan_site(L.dgu, L.d, plan->k_h3), fused ? 1 : bp));
    }
    LAROSA_TRY(tap_copy(T.h4, W.h4, sizeof(float) * B * L.inter, st));
    // ---- h4 -> down; epilogue r_mid + y_down (-> adapter input, or the next layer's r) ------------
    if (!fused && on(7)) LAROSA_TRY(rule_topk(3, W.h4, L.inter, plan->k_h4, -1.0f));
    LAROSA_TRY(tap_topk(W.h4, L.inter, plan->k_h4, -1.0f, T.idx_h4, T.vals_h4));
    const bool merged = w->adapter && w->adapter_in_down;
    if (merged && on(8)) {
        // r_next = r_mid A_l + h4[S4] W_down Q_{l+1}: one fixed-point accumulator, finalised once
        GemvArgs a = site_gemv(3, W.h4, L.inter, plan->k_h4, -1.0f, w->w_down, L.d, W.acc_down);
        a.zero_hist = fused ? W.sel[2].hist : nullptr;
        a.zero_words = kSelHistTotal;
        a.tl = tl_slot(4);
        if (fused) {
            a.W2 = w->adapter;
            a.x2 = W.rmid;
            a.d2 = (int)L.d;
            epi(a, 2, EPI_STORE, nullptr, s->resid, 0);
            a.out_host = s->host_out;
            if (w->w4_codes[3])
                LAROSA_TRY(launch_gemv_w4(a, w->w4_codes[3], w->w4_scales[3], st));
            else
                LAROSA_TRY(launch_gemv(a, plan_gemv_comp(L.d, plan->k_h4, L.inter, L.d), 1, st));
        } else {
            a.epi = EPI_NONE;
            LAROSA_TRY(launch_gemv(a, plan_site(L.d, L.inter, plan->k_h4), bp, st));
            GemvArgs b = gemv_args_base();
            b.W = w->adapter;
            b.ld = L.d;
            b.d_out = (int)L.d;
            b.mode = GEMV_DENSE;
            b.x = W.rmid;
            b.ldx = L.d;
            b.d_in = (int)L.d;
            b.batch = B;
            b.acc = W.acc_down;
            b.acc_ld = L.d;
            if (img_path) b.img = W.img_raw[1];
            epi(b, 3, EPI_STORE, nullptr, s->resid, 0);
            b.tl = tl_slot(5);
            LAROSA_TRY(launch_gemv(b, plan_gemv(L.d, L.d, bp, GEMV_DENSE, L.d), bp, st));
        }
        return LAROSA_OK;
    }
    if (merged) return LAROSA_OK;   // profiling mask without the down launch
    if (on(8)) {
        GemvArgs a = site_gemv(3, W.h4, L.inter, plan->k_h4, -1.0f, w->w_down, L.d, W.acc_down);
        if (w->adapter) {
            epi(a, 2, EPI_RESID, W.rmid, W.radp, -1);
        } else {
            epi(a, 2, EPI_RESID, W.rmid, s->resid, 0);
            a.out_host = s->host_out;
        }
        a.zero_hist = fused ? W.sel[2].hist : nullptr;   // h3's consumer (gate|up) is done
        a.tl = tl_slot(4);
        a.zero_words = kSelHistTotal;
        LAROSA_TRY(site_launch(a, 3, plan_site(L.d, L.inter, plan->k_h4), fused ? 1 : bp));
    }
    // ---- residual adapter r <- (r_mid + y_down) . A_l (dense GEMV) -------------------------
    if (w->adapter) {
        LAROSA_TRY(tap_copy(T.r_out, W.radp, sizeof(float) * B * L.d, st));
        if (on(9)) {
            const GemvPlan p = plan_gemv(L.d, L.d, bp, GEMV_DENSE, L.d);
            GemvArgs a = gemv_args_base();
            a.W = w->adapter;
            a.ld = L.d;
            a.d_out = (int)L.d;
            a.mode = GEMV_DENSE;
            a.x = W.radp;
            a.ldx = L.d;
            a.d_in = (int)L.d;
            a.batch = B;
            a.acc = W.acc_adp;
            a.acc_ld = L.d;
            epi(a, 3, EPI_STORE, nullptr, s->resid, 0);
            a.out_host = s->host_out;
            a.tl = tl_slot(5);
            LAROSA_TRY(launch_gemv(a, p, bp, st));
        }
    } else {
        LAROSA_TRY(tap_copy(T.r_out, s->resid, sizeof(float) * B * L.d, st));
    }
    return LAROSA_OK;
}

// ============================================================================== sharded layer
namespace {
struct ShardWs {
    SiteSel sel;                       // batch 1: selection data of the phase input (rebuilt each phase)
    ThreshOut* thr;                    // batch > 1: every token's Top-K rule of the phase input
    unsigned char *img, *img2;         // batch >= 8: token images of the phase input / of resid
    unsigned long long* acc;           // local projection accumulators [batch][largest phase]
    float* attn_part;
    unsigned* attn_cnt;
    unsigned* tickets;
};
struct ShardDims {
    int64_t d, inter, nq, hq_l, hkv_l, hd, dl, il, qkv_l;
    int G, batch;
};
ShardDims shard_dims(const larosa_layer_weights* w, const larosa_shard* sh) {
    ShardDims S;
    const int64_t n = sh->world;
    S.d = w->d;
    S.inter = w->inter;
    S.hd = w->head_dim;
    S.nq = w->n_q_heads * w->head_dim;
    S.hq_l = w->n_q_heads / n;
    S.hkv_l = w->n_kv_heads / n;
    S.dl = w->d / n;
    S.il = w->inter / n;
    S.qkv_l = (S.hq_l + 2 * S.hkv_l) * S.hd;
    S.G = (int)(S.hkv_l > 0 ? S.hq_l / S.hkv_l : 1);
    S.batch = sh->batch < 1 ? 1 : sh->batch;
    return S;
}
void carve_shard(Carver& c, const ShardDims& S, int64_t max_ctx, ShardWs* o) {
    ShardWs tmp;
    ShardWs* q = o ? o : &tmp;
    const int64_t dmax = std::max(std::max(S.d, S.nq), S.inter);
    const int64_t omax = std::max(std::max(S.qkv_l, S.dl), 2 * S.il);
    q->acc = c.take<unsigned long long>((size_t)S.batch * omax);
    q->sel.hist = c.take<uint32_t>(kSelHistAlloc);
    q->sel.pool = c.take<uint2>((size_t)kSelFine * kPoolCap);
    q->sel.ssq = c.take<float>((size_t)(dmax + kSliceCols - 1) / kSliceCols);
    q->thr = c.take<ThreshOut>((size_t)S.batch);
    q->img = S.batch >= 8 ? c.take<unsigned char>(img_bytes(dmax)) : nullptr;
    q->img2 = S.batch >= 8 ? c.take<unsigned char>(img_bytes(S.d)) : nullptr;
    const int ch = attn_chunk(max_ctx, (int)(S.batch * S.hq_l));
    const int nch = (int)((max_ctx + ch - 1) / ch);
    q->attn_part = c.take<float>((size_t)S.batch * S.hq_l * nch * (S.hd + 2));
    q->attn_cnt = c.counters(kAttnCounterBase);
    q->tickets = c.counters(kGemvTicketBase);
}
larosa_status validate_shard(const larosa_layer_weights* w, const larosa_shard* sh) {
    if (!w || !sh) return fail(LAROSA_EINVAL, "shard: NULL struct");
    const int64_t n = sh->world;
    if (n < 1 || sh->rank < 0 || sh->rank >= n) return fail(LAROSA_EINVAL, "shard: bad rank/world");
    if (sh->batch < 1) return fail(LAROSA_EINVAL, "shard: batch < 1");
    for (int j = 0; j < 4; ++j)
        if (w->w4_codes[j] || w->w4_scales[j]) return fail(LAROSA_EUNSUPPORTED, "shard: W4 sites are not sharded");
    if (sh->batch > LAROSA_MAX_BATCH) return fail(LAROSA_EUNSUPPORTED, "shard: batch > %d", LAROSA_MAX_BATCH);
    if (w->n_q_heads % n || w->n_kv_heads % n) return fail(LAROSA_EUNSUPPORTED, "shard: heads %% world != 0");
    if (w->d % (8 * n)) return fail(LAROSA_EUNSUPPORTED, "shard: d %% (8 world) != 0");
    if (w->inter % (LAROSA_GU_BLOCK * n)) return fail(LAROSA_EUNSUPPORTED, "shard: inter %% (64 world) != 0");
    if (w->head_dim != 64 && w->head_dim != 128) return fail(LAROSA_EUNSUPPORTED, "shard: head_dim must be 64 or 128");
    if (w->d > LAROSA_MAX_DIM || w->inter > LAROSA_MAX_DIM) return fail(LAROSA_EUNSUPPORTED, "shard: dims too large");
    if ((int64_t)sh->batch * (w->n_q_heads / n) > (int64_t)kAttnGroupCounterOff)
        return fail(LAROSA_EUNSUPPORTED, "shard: batch * Hq/n too large");
    return LAROSA_OK;
}
}  // namespace

extern "C" size_t larosa_shard_workspace_size(const larosa_layer_weights* w, const larosa_shard* shard,
                                              int64_t max_ctx) {
    if (validate_shard(w, shard) != LAROSA_OK || max_ctx <= 0) return 0;
    Carver c(nullptr);
    carve_shard(c, shard_dims(w, shard), max_ctx, nullptr);
    return c.size();
}

extern "C" larosa_status larosa_sparse_layer_shard_phase(const larosa_layer_weights* w, const larosa_layer_plan* plan,
                                                         const larosa_shard* sh, int32_t phase, const float* x,
                                                         const float* resid, float* out, uint16_t* k_cache,
                                                         uint16_t* v_cache, const int32_t* pos, int64_t max_ctx,
                                                         void* ws, size_t ws_bytes, larosa_stream_t stream) {
    LAROSA_TRY(validate_shard(w, sh));
    if (!plan || !x || !out) return fail(LAROSA_EINVAL, "shard_phase: NULL pointer");
    if (phase < 0 || phase > 4) return fail(LAROSA_EINVAL, "shard_phase: phase must be 0..4");
    if ((phase == 1 || phase == 3) && !resid) return fail(LAROSA_EINVAL, "shard_phase: phase %d needs resid", phase);
    if (phase == 0 && (!k_cache || !v_cache || !pos || max_ctx <= 0)) return fail(LAROSA_EINVAL, "shard_phase: KV state");
    const size_t need = larosa_shard_workspace_size(w, sh, max_ctx > 0 ? max_ctx : 1);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "shard_phase: workspace %zu < %zu", ws_bytes, need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const ShardDims S = shard_dims(w, sh);
    const int B = S.batch, bp = pad_batch(B);
    const bool fused = B == 1;
    Carver c(ws);
    ErrScope err_scope(c);
    ShardWs W;
    carve_shard(c, S, max_ctx > 0 ? max_ctx : 1, &W);
    const int r = sh->rank;
    if (w->adapter_mid) return fail(LAROSA_EUNSUPPORTED, "shard_phase: block-wise rotation (adapter_mid) not supported");
    const bool merged = w->adapter && w->adapter_in_down;   // 4 phases: the adapter rides with phase 3
    if (merged && phase == 4) return fail(LAROSA_EINVAL, "shard_phase: no phase 4 when adapter_in_down");
    // phase -> (site input width, k, RMS eps, weights, local output width)
    int64_t din = S.d, k = 0, dout = 0;
    float eps = -1.0f;
    const uint16_t* Wt = nullptr;
    switch (phase) {
        case 0: din = S.d; k = plan->k_h1; eps = w->rms_eps; Wt = w->w_qkv; dout = S.qkv_l; break;
        case 1: din = S.nq; k = plan->k_h2; Wt = w->w_o; dout = S.dl; break;
        case 2: din = S.d; k = plan->k_h3; eps = w->rms_eps; Wt = w->w_gu; dout = 2 * S.il; break;
        case 3: din = S.inter; k = plan->k_h4; Wt = w->w_down; dout = S.dl; break;
        default: din = S.d; Wt = w->adapter; dout = S.dl; break;
    }
    if (!Wt) return fail(LAROSA_EINVAL, "shard_phase: NULL weight for phase %d", phase);
    if (k < 0 || k > din) return fail(LAROSA_EINVAL, "shard_phase: k outside [0, D_in]");
    const void* ptrs[] = {x, resid, out, Wt, w->adapter, k_cache, v_cache};
    for (const void* q : ptrs)
        if (q && !aligned16(q)) return fail(LAROSA_EINVAL, "shard_phase: pointers must be 16-byte aligned");
    PeerOut peer;
    memset(&peer, 0, sizeof(peer));
    if (sh->peer_dst || sh->peer_flag) {
        if (!sh->peer_dst || !sh->peer_flag || sh->peer_ld <= 0)
            return fail(LAROSA_EINVAL, "shard_phase: peer_dst, peer_flag and peer_ld go together");
        peer.dst = reinterpret_cast<const unsigned long long*>(sh->peer_dst);
        peer.flag = reinterpret_cast<const unsigned long long*>(sh->peer_flag);
        peer.n = sh->world;
        peer.ld = (int)sh->peer_ld;
    }
    GemvArgs a = gemv_args_base();
    a.W = Wt;
    a.ld = dout;
    a.d_out = (int)dout;
    a.x = x;
    a.ldx = din;
    a.d_in = (int)din;
    a.batch = B;
    a.acc = W.acc;
    a.acc_ld = dout;
    GemvPlan p;
    bool dense2 = false;   // batch > 1, merged phase 3: a dense adapter GEMV into the same accumulators
    const bool img_path = !fused && use_tc_gemv(bp) && W.img;
    if (phase == 4) {
        a.mode = GEMV_DENSE;
        p = plan_gemv(dout, din, bp, GEMV_DENSE, din);
        if (img_path) {
            LAROSA_TRY(launch_dense_image(x, din, din, B, W.img, st));
            a.img = W.img;
        }
    } else if (fused) {
        // the gathered vector is identical on every rank -> identical selection data
        SiteSel sel = W.sel;
        if (eps < 0.f) sel.ssq = nullptr;
        LAROSA_TRY(cuda_check(launch(select_prep_kernel, dim3(n_slices_of(din)), dim3(kPrepThreads), 0, st, x, (int)din,
                                     sel, c.counters(kPrepBarrier), (float*)nullptr),
                              "select prep launch"));
        a.mode = GEMV_SELECT;
        a.sel = sel;
        a.sel_nssq = (int)((din + kSliceCols - 1) / kSliceCols);
        a.sel_k = (int)k;
        a.sel_eps = eps;
        p = plan_gemv(dout, k, 1, GEMV_SELECT, din);
        if (phase == 3 && merged) {   // + the dense r_mid rows of this rank's adapter columns
            a.W2 = w->adapter;
            a.x2 = resid;
            a.d2 = (int)S.d;
            p = plan_gemv_comp(dout, k, din, S.d);
        }
    } else {
        // batch > 1: every token's exact rule from the cluster Top-K kernel on the gathered input
        // (identical on every rank), then the union GEMV (THRESH; tcgen05 at batch >= 8)
        TopkKernelArgs tk = topk_args_base();   // every token's rule (the cluster Top-K kernel)
        tk.x = x;
        tk.ldx = din;
        tk.d = (int)din;
        tk.k = (int)k;
        tk.rms_eps = eps;
        tk.rule_out = W.thr;
        LAROSA_TRY(launch_topk(tk, B, st));
        if (img_path) {                          // and the token image from it
            const int groups = (int)((din + 7) / 8);
            LAROSA_TRY(cuda_check(launch(rule_apply_image_kernel, dim3((unsigned)((groups + 255) / 256), B), dim3(256), 0,
                                         st, x, din, (int)din, (const ThreshOut*)W.thr, W.img, (unsigned char*)nullptr),
                                  "rule_apply_image launch"));
        }
        a.mode = GEMV_THRESH;
        a.thr = W.thr;
        if (img_path) a.img = W.img;
        p = plan_gemv(dout, din, bp, GEMV_THRESH, din);
        dense2 = phase == 3 && merged;
    }
    if (phase != 0) {
        a.epi = phase == 2 ? EPI_SILU : ((phase == 4 || (phase == 3 && merged)) ? EPI_STORE : EPI_RESID);
        a.tickets = W.tickets;
        if (phase == 1 || (phase == 3 && !merged)) {
            a.res = resid + (size_t)r * S.dl;   // this rank's columns of r (phase 1) / r_mid (phase 3)
            a.res_ld = S.d;
        }
        a.out = out;
        a.out_ld = phase == 2 ? S.il : S.dl;
        if (!dense2) {
            a.peer = peer;
            return launch_gemv(a, p, fused ? 1 : bp, st);
        }
        // the sparse down columns leave their sums; the dense adapter GEMV (r_mid rows) finalises
        const int epi_mode = a.epi;
        a.epi = EPI_NONE;
        LAROSA_TRY(launch_gemv(a, p, bp, st));
        GemvArgs b2 = gemv_args_base();
        b2.W = w->adapter;
        b2.ld = dout;
        b2.d_out = (int)dout;
        b2.mode = GEMV_DENSE;
        b2.x = resid;
        b2.ldx = S.d;
        b2.d_in = (int)S.d;
        b2.batch = B;
        b2.acc = W.acc;
        b2.acc_ld = dout;
        b2.epi = epi_mode;
        b2.tickets = W.tickets;
        b2.out = out;
        b2.out_ld = S.dl;
        b2.peer = peer;
        if (img_path) {
            LAROSA_TRY(launch_dense_image(resid, S.d, S.d, B, W.img2, st));
            b2.img = W.img2;
        }
        return launch_gemv(b2, plan_gemv(dout, S.d, bp, GEMV_DENSE, S.d), bp, st);
    }
    // phase 0: QKV over the local heads (EPI_NONE) then attention writes the local h2
    LAROSA_TRY(launch_gemv(a, p, fused ? 1 : bp, st));
    AttnArgs aa;
    memset(&aa, 0, sizeof(aa));
    aa.acc = W.acc;
    aa.acc_ld = S.qkv_l;
    aa.bias = w->b_qkv;
    aa.theta = w->rope_theta;
    aa.kc = k_cache;
    aa.vc = v_cache;
    aa.pos = pos;
    aa.max_ctx = max_ctx;
    aa.hq = (int)S.hq_l;
    aa.hkv = (int)S.hkv_l;
    aa.hd = (int)S.hd;
    aa.chunk = attn_chunk(max_ctx, (int)(B * S.hq_l));
    aa.n_chunks = (int)((max_ctx + aa.chunk - 1) / aa.chunk);
    aa.part = W.attn_part;
    aa.counters = W.attn_cnt;
    aa.out = out;
    aa.peer = peer;
    return launch_attention(aa, (int)(B * S.hq_l), (int)S.hd, S.G, st);
}

extern "C" larosa_status larosa_shard_wait(const uint32_t* flag, uint32_t* expected, uint32_t count,
                                           larosa_stream_t stream) {
    if (!flag || !expected) return fail(LAROSA_EINVAL, "shard_wait: NULL pointer");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    return cuda_check(launch(peer_wait_kernel, dim3(1), dim3(32), 0, st, flag, expected, count), "shard_wait launch");
}

extern "C" larosa_status larosa_peer_push(const float* src, int32_t batch, int64_t d_local, int64_t src_ld,
                                          const uint64_t* peer_dst, const uint64_t* peer_flag, int32_t world,
                                          int64_t peer_ld, larosa_stream_t stream) {
    if (!src || !peer_dst || !peer_flag) return fail(LAROSA_EINVAL, "peer_push: NULL pointer");
    if (batch < 1 || d_local <= 0 || src_ld < d_local || world < 1 || peer_ld < d_local)
        return fail(LAROSA_EINVAL, "peer_push: bad sizes");
    if ((int64_t)batch * d_local > INT32_MAX) return fail(LAROSA_EUNSUPPORTED, "peer_push: too large");
    PeerOut peer;
    peer.dst = reinterpret_cast<const unsigned long long*>(peer_dst);
    peer.flag = reinterpret_cast<const unsigned long long*>(peer_flag);
    peer.n = world;
    peer.ld = (int)peer_ld;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t n = (int64_t)batch * d_local;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    return cuda_check(launch(peer_push_kernel, dim3(grid), dim3(256), 0, st, src, batch, (int)d_local, src_ld, peer),
                      "peer_push launch");
}

// gathered [world][batch][d_local] (rank-major all-gather) -> out [batch][world * d_local]
extern "C" larosa_status larosa_shard_gather_permute(const float* gathered, int32_t world, int32_t batch,
                                                     int64_t d_local, float* out, larosa_stream_t stream) {
    if (!gathered || !out) return fail(LAROSA_EINVAL, "shard_gather_permute: NULL pointer");
    if (world < 1 || batch < 1 || d_local <= 0) return fail(LAROSA_EINVAL, "shard_gather_permute: bad sizes");
    if ((const void*)gathered == (const void*)out) return fail(LAROSA_EINVAL, "shard_gather_permute: out aliases input");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t n = (int64_t)world * batch * d_local;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    return cuda_check(launch(gather_permute_kernel, dim3(grid), dim3(256), 0, st, gathered, world, batch, d_local, out),
                      "gather_permute launch");
}

extern "C" larosa_status larosa_argmax(const float* logits, int32_t batch, int64_t n, int64_t ld, int32_t* out,
                                       larosa_stream_t stream) {
    if (!logits || !out) return fail(LAROSA_EINVAL, "argmax: NULL pointer");
    if (batch < 1 || n <= 0 || ld < n) return fail(LAROSA_EINVAL, "argmax: bad sizes");
    if (n > INT32_MAX) return fail(LAROSA_EUNSUPPORTED, "argmax: n too large");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    return cuda_check(launch(argmax_kernel, dim3(batch), dim3(kRowThreads), 0, st, logits, ld, (int)n, out),
                      "argmax launch");
}



// ============================================================================== N1 calibration
extern "C" size_t larosa_calib_covariance_workspace_size(int64_t n_tok, int64_t d) {
    if (n_tok <= 0 || d <= 0) return 0;
    return (size_t)n_tok * d * 2 + 1024;   // X^T (bf16) for the tensor-core path
}

extern "C" larosa_status larosa_calib_covariance(const uint16_t* X, int64_t n_tok, int64_t d, float scale,
                                                 int32_t accumulate, float* C, void* ws, size_t ws_bytes,
                                                 larosa_stream_t stream) {
    if (!X || !C) return fail(LAROSA_EINVAL, "calib_covariance: NULL pointer");
    if (n_tok <= 0 || d <= 0) return fail(LAROSA_EINVAL, "calib_covariance: n_tok, d must be > 0");
    if (d > 65536 || n_tok > (1 << 30)) return fail(LAROSA_EUNSUPPORTED, "calib_covariance: too large");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const bool tc = d % kFoldBM == 0 && n_tok % kFoldBK == 0 && fold_bn(d) != 0 && aligned16(X) && aligned16(C) &&
                    env_int("LAROSA_FOLD_SIMT", 0) == 0;
    if (!tc) {
        const dim3 g((unsigned)((d + 31) / 32), (unsigned)((d + 31) / 32));
        covariance_simt_kernel<<<g, 256, 0, st>>>(X, (int)n_tok, (int)d, scale, accumulate, C);
        return cuda_check(cudaGetLastError(), "covariance kernel");
    }
    const size_t need = larosa_calib_covariance_workspace_size(n_tok, d);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "calib_covariance: workspace %zu < %zu", ws_bytes, need);
    // X^T [d][n] (K = tokens contiguous) serves as both K-major operands: C = Xt . Xt^T
    uint16_t* xt = static_cast<uint16_t*>(ws);
    const dim3 tb(32, 8);
    transpose_bf16_kernel<<<dim3((unsigned)((d + 31) / 32), (unsigned)((n_tok + 31) / 32)), tb, 0, st>>>(
        X, xt, (int)n_tok, (int)d);
    LAROSA_TRY(cuda_check(cudaGetLastError(), "transpose"));
    CUtensorMap a0, b0;
    const int bn = fold_bn(d);
    if (!make_kmajor_map(&a0, xt, d, n_tok, kFoldBM) || !make_kmajor_map(&b0, xt, d, n_tok, bn))
        return fail(LAROSA_ECUDA, "calib_covariance: tensor map");
    const cudaError_t e =
        bn == 256 ? launch_fold_tc<256, false, false, true>(a0, a0, b0, b0, C, (int)d, (int)d, (int)n_tok, st, scale,
                                                             accumulate)
                  : launch_fold_tc<128, false, false, true>(a0, a0, b0, b0, C, (int)d, (int)d, (int)n_tok, st, scale,
                                                             accumulate);
    return cuda_check(e, "covariance tcgen05 launch");
}

namespace {
std::mutex g_solver_mu;   // the Jacobi sweep graph is captured per call on a private stream
struct JacobiWs {
    double *A, *V, *part, *norms;
    int* pq;
    double2* cs;
    int* order;
};
constexpr int kJacobiNormCtas = 512;
void carve_jacobi(Carver& c, int64_t d, JacobiWs* o) {
    JacobiWs tmp;
    JacobiWs* q = o ? o : &tmp;
    const int64_t n = d + (d & 1);
    q->A = c.take<double>((size_t)n * n);
    q->V = c.take<double>((size_t)n * n);
    q->part = c.take<double>(2 * kJacobiNormCtas);
    q->norms = c.take<double>(2);
    q->pq = c.take<int>((size_t)n);
    q->cs = c.take<double2>((size_t)n / 2);
    q->order = c.take<int>((size_t)d);
}
}  // namespace

extern "C" size_t larosa_pca_rotation_workspace_size(int64_t d) {
    if (d <= 0 || d > 32768) return 0;
    Carver c(nullptr);
    carve_jacobi(c, d, nullptr);
    return c.size();
}

extern "C" larosa_status larosa_pca_rotation(const float* C, int64_t d, float* Q, float* lam, void* ws,
                                             size_t ws_bytes, larosa_stream_t stream) {
    if (!C || !Q || !lam) return fail(LAROSA_EINVAL, "pca_rotation: NULL pointer");
    if (d <= 0) return fail(LAROSA_EINVAL, "pca_rotation: d must be > 0");
    if (d > 32768) return fail(LAROSA_EUNSUPPORTED, "pca_rotation: d > 32768");
    const size_t need = larosa_pca_rotation_workspace_size(d);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "pca_rotation: workspace %zu < %zu", ws_bytes, need);
    std::lock_guard<std::mutex> lk(g_solver_mu);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Carver c(ws);
    ErrScope err_scope(c);
    JacobiWs J;
    carve_jacobi(c, d, &J);
    const int di = (int)d, n = di + (di & 1), npairs = n / 2;
    jacobi_init_kernel<<<1024, 256, 0, st>>>(C, J.A, J.V, di, n);
    LAROSA_TRY(cuda_check(cudaGetLastError(), "pca: init"));
    // one sweep (n - 1 rounds of disjoint rotations) as a CUDA graph on a private stream
    cudaStream_t ps;
    LAROSA_TRY(cuda_check(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking), "pca: stream"));
    cudaEvent_t ev;
    LAROSA_TRY(cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "pca: event"));
    LAROSA_TRY(cuda_check(cudaEventRecord(ev, st), "pca: event record"));
    LAROSA_TRY(cuda_check(cudaStreamWaitEvent(ps, ev, 0), "pca: stream wait"));
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    larosa_status status = LAROSA_OK;
    do {
        if (cudaStreamBeginCapture(ps, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            status = fail(LAROSA_ECUDA, "pca: begin capture");
            break;
        }
        const dim3 ga((unsigned)((npairs + 15) / 16), (unsigned)((npairs + 15) / 16));
        const unsigned gv = (unsigned)(((size_t)n * npairs + 255) / 256);
        for (int r = 0; r < n - 1; ++r) {
            jacobi_angles_kernel<<<(npairs + 127) / 128, 128, 0, ps>>>(J.A, n, r, J.pq, J.cs);
            jacobi_rotate_a_kernel<<<ga, 256, 0, ps>>>(J.A, n, npairs, J.pq, J.cs);
            jacobi_rotate_v_kernel<<<gv, 256, 0, ps>>>(J.V, n, npairs, J.pq, J.cs);
        }
        jacobi_norms_kernel<<<kJacobiNormCtas, 256, 0, ps>>>(J.A, n, J.part);
        jacobi_norms_final_kernel<<<1, 32, 0, ps>>>(J.part, kJacobiNormCtas, J.norms);
        if (cudaStreamEndCapture(ps, &graph) != cudaSuccess || !graph) {
            status = fail(LAROSA_ECUDA, "pca: end capture");
            break;
        }
        if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
            status = fail(LAROSA_ECUDA, "pca: graph instantiate");
            break;
        }
        // sweeps until off(A) <= 1e-12 ||A||_F (the oracle's criterion, Z8), at most 100
        bool done = false;
        for (int sweep = 0; sweep < 100 && status == LAROSA_OK; ++sweep) {
            double h[2];
            if (cudaGraphLaunch(exec, ps) != cudaSuccess ||
                cudaMemcpyAsync(h, J.norms, sizeof(h), cudaMemcpyDeviceToHost, ps) != cudaSuccess ||
                cudaStreamSynchronize(ps) != cudaSuccess) {
                status = fail(LAROSA_ECUDA, "pca: sweep");
                break;
            }
            if (std::sqrt(h[0]) <= 1e-12 * std::sqrt(h[1])) {
                done = true;
                break;
            }
        }
        if (status == LAROSA_OK && !done) status = fail(LAROSA_ECUDA, "pca: Jacobi did not converge in 100 sweeps");
        if (status != LAROSA_OK) break;
        eig_rank_kernel<<<(di + 255) / 256, 256, 0, ps>>>(J.A, di, n, J.order);
        pca_order_sign_kernel<<<(unsigned)di, 256, 0, ps>>>(J.V, J.A, J.order, di, n, Q, lam);
        if (cudaGetLastError() != cudaSuccess || cudaEventRecord(ev, ps) != cudaSuccess ||
            cudaStreamWaitEvent(st, ev, 0) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
            status = fail(LAROSA_ECUDA, "pca: order/sign");
    } while (false);
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    cudaEventDestroy(ev);
    cudaStreamDestroy(ps);
    return status;
}

// ============================================================================== N3 W4A16
static_assert(LAROSA_W4_GROUP == kW4Group, "W4 group size mismatch");
extern "C" larosa_status larosa_quantize_w4(const uint16_t* W, int64_t d_in, int64_t d_out, uint8_t* Wq, uint16_t* S,
                                            larosa_stream_t stream) {
    if (!W || !Wq || !S) return fail(LAROSA_EINVAL, "quantize_w4: NULL pointer");
    if (d_in <= 0 || d_out <= 0) return fail(LAROSA_EINVAL, "quantize_w4: d_in, d_out must be > 0");
    if (d_out % kSliceCols) return fail(LAROSA_EUNSUPPORTED, "quantize_w4: d_out %% 256 != 0");
    const int64_t units = d_in * (d_out / kW4Group);
    if (units > (int64_t)1 << 30) return fail(LAROSA_EUNSUPPORTED, "quantize_w4: too large");
    const unsigned blocks = (unsigned)((units + 7) / 8);
    quantize_w4_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(W, (int)d_in, (int)d_out, Wq, S);
    return cuda_check(cudaGetLastError(), "quantize_w4 launch");
}

extern "C" size_t larosa_topk_sparse_gemv_w4_workspace_size(int64_t d_in, int64_t d_out) {
    return larosa_topk_sparse_gemv_workspace_size(d_in, d_out);
}

extern "C" larosa_status larosa_topk_sparse_gemv_w4(const float* x, int64_t d_in, int64_t k, float rms_eps,
                                                    const uint8_t* Wq, const uint16_t* S, int64_t d_out, float* y,
                                                    int32_t prepared, void* ws, size_t ws_bytes,
                                                    larosa_stream_t stream) {
    if (!x || !Wq || !S || !y) return fail(LAROSA_EINVAL, "topk_sparse_gemv_w4: NULL pointer");
    if (d_in <= 0 || d_out <= 0) return fail(LAROSA_EINVAL, "topk_sparse_gemv_w4: d_in, d_out must be > 0");
    if (k < 0 || k > d_in) return fail(LAROSA_EINVAL, "topk_sparse_gemv_w4: k outside [0, d_in]");
    if (d_in > LAROSA_MAX_DIM || d_in % 8) return fail(LAROSA_EUNSUPPORTED, "topk_sparse_gemv_w4: d_in");
    if (d_out % kSliceCols || d_out > (int64_t)65536)
        return fail(LAROSA_EUNSUPPORTED, "topk_sparse_gemv_w4: d_out must be a multiple of 256 (<= 65536)");
    if (!aligned16(Wq) || !aligned16(x) || !aligned16(y) || (reinterpret_cast<uintptr_t>(S) & 3))
        return fail(LAROSA_EINVAL, "topk_sparse_gemv_w4: alignment (Wq, x, y 16 B; S 4 B)");
    const size_t need = larosa_topk_sparse_gemv_workspace_size(d_in, d_out);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "topk_sparse_gemv_w4: workspace %zu < %zu", ws_bytes, need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Carver c(ws);
    ErrScope err_scope(c);
    unsigned long long* acc;
    SiteSel sel;
    carve_topk_gemv(c, d_in, d_out, &acc, &sel);
    if (rms_eps < 0.f) sel.ssq = nullptr;
    if (!prepared)
        LAROSA_TRY(cuda_check(launch(select_prep_kernel, dim3(n_slices_of(d_in)), dim3(kPrepThreads), 0, st, x, (int)d_in,
                                     sel, c.counters(kPrepBarrier), (float*)nullptr),
                              "select prep launch"));
    GemvArgs a = gemv_args_base();
    a.ld = d_out;
    a.d_out = (int)d_out;
    a.mode = GEMV_SELECT;
    a.x = x;
    a.ldx = d_in;
    a.d_in = (int)d_in;
    a.sel = sel;
    a.sel_nssq = (int)((d_in + kSliceCols - 1) / kSliceCols);
    a.sel_k = (int)k;
    a.sel_eps = rms_eps;
    a.batch = 1;
    a.acc = acc;
    a.acc_ld = d_out;
    a.epi = EPI_STORE;
    a.tickets = c.counters(kGemvTicketBase);
    a.out = y;
    a.out_ld = d_out;
    return launch_gemv_w4(a, Wq, S, st);
}

// ============================================================================== N2 prefill
namespace {
struct PrefillWs {
    uint16_t *xh, *xl;
    uint8_t* anyk;
    int64_t n_pad;
};
void carve_prefill(Carver& c, int64_t n_tok, int64_t d_in, int split, PrefillWs* o) {
    PrefillWs tmp;
    PrefillWs* q = o ? o : &tmp;
    q->n_pad = (n_tok + kPfTok - 1) / kPfTok * kPfTok;
    q->xh = c.take<uint16_t>((size_t)n_tok * d_in);
    q->xl = split ? c.take<uint16_t>((size_t)n_tok * d_in) : nullptr;
    q->anyk = c.take<uint8_t>((size_t)((d_in + kPfK - 1) / kPfK) * q->n_pad);
}
}  // namespace

extern "C" size_t larosa_prefill_sparse_gemm_workspace_size(int64_t n_tok, int64_t d_in, int32_t split) {
    if (n_tok <= 0 || d_in <= 0) return 0;
    Carver c(nullptr);
    carve_prefill(c, n_tok, d_in, split, nullptr);
    return c.size();
}

extern "C" larosa_status larosa_prefill_sparse_gemm(const float* X, int64_t n_tok, int64_t d_in, int64_t k,
                                                    float rms_eps, const uint16_t* W, int64_t d_out, float* Y,
                                                    int32_t split, void* ws, size_t ws_bytes, larosa_stream_t stream) {
    if (!X || !W || !Y) return fail(LAROSA_EINVAL, "prefill_sparse_gemm: NULL pointer");
    if (n_tok <= 0 || d_in <= 0 || d_out <= 0) return fail(LAROSA_EINVAL, "prefill_sparse_gemm: sizes must be > 0");
    if (k < 0 || k > d_in) return fail(LAROSA_EINVAL, "prefill_sparse_gemm: k outside [0, d_in]");
    if (d_in > LAROSA_MAX_DIM) return fail(LAROSA_EUNSUPPORTED, "prefill_sparse_gemm: d_in > %d", LAROSA_MAX_DIM);
    if (d_in % 8 || d_out % 8) return fail(LAROSA_EUNSUPPORTED, "prefill_sparse_gemm: d_in and d_out must be multiples of 8");
    if (n_tok > 65535 * (int64_t)kPfTok || d_out > (int64_t)65535 * kPfCols)
        return fail(LAROSA_EUNSUPPORTED, "prefill_sparse_gemm: too large");
    if (!aligned16(W)) return fail(LAROSA_EINVAL, "prefill_sparse_gemm: W must be 16-byte aligned");
    const size_t need = larosa_prefill_sparse_gemm_workspace_size(n_tok, d_in, split);
    if (!ws || ws_bytes < need) return fail(LAROSA_EWORKSPACE, "prefill_sparse_gemm: workspace %zu < %zu", ws_bytes, need);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Carver c(ws);
    ErrScope err_scope(c);
    PrefillWs P;
    carve_prefill(c, n_tok, d_in, split, &P);
    // every token's exact Top-K (Z10) + RMS scale -> masked bf16 rows and per-block "any kept"
    const size_t rsmem = (size_t)d_in * 4 + 128;
    LAROSA_TRY(cuda_check(allow_smem(prefill_rule_mask_kernel, rsmem), "cudaFuncSetAttribute(prefill rule)"));
    LAROSA_TRY(cuda_check(launch(prefill_rule_mask_kernel, dim3((unsigned)n_tok), dim3(kPfThreads), rsmem, st, X,
                                 (int)n_tok, (int)d_in, (int)k, rms_eps, P.xh, P.xl, P.anyk, (int)P.n_pad),
                          "prefill rule launch"));
    CUtensorMap tw, txh, txl;
    if (!make_w_mn_map(&tw, W, d_in, d_out, d_out) || !make_kmajor_map(&txh, P.xh, n_tok, d_in, kPfTok) ||
        (split && !make_kmajor_map(&txl, P.xl, n_tok, d_in, kPfTok)))
        return fail(LAROSA_ECUDA, "prefill_sparse_gemm: tensor map");
    if (!split) txl = txh;
    const dim3 grid((unsigned)((d_out + kPfCols - 1) / kPfCols), (unsigned)((n_tok + kPfTok - 1) / kPfTok));
    if (split) {
        LAROSA_TRY(cuda_check(allow_smem(prefill_tc_kernel<true>, pf_smem_bytes(true)), "cudaFuncSetAttribute(prefill)"));
        return cuda_check(launch(prefill_tc_kernel<true>, grid, dim3(kPfGemmThreads), pf_smem_bytes(true), st, tw, txh,
                                 txl, (const uint8_t*)P.anyk, (int)P.n_pad, (int)n_tok, (int)d_in, (int)d_out, Y),
                          "prefill gemm launch");
    }
    LAROSA_TRY(cuda_check(allow_smem(prefill_tc_kernel<false>, pf_smem_bytes(false)), "cudaFuncSetAttribute(prefill)"));
    return cuda_check(launch(prefill_tc_kernel<false>, grid, dim3(kPfGemmThreads), pf_smem_bytes(false), st, tw, txh,
                             txl, (const uint8_t*)P.anyk, (int)P.n_pad, (int)n_tok, (int)d_in, (int)d_out, Y),
                      "prefill gemm launch");
}
