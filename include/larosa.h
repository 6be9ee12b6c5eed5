/* larosa.h — C ABI of the LaRoSA decode hot path on B200 (sm_100a).
 *
 * LaRoSA (arXiv 2507.01299, "Layerwise Rotated Sparse Activation"); PAPER.md line
 * numbers are cited as P:n.  The method: each token's hidden vector x is rotated by
 * a layerwise orthogonal Q_l, Top-K magnitude-sparsified with
 * k = alpha (1 - p) D_in (eq. 2), and the kept entries drive a GEMV over the
 * folded weights (W Q)^T that streams only the kept weight columns.
 *
 * Conventions:
 *  - Every weight is stored as Wc = W_pt^T, row-major [d_in][ld] bf16 (raw uint16
 *    bits), i.e. the paper's "column-major W" (P:414 (1)): kept input channel j is
 *    the contiguous row Wc[j][0 .. d_out).  A projection is y = x . Wc.
 *  - All pointers are DEVICE pointers unless marked (host).  All calls are
 *    asynchronous on `stream` and CUDA-graph capturable: no allocation, no host sync,
 *    no device-wide memset.  The caller owns every buffer.
 *  - Workspaces: sized by the matching *_workspace_size() query, 256-byte aligned,
 *    and ZERO-FILLED ONCE by the caller when allocated.  They hold the GEMVs' 64-bit
 *    fixed-point accumulators and tickets, which every call restores to zero, so a
 *    workspace must be reused only for calls of the same kind and shapes (or be zeroed
 *    again), and not by two calls that can run concurrently.
 *  - Errors: arguments are validated synchronously and a status is returned; no
 *    exception crosses the ABI.  Launch errors return LAROSA_ECUDA (from
 *    cudaGetLastError).  Faults inside kernels surface at the caller's next sync.
 *    larosa_last_error() gives a thread-local message for the last non-OK status.
 *  - Preconditions not checked on the hot path: inputs finite,
 *    per-token index lists ascending and unique.
 *  - Determinism: every reduction runs in a fixed order (no floating-point atomics),
 *    so results are bit-reproducible for a given shape and batch.
 *  - Re-entrant; concurrent calls on different streams with different workspaces
 *    are allowed.
 */
#ifndef LAROSA_H
#define LAROSA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LAROSA_ABI_VERSION 7
#define LAROSA_MAX_BATCH 16          /* decode batch 1..16 (BASELINE.json north_star) */
#define LAROSA_MAX_DIM 32768         /* largest D_in of any site (Qwen2.5-72B I = 29568) */
#define LAROSA_GU_BLOCK 64           /* gate|up interleave block, see larosa_pack_gate_up */

typedef struct CUstream_st* larosa_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    LAROSA_OK = 0,
    LAROSA_EINVAL = 1,       /* null pointer, k > d, d <= 0, batch < 1, misaligned pointer   */
    LAROSA_ESHAPE = 2,       /* inconsistent dimensions between arguments                     */
    LAROSA_EUNSUPPORTED = 3, /* e.g. ld % 8 != 0 or d_out % 8 != 0 (16-byte rows), batch > 16 */
    LAROSA_ECUDA = 4,        /* a CUDA runtime call or kernel launch failed                   */
    LAROSA_ENCCL = 5,        /* reserved for collective errors (collectives are the caller's) */
    LAROSA_EWORKSPACE = 6    /* workspace pointer NULL or smaller than the size query         */
} larosa_status;

int larosa_abi_version(void);

/* Device-side error bits of a workspace (every call that carves a workspace records here):
 *   LAROSA_ERR_KEEP_ALL      a SELECT GEMV found its site histogram inconsistent and used the
 *                            keep-all rule (sparse -> dense; never expected: a bug indicator);
 *   LAROSA_ERR_FIX_OVERFLOW  a GEMV column could leave the +-2^31 range of the 64-bit fixed point
 *                            (32 fraction bits) of the deterministic split-K reduction: one of its
 *                            n partials had |s| >= 2^31 / n (sufficient for no overflow otherwise).
 * Reads the word into *flags (host), optionally clears it; synchronises the stream.  The
 * workspace header's last counter word holds it (zero at rest like the others). */
#define LAROSA_ERR_KEEP_ALL 1u
#define LAROSA_ERR_FIX_OVERFLOW 2u
larosa_status larosa_error_flags(void* ws, int32_t clear, uint32_t* flags /* host */, larosa_stream_t stream);
const char* larosa_status_string(int status);
/* Thread-local detail of the last non-OK status returned on this thread. */
const char* larosa_last_error(void);

/* ------------------------------------------------------------------------------
 * Kept count (host, fp64).  k = alpha (1 - p) D_in.
 * Rounded half away from zero and clamped to [0, d_in]; p == 0 is
 * the dense "0%" configuration, k = d_in (Z16).  EINVAL if k_out is NULL, d_in <= 0,
 * p outside [0, 1] or alpha < 0.
 * ------------------------------------------------------------------------------ */
larosa_status larosa_compute_k(double alpha, double p, int64_t d_in, int64_t* k_out /* host */);

/* Sparsity-coefficient constraints (App. B):
 *   alpha2 = 4 - 3 alpha1,  alpha4 = (2 + M - 2 alpha3) / M.
 * EINVAL if m <= 0, a pointer is NULL or a resulting coefficient is <= 0. */
larosa_status larosa_solve_alpha(double alpha1, double alpha3, double m,
                                 double* alpha2 /* host */, double* alpha4 /* host */);

/* ------------------------------------------------------------------------------
 * Offline fold (eq. before_merge -> after_merge; §3.2).
 *  side = LAROSA_LEFT_QT : Wout = Q^T diag(gamma) W.  W [rows = d][cols = d_out],
 *      Q [d][d] fp32 row-major (Q[:, i] = i-th principal direction),
 *      gamma [d] fp32 or NULL (RMSNorm gain folded into W's input rows).
 *      Used for W_qkv (h1) and W_gate|up (h3).
 *  side = LAROSA_RIGHT_Q : Wout = W Q.  W [rows = d_in][cols = d], Q [d][d]; gamma
 *      must be NULL.  Used for W_o and W_down so the block output stays in Q_l's
 *      basis (Z21).
 *  (The residual adapter A_l = Q_l^T Q_{l+1}, has its own call below that keeps
 *  both fp32 factors split: larosa_residual_adapter.)
 *  W, Wout bf16 row-major with leading dimension `cols`; Wout must not alias W.
 *  Arithmetic: Q (times gamma) is split into bf16 hi + lo parts, the products run on
 *  the tcgen05 tensor cores with fp32 accumulation in TMEM, and Wout is rounded to
 *  bf16 (RNE) once.  rows, cols must be multiples of 64 (EUNSUPPORTED otherwise).
 * ------------------------------------------------------------------------------ */
enum { LAROSA_LEFT_QT = 0, LAROSA_RIGHT_Q = 1 };
size_t larosa_fold_workspace_size(int64_t rows, int64_t cols, int side);
larosa_status larosa_fold_rotation(const float* Q, const float* gamma, const uint16_t* W,
                                   uint16_t* Wout, int64_t rows, int64_t cols, int side,
                                   void* ws, size_t ws_bytes, larosa_stream_t stream);

/* ------------------------------------------------------------------------------
 * Residual adapter A_l = Q_l^T Q_{l+1}   ("residual adapters").
 *  Q_l, Q_next: fp32 [d][d] row-major (device); A: bf16 [d][d] row-major (device,
 *  caller-owned, must not alias either factor).  BOTH factors are split into bf16
 *  hi + lo parts and the three significant products (hi.hi + lo.hi + hi.lo) run on
 *  the tcgen05 tensor cores into one fp32 TMEM accumulator; A is rounded to bf16 (RNE)
 *  ONCE -- unlike the LEFT_QT fold of a bf16-rounded Q_{l+1}, which rounds twice.
 *  d < 128 or d % 128 != 0 uses an fp32 CUDA-core kernel (same single rounding).
 *  d must be a multiple of 64 (EUNSUPPORTED).  Workspace: larosa_residual_adapter_
 *  workspace_size(d) bytes (scratch; no zero-fill needed).
 * ------------------------------------------------------------------------------ */
size_t larosa_residual_adapter_workspace_size(int64_t d);
larosa_status larosa_residual_adapter(const float* Q_l, const float* Q_next, uint16_t* A, int64_t d,
                                      void* ws, size_t ws_bytes, larosa_stream_t stream);

/* Pack separate gate and up weights Wg, Wu [d][inter] into the fused layout the layer
 * uses: Wgu [d][2*inter] with column block t of width 2*LAROSA_GU_BLOCK holding
 * gate columns [t*B, t*B+B) followed by up columns [t*B, t*B+B) (B = LAROSA_GU_BLOCK),
 * so one GEMV tile owns matching gate/up pairs for the SiLU(g)*u epilogue.
 * inter must be a multiple of LAROSA_GU_BLOCK.  Works equally before or after the
 * (left) fold, which acts on rows. */
larosa_status larosa_pack_gate_up(const uint16_t* Wg, const uint16_t* Wu, uint16_t* Wgu,
                                  int64_t d, int64_t inter, larosa_stream_t stream);

/* ------------------------------------------------------------------------------
 * Rotate + Top-K  (RMS scale P:1444-1447).
 * Per token b in [0, batch):
 *   xr = x[b] . R            (R bf16 [d][d]; R == NULL -> identity, Top-K only:
 *                             the h2/h4 sites use Q = I)
 *   S  = the k largest |xr_i|; ties -> the lower index wins; exactly k
 *        indices even if some values are 0 (Z11); idx[b][0..k) ascending.
 *   vals[b][t] = xr[idx[b][t]] * s,  s = 1/sqrt(mean(xr^2) + rms_eps) if rms_eps >= 0
 *        (RMSNorm with gains folded into the next weights: h1, h3), else s = 1.
 *   Selection is taken on the unscaled xr (s > 0 cannot reorder).
 * x fp32 [batch][d]; xr_out fp32 [batch][d] or NULL; idx int32 [batch][k];
 * vals fp32 [batch][k]; mask uint32 [batch][ceil(d/32)] or NULL (bit i%32 of word
 * i/32 set iff i kept).  xr_out may alias x only when R == NULL.
 * Rotation: fp32 accumulation of bf16 R products in a fixed order.  Top-K: exact
 * radix select on the uint32 keys bits(|xr|) (monotone for finite values).
 * ------------------------------------------------------------------------------ */
size_t larosa_rotate_topk_workspace_size(int32_t batch, int64_t d);
larosa_status larosa_rotate_topk(const float* x, const uint16_t* R, int32_t batch, int64_t d,
                                 int64_t k, float rms_eps, float* xr_out, int32_t* idx,
                                 float* vals, uint32_t* mask, void* ws, size_t ws_bytes,
                                 larosa_stream_t stream);

/* ------------------------------------------------------------------------------
 * Sparse GEMV over kept columns (eq. after_merge; kernel recipe P:414).
 *   y[b][o] = (bias ? bias[o] : 0) + sum_{t<k} vals[b][t] * W[idx[b][t]][o],
 *   o in [0, d_out), b in [0, batch).
 * W bf16 [d_in][ld]; idx int32 [batch][k] (ascending, unique, < d_in);
 * vals fp32 [batch][k]; bias bf16 [d_out] or NULL; y fp32 [batch][d_out].
 * batch > 1 streams the union U of the tokens' kept rows exactly once; a token
 * contributes 0 on rows it did not keep (per-token results stay exact).
 * Bytes moved ~ |U| * d_out * 2.  Requires ld % 8 == 0, d_out % 8 == 0 and a
 * 16-byte aligned W (EUNSUPPORTED / EINVAL otherwise).  k == 0 gives y = bias.
 * ------------------------------------------------------------------------------ */
size_t larosa_sparse_gemv_workspace_size(int32_t batch, int64_t d_in, int64_t k, int64_t d_out);
larosa_status larosa_sparse_gemv(const uint16_t* W, int64_t d_in, int64_t d_out, int64_t ld,
                                 const int32_t* idx, const float* vals, int32_t batch, int64_t k,
                                 const uint16_t* bias, float* y, void* ws, size_t ws_bytes,
                                 larosa_stream_t stream);

/* ------------------------------------------------------------------------------
 * Fused Top-K + sparse GEMV, batch 1 (P:414 (2): sparsification fused into the GEMV;
 * SPEC fused_topk_gemv S:397-405):
 *   S = Top-K of |x| (k largest, ties -> lower index), s as in rotate_topk,
 *   y[o] = (bias ? bias[o] : 0) + sum_{j in S} x[j] * s * W[j][o].
 * No index list is materialised: a preparation kernel builds the 4096-bin histogram of
 * the keys' top 12 bits (and the RMS partials), then every CTA of the GEMV derives the
 * exact selection rule itself and streams an exactly balanced share of the kept rows.
 * x fp32 [d_in] (d_in % 4 == 0, 16-byte aligned); W bf16 [d_in][ld]; y fp32 [d_out].
 * Same W / ld / d_out / alignment requirements as larosa_sparse_gemv.
 * ------------------------------------------------------------------------------ */
size_t larosa_topk_sparse_gemv_workspace_size(int64_t d_in, int64_t d_out);
/* prepared != 0: the workspace already holds x's selection data from an earlier call with
 * the same x and rms_eps sign (then only the GEMV kernel is launched). */
larosa_status larosa_topk_sparse_gemv(const float* x, int64_t d_in, int64_t k, float rms_eps,
                                      const uint16_t* W, int64_t d_out, int64_t ld,
                                      const uint16_t* bias, float* y, int32_t prepared, void* ws,
                                      size_t ws_bytes, larosa_stream_t stream);

/* Fused Top-K + sparse GEMV plus a dense second operand into the same outputs (batch 1):
 *   y[o] = sum_{j in S} x[j] s W[j][o] + sum_{m < d2} x2[m] W2[m][o],
 * S and s as in larosa_topk_sparse_gemv.  This is the down site with the residual adapter
 * folded beside it (larosa_layer_weights.adapter_in_down: x = h4, W = Wd Q_{l+1}, x2 = r_mid,
 * W2 = A_l; P:388 by linearity).  The dense rows stream in CTAs of the same launch that need
 * no selection rule.  W2 bf16 [d2][ld] (16-byte aligned), x2 fp32 [d2], 1 <= d2 <= 32768;
 * the other arguments and the workspace are those of larosa_topk_sparse_gemv. */
larosa_status larosa_topk_sparse_gemv_dense2(const float* x, int64_t d_in, int64_t k, float rms_eps,
                                             const uint16_t* W, int64_t d_out, int64_t ld, const float* x2,
                                             const uint16_t* W2, int64_t d2, float* y, int32_t prepared,
                                             void* ws, size_t ws_bytes, larosa_stream_t stream);

/* Introspection (host): the launch plan larosa_sparse_gemv uses for this shape.
 * info (host, 8 ints) = {columns per CTA, column slices, kept-row splits, warps per CTA,
 * cp.async ring stages per warp, rows per stage, dynamic smem bytes, CTAs}. */
larosa_status larosa_gemv_plan_info(int64_t d_out, int64_t nrows_max, int32_t batch, int32_t* info);

/* ------------------------------------------------------------------------------
 * Decode-step ends (Q_0 is merged into the embedding, Q_L into
 * the head; the head is dense, the paper does not sparsify it).
 * larosa_embed: resid[b][:] = E'[tokens[b]][:] as fp32, E' = E Q_0 bf16 [vocab][d];
 *   tokens int32 [batch] in [0, vocab) (not checked on device).
 * larosa_lm_head: logits[b] = (r_b s_b) H' with s_b = 1/sqrt(mean(r_b^2) + rms_eps) (final
 *   RMSNorm; its gain is folded into H' = Q_L^T diag(gamma_f) H, LEFT fold), dense GEMV over
 *   H' bf16 [d][vocab] (fixed-point accumulation, fp32 out); next_token[b] = arg-max of
 *   logits[b], the lowest index on exact ties.  logits may be NULL (workspace scratch).
 *   vocab % 8 == 0, d % 8 == 0, batch <= 16.
 * ------------------------------------------------------------------------------ */
larosa_status larosa_embed(const uint16_t* E, int64_t vocab, int64_t d, const int32_t* tokens, int32_t batch,
                           float* resid, larosa_stream_t stream);
size_t larosa_lm_head_workspace_size(int32_t batch, int64_t d, int64_t vocab);
larosa_status larosa_lm_head(const float* resid, int32_t batch, int64_t d, const uint16_t* H, int64_t vocab,
                             float rms_eps, float* logits, int32_t* next_token, void* ws, size_t ws_bytes,
                             larosa_stream_t stream);

/* ------------------------------------------------------------------------------
 * One LaRoSA decoder layer on pre-folded weights (Fig. 2; §8(a) a6):
 *   r (residual, Q_l basis) -> h1: Top-K k_h1 of r, RMS scale -> sparse GEMV W_qkv
 *   (+bias, RoPE, append k/v at pos) -> GQA decode attention -> h2: Top-K k_h2 ->
 *   sparse GEMV W_o, r += -> h3: Top-K k_h3 of r, RMS scale -> sparse GEMV W_gate|up,
 *   h4 = SiLU(g) * u -> Top-K k_h4 -> sparse GEMV W_down, r += ->
 *   r <- r . A_l (dense adapter GEMV) unless adapter == NULL
 *   (adapter_in_down: r <- r_mid A_l + y_down in the down launch, see below).
 * Weights (all bf16, Wc layout):
 *   w_qkv [d][(Hq + 2 Hkv) hd] = Q_l^T diag(gamma_attn) [Wq | Wk | Wv]
 *   b_qkv [(Hq + 2 Hkv) hd] or NULL (Qwen2.5; unchanged by an input-side fold, Z28)
 *   w_o [Hq hd][d] = Wo Q_l;  w_gu [d][2 inter] = packed Q_l^T diag(gamma_mlp) [Wg | Wu]
 *   w_down [inter][d] = Wd Q_l (Wd Q_{l+1} if adapter_in_down);
 *   adapter [d][d] = Q_l^T Q_{l+1} or NULL.
 * Glue (not paper content): RoPE = HF rotate_half with pairs (i, i+hd/2),
 * inv_freq = theta^(-2i/hd), angle = pos * inv_freq; q-head h reads kv-head
 * floor(h Hkv / Hq); softmax scale 1/sqrt(hd) in fp32; KV cache bf16.
 * State: resid fp32 [batch][d] in/out; k_cache, v_cache bf16 [batch][Hkv][max_ctx][hd];
 * pos int32 [batch] (device): token b is written at position pos[b] and attends to
 * [0, pos[b]]; requires pos[b] < max_ctx (not checked on device).
 * Constraints: hd == 128 or 64 (hd % 16 == 0), Hq % Hkv == 0, d % 8 == 0,
 * inter % LAROSA_GU_BLOCK == 0, Hq*hd and (Hq+2Hkv)*hd multiples of 8.
 * Taps (optional, may be NULL; each member may be NULL): device buffers that receive
 * the intermediates for parity checks.  Sharded use: pass this rank's
 * output rows; collectives are issued by the caller between layers.
 * ------------------------------------------------------------------------------ */
typedef struct {
    const uint16_t* w_qkv;
    const uint16_t* b_qkv;
    const uint16_t* w_o;
    const uint16_t* w_gu;
    const uint16_t* w_down;
    const uint16_t* adapter;
    int64_t d, inter, n_q_heads, n_kv_heads, head_dim;
    float rope_theta, rms_eps;
    /* Nonzero: the adapter is folded into the down projection's output side,
     * w_down [inter][d] = Wd Q_{l+1} (= (Wd Q_l) A_l; SURVEY §8(e) "4-gather form"), and the
     * layer computes r_next = r_mid A_l + Top-K(h4) w_down (equal to the literal
     * (r_mid + y_down) A_l of P:388 by linearity).  Requires adapter != NULL.  At batch 1 the
     * dense r_mid rows of A_l stream in the same launch as the down site's kept rows (their
     * CTAs need no selection rule and prefetch before the dependency wait); the r_out tap is
     * not written.  0: the literal form (down folded with Q_l, separate adapter GEMV). */
    int32_t adapter_in_down;
    /* Block-wise rotation Q_B (Table 6): [d][d] = Q_a^T Q_m or NULL.  When set, the
     * attention block runs in Q_a's basis and the MLP block in Q_m's: w_o = Wo Q_m (output side),
     * w_gu folded with Q_m (input side), and r_mid = r A_mid + Top-K(h2) w_o (the dense r rows of
     * A_mid ride in the O launch like the adapter beside down); adapter / w_down then close from
     * Q_m's basis (adapter = Q_m^T Q_a', or w_down = Wd Q_a' with adapter_in_down).  NULL: Q_L
     * (one rotation per layer).  Not supported by larosa_sparse_layer_shard_phase. */
    const uint16_t* adapter_mid;
    /* W4A16 sites (ABI 6): for site s (0 QKV, 1 O, 2 gate|up, 3 down) either NULL
     * (the bf16 w_* above) or the int4 codes [d_in][d_out/2] and fp16 group scales
     * [d_in][d_out/128] of larosa_quantize_w4 of that (folded) weight; the site then streams the
     * codes with the same fused Top-K prologue and epilogue (batch 1 only, EUNSUPPORTED otherwise;
     * with adapter_in_down the adapter rows stream as bf16 companion CTAs of the W4 down launch). */
    const uint8_t* w4_codes[4];
    const uint16_t* w4_scales[4];
} larosa_layer_weights;

typedef struct {
    int64_t k_h1, k_h2, k_h3, k_h4;
    int64_t k_next_h1;   /* reserved (0) */
} larosa_layer_plan;

typedef struct {
    float* resid;
    uint16_t* k_cache;
    uint16_t* v_cache;
    const int32_t* pos;
    int64_t max_ctx;
    int32_t batch;
    /* Batch 1 only: nonzero iff `resid` is exactly what the previous larosa_sparse_layer
     * call on this same workspace wrote (the next layer of a decode step), untouched since.
     * That call's last epilogue already produced the h1 key histogram and RMS partials of
     * resid, so the preparation kernel is skipped.  0 is always correct. */
    int32_t chained;
    /* Batch 1, optional (NULL = unused): pinned, device-mapped host buffers of d floats.
     * host_in (only when chained == 0): the step's input residual is read from it by the
     * preparation kernel, which also writes resid -- the host-to-device transfer happens inside
     * the layer's first kernel.  host_out: the layer's last epilogue also writes r_next there
     * (device-to-host inside the kernel; complete when the stream reaches the layer's end). */
    const float* host_in;
    float* host_out;
} larosa_layer_state;

typedef struct {
    int32_t* idx_h1; float* vals_h1;   /* [batch][k_h1] */
    float* q;                          /* [batch][Hq hd] after bias + RoPE            */
    float* h2;                         /* [batch][Hq hd] attention output             */
    int32_t* idx_h2; float* vals_h2;   /* [batch][k_h2]                               */
    float* r_mid;                      /* [batch][d] residual after the O projection  */
    int32_t* idx_h3; float* vals_h3;   /* [batch][k_h3]                               */
    float* h4;                         /* [batch][inter] SiLU(g) * u                  */
    int32_t* idx_h4; float* vals_h4;   /* [batch][k_h4]                               */
    float* r_out;                      /* [batch][d] residual before the adapter      */
} larosa_layer_taps;

size_t larosa_layer_workspace_size(const larosa_layer_weights* w, int32_t batch, int64_t max_ctx);

/* Profiling aid (not for production): bitmask of the kernels larosa_sparse_layer launches
 * (default -1 = all; results are meaningless otherwise).  Bits: 0 h1 preparation (batch 1)
 * or Top-K h1 (batch > 1), 1 QKV GEMV, 2 attention, 3 Top-K h2 (batch > 1), 4 O GEMV,
 * 5 Top-K h3 (batch > 1), 6 gate|up GEMV, 7 Top-K h4 (batch > 1), 8 down GEMV, 9 adapter
 * GEMV.  Process-wide, not thread-safe.  Also settable through the LAROSA_LAYER_PHASES
 * environment variable. */
#define LAROSA_PHASES_GEMV_ONLY 0x352
void larosa_debug_set_layer_phases(int mask);
/* Profiling aid: device buffer of n_slots x 1024 x 16 uint64 %globaltimer stamps (ns), one
 * block per kernel of a batch-1 larosa_sparse_layer call (0 QKV, 1 attention, 2 O, 3 gate|up,
 * 4 down, 5 adapter), one row per CTA (linear id < 1024): [0] entry, [1] after the dependency
 * wait, [2] after the prologue, [3] after the main loop, [4] exit.  NULL disables.
 * Process-wide, not thread-safe. */
void larosa_debug_set_timeline(void* dev_buf, int n_slots);
larosa_status larosa_sparse_layer(const larosa_layer_weights* w, const larosa_layer_plan* plan,
                                  const larosa_layer_state* state, const larosa_layer_taps* taps,
                                  void* ws, size_t ws_bytes, larosa_stream_t stream);

/* ------------------------------------------------------------------------------
 * Row-sharded layer for multi-GPU decode (batch 1..16).  Every rank holds the
 * output columns ("rows" of nn.Linear) of each projection and the replicated residual:
 *   w_qkv  [d][(Hq/n + 2 Hkv/n) hd]   this rank's q heads [r Hq/n, ..) | k heads | v heads
 *   b_qkv  [(Hq/n + 2 Hkv/n) hd] or NULL
 *   w_o    [Hq hd][d/n]    w_gu [d][2 inter/n] (packed as larosa_pack_gate_up, the same
 *   inter/n range of gate and up)    w_down [inter][d/n]    adapter [d][d/n] or NULL
 * (the larosa_layer_weights struct keeps the FULL model dims; shard->world = n).
 * The layer runs as 5 phases; after each the caller all-gathers `out` into the next phase's
 * `x` (x, resid [batch][full width]; out [batch][local width]).  At batch 1 the rank-major
 * gather is already the column order; at batch > 1 larosa_shard_gather_permute turns the
 * gathered [world][batch][local] blocks into [batch][full]:
 *   0: x = r (full)      -> Top-K h1 (RMS) -> QKV (local heads, RoPE, local KV append)
 *                           -> attention (local heads)                 -> out = h2 [Hq hd / n]
 *   1: x = h2 (full)     -> Top-K h2 -> O (local cols)    -> out = r_mid cols = r + y_o [d/n]
 *   2: x = r_mid (full)  -> Top-K h3 (RMS) -> gate|up (local) -> out = SiLU(g) u [inter/n]
 *   3: x = h4 (full)     -> Top-K h4 -> down (local cols) -> out = r_mid + y_down [d/n]
 *   4: x = that (full)   -> adapter (dense, local cols)   -> out = r_next cols [d/n]
 *      (phase 4 is skipped when adapter == NULL: phase 3's output is r_next)
 * With adapter_in_down (w_down = Wd Q_{l+1}, SURVEY §8(e) "4-gather form"): phase 3 computes
 *   out = r_next cols = r_mid A_l[:, cols] + Top-K(h4) w_down[:, cols] (resid = the full r_mid),
 *   and there is no phase 4 (EINVAL): 4 all-gathers per layer.
 * resid = the full residual r (phases 1, 3 read r resp. r_mid from it: pass phase 0's x for
 * phase 1 and phase 2's x for phase 3).  Every rank derives the identical Top-K rule from
 * the identical gathered vector, so kept sets agree across ranks by construction.
 * k_cache / v_cache: this rank's [batch][Hkv/n][max_ctx][hd]; pos [batch].  Requires
 * Hq % n == 0, Hkv % n == 0, d % (8 n) == 0, inter % (64 n) == 0 (an MLP width that is not,
 * e.g. Qwen2.5-72B's 29568 at n = 4, 8, is padded with zero gate/up columns and zero down rows:
 * their h4 entries are exactly 0 and the Top-K with k_h4 <= the true width never prefers them
 * over a real entry, lower index winning ties -- the padded layer computes the same function;
 * model.shard_layer does this).  Batch 1: the fused SELECT GEMVs; batch > 1: the cluster Top-K
 * rule kernel and the union GEMV (tcgen05 at batch >= 8).  One workspace per rank and batch
 * (size query with the shard), zero-filled once.  W4 sites (w4_codes) are EUNSUPPORTED here.
 * ------------------------------------------------------------------------------ */
typedef struct {
    int32_t rank, world;
    int32_t batch;       /* tokens per step, 1..16 (ABI 5) */
    /* P2P push of the phase output instead of an all-gather (ABI 7; NULL = off):
     * DEVICE arrays of `world` addresses -- peer_dst[p]: rank p's gathered buffer for this phase's
     * output ([batch][peer_ld] fp32, e.g. torch symmetric memory mapped over NVLink), already offset
     * to THIS rank's first column; peer_flag[p]: rank p's uint32 arrival counter.  The kernel that
     * produces `out` also stores every value into every rank's buffer and then adds the number of
     * values it stored to every rank's counter (release, system scope); each rank then calls
     * larosa_shard_wait(its counter, batch * world * d_local) before reading its buffer. */
    const uint64_t* peer_dst;
    const uint64_t* peer_flag;
    int64_t peer_ld;
} larosa_shard;
size_t larosa_shard_workspace_size(const larosa_layer_weights* w, const larosa_shard* shard, int64_t max_ctx);
larosa_status larosa_sparse_layer_shard_phase(const larosa_layer_weights* w, const larosa_layer_plan* plan,
                                              const larosa_shard* shard, int32_t phase, const float* x,
                                              const float* resid, float* out, uint16_t* k_cache,
                                              uint16_t* v_cache, const int32_t* pos, int64_t max_ctx, void* ws,
                                              size_t ws_bytes, larosa_stream_t stream);

/* The consumer side of the P2P push (ABI 7): *expected += count, then wait (one device thread,
 * acquire at system scope) until the arrival counter *flag has reached *expected (wrap-safe).
 * expected: a device word of the caller's, zero at first use, only ever touched by this call.
 * Graph capturable; the following kernels in the stream see every pushed value. */
larosa_status larosa_shard_wait(const uint32_t* flag, uint32_t* expected, uint32_t count, larosa_stream_t stream);

/* P2P all-gather of an arbitrary [batch][d_local] fp32 slice (src row stride src_ld): every value
 * into every rank's buffer (peer_dst / peer_flag / peer_ld as in larosa_shard), then the counters
 * (the LM head's logits in the sharded decode step).  ABI 7. */
larosa_status larosa_peer_push(const float* src, int32_t batch, int64_t d_local, int64_t src_ld,
                               const uint64_t* peer_dst, const uint64_t* peer_flag, int32_t world,
                               int64_t peer_ld, larosa_stream_t stream);

/* gathered fp32 [world][batch][d_local] (an NCCL all_gather_into_tensor of every rank's
 * [batch][d_local] phase output) -> out [batch][world * d_local] (the full vectors in column
 * order).  out must not alias gathered.  Asynchronous. */
larosa_status larosa_shard_gather_permute(const float* gathered, int32_t world, int32_t batch,
                                          int64_t d_local, float* out, larosa_stream_t stream);

/* Greedy token of each row: out[b] = arg-max_{i < n} logits[b][i] (row stride ld), the lowest
 * index on exact ties -- the decode step's last operation, here for a vocabulary gathered from
 * column-sharded LM heads.  Asynchronous. */
larosa_status larosa_argmax(const float* logits, int32_t batch, int64_t n, int64_t ld, int32_t* out,
                            larosa_stream_t stream);

/* ------------------------------------------------------------------------------
 * Calibration of the rotation (§4.2, eq. 1):
 * larosa_calib_covariance: C[d][d] fp32 = scale * X^T X (+ C if accumulate != 0) over
 *   calibration activations X bf16 [n_tok][d] row-major (one layer's residual-stream inputs).
 *   Eq. 1 is Cov = (1/M) sum_i X_i^T X_i over M sequences, uncentered: pass
 *   scale = 1/M and accumulate the sequences (or any batching of their tokens).  tcgen05
 *   path when d % 128 == 0, n_tok % 64 == 0 and X, C are 16-byte aligned (workspace: the
 *   size query); otherwise a CUDA-core kernel (no workspace needed).  Asynchronous.
 * larosa_pca_rotation: Q fp32 [d][d] row-major with Q[:, i] the eigenvector of the i-th
 *   largest eigenvalue of C (symmetrised), lam fp32 [d] the eigenvalues descending (negative
 *   round-off clamped to 0); each eigenvector's largest-|entry| component is positive (lowest
 *   row on ties) -- SURVEY Z7.  Our fp64 cyclic two-sided Jacobi (the oracle's rotation, Z8)
 *   parallelised by a round-robin ordering: each sweep is d-1 rounds of d/2 disjoint rotations
 *   applied at once (captured as one CUDA graph), until off(A) <= 1e-12 ||A||_F, at most 100
 *   sweeps.  Synchronises the stream; LAROSA_ECUDA if it does not converge.  Offline path
 *   (workspace: 2 d^2 doubles + small arrays).
 * ------------------------------------------------------------------------------ */
size_t larosa_calib_covariance_workspace_size(int64_t n_tok, int64_t d);
larosa_status larosa_calib_covariance(const uint16_t* X, int64_t n_tok, int64_t d, float scale, int32_t accumulate,
                                      float* C, void* ws, size_t ws_bytes, larosa_stream_t stream);
size_t larosa_pca_rotation_workspace_size(int64_t d);
larosa_status larosa_pca_rotation(const float* C, int64_t d, float* Q, float* lam, void* ws, size_t ws_bytes,
                                  larosa_stream_t stream);

/* ------------------------------------------------------------------------------
 * W4A16 (the paper's compatibility with weight quantisation):
 * group-quantised int4 weights in the column-major layout, group size LAROSA_W4_GROUP along
 * the output dimension of each input row:
 *   Wq uint8 [d_in][d_out / 2]: byte b of row j = columns 2b (low nibble), 2b + 1 (high)
 *   S  fp16 bits [d_in][d_out / LAROSA_W4_GROUP];  w[j][o] = (q - 8) * S[j][o / group]
 * larosa_quantize_w4: from bf16 W [d_in][d_out]: scale = RNE_fp16(max |w| / 7) per (row,
 *   group) (fp32 divide), q = clamp(rint(w / scale) + 8, 0, 15) (fp32 divide; scale 0 -> 8).
 *   d_out % 256 == 0.  Asynchronous.
 * larosa_topk_sparse_gemv_w4: larosa_topk_sparse_gemv on these weights,
 *   y[o] = sum_{j in S} x[j] s w[j][o]; same selection (Top-K of |x|, ties -> lower index),
 *   workspace and `prepared` semantics; d_out % 256 == 0; Wq, x, y 16-byte aligned, S 4-byte.
 * ------------------------------------------------------------------------------ */
#define LAROSA_W4_GROUP 128
larosa_status larosa_quantize_w4(const uint16_t* W, int64_t d_in, int64_t d_out, uint8_t* Wq, uint16_t* S,
                                 larosa_stream_t stream);
size_t larosa_topk_sparse_gemv_w4_workspace_size(int64_t d_in, int64_t d_out);
larosa_status larosa_topk_sparse_gemv_w4(const float* x, int64_t d_in, int64_t k, float rms_eps, const uint8_t* Wq,
                                         const uint16_t* S, int64_t d_out, float* y, int32_t prepared, void* ws,
                                         size_t ws_bytes, larosa_stream_t stream);

/* ------------------------------------------------------------------------------
 * Prefill (full sparsification of prompt tokens): n_tok tokens, each
 * with its own exact Top-K (ties -> lower index) and RMS scale as larosa_rotate_topk (R = NULL):
 *   Y[t][o] = sum_{j in S_t} X[t][j] s_t W[j][o]
 * X fp32 [n_tok][d_in], W bf16 [d_in][d_out] (Wc layout, 16-byte aligned), Y fp32 [n_tok][d_out].
 * All on our kernels: a per-token selection kernel (exact k-th key by a bitwise search of
 * block-wide counts, index tie-break, fixed-order RMS sum) writes the masked activations
 * x_j s_t (0 where not kept) as bf16 -- split = 1 also writes the bf16 remainder, ~16 mantissa
 * bits in total -- and a tcgen05 GEMM (128 output columns x 256 tokens per CTA, TMA operands, TMEM
 * accumulator) multiplies them with W, skipping every 64-row block of W that no token of its
 * 256-token tile keeps.  split = 0: one bf16 MMA per block (activation rounding 2^-9 relative:
 * max |dY| / ||Y||_2 ~ 3e-5 at d_out 22016, inside north_star's 1e-3); split = 1: two MMAs.
 * d_in, d_out multiples of 8; d_in <= 32768.  Workspace: the size query (scratch, no zero-fill).
 * ------------------------------------------------------------------------------ */
size_t larosa_prefill_sparse_gemm_workspace_size(int64_t n_tok, int64_t d_in, int32_t split);
larosa_status larosa_prefill_sparse_gemm(const float* X, int64_t n_tok, int64_t d_in, int64_t k, float rms_eps,
                                         const uint16_t* W, int64_t d_out, float* Y, int32_t split, void* ws,
                                         size_t ws_bytes, larosa_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* LAROSA_H */
