"""LaRoSA fp64 CPU oracle — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  It shares no code with
``paper_2507_01299_b200/`` (the CUDA path) and imports nothing from it: its bf16
codec, Top-K, GEMV, RoPE, attention and k-rule are written here, independently,
in float64, straight from the paper (PAPER.md = /root/reference/PAPER.md,
"P:n" = line n) and the readings listed in DESIGN.md §3 ("Z" numbers follow
SURVEY.md §8(c)).

Conventions: every weight is ``Wc = W_pt^T`` stored
row-major ``[d_in][d_out]`` (the paper's "column-major W", P:414 (1)); a
projection is ``y = x · Wc``.  Bf16 tensors arrive as their raw uint16 bits and
are widened exactly (bits << 16 -> float32 -> float64).

Every function cites the passage it follows.  Functions with no independent pin
say so ("parity unpinned") — see DESIGN.md §4.  Pins live in
``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "bf16_to_f64", "f64_to_bf16_rne", "covariance", "jacobi_eigh", "build_rotation",
    "residual_adapter", "fold_left_qt", "fold_right_q", "rotate", "rms_scale", "topk",
    "topk_mask", "sparse_gemv", "dense_gemv", "compute_k", "solve_alpha", "site_ks",
    "std_normal_pdf", "std_normal_cdf", "std_normal_inv_cdf", "theory_relative_error",
    "rope", "decode_attention", "silu", "rmsnorm", "dense_block", "larosa_block", "build_rotation_lapack",
    "actual_sparsity", "embed", "lm_head", "greedy", "larosa_decode_step", "quantize_w4", "dequantize_w4",
    "W4_GROUP",
]


# ----------------------------------------------------------------------------------
# bf16 codec (own implementation; weights are bf16, math is fp64 here)
# ----------------------------------------------------------------------------------
def bf16_to_f64(bits) -> np.ndarray:
    """Widen raw bf16 bit patterns (uint16) to float64 exactly: bf16 is the top half of
    an IEEE float32, so (bits << 16) reinterpreted as float32 is the exact value."""
    b = np.asarray(bits).astype(np.uint16).astype(np.uint32) << np.uint32(16)
    with np.errstate(invalid="ignore"):          # NaN payloads widen as NaN
        return b.view(np.float32).astype(np.float64)


def f64_to_bf16_rne(x) -> np.ndarray:
    """Round float64 values directly to bf16 (round-to-nearest-even, one rounding) and
    return the uint16 bit patterns.  bf16 has 8 significant bits and float32's exponent
    range, so the rounding quantum of |x| in [2^e, 2^(e+1)) is 2^(e-7); below the
    smallest normal 2^-126 the quantum is the subnormal step 2^-133.  x/q and r*q are
    exact power-of-two scalings and np.rint rounds half to even."""
    x = np.asarray(x, dtype=np.float64)
    _, e = np.frexp(x)                       # x = f * 2^e, f in [0.5, 1)  ->  floor(log2|x|) = e-1
    q = np.ldexp(1.0, np.maximum(e - 1 - 7, -133))
    r = np.rint(x / q) * q                   # exactly representable in bf16 (hence float32)
    return (r.astype(np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


# ----------------------------------------------------------------------------------
# O-1 covariance, O-2 PCA rotation  (§4.2)
# ----------------------------------------------------------------------------------
def covariance(seqs) -> np.ndarray:
    """Cov(X_l, X_l^T) = (1/M) * sum_{i=1..M} (X_l^i)^T X_l^i   (eq. 1).

    Readings: the D x D feature covariance (Z2: the printed X X^T is N x N), i = 1..M
    (Z3), uncentered (Z4).  Each X_l^i is an [N_i, D] array of one sequence's layer-input
    activations.  Accumulated in sequence order; the upper triangle is mirrored so the
    result is exactly symmetric."""
    seqs = [np.asarray(s, dtype=np.float64) for s in seqs]
    if not seqs:
        raise ValueError("covariance: no sequences")
    d = seqs[0].shape[1]
    c = np.zeros((d, d))
    for x in seqs:
        if x.ndim != 2 or x.shape[1] != d:
            raise ValueError("covariance: dimension mismatch")
        c += x.T @ x
    c /= len(seqs)
    return np.triu(c) + np.triu(c, 1).T


def jacobi_eigh(a, max_sweeps: int = 100, tol: float = 1e-12):
    """Cyclic Jacobi eigen-solver for a symmetric matrix (Z8).

    Classical stable rotation: theta = (a_qq - a_pp) / (2 a_pq),
    t = sgn(theta) / (|theta| + sqrt(1 + theta^2)), c = 1/sqrt(1+t^2), s = t c;
    columns/rows p, q of A and columns p, q of V are rotated.  Sweeps until the
    off-diagonal Frobenius norm <= tol * ||A||_F, at most max_sweeps (else error).
    Returns (eigenvalues in diagonal order, V with A = V diag(lam) V^T)."""
    a = np.array(a, dtype=np.float64, copy=True)
    n = a.shape[0]
    if a.shape != (n, n):
        raise ValueError("jacobi_eigh: not square")
    norm_f = np.linalg.norm(a)
    if np.max(np.abs(a - a.T)) > 1e-10 * max(norm_f, 1e-300):
        raise ValueError("jacobi_eigh: not symmetric")
    v = np.eye(n)
    for _ in range(max_sweeps + 1):
        off = float(np.linalg.norm(a - np.diag(np.diag(a))))
        if off <= tol * norm_f:
            return np.diag(a).copy(), v
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = a[p, q]
                if apq == 0.0:
                    continue
                theta = (a[q, q] - a[p, p]) / (2.0 * apq)
                if abs(theta) > 1e150:                 # theta^2 would overflow: t -> 1/(2 theta)
                    t = 0.5 / theta
                else:
                    sgn = 1.0 if theta >= 0.0 else -1.0
                    t = sgn / (abs(theta) + math.sqrt(1.0 + theta * theta))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = t * c
                ap = a[:, p].copy()
                aq = a[:, q].copy()
                a[:, p] = c * ap - s * aq
                a[:, q] = s * ap + c * aq
                ap = a[p, :].copy()
                aq = a[q, :].copy()
                a[p, :] = c * ap - s * aq
                a[q, :] = s * ap + c * aq
                a[p, q] = 0.0
                a[q, p] = 0.0
                vp = v[:, p].copy()
                vq = v[:, q].copy()
                v[:, p] = c * vp - s * vq
                v[:, q] = s * vp + c * vq
    raise RuntimeError(f"jacobi_eigh: no convergence after {max_sweeps} sweeps (off={off:.3e})")


def build_rotation(cov):
    """Q_l = eigenvectors of Cov sorted by eigenvalue, descending   (§4.2).

    Readings (Z7): stable order on exact ties; eigenvalues >= -1e-8 tr(C) are clamped to
    0 (else error); sign: the largest-|entry| component of each eigenvector is made
    positive (lowest row index on ties).  Returns (Q, lam) with Q[:, i] = v_i."""
    cov = np.asarray(cov, dtype=np.float64)
    lam, v = jacobi_eigh(cov)
    tr = float(np.trace(cov))
    if np.any(lam < -1e-8 * abs(tr)):
        raise ValueError("build_rotation: covariance is not positive semidefinite")
    lam = np.where(lam < 0.0, 0.0, lam)
    order = np.argsort(-lam, kind="stable")
    lam = lam[order]
    q = v[:, order].copy()
    for i in range(q.shape[1]):
        j = int(np.argmax(np.abs(q[:, i])))      # argmax returns the lowest index on ties
        if q[j, i] < 0.0:
            q[:, i] = -q[:, i]
    return q, lam


def build_rotation_lapack(cov):
    """build_rotation with LAPACK's symmetric eigensolver (numpy.linalg.eigh, fp64) in place of the
    cyclic Jacobi loop, for widths where the pure-Python Jacobi sweep is too slow (d = 4096); the
    same ordering (descending, stable on exact ties), clamp and sign rule (Z7).  A library routine as
    one step (the eigendecomposition); pinned against jacobi_eigh / build_rotation at small d."""
    cov = np.asarray(cov, dtype=np.float64)
    if np.max(np.abs(cov - cov.T)) > 1e-10 * max(np.linalg.norm(cov), 1e-300):
        raise ValueError("build_rotation_lapack: not symmetric")
    lam, v = np.linalg.eigh(0.5 * (cov + cov.T))
    tr = float(np.trace(cov))
    if np.any(lam < -1e-8 * abs(tr)):
        raise ValueError("build_rotation_lapack: covariance is not positive semidefinite")
    lam = np.where(lam < 0.0, 0.0, lam)
    order = np.argsort(-lam, kind="stable")
    lam = lam[order]
    q = v[:, order].copy()
    for i in range(q.shape[1]):
        j = int(np.argmax(np.abs(q[:, i])))
        if q[j, i] < 0.0:
            q[:, i] = -q[:, i]
    return q, lam


def residual_adapter(q_l, q_next) -> np.ndarray:
    """A_l = Q_l^T Q_{l+1}, applied to each layer's output   (§4.2)."""
    return np.asarray(q_l, dtype=np.float64).T @ np.asarray(q_next, dtype=np.float64)


# ----------------------------------------------------------------------------------
# O-3 fold  (P:402-410 eqs. before_merge/after_merge; §3.2; Z6, Z21)
# ----------------------------------------------------------------------------------
def fold_left_qt(q, wc, gamma=None) -> np.ndarray:
    """Input-side fold Wc' = Q^T diag(gamma) Wc.

    Eq. after_merge writes the merged weight as (W Q)^T; with Wc = W^T
    (Z1) that is Q^T Wc.  The RMSNorm gain gamma, if given, is folded into Wc's input
    rows first (Z6) so the norm commutes with Q."""
    q = np.asarray(q, dtype=np.float64)
    w = np.asarray(wc, dtype=np.float64)
    if gamma is not None:
        w = np.asarray(gamma, dtype=np.float64)[:, None] * w
    return q.T @ w


def fold_right_q(wc, q) -> np.ndarray:
    """Output-side fold Wc' = Wc Q (W_o, W_down: the attention/MLP block then emits its
    output already rotated by Q, "if W_o is right-multiplied by ... Q"; Z21)."""
    return np.asarray(wc, dtype=np.float64) @ np.asarray(q, dtype=np.float64)


# ----------------------------------------------------------------------------------
# O-4 rotate, O-5 RMS, O-6 Top-K, O-7 masked GEMV   (§4.3)
# ----------------------------------------------------------------------------------
def rotate(x, r) -> np.ndarray:
    """x~ = x Q (eq. before_merge).  R = Q_l or the adapter A_l (Z20)."""
    return np.asarray(x, dtype=np.float64) @ np.asarray(r, dtype=np.float64)


def rms_scale(xr, eps: float) -> float:
    """s = 1 / sqrt(mean(x~^2) + eps): RMSNorm with gains folded into the weights leaves
    only this scalar (Z25)."""
    xr = np.asarray(xr, dtype=np.float64)
    return 1.0 / math.sqrt(float(np.sum(xr * xr)) / xr.shape[-1] + eps)


def topk(xr, k: int) -> np.ndarray:
    """S_k: indices of the k largest |x~_i|   (eq. 2; Z9).

    Tie-break (Z10): the total order is (|x~_i| descending, i ascending), i.e. the lower
    index wins.  Exactly k indices are returned (zeros may be kept, Z11), sorted
    ascending.  Inputs must be finite (Z12)."""
    xr = np.asarray(xr, dtype=np.float64)
    d = xr.shape[0]
    if not 0 <= k <= d:
        raise ValueError("topk: k out of range")
    if not np.all(np.isfinite(xr)):
        raise ValueError("topk: non-finite input")
    order = np.lexsort((np.arange(d), -np.abs(xr)))   # last key is primary
    return np.sort(order[:k]).astype(np.int64)


def topk_mask(idx, d: int) -> np.ndarray:
    """uint32 bitmask of the kept set: bit (i % 32) of word i // 32."""
    m = np.zeros((d + 31) // 32, dtype=np.uint32)
    for i in np.asarray(idx, dtype=np.int64):
        m[i // 32] |= np.uint32(1) << np.uint32(i % 32)
    return m


def actual_sparsity(x) -> float:
    """p = (1/D) sum_i 1(x_i = 0)   (eq. standard_Sparsity)."""
    x = np.asarray(x, dtype=np.float64)
    return float(np.count_nonzero(x == 0.0)) / x.shape[0]


def sparse_gemv(wc, idx, vals, bias=None) -> np.ndarray:
    """y_o = b_o + sum_{j in S} v_j Wc[j][o]   (P:407-410 eq. after_merge; P:414 (3)).

    Only the kept rows of the column-major weight are touched.  ``wc`` is float64
    [d_in][d_out]; idx ascending; the sum is a library matmul over the kept rows."""
    wc = np.asarray(wc, dtype=np.float64)
    idx = np.asarray(idx, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    y = vals @ wc[idx] if idx.size else np.zeros(wc.shape[1])
    if bias is not None:
        y = y + np.asarray(bias, dtype=np.float64)
    return y


def dense_gemv(wc, x, bias=None) -> np.ndarray:
    """Y = X W^T with Wc = W^T (eq. linear_mapping)."""
    y = np.asarray(x, dtype=np.float64) @ np.asarray(wc, dtype=np.float64)
    if bias is not None:
        y = y + np.asarray(bias, dtype=np.float64)
    return y


# ----------------------------------------------------------------------------------
# O-9 k and alpha  (App. B)
# ----------------------------------------------------------------------------------
def compute_k(alpha: float, p: float, d_in: int) -> int:
    """k = alpha (1 - p) D_in.

    Readings: round half away from zero in fp64, clamp to [0, D_in] (Z13, Z15); p = 0
    means the dense "0%" configuration, k = D_in at every site (Z16)."""
    if p == 0.0:
        return int(d_in)
    v = alpha * (1.0 - p) * d_in
    k = int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))
    return max(0, min(int(d_in), k))


def solve_alpha(alpha1: float, alpha3: float, m: float):
    """alpha2 = 4 - 3 alpha1;  alpha4 = (2 + M - 2 alpha3) / M   (App. B)."""
    return 4.0 - 3.0 * alpha1, (2.0 + m - 2.0 * alpha3) / m


def site_ks(p: float, alphas, d: int, inter: int):
    """Per-site kept counts (k_h1, k_h2, k_h3, k_h4) for a layer with hidden d and MLP
    width inter; h1, h2, h3 have D_in = d (h2 = Hq*hd = d), h4 has D_in = inter."""
    a1, a2, a3, a4 = alphas
    return (compute_k(a1, p, d), compute_k(a2, p, d), compute_k(a3, p, d), compute_k(a4, p, inter))


# ----------------------------------------------------------------------------------
# O-10 Theorem A.1
# ----------------------------------------------------------------------------------
def std_normal_pdf(t: float) -> float:
    """phi(t) = exp(-t^2/2) / sqrt(2 pi)."""
    return math.exp(-0.5 * t * t) / math.sqrt(2.0 * math.pi)


def std_normal_cdf(t: float) -> float:
    """Phi(t) = erfc(-t/sqrt2) / 2."""
    return 0.5 * math.erfc(-t / math.sqrt(2.0))


def std_normal_inv_cdf(u: float) -> float:
    """Phi^{-1}(u): Abramowitz-Stegun 26.2.23 rational guess (|err| < 4.5e-4) refined by
    Newton steps on the erfc-based Phi (SPEC S:52-69 design)."""
    if not 0.0 < u < 1.0:
        raise ValueError("std_normal_inv_cdf: u outside (0, 1)")
    pl = u if u < 0.5 else 1.0 - u
    t = math.sqrt(-2.0 * math.log(pl))
    z = t - (2.515517 + 0.802853 * t + 0.010328 * t * t) / (
        1.0 + 1.432788 * t + 0.189269 * t * t + 0.001308 * t * t * t)
    z = -z if u < 0.5 else z
    for _ in range(4):
        z -= (std_normal_cdf(z) - u) / std_normal_pdf(z)
    return z


def theory_relative_error(k: int, d: int) -> float:
    """Theorem A.1: E||y - y^S|| / E||y|| = sqrt(1 - k/D - 2 tau phi(tau)),
    tau = Phi^{-1}(1 - k/(2D)).  k = D -> 0; k = 0 -> 1 (limit)."""
    if not 0 <= k <= d:
        raise ValueError("theory_relative_error: k out of range")
    if k == d:
        return 0.0
    if k == 0:
        return 1.0
    tau = std_normal_inv_cdf(1.0 - k / (2.0 * d))
    return math.sqrt(max(0.0, 1.0 - k / d - 2.0 * tau * std_normal_pdf(tau)))


# ----------------------------------------------------------------------------------
# O-8 decoder block (Fig. 2; §3.1; glue conventions Z27)
# ----------------------------------------------------------------------------------
def rmsnorm(x, gamma, eps: float) -> np.ndarray:
    """RMSNorm(x) = gamma * x / sqrt(mean(x^2) + eps)."""
    x = np.asarray(x, dtype=np.float64)
    return np.asarray(gamma, dtype=np.float64) * x * rms_scale(x, eps)


def silu(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    return x / (1.0 + np.exp(-x))


def rope(v, pos: int, theta: float) -> np.ndarray:
    """HF rotate_half RoPE on one head vector of size hd (Z27; plumbing, not paper
    content): pairs (i, i + hd/2), inv_freq_i = theta^(-2i/hd), angle = pos * inv_freq_i."""
    v = np.asarray(v, dtype=np.float64)
    hd = v.shape[0]
    half = hd // 2
    i = np.arange(half, dtype=np.float64)
    ang = pos * theta ** (-2.0 * i / hd)
    c, s = np.cos(ang), np.sin(ang)
    out = np.empty(hd)
    out[:half] = v[:half] * c - v[half:] * s
    out[half:] = v[half:] * c + v[:half] * s
    return out


def decode_attention(q, k_cache, v_cache, ctx_len: int) -> np.ndarray:
    """One-token causal attention over positions [0, ctx_len) (Z27): GQA q-head h reads
    kv-head floor(h * Hkv / Hq); scale 1/sqrt(hd); softmax in fp64.
    q: [Hq, hd]; k_cache/v_cache: [Hkv, >=ctx_len, hd].  Returns [Hq * hd]."""
    q = np.asarray(q, dtype=np.float64)
    kc = np.asarray(k_cache, dtype=np.float64)
    vc = np.asarray(v_cache, dtype=np.float64)
    hq, hd = q.shape
    hkv = kc.shape[0]
    out = np.empty((hq, hd))
    for h in range(hq):
        g = (h * hkv) // hq
        sc = kc[g, :ctx_len] @ q[h] / math.sqrt(hd)
        w = np.exp(sc - np.max(sc))
        w /= np.sum(w)
        out[h] = w @ vc[g, :ctx_len]
    return out.reshape(-1)


def _split_qkv(y, hq, hkv, hd):
    q = y[: hq * hd].reshape(hq, hd)
    k = y[hq * hd: (hq + hkv) * hd].reshape(hkv, hd)
    v = y[(hq + hkv) * hd:].reshape(hkv, hd)
    return q, k, v


def _kv_store(x, kv_bf16: bool):
    """Z27: the KV cache is stored in bf16 (RNE); kv_bf16=False keeps fp64 (pure math)."""
    return bf16_to_f64(f64_to_bf16_rne(x)) if kv_bf16 else x


def dense_block(r, w, cfg, k_cache, v_cache, pos: int, kv_bf16: bool = False):
    """The unrotated, unsparsified pre-norm decoder layer (P:1381 block structure):
    h1 = RMSNorm(r) -> QKV (+bias, RoPE) -> attention -> h2 -> O -> r += ;
    h3 = RMSNorm(r) -> gate|up -> h4 = SiLU(g) * u -> down -> r += .
    ``w``: dict of float64 Wc matrices wq/wk/wv/wo/wg/wu/wd (+ bq/bk/bv, gamma1/2);
    ``k_cache``/``v_cache``: float64 [Hkv, max_ctx, hd], position ``pos`` is written.
    Returns (r_out, dict of intermediates)."""
    hq, hkv, hd, eps, theta = cfg["hq"], cfg["hkv"], cfg["hd"], cfg["eps"], cfg["theta"]
    h1 = rmsnorm(r, w["gamma1"], eps)
    q = dense_gemv(w["wq"], h1, w.get("bq")).reshape(hq, hd)
    k = dense_gemv(w["wk"], h1, w.get("bk")).reshape(hkv, hd)
    v = dense_gemv(w["wv"], h1, w.get("bv")).reshape(hkv, hd)
    q = np.stack([rope(q[h], pos, theta) for h in range(hq)])
    k = np.stack([rope(k[h], pos, theta) for h in range(hkv)])
    k_cache[:, pos] = _kv_store(k, kv_bf16)
    v_cache[:, pos] = _kv_store(v, kv_bf16)
    h2 = decode_attention(q, k_cache, v_cache, pos + 1)
    r = r + dense_gemv(w["wo"], h2)
    h3 = rmsnorm(r, w["gamma2"], eps)
    h4 = silu(dense_gemv(w["wg"], h3)) * dense_gemv(w["wu"], h3)
    r = r + dense_gemv(w["wd"], h4)
    return r, {"h1": h1, "h2": h2, "h3": h3, "h4": h4, "q": q}


def larosa_block(r, wf, cfg, ks, k_cache, v_cache, pos: int, adapter=None, kv_bf16: bool = False,
                 adapter_in_down: bool = False, adapter_mid=None):
    """The LaRoSA layer on folded weights, step by step as Fig. 2 and
    eqs. before/after_merge:

      r is the residual stream in Q_l's basis;
      h1: S1 = Top-K_{k1}(r), vals = r[S1] * s(r)   (RMS scale, gains folded, Z25)
          y = sparse GEMV over Wqkv' = Q^T diag(g1) Wqkv (+bias), RoPE, attention -> h2
      h2: S2 = Top-K_{k2}(h2) (Q = I at h2) -> O' = Wo Q  -> r += y
      h3: S3 = Top-K_{k3}(r), vals = r[S3] * s(r)  -> gate|up' = Q^T diag(g2) W -> h4
      h4: S4 = Top-K_{k4}(h4) (Q = I) -> down' = Wd Q -> r += y
      adapter: r_next = r A_l, A_l = Q_l^T Q_{l+1}   (Z20)

    ``wf``: dict of float64 folded matrices wqkv/wo/wg/wu/wd (+ bqkv);
    ``ks``: (k1, k2, k3, k4).  Returns (r_next, intermediates incl. idx per site).

    ``adapter_in_down``: the adapter is folded into the down projection's output side,
    wd = Wd Q_{l+1} = (Wd Q_l) A_l (the "4-gather form"; reading R4).
    By linearity of the adapter, (r_mid + y_down Q_l-basis) A_l = r_mid A_l + y_down',
    so r_next = r_mid A_l + h4[S4] wd; the down site's selection S4 is unchanged (it is taken
    on h4, before the projection).

    ``adapter_mid``: the block-wise rotation Q_B of the paper's ablation (Table 6, P:204-215;
    SURVEY §8(f) N4): the attention block runs in Q_a's basis and the MLP block in Q_m's, with
    A_mid = Q_a^T Q_m applied to the residual between them, folded beside O like the adapter
    beside down: wo = Wo Q_m, r_mid = r A_mid + h2[S2] wo; gate|up are folded with Q_m (input
    side) and down / the closing adapter carry the residual from Q_m's basis onward."""
    hq, hkv, hd, eps, theta = cfg["hq"], cfg["hkv"], cfg["hd"], cfg["eps"], cfg["theta"]
    k1, k2, k3, k4 = ks
    out = {}
    s1 = topk(r, k1)
    v1 = r[s1] * rms_scale(r, eps)
    y = sparse_gemv(wf["wqkv"], s1, v1, wf.get("bqkv"))
    q, k, v = _split_qkv(y, hq, hkv, hd)
    q = np.stack([rope(q[h], pos, theta) for h in range(hq)])
    k = np.stack([rope(k[h], pos, theta) for h in range(hkv)])
    k_cache[:, pos] = _kv_store(k, kv_bf16)
    v_cache[:, pos] = _kv_store(v, kv_bf16)
    h2 = decode_attention(q, k_cache, v_cache, pos + 1)
    s2 = topk(h2, k2)
    if adapter_mid is not None:
        r = rotate(r, adapter_mid) + sparse_gemv(wf["wo"], s2, h2[s2])
    else:
        r = r + sparse_gemv(wf["wo"], s2, h2[s2])
    r_mid = r.copy()
    s3 = topk(r, k3)
    v3 = r[s3] * rms_scale(r, eps)
    h4 = silu(sparse_gemv(wf["wg"], s3, v3)) * sparse_gemv(wf["wu"], s3, v3)
    s4 = topk(h4, k4)
    y_down = sparse_gemv(wf["wd"], s4, h4[s4])
    if adapter_in_down:
        if adapter is None:
            raise ValueError("adapter_in_down needs the adapter A_l")
        r = rotate(r_mid, adapter) + y_down
        out.update(idx1=s1, idx2=s2, idx3=s3, idx4=s4, q=q, h2=h2, r_mid=r_mid, h4=h4, r_out=None)
        return r, out
    r = r + y_down
    out.update(idx1=s1, idx2=s2, idx3=s3, idx4=s4, q=q, h2=h2, r_mid=r_mid, h4=h4, r_out=r.copy())
    if adapter is not None:
        r = rotate(r, adapter)
    return r, out


# ----------------------------------------------------------------------------------
# W4A16 weights (quantisation compatibility P:306-344).  The format is this
# implementation's (the paper fixes none): symmetric int4 per (input row, group of 128 outputs).
# The integer decisions are taken in fp32 as the header states (the kernel's precision).
# ----------------------------------------------------------------------------------
W4_GROUP = 128


def quantize_w4(wc_bf16_bits):
    """(codes uint8 [d_in][d_out] in [0, 15], scale fp16 bits [d_in][d_out/128]) of a bf16
    weight: scale = RNE_fp16(max|w| / 7) (fp32 divide), q = clamp(rint(w / scale) + 8, 0, 15)
    (fp32 divide, rint = round half to even); scale 0 -> q = 8."""
    w = bf16_to_f64(wc_bf16_bits).astype(np.float32)
    d_in, d_out = w.shape
    if d_out % W4_GROUP:
        raise ValueError("quantize_w4: d_out % 128 != 0")
    g = w.reshape(d_in, d_out // W4_GROUP, W4_GROUP)
    amax = np.max(np.abs(g), axis=2)
    scale16 = (amax / np.float32(7.0)).astype(np.float16)
    s = scale16.astype(np.float32)[:, :, None]
    with np.errstate(divide="ignore", invalid="ignore"):
        q = np.where(s > 0, np.clip(np.rint(g / s) + 8, 0, 15), 8)
    return q.reshape(d_in, d_out).astype(np.uint8), scale16.view(np.uint16)


def dequantize_w4(codes, scale_bits) -> np.ndarray:
    """w[j][o] = (q[j][o] - 8) * S[j][o / 128] in fp64."""
    codes = np.asarray(codes, dtype=np.float64)
    s = np.asarray(scale_bits, dtype=np.uint16).view(np.float16).astype(np.float64)
    return (codes - 8.0) * np.repeat(s, W4_GROUP, axis=1)


# ----------------------------------------------------------------------------------
# decode step: embedding -> L LaRoSA layers -> final RMS -> LM head
# ----------------------------------------------------------------------------------
def embed(e_folded, token: int) -> np.ndarray:
    """The residual stream enters layer 0 in Q_0's basis: r_0 = e_token Q_0, i.e. the row
    of the folded embedding E' = E Q_0 ("Q_0 ... merged into the embedding")."""
    return np.asarray(e_folded, dtype=np.float64)[int(token)].copy()


def lm_head(r, h_folded, eps: float) -> np.ndarray:
    """logits = RMSNorm(r_L) H with r_L in Q_L's basis and the final RMSNorm gain and Q_L
    folded into the head, H' = Q_L^T diag(gamma_f) H (Z6 for the gain): since Q_L
    is orthogonal, RMSNorm commutes with it and only the scale s remains:
    logits = (r s) H'.  The head is dense (the paper does not sparsify it)."""
    r = np.asarray(r, dtype=np.float64)
    return dense_gemv(h_folded, r * rms_scale(r, eps))


def greedy(logits) -> int:
    """Greedy decoding: the arg-max logit, the lowest index on exact ties."""
    logits = np.asarray(logits, dtype=np.float64)
    return int(np.flatnonzero(logits == logits.max())[0])


def larosa_decode_step(token: int, e_folded, layers, cfg, ks, caches, pos: int, h_folded, eps: float,
                       kv_bf16: bool = False):
    """One decode token through the whole model (a7): r = embed; for each layer,
    larosa_block (its own adapter A_l into the next layer's basis; the last layer's adapter
    is None when the head holds Q_L); logits = lm_head(r); next token = greedy(logits).
    ``layers``: list of (wf, adapter) pairs; ``caches``: list of (k_cache, v_cache),
    updated at ``pos``.  Returns (next_token, logits, final residual)."""
    r = embed(e_folded, token)
    for (wf, adapter), (kc, vc) in zip(layers, caches):
        r, _ = larosa_block(r, wf, cfg, ks, kc, vc, pos, adapter=adapter, kv_bf16=kv_bf16)
    logits = lm_head(r, h_folded, eps)
    return greedy(logits), logits, r
