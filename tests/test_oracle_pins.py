"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test names the oracle function it pins and what fixes the expected value:
a worked example (tests/golden/*.json, cited), a closed form, an invariant, a
library routine for a special case (LAPACK eigh, scipy's normal quantile, torch's
bf16 cast), or brute force on tiny inputs.  See DESIGN.md §4 for the table.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch
from scipy.stats import norm

import oracle as O
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


WE = _gold("worked_examples.json")


# ------------------------------------------------------------------ bf16 codec
def test_bf16_worked_examples():
    for ex in WE["bf16"]:
        assert int(O.f64_to_bf16_rne(ex["f32"])) == ex["bits"], ex["cite"]
        assert O.bf16_to_f64(np.uint16(ex["bits"])) == O.bf16_to_f64(O.f64_to_bf16_rne(ex["f32"]))


def test_bf16_exhaustive_roundtrip():
    """Every finite bf16 bit pattern widens and re-encodes to itself."""
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    v = O.bf16_to_f64(bits)
    fin = np.isfinite(v)
    back = O.f64_to_bf16_rne(v[fin])
    # -0 and +0 keep their own patterns
    assert np.array_equal(back, bits[fin])


def test_bf16_matches_torch_rne_on_fp32_inputs():
    """torch's float32->bfloat16 cast is RNE; fp32 inputs are exact in fp64 so both
    see the same value and must agree bit for bit (incl. subnormal range)."""
    g = torch.Generator().manual_seed(5)
    x = torch.randn(200000, generator=g) * torch.pow(2.0, torch.randint(-140, 60, (200000,), generator=g).float())
    x = x[torch.isfinite(x)]
    ref = x.to(torch.bfloat16).view(torch.int16).numpy().astype(np.uint16)
    got = O.f64_to_bf16_rne(x.numpy().astype(np.float64))
    finite = np.isfinite(O.bf16_to_f64(ref))
    assert np.array_equal(got[finite], ref[finite])


# ------------------------------------------------------------------ covariance
def test_covariance_single_token_is_outer_product():
    x = np.array([[1.0, -2.0, 0.5]])
    assert np.array_equal(O.covariance([x]), np.outer(x[0], x[0]))


def test_covariance_duplicate_sequences_idempotent():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((5, 6))
    assert np.allclose(O.covariance([x, x]), O.covariance([x]), rtol=0, atol=1e-14)


def test_covariance_brute_force_loop():
    rng = np.random.default_rng(1)
    seqs = [rng.standard_normal((n, 8)) for n in (3, 5, 2)]
    c = np.zeros((8, 8))
    for s in seqs:
        for t in range(s.shape[0]):
            for a in range(8):
                for b in range(8):
                    c[a, b] += s[t, a] * s[t, b]
    c /= 3
    assert np.allclose(O.covariance(seqs), c, rtol=1e-13, atol=1e-13)
    cc = O.covariance(seqs)
    assert np.array_equal(cc, cc.T)


# ------------------------------------------------------------------ PCA rotation
@pytest.mark.parametrize("ex", WE["eigh"])
def test_build_rotation_worked_examples(ex):
    q, lam = O.build_rotation(np.array(ex["A"]))
    assert np.allclose(lam, ex["lam"], atol=1e-12)
    assert np.allclose(q, np.array(ex["Q"]), atol=1e-12), ex["cite"]


def test_build_rotation_matches_lapack_distinct_eigenvalues():
    """Special case that reduces to a library routine: LAPACK eigh (numpy) with the same
    descending order and sign rule must give the same Q for distinct eigenvalues."""
    rng = np.random.default_rng(2)
    d = 32
    b = rng.standard_normal((d, d))
    c = b @ b.T / d
    q, lam = O.build_rotation(c)
    w, v = np.linalg.eigh(c)
    order = np.argsort(-w)
    w, v = w[order], v[:, order]
    for i in range(d):
        j = int(np.argmax(np.abs(v[:, i])))
        if v[j, i] < 0:
            v[:, i] = -v[:, i]
    assert np.allclose(lam, w, rtol=1e-10, atol=1e-12)
    assert np.allclose(q, v, atol=1e-8)


@pytest.mark.parametrize("d", [64, 256])
def test_jacobi_invariants(d):
    """Q^T Q = I (BASELINE: 1e-6; expect ~1e-14), reconstruction <= 1e-7 ||C||_F,
    Q^T C Q diagonal with descending diagonal (the defining PCA property)."""
    rng = np.random.default_rng(d)
    b = rng.standard_normal((d, d))
    c = b @ b.T
    q, lam = O.build_rotation(c)
    assert np.max(np.abs(q.T @ q - np.eye(d))) < 1e-12
    assert np.linalg.norm(q @ np.diag(lam) @ q.T - c) <= 1e-7 * np.linalg.norm(c)
    t = q.T @ c @ q
    assert np.max(np.abs(t - np.diag(np.diag(t)))) <= 1e-9 * np.linalg.norm(c)
    assert np.all(np.diff(np.diag(t)) <= 1e-9 * np.linalg.norm(c))


def test_toy_calibration_rotation():
    """C1: the toy calibration set has distinct eigenvalues 2^(-i/4) (scaled), so Q is
    unique up to sign; rotated coordinates' variances come out descending."""
    seqs = [s.numpy() for s in synth.toy_calibration()]
    c = O.covariance(seqs)
    q, lam = O.build_rotation(c)
    assert np.max(np.abs(q.T @ q - np.eye(64))) < 1e-12
    z = np.concatenate(seqs) @ q
    second_moment = np.mean(z * z, axis=0)
    # Cov sums each sequence's X^T X and divides by M sequences: lam = N_tok * E[z_i^2]
    assert np.allclose(second_moment * seqs[0].shape[0], lam, rtol=1e-9)
    assert np.all(np.diff(lam) <= 0)


# ------------------------------------------------------------------ fold / adapter / rotate
def test_fold_computational_invariance():
    """(x Q)(Q^T diag(g) Wc) = (x * g) Wc and (y Wc Q) Q^T = y Wc."""
    rng = np.random.default_rng(3)
    d, dout = 48, 80
    q = synth.haar_orthogonal(d, 4).numpy()
    wc = rng.standard_normal((d, dout))
    g = 1 + 0.1 * rng.standard_normal(d)
    x = rng.standard_normal(d)
    lhs = O.rotate(x, q) @ O.fold_left_qt(q, wc, g)
    assert np.allclose(lhs, (x * g) @ wc, rtol=0, atol=1e-12 * np.linalg.norm((x * g) @ wc))
    w2 = rng.standard_normal((dout, d))
    y = rng.standard_normal(dout)
    assert np.allclose(O.fold_right_q(w2, q) @ q.T, w2, atol=1e-12)
    assert np.allclose(y @ O.fold_right_q(w2, q), (y @ w2) @ q, atol=1e-12)


def test_fold_identity_is_bit_identical():
    wc = O.bf16_to_f64(synth.gaussian_bf16((16, 24), 1, 0.25).numpy())
    assert np.array_equal(O.fold_left_qt(np.eye(16), wc), wc)
    assert np.array_equal(O.fold_right_q(wc.T, np.eye(16)), wc.T)


def test_adapter_identities():
    q = synth.haar_orthogonal(32, 9).numpy()
    q2 = synth.haar_orthogonal(32, 10).numpy()
    assert np.allclose(O.residual_adapter(q, q), np.eye(32), atol=1e-13)
    a = O.residual_adapter(q, q2)
    assert np.max(np.abs(a.T @ a - np.eye(32))) < 1e-13
    assert np.array_equal(O.residual_adapter(np.eye(4), np.eye(4)), np.eye(4))


def test_rotate_preserves_norm_and_inverts():
    rng = np.random.default_rng(4)
    q = synth.haar_orthogonal(40, 11).numpy()
    x = rng.standard_normal(40)
    xr = O.rotate(x, q)
    assert abs(np.linalg.norm(xr) - np.linalg.norm(x)) < 1e-13 * np.linalg.norm(x)
    assert np.allclose(xr @ q.T, x, atol=1e-13)


def test_rms_scale_closed_form():
    x = np.full(8, -3.0)
    assert O.rms_scale(x, 0.0) == pytest.approx(1 / 3.0, rel=1e-15)
    q = synth.haar_orthogonal(8, 3).numpy()
    y = np.arange(8.0) - 3
    assert O.rms_scale(y @ q, 1e-6) == pytest.approx(O.rms_scale(y, 1e-6), rel=1e-13)


# ------------------------------------------------------------------ Top-K
@pytest.mark.parametrize("ex", WE["topk"])
def test_topk_worked_examples(ex):
    assert O.topk(np.array(ex["x"]), ex["k"]).tolist() == ex["idx"], ex["cite"]


def _brute_topk(x, k):
    """Z10 characterisation: the lexicographically smallest ascending index set S, |S| = k,
    with min_{i in S} |x_i| >= max_{j not in S} |x_j|."""
    n = len(x)
    a = np.abs(x)
    for s in itertools.combinations(range(n), k):   # lexicographic order
        rest = [j for j in range(n) if j not in s]
        if not s or not rest or min(a[list(s)]) >= max(a[rest]):
            return list(s)
    raise AssertionError


def test_topk_brute_force_small():
    rng = np.random.default_rng(6)
    for trial in range(300):
        n = int(rng.integers(1, 11))
        # integer-valued entries with signs: many exact |.| ties, zeros and -0
        x = rng.integers(-3, 4, n).astype(np.float64)
        x[rng.random(n) < 0.1] = -0.0
        k = int(rng.integers(0, n + 1))
        got = O.topk(x, k).tolist()
        assert got == _brute_topk(x, k), (x, k)


def test_topk_exact_sparsity_every_token():
    """'TopK 50.0 (+-0.0)': exactly k kept for every token incl. token 0."""
    x = synth.residual_activation(32, 256, 3).numpy()
    for t in range(32):
        idx = O.topk(x[t], 128)
        dense = np.zeros(256)
        dense[idx] = x[t][idx]
        assert len(idx) == 128 and len(set(idx.tolist())) == 128
        assert O.actual_sparsity(dense) == 0.5
        assert np.all(np.diff(idx) > 0)


def test_topk_mask_bits():
    m = O.topk_mask([0, 31, 32, 65], 70)
    assert m.tolist() == [0x80000001, 0x1, 0x2]


# ------------------------------------------------------------------ k and alpha
@pytest.mark.parametrize("ex", WE["compute_k"])
def test_compute_k_worked_examples(ex):
    assert O.compute_k(ex["alpha"], ex["p"], ex["d"]) == ex["k"], ex["cite"]


def test_alpha_table():
    """App. B table: alpha2 exact; alpha4 within 0.01 of the printed value
    (printed to 2 decimals; Z17), with the true M for Qwen2.5-72B (Z18)."""
    for row in _gold("alpha_table.json")["rows"]:
        a2, a4 = O.solve_alpha(row["a1"], row["a3"], row["M_true"])
        assert a2 == pytest.approx(row["a2"], abs=1e-12), row["model"]
        assert abs(a4 - row["a4"]) <= 0.01, row["model"]
        assert 3 * row["a1"] + a2 == pytest.approx(4.0, abs=1e-12)
        assert 2 * row["a3"] + row["M_true"] * a4 == pytest.approx(2 + row["M_true"], abs=1e-12)


def test_site_ks_survey_appendix_rows():
    """Derived k rows of SURVEY App. A (e.g. LLaMA3-8B 40% paper-alpha 1966/3932/1966/9585)
    follow from the rule; a dropped (1-p) or swapped site would change them."""
    a2, a4 = O.solve_alpha(0.8, 0.8, 3.5)
    assert O.site_ks(0.4, (0.8, a2, 0.8, a4), 4096, 14336) == (1966, 3932, 1966, 9585)
    a2, a4 = O.solve_alpha(0.9, 0.8, 11008 / 4096)
    assert O.site_ks(0.5, (0.9, a2, 0.8, a4), 4096, 11008) == (1843, 2662, 1638, 6323)
    assert O.site_ks(0.5, (1, 1, 1, 1), 4096, 11008) == (2048, 2048, 2048, 5504)


# ------------------------------------------------------------------ GEMV
@pytest.mark.parametrize("ex", WE["gemv"])
def test_gemv_worked_example(ex):
    wc = np.array(ex["W_pt"]).T
    assert O.dense_gemv(wc, ex["x"]).tolist() == ex["y"]
    assert O.sparse_gemv(wc, [0, 1], ex["x"]).tolist() == ex["y"]


def test_sparse_gemv_special_cases_vs_loops():
    rng = np.random.default_rng(8)
    wc = rng.standard_normal((12, 7))
    b = rng.standard_normal(7)
    x = rng.standard_normal(12)
    # k = D reduces to the dense GEMV, computed here by explicit loops
    loop = [b[o] + sum(x[j] * wc[j, o] for j in range(12)) for o in range(7)]
    assert np.allclose(O.sparse_gemv(wc, np.arange(12), x, b), loop, atol=1e-13)
    assert np.array_equal(O.sparse_gemv(wc, np.arange(0), np.zeros(0), b), b)      # k = 0
    assert np.allclose(O.sparse_gemv(wc, [5], [2.5]), 2.5 * wc[5], atol=0)        # k = 1


# ------------------------------------------------------------------ Theorem A.1
@pytest.mark.parametrize("ex", WE["normal"])
def test_normal_functions_worked(ex):
    if ex["fn"] == "inv_cdf":
        assert abs(O.std_normal_inv_cdf(ex["u"]) - ex["value"]) <= ex["tol"]
    else:
        assert abs(O.std_normal_pdf(ex["t"]) - ex["value"]) <= ex["tol"]


def test_inv_cdf_vs_scipy():
    for u in np.linspace(1e-6, 1 - 1e-6, 501):
        assert abs(O.std_normal_inv_cdf(u) - norm.ppf(u)) < 1e-8
        assert abs(O.std_normal_cdf(O.std_normal_inv_cdf(u)) - u) < 1e-12


@pytest.mark.parametrize("ex", WE["theorem_a1"])
def test_theorem_worked(ex):
    d = 4096
    k = int(round(ex["keep"] * d))
    assert abs(O.theory_relative_error(k, d) - ex["value"]) <= ex["tol"], ex["cite"]


def test_theorem_monotone():
    v = [O.theory_relative_error(k, 100) for k in range(101)]
    assert all(a >= b for a, b in zip(v, v[1:]))


def test_theorem_matches_monte_carlo_topk():
    """The relative error of the oracle's real Top-K on i.i.d. Gaussian x~, W~ matches
    Theorem A.1 within 2% at D = 4096.  A wrong selection (e.g. k
    random entries: sqrt(1-k/D)) or a dropped term fails by > 2x."""
    d, dout, n = 4096, 256, 400
    g = np.random.default_rng(12)
    w = g.standard_normal((d, dout))
    x = g.standard_normal((n, d))
    y = x @ w
    for keep in (0.25, 0.5, 0.75):
        k = int(keep * d)
        ys = np.stack([O.sparse_gemv(w, s, x[i][s]) for i in range(n) for s in [O.topk(x[i], k)]])
        num = np.mean(np.linalg.norm(y - ys, axis=1))
        den = np.mean(np.linalg.norm(y, axis=1))
        th = O.theory_relative_error(k, d)
        assert abs(num / den - th) / th < 0.02, (keep, num / den, th)
        rms = math.sqrt(np.mean(np.sum((y - ys) ** 2, 1)) / np.mean(np.sum(y ** 2, 1)))
        assert abs(rms - th) / th < 0.02


# ------------------------------------------------------------------ glue: RoPE / attention
def test_rope_closed_forms():
    v = np.array([1.0, 0.0])                         # hd = 2: a plain 2-D rotation by pos rad
    assert np.allclose(O.rope(v, 1, 10000.0), [math.cos(1), math.sin(1)], atol=1e-15)
    rng = np.random.default_rng(1)
    u = rng.standard_normal(16)
    assert np.array_equal(O.rope(u, 0, 1e4), u)
    assert np.allclose(O.rope(O.rope(u, 3, 1e4), 4, 1e4), O.rope(u, 7, 1e4), atol=1e-12)
    assert abs(np.linalg.norm(O.rope(u, 9, 1e4)) - np.linalg.norm(u)) < 1e-12


def test_attention_special_cases():
    rng = np.random.default_rng(2)
    q = rng.standard_normal((4, 8))
    kc = rng.standard_normal((2, 5, 8))
    vc = rng.standard_normal((2, 5, 8))
    out = O.decode_attention(q, kc, vc, 1).reshape(4, 8)
    assert np.allclose(out[0], vc[0, 0]) and np.allclose(out[1], vc[0, 0])   # GQA: heads 0,1 -> kv 0
    assert np.allclose(out[2], vc[1, 0]) and np.allclose(out[3], vc[1, 0])
    kc2 = np.repeat(kc[:, :1], 5, axis=1)                                      # equal keys -> mean of v
    out2 = O.decode_attention(q, kc2, vc, 5).reshape(4, 8)
    assert np.allclose(out2[3], vc[1].mean(0), atol=1e-14)


# ------------------------------------------------------------------ block invariance (O-8)
def _toy_layer(seed, d=64, inter=128, hq=4, hkv=2, hd=16, bias=False):
    rng = np.random.default_rng(seed)
    w = {
        "wq": rng.standard_normal((d, hq * hd)) / math.sqrt(d),
        "wk": rng.standard_normal((d, hkv * hd)) / math.sqrt(d),
        "wv": rng.standard_normal((d, hkv * hd)) / math.sqrt(d),
        "wo": rng.standard_normal((hq * hd, d)) / math.sqrt(hq * hd),
        "wg": rng.standard_normal((d, inter)) / math.sqrt(d),
        "wu": rng.standard_normal((d, inter)) / math.sqrt(d),
        "wd": rng.standard_normal((inter, d)) / math.sqrt(inter),
        "gamma1": 1 + 0.1 * rng.standard_normal(d),
        "gamma2": 1 + 0.1 * rng.standard_normal(d),
    }
    if bias:
        for n, m in (("bq", hq), ("bk", hkv), ("bv", hkv)):
            w[n] = 0.02 * rng.standard_normal(m * hd)
    cfg = dict(hq=hq, hkv=hkv, hd=hd, eps=1e-6, theta=10000.0)
    return w, cfg


def _fold_layer(w, q_l, q_down=None):
    wqkv = np.concatenate([w["wq"], w["wk"], w["wv"]], axis=1)
    wf = {
        "wqkv": O.fold_left_qt(q_l, wqkv, w["gamma1"]),
        "wo": O.fold_right_q(w["wo"], q_l),
        "wg": O.fold_left_qt(q_l, w["wg"], w["gamma2"]),
        "wu": O.fold_left_qt(q_l, w["wu"], w["gamma2"]),
        "wd": O.fold_right_q(w["wd"], q_l if q_down is None else q_down),
    }
    if "bq" in w:
        wf["bqkv"] = np.concatenate([w["bq"], w["bk"], w["bv"]])
    return wf


@pytest.mark.parametrize("bias", [False, True])
def test_block_p0_equals_dense_two_layers(bias):
    """Computational invariance end to end (S:615 acceptance #1): two rotated
    folded layers with adapter A_0 = Q_0^T Q_1 at k = D reproduce the dense layers:
    r_out^larosa = r_out^dense Q_{l+1}, within 1e-10 relative in fp64."""
    d, ctx = 64, 6
    layers = [_toy_layer(100 + l, bias=bias) for l in range(2)]
    qs = [synth.haar_orthogonal(d, 200 + l).numpy() for l in range(3)]
    cfg = layers[0][1]
    rng = np.random.default_rng(7)
    caches_d = [[rng.standard_normal((2, ctx, 16)) for _ in range(2)] for _ in range(2)]
    caches_r = [[c.copy() for c in cc] for cc in caches_d]
    r = rng.standard_normal(d)
    rr = r @ qs[0]
    pos = ctx - 1
    full = (d, d, d, 128)
    for l in range(2):
        w = layers[l][0]
        r, _ = O.dense_block(r, w, cfg, caches_d[l][0], caches_d[l][1], pos)
        rr, _ = O.larosa_block(rr, _fold_layer(w, qs[l]), cfg, full, caches_r[l][0], caches_r[l][1], pos,
                               adapter=O.residual_adapter(qs[l], qs[l + 1]))
        assert np.linalg.norm(rr - r @ qs[l + 1]) <= 1e-10 * np.linalg.norm(r)
    # the rotated embedding/head folds cancel: r_L Q_L^T is the dense output
    assert np.allclose(rr @ qs[2].T, r, atol=1e-10 * np.linalg.norm(r))


@pytest.mark.parametrize("p", [0.0, 0.5])
def test_block_adapter_in_down_equals_adapter_form(p):
    """The adapter folded into the down projection (wd = Wd Q_{l+1}) equals the
    paper's literal form r_next = (r_mid + y_down) A_l (Z20) at any sparsity: the same
    index sets at every site and r_next within 1e-12 relative (fp64, linearity of A_l).  At
    p = 0 both reproduce the dense layer rotated into Q_{l+1}'s basis."""
    d, ctx = 64, 6
    w, cfg = _toy_layer(700, bias=True)
    q0, q1 = (synth.haar_orthogonal(d, 710 + i).numpy() for i in range(2))
    rng = np.random.default_rng(3)
    kc, vc = rng.standard_normal((2, ctx, 16)), rng.standard_normal((2, ctx, 16))
    r = rng.standard_normal(d) * (1 + 5 * (rng.random(d) < 0.05))
    ks = O.site_ks(p, (1, 1, 1, 1), d, 128)
    a = O.residual_adapter(q0, q1)
    lit, i_lit = O.larosa_block(r @ q0, _fold_layer(w, q0), cfg, ks, kc.copy(), vc.copy(), ctx - 1, adapter=a)
    mrg, i_mrg = O.larosa_block(r @ q0, _fold_layer(w, q0, q1), cfg, ks, kc.copy(), vc.copy(), ctx - 1, adapter=a,
                                adapter_in_down=True)
    for site in ("idx1", "idx2", "idx3", "idx4"):
        assert np.array_equal(i_lit[site], i_mrg[site])
    assert np.linalg.norm(mrg - lit) <= 1e-12 * np.linalg.norm(lit)
    if p == 0.0:
        ref, _ = O.dense_block(r, w, cfg, kc.copy(), vc.copy(), ctx - 1)
        assert np.linalg.norm(mrg - ref @ q1) <= 1e-10 * np.linalg.norm(ref)
    with pytest.raises(ValueError):
        O.larosa_block(r @ q0, _fold_layer(w, q0, q1), cfg, ks, kc.copy(), vc.copy(), ctx - 1, adapter_in_down=True)


@pytest.mark.parametrize("merged", [False, True])
def test_block_wise_rotation_qb_p0_equals_dense(merged):
    """Q_B (Table 6): the attention block in Q_a's basis, the MLP block in Q_m's,
    A_mid = Q_a^T Q_m folded beside O (wo = Wo Q_m, r_mid = r A_mid + y_o) and the closing
    adapter Q_m^T Q_a' (or wd = Wd Q_a' beside down).  At k = D two chained layers reproduce the
    dense layers rotated into the next layer's attention basis (computational invariance,
    P:1444-1448), to 1e-10 in fp64."""
    d, ctx = 64, 6
    layers = [_toy_layer(800 + l, bias=True) for l in range(2)]
    qa = [synth.haar_orthogonal(d, 810 + l).numpy() for l in range(3)]
    qm = [synth.haar_orthogonal(d, 820 + l).numpy() for l in range(2)]
    cfg = layers[0][1]
    rng = np.random.default_rng(8)
    caches_d = [[rng.standard_normal((2, ctx, 16)) for _ in range(2)] for _ in range(2)]
    caches_r = [[c.copy() for c in cc] for cc in caches_d]
    r = rng.standard_normal(d)
    rr = r @ qa[0]
    full = (d, d, d, 128)
    for l in range(2):
        w = layers[l][0]
        r, _ = O.dense_block(r, w, cfg, caches_d[l][0], caches_d[l][1], ctx - 1)
        wqkv = np.concatenate([w["wq"], w["wk"], w["wv"]], axis=1)
        wf = {"wqkv": O.fold_left_qt(qa[l], wqkv, w["gamma1"]), "wo": O.fold_right_q(w["wo"], qm[l]),
              "wg": O.fold_left_qt(qm[l], w["wg"], w["gamma2"]), "wu": O.fold_left_qt(qm[l], w["wu"], w["gamma2"]),
              "wd": O.fold_right_q(w["wd"], qa[l + 1] if merged else qm[l]),
              "bqkv": np.concatenate([w["bq"], w["bk"], w["bv"]])}
        rr, _ = O.larosa_block(rr, wf, cfg, full, caches_r[l][0], caches_r[l][1], ctx - 1,
                               adapter=O.residual_adapter(qm[l], qa[l + 1]), adapter_in_down=merged,
                               adapter_mid=O.residual_adapter(qa[l], qm[l]))
        assert np.linalg.norm(rr - r @ qa[l + 1]) <= 1e-10 * np.linalg.norm(r)


def test_block_exact_sparsity_and_monotone_error():
    """Per-site kept counts are exactly k for every token and the mean relative
    output error is non-decreasing in p over 5 seeds."""
    d = 64
    errs = {p: [] for p in (0.0, 0.25, 0.5, 0.75)}
    for seed in range(5):
        w, cfg = _toy_layer(300 + seed)
        q = synth.haar_orthogonal(d, 400 + seed).numpy()
        wf = _fold_layer(w, q)
        rng = np.random.default_rng(seed)
        kc = rng.standard_normal((2, 8, 16))
        vc = rng.standard_normal((2, 8, 16))
        for tok in range(4):
            r = rng.standard_normal(d) * (1 + 5 * (rng.random(d) < 0.05))
            ref, _ = O.dense_block(r, w, cfg, kc.copy(), vc.copy(), 7)
            for p in errs:
                ks = O.site_ks(p, (1, 1, 1, 1), d, 128)
                out, inter = O.larosa_block(r @ q, wf, cfg, ks, kc.copy(), vc.copy(), 7)
                for site, kk in zip(("idx1", "idx2", "idx3", "idx4"), ks):
                    assert len(inter[site]) == kk
                errs[p].append(np.linalg.norm(out @ q.T - ref) / np.linalg.norm(ref))
    means = [np.mean(errs[p]) for p in sorted(errs)]
    assert means[0] < 1e-12
    assert all(a <= b for a, b in zip(means, means[1:])), means


def test_greedy_lowest_index_on_ties():
    assert O.greedy([1.0, 3.0, 3.0, 2.0]) == 1
    assert O.greedy([-5.0, -1.0, -1.0]) == 1
    rng = np.random.default_rng(0)
    for _ in range(50):
        v = rng.integers(-3, 4, 17).astype(np.float64)
        best = max(range(17), key=lambda i: (v[i], -i))        # brute force: max value, lowest index
        assert O.greedy(v) == best


def test_decode_step_p0_equals_dense_model():
    """a7 end to end at k = D: embedding E' = E Q_0, two folded layers
    (adapter A_0 = Q_0^T Q_1, the last layer's basis folded into the head
    H' = Q_1^T diag(gamma_f) H) reproduce the dense model's logits within 1e-10 relative and
    pick the same greedy token."""
    d, ctx, vocab = 64, 6, 50
    layers = [_toy_layer(500 + l) for l in range(2)]
    cfg = layers[0][1]
    qs = [synth.haar_orthogonal(d, 600 + l).numpy() for l in range(2)]
    rng = np.random.default_rng(11)
    E = rng.standard_normal((vocab, d))
    H = rng.standard_normal((d, vocab)) / math.sqrt(d)
    gf = 1 + 0.1 * rng.standard_normal(d)
    caches_d = [[rng.standard_normal((2, ctx, 16)) for _ in range(2)] for _ in range(2)]
    caches_r = [[c.copy() for c in cc] for cc in caches_d]
    pos, tok = ctx - 1, 17
    # dense reference
    r = E[tok].copy()
    for l in range(2):
        r, _ = O.dense_block(r, layers[l][0], cfg, caches_d[l][0], caches_d[l][1], pos)
    ref_logits = O.dense_gemv(H, O.rmsnorm(r, gf, cfg["eps"]))
    # LaRoSA model on folded weights
    folded = [(_fold_layer(layers[0][0], qs[0]), O.residual_adapter(qs[0], qs[1])),
              (_fold_layer(layers[1][0], qs[1]), None)]
    e_f = E @ qs[0]
    h_f = O.fold_left_qt(qs[1], H, gf)
    nxt, logits, _ = O.larosa_decode_step(tok, e_f, folded, cfg, (d, d, d, 128), caches_r, pos, h_f, cfg["eps"])
    assert np.linalg.norm(logits - ref_logits) <= 1e-10 * np.linalg.norm(ref_logits)
    assert nxt == int(np.argmax(ref_logits))


# ------------------------------------------------------------------ W4A16 (N3)
def test_w4_worked_example_and_error_bound():
    """A hand-computed group (bf16(0.7) = 0.69921875 = max |w|; 0.69921875 / 7 = 0.09988839...
    -> nearest fp16 1637 * 2^-14 = 0.09991455078125 (vs 1636 * 2^-14); w / s rounded half-to-even) and the quantisation bound |w - deq| <= s / 2 on random groups
    (interior codes), codes in [0, 15], an all-zero group -> scale 0, codes 8, deq 0."""
    row = np.zeros((1, 128), dtype=np.float32)
    row[0, :6] = [0.7, -0.35, 0.05, -0.7, 0.25, 0.0]
    q, sb = O.quantize_w4(O.f64_to_bf16_rne(row))
    s = float(np.uint16(sb[0, 0]).view(np.float16))
    assert s == 0.09991455078125
    wb = O.bf16_to_f64(O.f64_to_bf16_rne(row))[0]
    # by hand: 0.69921875/s = 6.998 -> 7; -0.349609375/s = -3.499 -> -3; 0.0500488/s = 0.5009
    # -> 1 (above the midpoint); 0.25/s = 2.5021 -> 3
    assert list(q[0, :6].astype(int) - 8) == [7, -3, 1, -7, 3, 0]
    assert np.all(q[0, 6:] == 8)
    zq, zs = O.quantize_w4(np.zeros((1, 256), dtype=np.uint16))
    assert np.all(zq == 8) and np.all(zs == 0) and np.all(O.dequantize_w4(zq, zs) == 0)
    rng = np.random.default_rng(0)
    w = O.f64_to_bf16_rne(rng.standard_normal((8, 512)).astype(np.float32) * 0.02)
    q, sb = O.quantize_w4(w)
    assert q.max() <= 15 and q.min() >= 0
    deq = O.dequantize_w4(q, sb)
    wf = O.bf16_to_f64(w)
    sc = np.repeat(sb.view(np.float16).astype(np.float64), 128, axis=1)
    assert np.all(np.abs(wf - deq) <= sc / 2 * (1 + 1e-3) + 1e-12)


# ------------------------------------------------------------------ glue pins with hand-computed values
# (VERDICT r1 "What's weak" 1: the closed forms above hold for ANY RoPE frequency schedule or pairing,
#  and softmax special cases are scale-invariant; these fix the Z27 conventions numerically.)
def test_rope_hand_values_hd8():
    """Z27 (HF rotate_half): pairs (i, i + hd/2), inv_freq_i = theta^(-2i/hd).  With hd = 8 and
    theta = 10^4 the frequencies are exactly 1, 0.1, 0.01, 0.001, so at pos = 3 basis vector e_i
    (i < 4) rotates by 3*10^-i rad into coordinate i + 4, and e_{i+4} into -sin at i.  An
    interleaved pairing (2i, 2i+1) or the schedule theta^(-i/hd) fails this."""
    hd, pos, theta = 8, 3, 1e4
    for i, ang in enumerate((3.0, 0.3, 0.03, 0.003)):
        e = np.zeros(hd); e[i] = 1.0
        want = np.zeros(hd); want[i] = math.cos(ang); want[i + 4] = math.sin(ang)
        assert np.allclose(O.rope(e, pos, theta), want, atol=1e-15, rtol=0), i
        e2 = np.zeros(hd); e2[i + 4] = 1.0
        want2 = np.zeros(hd); want2[i] = -math.sin(ang); want2[i + 4] = math.cos(ang)
        assert np.allclose(O.rope(e2, pos, theta), want2, atol=1e-15, rtol=0), i


def test_rope_hand_values_hd4():
    """hd = 4, theta = 100: inv_freq = (1, 100^(-1/2) = 0.1); pos = 2 -> angles (2, 0.2).
    v = (1, 2, 3, 4): out = (1 c2 - 3 s2, 2 c.2 - 4 s.2, 3 c2 + 1 s2, 4 c.2 + 2 s.2)."""
    c2, s2, c02, s02 = math.cos(2.0), math.sin(2.0), math.cos(0.2), math.sin(0.2)
    want = [1 * c2 - 3 * s2, 2 * c02 - 4 * s02, 3 * c2 + 1 * s2, 4 * c02 + 2 * s02]
    assert np.allclose(O.rope(np.array([1.0, 2.0, 3.0, 4.0]), 2, 100.0), want, atol=1e-14, rtol=0)


@pytest.mark.parametrize("hd", [4, 16])
def test_attention_scale_hand_values(hd):
    """Two cached positions, k_0 = 0 and k_1 = c * ones(hd) with c = ln(3) / sqrt(hd), query ones:
    the scores are (0, ln 3) only with the 1/sqrt(hd) scale (Z27), so the softmax weights are
    exactly (1/4, 3/4) and the output is 1/4 v_0 + 3/4 v_1.  Without the scale the weights would
    be (1, 3^sqrt(hd)) / (1 + 3^sqrt(hd)); with 1/hd, (1, 3^(1/sqrt(hd)))/(...)."""
    c = math.log(3.0) / math.sqrt(hd)
    q = np.ones((1, hd))
    kc = np.zeros((1, 2, hd)); kc[0, 1] = c
    vc = np.zeros((1, 2, hd)); vc[0, 0, 0] = 1.0; vc[0, 1, 1] = 1.0
    out = O.decode_attention(q, kc, vc, 2)
    want = np.zeros(hd); want[0] = 0.25; want[1] = 0.75
    assert np.allclose(out, want, atol=1e-14, rtol=0)
    # causal: ctx_len = 1 ignores position 1 entirely
    assert np.allclose(O.decode_attention(q, kc, vc, 1), vc[0, 0], atol=0)


def test_silu_closed_forms():
    """SiLU(x) = x * sigma(x): sigma(+-ln 3) = 3/4, 1/4 exactly, sigma(0) = 1/2; large |x| -> x, 0."""
    ln3 = math.log(3.0)
    got = O.silu(np.array([0.0, ln3, -ln3, 2 * math.log(2.0), 60.0, -60.0]))
    want = [0.0, 0.75 * ln3, -0.25 * ln3, 2 * math.log(2.0) * 0.8, 60.0, -60.0 * math.exp(-60.0)]
    assert np.allclose(got, want, rtol=1e-14, atol=1e-300)


def _wiring_layer():
    """A hand-built d = 8 layer (hq = 2, hkv = 1, hd = 4, inter = 8, eps = 0, pos = 0 so RoPE is
    the identity and the attention over one cached position returns v).  Rows a correct Top-K
    never keeps are filled with 100-1000, so a wrong kept set anywhere changes the output by
    orders of magnitude.  The expected kept sets and vectors are derived by hand in
    test_block_site_wiring_hand_built."""
    d = 8
    e = np.eye(d)
    wqkv = np.zeros((d, 16))                       # q cols 0-7 and k cols 8-11 stay 0
    for j, c in ((0, 0), (1, 1), (4, 2), (5, 3)):
        wqkv[j, 12 + c] = 1.0                      # v_c <- kept value of row j
    for j in (2, 3, 6, 7):
        wqkv[j, 12:] = 100.0
    wo = np.full((d, d), 100.0)
    wo[0], wo[2], wo[4], wo[6] = e[0], -e[2], 0.5 * e[1], e[3]
    wg = np.full((d, d), 1000.0)
    wg[0] = [100, -100, 0, 0, 0, 0, 0, 0]          # x vals3[0]/s3 = 6   -> (600, -600) at 0, 1
    wg[2] = [0, 0, 200, 0, 0, 0, 0, 0]             # x 2.5 -> 500 at 2
    wg[4] = [0, 0, 0, -200, 0, 0, 0, 0]            # x -3  -> 600 at 3
    wg[5] = [0, 0, 0, 0, 300, -300, 300, 300]      # x 2   -> (600, -600, 600, 600) at 4-7
    wu = np.full((d, d), 1000.0)
    wu[0] = 1.0                                    # U = 6 everywhere ...
    wu[2] = [0, 0, 2, 0, 0, 0, 0, 0]               # ... + 5 at 2
    wu[4] = [0, 0, 0, 1, 0, 0, 0, 0]               # ... - 3 at 3
    wu[5] = [0, 0, 0, 0, 0.5, 0, -1, 0]            # ... + 1 at 4, - 2 at 6
    wd = np.full((d, d), 1e3)
    wd[0], wd[2], wd[4] = 0.01 * e[6], 0.01 * e[7], -0.01 * e[0]
    return {"wqkv": wqkv, "wo": wo, "wg": wg, "wu": wu, "wd": wd}


@pytest.mark.parametrize("in_down", [False, True])
def test_block_site_wiring_hand_built(in_down):
    """p > 0 site wiring of larosa_block (Fig. 2; eqs.; Z10, Z25, Z20):
    every kept set and intermediate below is derived by hand.

      r = (4,-1,1,1,-3,2,0,0): mean r^2 = 4 -> s1 = 1/2; |r| top-4 with the lower index winning
          the three-way tie at |1| -> S1 = {0,1,4,5}; vals1 = r[S1] s1 = (2,-0.5,-1.5,1) = v
      h2 = (v, v) (both q heads read kv head 0) -> top-4 of |h2| = (2,.5,1.5,1,2,.5,1.5,1):
          S2 = {0,2,4,6}, vals2 = (2,-1.5,2,-1.5) (no RMS scale at h2)
      y_o = (2, 1, 1.5, -1.5, 0...) -> r_mid = (6,0,2.5,-0.5,-3,2,0,0); S3 = {0,2,4,5}
          (top-4 of |r_mid|: 6, 3, 2.5, 2; taking it on r instead gives {0,1,4,5}),
          s3 = 1/sqrt(55.5/8), vals3 = s3 (6, 2.5, -3, 2)
      g = s3 (600,-600,500,600,600,-600,600,600): SiLU(g) = g where g > 0 and ~0 where g < 0
          (|g| > 200); u = s3 (6,6,11,3,7,6,4,6); h4 = s3^2 (3600,0,5500,1800,4200,0,2400,3600)
      k4 = 3: S4 = {0,2,4} (3600 at 0 and 7 tie: the lower index wins), vals4 = h4[S4]
      y_down = s3^2 (-42,0,0,0,0,0,36,55); r_out = r_mid + y_down; r_next = r_out A."""
    w = _wiring_layer()
    cfg = dict(hq=2, hkv=1, hd=4, eps=0.0, theta=10000.0)
    r = np.array([4.0, -1, 1, 1, -3, 2, 0, 0])
    a = np.zeros((8, 8))
    for i, (j, sg) in enumerate(zip((7, 6, 5, 4, 3, 2, 1, 0), (1, -1, 1, 1, -1, 1, -1, 1))):
        a[i, j] = sg                                   # a signed permutation: orthogonal
    wf = dict(w)
    if in_down:
        wf["wd"] = w["wd"] @ a
    kc, vc = np.zeros((1, 2, 4)), np.zeros((1, 2, 4))
    out, inter = O.larosa_block(r, wf, cfg, (4, 4, 4, 3), kc, vc, 0, adapter=a, adapter_in_down=in_down)
    assert list(inter["idx1"]) == [0, 1, 4, 5]
    assert list(inter["idx2"]) == [0, 2, 4, 6]
    assert list(inter["idx3"]) == [0, 2, 4, 5]
    assert list(inter["idx4"]) == [0, 2, 4]
    assert np.array_equal(vc[0, 0], [2.0, -0.5, -1.5, 1.0]) and np.all(kc == 0)
    assert np.array_equal(inter["h2"], [2.0, -0.5, -1.5, 1.0] * 2)
    assert np.array_equal(inter["r_mid"], [6.0, 0, 2.5, -0.5, -3, 2, 0, 0])
    s3sq = 8.0 / 55.5
    h4 = s3sq * np.array([3600.0, 0, 5500, 1800, 4200, 0, 2400, 3600])
    assert np.allclose(inter["h4"], h4, rtol=1e-13, atol=1e-12)
    r_out = np.array([6.0, 0, 2.5, -0.5, -3, 2, 0, 0]) + s3sq * np.array([-42.0, 0, 0, 0, 0, 0, 36, 55])
    assert np.allclose(out, r_out @ a, rtol=1e-13, atol=1e-13)


def test_build_rotation_lapack_equals_jacobi():
    """build_rotation_lapack (LAPACK eigh as the eigendecomposition step) equals the Jacobi
    build_rotation on distinct-eigenvalue covariances (same order and sign rule, Z7)."""
    for d, seed in ((8, 1), (48, 2)):
        seqs = synth.toy_calibration(d=d, n_seq=8, n_tok=16, seed=seed)
        C = O.covariance([s.numpy() for s in seqs])
        q1, l1 = O.build_rotation(C)
        q2, l2 = O.build_rotation_lapack(C)
        assert np.max(np.abs(l1 - l2)) <= 1e-12 * l1[0]
        assert np.max(np.abs(q1 - q2)) <= 1e-9
