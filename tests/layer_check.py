"""Site-wise (P6) parity of one GPU layer run against the oracle: every
site's GPU input vector, read from the layer taps, is fed to the oracle; Top-K index lists must
be bit-identical (P1) and the GEMV / glue outputs within 1e-5 of their norm (north_star's bound
is 1e-3).  Shared by the layer and decode-step tests; comparisons only."""
import numpy as np

import oracle as O

TOL = 1e-5


def w64(bits):
    return O.bf16_to_f64(bits.detach().cpu().numpy().view(np.uint16))


def f64(t):
    return t.detach().cpu().numpy().astype(np.float64)


def bf16_ulp(x):
    """Spacing of the bf16 grid at |x| (8 significant bits)."""
    _, e = np.frexp(np.abs(x))
    return np.ldexp(1.0, e - 8)


def rel_max(got, ref):
    return float(np.max(np.abs(got - ref)) / max(np.linalg.norm(ref), 1e-300))


def unpack_gu(wgu, inter, block=64):
    """Inverse of larosa_pack_gate_up's documented layout (include/larosa.h)."""
    d = wgu.shape[0]
    blk = wgu.reshape(d, inter // block, 2, block)
    return blk[:, :, 0, :].reshape(d, inter), blk[:, :, 1, :].reshape(d, inter)


class OracleWeights:
    """fp64 views of one folded layer's bf16 weights (widened exactly)."""

    def __init__(self, lw):
        self.wqkv, self.wo, self.wd = w64(lw.w_qkv), w64(lw.w_o), w64(lw.w_down)
        self.wg, self.wu = unpack_gu(w64(lw.w_gu), lw.inter)
        self.bqkv = w64(lw.b_qkv) if lw.b_qkv is not None else None
        self.adapter = w64(lw.adapter) if lw.adapter is not None else None
        self.adapter_mid = w64(lw.adapter_mid) if getattr(lw, "adapter_mid", None) is not None else None
        self.merged = bool(lw.adapter_in_down)

    def wf(self):
        d = {"wqkv": self.wqkv, "wo": self.wo, "wd": self.wd, "wg": self.wg, "wu": self.wu}
        if self.bqkv is not None:
            d["bqkv"] = self.bqkv
        return d


def p6_layer(ow, shape, plan, tp, b, r, kc0_b, kc_gpu_b, vc_gpu_b, pos_b, out_gpu_b):
    """P6 for token b of one layer.  r: the layer input (fp64); kc0_b: the token's K cache
    before the step (uint16 bits [Hkv][max_ctx][hd]); kc_gpu_b / vc_gpu_b: after the step;
    out_gpu_b: the layer's output residual (fp64)."""
    k1, k2, k3, k4 = plan
    hq, hkv, hd = shape.hq, shape.hkv, shape.hd
    nq = hq * hd
    # h1
    i1 = tp["idx_h1"][b].cpu().numpy()
    assert np.array_equal(i1, O.topk(r, k1)), "h1 Top-K"
    assert np.allclose(f64(tp["vals_h1"][b]), r[i1] * O.rms_scale(r, shape.rms_eps), rtol=2e-6)
    y = O.sparse_gemv(ow.wqkv, i1, f64(tp["vals_h1"][b]), ow.bqkv)
    q = np.concatenate([O.rope(y[h * hd:(h + 1) * hd], pos_b, shape.rope_theta) for h in range(hq)])
    assert rel_max(f64(tp["q"][b]), q) <= TOL, "q"
    kn = np.concatenate([O.rope(y[nq + h * hd: nq + (h + 1) * hd], pos_b, shape.rope_theta) for h in range(hkv)])
    vn = y[nq + hkv * hd:]
    kg = O.bf16_to_f64(kc_gpu_b[:, pos_b, :]).reshape(-1)
    vg = O.bf16_to_f64(vc_gpu_b[:, pos_b, :]).reshape(-1)
    # bf16 storage of the new k/v: within one bf16 ulp of the exact value (the GPU rounds its
    # fp32 result, whose ~1e-7 relative error may cross a rounding midpoint)
    assert np.all(np.abs(kg - kn) <= bf16_ulp(kn) + 1e-6 * np.linalg.norm(kn)), "k append"
    assert np.all(np.abs(vg - vn) <= bf16_ulp(vn) + 1e-6 * np.linalg.norm(vn)), "v append"
    assert np.array_equal(np.delete(kc_gpu_b, pos_b, axis=1), np.delete(kc0_b, pos_b, axis=1)), "cache untouched"
    h2 = O.decode_attention(f64(tp["q"][b]).reshape(hq, hd), O.bf16_to_f64(kc_gpu_b), O.bf16_to_f64(vc_gpu_b),
                            pos_b + 1)
    assert rel_max(f64(tp["h2"][b]), h2) <= TOL, "attention"
    # h2 -> O
    h2g = f64(tp["h2"][b])
    i2 = tp["idx_h2"][b].cpu().numpy()
    assert np.array_equal(i2, O.topk(h2g, k2)), "h2 Top-K"
    assert np.array_equal(f64(tp["vals_h2"][b]), h2g[i2])
    rbase = O.rotate(r, ow.adapter_mid) if ow.adapter_mid is not None else r
    rmid = rbase + O.sparse_gemv(ow.wo, i2, h2g[i2])
    assert rel_max(f64(tp["r_mid"][b]), rmid) <= TOL, "r_mid"
    # h3 -> gate|up
    rm = f64(tp["r_mid"][b])
    i3 = tp["idx_h3"][b].cpu().numpy()
    assert np.array_equal(i3, O.topk(rm, k3)), "h3 Top-K"
    v3 = f64(tp["vals_h3"][b])
    assert np.allclose(v3, rm[i3] * O.rms_scale(rm, shape.rms_eps), rtol=2e-6)
    h4 = O.silu(O.sparse_gemv(ow.wg, i3, v3)) * O.sparse_gemv(ow.wu, i3, v3)
    assert rel_max(f64(tp["h4"][b]), h4) <= TOL, "h4"
    # h4 -> down (+ adapter)
    h4g = f64(tp["h4"][b])
    i4 = tp["idx_h4"][b].cpu().numpy()
    assert np.array_equal(i4, O.topk(h4g, k4)), "h4 Top-K"
    if ow.merged:   # r_next = r_mid A_l + h4[S4] (Wd Q_{l+1}) in one accumulator
        rn = O.rotate(rm, ow.adapter) + O.sparse_gemv(ow.wd, i4, h4g[i4])
        assert rel_max(out_gpu_b, rn) <= TOL, "r_next (adapter beside down)"
        return
    rout = rm + O.sparse_gemv(ow.wd, i4, h4g[i4])
    assert rel_max(f64(tp["r_out"][b]), rout) <= TOL, "r_out"
    if ow.adapter is None:
        assert rel_max(out_gpu_b, f64(tp["r_out"][b])) <= 0.0 + 1e-12, "no adapter: output = r_out"
        return
    rn = O.rotate(f64(tp["r_out"][b]), ow.adapter)
    assert rel_max(out_gpu_b, rn) <= TOL, "adapter"


def layer_sites(tp, b, inter, r_ref, r_gpu, tag=""):
    """One layer's four sites for the P5 walk (tests/parity.py)."""
    return [(f"{tag}h1", tp["idx_h1"][b].cpu().numpy(), inter["idx1"], r_gpu, r_ref),
            (f"{tag}h2", tp["idx_h2"][b].cpu().numpy(), inter["idx2"], f64(tp["h2"][b]), inter["h2"]),
            (f"{tag}h3", tp["idx_h3"][b].cpu().numpy(), inter["idx3"], f64(tp["r_mid"][b]), inter["r_mid"]),
            (f"{tag}h4", tp["idx_h4"][b].cpu().numpy(), inter["idx4"], f64(tp["h4"][b]), inter["h4"])]


def lm_head_chunked(r, h_bits, eps, chunk=16384):
    """The oracle's lm_head (O: logits = (r s) H') evaluated over column blocks of the folded
    head, so the fp64 copy of a 128k-vocab head never exists at once (same sums per column)."""
    v = h_bits.shape[1]
    out = np.empty(v)
    for c0 in range(0, v, chunk):
        out[c0:c0 + chunk] = O.lm_head(r, w64(h_bits[:, c0:c0 + chunk]), eps)
    return out
