"""GPU parity of the W4A16 decoder layer and decode step (larosa.h ABI 6):
larosa_sparse_layer with int4 weights at some or all of its four sites (batch 1: the fused
Top-K prologue of the bf16 path, then the int4 stream; either adapter form), site by site
against the oracle (P6, tests/layer_check.py).  The oracle quantises the folded bf16 weights
itself (O.quantize_w4, P:306-344 reading in DESIGN.md), the GPU codes and scales must equal its
codes bit for bit, and the oracle's dequantised matrices stand in for the bf16 ones."""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from layer_check import OracleWeights, f64, p6_layer, unpack_gu
from paper_2507_01299_b200 import larosa as LZ
from paper_2507_01299_b200 import model as M
from test_gpu_layer import SMALL, SMALL_MHA, build, run_layer

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def unpack_codes(Wq):
    b = Wq.cpu().numpy()
    q = np.empty((b.shape[0], b.shape[1] * 2), dtype=np.uint8)
    q[:, 0::2] = b & 15
    q[:, 1::2] = b >> 4
    return q


def oracle_weights_w4(lw4, inter):
    """OracleWeights of the layer with the oracle's own dequantised int4 matrices at the W4 sites
    (lw4 keeps its bf16 copies); the GPU codes/scales are checked equal to the oracle's."""
    ow = OracleWeights(lw4)
    for j, qs in enumerate(lw4.w4):
        if qs is None:
            continue
        q, s = O.quantize_w4(getattr(lw4, M.W4_SITES[j]).cpu().numpy().view(np.uint16))
        assert np.array_equal(unpack_codes(qs[0]), q), f"site {j} codes"
        assert np.array_equal(qs[1].cpu().numpy().view(np.uint16), s), f"site {j} scales"
        wd = O.dequantize_w4(q, s)
        if j == 0:
            ow.wqkv = wd
        elif j == 1:
            ow.wo = wd
        elif j == 2:
            ow.wg, ow.wu = unpack_gu(wd, inter)
        else:
            ow.wd = wd
    return ow


@pytest.mark.parametrize("shape,ctx,p,sites,adapter", [
    (SMALL, 7, 0.5, (0, 1, 2, 3), True), (SMALL_MHA, 40, 0.4, (0, 3), True), (SMALL, 20, 0.5, (1, 2), False),
    (synth.MODELS["llama3-8b"], 200, 0.4, (0, 1, 2, 3), True),
    (synth.MODELS["qwen2.5-7b"], 77, 0.25, (0, 1, 2, 3), True),   # QKV bias on the W4 QKV site
    (synth.MODELS["llama2-7b"], 256, 0.5, (2, 3), False),
    # adapter folded beside down (W4 codes of W_down Q_{l+1}, the adapter rows as bf16 companion CTAs)
    (SMALL, 9, 0.5, (0, 1, 2, 3), "merged"), (SMALL_MHA, 30, 0.25, (3,), "merged"),
    (synth.MODELS["llama3-8b"], 150, 0.4, (0, 1, 2, 3), "merged"),
    (synth.MODELS["mistral-7b"], 90, 0.6, (0, 1, 2, 3), "merged")])
def test_w4_layer_p6_sitewise(shape, ctx, p, sites, adapter):
    max_ctx = max(ctx, 64)
    _, _, _, lw, plan, resid, kc0, vc0, pos = build(shape, 13, 1, ctx, max_ctx, p, with_adapter=bool(adapter),
                                                    merged=adapter == "merged")
    lw4 = M.quantize_layer_w4(lw, sites)
    st, tp = run_layer(lw4, plan, resid, kc0, vc0, pos)
    ow = oracle_weights_w4(lw4, shape.inter)
    p6_layer(ow, shape, plan, tp, 0, resid[0].numpy().astype(np.float64), kc0[0].numpy().view(np.uint16),
             st.k_cache[0].cpu().numpy().view(np.uint16), st.v_cache[0].cpu().numpy().view(np.uint16), int(pos[0]),
             f64(st.resid[0]))
    # repeatable: the same inputs give the same bits
    st2, _ = run_layer(lw4, plan, resid, kc0, vc0, pos)
    assert torch.equal(st2.resid, st.resid)


def test_w4_layer_only_w4_weights():
    """The bf16 copies released (NULL w_* at W4 sites): the layer reads only the int4 weights."""
    shape = SMALL
    _, _, _, lw, plan, resid, kc0, vc0, pos = build(shape, 17, 1, 9, 64, 0.5)
    lw4 = M.quantize_layer_w4(lw)
    ref, _ = run_layer(lw4, plan, resid, kc0, vc0, pos)
    lw4d = M.quantize_layer_w4(lw, drop_bf16=True)
    assert lw4d.w_qkv is None and lw4d.w_down is None
    got, _ = run_layer(lw4d, plan, resid, kc0, vc0, pos)
    assert torch.equal(got.resid, ref.resid)


def test_w4_layer_rejections():
    shape = SMALL
    _, _, _, lw, plan, resid, kc0, vc0, pos = build(shape, 19, 2, 9, 64, 0.5)
    lw4 = M.quantize_layer_w4(lw, (0,))
    st = LZ.LayerState(resid.clone().to(DEV), kc0.clone().to(DEV), vc0.clone().to(DEV), pos.to(DEV))
    with pytest.raises(RuntimeError, match="W4 sites need batch 1"):
        LZ.sparse_layer(lw4, plan, st)


def test_w4_decode_step_llama3_8b():
    """Two chained W4 layers (adapter beside down) + the LM head (batch 1, the decode step of the W4
    bench extra):
    P6 at every site of both layers and the logits on the GPU's final residual."""
    shape = synth.MODELS["llama3-8b"]
    n_layers, max_ctx, ctx, p = 2, 256, 180, 0.4
    model = M.synth_decode_model(shape, n_layers, DEV, seed=5, vocab=32768, adapter_in_down=True)
    model.layers = [M.quantize_layer_w4(w) for w in model.layers]
    run = M.DecodeRunner(model, 1, max_ctx, DEV)
    g = torch.Generator().manual_seed(23)
    kv0 = []
    for kc, vc in run.kv:
        a = synth.gaussian_bf16(kc.shape, int(torch.randint(0, 10 ** 6, (1,), generator=g)), 1.0)
        b = synth.gaussian_bf16(vc.shape, int(torch.randint(0, 10 ** 6, (1,), generator=g)), 1.0)
        kc.copy_(a)
        vc.copy_(b)
        kv0.append(a.numpy().view(np.uint16))
    run.tokens.copy_(torch.tensor([1234], dtype=torch.int32))
    run.pos.copy_(torch.tensor([ctx - 1], dtype=torch.int32))
    plan = M.site_plan(shape, p)
    taps = [LZ.make_taps(w, plan, 1, DEV) for w in model.layers]
    nxt = run.step(plan, taps=taps).cpu().numpy()
    torch.cuda.synchronize()
    r_final = run.resid.cpu().numpy().astype(np.float64)
    for l, w in enumerate(model.layers):
        ow = oracle_weights_w4(w, shape.inter)
        r_in = f64(taps[l]["r_in"][0])
        out = f64(taps[l + 1]["r_in"][0]) if l + 1 < n_layers else r_final[0]
        kc, vc = run.kv[l]
        p6_layer(ow, shape, plan, taps[l], 0, r_in, kv0[l][0], kc[0].cpu().numpy().view(np.uint16),
                 vc[0].cpu().numpy().view(np.uint16), ctx - 1, out)
    logits = run.logits.cpu().numpy().astype(np.float64)[0]
    ref = O.lm_head(r_final[0], O.bf16_to_f64(model.head.cpu().numpy().view(np.uint16)), shape.rms_eps)
    assert np.max(np.abs(logits - ref)) <= 1e-5 * np.linalg.norm(ref)
    assert int(nxt[0]) == int(np.argmax(logits))


@pytest.mark.parametrize("merged", [False, True])
def test_w4_layer_edge_k(merged):
    """W4 sites at the edge counts (k = 0, 1, D - 1, D and the reverse), P6 against the oracle."""
    shape = SMALL
    nq = shape.hq * shape.hd
    for plan in ((0, 1, shape.d - 1, shape.inter), (shape.d, nq - 1, 1, 0)):
        _, _, _, lw, _, resid, kc0, vc0, pos = build(shape, 41, 1, 12, 64, 0.5, with_adapter=True, merged=merged)
        lw4 = M.quantize_layer_w4(lw)
        st, tp = run_layer(lw4, plan, resid, kc0, vc0, pos)
        ow = oracle_weights_w4(lw4, shape.inter)
        p6_layer(ow, shape, plan, tp, 0, resid[0].numpy().astype(np.float64), kc0[0].numpy().view(np.uint16),
                 st.k_cache[0].cpu().numpy().view(np.uint16), st.v_cache[0].cpu().numpy().view(np.uint16),
                 int(pos[0]), f64(st.resid[0]))
