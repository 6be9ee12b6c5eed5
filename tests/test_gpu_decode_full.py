"""Full-size parity of the decode step the bench times (BASELINE configs[2]: LLaMA3-8B, GQA
32/8 x 128, I = 14336, the full 128,256-token LM head), at batch 1 (fused SELECT GEMVs, companion
adapter rows) and batch 16 (tcgen05 THRESH GEMVs over the union, tcgen05 DENSE head), p = 0.4,
two chained layers with the adapter folded beside down (the bench's form):

  P6  every site of every layer, every token: the GPU's own site inputs fed to the oracle
      (tests/layer_check.py): kept sets bit-identical, outputs within 1e-5 of their norm;
      the LM head's logits against the oracle's lm_head on the GPU's final residual, and
      the greedy token on the GPU's own logits;
  P5  the oracle's independent chain (embedding -> 2 layers -> head) for sampled tokens: index
      sets equal at every site or a certified near-tie swap (tests/parity.py), logits 1e-4.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from layer_check import OracleWeights, f64, layer_sites, lm_head_chunked, p6_layer, rel_max, w64
from parity import walk_chain
from paper_2507_01299_b200 import larosa as LZ
from paper_2507_01299_b200 import model as M

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.mark.parametrize("batch", [1, 16])
def test_llama3_8b_decode_step_full_size(batch):
    shape = synth.MODELS["llama3-8b"]
    n_layers, max_ctx, ctx, p = 2, 256, 200, 0.4
    model = M.synth_decode_model(shape, n_layers, DEV, seed=3, adapter_in_down=True)
    run = M.DecodeRunner(model, batch, max_ctx, DEV)
    g = torch.Generator().manual_seed(11)
    kv0 = []
    for kc, vc in run.kv:
        a = synth.gaussian_bf16(kc.shape, int(torch.randint(0, 10 ** 6, (1,), generator=g)), 1.0)
        b = synth.gaussian_bf16(vc.shape, int(torch.randint(0, 10 ** 6, (1,), generator=g)), 1.0)
        kc.copy_(a)
        vc.copy_(b)
        kv0.append((a.numpy().view(np.uint16), b.numpy().view(np.uint16)))
    tokens = torch.randint(0, shape.vocab, (batch,), generator=g, dtype=torch.int32)
    pos = torch.randint(ctx // 2, ctx, (batch,), generator=g, dtype=torch.int32)   # ragged positions
    run.tokens.copy_(tokens)
    run.pos.copy_(pos)
    plan = M.site_plan(shape, p)
    taps = [LZ.make_taps(w, plan, batch, DEV) for w in model.layers]
    nxt = run.step(plan, taps=taps).cpu().numpy()
    torch.cuda.synchronize()
    logits_gpu = run.logits.cpu().numpy().astype(np.float64)
    r_final = run.resid.cpu().numpy().astype(np.float64)
    kv_gpu = [(kc.cpu().numpy().view(np.uint16), vc.cpu().numpy().view(np.uint16)) for kc, vc in run.kv]
    ows = [OracleWeights(w) for w in model.layers]
    # P6: every layer, every token, on the GPU's own inputs
    for l, ow in enumerate(ows):
        for b in range(batch):
            r_in = f64(taps[l]["r_in"][b])
            out_b = f64(taps[l + 1]["r_in"][b]) if l + 1 < n_layers else r_final[b]
            p6_layer(ow, shape, plan, taps[l], b, r_in, kv0[l][0][b], kv_gpu[l][0][b], kv_gpu[l][1][b], int(pos[b]),
                     out_b)
    # embedding row (exact widening) and the LM head on the GPU's final residual
    e_rows = w64(model.embed[tokens.long().to(DEV)])
    for b in range(batch):
        assert np.array_equal(f64(taps[0]["r_in"][b]), e_rows[b])
    sample = sorted({0, batch // 3, batch - 1})
    for b in sample:
        ref = lm_head_chunked(r_final[b], model.head, shape.rms_eps)
        assert rel_max(logits_gpu[b], ref) <= 1e-5
    for b in range(batch):
        assert int(nxt[b]) == O.greedy(logits_gpu[b])          # arg-max of the GPU's own logits: exact
    # P5: the oracle's independent chain for the sampled tokens
    wfs = [ow.wf() for ow in ows]
    cfg = dict(hq=shape.hq, hkv=shape.hkv, hd=shape.hd, eps=shape.rms_eps, theta=shape.rope_theta)
    for b in sample:
        r = O.embed(e_rows, b)
        sites = []
        for l, ow in enumerate(ows):
            kc = O.bf16_to_f64(kv0[l][0][b])
            vc = O.bf16_to_f64(kv0[l][1][b])
            r_in = r
            r, inter = O.larosa_block(r, wfs[l], cfg, plan, kc, vc, int(pos[b]), adapter=ow.adapter, kv_bf16=True,
                                      adapter_in_down=ow.merged)
            sites += layer_sites(taps[l], b, inter, r_in, f64(taps[l]["r_in"][b]), tag=f"token{b}.layer{l}.")
        swap = walk_chain(sites)
        if swap is not None:
            continue                                               # certified; chains diverge from here
        ref = lm_head_chunked(r, model.head, shape.rms_eps)
        assert rel_max(logits_gpu[b], ref) <= 1e-4
