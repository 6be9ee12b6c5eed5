"""GPU parity of the whole decode step: embed -> L LaRoSA layers -> final
RMS + LM head -> greedy token, against the oracle's larosa_decode_step run on the GPU's own
folded weights (independent chain, P5 protocol: index sets must agree at every site of every
layer unless a certified near-tie swaps them, then the test is skipped and reported)."""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from parity import walk_chain
from paper_2507_01299_b200 import larosa as LZ
from paper_2507_01299_b200 import model as M

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
SMALL = synth.ModelShape("small", 256, 512, 4, 2, 64, 3, 512, True, 1e-6, 10000.0)


def w64(bits):
    return O.bf16_to_f64(bits.detach().cpu().numpy().view(np.uint16))


def unpack_gu(wgu, inter):
    B = LZ.LAROSA_GU_BLOCK
    d = wgu.shape[0]
    blk = wgu.reshape(d, inter // B, 2, B)
    return blk[:, :, 0, :].reshape(d, inter), blk[:, :, 1, :].reshape(d, inter)


def f64(t):
    return t.detach().cpu().numpy().astype(np.float64)


def layer_sites(tp, b, inter, r_ref, tag=""):
    """One layer's four sites for the P5 walk (tests/parity.py); h1's GPU vector is the layer
    input the binding tapped (r_in)."""
    return [(f"{tag}h1", tp["idx_h1"][b].cpu().numpy(), inter["idx1"], f64(tp["r_in"][b]), r_ref),
            (f"{tag}h2", tp["idx_h2"][b].cpu().numpy(), inter["idx2"], f64(tp["h2"][b]), inter["h2"]),
            (f"{tag}h3", tp["idx_h3"][b].cpu().numpy(), inter["idx3"], f64(tp["r_mid"][b]), inter["r_mid"]),
            (f"{tag}h4", tp["idx_h4"][b].cpu().numpy(), inter["idx4"], f64(tp["h4"][b]), inter["h4"])]


def oracle_layers(model):
    out = []
    for w in model.layers:
        wf = {"wqkv": w64(w.w_qkv), "wo": w64(w.w_o), "wd": w64(w.w_down)}
        wf["wg"], wf["wu"] = unpack_gu(w64(w.w_gu), w.inter)
        if w.b_qkv is not None:
            wf["bqkv"] = w64(w.b_qkv)
        out.append((wf, w64(w.adapter) if w.adapter is not None else None, bool(w.adapter_in_down)))
    return out


@pytest.mark.parametrize("batch,p,merged", [(1, 0.5, False), (3, 0.4, False), (16, 0.5, False), (1, 0.5, True),
                                            (3, 0.4, True), (16, 0.5, True)])
def test_decode_step_vs_oracle(batch, p, merged):
    shape = SMALL
    model = M.synth_decode_model(shape, shape.layers, DEV, seed=1, adapter_in_down=merged)
    max_ctx, ctx = 32, 9
    run = M.DecodeRunner(model, batch, max_ctx, DEV)
    g = torch.Generator().manual_seed(3)
    kvs0 = []
    for kc, vc in run.kv:
        a = synth.gaussian_bf16(kc.shape, int(torch.randint(0, 10 ** 6, (1,), generator=g)), 1.0)
        b = synth.gaussian_bf16(vc.shape, int(torch.randint(0, 10 ** 6, (1,), generator=g)), 1.0)
        kc.copy_(a)
        vc.copy_(b)
        kvs0.append((a, b))
    tokens = torch.randint(0, shape.vocab, (batch,), generator=g, dtype=torch.int32)
    pos = torch.full((batch,), ctx - 1, dtype=torch.int32)
    run.tokens.copy_(tokens)
    run.pos.copy_(pos)
    plan = M.site_plan(shape, p)
    taps = [LZ.make_taps(w, plan, batch, DEV) for w in model.layers]
    nxt = run.step(plan, taps=taps).cpu().numpy()
    torch.cuda.synchronize()
    e_f, h_f = w64(model.embed), w64(model.head)
    layers = oracle_layers(model)
    cfg = dict(hq=shape.hq, hkv=shape.hkv, hd=shape.hd, eps=shape.rms_eps, theta=shape.rope_theta)
    logits_gpu = run.logits.cpu().numpy().astype(np.float64)
    for b in range(batch):
        caches = [(O.bf16_to_f64(a[b].numpy().view(np.uint16)), O.bf16_to_f64(c[b].numpy().view(np.uint16)))
                  for a, c in kvs0]
        # oracle chain, layer by layer, checking index sets against the GPU taps
        r = O.embed(e_f, int(tokens[b]))
        sites = []
        for l, ((wf, adp, mrg), (kc, vc)) in enumerate(zip(layers, caches)):
            r_in = r
            r, inter = O.larosa_block(r, wf, cfg, plan, kc, vc, int(pos[b]), adapter=adp, kv_bf16=True,
                                      adapter_in_down=mrg)
            sites += layer_sites(taps[l], b, inter, r_in, tag=f"layer{l}.")
        swap = walk_chain(sites)
        if swap is not None:
            pytest.skip(f"certified near-tie swap at {swap} (P5, reported)")
        logits = O.lm_head(r, h_f, shape.rms_eps)
        err = np.max(np.abs(logits_gpu[b] - logits)) / np.linalg.norm(logits)
        assert err <= 1e-4, err
        assert int(nxt[b]) == O.greedy(logits_gpu[b])      # arg-max on the GPU's own logits: exact
        top2 = np.sort(logits)[-2:]
        if top2[1] - top2[0] > 1e-3 * np.abs(top2).max():   # unambiguous -> the same token
            assert int(nxt[b]) == O.greedy(logits)


def test_embed_and_argmax_exact():
    vocab, d = 1000, 256
    E = synth.gaussian_bf16((vocab, d), 5, 1.0).to(DEV)
    tok = torch.tensor([0, 999, 17, 17], dtype=torch.int32, device=DEV)
    r = LZ.embed(E, tok)
    assert torch.equal(r.cpu(), torch.from_numpy(w64(E)[tok.cpu().numpy()].astype(np.float32)))
    # argmax with ties: lowest index wins
    H = torch.zeros((d, 64), dtype=torch.bfloat16)
    H[:, 5] = 1.0
    H[:, 9] = 1.0
    Hb = H.view(torch.int16).contiguous().to(DEV)
    x = torch.ones((2, d), device=DEV)
    nt, lg = LZ.lm_head(x, Hb, 1e-6, logits=torch.empty((2, 64), device=DEV))
    assert nt.cpu().tolist() == [5, 5]
