"""GPU parity of the row-sharded layer phases (larosa_sparse_layer_shard_phase)
by single-GPU emulation of n ranks in lockstep (each phase runs for every virtual rank, then
the shards are concatenated in rank order -- what all_gather_into_tensor does over NCCL).
Every phase output of every rank is checked against the oracle phase on the same gathered
GPU inputs (P6 style, 1e-5 of the norm), and the final residual against the unsharded GPU
layer (P5 style: equal index sets -> 1e-4)."""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from paper_2507_01299_b200 import larosa as LZ
from paper_2507_01299_b200 import model as M

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
SMALL_MHA = synth.ModelShape("small-mha", 512, 1024, 4, 4, 128, 2, 256, True, 1e-5, 10000.0)


def w64(bits):
    return O.bf16_to_f64(bits.detach().cpu().numpy().view(np.uint16))


def f64(t):
    return t.detach().cpu().numpy().astype(np.float64)


def rel_max(got, ref):
    return float(np.max(np.abs(got - ref)) / max(np.linalg.norm(ref), 1e-300))


def unpack_gu(wgu):
    d = wgu.shape[0]
    blk = wgu.reshape(d, -1, 2, LZ.LAROSA_GU_BLOCK)
    return blk[:, :, 0, :].reshape(d, -1), blk[:, :, 1, :].reshape(d, -1)


@pytest.mark.parametrize("world,p,merged", [(1, 0.5, False), (2, 0.5, False), (4, 0.4, False), (1, 0.5, True),
                                            (2, 0.5, True), (4, 0.4, True)])
def test_shard_phases_emulated(world, p, merged):
    """merged: the adapter folded beside down (4 phases / 4 all-gathers)."""
    shape = SMALL_MHA
    orig = M.synth_original_layer(shape, 21, device=DEV)
    q_l = synth.haar_orthogonal(shape.d, 31, device=DEV, dtype=torch.float32)
    q_n = synth.haar_orthogonal(shape.d, 32, device=DEV, dtype=torch.float32)
    lw = M.fold_layer(orig, shape, q_l, q_n, adapter_in_down=merged)
    plan = M.site_plan(shape, p)
    max_ctx, pos = 32, 20
    kc = synth.gaussian_bf16((1, shape.hkv, max_ctx, shape.hd), 41, 1.0, DEV)
    vc = synth.gaussian_bf16((1, shape.hkv, max_ctx, shape.hd), 42, 1.0, DEV)
    r0 = synth.residual_activation(1, shape.d, 43).to(DEV)
    posd = torch.tensor([pos], dtype=torch.int32, device=DEV)
    # unsharded reference run
    ref_state = LZ.LayerState(r0.clone(), kc.clone(), vc.clone(), posd)
    LZ.sparse_layer(lw, plan, ref_state)
    # emulated ranks
    ranks = [M.ShardedLayer(M.shard_layer(lw, r, world), r, world, max_ctx, DEV) for r in range(world)]
    kvs = [(M.shard_kv(kc, r, world), M.shard_kv(vc, r, world)) for r in range(world)]
    r_full = r0[0].clone()
    last = ranks[0].n_phases() - 1
    cfg_eps, hd = shape.rms_eps, shape.hd
    for ph in range(last + 1):
        outs = []
        for rk, (kcr, vcr) in zip(ranks, kvs):
            x, res = rk.inputs(ph, r_full)
            x_np, res_np = f64(x), (f64(res) if res is not None else None)
            kc_before = O.bf16_to_f64(kcr[0].cpu().numpy().view(np.uint16))
            vc_before = O.bf16_to_f64(vcr[0].cpu().numpy().view(np.uint16))
            out = rk.run_phase(ph, x, res, kcr, vcr, posd, plan)
            torch.cuda.synchronize()
            # oracle phase on the same inputs
            w = rk.w
            k1, k2, k3, k4 = plan
            n = world
            dl = shape.d // n
            if ph == 0:
                s = O.topk(x_np, k1)
                y = O.sparse_gemv(w64(w.w_qkv), s, x_np[s] * O.rms_scale(x_np, cfg_eps),
                                  w64(w.b_qkv) if w.b_qkv is not None else None)
                hq, hkv = shape.hq // n, shape.hkv // n
                qh = np.stack([O.rope(y[h * hd:(h + 1) * hd], pos, shape.rope_theta) for h in range(hq)])
                kn = np.stack([O.rope(y[(hq + h) * hd:(hq + h + 1) * hd], pos, shape.rope_theta) for h in range(hkv)])
                vn = y[(hq + hkv) * hd:].reshape(hkv, hd)
                kc_before[:, pos] = O.bf16_to_f64(O.f64_to_bf16_rne(kn))
                vc_before[:, pos] = O.bf16_to_f64(O.f64_to_bf16_rne(vn))
                ref = O.decode_attention(qh, kc_before, vc_before, pos + 1)
                tol = 1e-4       # q goes through RoPE and the bf16 KV append before attention
            elif ph == 1:
                s = O.topk(x_np, k2)
                ref = res_np[rk.rank * dl:(rk.rank + 1) * dl] + O.sparse_gemv(w64(w.w_o), s, x_np[s])
                tol = 1e-5
            elif ph == 2:
                s = O.topk(x_np, k3)
                wg, wu = unpack_gu(w64(w.w_gu))
                v = x_np[s] * O.rms_scale(x_np, cfg_eps)
                ref = O.silu(O.sparse_gemv(wg, s, v)) * O.sparse_gemv(wu, s, v)
                tol = 1e-5
            elif ph == 3 and merged:   # r_next cols = r_mid A_l[:, cols] + h4[S4] (Wd Q_{l+1})[:, cols]
                s = O.topk(x_np, k4)
                ref = O.dense_gemv(w64(w.adapter), res_np) + O.sparse_gemv(w64(w.w_down), s, x_np[s])
                tol = 1e-5
            elif ph == 3:
                s = O.topk(x_np, k4)
                ref = res_np[rk.rank * dl:(rk.rank + 1) * dl] + O.sparse_gemv(w64(w.w_down), s, x_np[s])
                tol = 1e-5
            else:
                ref = O.dense_gemv(w64(w.adapter), x_np)
                tol = 1e-5
            assert rel_max(f64(out), ref) <= tol, (ph, rk.rank)
            outs.append(out.clone())
        gathered = torch.cat(outs)
        if ph == last:
            r_full.copy_(gathered)
        else:
            ranks[0].full[ph].copy_(gathered)
            for rk in ranks[1:]:
                rk.full[ph].copy_(gathered)
    got, ref = f64(r_full), f64(ref_state.resid[0])
    assert rel_max(got, ref) <= 1e-4
