"""Host logic of the row-sharded multi-GPU layer, on CPU with a real gloo
process group (world size 2): every rank takes its shard with model.shard_layer, computes
each of the five phases on it with the fp64 ORACLE primitives (the same phase contract as
larosa_sparse_layer_shard_phase), and all-gathers the phase outputs with
torch.distributed.all_gather_into_tensor.  The gathered result must equal the unsharded
oracle layer bit for bit: the column partition (heads, d/n, packed gate|up blocks), the
phase inputs and the rank-major gather order are what is under test."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth
from paper_2507_01299_b200 import larosa as LZ
from paper_2507_01299_b200 import model as M

D, INTER, HQ, HKV, HD, CTX = 128, 256, 4, 2, 16, 6
B_GU = LZ.LAROSA_GU_BLOCK


def pack_gu(wg, wu):
    d, inter = wg.shape
    return np.stack([wg.reshape(d, inter // B_GU, B_GU), wu.reshape(d, inter // B_GU, B_GU)], axis=2).reshape(d, -1)


def unpack_gu(wgu):
    d = wgu.shape[0]
    blk = wgu.reshape(d, -1, 2, B_GU)
    return blk[:, :, 0, :].reshape(d, -1), blk[:, :, 1, :].reshape(d, -1)


def toy(seed):
    rng = np.random.default_rng(seed)
    nq, nk = HQ * HD, HKV * HD
    w = {"wqkv": rng.standard_normal((D, nq + 2 * nk)) / math.sqrt(D),
         "bqkv": 0.02 * rng.standard_normal(nq + 2 * nk),
         "wo": rng.standard_normal((nq, D)) / math.sqrt(nq),
         "wg": rng.standard_normal((D, INTER)) / math.sqrt(D),
         "wu": rng.standard_normal((D, INTER)) / math.sqrt(D),
         "wd": rng.standard_normal((INTER, D)) / math.sqrt(INTER),
         "adapter": synth.haar_orthogonal(D, seed + 1).numpy()}
    kc = rng.standard_normal((HKV, CTX, HD))
    vc = rng.standard_normal((HKV, CTX, HD))
    r = rng.standard_normal(D)
    return w, kc, vc, r


def layer_weights(w, merged=False):
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))   # noqa: E731
    return LZ.LayerWeights(w_qkv=t(w["wqkv"]), w_o=t(w["wo"]), w_gu=t(pack_gu(w["wg"], w["wu"])), w_down=t(w["wd"]),
                           d=D, inter=INTER, n_q_heads=HQ, n_kv_heads=HKV, head_dim=HD, rope_theta=10000.0,
                           rms_eps=1e-6, b_qkv=t(w["bqkv"]), adapter=t(w["adapter"]), adapter_in_down=merged)


def oracle_phase(ph, ws, plan, x, resid, kc, vc, pos, rank, world, merged=False):
    """The phase contract of larosa_sparse_layer_shard_phase, computed with oracle primitives."""
    k1, k2, k3, k4 = plan
    n = lambda t: t.numpy()   # noqa: E731
    dl = D // world
    if ph == 0:
        s = O.topk(x, k1)
        y = O.sparse_gemv(n(ws.w_qkv), s, x[s] * O.rms_scale(x, 1e-6), n(ws.b_qkv))
        hq, hkv = HQ // world, HKV // world
        q = y[:hq * HD].reshape(hq, HD)
        k = y[hq * HD:(hq + hkv) * HD].reshape(hkv, HD)
        v = y[(hq + hkv) * HD:].reshape(hkv, HD)
        q = np.stack([O.rope(q[h], pos, 10000.0) for h in range(hq)])
        k = np.stack([O.rope(k[h], pos, 10000.0) for h in range(hkv)])
        kc[:, pos] = k
        vc[:, pos] = v
        return O.decode_attention(q, kc, vc, pos + 1)
    if ph == 1:
        s = O.topk(x, k2)
        return resid[rank * dl:(rank + 1) * dl] + O.sparse_gemv(n(ws.w_o), s, x[s])
    if ph == 2:
        s = O.topk(x, k3)
        wg, wu = unpack_gu(n(ws.w_gu))
        v = x[s] * O.rms_scale(x, 1e-6)
        return O.silu(O.sparse_gemv(wg, s, v)) * O.sparse_gemv(wu, s, v)
    if ph == 3 and merged:   # adapter folded beside down: r_next cols = r_mid A[:, cols] + y_down cols
        s = O.topk(x, k4)
        return O.rotate(resid, n(ws.adapter)) + O.sparse_gemv(n(ws.w_down), s, x[s])
    if ph == 3:
        s = O.topk(x, k4)
        return resid[rank * dl:(rank + 1) * dl] + O.sparse_gemv(n(ws.w_down), s, x[s])
    return O.dense_gemv(n(ws.adapter), x)


def worker(rank, world, port, q, merged=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, kc, vc, r = toy(5)
        plan = O.site_ks(0.5, (1, 1, 1, 1), D, INTER)
        plan = (plan[0], O.compute_k(1.0, 0.5, HQ * HD), plan[2], plan[3])
        ws = M.shard_layer(layer_weights(w, merged), rank, world)
        hk = HKV // world
        kc_l, vc_l = kc[rank * hk:(rank + 1) * hk].copy(), vc[rank * hk:(rank + 1) * hk].copy()
        pos = CTX - 1
        full = {}
        x = r.copy()
        for ph in range(4 if merged else 5):
            xin = {0: r, 1: full.get(0), 2: full.get(1), 3: full.get(2), 4: full.get(3)}[ph]
            res = {1: r, 3: full.get(1)}.get(ph)
            out = torch.from_numpy(oracle_phase(ph, ws, plan, xin, res, kc_l, vc_l, pos, rank, world, merged))
            g = torch.empty(out.numel() * world, dtype=out.dtype)
            dist.all_gather_into_tensor(g, out)
            full[ph] = g.numpy()
        # unsharded reference
        wf = {"wqkv": w["wqkv"], "bqkv": w["bqkv"], "wo": w["wo"], "wg": w["wg"], "wu": w["wu"], "wd": w["wd"]}
        cfg = dict(hq=HQ, hkv=HKV, hd=HD, eps=1e-6, theta=10000.0)
        ref, inter = O.larosa_block(r, wf, cfg, plan, kc.copy(), vc.copy(), pos, adapter=w["adapter"],
                                    adapter_in_down=merged)
        last = full[3] if merged else full[4]
        ok = (np.array_equal(full[0], inter["h2"]) and np.array_equal(full[1], inter["r_mid"])
              and np.array_equal(full[2], inter["h4"]) and np.array_equal(last, ref)
              and (merged or np.array_equal(full[3], inter["r_out"])))
        q.put((rank, ok, float(np.max(np.abs(last - ref)))))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,merged", [(2, False), (2, True)])
def test_sharded_layer_gloo_equals_unsharded(world, merged):
    """merged: the adapter folded beside down -- 4 phases / 4 all-gathers."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q, merged)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res


def test_shard_layer_partition_covers_columns():
    """Concatenating the shards' columns in rank order rebuilds every projection (the gather
    order the phases rely on); q/k/v heads stay grouped per rank."""
    w, *_ = toy(9)
    lw = layer_weights(w)
    for world in (1, 2):
        sh = [M.shard_layer(lw, r, world) for r in range(world)]
        for name in ("w_o", "w_gu", "w_down", "adapter"):
            assert torch.equal(torch.cat([getattr(s, name) for s in sh], dim=1), getattr(lw, name))
        nq, nk = HQ * HD, HKV * HD
        ql, kl = nq // world, nk // world
        cat = torch.cat([s.w_qkv for s in sh], dim=1)
        q = torch.cat([cat[:, r * (ql + 2 * kl):r * (ql + 2 * kl) + ql] for r in range(world)], dim=1)
        assert torch.equal(q, lw.w_qkv[:, :nq])


def test_shard_inter_padding_is_exact():
    """model.shard_inter / pad_inter (larosa.h: an MLP width that is not a multiple of 64 n is
    zero-padded): Qwen2.5-72B's 29568 -> 29696 at n = 4 and 8, unchanged at n = 1, 2; the padded
    packed gate|up keeps every original column block in place and appends zero blocks; down gets
    zero rows; each rank's shard then holds exactly 2 inter_p / n gate|up columns."""
    assert M.shard_inter(29568, 1) == 29568 and M.shard_inter(29568, 2) == 29568
    assert M.shard_inter(29568, 4) == 29696 and M.shard_inter(29568, 8) == 29696
    assert M.shard_inter(28672, 8) == 28672 and M.shard_inter(14336, 8) == 14336
    w, *_ = toy(13)
    lw = layer_weights(w)
    inter_p = INTER + 2 * B_GU
    pw = M.pad_inter(lw, inter_p)
    assert pw.inter == inter_p
    assert torch.equal(pw.w_gu[:, :2 * INTER], lw.w_gu) and torch.all(pw.w_gu[:, 2 * INTER:] == 0)
    assert torch.equal(pw.w_down[:INTER], lw.w_down) and torch.all(pw.w_down[INTER:] == 0)
    g, u = unpack_gu(pw.w_gu.numpy())
    g0, u0 = unpack_gu(lw.w_gu.numpy())
    assert np.array_equal(g[:, :INTER], g0) and np.array_equal(u[:, :INTER], u0)
    # the padded layer computes the same function (oracle, p = 0.5): padded h4 entries are 0 and
    # never selected, the output is identical
    wf = {"wqkv": w["wqkv"], "bqkv": w["bqkv"], "wo": w["wo"], "wg": w["wg"], "wu": w["wu"], "wd": w["wd"]}
    wp = dict(wf, wg=g, wu=u, wd=pw.w_down.numpy())
    cfg = dict(hq=HQ, hkv=HKV, hd=HD, eps=1e-6, theta=10000.0)
    _, kc, vc, r = toy(13)
    plan = O.site_ks(0.5, (1, 1, 1, 1), D, INTER)
    a, ia = O.larosa_block(r, wf, cfg, plan, kc.copy(), vc.copy(), CTX - 1, adapter=w["adapter"])
    b, ib = O.larosa_block(r, wp, cfg, plan, kc.copy(), vc.copy(), CTX - 1, adapter=w["adapter"])
    assert np.array_equal(ia["idx4"], ib["idx4"]) and np.all(ib["h4"][INTER:] == 0)
    assert np.array_equal(a, b)


def worker_batch(rank, world, port, q):
    """Batch-2 phase outputs gathered rank-major [world][batch][local] and re-ordered to
    [batch][full] (the larosa_shard_gather_permute contract) reproduce the unsharded oracle layer
    for both tokens."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, kc, vc, r0 = toy(21)
        rng = np.random.default_rng(3)
        rs = [r0, rng.standard_normal(D)]
        plan = O.site_ks(0.4, (1, 1, 1, 1), D, INTER)
        plan = (plan[0], O.compute_k(1.0, 0.4, HQ * HD), plan[2], plan[3])
        ws = M.shard_layer(layer_weights(w, True), rank, world)
        hk = HKV // world
        pos = CTX - 1
        full = {}
        caches = [(kc[rank * hk:(rank + 1) * hk].copy(), vc[rank * hk:(rank + 1) * hk].copy()) for _ in rs]
        for ph in range(4):
            outs = []
            for b in range(2):
                xin = rs[b] if ph == 0 else full[ph - 1][b]
                res = {1: rs[b], 3: full.get(1, [None, None])[b]}.get(ph)
                outs.append(oracle_phase(ph, ws, plan, xin, res, *caches[b], pos, rank, world, True))
            out = torch.from_numpy(np.stack(outs))                     # [batch][local]
            g = torch.empty(out.numel() * world, dtype=out.dtype)
            dist.all_gather_into_tensor(g, out.reshape(-1))
            full[ph] = g.numpy().reshape(world, 2, -1).transpose(1, 0, 2).reshape(2, -1)   # permute
        wf = {"wqkv": w["wqkv"], "bqkv": w["bqkv"], "wo": w["wo"], "wg": w["wg"], "wu": w["wu"], "wd": w["wd"]}
        cfg = dict(hq=HQ, hkv=HKV, hd=HD, eps=1e-6, theta=10000.0)
        ok = True
        for b in range(2):
            ref, _ = O.larosa_block(rs[b], wf, cfg, plan, kc.copy(), vc.copy(), pos, adapter=w["adapter"],
                                    adapter_in_down=True)
            ok &= bool(np.max(np.abs(full[3][b] - ref)) <= 1e-12 * np.linalg.norm(ref))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_sharded_layer_gloo_batch2_gather_order():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker_batch, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_peer_space_layout():
    """P2P arena (model.PeerSpace): the same take() sequence gives the same offsets on every rank,
    so rank p's copy of a buffer is bases[p] + offset; targets point at this rank's column block;
    takes are 256-byte aligned and zeroed; an over-full arena raises."""
    import torch
    from paper_2507_01299_b200 import model as M
    world = 3
    spaces = M.PeerSpace.emulated(8192, "cpu", world)
    bufs = []
    for sp in spaces:
        sp.arena.fill_(7)
        a = sp.take((2, 10))
        f = sp.take((8,), torch.int32)
        b = sp.take((3, 5))
        bufs.append((a, f, b))
        assert (a == 0).all() and (f == 0).all()
    offs = [[t.data_ptr() - sp.arena.data_ptr() for t in bs] for sp, bs in zip(spaces, bufs)]
    assert all(o == offs[0] for o in offs) and offs[0] == [0, 256, 512]
    for r, sp in enumerate(spaces):
        a, f, b = bufs[r]
        tg = sp.target(a, col0=r * 3, flag=f[2:3])
        assert tg.ld == 10
        assert tg.dst.tolist() == [spaces[p].arena.data_ptr() + 4 * r * 3 for p in range(world)]
        assert tg.flag.tolist() == [spaces[p].arena.data_ptr() + 256 + 8 for p in range(world)]
    with pytest.raises(ValueError):
        spaces[0].take((4096,))
