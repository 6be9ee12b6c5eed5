"""Model assembly for the LaRoSA decode path: synthetic random-init layers of the paper's
model shapes, folded with the library's own fold (SURVEY §3.1 offline transform), and a
whole-model decode runner (embedding -> layers -> LM head) driven through the C ABI.

Everything computed here runs in liblarosa kernels; torch only allocates, draws the
seeded random weights (synth) and moves tensors.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch

import synth
from . import larosa as LZ


@dataclass
class OriginalLayer:
    """Unrotated layer weights, Wc layout ([d_in][d_out]) bf16 bits (int16)."""
    wqkv: torch.Tensor     # [d][(hq + 2 hkv) hd]  = [Wq | Wk | Wv]
    wo: torch.Tensor       # [hq hd][d]
    wg: torch.Tensor       # [d][inter]
    wu: torch.Tensor       # [d][inter]
    wd: torch.Tensor       # [inter][d]
    gamma1: torch.Tensor   # fp32 [d]  attention RMSNorm gain
    gamma2: torch.Tensor   # fp32 [d]  MLP RMSNorm gain
    bqkv: Optional[torch.Tensor] = None   # bf16 bits [(hq + 2 hkv) hd]


def synth_original_layer(shape: synth.ModelShape, seed: int, device="cpu") -> OriginalLayer:
    """W ~ N(0, 1/D_in) -> bf16, gains 1 + N(0, 0.1^2), QKV bias N(0, 0.02^2)."""
    d, inter, nq = shape.d, shape.inter, shape.hq * shape.hd
    s = 1000 * seed
    return OriginalLayer(
        wqkv=synth.gaussian_bf16((d, shape.qkv_out), s + 1, d ** -0.5, device),
        wo=synth.gaussian_bf16((nq, d), s + 2, nq ** -0.5, device),
        wg=synth.gaussian_bf16((d, inter), s + 3, d ** -0.5, device),
        wu=synth.gaussian_bf16((d, inter), s + 4, d ** -0.5, device),
        wd=synth.gaussian_bf16((inter, d), s + 5, inter ** -0.5, device),
        gamma1=1.0 + 0.1 * synth.gaussian((d,), s + 6, device=device),
        gamma2=1.0 + 0.1 * synth.gaussian((d,), s + 7, device=device),
        bqkv=synth.gaussian_bf16((shape.qkv_out,), s + 8, 0.02, device) if shape.qkv_bias else None,
    )


def fold_layer(orig: OriginalLayer, shape: synth.ModelShape, q_l: torch.Tensor,
               q_next: Optional[torch.Tensor], adapter_in_down: bool = False,
               q_mlp: Optional[torch.Tensor] = None) -> LZ.LayerWeights:
    """Offline transform of one layer (eqs. before/after_merge P:402-410, §3.2):
    W_qkv' = Q_l^T diag(g1) W_qkv;  W_o' = W_o Q_l;  W_gate|up' = Q_l^T diag(g2) [Wg | Wu]
    (packed);  W_down' = W_down Q_l;  A_l = Q_l^T Q_{l+1} (larosa_residual_adapter: both
    fp32 factors split hi + lo, one bf16 rounding).   q_l, q_next: fp32 on device.
    adapter_in_down (needs q_next): W_down' = W_down Q_{l+1} = (W_down Q_l) A_l, and the
    layer computes r_next = r_mid A_l + y_down (larosa.h).
    q_mlp (block-wise rotation Q_B, Table 6): the MLP block runs in q_mlp's basis: W_o' = W_o Q_m,
    W_gate|up' = Q_m^T diag(g2) [Wg | Wu], A_mid = Q_l^T Q_m, and down / the adapter close from
    Q_m (A = Q_m^T Q_{l+1}, or W_down' = W_down Q_{l+1} beside down)."""
    dev = orig.wqkv.device
    L, R = LZ.LAROSA_LEFT_QT, LZ.LAROSA_RIGHT_Q
    g1 = orig.gamma1.to(dev, torch.float32).contiguous()
    g2 = orig.gamma2.to(dev, torch.float32).contiguous()
    w_qkv = LZ.fold_rotation(q_l, orig.wqkv, L, gamma=g1)
    q_m = q_mlp if q_mlp is not None else q_l
    w_o = LZ.fold_rotation(q_m, orig.wo, R)
    wg = LZ.fold_rotation(q_m, orig.wg, L, gamma=g2)
    wu = LZ.fold_rotation(q_m, orig.wu, L, gamma=g2)
    w_gu = LZ.pack_gate_up(wg, wu)
    del wg, wu
    merged = adapter_in_down and q_next is not None
    w_down = LZ.fold_rotation(q_next if merged else q_m, orig.wd, R)
    adapter = None
    if q_next is not None:
        adapter = LZ.residual_adapter(q_m, q_next)
    adapter_mid = None
    if q_mlp is not None:
        adapter_mid = LZ.residual_adapter(q_l, q_mlp)
    return LZ.LayerWeights(w_qkv=w_qkv, w_o=w_o, w_gu=w_gu, w_down=w_down, d=shape.d, inter=shape.inter,
                           n_q_heads=shape.hq, n_kv_heads=shape.hkv, head_dim=shape.hd,
                           rope_theta=shape.rope_theta, rms_eps=shape.rms_eps,
                           b_qkv=orig.bqkv.contiguous() if orig.bqkv is not None else None, adapter=adapter,
                           adapter_in_down=merged, adapter_mid=adapter_mid)


W4_SITES = ("w_qkv", "w_o", "w_gu", "w_down")


def quantize_layer_w4(lw: LZ.LayerWeights, sites=(0, 1, 2, 3), drop_bf16: bool = False) -> LZ.LayerWeights:
    """The layer with W4A16 weights (larosa_quantize_w4 of the folded bf16 weights) at the given
    sites (0 QKV, 1 O, 2 gate|up, 3 down): the folded weights as they are (with
    adapter_in_down the down weight is W_down Q_{l+1}); drop_bf16 releases the bf16 copies."""
    w4 = [LZ.quantize_w4(getattr(lw, W4_SITES[j])) if j in sites else None for j in range(4)]
    kw = {W4_SITES[j]: None for j in sites} if drop_bf16 else {}
    return dataclasses.replace(lw, w4=w4, **kw)


def site_plan(shape: synth.ModelShape, p: float, alpha_mode: str = "uniform") -> tuple:
    """Per-site kept counts (k_h1, k_h2, k_h3, k_h4) via larosa_compute_k with
    uniform alpha or the paper's App. B coefficients (alpha2/alpha4 from the constraints)."""
    if alpha_mode == "uniform":
        a = (1.0, 1.0, 1.0, 1.0)
    else:
        a1, a3 = synth.PAPER_ALPHA[shape.name]
        a2, a4 = LZ.solve_alpha(a1, a3, shape.inter / shape.d)
        a = (a1, a2, a3, a4)
    nq = shape.hq * shape.hd
    return (LZ.compute_k(a[0], p, shape.d), LZ.compute_k(a[1], p, nq), LZ.compute_k(a[2], p, shape.d),
            LZ.compute_k(a[3], p, shape.inter))


@dataclass
class DecodeModel:
    """A whole LaRoSA model for decoding: folded embedding E' = E Q_0,
    L folded layers (layer l's adapter A_l = Q_l^T Q_{l+1}; the last layer has none), and the
    folded head H' = Q_{L-1}^T diag(gamma_f) H."""
    shape: synth.ModelShape
    embed: torch.Tensor            # bf16 bits [vocab, d]
    layers: List[LZ.LayerWeights]
    head: torch.Tensor             # bf16 bits [d, vocab]


def synth_decode_model(shape: synth.ModelShape, n_layers: int, device, seed: int = 0,
                       vocab: Optional[int] = None, adapter_in_down: bool = False, w4: bool = False) -> DecodeModel:
    """Random-init model of the given shape (synthetic weights), folded with
    the library's own tensor-core fold; w4: every layer's four sites as W4A16 weights (the bf16
    copies released)."""
    vocab = vocab or shape.vocab
    d = shape.d
    qs = [synth.haar_orthogonal(d, 7000 + 100 * seed + l, device=device, dtype=torch.float32)
          for l in range(n_layers)]
    E = synth.gaussian_bf16((vocab, d), 9000 + seed, 1.0, device)
    e_f = LZ.fold_rotation(qs[0], E, LZ.LAROSA_RIGHT_Q)
    del E
    layers = []
    for l in range(n_layers):
        orig = synth_original_layer(shape, 10 * seed + l + 1, device=device)
        lw = fold_layer(orig, shape, qs[l], qs[l + 1] if l + 1 < n_layers else None,
                        adapter_in_down=adapter_in_down)
        layers.append(quantize_layer_w4(lw, drop_bf16=True) if w4 else lw)
        del lw
        del orig
    H = synth.gaussian_bf16((d, vocab), 9100 + seed, d ** -0.5, device)
    gf = (1.0 + 0.1 * synth.gaussian((d,), 9200 + seed, device=device)).float().contiguous()
    h_f = LZ.fold_rotation(qs[-1], H, LZ.LAROSA_LEFT_QT, gamma=gf)
    del H
    return DecodeModel(shape=shape, embed=e_f, layers=layers, head=h_f)


class DecodeRunner:
    """Runs decode steps of a DecodeModel through the C ABI: embed -> larosa_sparse_layer per
    layer (batch 1: layers after the first reuse the previous layer's selection data) ->
    larosa_lm_head (greedy).  All buffers are preallocated so a step is CUDA-graph capturable."""

    def __init__(self, model: DecodeModel, batch: int, max_ctx: int, device):
        self.m = model
        self.batch = batch
        self.max_ctx = max_ctx
        s = model.shape
        w0 = model.layers[0]
        self.ws = torch.zeros(LZ.layer_workspace_size(w0, batch, max_ctx), dtype=torch.uint8, device=device)
        self.kv = [(torch.zeros((batch, w.n_kv_heads, max_ctx, w.head_dim), dtype=torch.int16, device=device),
                    torch.zeros((batch, w.n_kv_heads, max_ctx, w.head_dim), dtype=torch.int16, device=device))
                   for w in model.layers]
        self.resid = torch.zeros((batch, s.d), dtype=torch.float32, device=device)
        self.tokens = torch.zeros((batch,), dtype=torch.int32, device=device)
        self.next_tokens = torch.zeros((batch,), dtype=torch.int32, device=device)
        self.pos = torch.zeros((batch,), dtype=torch.int32, device=device)
        vocab = model.head.shape[1]
        self.logits = torch.zeros((batch, vocab), dtype=torch.float32, device=device)
        self.head_ws = torch.zeros(LZ.lib().larosa_lm_head_workspace_size(batch, s.d, vocab), dtype=torch.uint8,
                                   device=device)

    def step(self, plan: Sequence[int], taps: Optional[List[dict]] = None, stream=None):
        """One token for every sequence: reads self.tokens / self.pos, writes self.next_tokens
        and self.logits (and the KV caches at pos)."""
        LZ.embed(self.m.embed, self.tokens, out=self.resid, stream=stream)
        for l, (w, (kc, vc)) in enumerate(zip(self.m.layers, self.kv)):
            st = LZ.LayerState(self.resid, kc, vc, self.pos, chained=l > 0)
            LZ.sparse_layer(w, plan, st, taps=taps[l] if taps else None, ws=self.ws, stream=stream)
        LZ.lm_head(self.resid, self.m.head, self.m.shape.rms_eps, logits=self.logits, next_token=self.next_tokens,
                   ws=self.head_ws, stream=stream)
        return self.next_tokens


# ------------------------------------------------------------------------------- multi-GPU
def shard_inter(inter: int, world: int) -> int:
    """The MLP width a world-size-n shard uses: inter rounded up to a multiple of 64 n (the
    gate|up interleave block per rank).  Qwen2.5-72B: 29568 -> 29696 at n = 4, 8 (larosa.h)."""
    q = LZ.LAROSA_GU_BLOCK * world
    return (inter + q - 1) // q * q


def pad_inter(w: LZ.LayerWeights, inter_p: int) -> LZ.LayerWeights:
    """Zero-pad the MLP width to inter_p: extra zero gate|up column blocks (SiLU(0) * 0 = 0, so the
    padded h4 entries are exactly 0) and zero down rows (never selected while k_h4 <= the true
    width: a real entry beats a padded 0, the lower index winning ties).  Same function."""
    if inter_p == w.inter:
        return w
    extra = inter_p - w.inter
    gu = torch.cat([w.w_gu, torch.zeros((w.d, 2 * extra), dtype=w.w_gu.dtype, device=w.w_gu.device)], dim=1)
    dn = torch.cat([w.w_down, torch.zeros((extra, w.w_down.shape[1]), dtype=w.w_down.dtype, device=w.w_down.device)])
    return LZ.LayerWeights(**{**w.__dict__, "w_gu": gu.contiguous(), "w_down": dn.contiguous(), "inter": inter_p})


def shard_layer(w: LZ.LayerWeights, rank: int, world: int) -> LZ.LayerWeights:
    """This rank's output columns of every projection (SURVEY §8(e) partitioning; offline data
    layout, like loading a checkpoint shard): q heads [r Hq/n, (r+1) Hq/n) with the matching
    kv heads, d/n columns of W_o / W_down / adapter, the same inter/n range of gate and up (a
    contiguous column range of the packed W_gate|up).  Dims stay the full model's; an MLP width
    that is not a multiple of 64 n is zero-padded first (pad_inter)."""
    w = pad_inter(w, shard_inter(w.inter, world))
    n, hd = world, w.head_dim
    nq, nk = w.n_q_heads * hd, w.n_kv_heads * hd
    ql, kl = nq // n, nk // n
    dl, il = w.d // n, w.inter // n

    def cols(t, a, b):
        return t[..., a:b].contiguous() if t is not None else None

    def qkv(t):
        if t is None:
            return None
        return torch.cat([t[..., rank * ql:(rank + 1) * ql], t[..., nq + rank * kl:nq + (rank + 1) * kl],
                          t[..., nq + nk + rank * kl:nq + nk + (rank + 1) * kl]], dim=-1).contiguous()

    return LZ.LayerWeights(w_qkv=qkv(w.w_qkv), w_o=cols(w.w_o, rank * dl, (rank + 1) * dl),
                           w_gu=cols(w.w_gu, rank * 2 * il, (rank + 1) * 2 * il),
                           w_down=cols(w.w_down, rank * dl, (rank + 1) * dl), d=w.d, inter=w.inter,
                           n_q_heads=w.n_q_heads, n_kv_heads=w.n_kv_heads, head_dim=hd, rope_theta=w.rope_theta,
                           rms_eps=w.rms_eps, b_qkv=qkv(w.b_qkv),
                           adapter=cols(w.adapter, rank * dl, (rank + 1) * dl), adapter_in_down=w.adapter_in_down)


def shard_kv(cache: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """This rank's kv heads of a [B][Hkv][ctx][hd] cache."""
    h = cache.shape[1] // world
    return cache[:, rank * h:(rank + 1) * h].contiguous()


class PeerSpace:
    """The buffer arena of the P2P push: every rank carves the same layout from
    its arena, so a buffer's offset names it on every rank; bases[p] = rank p's arena address.  On a
    multi-GPU run the arena is torch symmetric memory (``PeerSpace.symmetric``: peer addresses mapped
    over NVLink); the single-GPU lockstep emulation uses one ordinary arena per emulated rank
    (``PeerSpace.emulated``)."""

    ALIGN = 256

    def __init__(self, arena: torch.Tensor, bases: Sequence[int], rank: int):
        self.arena, self.bases, self.rank, self.off = arena, [int(b) for b in bases], rank, 0
        self.world = len(self.bases)

    def take(self, shape, dtype=torch.float32) -> torch.Tensor:
        """A zeroed view of the next free bytes (the same offset on every rank for the same calls)."""
        n = int(np.prod(shape)) * torch.tensor([], dtype=dtype).element_size()
        if self.off + n > self.arena.numel():
            raise ValueError("PeerSpace: arena too small")
        t = self.arena[self.off:self.off + n].view(dtype).view(*shape)
        t.zero_()
        self.off += (n + self.ALIGN - 1) // self.ALIGN * self.ALIGN
        return t

    def addr(self, t: torch.Tensor, rank: int) -> int:
        return self.bases[rank] + (t.data_ptr() - self.arena.data_ptr())

    def target(self, buf: torch.Tensor, col0: int, flag: torch.Tensor) -> LZ.PeerTarget:
        """Push into every rank's copy of buf [batch][full] at column col0, counted on flag."""
        dev = self.arena.device
        dst = torch.tensor([self.addr(buf, p) + 4 * col0 for p in range(self.world)], dtype=torch.int64, device=dev)
        fl = torch.tensor([self.addr(flag, p) for p in range(self.world)], dtype=torch.int64, device=dev)
        return LZ.PeerTarget(dst, fl, buf.shape[-1])

    @staticmethod
    def symmetric(nbytes: int, device, group=None) -> "PeerSpace":
        """A torch symmetric-memory arena, rendezvous over `group` (collective: every rank calls it)."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        arena = symm_mem.empty(nbytes, dtype=torch.uint8, device=device)
        hdl = symm_mem.rendezvous(arena, group if group is not None else dist.group.WORLD)
        return PeerSpace(arena, list(hdl.buffer_ptrs), hdl.rank)

    @staticmethod
    def emulated(nbytes: int, device, world: int) -> List["PeerSpace"]:
        arenas = [torch.zeros(nbytes, dtype=torch.uint8, device=device) for _ in range(world)]
        bases = [a.data_ptr() for a in arenas]
        return [PeerSpace(a, bases, r) for r, a in enumerate(arenas)]


def shard_layer_peer_bytes(shape_d: int, nq: int, inter_p: int, batch: int) -> int:
    """Arena bytes one ShardedLayer takes in P2P mode (4 gathered buffers + counters)."""
    a = PeerSpace.ALIGN
    rnd = lambda n: (n + a - 1) // a * a
    return sum(rnd(batch * w * 4) for w in (nq, shape_d, inter_p, shape_d)) + rnd(8 * 4)


class ShardedLayer:
    """One rank's view of a row-sharded LaRoSA layer (batch 1..16): four or five library phases,
    each followed by an exchange of the phase output.  NCCL: ``allgather(local, gathered)`` is
    torch.distributed.all_gather_into_tensor (CUDA-graph capturable): rank-major
    [world][batch][local]; at batch 1 that is already the column order, at batch > 1
    larosa_shard_gather_permute reorders it to [batch][full].  P2P (``space`` given, SURVEY §8(e)
    v2): the kernel producing a phase output stores it straight into every rank's gathered buffer
    (this layer's buffers live in the PeerSpace arena; the last phase writes the residual ``resid``,
    also in the arena) and bumps every rank's counter; larosa_shard_wait then orders the next phase
    after all ranks' pushes.  Each layer has its own buffers and counters, so a rank that runs ahead
    never overwrites a buffer a slower rank still reads (every phase needs every rank's output)."""

    def __init__(self, w_shard: LZ.LayerWeights, rank: int, world: int, max_ctx: int, device, batch: int = 1,
                 space: Optional[PeerSpace] = None, resid: Optional[torch.Tensor] = None):
        self.w, self.rank, self.world, self.max_ctx, self.batch = w_shard, rank, world, max_ctx, batch
        d, nq, inter = w_shard.d, w_shard.n_q_heads * w_shard.head_dim, w_shard.inter
        n, B = world, batch
        f32 = dict(dtype=torch.float32, device=device)
        self.ws = torch.zeros(LZ.shard_workspace_size(w_shard, rank, world, max_ctx, batch), dtype=torch.uint8,
                              device=device)
        self.local = {0: torch.zeros((B, nq // n), **f32), 1: torch.zeros((B, d // n), **f32),
                      2: torch.zeros((B, inter // n), **f32), 3: torch.zeros((B, d // n), **f32),
                      4: torch.zeros((B, d // n), **f32)}
        self.space = space
        if space is None:
            self.full = {0: torch.zeros((B, nq), **f32), 1: torch.zeros((B, d), **f32),
                         2: torch.zeros((B, inter), **f32), 3: torch.zeros((B, d), **f32)}
            self.stage = torch.zeros((n * B * max(nq, d, inter) // n,), **f32) if B > 1 else None
        else:
            if resid is None or resid.shape != (B, d):
                raise ValueError("ShardedLayer: P2P mode needs the arena residual [batch][d]")
            self.full = {0: space.take((B, nq)), 1: space.take((B, d)), 2: space.take((B, inter)),
                         3: space.take((B, d))}
            self.flags = space.take((8,), torch.int32)           # arrival counters (peers add into them)
            self.expected = torch.zeros((8,), dtype=torch.int32, device=device)
            last = self.n_phases() - 1
            widths = {0: nq, 1: d, 2: inter, 3: d, 4: d}
            self.targets = {ph: space.target(resid if ph == last else self.full[ph], rank * widths[ph] // n,
                                             self.flags[ph:ph + 1]) for ph in range(last + 1)}
            self.counts = {ph: B * widths[ph] for ph in range(last + 1)}

    def run_phase(self, phase: int, x: torch.Tensor, resid: Optional[torch.Tensor], k_cache, v_cache, pos,
                  plan, stream=None) -> torch.Tensor:
        LZ.shard_phase(self.w, plan, self.rank, self.world, phase, x, self.local[phase], self.ws, resid=resid,
                       k_cache=k_cache, v_cache=v_cache, pos=pos, max_ctx=self.max_ctx, stream=stream,
                       peer=self.targets[phase] if self.space is not None else None)
        return self.local[phase]

    def wait_phase(self, phase: int, stream=None):
        """P2P: until every rank's push of this phase output has landed in this rank's buffer."""
        LZ.shard_wait(self.flags[phase:phase + 1], self.expected[phase:phase + 1], self.counts[phase], stream)

    def n_phases(self) -> int:
        """5 with the literal adapter phase; 4 without an adapter or with it folded beside down."""
        return 5 if self.w.adapter is not None and not self.w.adapter_in_down else 4

    def inputs(self, phase: int, r: torch.Tensor):
        """(x, resid) of a phase given the layer input r [batch][d] and the gathered earlier outputs."""
        if phase == 0:
            return r, None
        if phase == 1:
            return self.full[0], r
        if phase == 2:
            return self.full[1], None
        if phase == 3:
            return self.full[2], self.full[1]
        return self.full[3], None

    def gather(self, local: torch.Tensor, full: torch.Tensor, allgather, stream=None):
        """All ranks' phase outputs -> the full [batch][width] vector(s)."""
        if self.batch == 1:
            allgather(local.view(-1), full.view(-1))
            return
        st = self.stage[:local.numel() * self.world]
        allgather(local.view(-1), st)
        LZ.shard_gather_permute(st, self.world, self.batch, full, stream=stream)

    def forward(self, r: torch.Tensor, k_cache, v_cache, pos, plan, allgather, stream=None) -> torch.Tensor:
        """r: the full residual [batch][d] (replicated); returns it updated in place (next layer's input).
        P2P mode: r must be the arena residual the layer was built with; allgather is unused."""
        last = self.n_phases() - 1
        for ph in range(last + 1):
            x, res = self.inputs(ph, r)
            out = self.run_phase(ph, x, res, k_cache, v_cache, pos, plan, stream)
            if self.space is not None:
                self.wait_phase(ph, stream)
            else:
                self.gather(out, r if ph == last else self.full[ph], allgather, stream)
        return r


class ShardedDecodeModel:
    """One rank's share of a whole LaRoSA model for row-sharded decoding (SURVEY §8(a) a7 with
    §8(e)): the replicated folded embedding E' = E Q_0, every layer's shard, and the rank's vocab
    columns of the folded head H' = Q_{L-1}^T diag(gamma_f) H (the head is column-sharded too:
    every rank computes its logits slice, an all-gather reassembles the logits, greedy on them)."""

    def __init__(self, shape: synth.ModelShape, n_layers: int, rank: int, world: int, device, seed: int = 0,
                 adapter_in_down: bool = True, vocab: Optional[int] = None):
        self.shape, self.rank, self.world = shape, rank, world
        vocab = vocab or shape.vocab
        if vocab % (8 * world):
            raise ValueError("vocab must be a multiple of 8 * world")
        d = shape.d
        q_prev = synth.haar_orthogonal(d, 7000 + 100 * seed, device=device, dtype=torch.float32)
        E = synth.gaussian_bf16((vocab, d), 9000 + seed, 1.0, device)
        self.embed = LZ.fold_rotation(q_prev, E, LZ.LAROSA_RIGHT_Q)
        del E
        self.layers = []
        for l in range(n_layers):
            q_next = synth.haar_orthogonal(d, 7000 + 100 * seed + l + 1, device=device, dtype=torch.float32) \
                if l + 1 < n_layers else None
            full = fold_layer(synth_original_layer(shape, 10 * seed + l + 1, device=device), shape, q_prev, q_next,
                              adapter_in_down=adapter_in_down)
            self.layers.append(shard_layer(full, rank, world))
            del full
            q_prev = q_next if q_next is not None else q_prev
        vl = vocab // world
        H = synth.gaussian_bf16((d, vocab), 9100 + seed, d ** -0.5, device)
        gf = (1.0 + 0.1 * synth.gaussian((d,), 9200 + seed, device=device)).float().contiguous()
        self.head = LZ.fold_rotation(q_prev, H[:, rank * vl:(rank + 1) * vl].contiguous(), LZ.LAROSA_LEFT_QT, gamma=gf)
        del H
        self.vocab = vocab
        torch.cuda.empty_cache()


class ShardedDecodeRunner:
    """Decode steps of a ShardedDecodeModel on this rank (batch 1..16): embed (replicated) ->
    every layer's ShardedLayer.forward (4 all-gathers per layer with the adapter beside down) ->
    this rank's LM-head slice -> all-gather of the logits -> greedy.  ``allgather`` as in
    ShardedLayer; CUDA-graph capturable."""

    @staticmethod
    def peer_bytes(model: "ShardedDecodeModel", batch: int) -> int:
        """Arena bytes of the P2P mode (every layer's buffers, the residual, the logits, counters)."""
        s, w0 = model.shape, model.layers[0]
        a = PeerSpace.ALIGN
        rnd = lambda n: (n + a - 1) // a * a
        per = shard_layer_peer_bytes(s.d, s.hq * s.hd, w0.inter, batch)
        return len(model.layers) * per + rnd(batch * s.d * 4) + rnd(batch * model.vocab * 4) + rnd(8 * 4)

    def __init__(self, model: ShardedDecodeModel, batch: int, max_ctx: int, device,
                 space: Optional[PeerSpace] = None):
        self.m, self.batch, self.space = model, batch, space
        s, n, r = model.shape, model.world, model.rank
        f32 = dict(dtype=torch.float32, device=device)
        if space is not None:   # P2P: the residual, every layer's gathered buffers and the logits in the arena
            self.resid = space.take((batch, s.d))
            self.shards = [ShardedLayer(w, r, n, max_ctx, device, batch, space=space, resid=self.resid)
                           for w in model.layers]
            self.logits = space.take((batch, model.vocab))
            self.head_flag = space.take((8,), torch.int32)
            self.head_expected = torch.zeros((8,), dtype=torch.int32, device=device)
            self.head_target = space.target(self.logits, r * (model.vocab // n), self.head_flag[0:1])
        else:
            self.resid = torch.zeros((batch, s.d), **f32)
            self.shards = [ShardedLayer(w, r, n, max_ctx, device, batch) for w in model.layers]
            self.logits = torch.zeros((batch, model.vocab), **f32)
        hk = s.hkv // n
        self.kv = [(torch.zeros((batch, hk, max_ctx, s.hd), dtype=torch.int16, device=device),
                    torch.zeros((batch, hk, max_ctx, s.hd), dtype=torch.int16, device=device)) for _ in model.layers]
        self.tokens = torch.zeros((batch,), dtype=torch.int32, device=device)
        self.next_tokens = torch.zeros((batch,), dtype=torch.int32, device=device)
        self.pos = torch.zeros((batch,), dtype=torch.int32, device=device)
        vl = model.vocab // n
        self.logits_local = torch.zeros((batch, vl), **f32)
        self.stage = torch.zeros((n * batch * vl,), **f32)
        self.local_tok = torch.zeros((batch,), dtype=torch.int32, device=device)
        self.head_ws = torch.zeros(LZ.lib().larosa_lm_head_workspace_size(batch, s.d, vl), dtype=torch.uint8,
                                   device=device)

    def step(self, plan: Sequence[int], allgather, stream=None):
        LZ.embed(self.m.embed, self.tokens, out=self.resid, stream=stream)
        for sh, (kc, vc) in zip(self.shards, self.kv):
            sh.forward(self.resid, kc, vc, self.pos, plan, allgather, stream)
        LZ.lm_head(self.resid, self.m.head, self.m.shape.rms_eps, logits=self.logits_local,
                   next_token=self.local_tok, ws=self.head_ws, stream=stream)
        if self.space is not None:
            self.push_logits(stream)
            self.wait_logits(stream)
        elif self.batch == 1:
            allgather(self.logits_local.view(-1), self.logits.view(-1))
        else:
            allgather(self.logits_local.view(-1), self.stage)
            LZ.shard_gather_permute(self.stage, self.m.world, self.batch, self.logits, stream=stream)
        LZ.argmax(self.logits, self.next_tokens, stream=stream)
        return self.next_tokens

    def push_logits(self, stream=None):
        LZ.peer_push(self.logits_local, self.head_target, self.m.world, stream)

    def wait_logits(self, stream=None):
        LZ.shard_wait(self.head_flag[0:1], self.head_expected[0:1], self.batch * self.m.vocab, stream)
