"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck, ONE tool per gpurun
call): batch-1 / 3 / 16 layers (SELECT, THRESH + tcgen05, both adapter forms, Q_B), a 2-layer
decode step with the LM head, the shard phases at n = 2 (B = 1 and 3), the prefill GEMM, the
fused Top-K GEMVs, the fold and the PCA rotation, all on toy shapes."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2507_01299_b200 import larosa as LZ
from paper_2507_01299_b200 import model as M

dev = "cuda:0"
shape = synth.ModelShape("san", 256, 512, 4, 2, 64, 2, 512, True, 1e-6, 10000.0)
for B, merged, qb in ((1, True, False), (1, False, True), (3, True, False), (16, False, False), (16, True, True)):
    orig = M.synth_original_layer(shape, 1, device=dev)
    ql = synth.haar_orthogonal(shape.d, 2, device=dev, dtype=torch.float32)
    qn = synth.haar_orthogonal(shape.d, 3, device=dev, dtype=torch.float32)
    qm = synth.haar_orthogonal(shape.d, 4, device=dev, dtype=torch.float32) if qb else None
    lw = M.fold_layer(orig, shape, ql, qn, adapter_in_down=merged, q_mlp=qm)
    plan = M.site_plan(shape, 0.5)
    for max_ctx in (64, 300):
        st = LZ.LayerState(synth.residual_activation(B, shape.d, 5).to(dev),
                           synth.gaussian_bf16((B, shape.hkv, max_ctx, shape.hd), 6, 1.0, dev),
                           synth.gaussian_bf16((B, shape.hkv, max_ctx, shape.hd), 7, 1.0, dev),
                           torch.full((B,), max_ctx - 2, dtype=torch.int32, device=dev))
        taps = LZ.make_taps(lw, plan, B, dev)
        LZ.sparse_layer(lw, plan, st, taps=taps)
        LZ.sparse_layer(lw, plan, st)
torch.cuda.synchronize()
model = M.synth_decode_model(shape, 2, dev, seed=1, adapter_in_down=True)
for B in (1, 4):
    run = M.DecodeRunner(model, B, 32, dev)
    run.pos.fill_(10)
    run.step(M.site_plan(shape, 0.5))
torch.cuda.synchronize()
shape2 = synth.ModelShape("san2", 256, 512, 4, 4, 64, 2, 512, True, 1e-6, 10000.0)
lw2 = M.fold_layer(M.synth_original_layer(shape2, 3, device=dev), shape2,
                   synth.haar_orthogonal(256, 8, device=dev, dtype=torch.float32),
                   synth.haar_orthogonal(256, 9, device=dev, dtype=torch.float32), adapter_in_down=True)
for B in (1, 3):
    ranks = [M.ShardedLayer(M.shard_layer(lw2, r, 2), r, 2, 32, dev, B) for r in range(2)]
    kvs = [(torch.zeros((B, 2, 32, 64), dtype=torch.int16, device=dev),
            torch.zeros((B, 2, 32, 64), dtype=torch.int16, device=dev)) for _ in range(2)]
    r0 = synth.residual_activation(B, 256, 10).to(dev)
    pos = torch.full((B,), 5, dtype=torch.int32, device=dev)
    for ph in range(ranks[0].n_phases()):
        outs = []
        for rk, (kc, vc) in zip(ranks, kvs):
            x, res = rk.inputs(ph, r0)
            outs.append(rk.run_phase(ph, x, res, kc, vc, pos, M.site_plan(shape2, 0.5)).clone())
        stacked = torch.stack(outs).reshape(-1)
        for rk in ranks:
            rk.gather(outs[rk.rank], r0 if ph == ranks[0].n_phases() - 1 else rk.full[ph],
                      lambda l, d_: d_.copy_(stacked))
torch.cuda.synchronize()
X = torch.randn((300, 256), device=dev)
W = synth.gaussian_bf16((256, 384), 11, 0.06, dev)
for split in (False, True):
    LZ.prefill_sparse_gemm(X, 100, W, rms_eps=1e-6, split=split)
x = torch.randn((256,), device=dev)
LZ.topk_sparse_gemv(x, 100, W, rms_eps=1e-6)
LZ.rotate_topk(torch.randn((3, 256), device=dev), synth.bf16_bits(synth.haar_orthogonal(256, 1)).to(dev), 100,
               rms_eps=1e-5, want_xr=True)
C = torch.randn((256, 256), device=dev)
C = C @ C.T
LZ.pca_rotation(C)
LZ.pca_rotation(C[:129, :129].contiguous())
LZ.fold_rotation(synth.haar_orthogonal(256, 2, device=dev, dtype=torch.float32), W, LZ.LAROSA_LEFT_QT)
torch.cuda.synchronize()
print("sanitize workload done")
