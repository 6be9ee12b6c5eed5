"""One LLaMA3-8B layer at batch B (default 16), a few decode steps (for an ncu launch list)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402
from paper_2507_01299_b200 import model as M  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
shape = synth.MODELS["llama3-8b"]
dev = "cuda:0"
q0 = synth.haar_orthogonal(shape.d, 1, device=dev, dtype=torch.float32)
q1 = synth.haar_orthogonal(shape.d, 2, device=dev, dtype=torch.float32)
lw = M.fold_layer(M.synth_original_layer(shape, 1, device=dev), shape, q0, q1)
ctx = 256
kc = synth.gaussian_bf16((B, shape.hkv, ctx, shape.hd), 3, 1.0, dev)
vc = synth.gaussian_bf16((B, shape.hkv, ctx, shape.hd), 4, 1.0, dev)
pos = torch.full((B,), ctx - 1, dtype=torch.int32, device=dev)
resid = synth.residual_activation(B, shape.d, 5).to(dev)
plan = M.site_plan(shape, 0.4)
for i in range(4):
    LZ.sparse_layer(lw, plan, LZ.LayerState(resid, kc, vc, pos))
torch.cuda.synchronize()
print("probe ok")
