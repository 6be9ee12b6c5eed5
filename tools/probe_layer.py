"""One layer (LLaMA2-7B, or argv[2]), a few decode steps at p = argv[1] (for an ncu capture)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402
from paper_2507_01299_b200 import model as M  # noqa: E402

shape = synth.MODELS[sys.argv[2] if len(sys.argv) > 2 else "llama2-7b"]
p = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
dev = "cuda:0"
q0 = synth.haar_orthogonal(shape.d, 1, device=dev, dtype=torch.float32)
q1 = synth.haar_orthogonal(shape.d, 2, device=dev, dtype=torch.float32)
lw = M.fold_layer(M.synth_original_layer(shape, 1, device=dev), shape, q0, q1, adapter_in_down=True)
ctx = 256
kc = synth.gaussian_bf16((1, shape.hkv, ctx, shape.hd), 3, 1.0, dev)
vc = synth.gaussian_bf16((1, shape.hkv, ctx, shape.hd), 4, 1.0, dev)
pos = torch.full((1,), ctx - 1, dtype=torch.int32, device=dev)
resid = synth.residual_activation(1, shape.d, 5).to(dev)
plan = M.site_plan(shape, p)
torch.cuda.synchronize()
for i in range(6):
    LZ.sparse_layer(lw, plan, LZ.LayerState(resid, kc, vc, pos, chained=i > 0))
torch.cuda.synchronize()
print("probe ok")
