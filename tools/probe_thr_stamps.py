"""Timestamps inside the threshold kernels of one LLaMA2-7B layer step (profiling)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402
from paper_2507_01299_b200 import model as M  # noqa: E402

shape = synth.MODELS["llama2-7b"]
dev = "cuda:0"
q0 = synth.haar_orthogonal(shape.d, 1, device=dev, dtype=torch.float32)
q1 = synth.haar_orthogonal(shape.d, 2, device=dev, dtype=torch.float32)
lw = M.fold_layer(M.synth_original_layer(shape, 1, device=dev), shape, q0, q1)
ctx = 256
kc = synth.gaussian_bf16((1, shape.hkv, ctx, shape.hd), 3, 1.0, dev)
vc = synth.gaussian_bf16((1, shape.hkv, ctx, shape.hd), 4, 1.0, dev)
pos = torch.full((1,), ctx - 1, dtype=torch.int32, device=dev)
resid = synth.residual_activation(1, shape.d, 5).to(dev)
plan = M.site_plan(shape, 0.5)
buf = torch.zeros(128, dtype=torch.int64, device=dev)
L = LZ.lib()
L.larosa_debug_set_thresh_stamps.argtypes = [ctypes.c_void_p]
for it in range(5):
    L.larosa_debug_set_thresh_stamps(ctypes.c_void_p(buf.data_ptr()) if it == 4 else None)
    LZ.sparse_layer(lw, plan, LZ.LayerState(resid, kc, vc, pos))
    torch.cuda.synchronize()
b = buf.cpu().tolist()
for s in range(4):
    st = b[32 * s: 32 * s + 32]
    t0 = st[0]
    print(f"site {s}: gtimer " + " ".join(f"{(st[i] - t0) / 1000:.2f}" for i in range(6)) + f"  (us since CTA0 start; bucket={st[15]})")
    c = st[16:32]
    print("        clock64 from stamp 2: " + ", ".join(f"s{i}={c[i] - c[2]}" for i in (2, 6, 7, 8, 3, 4, 5)))
