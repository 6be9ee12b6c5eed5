"""Debug aid: clock64 phase stamps of the last compute_rule call of a chained layer (the
adapter's rule for the next layer's h1)."""
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
kc = synth.gaussian_bf16((1, shape.hkv, 256, shape.hd), 3, 1.0, dev)
vc = synth.gaussian_bf16((1, shape.hkv, 256, shape.hd), 4, 1.0, dev)
pos = torch.full((1,), 255, dtype=torch.int32, device=dev)
resid = synth.residual_activation(1, shape.d, 5).to(dev)
plan = M.site_plan(shape, 0.5)
L = LZ.lib()
L.larosa_debug_read_rule_stamps.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_longlong * 16)()
for i in range(4):
    LZ.sparse_layer(lw, plan, LZ.LayerState(resid, kc, vc, pos, chained=i > 0))
    torch.cuda.synchronize()
    L.larosa_debug_read_rule_stamps(ctypes.byref(buf))
    b = list(buf)
    print("cnt", b[8], "rem", b[9], "fallback", b[10], "| coarse", b[1] - b[0], "fine", b[2] - b[1], "rank", b[3] - b[2],
          "to-sync", b[4] - b[0], "sync", b[5] - b[4], "tail", b[6] - b[5], "total", b[6] - b[0],
          "| first call: coarse", b[12], "fine", b[13], "total", b[14])
