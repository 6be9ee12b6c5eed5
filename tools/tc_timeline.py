"""In-graph timeline of one batch-B LLaMA3-8B layer (default B = 16, the tcgen05 GEMV path):
per stamped kernel, the spread of CTA entries and the median CTA's phases (dependency wait,
prologue, main loop, tail), all in us.   python tools/tc_timeline.py [B] [p]"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402
from paper_2507_01299_b200 import model as M  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
P = float(sys.argv[2]) if len(sys.argv) > 2 else 0.4
dev = "cuda:0"
shape = synth.MODELS["llama3-8b"]
n = 4
qs = [synth.haar_orthogonal(shape.d, 100 + i, device=dev, dtype=torch.float32) for i in range(n + 1)]
layers = [M.fold_layer(M.synth_original_layer(shape, i + 1, device=dev), shape, qs[i], qs[i + 1]) for i in range(n)]
ctx = 256
kv = [(synth.gaussian_bf16((B, shape.hkv, ctx, shape.hd), 900 + i, 1.0, dev),
       synth.gaussian_bf16((B, shape.hkv, ctx, shape.hd), 950 + i, 1.0, dev)) for i in range(n)]
pos = torch.full((B,), ctx - 1, dtype=torch.int32, device=dev)
resid = synth.residual_activation(B, shape.d, 7).to(dev)
plan = M.site_plan(shape, P)
wsb = torch.zeros(LZ.layer_workspace_size(layers[0], B, ctx), dtype=torch.uint8, device=dev)
L = LZ.lib()
L.larosa_debug_set_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.larosa_debug_set_timeline.restype = None
tl = torch.zeros((n, 6, 1024, 16), dtype=torch.int64, device=dev)
for i in range(n):
    LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos, chained=i > 0), ws=wsb)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(n):
        L.larosa_debug_set_timeline(ctypes.c_void_p(tl[i].data_ptr()), 6)
        LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos, chained=True), ws=wsb)
    L.larosa_debug_set_timeline(None, 0)
acc = []
for r in range(13):
    tl.zero_()
    g.replay()
    torch.cuda.synchronize()
    if r >= 3:
        acc.append(tl.cpu().numpy().astype(np.float64))
names = ["qkv", "attention", "o", "gate_up", "down", "adapter"]
out = {"batch": B, "p": P, "kernels": {}}
for k, name in enumerate(names):
    st = {}
    for a in acc:
        for li in range(1, n):
            cur = a[li][k]
            live = cur[:, 0] > 0
            if not live.any():
                continue
            c = cur[live]
            t0 = c[:, 0].min()
            st.setdefault("ctas", []).append(int(live.sum()))
            st.setdefault("entry_spread", []).append(np.percentile(c[:, 0] - t0, 100))
            st.setdefault("wait_med", []).append(np.median(c[:, 1] - c[:, 0]))
            st.setdefault("prologue_med", []).append(np.median(c[:, 2] - c[:, 1]))
            st.setdefault("loop_med", []).append(np.median(c[:, 3] - c[:, 2]))
            st.setdefault("loop_max", []).append(np.max(c[:, 3] - c[:, 2]))
            st.setdefault("tail_med", []).append(np.median(c[:, 4] - c[:, 3]))
            st.setdefault("tail_max", []).append(np.max(c[:, 4] - c[:, 3]))
            st.setdefault("span", []).append(c[:, 4].max() - c[:, 1].min())
    out["kernels"][name] = {key: round(float(np.mean(v)) / (1 if key == "ctas" else 1e3), 2) for key, v in st.items()}
print(json.dumps(out))
