"""In-graph microseconds per LLaMA3-8B layer at batch 1 (4 chained layer copies, adapter beside
down, ctx 256) for the current environment (tuning knobs are read once per process).  JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2507_01299_b200 import larosa as LZ
from paper_2507_01299_b200 import model as M
DEV = "cuda:0"
shape = synth.MODELS[os.environ.get("MODEL", "llama3-8b")]
p = float(os.environ.get("P", "0.4"))
n = 6
qs = [synth.haar_orthogonal(shape.d, 100 + i, device=DEV, dtype=torch.float32) for i in range(n + 1)]
layers = [M.fold_layer(M.synth_original_layer(shape, i + 1, device=DEV), shape, qs[i], qs[i + 1], adapter_in_down=True)
          for i in range(n)]
ctx = 256
kv = [(synth.gaussian_bf16((1, shape.hkv, ctx, shape.hd), 900 + i, 1.0, DEV),
       synth.gaussian_bf16((1, shape.hkv, ctx, shape.hd), 950 + i, 1.0, DEV)) for i in range(n)]
pos = torch.full((1,), ctx - 1, dtype=torch.int32, device=DEV)
resid = synth.residual_activation(1, shape.d, 7).to(DEV)
wsb = torch.zeros(LZ.layer_workspace_size(layers[0], 1, ctx), dtype=torch.uint8, device=DEV)
plan = M.site_plan(shape, p)
for i in range(n):
    LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos, chained=i > 0), ws=wsb)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(n):
        LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos, chained=True), ws=wsb)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
res = []
for trial in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) * 1e3 / (100 * n))
res.sort()
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("LAROSA")}, "p": p,
                  "layer_us_median": res[2], "layer_us_min": res[0]}))
