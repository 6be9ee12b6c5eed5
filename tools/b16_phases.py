"""In-graph time of the batch-16 LLaMA3-8B layer (4 chained layer copies, adapter beside down,
p = 0.4) with all kernels, and without the rule kernels / the GEMVs / attention
(larosa_debug_set_layer_phases), for the current env (LAROSA_RULE_KERNEL etc.).  JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2507_01299_b200 import larosa as LZ
from paper_2507_01299_b200 import model as M
DEV = "cuda:0"
B = int(os.environ.get("B", "16"))
shape = synth.MODELS[os.environ.get("MODEL", "llama3-8b")]
n = 4
qs = [synth.haar_orthogonal(shape.d, 100 + i, device=DEV, dtype=torch.float32) for i in range(n + 1)]
layers = [M.fold_layer(M.synth_original_layer(shape, i + 1, device=DEV), shape, qs[i], qs[i + 1], adapter_in_down=True)
          for i in range(n)]
ctx = 256
kv = [(synth.gaussian_bf16((B, shape.hkv, ctx, shape.hd), 900 + i, 1.0, DEV),
       synth.gaussian_bf16((B, shape.hkv, ctx, shape.hd), 950 + i, 1.0, DEV)) for i in range(n)]
pos = torch.full((B,), ctx - 1, dtype=torch.int32, device=DEV)
resid = synth.residual_activation(B, shape.d, 7).to(DEV)
wsb = torch.zeros(LZ.layer_workspace_size(layers[0], B, ctx), dtype=torch.uint8, device=DEV)
plan = M.site_plan(shape, float(os.environ.get("P", "0.4")))

def timed(mask, reps=50):
    LZ.lib().larosa_debug_set_layer_phases(mask)
    for i in range(n):
        LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos), ws=wsb)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(n):
            LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos), ws=wsb)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    LZ.lib().larosa_debug_set_layer_phases(-1)
    return e0.elapsed_time(e1) * 1e3 / (reps * n)

ALL = 2047
res = {"B": B, "env": {k: v for k, v in os.environ.items() if k.startswith("LAROSA")}, "layer_us": timed(ALL),
       "no_rules_us": timed(ALL & ~(1 | 8 | 32 | 128)), "no_attention_us": timed(ALL & ~4),
       "rules_attention_only_us": timed(1 | 4 | 8 | 32 | 128), "gemvs_only_us": timed(2 | 16 | 64 | 256 | 512)}
print(json.dumps(res))
