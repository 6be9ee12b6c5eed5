"""Block step time (us) of the bench workload, quick: python tools/layer_us.py [p] [steps].
Env knobs (LAROSA_COMP_PCT, ...) are read by the library at first use."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402
from paper_2507_01299_b200 import model as M  # noqa: E402

p = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
merged = os.environ.get("ADAPTER", "down") == "down"
dev = "cuda:0"
shape = synth.MODELS["llama2-7b"]
layers = bench.build_stack(shape, dev, bench.N_COPIES, merged=merged)
kv = [(synth.gaussian_bf16((1, shape.hkv, bench.CTX, shape.hd), 900 + i, 1.0, dev),
       synth.gaussian_bf16((1, shape.hkv, bench.CTX, shape.hd), 950 + i, 1.0, dev)) for i in range(bench.N_COPIES)]
pos = torch.full((1,), bench.CTX - 1, dtype=torch.int32, device=dev)
ws = torch.zeros(LZ.layer_workspace_size(layers[0], 1, bench.CTX), dtype=torch.uint8, device=dev)
resid = synth.residual_activation(1, shape.d, seed=77).to(dev)
plan = M.site_plan(shape, p)
graphs = bench.capture_graphs(layers, kv, resid, pos, plan, ws)
bench.run_steps(graphs, 100, 0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = []
for t in range(3):
    e0.record()
    bench.run_steps(graphs, steps, 0)
    e1.record()
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) * 1e3 / steps)
print(f"{os.environ.get('TAG', '')} p={p} block_us={min(res):.2f} all={[round(r, 2) for r in res]}")
