"""Quick: W4A16 vs bf16 fused Top-K GEMV per LLaMA2-7B site (isolated, graph-replayed)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
from paper_2507_01299_b200 import model as M
shape = synth.MODELS["llama2-7b"]
layers = bench.build_stack(shape, "cuda:0", 8, merged=False)
plan = M.site_plan(shape, 0.5)
w4 = bench.w4_sites_extra(layers, plan, shape, "cuda:0")
bf = bench.time_gemv_sites(layers, plan, shape, "cuda:0")
print(json.dumps({k: {"w4_us": round(v["us"], 2), "w4_gbs": round(v["gbs"]), "bf16_us": round(bf[k]["us"], 2)} for k, v in w4.items()}))
