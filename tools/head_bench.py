"""LM head (larosa_lm_head: final RMS + dense GEMV over H' + greedy) time at LLaMA3-8B shapes."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2507_01299_b200 import larosa as LZ
dev = "cuda:0"
d, V = 4096, 128256
Hs = [synth.gaussian_bf16((d, V), 10 + i, d ** -0.5, dev) for i in range(3)]
out = {}
for B in (1, 16):
    r = torch.randn((B, d), device=dev)
    lg = torch.empty((B, V), device=dev)
    nt = torch.empty((B,), dtype=torch.int32, device=dev)
    ws = torch.zeros(LZ.lib().larosa_lm_head_workspace_size(B, d, V), dtype=torch.uint8, device=dev)
    for i in range(3):
        LZ.lm_head(r, Hs[i % 3], 1e-5, logits=lg, next_token=nt, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(30):
        LZ.lm_head(r, Hs[i % 3], 1e-5, logits=lg, next_token=nt, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 30
    out[f"B{B}"] = {"us": us, "gbs": d * V * 2 / us / 1e3}
x = torch.randn((1, d), device=dev, dtype=torch.bfloat16)
Wb = [h.view(torch.bfloat16) for h in Hs]
for i in range(3):
    torch.matmul(x, Wb[i])
torch.cuda.synchronize()
e0.record()
for i in range(30):
    torch.matmul(x, Wb[i % 3])
e1.record()
torch.cuda.synchronize()
out["cublas_B1_us"] = e0.elapsed_time(e1) * 1e3 / 30
print(json.dumps(out))
