"""Time the batch-16 tcgen05 sparse GEMV standalone (all rows kept): tc_probe.py d_in d_out."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402

d_in, d_out, B = int(sys.argv[1]), int(sys.argv[2]), 16
Ws = [synth.gaussian_bf16((d_in, d_out), 3 + i, d_in ** -0.5).cuda() for i in range(4)]
x = synth.residual_activation(B, d_in, 4).cuda()
_, idx, vals, _ = LZ.rotate_topk(x, None, d_in)
y = torch.empty((B, d_out), device="cuda")
for i in range(3):
    LZ.sparse_gemv(Ws[i % 4], idx, vals, out=y)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(16):
        LZ.sparse_gemv(Ws[i % 4], idx, vals, out=y)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 80
print(os.environ.get("LAROSA_TC_DBG", "0"), d_in, d_out, f"{us:.2f} us  {d_in * d_out * 2 / us / 1e3:.0f} GB/s")
