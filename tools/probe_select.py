"""A few standalone fused Top-K + sparse GEMV calls (batch 1) for ncu: d_in 4096 -> d_out 4096,
k = 2048 (LLaMA2-7B W_o at 50%)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402

d_in = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d_out = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
k = d_in // 2
xs = [synth.residual_activation(1, d_in, seed=s)[0].cuda() for s in range(4)]
W = synth.gaussian_bf16((d_in, d_out), 1, d_in ** -0.5, "cuda")
for i in range(6):
    LZ.topk_sparse_gemv(xs[i % 4], k, W)
torch.cuda.synchronize()
print("ok")
