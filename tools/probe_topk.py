"""Top-K probe for ncu: batch-16 rotate_topk (R = NULL) on LLaMA-shaped widths."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
x = synth.residual_activation(16, d, 5).cuda()
for _ in range(4):
    LZ.rotate_topk(x, None, d // 2, rms_eps=1e-5)
torch.cuda.synchronize()
print("probe ok")
