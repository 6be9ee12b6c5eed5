"""Debug aid: one batch-8 sparse GEMV through the tcgen05 path vs the CUDA-core path."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402

d_in, d_out, k, B = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
W = synth.gaussian_bf16((d_in, d_out), 3, d_in ** -0.5).cuda()
x = synth.residual_activation(B, d_in, 4).cuda()
_, idx, vals, _ = LZ.rotate_topk(x, None, k)
y = LZ.sparse_gemv(W, idx, vals)
torch.cuda.synchronize()
Wf = O.bf16_to_f64(W.cpu().numpy().view(np.uint16))
for b in range(B):
    ref = O.sparse_gemv(Wf, idx[b].cpu().numpy(), vals[b].cpu().numpy().astype(np.float64))
    print(b, float(np.max(np.abs(y[b].cpu().numpy() - ref)) / np.linalg.norm(ref)))
