"""Debug aid: fused Top-K + GEMV with W = I shows the kept set and values directly."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402

for (d, k) in [(64, 32), (4096, 1638), (4096, 2048)]:
    x = synth.residual_activation(1, d, seed=d + k)[0]
    eye = torch.eye(d, dtype=torch.bfloat16).view(torch.int16).contiguous()
    y = LZ.topk_sparse_gemv(x.cuda(), k, eye.cuda()).cpu().numpy()
    xd = x.numpy().astype(np.float64)
    idx = O.topk(xd, k)
    exp = np.zeros(d)
    exp[idx] = xd[idx]
    bad = np.where(np.abs(y - exp) > 1e-6 * np.abs(xd).max())[0]
    print(d, k, "nonzero", int((y != 0).sum()), "bad", bad[:10].tolist(),
          [(int(i), float(y[i]), float(exp[i]), hex(np.float32(xd[i]).view(np.uint32) & 0x7fffffff)) for i in bad[:4]],
          "thr key", hex(np.float32(np.sort(np.abs(xd))[::-1][k - 1]).view(np.uint32)))
