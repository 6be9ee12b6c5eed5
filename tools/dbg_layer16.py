"""Debug aid: batch-16 layer, new-k accuracy vs the oracle (tcgen05 vs CUDA-core GEMV)."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import synth  # noqa: E402
from test_gpu_layer import SMALL, build, run_layer, w64, f64  # noqa: E402

batch, ctx, p = 16, 30, 0.5
orig, q_l, q_n, lw, plan, resid, kc0, vc0, pos = build(SMALL, 3, batch, ctx, 64, p)
st, tp = run_layer(lw, plan, resid, kc0, vc0, pos)
hd, hq, hkv = SMALL.hd, SMALL.hq, SMALL.hkv
nq = hq * hd
kc_gpu = st.k_cache.cpu().numpy().view(np.uint16)
worst = 0
for b in range(batch):
    i1 = tp["idx_h1"][b].cpu().numpy()
    y = O.sparse_gemv(w64(lw.w_qkv), i1, f64(tp["vals_h1"][b]), w64(lw.b_qkv))
    pb = int(pos[b])
    kn = np.concatenate([O.rope(y[nq + h * hd: nq + (h + 1) * hd], pb, SMALL.rope_theta) for h in range(hkv)])
    kg = O.bf16_to_f64(kc_gpu[b, :, pb, :]).reshape(-1)
    e = np.abs(kg - kn) / np.maximum(np.abs(kn), 1e-9)
    worst = max(worst, e.max())
    if b < 3:
        j = int(np.argmax(e))
        print(b, "max rel", e.max(), "at", j, kg[j], kn[j], "norm-rel", np.max(np.abs(kg - kn)) / np.linalg.norm(kn))
print("worst", worst, "bf16 half-ulp", 2 ** -9)
