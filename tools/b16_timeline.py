"""In-graph timeline of the batch-16 layer's tcgen05 image GEMVs (%globaltimer stamps via
larosa_debug_set_timeline): per GEMV launch, the dependency release, the accumulator-ready time,
the ticket and the exit, relative to the launch's first CTA entry; LLaMA3-8B, adapter beside down,
4 chained layer copies.   python tools/b16_timeline.py [--p 0.4]"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402
from paper_2507_01299_b200 import model as M  # noqa: E402

DEV = "cuda:0"
NAMES = ["qkv", "attention", "o", "gate_up", "down", "adapter"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=float, default=0.4)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    shape, B, n, ctx = synth.MODELS["llama3-8b"], 16, 4, 256
    qs = [synth.haar_orthogonal(shape.d, 100 + i, device=DEV, dtype=torch.float32) for i in range(n + 1)]
    layers = [M.fold_layer(M.synth_original_layer(shape, i + 1, device=DEV), shape, qs[i], qs[i + 1],
                           adapter_in_down=True) for i in range(n)]
    kv = [(synth.gaussian_bf16((B, shape.hkv, ctx, shape.hd), 900 + i, 1.0, DEV),
           synth.gaussian_bf16((B, shape.hkv, ctx, shape.hd), 950 + i, 1.0, DEV)) for i in range(n)]
    pos = torch.full((B,), ctx - 1, dtype=torch.int32, device=DEV)
    resid = synth.residual_activation(B, shape.d, 7).to(DEV)
    wsb = torch.zeros(LZ.layer_workspace_size(layers[0], B, ctx), dtype=torch.uint8, device=DEV)
    plan = M.site_plan(shape, args.p)
    L = LZ.lib()
    L.larosa_debug_set_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.larosa_debug_set_timeline.restype = None
    tl = torch.zeros((n, 10, 1024, 16), dtype=torch.int64, device=DEV)
    for i in range(n):
        LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos), ws=wsb)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(n):
            L.larosa_debug_set_timeline(ctypes.c_void_p(tl[i].data_ptr()), 10)
            LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos), ws=wsb)
        L.larosa_debug_set_timeline(None, 0)
    acc = []
    for r in range(args.reps + 3):
        tl.zero_()
        g.replay()
        torch.cuda.synchronize()
        if r >= 3:
            acc.append(tl.cpu().numpy().astype(np.float64))
    out = {"p": args.p, "batch": B, "kernels": {}}
    for k in (0, 2, 3, 4, 5):
        st = {}
        for a in acc:
            for li in range(1, n):
                cur = a[li][k]
                live = cur[:, 0] > 0
                if not live.any():
                    continue
                c = cur[live]
                t0 = c[:, 0].min()
                for i, key in ((1, "wait"), (3, "acc_ready"), (12, "ticket"), (13, "epi"), (4, "exit")):
                    col = c[:, i][c[:, i] > 0] - t0
                    if col.size:
                        for q, qn in ((50, "med"), (100, "max")):
                            st.setdefault(f"{key}_{qn}", []).append(np.percentile(col, q))
                st.setdefault("ctas", []).append(int(live.sum()))
        out["kernels"][NAMES[k]] = {kk: round(float(np.mean(v)) / (1e3 if kk != "ctas" else 1), 2)
                                    for kk, v in st.items()}
    # attention (slot 1): phases relative to its dependency release
    st = {}
    for a in acc:
        for li in range(1, n):
            cur = a[li][1]
            live = cur[:, 1] > 0
            if not live.any():
                continue
            c = cur[live]
            t1 = c[:, 1].min()
            for i, key in ((0, "entry"), (2, "q_kv_ready"), (3, "scores_pv"), (6, "merged"), (4, "exit")):
                col = c[:, i][c[:, i] > 0] - t1
                if col.size:
                    st.setdefault(f"{key}_med", []).append(np.median(col))
                    st.setdefault(f"{key}_max", []).append(col.max())
            st.setdefault("ctas", []).append(int(live.sum()))
    out["kernels"]["attention"] = {kk: round(float(np.mean(v)) / (1e3 if kk != "ctas" else 1), 2) for kk, v in st.items()}
    # the Top-K rule kernels (slots 6-9: sites h1..h4), phases relative to their dependency release
    for si in range(4):
        st = {}
        for a in acc:
            for li in range(1, n):
                cur = a[li][6 + si]
                live = cur[:, 1] > 0
                if not live.any():
                    continue
                c = cur[live]
                t1 = c[:, 1].min()
                for i, key in ((2, "loaded"), (9, "hist0"), (10, "scan0"), (11, "gathered"), (5, "pass0/rule"),
                               (6, "pass1"), (8, "rule_image"), (4, "exit")):
                    col = c[:, i][c[:, i] > 0] - t1
                    if col.size:
                        st.setdefault(f"{key}_max", []).append(col.max())
                st.setdefault("ctas", []).append(int(live.sum()))
        out["kernels"][f"topk_h{si + 1}"] = {kk: round(float(np.mean(v)) / (1e3 if kk != "ctas" else 1), 2)
                                             for kk, v in st.items()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
