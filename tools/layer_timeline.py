"""In-graph timeline of the batch-1 layer kernels (%globaltimer stamps via
larosa_debug_set_timeline): per kernel, the dependency-wait release, prologue end, main-loop
end and exit, relative to the previous kernel's exit.  Chained CUDA graph over 4 layer
copies (weights >> L2).   python tools/layer_timeline.py [--p 0.5] [--model llama2-7b]"""
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
    ap.add_argument("--p", type=float, default=0.5)
    ap.add_argument("--model", default="llama2-7b")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--adapter", default="down", choices=["down", "separate"])
    ap.add_argument("--w4", action="store_true", help="W4A16 weights at all four sites")
    args = ap.parse_args()
    shape = synth.MODELS[args.model]
    n = 4
    qs = [synth.haar_orthogonal(shape.d, 100 + i, device=DEV, dtype=torch.float32) for i in range(n + 1)]
    merged = args.adapter == "down"
    layers = [M.fold_layer(M.synth_original_layer(shape, i + 1, device=DEV), shape, qs[i], qs[i + 1],
                           adapter_in_down=merged) for i in range(n)]
    if args.w4:
        layers = [M.quantize_layer_w4(w, drop_bf16=True) for w in layers]
    ctx = 256
    kv = [(synth.gaussian_bf16((1, shape.hkv, ctx, shape.hd), 900 + i, 1.0, DEV),
           synth.gaussian_bf16((1, shape.hkv, ctx, shape.hd), 950 + i, 1.0, DEV)) for i in range(n)]
    pos = torch.full((1,), ctx - 1, dtype=torch.int32, device=DEV)
    resid = synth.residual_activation(1, shape.d, 7).to(DEV)
    wsb = torch.zeros(LZ.layer_workspace_size(layers[0], 1, ctx), dtype=torch.uint8, device=DEV)
    plan = M.site_plan(shape, args.p)
    L = LZ.lib()
    L.larosa_debug_set_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.larosa_debug_set_timeline.restype = None
    tl = torch.zeros((n, 6, 1024, 16), dtype=torch.int64, device=DEV)
    for i in range(n):
        LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos, chained=i > 0), ws=wsb)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(n):
            L.larosa_debug_set_timeline(ctypes.c_void_p(tl[i].data_ptr()), 6)
            LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos, chained=True), ws=wsb)
        L.larosa_debug_set_timeline(None, 0)
    acc = []
    for r in range(args.reps + 3):
        tl.zero_()
        g.replay()
        torch.cuda.synchronize()
        if r >= 3:
            acc.append(tl.cpu().numpy().astype(np.float64))
    out = {"model": args.model, "p": args.p, "plan": list(plan), "w4": args.w4, "kernels": {}}
    last = 4 if merged else 5
    lay = []
    for a in acc:
        for li in range(1, n):
            lay.append(a[li][last][:, 4].max() - a[li - 1][last][:, 4].max())
    out["layer_us"] = round(float(np.mean(lay)) / 1e3, 2)
    groups = [(k, name, None) for k, name in enumerate(NAMES[:last + 1])]
    if merged:   # the down launch: SELECT CTAs (stamp 5 written) and dense companion CTAs
        groups[4] = (4, "down_select", True)
        groups.insert(5, (4, "down_companion", False))
    for k, name, sel in groups:
        stats = {}
        for a in acc:
            for li in range(1, n):
                prev = a[li - 1][last] if k == 0 else a[li][k - 1]
                t0 = prev[:, 4].max()                     # previous kernel's last exit
                cur = a[li][k]
                live = cur[:, 0] > 0
                if sel is not None:
                    live = live & ((cur[:, 5] > 0) == sel)
                c = cur[live] - t0
                for i, key in enumerate(["entry", "wait", "prologue", "loop", "exit", "sel_hist", "rule_coarse", "sel_mask",
                                          "rule_fine", "rule_pool", "rule_ssq", "list", "ticket", "epi", "lookup_data",
                                          "unused"]):
                    col = c[:, i]
                    col = col[cur[live][:, i] > 0]
                    if col.size:
                        for q, qn in ((0, "min"), (50, "med"), (100, "max")):
                            stats.setdefault(f"{key}_{qn}", []).append(np.percentile(col, q))
                stats.setdefault("ctas", []).append(int(live.sum()))
        out["kernels"][name] = {key: round(float(np.mean(v)) / (1e3 if key != "ctas" else 1), 2)
                                for key, v in stats.items()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
