"""Marginal in-graph cost of each kernel of the batch-1 LLaMA2-7B layer step (chained CUDA
graphs over 4 layer copies): t(all) - t(all but one), via larosa_debug_set_layer_phases.
Prints one JSON line.   python tools/layer_phases.py [--p 0.5]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402
from paper_2507_01299_b200 import model as M  # noqa: E402

DEV = "cuda:0"
BITS = {"qkv": 1, "attention": 2, "o": 4, "gate_up": 6, "down": 8, "adapter": 9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=float, default=0.5)
    ap.add_argument("--model", default="llama2-7b")
    ap.add_argument("--reps", type=int, default=400)
    args = ap.parse_args()
    shape = synth.MODELS[args.model]
    n = 4
    qs = [synth.haar_orthogonal(shape.d, 100 + i, device=DEV, dtype=torch.float32) for i in range(n + 1)]
    layers = [M.fold_layer(M.synth_original_layer(shape, i + 1, device=DEV), shape, qs[i], qs[i + 1]) for i in range(n)]
    ctx = 256
    kv = [(synth.gaussian_bf16((1, shape.hkv, ctx, shape.hd), 900 + i, 1.0, DEV),
           synth.gaussian_bf16((1, shape.hkv, ctx, shape.hd), 950 + i, 1.0, DEV)) for i in range(n)]
    pos = torch.full((1,), ctx - 1, dtype=torch.int32, device=DEV)
    resid = synth.residual_activation(1, shape.d, 7).to(DEV)
    wsb = torch.zeros(LZ.layer_workspace_size(layers[0], 1, ctx), dtype=torch.uint8, device=DEV)
    plan = M.site_plan(shape, args.p)

    def timed(mask):
        LZ.lib().larosa_debug_set_layer_phases(mask)
        for i in range(n):
            LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos, chained=i > 0), ws=wsb)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(n):
                LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos, chained=True), ws=wsb)
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = args.reps // n
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        LZ.lib().larosa_debug_set_layer_phases(-1)
        return e0.elapsed_time(e1) * 1e3 / (reps * n)

    full = timed(-1)
    out = {"model": args.model, "p": args.p, "plan": list(plan), "layer_us": round(full, 2), "marginal_us": {}}
    for name, bit in BITS.items():
        out["marginal_us"][name] = round(full - timed(-1 & ~(1 << bit)), 2)
    out["gemv_only_us"] = round(timed(sum(1 << b for k, b in BITS.items() if k != "attention")), 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
