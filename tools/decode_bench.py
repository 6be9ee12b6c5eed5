"""LLaMA3-8B-shaped full decode step: 32 folded random-init layers + LM head,
batch 1/4/16, p = 0.4 uniform alpha (and p = 0 for the overhead), KV context 256, one CUDA
graph per step; prints one JSON line with tok/s per batch."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01299_b200 import model as M  # noqa: E402


def time_graph(g, reps):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--batches", default="1,4,16")
    ap.add_argument("--ps", default="0.4,0.0")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    shape = synth.MODELS[args.model]
    L = args.layers or shape.layers
    dev = "cuda:0"
    model = M.synth_decode_model(shape, L, dev, seed=1)
    torch.cuda.synchronize()
    out = {"model": args.model, "layers": L, "ctx": 256, "results": {}}
    for B in [int(b) for b in args.batches.split(",")]:
        run = M.DecodeRunner(model, B, 256, dev)
        for kc, vc in run.kv:
            kc.copy_(synth.gaussian_bf16(kc.shape, 5, 1.0, dev))
            vc.copy_(synth.gaussian_bf16(vc.shape, 6, 1.0, dev))
        run.tokens.copy_(torch.arange(B, dtype=torch.int32) * 37 + 11)
        run.pos.fill_(255)
        for p in [float(x) for x in args.ps.split(",")]:
            plan = M.site_plan(shape, p)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                run.step(plan)
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                run.step(plan)
            ms = time_graph(g, args.reps)
            out["results"][f"B{B}_p{p}"] = {"ms_per_step": round(ms, 4), "tok_s": round(B * 1e3 / ms, 1),
                                            "plan": list(plan)}
        del run
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
