"""Per-call device timing of the C-ABI calls (CUDA graphs of back-to-back launches, CUDA
events): sparse GEMV per LLaMA2-7B site, rotate_topk (Top-K only) per site width, and one
decoder block.  Prints one JSON line.   python tools/micro.py [--p 0.5] [--reps 64]"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402
from paper_2507_01299_b200 import model as M  # noqa: E402

DEV = "cuda:0"


def graph_time(fn, reps, rounds=5):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(rounds):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (rounds * reps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=float, default=0.5)
    ap.add_argument("--reps", type=int, default=64)
    ap.add_argument("--what", default="gemv,topk,layer")
    args = ap.parse_args()
    shape = synth.MODELS["llama2-7b"]
    plan = M.site_plan(shape, args.p)
    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("LAROSA_")}}
    what = args.what.split(",")
    nq = shape.hq * shape.hd
    if "gemv" in what:
        sites = {"qkv": (shape.d, shape.qkv_out, plan[0]), "o": (nq, shape.d, plan[1]),
                 "gate_up": (shape.d, 2 * shape.inter, plan[2]), "down": (shape.inter, shape.d, plan[3]),
                 "adapter": (shape.d, shape.d, shape.d), "o_k16": (nq, shape.d, 16), "o_k256": (nq, shape.d, 256)}
        res = {}
        for name, (din, dout, k) in sites.items():
            ws = [synth.gaussian_bf16((din, dout), 10 * i + 1, din ** -0.5, DEV) for i in range(8)]
            ins = []
            for r in range(8):
                x = synth.residual_activation(1, din, 300 + r).to(DEV)
                _, idx, vals, _ = LZ.rotate_topk(x, None, k)
                ins.append((idx, vals))
            y = torch.empty((1, dout), device=DEV)
            us = graph_time(lambda i: LZ.sparse_gemv(ws[i % 8], *ins[i % 8], out=y), args.reps)
            byt = k * dout * 2
            info = (ctypes.c_int32 * 8)()
            LZ.lib().larosa_gemv_plan_info(ctypes.c_int64(dout), ctypes.c_int64(k), 1, info)  # see larosa.h
            res[name] = {"us": round(us, 2), "GBps": round(byt / us / 1e3, 1), "plan": list(info)}
            del ws
        out["gemv"] = res
    if "topk" in what:
        res = {}
        for d, k in ((4096, plan[0]), (11008, plan[3])):
            xs = [synth.residual_activation(1, d, 400 + r).to(DEV) for r in range(8)]
            idx = torch.empty((1, k), dtype=torch.int32, device=DEV)
            vals = torch.empty((1, k), device=DEV)
            L = LZ.lib()
            nb = L.larosa_rotate_topk_workspace_size(1, d)
            wsb = torch.zeros(nb, dtype=torch.uint8, device=DEV)

            def f(i):
                LZ._check(L.larosa_rotate_topk(LZ._ptr(xs[i % 8]), None, 1, d, k, 1e-5, None, LZ._ptr(idx),
                                               LZ._ptr(vals), None, LZ._ptr(wsb), wsb.numel(), LZ._stream()))
            res[f"d{d}"] = round(graph_time(f, args.reps), 2)
        out["topk_us"] = res
    if "layer" in what:
        layers = []
        qs = [synth.haar_orthogonal(shape.d, 100 + i, device=DEV, dtype=torch.float32) for i in range(5)]
        for i in range(4):
            layers.append(M.fold_layer(M.synth_original_layer(shape, i + 1, device=DEV), shape, qs[i], qs[i + 1]))
        ctx = 256
        kv = [(synth.gaussian_bf16((1, shape.hkv, ctx, shape.hd), 900 + i, 1.0, DEV),
               synth.gaussian_bf16((1, shape.hkv, ctx, shape.hd), 950 + i, 1.0, DEV)) for i in range(4)]
        pos = torch.full((1,), ctx - 1, dtype=torch.int32, device=DEV)
        resid = synth.residual_activation(1, shape.d, 7).to(DEV)
        wsb = torch.zeros(LZ.layer_workspace_size(layers[0], 1, ctx), dtype=torch.uint8, device=DEV)
        res = {}
        for p in (0.0, 0.5):
            pl = M.site_plan(shape, p)
            us = graph_time(lambda i: LZ.sparse_layer(layers[i % 4], pl, LZ.LayerState(resid, *kv[i % 4], pos),
                                                      ws=wsb), 32)
            res[str(p)] = round(us, 2)
        out["layer_us"] = res
    print(json.dumps(out))


if __name__ == "__main__":
    main()
