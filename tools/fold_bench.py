"""Time larosa_fold_rotation (tcgen05 vs CUDA-core) on LLaMA2-7B layer shapes; prints JSON.
FLOPs counted as 2 * M * N * K of the mathematical fold (the hi/lo split doubles the MMAs)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402


def main():
    dev = "cuda:0"
    d = 4096
    q = synth.haar_orthogonal(d, 1, device=dev, dtype=torch.float32)
    g = torch.ones(d, device=dev)
    res = {}
    for name, rows, cols, side in (("w_qkv (left)", 4096, 12288, 0), ("w_down (right)", 11008, 4096, 1)):
        W = synth.gaussian_bf16((rows, cols), 2, 0.02, dev)
        out = torch.empty_like(W)
        for simt in (0, 1):
            os.environ["LAROSA_FOLD_SIMT"] = str(simt)
            LZ.fold_rotation(q, W, side, gamma=g if side == 0 else None, out=out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record()
            for _ in range(reps):
                LZ.fold_rotation(q, W, side, gamma=g if side == 0 else None, out=out)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            flops = 2.0 * rows * cols * d
            res[f"{name} {'simt' if simt else 'tcgen05'}"] = {"ms": round(ms, 3), "tflops": round(flops / ms / 1e9, 1)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
