"""Standalone sparse-GEMV probe for ncu (no QR / fold noise): a few back-to-back
larosa_sparse_gemv launches on one LLaMA2-7B-shaped weight per site.
  python tools/probe_gemv.py [site ...]   sites: qkv o gate_up down adapter"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01299_b200 import larosa as LZ  # noqa: E402

SITES = {"qkv": (4096, 12288, 2048), "o": (4096, 4096, 2048), "gate_up": (4096, 22016, 2048),
         "down": (11008, 4096, 5504), "adapter": (4096, 4096, 4096)}


def main():
    names = sys.argv[1:] or list(SITES)
    dev = "cuda:0"
    for name in names:
        din, dout, k = SITES[name]
        ws = [synth.gaussian_bf16((din, dout), i, din ** -0.5, dev) for i in range(4)]
        ins = []
        for r in range(4):
            x = synth.residual_activation(1, din, 300 + r).to(dev)
            _, idx, vals, _ = LZ.rotate_topk(x, None, k)
            ins.append((idx, vals))
        y = torch.empty((1, dout), device=dev)
        for i in range(6):
            LZ.sparse_gemv(ws[i % 4], *ins[i % 4], out=y)
        torch.cuda.synchronize()
    print("probe ok")


if __name__ == "__main__":
    main()
