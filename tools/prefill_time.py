"""Time larosa_prefill_sparse_gemm (N2) vs cuBLAS dense bf16 on LLaMA2-7B gate|up (512 tokens, p=0.5)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import bench_extras as BX
from paper_2507_01299_b200 import model as M
dev = "cuda:0"
shape = synth.MODELS["llama2-7b"]
orig = M.synth_original_layer(shape, 1, device=dev)
q = synth.haar_orthogonal(shape.d, 2, device=dev, dtype=torch.float32)
lw = M.fold_layer(orig, shape, q, q)
res = {}
for n in (128, 512, 2048):
    res[n] = BX.prefill_extra([lw], shape, dev, n_tok=n)
print(json.dumps(res))
