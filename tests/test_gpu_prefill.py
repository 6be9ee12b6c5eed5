"""GPU parity of the prefill path: every prompt token keeps its own exact
Top-K (index sets bit-identical to the oracle's Top-K per token, checked through a one-hot
weight) and the outputs match the oracle's per-token masked GEMV."""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from paper_2507_01299_b200 import larosa as LZ

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def w64(bits):
    return O.bf16_to_f64(bits.detach().cpu().numpy().view(np.uint16))


@pytest.mark.parametrize("n,d_in,d_out,k,eps", [(40, 4096, 4096, 2048, 1e-5), (1, 64, 128, 32, -1.0),
                                                (128, 11008, 4096, 5504, -1.0), (17, 1000, 256, 0, -1.0),
                                                (33, 1000, 256, 1000, 1e-6)])
def test_prefill_vs_oracle(n, d_in, d_out, k, eps):
    X = torch.stack([synth.residual_activation(1, d_in, seed=100 + t)[0] for t in range(n)])
    W = synth.gaussian_bf16((d_in, d_out), 5 + d_in, d_in ** -0.5)
    Y = LZ.prefill_sparse_gemm(X.to(DEV), k, W.to(DEV), rms_eps=eps).cpu().numpy().astype(np.float64)
    Wf = w64(W)
    for t in range(n):
        x = X[t].numpy().astype(np.float64)
        idx = O.topk(x, k)
        s = O.rms_scale(x, eps) if eps >= 0 else 1.0
        ref = O.sparse_gemv(Wf, idx, x[idx] * s)
        assert np.max(np.abs(Y[t] - ref)) <= 1e-5 * max(np.linalg.norm(ref), 1e-30), t


def test_prefill_kept_sets_exact():
    """Integer-valued tokens with ties and a one-hot-coded weight: y identifies the kept set."""
    n, d, k = 24, 256, 100
    g = torch.Generator().manual_seed(4)
    X = torch.randint(-4, 5, (n, d), generator=g).float()
    W = torch.zeros((d, d), dtype=torch.bfloat16)
    W[torch.arange(d), torch.arange(d)] = 1.0
    Wb = W.view(torch.int16).contiguous()
    Y = LZ.prefill_sparse_gemm(X.to(DEV), k, Wb.to(DEV)).cpu().numpy()
    for t in range(n):
        x = X[t].numpy().astype(np.float64)
        ref = np.zeros(d)
        idx = O.topk(x, k)
        ref[idx] = x[idx]
        assert np.array_equal(Y[t], ref.astype(np.float32)), t
