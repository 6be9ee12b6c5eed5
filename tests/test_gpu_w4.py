"""GPU parity of the W4A16 path: larosa_quantize_w4 codes and scales
bit-identical to the oracle's quantisation (integer decisions in fp32 on both sides), and the
fused Top-K + int4 sparse GEMV against the oracle's masked GEMV over the dequantised weights."""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from paper_2507_01299_b200 import larosa as LZ

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def unpack(Wq):
    b = Wq.cpu().numpy()
    q = np.empty((b.shape[0], b.shape[1] * 2), dtype=np.uint8)
    q[:, 0::2] = b & 15
    q[:, 1::2] = b >> 4
    return q


@pytest.mark.parametrize("d_in,d_out", [(64, 256), (4096, 4096), (1000, 12288)])
def test_quantize_w4_bit_exact(d_in, d_out):
    W = synth.gaussian_bf16((d_in, d_out), 21 + d_in, d_in ** -0.5)
    W[3, :128] = 0   # an all-zero group
    Wq, S = LZ.quantize_w4(W.to(DEV))
    q_ref, s_ref = O.quantize_w4(W.numpy().view(np.uint16))
    assert np.array_equal(unpack(Wq), q_ref)
    assert np.array_equal(S.cpu().numpy().view(np.uint16), s_ref)


@pytest.mark.parametrize("d_in,d_out,k,eps", [(64, 256, 32, -1.0), (4096, 4096, 2048, 1e-5), (4096, 12288, 2048, 1e-5),
                                              (11008, 4096, 5504, -1.0), (4096, 22016 // 256 * 256, 1638, 1e-5),
                                              (1000, 512, 0, -1.0), (1000, 512, 1000, -1.0)])
def test_topk_sparse_gemv_w4_p3(d_in, d_out, k, eps):
    x = synth.residual_activation(1, d_in, seed=d_in + k)[0]
    W = synth.gaussian_bf16((d_in, d_out), 40 + d_in, d_in ** -0.5)
    Wq, S = LZ.quantize_w4(W.to(DEV))
    y = LZ.topk_sparse_gemv_w4(x.to(DEV), k, Wq, S, rms_eps=eps)
    q, s = O.quantize_w4(W.numpy().view(np.uint16))
    wd = O.dequantize_w4(q, s)
    xd = x.numpy().astype(np.float64)
    idx = O.topk(xd, k)
    sc = O.rms_scale(xd, eps) if eps >= 0 else 1.0
    ref = O.sparse_gemv(wd, idx, xd[idx] * sc)
    got = y.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(got - ref)) <= 1e-5 * max(np.linalg.norm(ref), 1e-30)
    # repeatable
    assert torch.equal(LZ.topk_sparse_gemv_w4(x.to(DEV), k, Wq, S, rms_eps=eps), y)
