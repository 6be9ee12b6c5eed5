"""Seeded synthetic input generators shared by tests/, bench.py and smoke().

This module holds NONE of LaRoSA's arithmetic (no rotation construction from data,
no fold, no Top-K, no GEMV, no k-rule): it only draws random numbers with the
shapes and distributions of the paper's workloads (DESIGN.md §5 "input recipe")
and returns them as torch CPU tensors / raw bf16 bit patterns.  Both the CUDA
path and the oracle consume what it returns; neither is imported here.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

__all__ = ["ModelShape", "MODELS", "PAPER_ALPHA", "gen", "gaussian", "gaussian_bf16",
           "haar_orthogonal", "residual_activation", "toy_calibration", "bf16_bits",
           "correlated_batch"]


@dataclass(frozen=True)
class ModelShape:
    """Public HF config shapes of the paper's models (no paper content
    beyond M = I/D)."""
    name: str
    d: int
    inter: int
    hq: int
    hkv: int
    hd: int
    layers: int
    vocab: int
    qkv_bias: bool
    rms_eps: float
    rope_theta: float

    @property
    def qkv_out(self) -> int:
        return (self.hq + 2 * self.hkv) * self.hd


MODELS = {
    "toy": ModelShape("toy", 64, 128, 4, 2, 16, 2, 256, False, 1e-6, 10000.0),
    "llama2-7b": ModelShape("llama2-7b", 4096, 11008, 32, 32, 128, 32, 32000, False, 1e-5, 10000.0),
    "llama3-8b": ModelShape("llama3-8b", 4096, 14336, 32, 8, 128, 32, 128256, False, 1e-5, 500000.0),
    "mistral-7b": ModelShape("mistral-7b", 4096, 14336, 32, 8, 128, 32, 32768, False, 1e-5, 1000000.0),
    "qwen2.5-7b": ModelShape("qwen2.5-7b", 3584, 18944, 28, 4, 128, 28, 152064, True, 1e-6, 1000000.0),
    "llama3-70b": ModelShape("llama3-70b", 8192, 28672, 64, 8, 128, 80, 128256, False, 1e-5, 500000.0),
    "qwen2.5-72b": ModelShape("qwen2.5-72b", 8192, 29568, 64, 8, 128, 80, 152064, True, 1e-6, 1000000.0),
}

# (alpha1, alpha3) from the App. B optimal-coefficient table; alpha2 and
# alpha4 are derived by the constraint solver of whichever side uses them.
PAPER_ALPHA = {
    "llama2-7b": (0.90, 0.80),
    "llama3-8b": (0.80, 0.80),
    "llama3-70b": (0.85, 0.75),
    "mistral-7b": (1.00, 0.80),
    "qwen2.5-7b": (0.80, 0.80),
    "qwen2.5-72b": (0.80, 0.80),
}


def gen(seed: int, device: str = "cpu") -> torch.Generator:
    return torch.Generator(device=device).manual_seed(int(seed))


def gaussian(shape, seed: int, std: float = 1.0, dtype=torch.float32, device: str = "cpu") -> torch.Tensor:
    return torch.randn(shape, generator=gen(seed, device), dtype=dtype, device=device) * std


def bf16_bits(t: torch.Tensor) -> torch.Tensor:
    """Round a float tensor to bf16 (torch's RNE) and return the raw bits as int16."""
    return t.to(torch.bfloat16).view(torch.int16)


def gaussian_bf16(shape, seed: int, std: float, device: str = "cpu") -> torch.Tensor:
    """N(0, std^2) weights rounded to bf16; returned as raw int16 bits [SURVEY §8(d) C2]."""
    return bf16_bits(gaussian(shape, seed, std, device=device))


def haar_orthogonal(d: int, seed: int, device: str = "cpu", dtype=torch.float64) -> torch.Tensor:
    """A Haar-random orthogonal matrix (QR of a Gaussian, R-diagonal sign fixed).
    Stands in for a PCA rotation at model size (Q is an input there)."""
    a = torch.randn((d, d), generator=gen(seed, device), dtype=dtype, device=device)
    q, r = torch.linalg.qr(a)
    return (q * torch.sign(torch.diagonal(r)).unsqueeze(0)).contiguous()


def residual_activation(batch: int, d: int, seed: int, outlier_frac: float = 0.005,
                        outlier_scale: float = 20.0) -> torch.Tensor:
    """Residual-stream-like token vectors: N(0, 1) with a fixed 0.5% of channels scaled
    x20 (massive-activation outlier channels) [SURVEY §8(d) C2]. fp32 [batch, d]."""
    x = gaussian((batch, d), seed)
    n_out = max(1, int(round(outlier_frac * d)))
    ch = torch.randperm(d, generator=gen(seed + 7919))[:n_out]
    x[:, ch] *= outlier_scale
    return x


def correlated_batch(batch: int, d: int, seed: int, spread: float = 0.5) -> torch.Tensor:
    """Regime R2 of SURVEY §8(d) C3: x_b = mu + spread * z_b (tokens share a direction,
    so their Top-K sets overlap)."""
    mu = gaussian((1, d), seed)
    return mu + spread * gaussian((batch, d), seed + 1)


def toy_calibration(d: int = 64, n_seq: int = 16, n_tok: int = 16, seed: int = 11):
    """Toy calibration set of SURVEY §8(d) C1: x = (z * sigma) R0^T, z ~ N(0, I),
    sigma_i = 2^(-i/8) (distinct eigenvalues), R0 Haar-orthogonal.  Returns a list of
    n_seq float64 [n_tok, d] arrays' torch tensors."""
    r0 = haar_orthogonal(d, seed)
    sigma = torch.pow(2.0, -torch.arange(d, dtype=torch.float64) / 8.0)
    g = gen(seed + 1)
    out = []
    for _ in range(n_seq):
        z = torch.randn((n_tok, d), generator=g, dtype=torch.float64)
        out.append((z * sigma) @ r0.T)
    return out
