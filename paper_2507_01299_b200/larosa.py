"""Thin Python binding of the C ABI in include/larosa.h (ctypes).

Argument marshalling only: every step of the hot path runs in the CUDA kernels of
``lib/liblarosa.so``.  PyTorch provides device memory and the current CUDA stream.
There is no CPU fallback: if the library is missing, or a call is made on CPU
tensors, this module raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LAROSA_LIB") or os.path.join(_HERE, "lib", "liblarosa.so")   # env: experiments only

LAROSA_LEFT_QT = 0
LAROSA_RIGHT_Q = 1
LAROSA_GU_BLOCK = 64
LAROSA_MAX_BATCH = 16

_c_i64 = ctypes.c_int64
_c_i32 = ctypes.c_int32
_vp = ctypes.c_void_p


class LarosaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"status {status}: {msg}")
        self.status = status


class LayerWeightsC(ctypes.Structure):
    _fields_ = [("w_qkv", _vp), ("b_qkv", _vp), ("w_o", _vp), ("w_gu", _vp), ("w_down", _vp),
                ("adapter", _vp), ("d", _c_i64), ("inter", _c_i64), ("n_q_heads", _c_i64),
                ("n_kv_heads", _c_i64), ("head_dim", _c_i64), ("rope_theta", ctypes.c_float),
                ("rms_eps", ctypes.c_float), ("adapter_in_down", _c_i32), ("adapter_mid", _vp),
                ("w4_codes", _vp * 4), ("w4_scales", _vp * 4)]


class LayerPlanC(ctypes.Structure):
    _fields_ = [("k_h1", _c_i64), ("k_h2", _c_i64), ("k_h3", _c_i64), ("k_h4", _c_i64), ("k_next_h1", _c_i64)]


class LayerStateC(ctypes.Structure):
    _fields_ = [("resid", _vp), ("k_cache", _vp), ("v_cache", _vp), ("pos", _vp),
                ("max_ctx", _c_i64), ("batch", _c_i32), ("chained", _c_i32), ("host_in", _vp), ("host_out", _vp)]


class LayerTapsC(ctypes.Structure):
    _fields_ = [("idx_h1", _vp), ("vals_h1", _vp), ("q", _vp), ("h2", _vp), ("idx_h2", _vp),
                ("vals_h2", _vp), ("r_mid", _vp), ("idx_h3", _vp), ("vals_h3", _vp), ("h4", _vp),
                ("idx_h4", _vp), ("vals_h4", _vp), ("r_out", _vp)]


class ShardC(ctypes.Structure):
    _fields_ = [("rank", _c_i32), ("world", _c_i32), ("batch", _c_i32), ("peer_dst", _vp), ("peer_flag", _vp),
                ("peer_ld", _c_i64)]


_LIB = None


def lib() -> ctypes.CDLL:
    """Load the in-tree liblarosa.so (raises if it was not built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"liblarosa.so not built ({LIB_PATH}); run __graft_entry__.build() or `make`")
    L = ctypes.CDLL(LIB_PATH)
    L.larosa_abi_version.restype = ctypes.c_int
    L.larosa_status_string.restype = ctypes.c_char_p
    L.larosa_status_string.argtypes = [ctypes.c_int]
    L.larosa_last_error.restype = ctypes.c_char_p
    L.larosa_compute_k.argtypes = [ctypes.c_double, ctypes.c_double, _c_i64, ctypes.POINTER(_c_i64)]
    L.larosa_solve_alpha.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    L.larosa_fold_workspace_size.restype = ctypes.c_size_t
    L.larosa_fold_workspace_size.argtypes = [_c_i64, _c_i64, ctypes.c_int]
    L.larosa_fold_rotation.argtypes = [_vp, _vp, _vp, _vp, _c_i64, _c_i64, ctypes.c_int, _vp, ctypes.c_size_t, _vp]
    L.larosa_pack_gate_up.argtypes = [_vp, _vp, _vp, _c_i64, _c_i64, _vp]
    L.larosa_residual_adapter_workspace_size.restype = ctypes.c_size_t
    L.larosa_residual_adapter_workspace_size.argtypes = [_c_i64]
    L.larosa_residual_adapter.argtypes = [_vp, _vp, _vp, _c_i64, _vp, ctypes.c_size_t, _vp]
    L.larosa_rotate_topk_workspace_size.restype = ctypes.c_size_t
    L.larosa_rotate_topk_workspace_size.argtypes = [_c_i32, _c_i64]
    L.larosa_rotate_topk.argtypes = [_vp, _vp, _c_i32, _c_i64, _c_i64, ctypes.c_float, _vp, _vp, _vp, _vp, _vp,
                                     ctypes.c_size_t, _vp]
    L.larosa_sparse_gemv_workspace_size.restype = ctypes.c_size_t
    L.larosa_sparse_gemv_workspace_size.argtypes = [_c_i32, _c_i64, _c_i64, _c_i64]
    L.larosa_sparse_gemv.argtypes = [_vp, _c_i64, _c_i64, _c_i64, _vp, _vp, _c_i32, _c_i64, _vp, _vp, _vp,
                                     ctypes.c_size_t, _vp]
    L.larosa_topk_sparse_gemv_workspace_size.restype = ctypes.c_size_t
    L.larosa_topk_sparse_gemv_workspace_size.argtypes = [_c_i64, _c_i64]
    L.larosa_topk_sparse_gemv.argtypes = [_vp, _c_i64, _c_i64, ctypes.c_float, _vp, _c_i64, _c_i64, _vp, _vp,
                                          _c_i32, _vp, ctypes.c_size_t, _vp]
    L.larosa_topk_sparse_gemv_dense2.argtypes = [_vp, _c_i64, _c_i64, ctypes.c_float, _vp, _c_i64, _c_i64, _vp, _vp,
                                                 _c_i64, _vp, _c_i32, _vp, ctypes.c_size_t, _vp]
    L.larosa_embed.argtypes = [_vp, _c_i64, _c_i64, _vp, _c_i32, _vp, _vp]
    L.larosa_quantize_w4.argtypes = [_vp, _c_i64, _c_i64, _vp, _vp, _vp]
    L.larosa_topk_sparse_gemv_w4_workspace_size.restype = ctypes.c_size_t
    L.larosa_topk_sparse_gemv_w4_workspace_size.argtypes = [_c_i64, _c_i64]
    L.larosa_topk_sparse_gemv_w4.argtypes = [_vp, _c_i64, _c_i64, ctypes.c_float, _vp, _vp, _c_i64, _vp, _c_i32, _vp,
                                             ctypes.c_size_t, _vp]
    L.larosa_prefill_sparse_gemm_workspace_size.restype = ctypes.c_size_t
    L.larosa_prefill_sparse_gemm_workspace_size.argtypes = [_c_i64, _c_i64, _c_i32]
    L.larosa_prefill_sparse_gemm.argtypes = [_vp, _c_i64, _c_i64, _c_i64, ctypes.c_float, _vp, _c_i64, _vp, _c_i32,
                                             _vp, ctypes.c_size_t, _vp]
    L.larosa_calib_covariance_workspace_size.restype = ctypes.c_size_t
    L.larosa_calib_covariance_workspace_size.argtypes = [_c_i64, _c_i64]
    L.larosa_calib_covariance.argtypes = [_vp, _c_i64, _c_i64, ctypes.c_float, _c_i32, _vp, _vp, ctypes.c_size_t, _vp]
    L.larosa_pca_rotation_workspace_size.restype = ctypes.c_size_t
    L.larosa_pca_rotation_workspace_size.argtypes = [_c_i64]
    L.larosa_pca_rotation.argtypes = [_vp, _c_i64, _vp, _vp, _vp, ctypes.c_size_t, _vp]
    L.larosa_lm_head_workspace_size.restype = ctypes.c_size_t
    L.larosa_lm_head_workspace_size.argtypes = [_c_i32, _c_i64, _c_i64]
    L.larosa_lm_head.argtypes = [_vp, _c_i32, _c_i64, _vp, _c_i64, ctypes.c_float, _vp, _vp, _vp, ctypes.c_size_t, _vp]
    L.larosa_shard_workspace_size.restype = ctypes.c_size_t
    L.larosa_shard_workspace_size.argtypes = [ctypes.POINTER(LayerWeightsC), ctypes.POINTER(ShardC), _c_i64]
    L.larosa_sparse_layer_shard_phase.argtypes = [ctypes.POINTER(LayerWeightsC), ctypes.POINTER(LayerPlanC),
                                                  ctypes.POINTER(ShardC), _c_i32, _vp, _vp, _vp, _vp, _vp, _vp,
                                                  _c_i64, _vp, ctypes.c_size_t, _vp]
    L.larosa_shard_gather_permute.argtypes = [_vp, _c_i32, _c_i32, _c_i64, _vp, _vp]
    L.larosa_shard_wait.argtypes = [_vp, _vp, ctypes.c_uint32, _vp]
    L.larosa_peer_push.argtypes = [_vp, _c_i32, _c_i64, _c_i64, _vp, _vp, _c_i32, _c_i64, _vp]
    L.larosa_error_flags.argtypes = [_vp, _c_i32, ctypes.POINTER(ctypes.c_uint32), _vp]
    L.larosa_error_flags.restype = ctypes.c_int
    L.larosa_argmax.argtypes = [_vp, _c_i32, _c_i64, _c_i64, _vp, _vp]
    L.larosa_debug_set_layer_phases.argtypes = [ctypes.c_int]
    L.larosa_debug_set_layer_phases.restype = None
    L.larosa_gemv_plan_info.argtypes = [_c_i64, _c_i64, _c_i32, ctypes.POINTER(_c_i32)]
    L.larosa_gemv_plan_info.restype = ctypes.c_int
    L.larosa_layer_workspace_size.restype = ctypes.c_size_t
    L.larosa_layer_workspace_size.argtypes = [ctypes.POINTER(LayerWeightsC), _c_i32, _c_i64]
    L.larosa_sparse_layer.argtypes = [ctypes.POINTER(LayerWeightsC), ctypes.POINTER(LayerPlanC),
                                      ctypes.POINTER(LayerStateC), ctypes.POINTER(LayerTapsC), _vp,
                                      ctypes.c_size_t, _vp]
    for name in ("larosa_compute_k", "larosa_solve_alpha", "larosa_fold_rotation", "larosa_pack_gate_up",
                 "larosa_residual_adapter",
                 "larosa_rotate_topk", "larosa_sparse_gemv", "larosa_topk_sparse_gemv", "larosa_sparse_layer",
                 "larosa_embed", "larosa_lm_head", "larosa_sparse_layer_shard_phase", "larosa_shard_gather_permute",
                 "larosa_argmax", "larosa_shard_wait", "larosa_peer_push"):
        getattr(L, name).restype = ctypes.c_int
    if L.larosa_abi_version() != 7:
        raise RuntimeError("liblarosa ABI version mismatch")
    _LIB = L
    return L


def _check(status: int):
    if status != 0:
        L = lib()
        raise LarosaError(status, f"{L.larosa_status_string(status).decode()} — {L.larosa_last_error().decode()}")


def _host_ptr(t: Optional[torch.Tensor]):
    """Pinned host tensor -> its address (device-accessible under unified addressing)."""
    if t is None:
        return None
    if t.is_cuda or not t.is_pinned() or not t.is_contiguous():
        raise ValueError("larosa: host buffers must be contiguous pinned host tensors")
    return ctypes.c_void_p(t.data_ptr())


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("larosa: tensors must live on a CUDA device (no CPU path)")
    if not t.is_contiguous():
        raise ValueError("larosa: tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class Workspace:
    """A zero-initialised device byte buffer reused across calls (kernels keep its tile
    counters self-resetting).  Not for concurrent calls."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != torch.device(device):
            self.buf = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)
        return self.buf


_WS = {}


def _ws(tag, nbytes: int, device) -> torch.Tensor:
    """Workspace per (call kind, shape signature): the library keeps accumulators zero
    between calls only for a fixed layout."""
    key = (tag, str(device))
    if key not in _WS:
        _WS[key] = Workspace()
    return _WS[key].get(nbytes, device)


# ------------------------------------------------------------------------------- host helpers
def abi_version() -> int:
    return lib().larosa_abi_version()


def compute_k(alpha: float, p: float, d_in: int) -> int:
    k = _c_i64(0)
    _check(lib().larosa_compute_k(float(alpha), float(p), int(d_in), ctypes.byref(k)))
    return k.value


def solve_alpha(alpha1: float, alpha3: float, m: float):
    a2, a4 = ctypes.c_double(0), ctypes.c_double(0)
    _check(lib().larosa_solve_alpha(float(alpha1), float(alpha3), float(m), ctypes.byref(a2), ctypes.byref(a4)))
    return a2.value, a4.value


# ------------------------------------------------------------------------------- device calls
def fold_rotation(Q: torch.Tensor, W: torch.Tensor, side: int, gamma: Optional[torch.Tensor] = None,
                  out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """LEFT_QT: Q^T diag(gamma) W; RIGHT_Q: W Q.  Q fp32 [d,d]; W bf16 bits (int16) [rows, cols]."""
    assert Q.dtype == torch.float32 and W.dtype in (torch.int16, torch.bfloat16)
    rows, cols = W.shape
    out = out if out is not None else torch.empty((rows, cols), dtype=torch.int16, device=W.device)
    L = lib()
    nb = L.larosa_fold_workspace_size(rows, cols, side)
    ws = _ws(("fold", rows, cols, side), nb, W.device)
    _check(L.larosa_fold_rotation(_ptr(Q), _ptr(gamma), _ptr(W), _ptr(out), rows, cols, side, _ptr(ws),
                                  ws.numel(), _stream(stream)))
    return out


def residual_adapter(Q_l: torch.Tensor, Q_next: torch.Tensor, out: Optional[torch.Tensor] = None,
                     stream=None) -> torch.Tensor:
    """A_l = Q_l^T Q_next with both fp32 factors split hi + lo, rounded to bf16 once."""
    assert Q_l.dtype == torch.float32 and Q_next.dtype == torch.float32 and Q_l.shape == Q_next.shape
    d = Q_l.shape[0]
    out = out if out is not None else torch.empty((d, d), dtype=torch.int16, device=Q_l.device)
    L = lib()
    nb = L.larosa_residual_adapter_workspace_size(d)
    ws = _ws(("adapter", d), nb, Q_l.device)
    _check(L.larosa_residual_adapter(_ptr(Q_l.contiguous()), _ptr(Q_next.contiguous()), _ptr(out), d, _ptr(ws),
                                     ws.numel(), _stream(stream)))
    return out


def pack_gate_up(Wg: torch.Tensor, Wu: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    d, inter = Wg.shape
    out = out if out is not None else torch.empty((d, 2 * inter), dtype=torch.int16, device=Wg.device)
    _check(lib().larosa_pack_gate_up(_ptr(Wg), _ptr(Wu), _ptr(out), d, inter, _stream(stream)))
    return out


def rotate_topk(x: torch.Tensor, R: Optional[torch.Tensor], k: int, rms_eps: float = -1.0,
                want_xr: bool = False, want_mask: bool = False, stream=None):
    """Returns (xr or None, idx [B,k] int32, vals [B,k] f32, mask [B,ceil(d/32)] int32 or None)."""
    assert x.dtype == torch.float32 and x.dim() == 2
    B, d = x.shape
    dev = x.device
    xr = torch.empty((B, d), dtype=torch.float32, device=dev) if want_xr else None
    idx = torch.empty((B, k), dtype=torch.int32, device=dev)
    vals = torch.empty((B, k), dtype=torch.float32, device=dev)
    mask = torch.empty((B, (d + 31) // 32), dtype=torch.int32, device=dev) if want_mask else None
    L = lib()
    nb = L.larosa_rotate_topk_workspace_size(B, d)
    ws = _ws(("rotate_topk", B, d), nb, dev)
    _check(L.larosa_rotate_topk(_ptr(x), _ptr(R), B, d, k, float(rms_eps), _ptr(xr), _ptr(idx), _ptr(vals),
                                _ptr(mask), _ptr(ws), ws.numel(), _stream(stream)))
    return xr, idx, vals, mask


def sparse_gemv(W: torch.Tensor, idx: torch.Tensor, vals: torch.Tensor, bias: Optional[torch.Tensor] = None,
                d_out: Optional[int] = None, out: Optional[torch.Tensor] = None, ws: Optional[torch.Tensor] = None,
                stream=None) -> torch.Tensor:
    """y[b] = bias + sum_t vals[b,t] W[idx[b,t]]  (W: bf16 bits [d_in, ld])."""
    d_in, ld = W.shape
    d_out = ld if d_out is None else d_out
    if idx.dim() == 1:
        idx, vals = idx.unsqueeze(0), vals.unsqueeze(0)
    B, k = idx.shape
    dev = W.device
    y = out if out is not None else torch.empty((B, d_out), dtype=torch.float32, device=dev)
    L = lib()
    nb = L.larosa_sparse_gemv_workspace_size(B, d_in, k, d_out)
    if ws is None:
        ws = _ws(("sparse_gemv", B, d_in, d_out), nb, dev)
    _check(L.larosa_sparse_gemv(_ptr(W), d_in, d_out, ld, _ptr(idx) if k else None, _ptr(vals) if k else None,
                                B, k, _ptr(bias), _ptr(y), _ptr(ws), ws.numel(), _stream(stream)))
    return y


def topk_sparse_gemv_workspace(d_in: int, d_out: int, device) -> torch.Tensor:
    return torch.zeros(lib().larosa_topk_sparse_gemv_workspace_size(d_in, d_out), dtype=torch.uint8, device=device)


def topk_sparse_gemv(x: torch.Tensor, k: int, W: torch.Tensor, rms_eps: float = -1.0,
                     bias: Optional[torch.Tensor] = None, d_out: Optional[int] = None,
                     out: Optional[torch.Tensor] = None, ws: Optional[torch.Tensor] = None, prepared: bool = False,
                     stream=None) -> torch.Tensor:
    """Batch 1: y = bias + sum_{j in TopK_k(|x|)} x_j s W[j]  (selection fused into the GEMV).
    prepared=True: ``ws`` already holds x's selection data (only the GEMV kernel launches)."""
    x = x.reshape(-1)
    d_in, ld = W.shape
    d_out = ld if d_out is None else d_out
    assert x.dtype == torch.float32 and x.numel() == d_in
    y = out if out is not None else torch.empty((d_out,), dtype=torch.float32, device=W.device)
    L = lib()
    nb = L.larosa_topk_sparse_gemv_workspace_size(d_in, d_out)
    if ws is None:
        ws = _ws(("topk_sparse_gemv", d_in, d_out), nb, W.device)
    _check(L.larosa_topk_sparse_gemv(_ptr(x), d_in, int(k), float(rms_eps), _ptr(W), d_out, ld, _ptr(bias), _ptr(y),
                                     int(prepared), _ptr(ws), ws.numel(), _stream(stream)))
    return y


def topk_sparse_gemv_dense2(x: torch.Tensor, k: int, W: torch.Tensor, x2: torch.Tensor, W2: torch.Tensor,
                            rms_eps: float = -1.0, out: Optional[torch.Tensor] = None,
                            ws: Optional[torch.Tensor] = None, prepared: bool = False, stream=None) -> torch.Tensor:
    """Batch 1: y = sum_{j in TopK_k(|x|)} x_j s W[j] + sum_m x2_m W2[m] (the down site with the
    adapter folded beside it; larosa_topk_sparse_gemv_dense2)."""
    x = x.reshape(-1)
    x2 = x2.reshape(-1)
    d_in, ld = W.shape
    d2 = W2.shape[0]
    assert x.dtype == torch.float32 and x.numel() == d_in and x2.dtype == torch.float32 and x2.numel() == d2
    assert W2.shape[1] == ld
    y = out if out is not None else torch.empty((ld,), dtype=torch.float32, device=W.device)
    L = lib()
    nb = L.larosa_topk_sparse_gemv_workspace_size(d_in, ld)
    if ws is None:
        ws = _ws(("topk_sparse_gemv", d_in, ld), nb, W.device)
    _check(L.larosa_topk_sparse_gemv_dense2(_ptr(x), d_in, int(k), float(rms_eps), _ptr(W), ld, ld, _ptr(x2), _ptr(W2),
                                            d2, _ptr(y), int(prepared), _ptr(ws), ws.numel(), _stream(stream)))
    return y


LAROSA_W4_GROUP = 128


def quantize_w4(W: torch.Tensor, stream=None):
    """(Wq uint8 [d_in, d_out/2], S fp16 bits int16 [d_in, d_out/128]) of bf16 bits W [d_in, d_out]
    (larosa_quantize_w4; symmetric int4 per row and group of 128 outputs)."""
    d_in, d_out = W.shape
    Wq = torch.empty((d_in, d_out // 2), dtype=torch.uint8, device=W.device)
    S = torch.empty((d_in, d_out // LAROSA_W4_GROUP), dtype=torch.int16, device=W.device)
    _check(lib().larosa_quantize_w4(_ptr(W), d_in, d_out, _ptr(Wq), _ptr(S), _stream(stream)))
    return Wq, S


def topk_sparse_gemv_w4(x: torch.Tensor, k: int, Wq: torch.Tensor, S: torch.Tensor, rms_eps: float = -1.0,
                        out: Optional[torch.Tensor] = None, ws: Optional[torch.Tensor] = None, prepared: bool = False,
                        stream=None) -> torch.Tensor:
    """Batch 1: y = sum_{j in TopK_k(|x|)} x_j s w4[j] (W4A16 weights; larosa_topk_sparse_gemv_w4)."""
    x = x.reshape(-1)
    d_in = Wq.shape[0]
    d_out = Wq.shape[1] * 2
    y = out if out is not None else torch.empty((d_out,), dtype=torch.float32, device=Wq.device)
    L = lib()
    nb = L.larosa_topk_sparse_gemv_w4_workspace_size(d_in, d_out)
    if ws is None:
        ws = _ws(("topk_sparse_gemv_w4", d_in, d_out), nb, Wq.device)
    _check(L.larosa_topk_sparse_gemv_w4(_ptr(x), d_in, int(k), float(rms_eps), _ptr(Wq), _ptr(S), d_out, _ptr(y),
                                        int(prepared), _ptr(ws), ws.numel(), _stream(stream)))
    return y


def prefill_sparse_gemm(X: torch.Tensor, k: int, W: torch.Tensor, rms_eps: float = -1.0,
                        out: Optional[torch.Tensor] = None, split: bool = False, stream=None) -> torch.Tensor:
    """Y[t] = sum_{j in TopK_k(|X[t]|)} X[t][j] s_t W[j] for every prompt token t (N2).
    split: bf16 hi + lo activations (two MMAs) instead of one bf16 operand."""
    n, d_in = X.shape
    d_out = W.shape[1]
    Y = out if out is not None else torch.empty((n, d_out), dtype=torch.float32, device=W.device)
    L = lib()
    nb = L.larosa_prefill_sparse_gemm_workspace_size(n, d_in, int(split))
    ws = _ws(("prefill", n, d_in, int(split)), nb, W.device)
    _check(L.larosa_prefill_sparse_gemm(_ptr(X.contiguous()), n, d_in, int(k), float(rms_eps), _ptr(W), d_out, _ptr(Y),
                                        int(split), _ptr(ws), ws.numel(), _stream(stream)))
    return Y


def calib_covariance(X: torch.Tensor, scale: float = 1.0, out: Optional[torch.Tensor] = None,
                     accumulate: bool = False, stream=None) -> torch.Tensor:
    """C = scale * X^T X (+ C): X bf16 bits (int16) [n_tok, d] of calibration activations (eq. 1,
    P:380-383; pass scale = 1/M and accumulate over the M sequences)."""
    n, d = X.shape
    C = out if out is not None else torch.zeros((d, d), dtype=torch.float32, device=X.device)
    L = lib()
    nb = L.larosa_calib_covariance_workspace_size(n, d)
    ws = _ws(("calib_cov", n, d), nb, X.device)
    _check(L.larosa_calib_covariance(_ptr(X), n, d, float(scale), int(accumulate), _ptr(C), _ptr(ws), ws.numel(),
                                     _stream(stream)))
    return C


def pca_rotation(C: torch.Tensor, stream=None):
    """(Q, lam): eigenvectors of C as columns, eigenvalues descending, largest-|entry| component
    positive.  Synchronises the stream."""
    d = C.shape[0]
    L = lib()
    nb = L.larosa_pca_rotation_workspace_size(d)
    if nb == 0:
        raise LarosaError(1, "pca_rotation: bad d")
    ws = _ws(("pca", d), nb, C.device)
    Q = torch.empty((d, d), dtype=torch.float32, device=C.device)
    lam = torch.empty((d,), dtype=torch.float32, device=C.device)
    _check(L.larosa_pca_rotation(_ptr(C.contiguous()), d, _ptr(Q), _ptr(lam), _ptr(ws), ws.numel(), _stream(stream)))
    return Q, lam


LAROSA_ERR_KEEP_ALL = 1
LAROSA_ERR_FIX_OVERFLOW = 2


def error_flags(ws: torch.Tensor, clear: bool = True, stream=None) -> int:
    """The workspace's device error bits (LAROSA_ERR_*); synchronises the stream."""
    v = ctypes.c_uint32(0)
    _check(lib().larosa_error_flags(_ptr(ws), int(clear), ctypes.byref(v), _stream(stream)))
    return int(v.value)


_HEADER_WS = ("rotate_topk", "sparse_gemv", "topk_sparse_gemv", "topk_sparse_gemv_w4", "prefill", "pca", "lm_head",
              "layer")   # call kinds whose workspace starts with the counter header (larosa_error_flags)


def workspaces():
    """Every cached workspace buffer of a call kind that carries the error word (for tests)."""
    return [w.buf for (tag, _), w in _WS.items() if w.buf is not None and tag[0] in _HEADER_WS]


def shard_gather_permute(gathered: torch.Tensor, world: int, batch: int, out: torch.Tensor, stream=None):
    """[world][batch][local] (rank-major all-gather) -> out [batch][world * local]."""
    d_local = gathered.numel() // (world * batch)
    _check(lib().larosa_shard_gather_permute(_ptr(gathered), world, batch, d_local, _ptr(out), _stream(stream)))
    return out


@dataclass
class PeerTarget:
    """Where a sharded phase pushes its output (larosa_shard.peer_*): device int64 arrays of every
    rank's destination address (at this rank's first column) and arrival-counter address, and the
    token stride of the destination buffers (floats)."""
    dst: torch.Tensor    # int64 [world] on device
    flag: torch.Tensor   # int64 [world] on device
    ld: int


def shard_wait(flag: torch.Tensor, expected: torch.Tensor, count: int, stream=None):
    """Wait (on the device) until this rank's arrival counter has grown by `count` more values
    (larosa_shard_wait); flag / expected: one-element int32 device tensors."""
    _check(lib().larosa_shard_wait(_ptr(flag), _ptr(expected), ctypes.c_uint32(int(count) & 0xffffffff),
                                   _stream(stream)))


def peer_push(src: torch.Tensor, target: PeerTarget, world: int, stream=None):
    """Push a [batch][d_local] fp32 slice into every rank's buffer + counters (larosa_peer_push)."""
    B, dl = src.shape
    _check(lib().larosa_peer_push(_ptr(src), B, dl, src.stride(0), _ptr(target.dst), _ptr(target.flag), world,
                                  int(target.ld), _stream(stream)))


def argmax(logits: torch.Tensor, out: torch.Tensor, stream=None):
    """out[b] = arg-max of logits[b] (lowest index on ties)."""
    B, n = logits.shape
    _check(lib().larosa_argmax(_ptr(logits), B, n, logits.stride(0), _ptr(out), _stream(stream)))
    return out


def embed(E: torch.Tensor, tokens: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """resid[b] = E'[tokens[b]] (E' = E Q_0, bf16 bits [vocab, d]; tokens int32 [B] on device)."""
    vocab, d = E.shape
    B = tokens.numel()
    out = out if out is not None else torch.empty((B, d), dtype=torch.float32, device=E.device)
    _check(lib().larosa_embed(_ptr(E), vocab, d, _ptr(tokens), B, _ptr(out), _stream(stream)))
    return out


def lm_head(resid: torch.Tensor, H: torch.Tensor, rms_eps: float, logits: Optional[torch.Tensor] = None,
            next_token: Optional[torch.Tensor] = None, ws: Optional[torch.Tensor] = None, stream=None):
    """Final RMS scale + dense head GEMV (H' bf16 bits [d, vocab]) + greedy arg-max.
    Returns (next_token int32 [B], logits fp32 [B, vocab] or None)."""
    B, d = resid.shape
    vocab = H.shape[1]
    dev = resid.device
    nt = next_token if next_token is not None else torch.empty((B,), dtype=torch.int32, device=dev)
    L = lib()
    nb = L.larosa_lm_head_workspace_size(B, d, vocab)
    if ws is None:
        ws = _ws(("lm_head", B, d, vocab), nb, dev)
    _check(L.larosa_lm_head(_ptr(resid), B, d, _ptr(H), vocab, float(rms_eps), _ptr(logits), _ptr(nt), _ptr(ws),
                            ws.numel(), _stream(stream)))
    return nt, logits


@dataclass
class LayerWeights:
    """Folded bf16 (int16-bit) weights of one decoder layer in the Wc layout."""
    w_qkv: torch.Tensor
    w_o: torch.Tensor
    w_gu: torch.Tensor
    w_down: torch.Tensor
    d: int
    inter: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    rope_theta: float
    rms_eps: float
    b_qkv: Optional[torch.Tensor] = None
    adapter: Optional[torch.Tensor] = None
    adapter_in_down: bool = False   # w_down = Wd Q_{l+1}: r_next = r_mid A_l + y_down (larosa.h)
    adapter_mid: Optional[torch.Tensor] = None   # Q_B: A_mid = Q_a^T Q_m beside O (larosa.h)
    # W4A16 sites (ABI 6): per site (QKV, O, gate|up, down) None or (codes, scales) of quantize_w4
    w4: Optional[list] = None

    def c(self) -> LayerWeightsC:
        c = LayerWeightsC(_ptr(self.w_qkv), _ptr(self.b_qkv), _ptr(self.w_o), _ptr(self.w_gu), _ptr(self.w_down),
                          _ptr(self.adapter), self.d, self.inter, self.n_q_heads, self.n_kv_heads, self.head_dim,
                          float(self.rope_theta), float(self.rms_eps), int(self.adapter_in_down),
                          _ptr(self.adapter_mid))
        for j, qs in enumerate(self.w4 or []):
            if qs is not None:
                c.w4_codes[j] = _ptr(qs[0])
                c.w4_scales[j] = _ptr(qs[1])
        return c


@dataclass
class LayerState:
    resid: torch.Tensor      # fp32 [B, d]
    k_cache: torch.Tensor    # int16 [B, Hkv, max_ctx, hd]
    v_cache: torch.Tensor
    pos: torch.Tensor        # int32 [B] on device
    chained: bool = False    # resid was written by the previous layer call on the same workspace
    host_in: Optional[torch.Tensor] = None    # pinned host fp32 [1, d]: the input, read in-kernel
    host_out: Optional[torch.Tensor] = None   # pinned host fp32 [1, d]: the output, written in-kernel

    def c(self) -> LayerStateC:
        B = self.resid.shape[0]
        return LayerStateC(_ptr(self.resid), _ptr(self.k_cache), _ptr(self.v_cache), _ptr(self.pos),
                           self.k_cache.shape[2], B, int(self.chained), _host_ptr(self.host_in),
                           _host_ptr(self.host_out))


TAP_NAMES = [f[0] for f in LayerTapsC._fields_]


def make_taps(w: LayerWeights, plan: Sequence[int], batch: int, device) -> dict:
    k1, k2, k3, k4 = plan
    nq = w.n_q_heads * w.head_dim
    f32 = dict(dtype=torch.float32, device=device)
    i32 = dict(dtype=torch.int32, device=device)
    return {
        "idx_h1": torch.empty((batch, k1), **i32), "vals_h1": torch.empty((batch, k1), **f32),
        "q": torch.empty((batch, nq), **f32), "h2": torch.empty((batch, nq), **f32),
        "idx_h2": torch.empty((batch, k2), **i32), "vals_h2": torch.empty((batch, k2), **f32),
        "r_mid": torch.empty((batch, w.d), **f32),
        "idx_h3": torch.empty((batch, k3), **i32), "vals_h3": torch.empty((batch, k3), **f32),
        "h4": torch.empty((batch, w.inter), **f32),
        "idx_h4": torch.empty((batch, k4), **i32), "vals_h4": torch.empty((batch, k4), **f32),
        "r_out": torch.empty((batch, w.d), **f32),
        "r_in": torch.empty((batch, w.d), **f32),
    }


def layer_workspace_size(w: LayerWeights, batch: int, max_ctx: int) -> int:
    wc = w.c()
    return lib().larosa_layer_workspace_size(ctypes.byref(wc), batch, max_ctx)


def sparse_layer(w: LayerWeights, plan: Sequence[int], state: LayerState, taps: Optional[dict] = None,
                 ws: Optional[torch.Tensor] = None, stream=None):
    """One LaRoSA decoder layer in place on ``state`` (resid, KV cache)."""
    L = lib()
    wc = w.c()
    pc = LayerPlanC(*[int(k) for k in plan[:5]], *([0] if len(plan) < 5 else []))
    sc = state.c()
    B = state.resid.shape[0]
    nb = L.larosa_layer_workspace_size(ctypes.byref(wc), B, state.k_cache.shape[2])
    if ws is None:
        ws = _ws(("layer", w.d, w.inter, w.n_q_heads, w.n_kv_heads, w.head_dim, B, state.k_cache.shape[2]), nb,
                 state.resid.device)
    elif ws.numel() < nb:
        raise ValueError("sparse_layer: workspace too small")
    tc = None
    if taps is not None:
        tc = LayerTapsC(*[_ptr(taps.get(n)) for n in TAP_NAMES])
        if taps.get("r_in") is not None and state.host_in is None:   # debug tap: the layer's input
            with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream()):
                taps["r_in"].copy_(state.resid)
    _check(L.larosa_sparse_layer(ctypes.byref(wc), ctypes.byref(pc), ctypes.byref(sc),
                                 ctypes.byref(tc) if tc is not None else None, _ptr(ws), ws.numel(),
                                 _stream(stream)))


# ------------------------------------------------------------------------------- sharding
def shard_workspace_size(w: LayerWeights, rank: int, world: int, max_ctx: int, batch: int = 1) -> int:
    wc = w.c()
    sh = ShardC(rank, world, batch)
    n = lib().larosa_shard_workspace_size(ctypes.byref(wc), ctypes.byref(sh), max_ctx)
    if n == 0:
        raise LarosaError(3, "shard configuration unsupported (see larosa.h)")
    return n


def shard_phase(w: LayerWeights, plan: Sequence[int], rank: int, world: int, phase: int, x: torch.Tensor,
                out: torch.Tensor, ws: torch.Tensor, resid: Optional[torch.Tensor] = None,
                k_cache: Optional[torch.Tensor] = None, v_cache: Optional[torch.Tensor] = None,
                pos: Optional[torch.Tensor] = None, max_ctx: int = 0, stream=None,
                peer: Optional[PeerTarget] = None):
    """One phase of the row-sharded layer (larosa_sparse_layer_shard_phase); ``w`` holds this
    rank's shard with the FULL model dims.  x / resid [batch][full] (or [full] at batch 1),
    out [batch][local]; peer: also push the output to every rank (then shard_wait)."""
    wc = w.c()
    pc = LayerPlanC(*[int(k) for k in plan[:5]], *([0] if len(plan) < 5 else []))
    sh = ShardC(rank, world, x.shape[0] if x.dim() == 2 else 1)
    if peer is not None:
        sh.peer_dst = _ptr(peer.dst)
        sh.peer_flag = _ptr(peer.flag)
        sh.peer_ld = int(peer.ld)
    _check(lib().larosa_sparse_layer_shard_phase(ctypes.byref(wc), ctypes.byref(pc), ctypes.byref(sh), int(phase),
                                                 _ptr(x), _ptr(resid), _ptr(out), _ptr(k_cache), _ptr(v_cache),
                                                 _ptr(pos), int(max_ctx), _ptr(ws), ws.numel(), _stream(stream)))
