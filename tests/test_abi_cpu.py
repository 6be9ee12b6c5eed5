"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/larosa.h
declares, and its host logic (k rule, alpha constraints, argument validation) behaves as
the header states.  No kernel is launched here."""
import ctypes
import json
import os
import re

import pytest

import oracle as O
from paper_2507_01299_b200 import larosa as LZ

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "larosa.h")


def _declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(larosa_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = LZ.lib()
    names = _declared_functions()
    assert len(names) >= 14, names
    for n in names:
        assert hasattr(L, n), f"missing export {n}"
    assert L.larosa_abi_version() == 7


def test_status_strings():
    L = LZ.lib()
    for s in range(7):
        assert L.larosa_status_string(s).decode().startswith("LAROSA_")


def test_compute_k_matches_worked_examples_and_oracle():
    we = json.load(open(os.path.join(ROOT, "tests", "golden", "worked_examples.json")))
    for ex in we["compute_k"]:
        assert LZ.compute_k(ex["alpha"], ex["p"], ex["d"]) == ex["k"], ex["cite"]
    for a in (0.7, 0.8, 0.85, 1.0, 1.15, 1.6):
        for p in (0.0, 0.1, 0.25, 0.4, 0.5, 0.6, 0.75):
            for d in (64, 3584, 4096, 11008, 14336, 18944, 29568):
                assert LZ.compute_k(a, p, d) == O.compute_k(a, p, d)


def test_compute_k_rejects_bad_args():
    with pytest.raises(LZ.LarosaError) as e:
        LZ.compute_k(1.0, 1.5, 10)
    assert e.value.status == 1
    with pytest.raises(LZ.LarosaError):
        LZ.compute_k(1.0, 0.5, 0)
    with pytest.raises(LZ.LarosaError):
        LZ.compute_k(-1.0, 0.5, 10)


def test_solve_alpha_matches_paper_table():
    rows = json.load(open(os.path.join(ROOT, "tests", "golden", "alpha_table.json")))["rows"]
    for r in rows:
        a2, a4 = LZ.solve_alpha(r["a1"], r["a3"], r["M_true"])
        assert a2 == pytest.approx(r["a2"], abs=1e-12)
        assert abs(a4 - r["a4"]) <= 0.01
    with pytest.raises(LZ.LarosaError):
        LZ.solve_alpha(1.5, 0.8, 3.5)        # alpha2 = -0.5 infeasible


FAKE = ctypes.c_void_p(1 << 20)   # never dereferenced: validation fails first


def _status(fn, *args):
    return getattr(LZ.lib(), fn)(*args)


def test_sparse_gemv_validation():
    L = LZ.lib()
    ws = ctypes.c_void_p(1 << 21)
    # NULL W
    assert _status("larosa_sparse_gemv", None, 64, 128, 128, FAKE, FAKE, 1, 8, None, FAKE, ws, 1 << 30, None) == 1
    # k > d_in
    assert _status("larosa_sparse_gemv", FAKE, 64, 128, 128, FAKE, FAKE, 1, 65, None, FAKE, ws, 1 << 30, None) == 1
    # batch > 16
    assert _status("larosa_sparse_gemv", FAKE, 64, 128, 128, FAKE, FAKE, 17, 8, None, FAKE, ws, 1 << 30, None) == 3
    # d_out not a multiple of 8
    assert _status("larosa_sparse_gemv", FAKE, 64, 100, 100, FAKE, FAKE, 1, 8, None, FAKE, ws, 1 << 30, None) == 3
    # ld < d_out
    assert _status("larosa_sparse_gemv", FAKE, 64, 128, 64, FAKE, FAKE, 1, 8, None, FAKE, ws, 1 << 30, None) == 2
    # misaligned y
    assert _status("larosa_sparse_gemv", FAKE, 64, 128, 128, FAKE, FAKE, 1, 8, None, ctypes.c_void_p((1 << 20) + 4),
                   ws, 1 << 30, None) == 1
    # workspace too small
    assert _status("larosa_sparse_gemv", FAKE, 64, 128, 128, FAKE, FAKE, 1, 8, None, FAKE, ws, 16, None) == 6
    assert "workspace" in L.larosa_last_error().decode()


def test_rotate_topk_validation():
    ws = ctypes.c_void_p(1 << 21)
    assert _status("larosa_rotate_topk", None, None, 1, 64, 8, ctypes.c_float(-1), None, FAKE, FAKE, None, ws,
                   1 << 30, None) == 1
    assert _status("larosa_rotate_topk", FAKE, None, 1, 64, 65, ctypes.c_float(-1), None, FAKE, FAKE, None, ws,
                   1 << 30, None) == 1
    assert _status("larosa_rotate_topk", FAKE, None, 1, 40000, 8, ctypes.c_float(-1), None, FAKE, FAKE, None, ws,
                   1 << 30, None) == 3
    assert _status("larosa_rotate_topk", FAKE, FAKE, 1, 64, 8, ctypes.c_float(-1), FAKE, FAKE, FAKE, None, ws,
                   1 << 30, None) == 1   # xr_out aliases x with R


def test_fold_validation():
    ws = ctypes.c_void_p(1 << 21)
    assert _status("larosa_fold_rotation", FAKE, None, FAKE, ctypes.c_void_p(1 << 22), 100, 128, 0, ws, 1 << 30,
                   None) == 3
    assert _status("larosa_fold_rotation", FAKE, FAKE, FAKE, ctypes.c_void_p(1 << 22), 128, 128, 1, ws, 1 << 30,
                   None) == 1   # gamma with RIGHT_Q
    assert _status("larosa_fold_rotation", FAKE, None, FAKE, FAKE, 128, 128, 0, ws, 1 << 30, None) == 1  # alias
    # residual adapter: NULL, d % 64, aliasing, workspace too small
    assert _status("larosa_residual_adapter", None, FAKE, ctypes.c_void_p(1 << 22), 128, ws, 1 << 30, None) == 1
    assert _status("larosa_residual_adapter", FAKE, FAKE, ctypes.c_void_p(1 << 22), 100, ws, 1 << 30, None) == 3
    assert _status("larosa_residual_adapter", FAKE, FAKE, FAKE, 128, ws, 1 << 30, None) == 1
    assert _status("larosa_residual_adapter", FAKE, ctypes.c_void_p(1 << 23), ctypes.c_void_p(1 << 22), 128, ws, 16,
                   None) == 6
    assert _status("larosa_fold_rotation", FAKE, None, FAKE, ctypes.c_void_p(1 << 22), 128, 128, 7, ws, 1 << 30,
                   None) == 1


def test_layer_validation():
    L = LZ.lib()
    w = LZ.LayerWeightsC(FAKE, None, FAKE, FAKE, FAKE, None, 4096, 11008, 32, 32, 96, 1e4, 1e-5)
    p = LZ.LayerPlanC(2048, 2048, 2048, 5504)
    s = LZ.LayerStateC(FAKE, FAKE, FAKE, FAKE, 256, 1)
    ws = ctypes.c_void_p(1 << 21)
    assert L.larosa_sparse_layer(ctypes.byref(w), ctypes.byref(p), ctypes.byref(s), None, ws, 1 << 40, None) == 3
    w.head_dim = 128
    p.k_h4 = 20000
    assert L.larosa_sparse_layer(ctypes.byref(w), ctypes.byref(p), ctypes.byref(s), None, ws, 1 << 40, None) == 1
    p.k_h4 = 5504
    w.n_kv_heads = 5
    assert L.larosa_sparse_layer(ctypes.byref(w), ctypes.byref(p), ctypes.byref(s), None, ws, 1 << 40, None) == 2


def test_no_cpu_fallback():
    import torch
    with pytest.raises((ValueError, RuntimeError)):
        LZ.sparse_gemv(torch.zeros((64, 128), dtype=torch.int16), torch.zeros((1, 8), dtype=torch.int32),
                       torch.zeros((1, 8)))


def test_new_entry_points_validation():
    """Argument checks of the dense2, W4A16, calibration and layer-variant entry points (header
    contracts: NULL -> EINVAL, unsupported shapes -> EUNSUPPORTED, workspace -> EWORKSPACE)."""
    L = LZ.lib()
    ws = ctypes.c_void_p(1 << 21)
    f = ctypes.c_float
    # dense2: NULL x2 / W2, d2 out of range
    assert _status("larosa_topk_sparse_gemv_dense2", FAKE, 64, 8, f(-1), FAKE, 128, 128, None, FAKE, 64, FAKE, 0, ws,
                   1 << 30, None) == 1
    assert _status("larosa_topk_sparse_gemv_dense2", FAKE, 64, 8, f(-1), FAKE, 128, 128, FAKE, FAKE, 0, FAKE, 0, ws,
                   1 << 30, None) == 1
    # W4: d_out not a multiple of 256, k > d_in, NULL scales, workspace too small
    assert _status("larosa_quantize_w4", FAKE, 64, 200, FAKE, FAKE, None) == 3
    assert _status("larosa_quantize_w4", FAKE, 64, 256, None, FAKE, None) == 1
    assert _status("larosa_topk_sparse_gemv_w4", FAKE, 64, 65, f(-1), FAKE, FAKE, 256, FAKE, 0, ws, 1 << 30, None) == 1
    assert _status("larosa_topk_sparse_gemv_w4", FAKE, 64, 8, f(-1), FAKE, None, 256, FAKE, 0, ws, 1 << 30, None) == 1
    assert _status("larosa_topk_sparse_gemv_w4", FAKE, 64, 8, f(-1), FAKE, FAKE, 300, FAKE, 0, ws, 1 << 30, None) == 3
    assert _status("larosa_topk_sparse_gemv_w4", FAKE, 64, 8, f(-1), FAKE, FAKE, 256, FAKE, 0, ws, 16, None) == 6
    # calibration: NULL, bad dims; PCA: NULL, d too large
    assert _status("larosa_calib_covariance", None, 64, 64, f(1), 0, FAKE, ws, 1 << 30, None) == 1
    assert _status("larosa_calib_covariance", FAKE, 0, 64, f(1), 0, FAKE, ws, 1 << 30, None) == 1
    assert _status("larosa_pca_rotation", None, 64, FAKE, FAKE, ws, 1 << 30, None) == 1
    assert _status("larosa_pca_rotation", FAKE, 40000, FAKE, FAKE, ws, 1 << 30, None) == 3
    # layer: adapter_in_down without an adapter
    w = LZ.LayerWeightsC(FAKE, None, FAKE, FAKE, FAKE, None, 4096, 11008, 32, 32, 128, 1e4, 1e-5, 1, None)
    p = LZ.LayerPlanC(2048, 2048, 2048, 5504)
    s = LZ.LayerStateC(FAKE, FAKE, FAKE, FAKE, 256, 1)
    assert L.larosa_sparse_layer(ctypes.byref(w), ctypes.byref(p), ctypes.byref(s), None, ws, 1 << 40, None) == 1
    # host buffers need batch 1
    w.adapter_in_down = 0
    s3 = LZ.LayerStateC(FAKE, FAKE, FAKE, FAKE, 256, 2, 0, FAKE, None)
    assert L.larosa_sparse_layer(ctypes.byref(w), ctypes.byref(p), ctypes.byref(s3), None, ws, 1 << 40, None) == 1
    # W4 sites (ABI 6): codes without scales, batch > 1, D_out % 256 (gate|up of inter 11008 + 64), and a NULL bf16 weight without W4 codes
    s1 = LZ.LayerStateC(FAKE, FAKE, FAKE, FAKE, 256, 1)
    s2 = LZ.LayerStateC(FAKE, FAKE, FAKE, FAKE, 256, 2)
    w4 = LZ.LayerWeightsC(FAKE, None, FAKE, FAKE, FAKE, FAKE, 4096, 11008, 32, 32, 128, 1e4, 1e-5, 0, None)
    w4.w4_codes[0] = FAKE
    assert L.larosa_sparse_layer(ctypes.byref(w4), ctypes.byref(p), ctypes.byref(s1), None, ws, 1 << 40, None) == 1
    w4.w4_scales[0] = FAKE
    assert L.larosa_sparse_layer(ctypes.byref(w4), ctypes.byref(p), ctypes.byref(s2), None, ws, 1 << 40, None) == 3
    w4.w4_codes[3] = w4.w4_scales[3] = FAKE
    w4.inter = 11008 + 64
    w4.w4_codes[2] = w4.w4_scales[2] = FAKE
    assert L.larosa_sparse_layer(ctypes.byref(w4), ctypes.byref(p), ctypes.byref(s1), None, ws, 1 << 40, None) == 3
    w4.inter = 11008
    w4.w4_codes[2] = w4.w4_scales[2] = None
    w4.w_gu = None
    assert L.larosa_sparse_layer(ctypes.byref(w4), ctypes.byref(p), ctypes.byref(s1), None, ws, 1 << 40, None) == 1
    sh1 = LZ.ShardC(0, 1, 1)
    w4.w_gu = FAKE
    assert L.larosa_sparse_layer_shard_phase(ctypes.byref(w4), ctypes.byref(p), ctypes.byref(sh1), 1, FAKE, FAKE,
                                             FAKE, None, None, None, 0, ws, 1 << 40, None) == 3
    # shard phase: the block-wise rotation is not supported there
    w2 = LZ.LayerWeightsC(FAKE, None, FAKE, FAKE, FAKE, FAKE, 4096, 11008, 32, 32, 128, 1e4, 1e-5, 0, FAKE)
    sh = LZ.ShardC(0, 1, 1)
    assert L.larosa_sparse_layer_shard_phase(ctypes.byref(w2), ctypes.byref(p), ctypes.byref(sh), 1, FAKE, FAKE, FAKE,
                                             None, None, None, 0, ws, 1 << 40, None) in (1, 3)
    # shard batch: 0 is invalid, > 16 unsupported (ABI 5)
    w2.adapter_mid = None
    for b, st in ((0, 1), (17, 3)):
        shb = LZ.ShardC(0, 1, b)
        assert L.larosa_sparse_layer_shard_phase(ctypes.byref(w2), ctypes.byref(p), ctypes.byref(shb), 1, FAKE, FAKE,
                                                 FAKE, None, None, None, 0, ws, 1 << 40, None) == st
        assert L.larosa_shard_workspace_size(ctypes.byref(w2), ctypes.byref(shb), 256) == 0
    # P2P push (ABI 7): peer_dst without peer_flag, NULL pointers, bad sizes
    shp = LZ.ShardC(0, 1, 1)
    shp.peer_dst = FAKE
    w2.adapter_mid = None
    assert L.larosa_sparse_layer_shard_phase(ctypes.byref(w2), ctypes.byref(p), ctypes.byref(shp), 1, FAKE, FAKE,
                                             FAKE, None, None, None, 0, ws, 1 << 40, None) == 1
    assert L.larosa_shard_wait(None, FAKE, 1, None) == 1
    assert L.larosa_shard_wait(FAKE, None, 1, None) == 1
    assert L.larosa_peer_push(None, 1, 64, 64, FAKE, FAKE, 1, 64, None) == 1
    assert L.larosa_peer_push(FAKE, 1, 64, 32, FAKE, FAKE, 1, 64, None) == 1     # src_ld < d_local
    assert L.larosa_peer_push(FAKE, 1, 64, 64, FAKE, FAKE, 0, 64, None) == 1     # world 0
    # gather permute / argmax argument checks
    assert L.larosa_shard_gather_permute(None, 2, 1, 64, FAKE, None) == 1
    assert L.larosa_shard_gather_permute(FAKE, 0, 1, 64, ctypes.c_void_p(1 << 22), None) == 1
    assert L.larosa_shard_gather_permute(FAKE, 2, 1, 64, FAKE, None) == 1          # aliasing
    assert L.larosa_argmax(FAKE, 1, 100, 50, FAKE, None) == 1                      # ld < n
    assert L.larosa_argmax(None, 1, 100, 100, FAKE, None) == 1
