"""The selectable kernel variants (tuning switches read once per process, so each runs in its own
subprocess): the batch-16 rule / token-image paths (LAROSA_RULE_KERNEL 0: cluster Top-K +
gemv_tc; 1: rule_image_kernel; 2: cluster Top-K + rule_apply_image (default); 3: register-resident
rule_image) and the attention kernels (LAROSA_ATTN 1: split-KV ticket merge; 2: cluster DSMEM
merge; default: single pass).  Every variant computes the same exact kept sets, so the image paths
must agree with the default within fp32 rounding (their RMS sums run in different fixed orders)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, "%s")
import synth
from paper_2507_01299_b200 import larosa as LZ
from paper_2507_01299_b200 import model as M
dev = "cuda:0"
shape = synth.ModelShape("m", 512, 1024, 8, 2, 64, 2, 256, True, 1e-6, 10000.0)
B, max_ctx = int(sys.argv[1]), int(sys.argv[2])
lw = M.fold_layer(M.synth_original_layer(shape, 1, device=dev), shape,
                  synth.haar_orthogonal(512, 2, device=dev, dtype=torch.float32),
                  synth.haar_orthogonal(512, 3, device=dev, dtype=torch.float32), adapter_in_down=True)
st = LZ.LayerState(synth.residual_activation(B, 512, 5).to(dev),
                   synth.gaussian_bf16((B, 2, max_ctx, 64), 6, 1.0, dev), synth.gaussian_bf16((B, 2, max_ctx, 64), 7, 1.0, dev),
                   torch.full((B,), max_ctx - 3, dtype=torch.int32, device=dev))
LZ.sparse_layer(lw, M.site_plan(shape, 0.4), st)
torch.cuda.synchronize()
np.save(sys.argv[3], st.resid.cpu().numpy())
''' % ROOT


def run(env, B, max_ctx, tmp, tag):
    out = os.path.join(tmp, f"{tag}.npy")
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(B), str(max_ctx), out], env=e, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out).astype(np.float64)


def test_rule_kernel_variants(tmp_path):
    """Every rule / image path computes the same exact kept sets; their RMS scales are summed in
    different (each fixed) orders, so the outputs agree within fp32 rounding.  The default rule
    kernel (one CTA per token) and the cluster kernel (LAROSA_RULE_CTA=0) feed the same image."""
    ref = run({}, 16, 64, tmp_path, "default")
    outs = {m: run({"LAROSA_RULE_KERNEL": m}, 16, 64, tmp_path, f"rk{m}") for m in ("0", "1", "2", "3")}
    outs["cluster"] = run({"LAROSA_RULE_CTA": "0"}, 16, 64, tmp_path, "cluster")
    assert np.array_equal(outs["2"], ref)
    assert np.array_equal(outs["1"], outs["3"])
    for m, o in outs.items():
        for b in range(16):
            assert np.max(np.abs(o[b] - ref[b])) <= 1e-5 * np.linalg.norm(ref[b]), (m, b)


@pytest.mark.parametrize("B,max_ctx", [(1, 64), (3, 200), (16, 256)])
def test_attention_variants(tmp_path, B, max_ctx):
    ref = run({}, B, max_ctx, tmp_path, "default")
    for m in ("1", "2"):
        got = run({"LAROSA_ATTN": m}, B, max_ctx, tmp_path, f"attn{m}")
        for b in range(B):
            assert np.max(np.abs(got[b] - ref[b])) <= 1e-4 * np.linalg.norm(ref[b]), (m, b)
