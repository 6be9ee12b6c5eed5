"""Supplementary measurements for bench.py: the LLaMA2-7B block of BASELINE
configs[1] (the round-1 headline), the configs[3] Mistral/Qwen sweeps, the isolated SELECT GEMV
per site, the tcgen05 fold / calibration / prefill / W4A16 / rotation-variant legs, and the
row-sharded LLaMA3-70B workload of configs[4].  Imported by bench.py; every number here runs
through the C ABI (liblarosa.so) except the labelled cuBLAS baselines and the oracle leg."""
from __future__ import annotations

import json
import os
import time

import numpy as np
import torch

import synth
from bench import ClockSampler, dist_env, measured_peaks

CTX = 256
N_COPIES = 8
CONFIG_NAME_C2 = "LLaMA2-7B decoder block (4096 hidden, 11008 MLP) batch 1"


# ------------------------------------------------------------------------------------ oracle leg
def build_stack(shape, device, n_copies, seed=0, merged=True, variant="QL"):
    """variant: QL (one rotation per layer, the paper's method), QB (block-wise: attention and MLP
    blocks in their own bases, A_mid beside O), QM (one rotation for the whole model: no adapter)."""
    from paper_2507_01299_b200 import model as M
    qs = [synth.haar_orthogonal(shape.d, seed=100 + i, device=device, dtype=torch.float32) for i in range(n_copies + 1)]
    layers = []
    for i in range(n_copies):
        orig = M.synth_original_layer(shape, seed + i + 1, device=device)
        if variant == "QM":
            layers.append(M.fold_layer(orig, shape, qs[0], None))
        elif variant == "QB":
            qm = synth.haar_orthogonal(shape.d, seed=300 + i, device=device, dtype=torch.float32)
            layers.append(M.fold_layer(orig, shape, qs[i], qs[i + 1], adapter_in_down=merged, q_mlp=qm))
        else:
            layers.append(M.fold_layer(orig, shape, qs[i], qs[i + 1], adapter_in_down=merged))
        del orig
    torch.cuda.synchronize()
    return layers


def time_gemv_sites(layers, plan, shape, device, reps=48):
    """The dominant kernel in isolation: the batch-1 SELECT GEMV (gemv_kernel<1, SELECT>, the
    exact kernel of the layer step: fused Top-K prologue + kept-row stream + epilogue) per
    site, on selection data prepared once per input (larosa_topk_sparse_gemv prepared=1),
    back-to-back launches (PDL) in a CUDA graph, cycling the layer copies (weights >> L2) and
    8 inputs; CUDA events on the launching stream.  The adapter site runs at k = D; with the
    adapter folded beside the down projection it is the dense companion of the down launch
    (larosa_topk_sparse_gemv_dense2), as in the layer."""
    from paper_2507_01299_b200 import larosa as LZ
    k1, k2, k3, k4 = plan
    nq = shape.hq * shape.hd
    sites = [("qkv", "w_qkv", shape.d, shape.qkv_out, k1, shape.rms_eps), ("o", "w_o", nq, shape.d, k2, -1.0),
             ("gate_up", "w_gu", shape.d, 2 * shape.inter, k3, shape.rms_eps),
             ("down", "w_down", shape.inter, shape.d, k4, -1.0), ("adapter", "adapter", shape.d, shape.d, shape.d, -1.0)]
    merged = layers[0].adapter_in_down
    if merged:
        sites[3] = ("down+adapter", "w_down", shape.inter, shape.d, k4, -1.0)
        sites = sites[:4]
    res = {}
    stream = torch.cuda.current_stream()
    n_in = 8
    for name, attr, din, dout, k, eps in sites:
        xs = [synth.residual_activation(1, din, seed=500 + r)[0].to(device) for r in range(n_in)]
        wss = [LZ.topk_sparse_gemv_workspace(din, dout, device) for _ in range(n_in)]
        y = torch.empty((dout,), dtype=torch.float32, device=device)
        dense2 = name == "down+adapter"
        x2s = [synth.residual_activation(1, shape.d, seed=600 + r)[0].to(device) for r in range(n_in)] if dense2 else None

        def call(i, lw, prepared):
            if dense2:
                LZ.topk_sparse_gemv_dense2(xs[i], k, lw.w_down, x2s[i], lw.adapter, out=y, ws=wss[i], prepared=prepared)
            else:
                LZ.topk_sparse_gemv(xs[i], k, getattr(lw, attr), rms_eps=eps, out=y, ws=wss[i], prepared=prepared)

        for i in range(n_in):   # prepare each input's selection data once
            call(i, layers[0], False)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(reps):
                call(i % n_in, layers[i % len(layers)], True)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (5 * reps)
        alg = k * dout * 2 + din * 2 + dout * 4      # kept rows + 16-bit keys + y
        if dense2:
            alg += shape.d * dout * 2 + shape.d * 4    # + every adapter row and its value
        res[name] = {"us": us, "bytes": alg, "gbs": alg / us / 1e3, "k": k, "d_in": din, "d_out": dout}
    return res


def list_gemv_sweep_extra(device, peaks, shape_name="llama3-8b", ps=(0.25, 0.4, 0.5, 0.6), n_copies=8, reps=64):
    """north_star's "sparse-GEMV HBM GB/s (% of peak) vs sparsity": larosa_sparse_gemv (the LIST
    entry: the kept-index list and values given, as larosa_rotate_topk emits them; batch 1) on each
    projection of the layer, back-to-back launches in a CUDA graph cycling n_copies layer copies
    (weights >> L2); GB/s on the selected-column bytes k d_out 2 (+ the index/value list and y)."""
    from paper_2507_01299_b200 import larosa as LZ
    from paper_2507_01299_b200 import model as M
    shape = synth.MODELS[shape_name]
    layers = build_stack(shape, device, n_copies, seed=40)
    nq = shape.hq * shape.hd
    sites = [("qkv", "w_qkv", shape.d, shape.qkv_out), ("o", "w_o", nq, shape.d),
             ("gate_up", "w_gu", shape.d, 2 * shape.inter), ("down", "w_down", shape.inter, shape.d)]
    g0 = torch.Generator().manual_seed(77)
    out = {"workload": f"{shape.name} projections, batch 1, larosa_sparse_gemv (LIST)", "peak_gbs": peaks["hbm_gbs"]}
    stream = torch.cuda.current_stream()
    for p in ps:
        plan = M.site_plan(shape, p)
        row = {}
        tot_b, tot_us = 0, 0.0
        for (name, attr, din, dout), k in zip(sites, plan):
            n_in = 8
            idx = [torch.sort(torch.randperm(din, generator=g0)[:k])[0].to(torch.int32).to(device) for _ in range(n_in)]
            vals = [torch.randn((k,), generator=g0).to(device) for _ in range(n_in)]
            y = torch.empty((1, dout), dtype=torch.float32, device=device)
            ws = torch.zeros(LZ.lib().larosa_sparse_gemv_workspace_size(1, din, k, dout), dtype=torch.uint8,
                             device=device)
            LZ.sparse_gemv(getattr(layers[0], attr), idx[0], vals[0], out=y, ws=ws)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(reps):
                    LZ.sparse_gemv(getattr(layers[i % n_copies], attr), idx[i % n_in], vals[i % n_in], out=y, ws=ws)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(5):
                g.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (5 * reps)
            sel = k * dout * 2
            alg = sel + k * 8 + dout * 4
            row[name] = {"k": k, "us": round(us, 3), "selected_bytes": sel, "gbs": round(alg / us / 1e3, 1),
                         "frac": round(alg / us / 1e3 / peaks["hbm_gbs"], 3)}
            tot_b += alg
            tot_us += us
            del g
        row["all_sites"] = {"gbs": round(tot_b / tot_us / 1e3, 1), "frac": round(tot_b / tot_us / 1e3 / peaks["hbm_gbs"], 3)}
        out[str(p)] = row
    del layers
    torch.cuda.empty_cache()
    return out


def model_sweep_extra(device, models=("mistral-7b", "qwen2.5-7b"), ps=(0.0, 0.25, 0.4, 0.5, 0.6), steps=400,
                      copies=4, merged=True):
    """BASELINE configs[3]: per-layer sparsity sweep of the Mistral-7B and Qwen2.5-7B blocks (batch 1,
    ctx 256, uniform alpha, plus the paper's alpha at p = 0.5) against the dense bf16 GEMV time
    (cuBLAS on the same folded weights) and the HBM byte roofline of each plan."""
    from paper_2507_01299_b200 import larosa as LZ
    from paper_2507_01299_b200 import model as M
    peaks, _ = measured_peaks()
    out = {}
    for name in models:
        shape = synth.MODELS[name]
        layers = build_stack(shape, device, copies, seed=500, merged=merged)
        kv = [(synth.gaussian_bf16((1, shape.hkv, CTX, shape.hd), 900 + i, 1.0, device),
               synth.gaussian_bf16((1, shape.hkv, CTX, shape.hd), 950 + i, 1.0, device)) for i in range(copies)]
        pos = torch.full((1,), CTX - 1, dtype=torch.int32, device=device)
        ws_buf = torch.zeros(LZ.layer_workspace_size(layers[0], 1, CTX), dtype=torch.uint8, device=device)
        res = {}
        plans = [(str(p), M.site_plan(shape, p)) for p in ps] + [("0.5_paper_alpha", M.site_plan(shape, 0.5, "paper"))]
        nq = shape.hq * shape.hd
        for key, plan in plans:
            resid = synth.residual_activation(1, shape.d, seed=77).to(device)
            graphs = capture_graphs(layers, kv, resid, pos, plan, ws_buf)
            run_steps(graphs, 50, 0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run_steps(graphs, steps, 0)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / steps
            k1, k2, k3, k4 = plan
            wbytes = 2 * (k1 * shape.qkv_out + k2 * shape.d + k3 * 2 * shape.inter + k4 * shape.d + shape.d * shape.d)
            kvb = 2 * 2 * shape.hkv * shape.hd * CTX
            res[key] = {"block_us": us, "tok_s": 1e6 / us, "plan": list(plan), "bytes": wbytes + kvb,
                        "roofline_us": (wbytes + kvb) / peaks["hbm_gbs"] / 1e3,
                        "frac_of_roofline": (wbytes + kvb) / peaks["hbm_gbs"] / 1e3 / us}
            del graphs
        dense_us, _ = cublas_dense_us(layers, shape, device)
        res["cublas_dense_4gemv_us"] = dense_us
        res["speedup_vs_dense_at_0.5"] = dense_us / res["0.5"]["block_us"]
        out[name] = res
        del layers, kv, ws_buf
        torch.cuda.empty_cache()
    return out


def calibration_extra(device, d=4096, n_seq=16, n_tok=2048):
    """SURVEY §8(f) N1 at the paper's calibration size (16 sequences x 2048 tokens) for
    a d = 4096 layer: covariance on tcgen05 (TFLOP/s of 2 n d^2) and the fp64 PCA rotation."""
    from paper_2507_01299_b200 import larosa as LZ
    X = synth.gaussian_bf16((n_seq * n_tok, d), 3, 1.0, device)
    C = torch.zeros((d, d), dtype=torch.float32, device=device)
    LZ.calib_covariance(X, scale=1.0 / n_seq, out=C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        LZ.calib_covariance(X, scale=1.0 / n_seq, out=C)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    t0 = time.perf_counter()
    LZ.pca_rotation(C)
    pca_ms = (time.perf_counter() - t0) * 1e3
    return {"d": d, "tokens": n_seq * n_tok, "covariance_ms": ms, "covariance_tflops": 2.0 * n_seq * n_tok * d * d / ms / 1e9,
            "pca_rotation_ms": pca_ms}


def launch_decomposition(layers, kv, pos, ws_buf, plan, shape, device, reps=20):
    """Where each SELECT launch's time goes inside the block step (per-CTA %globaltimer stamps,
    larosa_debug_set_timeline; a separate run after the timed region): per site, the medians
    over CTAs of the prologue (previous kernel's last exit -> row list ready: dependency release,
    selection rule, mask and list), the stream (-> main loop done) and the tail (-> the last CTA's
    exit: split-K reduction, slice ticket, epilogue), and the stream phase's bandwidth on the
    site's kept-row bytes: over the median CTA's stream window, and over the whole span from the
    first CTA's prologue end to the last CTA's loop end (for down + adapter the companions start
    before the SELECT CTAs).  Supplementary to `roofline` (whole launches)."""
    import ctypes
    from paper_2507_01299_b200 import larosa as LZ
    L = LZ.lib()
    L.larosa_debug_set_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.larosa_debug_set_timeline.restype = None
    n = len(layers)
    tl = torch.zeros((n, 6, 1024, 16), dtype=torch.int64, device=device)
    resid = synth.residual_activation(1, shape.d, seed=7).to(device)
    for i in range(n):
        LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos, chained=i > 0), ws=ws_buf)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(n):
            L.larosa_debug_set_timeline(ctypes.c_void_p(tl[i].data_ptr()), 6)
            LZ.sparse_layer(layers[i], plan, LZ.LayerState(resid, *kv[i], pos, chained=True), ws=ws_buf)
        L.larosa_debug_set_timeline(None, 0)
    k1, k2, k3, k4 = plan
    nbytes = {"qkv": k1 * shape.qkv_out * 2, "o": k2 * shape.d * 2, "gate_up": k3 * 2 * shape.inter * 2,
              "down+adapter": (k4 + shape.d) * shape.d * 2}
    slots = {"qkv": (0, 5), "o": (2, 1), "gate_up": (3, 2), "down+adapter": (4, 3)}   # (slot, previous slot)
    res = {k: {"prologue_us": [], "stream_us": [], "tail_us": [], "span_us": []} for k in nbytes}
    for r in range(reps + 2):
        tl.zero_()
        g.replay()
        torch.cuda.synchronize()
        if r < 2:
            continue
        a = tl.cpu().numpy().astype(np.float64)
        for li in range(1, n):
            for name, (sl, prev) in slots.items():
                pv = a[li - 1][4] if sl == 0 else a[li][prev]
                t0 = pv[pv[:, 0] > 0][:, 4].max()
                cur = a[li][sl]
                cur = cur[cur[:, 0] > 0]
                pro = np.median(cur[:, 2]) - t0
                loop = np.median(cur[:, 3]) - t0
                res[name]["prologue_us"].append(pro / 1e3)
                res[name]["stream_us"].append((loop - pro) / 1e3)
                res[name]["tail_us"].append((cur[:, 4].max() - t0 - loop) / 1e3)
                res[name]["span_us"].append((cur[:, 3].max() - cur[:, 2].min()) / 1e3)
    out = {}
    for name, v in res.items():
        pro, stm, tail, span = (float(np.mean(v[k])) for k in ("prologue_us", "stream_us", "tail_us", "span_us"))
        out[name] = {"prologue_us": pro, "stream_us": stm, "tail_us": tail,
                     "stream_phase_gbs_median_cta": nbytes[name] / stm / 1e3 if stm > 0 else None,
                     "stream_phase_gbs_span": nbytes[name] / span / 1e3 if span > 0 else None}
    return out


def prefill_extra(layers, shape, device, p=0.5, n_tok=512, reps=20):
    """N2: a 512-token prompt through the LLaMA2-7B gate|up projection (4096 x 22016) with every
    token's own exact Top-K (larosa_prefill_sparse_gemm: our selection kernel + our tcgen05 masked
    GEMM; bf16 activations and the split hi + lo mode) vs cuBLAS's dense bf16 GEMM on unmasked
    activations: ms, tokens/s and TFLOP/s (useful 2 n k d_out, and the executed 2 n d_in d_out)."""
    from paper_2507_01299_b200 import larosa as LZ
    from paper_2507_01299_b200 import model as M
    k = M.site_plan(shape, p)[2]
    W = layers[0].w_gu
    d_in, d_out = W.shape
    X = torch.randn((n_tok, d_in), device=device)
    Y = torch.empty((n_tok, d_out), device=device)
    out = {"n_tok": n_tok, "k": k, "d_in": d_in, "d_out": d_out}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for split in (False, True):
        LZ.prefill_sparse_gemm(X, k, W, rms_eps=shape.rms_eps, out=Y, split=split)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            LZ.prefill_sparse_gemm(X, k, W, rms_eps=shape.rms_eps, out=Y, split=split)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out["split" if split else "bf16"] = {"ms": ms, "tok_s": n_tok / ms * 1e3,
                                             "useful_tflops": 2.0 * n_tok * k * d_out / ms / 1e9,
                                             "executed_tflops": 2.0 * n_tok * d_in * d_out * (2 if split else 1) / ms / 1e9}
    Xb, Wb = X.to(torch.bfloat16), W.view(torch.bfloat16)
    torch.matmul(Xb, Wb)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        torch.matmul(Xb, Wb)
    e1.record()
    torch.cuda.synchronize()
    out["cublas_dense_bf16_ms"] = e0.elapsed_time(e1) / reps
    out["speedup_vs_cublas_dense"] = out["cublas_dense_bf16_ms"] / out["bf16"]["ms"]
    return out


def w4_sites_extra(layers, plan, shape, device, reps=48):
    """N3: the batch-1 fused Top-K + sparse GEMV per LLaMA2-7B site on W4A16 weights (quantised
    from the same folded bf16 weights, 8 copies cycled), timed like the bf16 roofline leg:
    us, algorithmic GB/s (kept rows' int4 bytes + scales) and the speed-up over bf16 at the site."""
    from paper_2507_01299_b200 import larosa as LZ
    k1, k2, k3, k4 = plan
    nq = shape.hq * shape.hd
    sites = [("qkv", "w_qkv", shape.d, k1, shape.rms_eps), ("o", "w_o", nq, k2, -1.0),
             ("gate_up", "w_gu", shape.d, k3, shape.rms_eps), ("down", "w_down", shape.inter, k4, -1.0)]
    out = {}
    n_in = 8
    for name, attr, din, k, eps in sites:
        qw = [LZ.quantize_w4(getattr(l, attr)) for l in layers]
        dout = qw[0][0].shape[1] * 2
        xs = [synth.residual_activation(1, din, seed=500 + r)[0].to(device) for r in range(n_in)]
        wss = [LZ.topk_sparse_gemv_workspace(din, dout, device) for _ in range(n_in)]
        y = torch.empty((dout,), dtype=torch.float32, device=device)
        for i in range(n_in):
            LZ.topk_sparse_gemv_w4(xs[i], k, *qw[0], rms_eps=eps, out=y, ws=wss[i])
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(reps):
                LZ.topk_sparse_gemv_w4(xs[i % n_in], k, *qw[i % len(qw)], rms_eps=eps, out=y, ws=wss[i % n_in],
                                       prepared=True)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (5 * reps)
        alg = k * (dout // 2 + dout // 128 * 2) + din * 4 + dout * 4
        out[name] = {"us": us, "bytes": alg, "gbs": alg / us / 1e3, "k": k}
        del qw
    return out


def rotation_variants_extra(device, shape, steps=1000, copies=4, p=0.5):
    """Table 6's rotation variants on the LLaMA2-7B block (batch 1, ctx 256, p = 0.5): Q_L (one
    rotation per layer), Q_B (attention / MLP blocks rotated separately: one more D x D adapter,
    riding in the O launch) and Q_M (one rotation for the model: no adapter)."""
    from paper_2507_01299_b200 import larosa as LZ
    from paper_2507_01299_b200 import model as M
    plan = M.site_plan(shape, p)
    out = {}
    for v in ("QL", "QB", "QM"):
        layers = build_stack(shape, device, copies, seed=700, merged=True, variant=v)
        kv = [(synth.gaussian_bf16((1, shape.hkv, CTX, shape.hd), 900 + i, 1.0, device),
               synth.gaussian_bf16((1, shape.hkv, CTX, shape.hd), 950 + i, 1.0, device)) for i in range(copies)]
        pos = torch.full((1,), CTX - 1, dtype=torch.int32, device=device)
        ws_buf = torch.zeros(LZ.layer_workspace_size(layers[0], 1, CTX), dtype=torch.uint8, device=device)
        resid = synth.residual_activation(1, shape.d, seed=77).to(device)
        graphs = capture_graphs(layers, kv, resid, pos, plan, ws_buf)
        run_steps(graphs, 50, 0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run_steps(graphs, steps, 0)
        e1.record()
        torch.cuda.synchronize()
        out[v] = {"block_us": e0.elapsed_time(e1) * 1e3 / steps}
        del layers, kv, graphs, ws_buf
        torch.cuda.empty_cache()
    return out


def latency_consistency_extra(layers, kv, pos, ws_buf, shape, device, steps=600):
    """SURVEY §8(f) N4 / P:369-370: with exact per-token Top-K every token moves the
    same bytes, so per-token latency should be as steady as the dense step's.  Per-step device
    times (CUDA events around each chained step, fresh Top-K sets every step) at p = 0.5 and
    p = 0: percentiles and the coefficient of variation."""
    from paper_2507_01299_b200 import model as M
    out = {}
    for p in (0.5, 0.0):
        plan = M.site_plan(shape, p)
        resid = synth.residual_activation(1, shape.d, seed=91).to(device)
        graphs = capture_graphs(layers, kv, resid, pos, plan, ws_buf)
        run_steps(graphs, 50, 0)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        torch.cuda.synchronize()
        evs[0].record()
        for i in range(steps):
            graphs[i % len(graphs)].replay()
            evs[i + 1].record()
        torch.cuda.synchronize()
        t = np.array([evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(steps)])
        out[str(p)] = {"p10_us": float(np.percentile(t, 10)), "p50_us": float(np.percentile(t, 50)),
                       "p90_us": float(np.percentile(t, 90)), "p99_us": float(np.percentile(t, 99)),
                       "cv": float(np.std(t) / np.mean(t))}
    return out


def fold_extra(device):
    """larosa_fold_rotation on LLaMA2-7B layer shapes: tcgen05 TFLOP/s (2 M N K of the fold)."""
    from paper_2507_01299_b200 import larosa as LZ
    d = 4096
    q = synth.haar_orthogonal(d, 1, device=device, dtype=torch.float32)
    g = torch.ones(d, device=device)
    res = {}
    for name, rows, cols, side in (("w_qkv_left", 4096, 12288, 0), ("w_down_right", 11008, 4096, 1)):
        W = synth.gaussian_bf16((rows, cols), 2, 0.02, device)
        out = torch.empty_like(W)
        LZ.fold_rotation(q, W, side, gamma=g if side == 0 else None, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            LZ.fold_rotation(q, W, side, gamma=g if side == 0 else None, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        res[name] = {"ms": ms, "tflops": 2.0 * rows * cols * d / ms / 1e9}
    return res


def cublas_dense_us(layers, shape, device, reps=40):
    """Dense bf16 GEMV baseline (cuBLAS via torch.matmul) on the same folded weights."""
    nq = shape.hq * shape.hd
    mats = [("w_qkv", shape.d), ("w_o", nq), ("w_gu", shape.d), ("w_down", shape.inter)]
    tot = 0.0
    per = {}
    for attr, din in mats:
        x = torch.randn((1, din), device=device, dtype=torch.bfloat16)
        ws = [getattr(l, attr).view(torch.bfloat16) for l in layers]
        for i in range(3):
            torch.matmul(x, ws[i % len(ws)])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(reps):
            torch.matmul(x, ws[i % len(ws)])
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        per[attr] = us
        tot += us
    return tot, per


def capture_graphs(layers, stack_kv, resid, pos, plan, ws_buf, chained=True):
    """One CUDA graph per layer copy.  chained=True: the step's input residual is the
    previous step's output (its h1 histogram / RMS partials were produced by the previous
    layer's epilogue); chained=False adds the standalone h1 preparation kernel."""
    from paper_2507_01299_b200 import larosa as LZ
    graphs = []
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i, (w, (kc, vc)) in enumerate(zip(layers, stack_kv)):     # warm-up outside capture
            LZ.sparse_layer(w, plan, LZ.LayerState(resid, kc, vc, pos, chained=chained and i > 0), ws=ws_buf)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    for w, (kc, vc) in zip(layers, stack_kv):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            LZ.sparse_layer(w, plan, LZ.LayerState(resid, kc, vc, pos, chained=chained), ws=ws_buf)
        graphs.append(g)
    torch.cuda.synchronize()
    return graphs


def run_steps(graphs, k, start):
    for i in range(k):
        graphs[(start + i) % len(graphs)].replay()


def run_sharded(args):
    """BASELINE configs[4]: the LLaMA3-70B decode step (80 folded layers, d 8192, MLP 28672, GQA 64/8,
    128256 vocab; --model qwen2.5-72b for Qwen2.5-72B) row-sharded over the WORLD_SIZE ranks
    (SURVEY §8(e)): every rank holds its columns of every projection and of the LM head, the
    embedding and the residual are replicated; per layer 4 NCCL all-gathers (adapter beside down)
    plus one for the logits, the whole step captured in one CUDA graph.  value = tokens/s of the
    job (batch x steps / max-over-ranks CUDA-event time); strong scaling (the same model split)."""
    import torch.distributed as dist
    from paper_2507_01299_b200 import model as M
    ws_n, rank, local = dist_env()
    torch.cuda.set_device(local)
    device = f"cuda:{local}"
    if ws_n > 1:
        dist.init_process_group("nccl", device_id=torch.device(device))
    shape = synth.MODELS[getattr(args, "model", None) or "llama3-70b"]
    n_layers = getattr(args, "layers", None) or shape.layers
    B, max_ctx = args.batch, 256
    model = M.ShardedDecodeModel(shape, n_layers, rank, ws_n, device, seed=3, adapter_in_down=args.adapter == "down")
    collective = getattr(args, "collective", "nccl")
    if collective == "p2p":   # the phase kernels push into every rank's symmetric buffers
        if ws_n == 1 and not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(device))
        space = M.PeerSpace.symmetric(M.ShardedDecodeRunner.peer_bytes(model, B), device)
        run = M.ShardedDecodeRunner(model, B, max_ctx, device, space=space)
    else:
        run = M.ShardedDecodeRunner(model, B, max_ctx, device)
    for kc, vc in run.kv:
        kc.copy_(synth.gaussian_bf16(kc.shape, 5 + rank, 1.0, device))
        vc.copy_(synth.gaussian_bf16(vc.shape, 6 + rank, 1.0, device))
    run.tokens.copy_((torch.arange(B, dtype=torch.int32) * 7919 + 11) % shape.vocab)
    run.pos.fill_(max_ctx - 1)
    plan = M.site_plan(shape, args.p)

    def allgather(local_t, full_t):
        if ws_n > 1:
            dist.all_gather_into_tensor(full_t, local_t)
        else:
            full_t.copy_(local_t)

    def body():
        run.step(plan, allgather)
        run.tokens.copy_(run.next_tokens)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        body()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    for _ in range(args.warmup):
        g.replay()
    torch.cuda.synchronize()
    if ws_n > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if ws_n > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    n_ph = run.shards[0].n_phases()
    if rank == 0:
        out = {"metric": f"decode tokens/s ({shape.name} {n_layers}-layer decode step, row-sharded)",
               "value": B * args.steps / (ms / 1e3), "unit": "tok/s", "n_gpus": ws_n, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "bf16 weights, fp32 activations/accumulate", "data": "synthetic",
               "config": {"workload": f"{shape.name} decode step ({n_layers} layers, d {shape.d}, MLP {shape.inter}, "
                                      f"GQA {shape.hq}/{shape.hkv}), row-sharded", "batch": B, "sparsity": args.p,
                          "plan_k": list(plan), "ctx": max_ctx,
                          "parallelism": f"tp{ws_n} (row-sharded, NCCL all-gather x{n_ph}/layer + logits)"
                          if collective != "p2p" else
                          f"tp{ws_n} (row-sharded, P2P push from the phase kernels into symmetric memory "
                          f"x{n_ph}/layer + logits, device-side counters)", "collective": collective,
                          "l2": "inputs larger than L2: the step streams the whole sharded model"},
               "gpu_launches": None, "clocks": clk.summary()}
        print(json.dumps(out))
    if dist.is_initialized():
        dist.destroy_process_group()


def block_c2_extra(device, p=0.5, steps=2000, warmup=200, merged=True):
    """BASELINE configs[1]: one LLaMA2-7B decoder block, batch 1, ctx 256 (the round-1 headline):
    block tokens/s over 8 distinct layer copies (3.2 GB >> L2) with each step's input the previous
    output, the same block fed from / to pinned host memory (larosa_layer_state.host_in/out), the
    isolated SELECT GEMV per site (algorithmic GB/s), the in-step launch decomposition, the sparsity
    sweep and the cuBLAS dense GEMVs on the same weights."""
    from paper_2507_01299_b200 import larosa as LZ
    from paper_2507_01299_b200 import model as M
    shape = synth.MODELS["llama2-7b"]
    layers = build_stack(shape, device, N_COPIES, seed=0, merged=merged)
    kv = [(synth.gaussian_bf16((1, shape.hkv, CTX, shape.hd), 900 + i, 1.0, device),
           synth.gaussian_bf16((1, shape.hkv, CTX, shape.hd), 950 + i, 1.0, device)) for i in range(N_COPIES)]
    pos = torch.full((1,), CTX - 1, dtype=torch.int32, device=device)
    ws_buf = torch.zeros(LZ.layer_workspace_size(layers[0], 1, CTX), dtype=torch.uint8, device=device)
    resid0 = synth.residual_activation(1, shape.d, seed=77).to(device)
    peaks, _ = measured_peaks()

    def measure(pp):
        plan = M.site_plan(shape, pp)
        resid = resid0.clone()
        graphs = capture_graphs(layers, kv, resid, pos, plan, ws_buf)
        run_steps(graphs, warmup, 0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run_steps(graphs, steps, warmup)
        e1.record()
        torch.cuda.synchronize()
        return plan, e0.elapsed_time(e1) * 1e3 / steps

    plan, us = measure(p)
    out = {"workload": CONFIG_NAME_C2, "p": p, "plan": list(plan), "block_us": us, "block_tok_s": 1e6 / us}
    # e2e: host input / output inside the layer's first and last kernels
    h_in = torch.empty((1, shape.d), dtype=torch.float32).pin_memory()
    h_in.copy_(resid0.cpu())
    h_out = torch.empty((1, shape.d), dtype=torch.float32).pin_memory()
    resid = resid0.clone()
    io = []
    for w, (kc, vc) in zip(layers, kv):
        LZ.sparse_layer(w, plan, LZ.LayerState(resid, kc, vc, pos, host_in=h_in, host_out=h_out), ws=ws_buf)
    torch.cuda.synchronize()
    for w, (kc, vc) in zip(layers, kv):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            LZ.sparse_layer(w, plan, LZ.LayerState(resid, kc, vc, pos, host_in=h_in, host_out=h_out), ws=ws_buf)
        io.append(g)
    run_steps(io, warmup, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run_steps(io, steps, 0)
    e1.record()
    torch.cuda.synchronize()
    out["e2e_block_tok_s"] = steps / (e0.elapsed_time(e1) / 1e3)
    gem = time_gemv_sites(layers, plan, shape, device)
    bytes_step = sum(v["bytes"] for v in gem.values())
    us_gemv = sum(v["us"] for v in gem.values())
    out["select_gemv"] = {"achieved_gbs": bytes_step / us_gemv / 1e3, "frac": bytes_step / us_gemv / 1e3 / peaks["hbm_gbs"],
                          "algorithmic_bytes": bytes_step, "us": us_gemv, "per_site": gem}
    out["decomposition_in_step"] = launch_decomposition(layers[:4], kv[:4], pos, ws_buf, plan, shape, device) \
        if merged else None
    sweep = {}
    for pp in (0.0, 0.25, 0.4, 0.5, 0.6):
        pl, u = measure(pp)
        sweep[str(pp)] = {"block_us": u, "tok_s": 1e6 / u, "plan": list(pl)}
    dense_us, dense_per = cublas_dense_us(layers, shape, device)
    sweep["cublas_dense_4gemv_us"] = dense_us
    sweep["cublas_dense_per_gemv_us"] = dense_per
    out["sweep"] = sweep
    out["latency_consistency"] = latency_consistency_extra(layers, kv, pos, ws_buf, shape, device)
    w4 = w4_sites_extra(layers, plan, shape, device)
    out["w4a16_sites"] = {k: dict(v, bf16_us=gem[k if k != "down" else ("down+adapter" if merged else "down")]["us"])
                          for k, v in w4.items()}
    out["prefill_n2"] = prefill_extra(layers, shape, device)
    del layers, kv, ws_buf
    torch.cuda.empty_cache()
    return out
