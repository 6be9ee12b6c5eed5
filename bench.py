#!/usr/bin/env python
"""LaRoSA decode hot path benchmark (driver contract).

Workload (BASELINE.json configs[2], the largest single-GPU configuration): the LLaMA3-8B-shaped
full decode step -- 32 folded random-init layers (d 4096, MLP 14336, GQA 32/8 x 128), the
128,256-token LM head and greedy arg-max -- at batch 1 (default; --batch up to 16), sparsity
p = 0.4 with uniform alpha, KV context 256.  A *step* = one decode token for every sequence:
embedding row -> 32 x larosa_sparse_layer (per layer: Top-K(h1) + sparse QKV GEMV (+RoPE, KV
append) -> attention -> Top-K(h2) + sparse O GEMV -> Top-K(h3) + sparse gate|up GEMV (+SiLU*)
-> Top-K(h4) + sparse down GEMV with the residual adapter rows beside it) -> RMS + LM head ->
arg-max, the greedy token fed back as the next step's input, all replayed as one CUDA graph.
The weights (17 GB) are read once per step, so every step streams from HBM (>> 126 MB L2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--p 0.4] [--batch 1] [--impl reference]
                  [--workload decode|block|sharded-70b] [--no-extras] [--no-cpu-baseline]

N > 1 (torchrun): every rank runs its own decode stream of its own model copy (replicas,
weak scaling: an 8B model fits one B200, so the path does not shard), CUDA-event
time, max over ranks.  --workload sharded-70b: one LLaMA3-70B layer row-sharded over the ranks
with NCCL all-gathers (configs[4]); --workload block: the LLaMA2-7B block (configs[1]).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "decode tokens/s (LLaMA3-8B 32-layer decode step)"
UNIT = "tok/s"
MODEL = "llama3-8b"
CONFIG_NAME = "LLaMA3-8B full 32-layer decode step (GQA 32/8, 14336 MLP, 128256 vocab)"
CTX = 256


# ------------------------------------------------------------------------------------ utils
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.15)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def host_info():
    """nproc, CPU model and RAM of the box (the oracle's host is stated)."""
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    info["cpu"] = ln.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemTotal"):
                    info["ram_gb"] = round(int(ln.split()[1]) / 2 ** 20, 1)
                    break
    except OSError:
        pass
    return info


def source_hash():
    """Hash of the library sources and the launch-plan code: profiles/traffic.json is used only
    when it was measured at the same sources (tools/traffic.sh)."""
    h = hashlib.sha256()
    files = sorted(os.path.join(ROOT, "paper_2507_01299_b200", "csrc", f)
                   for f in os.listdir(os.path.join(ROOT, "paper_2507_01299_b200", "csrc")))
    files += [os.path.join(ROOT, "include", "larosa.h")]
    for p in files:
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


# ------------------------------------------------------------------------------------ step bytes
def step_bytes(shape, plan, unions, batch, ctx_lens, n_layers, w4=False):
    """Algorithmic bytes of one decode step (SURVEY §8(d) "algorithmic work per unit"):
    per layer  sum_sites |U_s| D_out,s 2  (|U_s| = k_s at batch 1; the measured union of the
    tokens' kept sets otherwise)  +  D^2 2 (adapter; the last layer has none)  +  the KV rows read
    (B 2 Hkv hd ctx 2); plus the LM head D V 2 and the embedding rows B D 2.  w4: a kept row of a
    site costs D_out / 2 code bytes + D_out / 128 fp16 scales instead of 2 D_out."""
    d, nq = shape.d, shape.hq * shape.hd
    douts = (shape.qkv_out, d, 2 * shape.inter, d)
    kv = sum(2 * shape.hkv * shape.hd * c * 2 for c in ctx_lens)
    row = (lambda n: n // 2 + 2 * (n // 128)) if w4 else (lambda n: 2 * n)
    tot = 0
    for l in range(n_layers):
        u = unions[l] if unions is not None else plan
        tot += sum(int(a) * row(b) for a, b in zip(u, douts)) + kv
        if l + 1 < n_layers:
            tot += d * d * 2
    return tot + d * shape.vocab * 2 + batch * d * 2


def measure_unions(run, plan, batch):
    """|U_s| per layer and site: the union of the batch's kept index sets, from one tapped step."""
    from paper_2507_01299_b200 import larosa as LZ
    taps = [LZ.make_taps(w, plan, batch, run.resid.device) for w in run.m.layers]
    run.step(plan, taps=taps)
    torch.cuda.synchronize()
    out = []
    for t in taps:
        u = []
        for s in (1, 2, 3, 4):
            idx = t[f"idx_h{s}"].cpu().numpy()
            u.append(int(np.unique(idx).size) if idx.size else 0)
        out.append(u)
    return out


def launches_per_step(batch, n_layers, merged=True):
    """Our kernels in one captured decode step: embed; per layer (batch 1) QKV, attention, O,
    gate|up, down (+ adapter rows) SELECT GEMVs -- 5 -- plus the h1 preparation kernel in the
    first layer; at batch > 1 a Top-K rule kernel before each of the 4 site GEMVs and a separate
    dense adapter GEMV (10 per layer, the last layer 9); LM head: RMS, GEMV, arg-max."""
    if batch == 1:
        per = [5 if merged else 6] * n_layers
        per[0] += 1
        per[-1] -= 0 if merged else 1
    else:
        per = [10] * n_layers
        per[-1] = 9
    return 1 + sum(per) + 3


# ------------------------------------------------------------------------------------ oracle leg
def oracle_decode_sample(shape, plan, n_tok, threads=None, seed=0):
    """The fp64 oracle (as it stands: oracle.larosa_block + oracle.lm_head) on the headline
    workload's shapes: n_tok tokens through ONE LLaMA3-8B layer plus one 1/8 slice of the LM head,
    extrapolated to the 32-layer step as 32 t_layer + 8 t_head_slice (a layer's fp64 weights are
    1.8 GB and the model's 64 GB, so the whole model is not materialised).  threads: BLAS threads
    (threadpoolctl), None = the library default.  Returns (tok/s, seconds measured, threads)."""
    import oracle as O
    from threadpoolctl import threadpool_limits, threadpool_info
    d, inter, nq = shape.d, shape.inter, shape.hq * shape.hd
    rng = np.random.default_rng(seed)

    def wbits(shape_, std):
        return O.f64_to_bf16_rne(rng.standard_normal(shape_, dtype=np.float32) * std)

    wf = {"wqkv": O.bf16_to_f64(wbits((d, shape.qkv_out), d ** -0.5)),
          "wo": O.bf16_to_f64(wbits((nq, d), nq ** -0.5)),
          "wg": O.bf16_to_f64(wbits((d, inter), d ** -0.5)),
          "wu": O.bf16_to_f64(wbits((d, inter), d ** -0.5)),
          "wd": O.bf16_to_f64(wbits((inter, d), inter ** -0.5))}
    adapter = O.bf16_to_f64(wbits((d, d), d ** -0.5))
    head_slice = O.bf16_to_f64(wbits((d, shape.vocab // 8), d ** -0.5))
    cfg = dict(hq=shape.hq, hkv=shape.hkv, hd=shape.hd, eps=shape.rms_eps, theta=shape.rope_theta)
    kc = rng.standard_normal((shape.hkv, CTX, shape.hd))
    vc = rng.standard_normal((shape.hkv, CTX, shape.hd))
    r0 = synth.residual_activation(1, d, seed=1).numpy()[0].astype(np.float64)
    with threadpool_limits(limits=threads):
        used = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
        O.larosa_block(r0, wf, cfg, plan, kc, vc, CTX - 1, adapter=adapter, kv_bf16=True, adapter_in_down=True)
        t0 = time.perf_counter()
        r = r0
        for _ in range(n_tok):
            r, _ = O.larosa_block(r, wf, cfg, plan, kc, vc, CTX - 1, adapter=adapter, kv_bf16=True,
                                  adapter_in_down=True)
        t_layer = (time.perf_counter() - t0) / n_tok
        t0 = time.perf_counter()
        O.lm_head(r, head_slice, shape.rms_eps)
        t_head = (time.perf_counter() - t0) * 8
    t_step = shape.layers * t_layer + t_head
    return 1.0 / t_step, n_tok * t_layer + t_head / 8, used


def cpu_baseline(shape, plan, n_tok=2):
    """Oracle tok/s on the box's host cores, 1 thread and all threads (results bit-identical:
    each output is one fixed-order dot product)."""
    nproc = os.cpu_count() or 1
    one, s1, _ = oracle_decode_sample(shape, plan, n_tok, threads=1)
    alln, s2, used = oracle_decode_sample(shape, plan, n_tok, threads=nproc)
    return {"value": alln, "unit": UNIT, "cores": used, "kind": "oracle",
            "sample": f"{n_tok} tokens through one LLaMA3-8B layer + 1/8 of the LM head (fp64 numpy oracle), "
                      f"extrapolated to the 32-layer step (32 t_layer + t_head); same p and plan",
            "extrapolated": True, "one_thread_tok_s": one, "all_threads_tok_s": alln,
            "measured_seconds": s1 + s2, "host": host_info()}


def run_reference(args):
    """--impl reference: the oracle (as it stands) on the same workload and metric; each step = one
    token through one layer + 1/8 head slice, extrapolated to the 32-layer step."""
    ws, rank, _ = dist_env()
    if ws > 1 and rank != 0:
        return
    import oracle as O
    shape = synth.MODELS[MODEL]
    plan = O.site_ks(args.p, (1, 1, 1, 1), shape.d, shape.inter)
    steps = max(1, min(args.steps, 6))                       # bounded CPU sample
    tok_s, secs, threads = oracle_decode_sample(shape, plan, steps)
    out = {"impl": "reference", "metric": METRIC, "value": tok_s, "unit": UNIT, "n_gpus": args.gpus,
           "steps": steps, "warmup": 1, "ms_per_step": 1e3 / tok_s, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": CONFIG_NAME, "sparsity": args.p, "alpha": "uniform", "ctx": CTX, "batch": 1},
           "cpu_baseline": {"value": tok_s, "unit": UNIT, "cores": threads, "kind": "oracle",
                            "sample": f"{steps} tokens through one LLaMA3-8B layer + 1/8 LM head (fp64 numpy "
                                      f"oracle), extrapolated to 32 layers + head", "host": host_info()},
           "e2e": {"value": tok_s, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


# ------------------------------------------------------------------------------------ GPU leg
def capture_step(run, plan, feedback=True):
    """One CUDA graph of a whole decode step; feedback=True appends the greedy token -> next
    input copy (device to device), so replays decode a real token sequence."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run.step(plan)
        if feedback:
            run.tokens.copy_(run.next_tokens)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run.step(plan)
        if feedback:
            run.tokens.copy_(run.next_tokens)
    torch.cuda.synchronize()
    return g


def timed_replays(g, k, ws_n=1, device=None):
    """k replays between two CUDA events on the replay stream (after a barrier + sync), max over ranks."""
    torch.cuda.synchronize()
    if ws_n > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if ws_n > 1:
        t = torch.tensor([ms], device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def reset_run(run, seed):
    for kc, vc in run.kv:
        kc.copy_(synth.gaussian_bf16(kc.shape, seed, 1.0, kc.device))
        vc.copy_(synth.gaussian_bf16(vc.shape, seed + 1, 1.0, vc.device))
    b = run.tokens.shape[0]
    run.tokens.copy_((torch.arange(b, dtype=torch.int32) * 7919 + 11) % run.m.shape.vocab)
    run.pos.fill_(CTX - 1)


def cublas_dense_step_ms(model, batch, device, reps=10):
    """cuBLAS bf16 dense GEMVs of the whole step (4 projections x 32 layers + the LM head, torch.matmul
    on the same weights, one CUDA graph); attention excluded (favours this baseline)."""
    x = {n: torch.randn((batch, n), device=device, dtype=torch.bfloat16) for n in {model.shape.d, model.shape.inter,
                                                                                   model.shape.hq * model.shape.hd}}
    mats = []
    for w in model.layers:
        mats += [(w.w_qkv, w.d), (w.w_o, w.n_q_heads * w.head_dim), (w.w_gu, w.d), (w.w_down, w.inter)]
    mats.append((model.head, model.shape.d))

    def body():
        for W, din in mats:
            torch.matmul(x[din], W.view(torch.bfloat16))

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        body()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    for _ in range(2):
        g.replay()
    return timed_replays(g, reps) / reps


def own_dense_model(model):
    """The same model without the method's additions (no adapter, every site at k = D: the SELECT
    GEMVs take the keep-all rule without a histogram lookup): the library's own dense chain."""
    from paper_2507_01299_b200 import larosa as LZ
    from paper_2507_01299_b200 import model as M
    layers = [LZ.LayerWeights(**{**w.__dict__, "adapter": None, "adapter_in_down": False}) for w in model.layers]
    return M.DecodeModel(shape=model.shape, embed=model.embed, layers=layers, head=model.head)


def w4_decode_extra(shape, device, peaks, ps=(0.0, 0.4, 0.5), steps=20):
    """N3: the same decode step with W4A16 weights at all four sites of every layer (larosa.h ABI 6;
    adapter beside down, bf16 head), batch 1, one CUDA graph per step (tests/test_gpu_w4_layer.py
    is its parity)."""
    from paper_2507_01299_b200 import model as M
    model = M.synth_decode_model(shape, shape.layers, device, seed=1, w4=True, adapter_in_down=True)
    run = M.DecodeRunner(model, 1, CTX, device)
    out = {"weights": "int4 codes + fp16 scales per 128 outputs, all 4 sites; adapter bf16 beside down "
                      "(companion CTAs of the W4 down launch); head bf16"}
    for pp in ps:
        pl = M.site_plan(shape, pp)
        reset_run(run, 5)
        t = decode_line(run, pl, steps)
        nb = step_bytes(shape, pl, None, 1, [CTX], shape.layers, w4=True)
        out[str(pp)] = {"ms_per_step": t, "tok_s": 1e3 / t, "plan": list(pl), "bytes": nb,
                        "frac": nb / (t * 1e-3) / 1e9 / peaks["hbm_gbs"]}
    del run, model
    torch.cuda.empty_cache()
    return out


def decode_line(run, plan, steps, reps_unions=True):
    g = capture_step(run, plan)
    for _ in range(3):
        g.replay()
    ms = timed_replays(g, steps) / steps
    del g
    return ms


def traffic_record(batch, p):
    """DRAM bytes per step measured by ncu (tools/traffic.sh) at the SAME library sources, else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            rec = json.load(f)
    except Exception:
        return None, "no profiles/traffic.json"
    key = f"B{batch}_p{p}"
    if rec.get("source_hash") != source_hash():
        return None, f"profiles/traffic.json measured at sources {rec.get('source_hash')} != {source_hash()}"
    e = rec.get("steps", {}).get(key)
    if not e:
        return None, f"no {key} entry in profiles/traffic.json"
    return e, "ncu dram__bytes_read.sum + dram__bytes_write.sum over every kernel of one step (tools/traffic.sh)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--p", type=float, default=0.4)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--impl", default="larosa", choices=["larosa", "reference"])
    ap.add_argument("--workload", default="decode", choices=["decode", "block", "sharded-70b"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="alias of --no-extras")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--traffic-probe", action="store_true",
                    help="build the model, warm up, then run exactly 2 steps eagerly (for ncu; no JSON)")
    ap.add_argument("--adapter", default="down", choices=["down", "separate"])
    ap.add_argument("--model", default=None, help="sharded-70b: llama3-70b (default) or qwen2.5-72b")
    ap.add_argument("--layers", type=int, default=None, help="sharded-70b: layer count (default: the model's)")
    ap.add_argument("--collective", default="nccl", choices=["nccl", "p2p"],
                    help="sharded-70b: NCCL all-gathers, or the phase kernels' P2P push into symmetric memory")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return
    import bench_extras as BX
    if args.workload == "sharded-70b":
        BX.run_sharded(args)
        return
    ws_n, rank, local = dist_env()
    torch.cuda.set_device(local)
    device = f"cuda:{local}"
    if ws_n > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(device))
    if args.workload == "block":
        out = BX.block_c2_extra(device, p=args.p if args.p != 0.4 else 0.5, steps=args.steps * 20,
                                warmup=args.warmup * 20, merged=args.adapter == "down")
        if rank == 0:
            print(json.dumps(out))
        return
    from paper_2507_01299_b200 import model as M

    shape = synth.MODELS[MODEL]
    merged = args.adapter == "down"
    B = args.batch
    model = M.synth_decode_model(shape, shape.layers, device, seed=1 + rank, adapter_in_down=merged)
    run = M.DecodeRunner(model, B, CTX, device)
    reset_run(run, 5)
    plan = M.site_plan(shape, args.p)

    if args.traffic_probe:   # tools/traffic.sh: ncu keeps only the kernels inside the NVTX range
        g = capture_step(run, plan)
        for _ in range(args.warmup):
            g.replay()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("traffic_step")
        g.replay()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        return

    with ClockSampler(local) as clk:
        g = capture_step(run, plan)
        for _ in range(args.warmup):
            g.replay()
        ms = timed_replays(g, args.steps, ws_n, device)
    clocks = clk.summary()
    ms_per_step = ms / args.steps
    value = ws_n * B * args.steps / (ms / 1e3)
    del g

    # ---- end to end through the public API: every step copies the step's input tokens from pinned
    # host memory and reads the greedy tokens back into pinned host memory, inside the timed region
    h_tok = torch.empty((args.steps + args.warmup, B), dtype=torch.int32).pin_memory()
    h_tok.copy_(torch.randint(0, shape.vocab, h_tok.shape, generator=synth.gen(3), dtype=torch.int32))
    h_out = torch.empty((args.steps + args.warmup, B), dtype=torch.int32).pin_memory()
    ge = capture_step(run, plan, feedback=False)

    def e2e_step(i):
        run.tokens.copy_(h_tok[i], non_blocking=True)
        ge.replay()
        h_out[i].copy_(run.next_tokens, non_blocking=True)

    for i in range(args.warmup):
        e2e_step(i)
    torch.cuda.synchronize()
    if ws_n > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        e2e_step(args.warmup + i)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if ws_n > 1:
        t = torch.tensor([e2e_ms], device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": ws_n * B * args.steps / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": B * 4,
           "d2h_bytes_per_step": B * 4, "api": "model.DecodeRunner.step (CUDA graph) + pinned token copies"}
    del ge

    # ---- roofline of the step: algorithmic bytes / step time --------------------------------------
    peaks, peak_kind = measured_peaks()
    unions = None if B == 1 else measure_unions(run, plan, B)
    reset_run(run, 5)
    nbytes = step_bytes(shape, plan, unions, B, [CTX] * B, shape.layers)
    achieved = nbytes / (ms_per_step * 1e-3) / 1e9
    traffic, traffic_src = traffic_record(B, args.p)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "frac_of_8tbs": achieved / 8000.0,
                "traffic": traffic["dram_bytes_per_step"] if traffic else None, "traffic_source": traffic_src,
                "kernel": "the whole decode step (every launch of the graph; the SELECT GEMVs are ~86% of its "
                          "kernel time, profiles/r02/)",
                "algorithmic_bytes_per_step": nbytes, "unions_per_layer": unions,
                "peak_kind": f"{peak_kind} copy (hbm_gbs)",
                "bound_tok_s": B * peaks["hbm_gbs"] * 1e9 / nbytes}
    if not (args.no_extras or args.no_sweep):
        gem = BX.time_gemv_sites([w for w in model.layers[:8]], plan, shape, device)
        gb = sum(v["bytes"] for v in gem.values())
        gu = sum(v["us"] for v in gem.values())
        roofline["dominant_kernel"] = {
            "kernel": "gemv_kernel<1, SELECT> (fused Top-K prologue + kept-row stream + epilogue), the 4 site "
                      "launches of one LLaMA3-8B layer (down with the adapter rows as companions), each timed "
                      "back to back in a CUDA graph over 8 layer copies",
            "achieved": gb / gu / 1e3, "frac": gb / gu / 1e3 / peaks["hbm_gbs"], "algorithmic_bytes": gb,
            "us": gu, "per_site": gem}

    extras = None
    if not (args.no_extras or args.no_sweep):
        extras = {}
        # sparsity sweep of the whole step, the dense baselines and batch 16
        sweep = {}
        for pp in (0.0, 0.25, 0.4, 0.5, 0.6):
            pl = M.site_plan(shape, pp)
            reset_run(run, 5)
            t = decode_line(run, pl, 20)
            sweep[str(pp)] = {"ms_per_step": t, "tok_s": B * 1e3 / t, "plan": list(pl),
                              "bytes": step_bytes(shape, pl, None, 1, [CTX], shape.layers) if B == 1 else None}
        dm = own_dense_model(model)
        drun = M.DecodeRunner(dm, B, CTX, device)
        reset_run(drun, 5)
        dense_own = decode_line(drun, M.site_plan(shape, 0.0), 20)
        del drun, dm
        dense_cublas = cublas_dense_step_ms(model, B, device)
        dense = min(dense_own, dense_cublas)
        dense_bytes = step_bytes(shape, M.site_plan(shape, 0.0), None, 1, [CTX], shape.layers) - \
            (shape.layers - 1) * shape.d * shape.d * 2
        for k, v in sweep.items():
            v["speedup_vs_dense"] = dense / v["ms_per_step"]
            if v["bytes"]:
                v["ideal_speedup_bytes"] = dense_bytes / v["bytes"]
                v["frac"] = v["bytes"] / (v["ms_per_step"] * 1e-3) / 1e9 / peaks["hbm_gbs"]
        extras["step_sweep"] = sweep
        extras["dense_baseline"] = {"own_dense_chain_ms": dense_own, "cublas_gemvs_ms": dense_cublas,
                                    "dense_ms": dense, "dense_bytes": dense_bytes,
                                    "note": "own: the same step without adapter at k = D (keep-all rule, no "
                                            "histogram lookup); cuBLAS: torch.matmul GEMVs of the 4 projections x "
                                            "32 + head, attention excluded; dense = the faster"}
        if B == 1:
            del run
            torch.cuda.empty_cache()
            b16 = {}
            run16 = M.DecodeRunner(model, 16, CTX, device)
            for pp in (0.4, 0.0):
                pl = M.site_plan(shape, pp)
                reset_run(run16, 5)
                t = decode_line(run16, pl, 10)
                ent = {"ms_per_step": t, "tok_s": 16e3 / t, "plan": list(pl)}
                if pp > 0:
                    un = measure_unions(run16, pl, 16)
                    nb16 = step_bytes(shape, pl, un, 16, [CTX] * 16, shape.layers)
                    ent.update(bytes=nb16, frac=nb16 / (t * 1e-3) / 1e9 / peaks["hbm_gbs"],
                               union_fraction=[round(float(np.mean([u[s] for u in un])) / dn, 4) for s, dn in
                                               enumerate((shape.d, shape.hq * shape.hd, shape.d, shape.inter))])
                b16[str(pp)] = ent
            dm = own_dense_model(model)
            d16 = M.DecodeRunner(dm, 16, CTX, device)
            reset_run(d16, 5)
            b16["dense_own_ms"] = decode_line(d16, M.site_plan(shape, 0.0), 10)
            b16["dense_cublas_ms"] = cublas_dense_step_ms(model, 16, device)
            del d16, dm, run16
            extras["batch16"] = b16
        del model
        torch.cuda.empty_cache()
        extras["w4a16_decode"] = w4_decode_extra(shape, device, peaks)
        extras["sparse_gemv_list_sweep"] = BX.list_gemv_sweep_extra(device, peaks)
        extras["block_llama2_7b_c2"] = BX.block_c2_extra(device)
        extras["model_sweep_configs3"] = BX.model_sweep_extra(device, merged=merged)
        extras["fold_tcgen05"] = BX.fold_extra(device)
        extras["calibration_n1"] = BX.calibration_extra(device)
        extras["rotation_variants"] = BX.rotation_variants_extra(device, synth.MODELS["llama2-7b"])

    cpu = None
    if rank == 0 and ws_n == 1 and not args.no_cpu_baseline:
        import oracle as O
        cpu = cpu_baseline(shape, O.site_ks(args.p, (1, 1, 1, 1), shape.d, shape.inter))

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws_n, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "bf16 weights, fp32 activations/accumulate", "data": "synthetic",
               "config": {"workload": CONFIG_NAME, "sparsity": args.p, "alpha": "uniform", "plan_k": list(plan),
                          "ctx": CTX, "batch": B, "layers": shape.layers, "vocab": shape.vocab,
                          "adapter": "folded beside down (one launch)" if merged else "separate GEMV",
                          "l2": "inputs larger than L2: every step streams the 17 GB model once",
                          "parallelism": f"replicas x{ws_n}" if ws_n > 1 else "single GPU",
                          "decode": "greedy tokens fed back (device), ctx 256"},
               "e2e": e2e, "gpu_launches": launches_per_step(B, shape.layers, merged) * args.steps,
               "clocks": clocks, "roofline": roofline, "cpu_baseline": cpu, "extras": extras}
        print(json.dumps(out))
    if ws_n > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
