#!/usr/bin/env python
"""Summarise tools/traffic.sh's ncu CSV (one decode step's kernels) into profiles/traffic.json,
keyed by the library source hash (bench.py reads `traffic` from it only at the same sources),
and print the launch list with per-kernel shares.
Usage: python tools/traffic_summarize.py gpurun_out/traffic_B1_p0.4.csv [B] [p]"""
import csv
import json
import os
import re
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def parse(path):
    rows = defaultdict(dict)
    names = {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        i = int(r["ID"])
        names[i] = r["Kernel Name"]
        v = r["Metric Value"].replace(",", "")
        try:
            rows[i][r["Metric Name"]] = float(v)
        except ValueError:
            pass
    return names, rows


def short(n):
    n = re.sub(r"\(.*", "", n)
    return n.replace("larosa::", "")


def main():
    path = sys.argv[1]
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    p = float(sys.argv[3]) if len(sys.argv) > 3 else 0.4
    names, rows = parse(path)
    tot_b = tot_t = 0.0
    per = defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in rows.items():
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        t = m.get("gpu__time_duration.sum", 0.0)
        # units: ncu reports bytes in byte multiples per its unit column; normalise via the unit-less value
        tot_b += b
        tot_t += t
        k = short(names[i])
        per[k][0] += 1
        per[k][1] += t
        per[k][2] += b
    import bench
    rec_path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        rec = json.load(open(rec_path))
    except Exception:
        rec = {}
    if rec.get("source_hash") != bench.source_hash():
        rec = {"source_hash": bench.source_hash(), "steps": {}}
    rec["steps"][f"B{B}_p{p}"] = {
        "dram_bytes_per_step": tot_b, "kernels_per_step": sum(v[0] for v in per.values()),
        "serialised_kernel_time_ns": tot_t,
        "per_kernel": {k: {"launches": v[0], "time_share": v[1] / tot_t, "dram_bytes": v[2]}
                       for k, v in sorted(per.items(), key=lambda kv: -kv[1][1])}}
    json.dump(rec, open(rec_path, "w"), indent=1)
    print(f"B={B} p={p}: {sum(v[0] for v in per.values())} kernels, DRAM {tot_b / 1e9:.3f} GB, "
          f"serialised {tot_t / 1e3:.1f} us")
    for k, v in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:60s} x{v[0]:4d}  {100 * v[1] / tot_t:5.1f}%  {v[1] / 1e3:8.1f} us  {v[2] / 1e6:9.1f} MB")


if __name__ == "__main__":
    main()
