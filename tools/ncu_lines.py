"""Aggregate ncu source-page warp-stall samples per CUDA source line for one profiled launch
(needs -lineinfo).  usage: python tools/ncu_lines.py REPORT.ncu-rep LAUNCH_INDEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, fname = [], None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] and len(r) > 6:          # a source line row (aggregated over its SASS)
        try:
            s = int(r[4])
        except ValueError:
            continue
        if s:
            res.append((s, fname, r[0], r[1].strip()[:80]))
tot = sum(t[0] for t in res)
print("total samples", tot)
for s, f, ln, src in sorted(res, key=lambda t: -t[0])[:top]:
    print(f"{100.0 * s / tot:5.1f}% {f}:{ln:>4} {src}")
