"""Executed warp-instructions per CUDA source line for one profiled launch (ncu source page).
usage: python tools/ncu_instr.py REPORT.ncu-rep LAUNCH_INDEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, res, f = None, [], None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] and hdr and len(r) > 8:
        try:
            ie = int(r[hdr.index("Instructions Executed")])
        except ValueError:
            continue
        if ie:
            res.append((ie, f, r[0], r[1].strip()[:90]))
tot = sum(x[0] for x in res)
print("warp-instructions executed", tot)
for ie, f, ln, src in sorted(res, key=lambda t: -t[0])[:top]:
    print(f"{ie:9d} {100 * ie / tot:5.1f}% {f}:{ln} {src}")
