"""Per-CUDA-source-line stall samples of one kernel in an ncu report
(``ncu -i rep --page source --print-source cuda,sass``).  Usage:
python tools/ncu_lines.py rep.ncu-rep [top-N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[2]
si = hdr.index("Warp Stall Sampling (All Samples)")
lines = {}
cur = None
total = 0
for r in rows[3:]:
    if len(r) <= si:
        continue
    if r[0]:
        if r[0].isdigit():
            cur = (int(r[0]), r[1][:90])
        continue
    try:
        v = int(r[si])
    except ValueError:
        continue
    lines[cur] = lines.get(cur, 0) + v
    total += v
for (ln, src), v in sorted(lines.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * v / max(total, 1):5.1f}%  {ln:5d}  {src}")
