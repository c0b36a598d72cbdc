"""Per-CUDA-line instruction and stall totals of one kernel in an ncu report:
python tools_ncu_lines.py rep kernel_regex [n]"""
import csv
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{rx}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ie = h.index("Instructions Executed")
ws = h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[hi + 1:]:
    if len(r) > ie and r[0] not in ("", "-"):
        try:
            data.append((int(r[ie] or 0), int(r[ws] or 0), int(r[0]), r[1]))
        except ValueError:
            pass
ti = sum(d[0] for d in data) or 1
tw = sum(d[1] for d in data) or 1
print(f"warp instructions {ti}  stall samples {tw}")
for i, w, ln, s in sorted(data, reverse=True)[:n]:
    print(f"{100 * i / ti:5.1f}% inst {100 * w / tw:5.1f}% stall  L{ln:5d} {s.strip()[:90]}")
