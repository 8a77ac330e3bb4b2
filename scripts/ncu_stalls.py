"""Warp-stall samples of an ncu report by reason, and the top lines per reason.

    python scripts/ncu_stalls.py gpurun_out/<name>.ncu-rep [n_lines]
"""
import csv
import io
import subprocess
import sys
from pathlib import Path

rep = Path(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
src = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
data = [r for r in rows[hdr + 1:] if len(r) > 8 and r[2] == "-"]
cu = rep.with_suffix(".cu")
text = cu.read_text().split("\n") if cu.exists() else []
cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = {h[i]: sum(int(r[i] or 0) for r in data) for i in cols}
allv = sum(tot.values()) or 1
for name, v in sorted(tot.items(), key=lambda x: -x[1]):
    if v / allv < 0.01:
        continue
    print(f"{name:26s} {100 * v / allv:5.1f}%")
    i = h.index(name)
    for r in sorted(data, key=lambda r: -int(r[i] or 0))[:n]:
        ln = int(r[0])
        line = text[ln - 1].strip() if ln - 1 < len(text) else r[1]
        print(f"      {ln:5d} {100 * int(r[i]) / allv:5.1f}%  {line[:90]}")
