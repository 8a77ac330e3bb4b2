"""Stall reasons summed over a line range of the profiled plan source.

    python scripts/ncu_range_stalls.py gpurun_out/<name>.ncu-rep FIRST LAST
"""
import csv
import io
import subprocess
import sys
from pathlib import Path

rep, a, b = Path(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
src = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
data = [r for r in rows[hdr + 1:] if len(r) > 8 and r[2] == "-"]
cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
allv = sum(int(r[i] or 0) for r in data for i in cols) or 1
sel = [r for r in data if a <= int(r[0]) <= b]
tot = {h[i]: sum(int(r[i] or 0) for r in sel) for i in cols}
s = sum(tot.values())
print(f"range {a}-{b}: {100 * s / allv:.1f}% of all stall samples")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k:26s} {100 * v / max(s, 1):5.1f}% of range")
