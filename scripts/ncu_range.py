"""Instructions / stall samples per source line inside a line range of the
profiled plan source (e.g. one device function).

    python scripts/ncu_range.py gpurun_out/<name>.ncu-rep FIRST LAST
"""
import csv
import io
import subprocess
import sys
from pathlib import Path

rep, a, b = Path(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
text = rep.with_suffix(".cu").read_text().split("\n")
src = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
data = [r for r in rows[hdr + 1:] if len(r) > 8 and r[2] == "-"]
te = sum(int(r[7]) for r in data) or 1
tot = 0
for r in data:
    ln = int(r[0])
    if a <= ln <= b and int(r[7]):
        tot += int(r[7])
        print(f"{ln:5d} inst {100 * int(r[7]) / te:5.2f}%  {text[ln - 1].strip()[:100]}")
print(f"range total {100 * tot / te:.2f}% of {te} warp-inst")
