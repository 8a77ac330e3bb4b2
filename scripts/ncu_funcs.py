"""Aggregate an fbx_pipeline ncu source page by device function / kernel region.

    python scripts/ncu_funcs.py gpurun_out/<name>.ncu-rep
"""
import csv
import io
import re
import subprocess
import sys
from pathlib import Path

rep = Path(sys.argv[1])
text = rep.with_suffix(".cu").read_text().split("\n")
# function / region boundaries: FBX_DI/FBX_NI definitions and the generated "// ----" markers
marks = []
for i, line in enumerate(text, 1):
    m = re.match(r"\s*(?:template <[^>]*>\s*)?(?:FBX_DI|FBX_NI|static FBX_DI)\s+[\w:<>,\s\*&]+?\s(\w+)\(", line)
    if m:
        marks.append((i, "fn " + m.group(1)))
    elif line.strip().startswith("// ----") or line.strip().startswith("// node "):
        marks.append((i, line.strip()[:60]))
    elif line.startswith("struct ") or line.startswith("extern \"C\""):
        marks.append((i, line.strip()[:40]))
marks.sort()
src = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
data = [r for r in rows[hdr + 1:] if len(r) > 8 and r[2] == "-"]
agg = {}
for r in data:
    ln = int(r[0])
    name = "?"
    for start, nm in marks:
        if start <= ln:
            name = nm
        else:
            break
    a = agg.setdefault(name, [0, 0])
    a[0] += int(r[4])
    a[1] += int(r[7])
ts = sum(v[0] for v in agg.values()) or 1
te = sum(v[1] for v in agg.values()) or 1
for nm, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:35]:
    print(f"inst {100 * e / te:5.1f}%  stall {100 * s / ts:5.1f}%  {nm}")
