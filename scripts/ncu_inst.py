"""Top source lines of an ncu report by executed warp-instructions, plus per-function totals.

    python scripts/ncu_inst.py gpurun_out/<name>.ncu-rep [n_lines]
"""
import csv
import io
import re
import subprocess
import sys
from pathlib import Path

rep = Path(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
src = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
data = [r for r in rows[hdr + 1:] if len(r) > 8 and r[2] == "-"]
cu = rep.with_suffix(".cu")
text = cu.read_text().split("\n") if cu.exists() else []
te = sum(int(r[7]) for r in data) or 1
# enclosing function of each line: last line above matching a definition
defs = []
for i, t in enumerate(text):
    m = re.match(r"\s*(?:template\s*<[^>]*>\s*)?(?:FBX_DI|__device__|extern \"C\" __global__)[^(]*?(\w+)\s*\(", t)
    if m:
        defs.append((i + 1, m.group(1)))
def fn_of(ln):
    name = "?"
    for d, nm in defs:
        if d <= ln:
            name = nm
        else:
            break
    return name
tot = {}
for r in data:
    f = fn_of(int(r[0]))
    tot[f] = tot.get(f, 0) + int(r[7])
print(f"warp-inst {te}")
for f, v in sorted(tot.items(), key=lambda x: -x[1])[:30]:
    print(f"  {100 * v / te:5.1f}%  {f}")
print()
for r in sorted(data, key=lambda r: -int(r[7]))[:n]:
    ln = int(r[0])
    line = text[ln - 1].strip() if ln - 1 < len(text) else r[1]
    print(f"{ln:5d} inst {100 * int(r[7]) / te:5.1f}%  {line[:100]}")
