"""Summarise an ncu report of fbx_pipeline: key metrics + top source lines.

    python scripts/ncu_lines.py gpurun_out/<name>.ncu-rep [n_lines]
"""
import csv
import io
import subprocess
import sys
from pathlib import Path

rep = Path(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
if rows:
    h, units, vals = rows[0], rows[1], rows[2]
    for m in METRICS:
        if m in h:
            j = h.index(m)
            print(f"{m:62s} {vals[j]:>16s} {units[j]}")
src = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
data = [r for r in rows[hdr + 1:] if len(r) > 8 and r[2] == "-"]
cu = rep.with_suffix(".cu")
text = cu.read_text().split("\n") if cu.exists() else []
ts = sum(int(r[4]) for r in data) or 1
te = sum(int(r[7]) for r in data) or 1
print(f"\nsamples {ts}  warp-inst {te}")
for r in sorted(data, key=lambda r: -int(r[4]))[:n]:
    ln = int(r[0])
    line = text[ln - 1].strip() if ln - 1 < len(text) else r[1]
    print(f"{ln:5d} stall {100 * int(r[4]) / ts:5.1f}%  inst {100 * int(r[7]) / te:5.1f}%  {line[:92]}")
