"""Record the measured DRAM traffic of fbx_pipeline for the bench's roofline line.

    python scripts/traffic.py gpurun_out/<name>.ncu-rep gpurun_out/<name>.log

Reads the ncu --set full capture (scripts/profile_kernel.sh) and the bench JSON
line of the same command (its ``roofline.plan_sha`` = sha256 of the generated plan source)
and writes profiles/traffic.json[<dag>]; bench.py uses the entry only while the
plan it compiles has that same hash.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rep, log = Path(sys.argv[1]), Path(sys.argv[2])
raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, vals = rows[0], rows[1], rows[2]


def metric(name, scale_units=True):
    j = h.index(name)
    v = float(vals[j].replace(",", ""))
    u = units[j]
    if scale_units:
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3,
              "ms": 1e6, "usecond": 1e3, "nsecond": 1, "msecond": 1e6}.get(u, 1)
    return v


line = next(x for x in reversed(log.read_text().splitlines()) if x.startswith("{"))
bench = json.loads(line)
dag = bench["config"]["workload"].split()[0]
rd, wr = metric("dram__bytes_read.sum"), metric("dram__bytes_write.sum")
entry = {
    "dram_bytes": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
    "ncu_duration_ns": int(metric("gpu__time_duration.sum")),
    "inst_executed": int(metric("smsp__inst_executed.sum", False)),
    "issue_active_pct": round(metric("smsp__issue_active.avg.pct_of_peak_sustained_active",
                                     False), 2),
    "algorithmic_bytes": bench["roofline"]["bytes_per_launch"]["total"],
    "plan_sha": bench["roofline"]["plan_sha"],
    "source": f"ncu --set full -k regex:fbx_pipeline -s 3 -c 1 ({rep.name})",
}
out = ROOT / "profiles" / "traffic.json"
doc = json.loads(out.read_text()) if out.exists() else {}
doc[dag] = entry
out.write_text(json.dumps(doc, indent=1) + "\n")
print(dag, json.dumps(entry))
