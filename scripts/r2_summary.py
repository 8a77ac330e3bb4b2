"""Write profiles/r2_final.md from the round-2 measurement captures in gpurun_out/
(scripts/round2_measure.sh): the launch list, the bench line's kernel split, and per
DAG the ncu metrics, top source lines, stall reasons and per-function split."""
import collections
import csv
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
P, G = ROOT / "profiles", ROOT / "gpurun_out"
out = ["# Round 2 final -- ncu of fbx_pipeline (one B200), launch list, bench lines\n",
       "Captures: `ncu --set full --clock-control none --import-source on -k regex:fbx_pipeline "
       "-s 3 -c 1` of `bench.py --dag <dag> --steps 1 --warmup 3` and the launch list of "
       "`bench.py --steps 2 --warmup 3` (scripts/round2_measure.sh) under gpurun.  Bench lines: "
       "profiles/r2_bench_dags.jsonl (five Appendix-B DAGs, 1M records each, goldens checked), "
       "profiles/r2_bench_full.json (the default line incl. the reference's CPU run), "
       "profiles/r2_bench_c5_100m.json (C5).  DRAM traffic per plan: profiles/traffic.json, "
       "keyed by the sha256 of the generated plan source (bench.py reads an entry when the "
       "plan it generates has the same hash).\n",
       "## Launch list (ncu gpu__time_duration, --clock-control none; cold-cache, serialised)\n```"]
rows = list(csv.reader(open(P / "r2_launches.csv")))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[start + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        agg.setdefault(r[ki][:60], []).append(float(r[vi].replace(",", "")))
for k, v in agg.items():
    out.append(f"{k:60s} n={len(v):3d} avg={sum(v) / len(v) / 1000:8.1f} us")
out.append("```")
full = json.loads((P / "r2_bench_full.json").read_text())
r = full["roofline"]
out.append("Per bench step (one CUDA graph replay): the side / basic table memsets, "
           "fbx_side_prep_all (index builds, one launch), k_idset_clear, k_state_reset, "
           "fbx_pipeline; k_flush is the L2 flush between steps (outside the timed events).  "
           f"Bench line (profiles/r2_bench_full.json): fbx_pipeline {r['kernel_ms']} ms of a "
           f"{full['ms_per_step']:.4f} ms step (CUDA events), index builds "
           f"{r['index_build_ms']} ms, frac {r['frac']}, traffic {r['traffic']} B per launch.\n")
for d, title in (("sign_heavy", "sign_heavy (C2)"), ("cross_heavy", "cross_heavy (C3)"),
                 ("lookup_heavy", "lookup_heavy (C4)")):
    rep = G / f"r2_full_{d}.ncu-rep"
    out.append(f"## {title}, 1M records\n```")
    out.append(subprocess.run(["python", "scripts/ncu_lines.py", str(rep), "16"],
                              capture_output=True, text=True, cwd=ROOT).stdout.rstrip())
    out.append("```")
    for scr in ("scripts/ncu_stalls.py", "scripts/ncu_funcs.py"):
        txt = subprocess.run(["python", scr, str(rep)], capture_output=True, text=True,
                             cwd=ROOT).stdout.rstrip().splitlines()[:25]
        if txt:
            out.append("```\n" + "\n".join(txt) + "\n```")
(P / "r2_final.md").write_text("\n".join(out) + "\n")
print("wrote", P / "r2_final.md")
