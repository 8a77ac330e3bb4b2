"""The command-line front end (the reference's cli.py on the B200 engine):
exit codes, gen-corpus, plan on CPU; run (both modes) on the GPU."""

from __future__ import annotations

import tempfile
from pathlib import Path

import pytest

from paper_2210_07768_b200 import cli
from paper_2210_07768_b200.engine import parse_report_block


def test_gen_corpus_and_plan(capsys):
    d = Path(tempfile.mkdtemp(prefix="fbxcli")) / "c"
    assert cli.main(["gen-corpus", "--out", str(d), "--instances", "400", "--users", "40"]) == 0
    out = capsys.readouterr().out
    assert "config:" in out and (d / "pipeline.json").exists()
    rep = d / "plan.txt"
    assert cli.main(["plan", "--config", str(d / "pipeline.json"), "--report", str(rep)]) == 0
    text = rep.read_text()
    assert text.startswith("plan: 7 operators, 2 layers") and "kernel: fbx_pipeline" in text


def test_usage_and_config_errors_exit_2(tmp_path, capsys):
    assert cli.main(["run", "--config", str(tmp_path / "missing.json")]) == 2
    (tmp_path / "bad.json").write_text('{"driver": "x"}')
    assert cli.main(["plan", "--config", str(tmp_path / "bad.json")]) == 2
    assert cli.main(["gen-corpus", "--out", str(tmp_path / "c"), "--users", "0"]) == 2
    assert "error:" in capsys.readouterr().err


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["pipelined", "staged"])
def test_run_both_modes(mode, capsys):
    """The 2k / 300 / seed-7 corpus (SURVEY Appendix B golden 0x483d13d62f945805)."""
    d = Path(tempfile.mkdtemp(prefix="fbxcli"))
    assert cli.main(["gen-corpus", "--out", str(d), "--instances", "2000", "--users", "300",
                     "--seed", "7"]) == 0
    capsys.readouterr()
    args = ["run", "--config", str(d / "pipeline.json"), "--mode", mode]
    if mode == "staged":
        args += ["--staging", str(d / "stage")]
    assert cli.main(args) == 0
    kv = parse_report_block(capsys.readouterr().out)
    assert kv["digest"] == "0x483d13d62f945805" and kv["instances"] == "1764"
    assert kv["mode"] == mode


def test_sharded_needs_torchrun(tmp_path, capsys, monkeypatch):
    d = tmp_path / "c"
    assert cli.main(["gen-corpus", "--out", str(d), "--instances", "400", "--users", "40"]) == 0
    monkeypatch.delenv("RANK", raising=False)
    assert cli.main(["run", "--config", str(d / "pipeline.json"), "--sharded"]) == 2
    assert "torchrun" in capsys.readouterr().err


@pytest.mark.gpu
def test_run_sharded_under_torchrun(tmp_path):
    """`torchrun -m ...cli run --sharded` with the box's one GPU: rank 0 prints the
    single run's report (the published 2k corpus digest)."""
    import subprocess
    import sys
    d = tmp_path / "c"
    assert cli.main(["gen-corpus", "--out", str(d), "--instances", "2000", "--users", "300",
                     "--seed", "7"]) == 0
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
                        "--master-port", "29531", "-m", "paper_2210_07768_b200.cli", "run",
                        "--config", str(d / "pipeline.json"), "--sharded"],
                       capture_output=True, text=True, cwd=root, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    kv = parse_report_block(r.stdout)
    assert kv["digest"] == "0x483d13d62f945805" and kv["instances"] == "1764"
