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


# ---- the reference's CLI behaviours (pkg/tests/test_cli.py), restated --------------

def _cli(capsys, argv):
    code = cli.main(argv)
    out = capsys.readouterr()
    return code, out.out, out.err


def test_gen_corpus_outputs_and_determinism(tmp_path, capsys):
    import filecmp
    code, out, _ = _cli(capsys, ["gen-corpus", "--out", str(tmp_path / "a"), "--instances",
                                 "200", "--users", "20"])
    assert code == 0
    names = [ln.split(":")[0] for ln in out.strip().splitlines()]
    assert names == sorted(names)
    assert set(names) == {"basic", "city_dict", "config", "user_events", "user_profile"}
    assert cli.main(["gen-corpus", "--out", str(tmp_path / "b"), "--instances", "200",
                     "--users", "20"]) == 0
    for name in ("user_events.fbxc", "user_profile.fbxc", "basic.fbxc", "city_dict.tsv",
                 "pipeline.json"):
        assert filecmp.cmp(tmp_path / "a" / name, tmp_path / "b" / name, shallow=False), name
    capsys.readouterr()
    code, out, _ = _cli(capsys, ["gen-corpus", "--out", str(tmp_path / "c"), "--instances",
                                 "150", "--views", "1"])
    assert code == 0
    assert {ln.split(":")[0] for ln in out.strip().splitlines()} == {"basic", "config",
                                                                    "user_events"}


def test_cli_usage_errors(tmp_path, capsys):
    code, _, err = _cli(capsys, ["gen-corpus", "--out", str(tmp_path), "--instances", "-5"])
    assert code == 2 and "error:" in err
    for argv in (["gen-corpus", "--out", str(tmp_path), "--views", "3"],
                 ["run", "--config", str(tmp_path / "x.json"), "--frobnicate"],
                 ["made-up-command"], ["run"]):
        with pytest.raises(SystemExit) as exc:
            cli.main(argv)
        assert exc.value.code == 2
    bad = tmp_path / "bad.json"
    bad.write_text('{"views": []}')
    assert cli.main(["run", "--config", str(bad)]) == 2


def test_thread_env_invalid_is_usage_error(tmp_path, capsys, monkeypatch):
    """FEATUREBOX_THREADS must be an integer >= 1 (device.py:81-96): a ConfigError
    when the run starts, exit 2 -- before any device work."""
    d = tmp_path / "c"
    assert cli.main(["gen-corpus", "--out", str(d), "--instances", "100", "--users", "9"]) == 0
    capsys.readouterr()
    monkeypatch.setenv("FEATUREBOX_THREADS", "many")
    code, _, err = _cli(capsys, ["run", "--config", str(d / "pipeline.json")])
    assert code == 2 and "FEATUREBOX_THREADS" in err


@pytest.fixture(scope="module")
def cli_corpus(tmp_path_factory):
    dest = tmp_path_factory.mktemp("clicorpus")
    assert cli.main(["gen-corpus", "--out", str(dest), "--instances", "600",
                     "--users", "80"]) == 0
    return dest


@pytest.mark.gpu
def test_run_modes_report_file_overrides(cli_corpus, capsys, tmp_path, monkeypatch):
    monkeypatch.delenv("FEATUREBOX_THREADS", raising=False)
    config = str(cli_corpus / "pipeline.json")
    code, out_st, _ = _cli(capsys, ["run", "--config", config, "--mode", "staged",
                                    "--staging", str(tmp_path / "st")])
    assert code == 0
    code, out_pp, _ = _cli(capsys, ["run", "--config", config, "--mode", "pipelined",
                                    "--report", str(tmp_path / "r.txt")])
    assert code == 0
    st, pp = parse_report_block(out_st), parse_report_block(out_pp)
    assert st["digest"] == pp["digest"] and (st["mode"], pp["mode"]) == ("staged", "pipelined")
    assert int(st["intermediate_bytes"]) > 0 and int(pp["intermediate_bytes"]) == 0
    assert parse_report_block((tmp_path / "r.txt").read_text()) == pp
    code, out, _ = _cli(capsys, ["run", "--config", config, "--batch-size", "100"])
    kv = parse_report_block(out)
    assert code == 0 and kv["batch_size"] == "100"
    assert int(kv["batches"]) == -(-int(kv["instances"]) // 100)
    digests = set()
    for workers in ("1", "3"):
        code, out, _ = _cli(capsys, ["run", "--config", config, "--workers", workers])
        kv = parse_report_block(out)
        assert code == 0 and kv["workers"] == workers
        digests.add(kv["digest"])
    assert len(digests) == 1
    monkeypatch.setenv("FEATUREBOX_THREADS", "1")
    code, out, _ = _cli(capsys, ["run", "--config", config, "--workers", "8"])
    assert code == 0 and parse_report_block(out)["workers"] == "1"


@pytest.mark.gpu
def test_run_empty_corpus_and_corrupt_data(tmp_path, capsys, cli_corpus):
    import shutil
    assert cli.main(["gen-corpus", "--out", str(tmp_path / "e"), "--instances", "0"]) == 0
    capsys.readouterr()
    code, out, _ = _cli(capsys, ["run", "--config", str(tmp_path / "e" / "pipeline.json")])
    kv = parse_report_block(out)
    assert code == 0 and (kv["instances"], kv["batches"], kv["digest"]) == \
        ("0", "0", "0x0000000000000000")
    work = tmp_path / "corpus"
    shutil.copytree(cli_corpus, work)
    blob = bytearray((work / "user_events.fbxc").read_bytes())
    blob[-30] ^= 0x55
    (work / "user_events.fbxc").write_bytes(blob)
    code, _, err = _cli(capsys, ["run", "--config", str(work / "pipeline.json"), "--mode",
                                 "staged"])
    assert code == 1 and "stage" in err and "clean" in err
