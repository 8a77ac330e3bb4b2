"""CPU: corpus, FBXC format, config/planner semantics, code generation + NVRTC,
and the C-ABI library surface (no GPU calls)."""

from __future__ import annotations

import hashlib
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, corpus

from paper_2210_07768_b200 import codegen, engine
from paper_2210_07768_b200.columns import (ChecksumError, ColumnImage, Kind, ViewImage, read_view,
                                           write_view)
from paper_2210_07768_b200.config import ConfigError, UnsupportedOnDevice, config_from_dict, load_config
from paper_2210_07768_b200.corpus import gen_corpus
from paper_2210_07768_b200.opgraph import expand_call_graph, layer_schedule
from paper_2210_07768_b200.workloads import DAGS, workload_config


def test_corpus_is_byte_identical_to_reference(goldens, tmp_path):
    for key, want in goldens["corpus_sha256"].items():
        rows, users, seed, views = map(int, key.split("_"))
        files = gen_corpus(tmp_path / key, rows=rows, users=users, seed=seed, views=views)
        got = {k: hashlib.sha256(Path(v).read_bytes()).hexdigest() for k, v in files.items()}
        assert got == want, key


@pytest.mark.parametrize("rows,users,seed,views", [(3000, 300, 7, 2), (1200, 200, 11, 1),
                                                   (4000, 5000, 2**40 + 3, 2), (0, 5, 1, 2)])
def test_fast_generator_is_byte_identical(rows, users, seed, views, tmp_path):
    from paper_2210_07768_b200.corpus import make_corpus, make_corpus_fast, write_corpus
    fa = write_corpus(make_corpus(rows, users, seed, views), tmp_path / "py")
    fb = write_corpus(make_corpus_fast(rows, users, seed, views), tmp_path / "c")
    for k in fa:
        assert fa[k].read_bytes() == fb[k].read_bytes(), k


def test_fbxc_roundtrip_and_crc(tmp_path):
    v = ViewImage.from_pydict([("a", Kind.INT64), ("s", Kind.UTF8), ("f", Kind.FLOAT32)],
                              {"a": [1, None, -3], "s": ["x", "é", None], "f": [0.5, None, 2.0]})
    p = write_view(v, tmp_path / "v.fbxc")
    r = read_view(p)
    for c in ("a", "s", "f"):
        assert r.columns[c].to_pylist() == v.columns[c].to_pylist()
    raw = bytearray(p.read_bytes())
    raw[-10] ^= 0xFF
    p.write_bytes(bytes(raw))
    with pytest.raises(ChecksumError):
        read_view(p)


# node / layer counts of the Appendix-B DAGs
@pytest.mark.parametrize("dag,nodes,layers", [("default", 7, 2), ("fig4", 8, 3),
                                              ("sign_heavy", 18, 2), ("cross_heavy", 18, 3),
                                              ("lookup_heavy", 24, 4)])
def test_layer_schedule_matches_reference_shape(dag, nodes, layers):
    c, d = corpus(2000, 300, 7)
    cfg = config_from_dict(workload_config(dag), d)
    dg = expand_call_graph(cfg.operators)
    plan = layer_schedule(dg)
    assert (len(dg.nodes), len(plan.layers)) == (nodes, layers)


def test_config_errors_mirror_reference(tmp_path):
    c, d = corpus(2000, 300, 7)
    raw = workload_config("default")
    raw["operators"][0]["body"]["fn"] = "nope:1"
    with pytest.raises(ConfigError):
        engine.prepare(config_from_dict(raw, d), compile_program=False)
    raw = workload_config("default")
    raw["emit"]["features"]["missing_col"] = 3
    with pytest.raises(ConfigError):
        engine.prepare(config_from_dict(raw, d), compile_program=False)
    raw = workload_config("default")
    raw["views"][0]["clean"]["filter"] = "nosuch < 3"
    with pytest.raises(ConfigError):
        engine.prepare(config_from_dict(raw, d), compile_program=False)
    (tmp_path / "bad.json").write_text("{")
    with pytest.raises(ConfigError):
        load_config(tmp_path / "bad.json")


def test_unsupported_constructs_are_plan_time_errors():
    c, d = corpus(2000, 300, 7)
    raw = workload_config("default")
    raw["views"][0]["clean"]["extract"] += [
        {"source": "meta", "path": f"u.k{i}", "output": f"k{i}", "kind": "utf8"} for i in range(8)]
    with pytest.raises(UnsupportedOnDevice):  # > 8 paths from one JSON source
        engine.prepare(config_from_dict(raw, d), compile_program=False)


def test_big_batch_plan_compiles():
    """batch_size > 1024: 512-row sub-tiles per chunk (merged after the run)."""
    c, d = corpus(2000, 300, 7)
    p = engine.prepare(config_from_dict(workload_config("sign_heavy", batch_size=100_000), d),
                       {"user_events": c.driver, "user_profile": c.profile}, c.basic)
    assert p.program.tiles_per_chunk == 196 and p.program.threads == 512
    assert p.cubin[:4] == b"\x7fELF"


def test_json_kind_plan_compiles():
    """Json-kind extraction (json.dumps re-serialisation) is generated on device."""
    c, d = corpus(2000, 300, 7)
    raw = workload_config("default")
    raw["views"][0]["clean"]["extract"].append(
        {"source": "meta", "path": "u", "output": "u_json", "kind": "json"})
    raw["operators"].append({"name": "uj", "inputs": ["u_json"], "outputs": ["uj"],
                             "body": {"fn": "hash:91"}})
    raw["emit"]["features"]["uj"] = 91
    p = engine.prepare(config_from_dict(raw, d),
                       {"user_events": c.driver, "user_profile": c.profile}, c.basic)
    assert p.cubin[:4] == b"\x7fELF"


def test_float_repr_plan_compiles():
    """str(Float32) (Python repr) is generated on device: the plan compiles."""
    c, d = corpus(2000, 300, 7)
    raw = workload_config("default")
    raw["operators"].append({"name": "sc", "inputs": ["score"], "outputs": ["sc"],
                             "pre": [{"fn": "lower"}], "body": {"fn": "hash:90"}})
    raw["emit"]["features"]["sc"] = 90
    p = engine.prepare(config_from_dict(raw, d),
                       {"user_events": c.driver, "user_profile": c.profile}, c.basic)
    assert p.cubin[:4] == b"\x7fELF"


def test_f32_repr_model_matches_python():
    """decimal_tables.f32_repr (model of fbx::f32_repr) == repr() of float32 values."""
    from paper_2210_07768_b200.decimal_tables import check_f32_repr
    assert check_f32_repr(60000) > 60000


@pytest.mark.parametrize("dag", DAGS)
def test_plans_compile_for_sm100a(dag):
    """Every Appendix-B plan generates and NVRTC-compiles to an sm_100a cubin."""
    c, d = corpus(2000, 300, 7)
    p = engine.prepare(config_from_dict(workload_config(dag), d),
                       {"user_events": c.driver, "user_profile": c.profile}, c.basic)
    assert p.cubin[:4] == b"\x7fELF"
    assert "fbx_pipeline" in p.program.kernels


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2210_07768_b200 import runtime
    L = runtime.lib()
    declared = set()
    for h in (ROOT / "include").glob("*.h"):
        declared |= set(re.findall(r"\b(fbx_\w+)\s*\(", h.read_text()))
    assert declared, "no declarations found"
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert L.fbx_version().decode().startswith("fbx")
    assert isinstance(L.fbx_error_message(None), bytes)
    assert ctypes.sizeof(ctypes.c_uint64) * 384 == 3072  # fbx_params


def test_engine_refuses_cpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c, d = corpus(2000, 300, 7)
    p = engine.prepare(config_from_dict(workload_config("default"), d),
                       {"user_events": c.driver, "user_profile": c.profile}, c.basic,
                       compile_program=False)
    with pytest.raises(RuntimeError):
        engine.Engine(p, {"user_events": c.driver, "user_profile": c.profile}, c.basic)


def test_unicode_lower_tables_current_and_exact():
    """Device lower() tables regenerate identically from this CPython, and the
    device algorithm (emulated) equals str.lower on fuzzed strings."""
    import random
    import unicodedata

    from paper_2210_07768_b200 import unicode_tables as U
    if unicodedata.unidata_version != "15.0.0":
        pytest.skip("tables are pinned to Unicode 15.0 (CPython 3.12)")
    assert U.render() == U.HEADER.read_text()
    rng = random.Random(5)
    alphabet = [chr(c) for c in list(range(0x20, 0x7F)) + [
        0xC0, 0xC9, 0xDF, 0x130, 0x131, 0x3A3, 0x3C3, 0x391, 0x1E9E, 0x10400, 0x345, 0x2126,
        0x212A, 0x1F88, 0x1FBC, 0x307, 0xAD, 0x2019, 0x1C4, 0x1C5, 0x24B6, 0x10A0, 0xFF21]]
    for _ in range(3000):
        s = "".join(rng.choice(alphabet) for _ in range(rng.randint(0, 12)))
        assert U.emulate_lower(s) == s.lower(), s


def test_decimal_to_double_model_and_tables():
    """The device's bracketing Eisel-Lemire (modelled exactly in Python) equals
    float() on random decimals; the generated power table is current."""
    from paper_2210_07768_b200 import decimal_tables as Dt
    assert Dt.render() == Dt.HEADER.read_text()
    slow = Dt.check_random(30000, 11)  # asserts equality for every non-slow case
    assert slow < 60


def test_f64_repr_model_matches_python():
    """decimal_tables.f64_repr (model of fbx::f64_repr) == repr() of doubles."""
    from paper_2210_07768_b200.decimal_tables import check_f64_repr
    assert check_f64_repr(20000) > 40000


def test_json_canon_model_matches_json_dumps():
    """jsoncanon.json_canon (model of fbx::json_canon) == json.dumps(sort_keys, (",", ":"))."""
    from paper_2210_07768_b200.jsoncanon import check_json_canon
    assert check_json_canon(4000) == 4000


@pytest.mark.parametrize("seed", [12, 1000, 1099])
def test_fast_generator_matches_reference_shard_files(seed, tmp_path):
    """The 1M-row shards the bench regenerates with the C generator are the exact
    files the unmodified reference generated for tests/golden/shard_goldens.json
    (sha256 of every file), so the per-shard reference digests apply to them."""
    import json
    from paper_2210_07768_b200.corpus import make_corpus_fast, write_corpus
    doc = json.loads((ROOT / "tests" / "golden" / "shard_goldens.json").read_text())
    want = next(r for r in doc["shards"] if r["seed"] == seed)["corpus_sha256"]
    files = write_corpus(make_corpus_fast(1_000_000, 5000, seed, 2), tmp_path)
    got = {k: hashlib.sha256(Path(v).read_bytes()).hexdigest() for k, v in files.items()}
    assert got == want


def test_shard_goldens_compose_to_c5():
    """C5's run digest is the XOR of its 100 independently generated shards."""
    import json
    doc = json.loads((ROOT / "tests" / "golden" / "shard_goldens.json").read_text())
    c5 = [r for r in doc["shards"] if r["dag"] == "default" and 1000 <= r["seed"] < 1100]
    assert len(c5) == 100 and sorted(r["seed"] for r in c5) == list(range(1000, 1100))
    x = 0
    for r in c5:
        x ^= int(r["digest"], 16)
    assert f"0x{x:016x}" == doc["c5"]["xor_digest"]
    assert sum(r["rows"] for r in c5) == 100_000_000


# ---- FBXC header validation: the reference's error types and messages --------------

def _fbxc_cases(tmp_path):
    """(name, bytes) of damaged FBXC files, as the reference's own tests make them
    (test_columnstore.py: bad magic, version 2, truncated, tiny) plus a cut
    column name, a cut directory and a body one byte long."""
    import struct as st
    from paper_2210_07768_b200.columns import ColumnImage, Kind, ViewImage, write_view
    v = ViewImage.from_pydict([("id", Kind.INT64), ("name", Kind.UTF8)],
                              {"id": [1, 2, None], "name": ["a", None, "ccc"]}, ("id",))
    path = tmp_path / "ok.fbxc"
    write_view(v, path)
    blob = path.read_bytes()
    bad_magic = b"XXXX" + blob[4:]
    v2 = blob[:4] + st.pack("<H", 2) + blob[6:]
    return {"bad_magic": bad_magic, "version": v2, "truncated": blob[:-5], "tiny": b"FB",
            "cut_name": blob[:22], "cut_directory": blob[:40], "long": blob + b"\0",
            "empty": b""}


def test_fbxc_header_errors_match_reference(tmp_path):
    import sys
    from conftest import reference_package_path
    from paper_2210_07768_b200 import columns as C
    ref = reference_package_path()
    for name, data in _fbxc_cases(tmp_path).items():
        f = tmp_path / f"{name}.fbxc"
        f.write_bytes(data)
        with pytest.raises(C.FormatError) as got:
            C.open_view(f)
        want = {"bad_magic": C.BadMagicError, "version": C.UnsupportedVersionError,
                "tiny": C.TruncatedError, "truncated": C.TruncatedError,
                "empty": C.TruncatedError}.get(name)
        if want is not None:
            assert type(got.value) is want, (name, got.value)
        if ref is None:
            continue
        if str(ref) not in sys.path:
            sys.path.insert(0, str(ref))
        import featurebox.columnstore as RC
        with pytest.raises(RC.FormatError) as exp:
            RC.open_view(f)
        assert type(got.value).__name__ == type(exp.value).__name__, name
        assert str(got.value) == str(exp.value), name


def test_fbxc_checksum_error_matches_reference(tmp_path):
    import sys
    from conftest import reference_package_path
    from paper_2210_07768_b200 import columns as C
    from paper_2210_07768_b200.columns import Kind, ViewImage, write_view
    v = ViewImage.from_pydict([("id", Kind.INT64)], {"id": [1, 2, 3]}, ("id",))
    f = tmp_path / "crc.fbxc"
    write_view(v, f)
    raw = bytearray(f.read_bytes())
    raw[-9] ^= 0x40
    f.write_bytes(bytes(raw))
    with pytest.raises(C.ChecksumError) as got:
        C.read_view(f)
    ref = reference_package_path()
    if ref is None:
        return
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import featurebox.columnstore as RC
    with pytest.raises(RC.ChecksumError) as exp:
        RC.read_columns(RC.open_view(f), None)
    assert str(got.value) == str(exp.value)
