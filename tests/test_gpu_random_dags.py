"""GPU: randomly generated operator DAGs (the reference's config schema) against the
CPU oracle -- every operator of the library (token / lower / trim / lookup pre-ops,
hash / concat bodies, mix / fold posts), chained through earlier operators' outputs,
over driver and side-view columns, emitted with the basic features.  Bit-exact CSR or the
same failure stage."""

from __future__ import annotations

import os
import random

import numpy as np
import pytest

import featurebox_oracle as O
from conftest import corpus

pytestmark = pytest.mark.gpu

STR_COLS = ["query", "city_x", "city"]
INT_COLS = ["age", "user_id"]
F32_COLS = ["score"]
TABLES = {"city_dict": {"path": "city_dict.tsv", "default": 0},
          "query_dict": {"path": "query_dict.tsv", "default": 3},
          "token_dict": {"path": "token_dict.tsv", "default": 0},
          "user_dict": {"path": "user_dict.tsv", "default": 7}}


def random_dag(seed: int):
    rng = random.Random(seed)
    ops, feats = [], {}
    str_outs: list[str] = []
    u64_outs: list[str] = []
    slot = 100
    for k in range(rng.randrange(2, 8)):
        name = f"op{k}"
        if rng.random() < 0.25 and (str_outs or True):
            # concat of 1..3 strings (pre-ops allowed), output str
            n_in = rng.randrange(1, 4)
            ins, pre = [], []
            for a in range(n_in):
                c = rng.choice(STR_COLS + str_outs + INT_COLS[:1])
                ins.append(c)
                if c in STR_COLS + str_outs and rng.random() < 0.5:
                    pre.append({"fn": rng.choice(["lower", "trim", "token: :0", "token: :1",
                                                  "token:,:0"]), "arg": a})
            op = {"name": name, "inputs": ins, "outputs": [f"{name}_s"],
                  "body": {"fn": rng.choice(["concat:|", "concat:", "concat: - "])}}
            if pre:
                op["pre"] = pre
            ops.append(op)
            str_outs.append(f"{name}_s")
            continue
        n_in = rng.randrange(1, 4)
        ins, pre = [], []
        for a in range(n_in):
            c = rng.choice(STR_COLS + INT_COLS + F32_COLS + str_outs + u64_outs)
            ins.append(c)
            r = rng.random()
            if c in STR_COLS + str_outs and r < 0.5:
                pre.append({"fn": rng.choice(["lower", "trim", "token: :0", "token: :2",
                                              "lookup:city_dict", "lookup:query_dict",
                                              "lookup:token_dict"]), "arg": a})
            elif c in ("user_id",) and r < 0.3:
                pre.append({"fn": "lookup:user_dict", "arg": a})
            elif c in u64_outs and r < 0.3:
                pre.append({"fn": rng.choice(["mix", "fold"]), "arg": a})
        outs = [f"{name}_h"]
        post = []
        if rng.random() < 0.5:
            outs = [f"{name}_h{j}" for j in range(rng.randrange(1, 3))]
            post = [{"fn": rng.choice(["mix", "fold", "id"])} for _ in outs]
        op = {"name": name, "inputs": ins, "outputs": outs, "body": {"fn": f"hash:{slot}"}}
        if pre:
            op["pre"] = pre
        if post:
            op["post"] = post
        ops.append(op)
        for o in outs:
            u64_outs.append(o)
            feats[o] = slot if rng.random() < 0.8 else 100  # some shared slots (dedup)
        slot += 1
    if not feats:
        ops.append({"name": "last", "inputs": ["query"], "outputs": ["last_h"],
                    "body": {"fn": "hash:99"}})
        feats["last_h"] = 99
    feats.update({"basic_a": 40, "basic_b": 41})
    return ops, feats


@pytest.mark.parametrize("seed", range(int(os.environ.get("FBX_RANDOM_DAGS", "24"))))
def test_random_dag_matches_oracle(seed):
    from paper_2210_07768_b200.config import ConfigError, config_from_dict
    from paper_2210_07768_b200.engine import run_views
    from paper_2210_07768_b200.workloads import workload_config
    c, d = corpus(3000, 400, 13 + seed % 3)
    raw = workload_config("default", batch_size=[512, 256, 100, 3000][seed % 4])
    ops, feats = random_dag(seed)
    raw["operators"] = ops
    raw["emit"] = {"features": feats}
    raw["tables"] = TABLES
    views = {"user_events": c.driver, "user_profile": c.profile}
    try:
        cfg = config_from_dict(raw, d)
    except ConfigError:
        pytest.skip("generated config rejected by the reference schema")
    tables, sizes = O.load_tables(raw["tables"], d)
    try:
        ref = O.run_pipelined(raw, views, c.basic, tables, sizes)
        ref_err = None
    except O.OracleError as e:
        ref, ref_err = None, e
    except ConfigError:
        pytest.skip("generated config rejected by the oracle")
    try:
        got = run_views(cfg, views, c.basic, collect=True)
        got_err = None
    except Exception as e:  # noqa: BLE001
        got, got_err = None, e
    if ref_err is not None:
        assert got_err is not None, f"oracle failed ({ref_err}), engine did not"
        assert getattr(got_err, "stage", None) == ref_err.stage, (got_err, ref_err)
        return
    assert got_err is None, got_err
    assert (got.report.digest, got.report.instances, got.report.signs) == \
        (ref.digest, ref.instances, ref.signs)
    np.testing.assert_array_equal(got.csr["ids"], np.array(ref.ids, np.uint64))
    np.testing.assert_array_equal(got.csr["offsets"], np.array(ref.offsets, np.uint64))
    np.testing.assert_array_equal(got.csr["slots"], np.array(ref.slots, np.uint16))
    np.testing.assert_array_equal(got.csr["signs"], np.array(ref.values, np.uint64))


@pytest.mark.parametrize("seed", range(int(os.environ.get("FBX_RANDOM_DAGS", "24")) // 2))
def test_random_dag_on_adversarial_records(seed, tmp_path):
    """Random DAGs over the adversarial records of test_gpu_edge (Unicode / ragged
    queries, escaped and malformed JSON, nulls, int / float corner values)."""
    import test_gpu_edge as E
    from paper_2210_07768_b200.config import ConfigError
    global STR_COLS, INT_COLS, F32_COLS
    saved = (STR_COLS, INT_COLS, F32_COLS)
    STR_COLS, INT_COLS, F32_COLS = ["query", "cx", "city"], ["age", "user_id", "tier"], ["score"]
    try:
        ops, feats = random_dag(1000 + seed)
    finally:
        STR_COLS, INT_COLS, F32_COLS = saved
    feats.pop("basic_b", None)
    feats = {k: (9 if k == "basic_a" else v) for k, v in feats.items()}
    drv, prof, bas = E._views(2500, 50 + seed)
    E._write_views(tmp_path, drv, prof, bas)
    raw = E._config([512, 64, 7][seed % 3], ops, feats, filt="age != -12345")
    raw["tables"] = {}
    for op in ops:  # the adversarial corpus has no dictionaries: lookups become trims
        for p in op.get("pre", []):
            if p["fn"].startswith("lookup:"):
                p["fn"] = "trim"
    try:
        ref, ref_err, got, got_err = E._run_both(raw, drv, prof, bas, tmp_path)
    except ConfigError:
        pytest.skip("generated config rejected")
    if ref_err is not None:
        assert got_err is not None, f"oracle failed ({ref_err}), engine did not"
        assert getattr(got_err, "stage", None) == ref_err.stage, (got_err, ref_err)
        return
    assert got_err is None, got_err
    assert (got.report.digest, got.report.instances, got.report.signs) == \
        (ref.digest, ref.instances, ref.signs)
    np.testing.assert_array_equal(got.csr["signs"], np.array(ref.values, np.uint64))
