"""CPU, build container only: the oracle against the UNMODIFIED reference
(/root/reference, imported read-only) on randomly generated operator DAGs, over the
reference corpus and over the adversarial records of test_gpu_edge.  The GPU tests
compare the device with the oracle on the same generators (test_gpu_random_dags.py),
so this pins the device to the reference transitively.  Skipped where the reference
is not mounted (the GPU box)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

import featurebox_oracle as O
from conftest import REFERENCE, corpus, reference_available

pytestmark = pytest.mark.skipif(not reference_available(), reason="reference not mounted")

N = int(os.environ.get("FBX_REFDIFF_DAGS", "16"))


def _ref_modules():
    if str(REFERENCE) not in sys.path:
        sys.path.insert(0, str(REFERENCE))
    import featurebox.pipeline as P
    from featurebox.featureops import FeatureConfigError
    return P, FeatureConfigError


def _reference_call(raw: dict, where, batches=None):
    """run_pipelined(load_config(cfg.json)) of the reference (its emitted
    mini-batches appended to `batches`); raises what the reference raises."""
    P, _ = _ref_modules()
    path = where / f"refdiff_{os.getpid()}.json"
    path.write_text(json.dumps(raw))
    orig = P.TrainingSink.consume
    if batches is not None:
        def consume(self, batch):
            batches.append(batch)
            return orig(self, batch)
        P.TrainingSink.consume = consume
    try:
        return P.run_pipelined(P.load_config(path))
    finally:
        P.TrainingSink.consume = orig
        path.unlink()


def _reference_run(raw: dict, where):
    """(report, None) or (None, failing stage | "config")."""
    P, FeatureConfigError = _ref_modules()
    try:
        return _reference_call(raw, where), None
    except P.StageError as e:
        return None, e.stage
    except (P.ConfigError, FeatureConfigError):
        return None, "config"


def _oracle_run(raw, views, basic, where):
    from paper_2210_07768_b200.config import ConfigError, config_from_dict
    try:
        config_from_dict(raw, where)
        tables, sizes = O.load_tables(raw.get("tables", {}), where)
        return O.run_pipelined(raw, views, basic, tables, sizes), None
    except O.OracleError as e:
        return None, e.stage
    except ConfigError:
        return None, "config"


def _compare(ref, ref_stage, mine, my_stage):
    assert ref_stage == my_stage, (ref_stage, my_stage)
    if ref is not None:
        assert (ref.digest, ref.instances, ref.signs, ref.batches) == \
            (mine.digest, mine.instances, mine.signs, mine.batches)
        assert (ref.rows_dropped, ref.rows_filtered) == (mine.malformed, mine.filtered)


@pytest.mark.parametrize("seed", range(N))
def test_random_dag_oracle_equals_reference(seed):
    from paper_2210_07768_b200.workloads import workload_config
    from test_gpu_random_dags import TABLES, random_dag
    c, d = corpus(3000, 400, 13 + seed % 3)
    raw = workload_config("default", batch_size=[512, 256, 100, 3000][seed % 4])
    raw["operators"], raw["emit"] = random_dag(seed)[0], {"features": random_dag(seed)[1]}
    raw["tables"] = TABLES
    ref, ref_stage = _reference_run(raw, d)
    mine, my_stage = _oracle_run(raw, {"user_events": c.driver, "user_profile": c.profile},
                                 c.basic, d)
    _compare(ref, ref_stage, mine, my_stage)


@pytest.mark.parametrize("seed", range(N // 2))
def test_random_dag_on_adversarial_records_oracle_equals_reference(seed, tmp_path):
    import test_gpu_edge as E
    import test_gpu_random_dags as R
    saved = (R.STR_COLS, R.INT_COLS, R.F32_COLS)
    R.STR_COLS, R.INT_COLS, R.F32_COLS = ["query", "cx", "city"], ["age", "user_id", "tier"], ["score"]
    try:
        ops, feats = R.random_dag(1000 + seed)
    finally:
        R.STR_COLS, R.INT_COLS, R.F32_COLS = saved
    feats.pop("basic_b", None)
    feats = {k: (9 if k == "basic_a" else v) for k, v in feats.items()}
    drv, prof, bas = E._views(2500, 50 + seed)
    E._write_views(tmp_path, drv, prof, bas)
    raw = E._config([512, 64, 7][seed % 3], ops, feats, filt="age != -12345")
    for op in ops:
        for p in op.get("pre", []):
            if p["fn"].startswith("lookup:"):
                p["fn"] = "trim"
    ref, ref_stage = _reference_run(raw, tmp_path)
    mine, my_stage = _oracle_run(raw, {"ev": drv, "pr": prof}, bas, tmp_path)
    _compare(ref, ref_stage, mine, my_stage)


@pytest.mark.parametrize("batch_size,seed", [(512, 1), (64, 2), (7, 3), (1000, 4)])
def test_adversarial_records_oracle_equals_reference(batch_size, seed, tmp_path):
    import test_gpu_edge as E
    drv, prof, bas = E._views(3000, seed)
    E._write_views(tmp_path, drv, prof, bas)
    raw = E._config(batch_size, E.OPS, E.FEATS)
    ref, ref_stage = _reference_run(raw, tmp_path)
    mine, my_stage = _oracle_run(raw, {"ev": drv, "pr": prof}, bas, tmp_path)
    _compare(ref, ref_stage, mine, my_stage)


# ---- the GPU edge tests, with the reference in the engine's seat ------------------------

class _RefRun:
    """The reference's run shaped like engine.run_views(..., collect=True)."""

    def __init__(self, report, batches):
        ids, labels, offs, slots, signs = [], [], [0], [], []
        for b in batches:
            for i in range(len(b)):
                ids.append(b.ids[i])
                labels.append(b.labels[i])
                for sl, sg in b.features[i]:
                    slots.append(sl)
                    signs.append(sg)
                offs.append(len(slots))
        self.report = report
        self.csr = {"ids": np.array(ids, np.uint64), "labels": np.array(labels, np.uint8),
                    "offsets": np.array(offs, np.uint64), "slots": np.array(slots, np.uint16),
                    "signs": np.array(signs, np.uint64)}


def _oracle_vs_reference(raw, drv, prof, bas, tmp):
    """test_gpu_edge._run_both with the unmodified reference instead of the engine."""
    tables, sizes = O.load_tables(raw.get("tables", {}), tmp)
    try:
        ref, ref_err = O.run_pipelined(raw, {"ev": drv, "pr": prof}, bas, tables, sizes), None
    except O.OracleError as e:
        ref, ref_err = None, e
    P, _ = _ref_modules()
    batches = []
    try:
        got, got_err = _RefRun(_reference_call(raw, tmp, batches), batches), None
    except P.StageError as e:
        got, got_err = None, e
    return ref, ref_err, got, got_err


EDGE_TESTS = [  # (test function name, parameter sets)
    ("test_adversarial_records_match_oracle", [{"batch_size": b, "seed": s} for b, s in
                                               [(2048, 5), (5000, 6)]]),
    ("test_json_fuzz_matches_oracle", [{"seed": 21}, {"seed": 22}]),
    ("test_tokens_long_and_ragged_queries_match_oracle", [{}]),
    ("test_json_kind_extraction_matches_oracle", [{"seed": 41}, {"seed": 42}]),
    ("test_filters_match_oracle", "filt"),
    ("test_type_error_mix_of_str", [{}]),
    ("test_lone_surrogate_hash_is_encode_error", [{}]),
    ("test_duplicate_instance_ids", [{}]),
    ("test_bad_labels", "label"),
    ("test_failure_placement_matches_reference", "case,batch_size"),
    ("test_json_float32_leaves_match_oracle", [{}]),
    ("test_json_float32_overflow_is_stage_error", "bad"),
    ("test_float32_str_repr_matches_oracle", [{}]),
    ("test_basic_view_duplicate_id_fails_prepare", [{"dst": -1, "src": 0}, {"dst": 5, "src": 6}]),
    ("test_pool_bytes_matches_reference", [dict(zip(("pool", "lpg", "batch_size", "ops"), c))
                                           for c in __import__("test_gpu_edge").POOL_CASES]),
]


def _edge_cases():
    import test_gpu_edge as E
    out = []
    for name, params in EDGE_TESTS:
        fn = getattr(E, name)
        if isinstance(params, str):  # the test's own parametrize marks
            keys = params.split(",")
            grids = {m.args[0]: m.args[1] for m in fn.pytestmark if m.name == "parametrize"}
            combos = [{}]
            for k in keys:
                combos = [dict(c, **{k: v}) for c in combos for v in grids[k]]
            params = combos
        out += [pytest.param(name, p, id=f"{name[5:]}-{'-'.join(str(v)[:12] for v in p.values())}")
                for p in params]
    return out


@pytest.mark.parametrize("name,params", _edge_cases())
def test_edge_case_oracle_equals_reference(name, params, tmp_path, monkeypatch):
    """Every success / failure assertion of test_gpu_edge evaluated with the oracle
    as the expectation and the reference as the implementation."""
    import test_gpu_edge as E
    import paper_2210_07768_b200.config as C
    P, _ = _ref_modules()
    monkeypatch.setattr(E, "_run_both", _oracle_vs_reference)
    monkeypatch.setattr(C, "StageError", P.StageError)
    getattr(E, name)(tmp_path=tmp_path, **params)
