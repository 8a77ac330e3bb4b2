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

import pytest

import featurebox_oracle as O
from conftest import REFERENCE, corpus, reference_available

pytestmark = pytest.mark.skipif(not reference_available(), reason="reference not mounted")

N = int(os.environ.get("FBX_REFDIFF_DAGS", "16"))


def _reference_run(raw: dict, where):
    """run_pipelined(load_config(cfg.json)) of the reference; (report, None) or (None, stage)."""
    if str(REFERENCE) not in sys.path:
        sys.path.insert(0, str(REFERENCE))
    from featurebox.pipeline import StageError, load_config, run_pipelined
    from featurebox.featureops import FeatureConfigError
    from featurebox.pipeline import ConfigError as RefConfigError
    path = where / f"refdiff_{os.getpid()}.json"
    path.write_text(json.dumps(raw))
    try:
        cfg = load_config(path)
    except (RefConfigError, FeatureConfigError):
        return None, "config"
    try:
        return run_pipelined(cfg), None
    except StageError as e:
        return None, e.stage
    except (RefConfigError, FeatureConfigError):
        return None, "config"
    finally:
        path.unlink()


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
