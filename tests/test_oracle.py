"""CPU: the oracle is pinned to the reference's known answers and goldens."""

from __future__ import annotations

import json
import struct

import numpy as np
import pytest

import featurebox_oracle as O
from conftest import GOLDEN, corpus, golden_run, reference_available

DAGS = ("default", "fig4", "sign_heavy", "cross_heavy", "lookup_heavy")


def test_fnv_known_answers():
    # reference tests/test_featureops.py:40-43, 65-69, 291
    assert O.fnv1a64(b"") == 0xCBF29CE484222325
    assert O.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert O.fnv1a64(b"hello") == 0xA430D84680AABD0B
    assert O.feature_sign(3, ["q"]) == 0xD942B1186C06365F == O.fnv1a64(b"\x00\x03q")
    assert O.make_fn("mix", {}).call(5) == 0xA8C7F332281A3146


def test_sign_examples_appendix_a():
    assert O.feature_sign(12, [O.fnv1a64(b"tokyo")]) == 0xAF6418975BA922F4
    assert O.feature_sign(12, [0.5]) == 0x5EC2947371569A16
    assert O.feature_sign(12, [5]) == 0x80D70A6929B36BC2
    assert O.feature_sign(12, ["5"]) == 0xD9247D186BECE074


def test_value_bytes_encodings():
    assert O.value_bytes("é") == "é".encode()
    assert O.value_bytes(-1) == b"\xff" * 8
    assert O.value_bytes(1.5) == struct.pack(">f", 1.5)
    with pytest.raises(TypeError):
        O.value_bytes(True)


def test_instance_digest_layout():
    # reference tests/test_pipeline.py:82-91
    msg = (7).to_bytes(8, "little") + b"\x01" + (3).to_bytes(2, "little") + (9).to_bytes(8, "little")
    assert O.instance_digest(7, 1, [(3, 9)]) == O.fnv1a64(msg)


def test_token_and_fold_semantics():
    tok = O.make_fn("token: :9", {}).call
    assert tok("a b") == "" and tok(None) is None
    assert O.make_fn("fold", {}).call(-5) == -4294967292


@pytest.mark.parametrize("dag", DAGS)
def test_oracle_matches_reference_minibatches(dag, goldens):
    c, d = corpus(2000, 300, 7)
    from paper_2210_07768_b200.workloads import workload_config
    cfg = workload_config(dag)
    tables, sizes = O.load_tables(cfg.get("tables", {}), d)
    r = O.run_pipelined(cfg, {"user_events": c.driver, "user_profile": c.profile}, c.basic,
                        tables, sizes)
    g = golden_run(goldens, 2000, 7, dag)
    assert f"0x{r.digest:016x}" == g["digest"]
    assert (r.instances, r.signs, r.batches) == (g["instances"], g["signs"], g["batches"])
    ref = np.load(GOLDEN / f"csr_{dag}.npz")
    np.testing.assert_array_equal(np.array(r.ids, np.uint64), ref["ids"])
    np.testing.assert_array_equal(np.array(r.offsets, np.uint64), ref["offsets"])
    np.testing.assert_array_equal(np.array(r.slots, np.uint16), ref["slots"])
    np.testing.assert_array_equal(np.array(r.values, np.uint64), ref["signs"])


def test_oracle_single_view(goldens):
    c, d = corpus(1200, 200, 11, views=1)
    cfg = json.loads((d / "pipeline.json").read_text())
    r = O.run_pipelined(cfg, {"user_events": c.driver}, c.basic, {}, {})
    g = golden_run(goldens, 1200, 11, "default", views=1)
    assert f"0x{r.digest:016x}" == g["digest"]


JSON_CASES = ['{"u": {"city": "tokyo"}}', '{"u":{"city":"a\\u00e9b"}}', '{"u": {"city": 5}}',
              '{"u": [1]}', "not json{", '{"u": {"city": "x"}, "u": 5}', '{"a":1,}', " [1] ",
              '{"u":{"city":"x"}}x', '{"u":{"city":"\\ud800"}}', '"s"', "NaN", '{"u":{}}',
              '{"u":{"city":"q","city":"r"}}', '{"\\u0075":{"city":"k"}}', "{", "",
              '{"u":{"city":"tab\there"}}', '{"u":{"city":"ok"},"n":-0.5e-3}', '1e400']


@pytest.mark.skipif(not reference_available(), reason="reference not mounted")
@pytest.mark.parametrize("doc", JSON_CASES)
def test_oracle_clean_matches_reference_clean(doc):
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    from featurebox.columnstore import ColumnBatch, Kind as RK
    from featurebox.viewpipe import CleanCounters, CleanPolicy, JsonExtraction, clean_views
    rb = ColumnBatch.from_pydict([("meta", RK.JSON)], {"meta": [doc, None]})
    pol = CleanPolicy(extractions=(JsonExtraction("meta", "u.city", "cx", RK.UTF8),))
    rc = CleanCounters()
    ref = clean_views(rb, pol, rc)
    t = O.Table({"meta": "json"}, [{"meta": doc}, {"meta": None}])
    oc = {}
    mine = O.clean(t, {"extract": [{"source": "meta", "path": "u.city", "output": "cx",
                                    "kind": "utf8"}]}, oc)
    assert [r["cx"] for r in mine.rows] == ref.columns["cx"].to_pylist()
    assert oc.get("malformed", 0) == rc.malformed_rows


@pytest.mark.parametrize("dag", DAGS)
def test_oracle_extract_matches_reference_extract_batch(dag):
    """The oracle's `_extract_batch` restatement vs the reference's outputs."""
    from paper_2210_07768_b200.columns import read_view
    from paper_2210_07768_b200.workloads import workload_config
    c, d = corpus(2000, 300, 7)
    cfg = workload_config(dag)
    tables, sizes = O.load_tables(cfg.get("tables", {}), d)
    plan = O.build_plan(cfg["operators"], tables, cfg["device"]["budget_bytes"], sizes)
    t = O.Table.from_view(read_view(GOLDEN / "joined_2k.fbxc"))
    out = O.extract(plan, t)
    ref = np.load(GOLDEN / f"extract_{dag}.npz")
    for col in [k for k in ref.files if "." not in k]:
        vals = [r[col] for r in out.rows]
        assert [v is None for v in vals] == list(ref[col + ".null"]), col
        if col + ".offsets" in ref.files:
            blob = b"".join(b"" if v is None else v.encode() for v in vals)
            assert blob == ref[col].tobytes(), col
        else:
            assert [0 if v is None else v for v in vals] == list(ref[col]), col
