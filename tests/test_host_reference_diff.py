"""CPU: the host-side drop-in surface against the UNMODIFIED reference (baseline/_ref
or /root/reference, imported read-only; skipped without it): the filter grammar,
the clean-policy and JSON-path validation, the feature-op helpers and the
dictionary-table loader give the same results, exception types and messages."""

from __future__ import annotations

import sys

import pytest

from conftest import reference_package_path

REF = reference_package_path()
pytestmark = pytest.mark.skipif(REF is None, reason="reference package not installed")


def _ref(mod):
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import importlib
    return importlib.import_module(f"featurebox.{mod}")


def _outcome(fn, *a, **kw):
    try:
        return ("ok", repr(fn(*a, **kw)))
    except Exception as exc:  # noqa: BLE001
        return ("err", type(exc).__name__, str(exc))


FILTERS = ["age <= 120", "score > -1.5", "city == 'nyc'", 'city != "sf"',
           "a == 1 or b == 2 and c == 3", "(a == 1 or b == 2) and c == 3", "a == 1 && b == 2",
           "a == 1 || b == 2", "", "age", "age <=", "age <= <=", "<= 120", "age ~ 5",
           "(age <= 120", "age <= 120)", "age <= 120 extra", "age <= 'x' @", "age <= 1e3",
           "x == -0.0", "x == 'it''s'", "x==1", "not x == 1", "x == 1 and",
           "x == 99999999999999999999999", "((a == 1))", "a == 1 or (b == 2 or c == 3)",
           "a == 'é'", "a >= 0.1 and b < 2 or not c == 'z'"]


@pytest.mark.parametrize("text", FILTERS)
def test_filter_grammar(text):
    from paper_2210_07768_b200.config import parse_filter
    assert _outcome(parse_filter, text) == _outcome(_ref("viewpipe").parse_filter, text)


@pytest.mark.parametrize("path", ["a", "u.city", "", "a..b", ".a", "a.", "a b", "é.x"])
def test_json_extraction_paths(path):
    from paper_2210_07768_b200.columns import Kind
    from paper_2210_07768_b200.config import JsonExtraction
    rv = _ref("viewpipe")
    rk = _ref("columnstore").Kind
    got = _outcome(JsonExtraction, "meta", path, "o", Kind.UTF8)
    want = _outcome(rv.JsonExtraction, "meta", path, "o", rk.UTF8)
    assert got[0] == want[0] and got[1:2] == want[1:2] if got[0] == "err" else got[0] == "ok"
    if got[0] == "err":
        assert got[2] == want[2]


def _policies(cfg, kind_mod):
    K = kind_mod
    X = cfg.JsonExtraction
    return [
        cfg.CleanPolicy(fills={"ghost": 1}),
        cfg.CleanPolicy(fills={"age": "old"}),
        cfg.CleanPolicy(fills={"age": True}),
        cfg.CleanPolicy(fills={"query": 3}),
        cfg.CleanPolicy(fills={"age": 2 ** 70}),
        cfg.CleanPolicy(extractions=(X("ghost", "a", "o", K.UTF8),)),
        cfg.CleanPolicy(extractions=(X("query", "a", "o", K.UTF8),)),
        cfg.CleanPolicy(extractions=(X("meta", "a", "age", K.UTF8),)),
        cfg.CleanPolicy(extractions=(X("meta", "a", "age", K.INT64),)),
        cfg.CleanPolicy(fills={"age": 0, "query": ""}),
    ]


def test_clean_policy_validation():
    from paper_2210_07768_b200 import config as C
    from paper_2210_07768_b200.columns import Kind
    rv, rc = _ref("viewpipe"), _ref("columnstore")
    ours = _policies(C, Kind)
    theirs = _policies(rv, rc.Kind)
    kinds = {"age": Kind.INT64, "query": Kind.UTF8, "meta": Kind.JSON}
    schema = rc.ColumnBatch.from_pydict([("age", rc.Kind.INT64), ("query", rc.Kind.UTF8),
                                         ("meta", rc.Kind.JSON)],
                                        {"age": [], "query": [], "meta": []}).schema
    for mine, ref in zip(ours, theirs):
        got = _outcome(C.validate_clean_policy, kinds, mine)
        want = _outcome(rv.validate_clean_policy, schema, ref)
        assert got == want, (mine, got, want)
    X, XR = C.JsonExtraction, rv.JsonExtraction
    dup = (lambda M, K: M.CleanPolicy(extractions=(M.JsonExtraction("meta", "a", "o", K.UTF8),
                                                   M.JsonExtraction("meta", "b", "o", K.UTF8))))
    assert _outcome(dup, C, Kind) == _outcome(dup, rv, rc.Kind)
    del X, XR


@pytest.mark.parametrize("s,d", [("a b  c", " "), ("", " "), ("x", "x"), ("a|b|", "|"),
                                 ("é é", " "), ("abc", "ab"), ("abc", ""), ("a b", "é")])
def test_split_string(s, d):
    from paper_2210_07768_b200.featureops import split_string
    assert _outcome(split_string, s, d) == _outcome(_ref("featureops").split_string, s, d)


@pytest.mark.parametrize("values,slot", [([b"a"], 0), ([b"", b"x"], 65535), ([b"q" * 70], 7),
                                         ([b"a", b"b", b"c"], 300), ([b"a"], 65536), ([], 3),
                                         ([b"a"], -1)])
def test_hash_combine_and_fnv(values, slot):
    from paper_2210_07768_b200.featureops import fnv1a64, hash_combine
    rf = _ref("featureops")
    assert _outcome(hash_combine, values, slot) == _outcome(rf.hash_combine, values, slot)
    for v in values:
        assert fnv1a64(v) == rf.fnv1a64(v)


SPECS = ["lower", "trim", "id", "mix", "fold", "token: :0", "token:,:3", "token::1", "token: ",
         "token: :-1", "token: :x", "hash:0", "hash:65535", "hash:65536", "hash:-1", "hash:x",
         "concat:", "concat:|", "lookup:ghost", "nope", "", "token:ab:1", "hash:07"]


@pytest.mark.parametrize("spec", SPECS)
def test_resolve_function_errors(spec):
    """Spec grammar errors (featureops.py:370-446): same exception type and text;
    accepted specs are accepted by both (the B200 side returns device op codes)."""
    from paper_2210_07768_b200.featureops import resolve_function
    got = _outcome(resolve_function, spec, {})
    want = _outcome(_ref("featureops").resolve_function, spec, {})
    assert got[0] == want[0], (spec, got, want)
    if got[0] == "err":
        assert got[1:] == want[1:], spec


@pytest.mark.parametrize("text", ["a\t1\nb\t2\n", "a\t1\na\t2\n", "a 1\n", "a\tx\n", "\t5\n",
                                  "a\t-1\n", "a\t18446744073709551616\n", "", "# c\na\t1\n",
                                  "a\t1\n\nb\t2\n", "é\t7\n"])
def test_load_dict_table(text, tmp_path):
    from paper_2210_07768_b200.featureops import load_dict_table
    f = tmp_path / "t.tsv"
    f.write_text(text, encoding="utf-8")
    got = _outcome(lambda: dict(load_dict_table(f, 0).entries))
    want = _outcome(lambda: dict(_ref("featureops").load_dict_table(f, 0).entries))
    assert got == want, (text, got, want)


# ---- load_config + prepare on mutated configs: the same ConfigError text ------------

def _mut(path, value):
    def m(raw):
        obj = raw
        for k in path[:-1]:
            obj = obj[k]
        if value is _DEL:
            del obj[path[-1]]
        else:
            obj[path[-1]] = value
    return m


_DEL = object()


def _append_ops(*ops):
    def m(raw):
        raw["operators"].extend(ops)
    return m


MUTATIONS = {
    "unknown_fn": _mut(["operators", 0, "body", "fn"], "warp:9"),
    "dup_outputs": lambda raw: raw["operators"][1].__setitem__("outputs",
                                                              raw["operators"][0]["outputs"]),
    "ghost_feature": lambda raw: raw["emit"]["features"].__setitem__("ghost_col", 40),
    "missing_join_key": _mut(["join", "keys"], ["no_such_key"]),
    "missing_label": _mut(["label_column"], "nope"),
    "ghost_filter": _mut(["views", 0, "clean", "filter"], "ghost > 3"),
    "bad_filter": _mut(["views", 0, "clean", "filter"], "age <"),
    "cycle": _append_ops({"name": "loop_a", "inputs": ["loop_b_out"], "outputs": ["loop_a_out"],
                          "body": {"fn": "hash:60"}},
                         {"name": "loop_b", "inputs": ["loop_a_out"], "outputs": ["loop_b_out"],
                          "body": {"fn": "hash:61"}}),
    "unknown_input": _mut(["operators", 0, "inputs"], ["never_heard_of_it"]),
    "batch_zero": _mut(["batch_size"], 0),
    "mode": _mut(["mode"], "turbo"),
    "slot_range": lambda raw: raw["emit"]["features"].__setitem__("x", 1 << 16),
    "no_views": _mut(["views"], []),
    "ghost_driver": _mut(["driver"], "ghost"),
    "fill_kind": lambda raw: raw["views"][0]["clean"]["fills"].__setitem__("age", "old"),
    "fill_unknown": lambda raw: raw["views"][0]["clean"]["fills"].__setitem__("ghost", 1),
    "no_basic": lambda raw: raw.__delitem__("basic"),
    "table_missing": lambda raw: raw["tables"].__setitem__("t2", {"path": "/nonexistent.tsv"}),
    "arity": _mut(["operators", 0, "body", "fn"], "lower"),
    "pool_bytes": lambda raw: raw.setdefault("device", {}).__setitem__("pool_bytes", 100),
    "queue_depth": _mut(["queue_depth"], 0),
    "workers_zero": _mut(["workers"], 0),
    "budget": lambda raw: raw.setdefault("device", {}).__setitem__("budget_bytes", -1),
    "dup_view": lambda raw: raw["views"].append(dict(raw["views"][0])),
    "no_join": lambda raw: raw.__delitem__("join"),
    "feature_not_int": lambda raw: raw["emit"]["features"].__setitem__("q_sig", "x"),
    "ghost_projection": _mut(["views", 0, "columns"], ["instance_id", "ghost"]),
    "projection_drops_label": _mut(["views", 0, "columns"], ["instance_id", "user_id", "query"]),
    "extract_kind": lambda raw: raw["views"][0]["clean"].__setitem__(
        "extract", [{"source": "meta", "path": "u.city", "output": "cx", "kind": "blob"}]),
    "extract_source": lambda raw: raw["views"][0]["clean"].__setitem__(
        "extract", [{"source": "query", "path": "u.city", "output": "cx", "kind": "utf8"}]),
    "table_default": lambda raw: [t.__setitem__("default", "x") for t in raw["tables"].values()],
    "table_path": lambda raw: [t.__setitem__("path", "/nope/none.tsv") for t in raw["tables"].values()],
    "op_no_body": lambda raw: raw["operators"][0].__delitem__("body"),
    "op_bad_pre": _mut(["operators", 0, "pre"], [{"fn": "hash:3"}]),
    "basic_columns": lambda raw: raw["basic"].__setitem__("columns", ["basic_a"]),
    "label_kind": _mut(["label_column"], "query"),
    "instance_kind": _mut(["instance_column"], "query"),
}


@pytest.mark.parametrize("case", sorted(MUTATIONS))
def test_config_mutations_fail_alike(case, tmp_path):
    import json
    from paper_2210_07768_b200 import engine, load_config
    rc = _ref("corpus")
    rp = _ref("pipeline")
    base = tmp_path / "c"
    paths = rc.gen_corpus(base, rows=200, users=20, seed=7, views=2)
    raw = json.loads(paths["config"].read_text())
    for v in raw["views"]:
        v["path"] = str(base / v["path"])
    raw["basic"]["path"] = str(base / raw["basic"]["path"])
    for t in raw.get("tables", {}).values():
        t["path"] = str(base / t["path"])
    raw["staging_dir"] = str(tmp_path / "staging")
    MUTATIONS[case](raw)
    f = tmp_path / "pipeline.json"
    f.write_text(json.dumps(raw))
    got = _outcome(lambda: engine.prepare(load_config(f), compile_program=False))
    want = _outcome(lambda: rp.prepare(rp.load_config(f)))
    assert got[0] == want[0] == "err", (case, got, want)
    assert got[1:] == want[1:], (case, got, want)


RUN_START = {
    "fusion": lambda raw: raw.setdefault("device", {}).__setitem__("fusion", "sideways"),
    "lanes": lambda raw: raw.setdefault("device", {}).__setitem__("lanes_per_group", 0),
    "work_groups": lambda raw: raw.setdefault("device", {}).__setitem__("work_groups", 0),
    "bandwidth": lambda raw: raw.setdefault("device", {}).__setitem__("bandwidth_bytes_per_s", 0),
    "fine": lambda raw: None,
}


@pytest.mark.parametrize("case", sorted(RUN_START))
def test_run_start_checks_fail_alike(case, tmp_path, monkeypatch):
    """Checks the reference makes when a run starts (its ExecContext): the same
    exception type and text before any data moves."""
    import json
    from paper_2210_07768_b200 import load_config
    from paper_2210_07768_b200.config import run_workers
    monkeypatch.delenv("FEATUREBOX_THREADS", raising=False)
    rc, rp = _ref("corpus"), _ref("pipeline")
    base = tmp_path / "c"
    paths = rc.gen_corpus(base, rows=50, users=5, seed=7, views=2)
    raw = json.loads(paths["config"].read_text())
    RUN_START[case](raw)
    f = base / "pipeline.json"
    f.write_text(json.dumps(raw))
    got = _outcome(lambda: run_workers(load_config(f)) and None)
    want = _outcome(lambda: rp._make_ctx(rp.prepare(rp.load_config(f))) and None)
    assert got == want, (case, got, want)
