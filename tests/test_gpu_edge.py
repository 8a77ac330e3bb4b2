"""GPU: adversarial records and error paths, engine vs the CPU oracle.

Edge cases follow SURVEY.md Appendix A and the reference's tests: JSON grammar
corners, escapes, duplicate keys, fills, exact int/float filters, null join
keys, shared emit slots, tokens past the end, upper-case lower(), tiny and odd
batch sizes -- and the failure modes (TypeError, UnicodeEncodeError, duplicate
ids, null / out-of-range labels) located by stage like the reference.
"""

from __future__ import annotations

import json
import random
import tempfile
from pathlib import Path

import numpy as np
import pytest

import featurebox_oracle as O

pytestmark = pytest.mark.gpu

JSON_DOCS = [
    '{"u": {"city": "tokyo", "tier": 2}, "src": "app"}', '{"u":{"city":"Kyoto"}}',
    '{"u": {"city": "a\\u00e9b"}}', '{"u": {"city": "\\ud83d\\ude00x"}}', '{"u": {"city": 5}}',
    '{"u": [1, 2]}', "not json{", '{"u": {"city": "x"}, "u": 5}', '{"a":1,}', " [1] ",
    '{"u":{"city":"x"}}x', '"s"', "NaN", '{"u":{}}', '{"u":{"city":"q","city":"r"}}',
    '{"\\u0075":{"city":"k"}}', "{", "", '{"u":{"city":"tab\\there"}}',
    '{"u":{"city":"ok"},"n":-0.5e-3}', "1e400", '{"u":{"city":"  padded  "}}',
    '{"u" : {"city" : "SP ACE"} }', '{"u":{"city":"a"},"x":[{"y":[1,{"z":null}]}]}',
    '{"u":{"city":"line\\nbreak"}}', '{"u":{"city":"\\"quoted\\""}}', "[]", "{}",
    '{"u":{"city":"x"},"t":true,"f":false,"n":null,"i":-Infinity}', '{"u":{"city":"é"}}',
    '{"u":{"city":"x"}', '{"u":{"city":"x"}}}', '{"u":{"city":"x"},}', '{"u":{"city":"x"} "v":1}',
    '{"u":{"city":01}}', '{"u":{"city":"\\x"}}', '{"u":{"city":"ctl\x01"}}', '{"u":{"city":"x"}}\n',
]
QUERIES = ["running shoes", "Coffee Beans", "  desk  ", "", "a  b", "x", "mechanical keyboard gravel bike",
           "ÉCOLE café", "tab\tsep", None, "ΟΔΟΣ ΑΣ.Σ", "İstanbul", "ΣΑΣ", "Ω\u0345x", "ŉ ǅ ß ẞ",
           "\U0001F600 SMILE", "ПРИВЕТ мир", "Σ", "A\u00adΣ", "x\u2019Σ y"]
LONG_QUERIES = ["w " * 30, "long query " * 6 + "x", " lead", "trail ", "a  b  c  d  e", "x" * 61,
                " " * 59 + "y", "q" * 60, "é " * 20 + "z"]


def _views(n, seed):
    from paper_2210_07768_b200.columns import Kind, ViewImage
    rng = random.Random(seed)
    ids, labels, users, queries, metas, ages = [], [], [], [], [], []
    for i in range(n):
        ids.append((i * 0x9E3779B97F4A7C15 + 12345) % (1 << 63) * (-1 if i % 7 == 0 else 1))
        labels.append(rng.choice([0, 1]))
        users.append(rng.choice([None] + list(range(40))) if rng.random() < 0.1 else rng.randrange(40))
        queries.append(rng.choice(QUERIES))
        metas.append(rng.choice(JSON_DOCS + [None]))
        ages.append(rng.choice([None, -5, 0, 18, 120, 121, 2**40, -2**62]))
    drv = ViewImage.from_pydict(
        [("instance_id", Kind.INT64), ("label", Kind.INT64), ("user_id", Kind.INT64),
         ("query", Kind.UTF8), ("meta", Kind.JSON), ("age", Kind.INT64)],
        {"instance_id": ids, "label": labels, "user_id": users, "query": queries,
         "meta": metas, "age": ages}, ("user_id",))
    pu, pc, ps = [], [], []
    for u in range(40):
        if u % 9 == 4:
            continue
        pu.append(u)
        pc.append(rng.choice([None, " tokyo", "Osaka ", "kyoto", "é", ""]))
        ps.append(rng.choice([None, 0.5, -0.0, 1e-7, 3.25, float("nan")]))
    prof = ViewImage.from_pydict([("user_id", Kind.INT64), ("city", Kind.UTF8),
                                  ("score", Kind.FLOAT32)],
                                 {"user_id": pu, "city": pc, "score": ps}, ("user_id",))
    bas = ViewImage.from_pydict([("instance_id", Kind.INT64), ("basic_a", Kind.INT64)],
                                {"instance_id": [x for j, x in enumerate(ids) if j % 11],
                                 "basic_a": [rng.choice([None, 7, -7]) for j in range(n) if j % 11]},
                                ("instance_id",))
    return drv, prof, bas


def _config(batch_size, ops, features, filt="age <= 120 and age != -5", tables=None):
    return {
        "driver": "ev", "batch_size": batch_size, "basic": {"path": "basic.fbxc"},
        "views": [{"name": "ev", "path": "ev.fbxc",
                   "clean": {"fills": {"query": ""},
                             "extract": [{"source": "meta", "path": "u.city", "output": "cx",
                                          "kind": "utf8"},
                                         {"source": "meta", "path": "u.tier", "output": "tier",
                                          "kind": "int64"}],
                             "filter": filt}},
                  {"name": "pr", "path": "pr.fbxc", "clean": {"fills": {"city": "unknown"}}}],
        "join": {"keys": ["user_id"]}, "tables": tables or {}, "operators": ops,
        "emit": {"features": features}, "device": {"budget_bytes": 65536}}


def _run_both(raw, drv, prof, bas, tmp: Path):
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.engine import run_views
    cfg = config_from_dict(raw, tmp)
    views = {"ev": drv, "pr": prof}
    tables, sizes = O.load_tables(raw.get("tables", {}), tmp)
    try:
        ref = O.run_pipelined(raw, views, bas, tables, sizes)
        ref_err = None
    except O.OracleError as e:
        ref, ref_err = None, e
    try:
        got = run_views(cfg, views, bas, collect=True, max_rows_per_launch=1 << 20)
        got_err = None
    except Exception as e:  # noqa: BLE001
        got, got_err = None, e
    return ref, ref_err, got, got_err


OPS = [
    {"name": "q_low", "inputs": ["query"], "outputs": ["q_low"], "pre": [{"fn": "lower"}],
     "body": {"fn": "hash:3"}},
    {"name": "q_tr", "inputs": ["query"], "outputs": ["q_tr"], "pre": [{"fn": "trim"}],
     "body": {"fn": "hash:4"}},
    {"name": "q_t5", "inputs": ["query"], "outputs": ["q_t5"], "pre": [{"fn": "token: :5"}],
     "body": {"fn": "hash:5"}},
    {"name": "x", "inputs": ["cx", "city", "score"], "outputs": ["x_m", "x_f"],
     "body": {"fn": "hash:6"}, "post": [{"fn": "mix"}, {"fn": "fold"}]},
    {"name": "cc", "inputs": ["city", "cx", "tier"], "outputs": ["cc"], "body": {"fn": "concat:/"}},
    {"name": "cc_sig", "inputs": ["cc"], "outputs": ["cc_sig"], "pre": [{"fn": "lower"}],
     "body": {"fn": "hash:7"}},
    {"name": "age_s", "inputs": ["age", "user_id"], "outputs": ["age_s"],
     "pre": [{"fn": "fold", "arg": 0}], "body": {"fn": "hash:8"}},
    {"name": "tier_s", "inputs": ["tier"], "outputs": ["tier_s"], "pre": [{"fn": "trim"}],
     "body": {"fn": "hash:9"}},
]
FEATS = {"q_low": 3, "q_tr": 4, "q_t5": 5, "x_m": 6, "x_f": 6, "cc_sig": 7, "age_s": 8,
         "tier_s": 9, "basic_a": 9}


def _write_views(tmp, drv, prof, bas):
    from paper_2210_07768_b200.columns import write_view
    write_view(drv, tmp / "ev.fbxc")
    write_view(prof, tmp / "pr.fbxc")
    write_view(bas, tmp / "basic.fbxc")


@pytest.mark.parametrize("batch_size,seed", [(512, 1), (64, 2), (7, 3), (1000, 4), (2048, 5),
                                             (5000, 6)])
def test_adversarial_records_match_oracle(batch_size, seed, tmp_path):
    drv, prof, bas = _views(3000, seed)
    _write_views(tmp_path, drv, prof, bas)
    raw = _config(batch_size, OPS, FEATS)
    ref, ref_err, got, got_err = _run_both(raw, drv, prof, bas, tmp_path)
    assert ref_err is None, ref_err
    assert got_err is None, got_err
    rep = got.report
    assert (rep.digest, rep.instances, rep.signs) == (ref.digest, ref.instances, ref.signs)
    assert (rep.rows_dropped, rep.rows_filtered) == (ref.malformed, ref.filtered)
    np.testing.assert_array_equal(got.csr["ids"], np.array(ref.ids, np.uint64))
    np.testing.assert_array_equal(got.csr["offsets"], np.array(ref.offsets, np.uint64))
    np.testing.assert_array_equal(got.csr["slots"], np.array(ref.slots, np.uint16))
    np.testing.assert_array_equal(got.csr["signs"], np.array(ref.values, np.uint64))


FUZZ_ALPHABET = ' "{}[]:,\\0123456789.-+eEtrufalsnNIycity\t\n\x01'


def _fuzz_docs(n, seed):
    """Short JSON-ish documents: random edits of the grammar corpus (covers the
    mask-mode reader for <= 60-byte docs and its byte-scanner fallback)."""
    rng = random.Random(seed)
    base = [d for d in JSON_DOCS if "\\ud8" not in d] + [
        '{"u": {"city": "a b", "tier": 1}}', '{"u":{"city":" ","tier":-0}}',
        '{ "u" : { "city" : "k" , "tier" : 12 } }', '{"u": {"tier": 3, "city": "z"}}']
    out = []
    for _ in range(n):
        d = list(rng.choice(base))
        for _ in range(rng.choice([0, 0, 1, 1, 2, 3])):
            op = rng.randrange(3)
            k = rng.randrange(len(d) + 1)
            if op == 0:
                d.insert(k, rng.choice(FUZZ_ALPHABET))
            elif op == 1 and d:
                del d[min(k, len(d) - 1)]
            elif d:
                d[min(k, len(d) - 1)] = rng.choice(FUZZ_ALPHABET)
        out.append("".join(d))
    return out


@pytest.mark.parametrize("seed", [21, 22])
def test_json_fuzz_matches_oracle(seed, tmp_path):
    from paper_2210_07768_b200.columns import ColumnImage, Kind
    drv, prof, bas = _views(4000, seed)
    docs = _fuzz_docs(4000, seed)
    drv.columns["meta"] = ColumnImage.from_values(Kind.JSON, docs)
    _write_views(tmp_path, drv, prof, bas)
    ops = [{"name": "c", "inputs": ["cx", "tier"], "outputs": ["c"], "body": {"fn": "hash:3"}},
           {"name": "d", "inputs": ["cx"], "outputs": ["d"], "body": {"fn": "hash:4"}}]
    raw = _config(256, ops, {"c": 3, "d": 4}, filt="age != -12345")
    ref, ref_err, got, got_err = _run_both(raw, drv, prof, bas, tmp_path)
    assert ref_err is None and got_err is None, (ref_err, got_err)
    assert (got.report.rows_dropped, got.report.rows_filtered) == (ref.malformed, ref.filtered)
    assert (got.report.digest, got.report.instances, got.report.signs) == \
        (ref.digest, ref.instances, ref.signs)
    np.testing.assert_array_equal(got.csr["signs"], np.array(ref.values, np.uint64))


def test_tokens_long_and_ragged_queries_match_oracle(tmp_path):
    """token splits over <= 60-byte queries (mask mode) and longer ones (scan)."""
    from paper_2210_07768_b200.columns import ColumnImage, Kind
    drv, prof, bas = _views(3000, 31)
    rng = random.Random(31)
    qs = [rng.choice(LONG_QUERIES + QUERIES) for _ in range(3000)]
    drv.columns["query"] = ColumnImage.from_values(Kind.UTF8, qs)
    _write_views(tmp_path, drv, prof, bas)
    ops = [{"name": f"t{i}", "inputs": ["query"], "outputs": [f"t{i}"],
            "pre": [{"fn": f"token: :{i}"}], "body": {"fn": f"hash:{10 + i}"}} for i in range(5)]
    ops.append({"name": "t9", "inputs": ["query"], "outputs": ["t9"],
                "pre": [{"fn": "token: :9"}], "body": {"fn": "hash:19"}})
    raw = _config(256, ops, {f"t{i}": 10 + i for i in (0, 1, 2, 3, 4, 9)}, filt="age != -12345")
    ref, ref_err, got, got_err = _run_both(raw, drv, prof, bas, tmp_path)
    assert ref_err is None and got_err is None, (ref_err, got_err)
    assert (got.report.digest, got.report.instances, got.report.signs) == \
        (ref.digest, ref.instances, ref.signs)
    np.testing.assert_array_equal(got.csr["signs"], np.array(ref.values, np.uint64))


@pytest.mark.parametrize("seed", [41, 42])
def test_json_kind_extraction_matches_oracle(seed, tmp_path):
    """Json-kind leaves (json.dumps(sort_keys=True, separators=(",", ":"))): random
    nested values, duplicate keys, escapes, non-ASCII, floats of every magnitude."""
    from paper_2210_07768_b200.columns import ColumnImage, Kind
    from paper_2210_07768_b200.jsoncanon import random_json_docs
    drv, prof, bas = _views(3000, seed)
    vals = random_json_docs(3000, seed)
    rng = random.Random(seed)
    metas = []
    for v in vals:
        r = rng.random()
        metas.append(None if r < 0.03 else ('{"u": {"city": %s, "tier": 1}}' % v if r < 0.9
                                           else '{"u": %s}' % v))
    drv.columns["meta"] = ColumnImage.from_values(Kind.JSON, metas)
    _write_views(tmp_path, drv, prof, bas)
    raw = _config(256, [], {}, filt="age != -12345")
    raw["views"][0]["clean"]["extract"] = [
        {"source": "meta", "path": "u.city", "output": "cx", "kind": "json"},
        {"source": "meta", "path": "u", "output": "uj", "kind": "json"}]
    raw["operators"] = [
        {"name": "c", "inputs": ["cx"], "outputs": ["c"], "body": {"fn": "hash:3"}},
        {"name": "u", "inputs": ["uj"], "outputs": ["u"], "body": {"fn": "hash:4"}},
        {"name": "cl", "inputs": ["cx"], "outputs": ["cl"], "pre": [{"fn": "lower"}],
         "body": {"fn": "hash:5"}}]
    raw["emit"] = {"features": {"c": 3, "u": 4, "cl": 5}}
    ref, ref_err, got, got_err = _run_both(raw, drv, prof, bas, tmp_path)
    assert ref_err is None and got_err is None, (ref_err, got_err)
    assert (got.report.rows_dropped, got.report.rows_filtered) == (ref.malformed, ref.filtered)
    assert (got.report.digest, got.report.instances, got.report.signs) == \
        (ref.digest, ref.instances, ref.signs)
    np.testing.assert_array_equal(got.csr["signs"], np.array(ref.values, np.uint64))


@pytest.mark.parametrize("filt", ["age < 120.5", "age >= -4611686018427387904", "age == 20.0",
                                  "age != 9999999999999999999999", "age > -1.5 or tier == 2",
                                  "(age < 30 or age > 60) and query != ''", "cx >= 'kyoto'",
                                  "tier <= 1 && cx != 'x'"])
def test_filters_match_oracle(filt, tmp_path):
    drv, prof, bas = _views(1500, 9)
    _write_views(tmp_path, drv, prof, bas)
    raw = _config(256, OPS[3:4], {"x_m": 6, "x_f": 7}, filt=filt)
    ref, ref_err, got, got_err = _run_both(raw, drv, prof, bas, tmp_path)
    assert ref_err is None and got_err is None, (ref_err, got_err)
    assert (got.report.digest, got.report.instances) == (ref.digest, ref.instances)
    assert (got.report.rows_dropped, got.report.rows_filtered) == (ref.malformed, ref.filtered)


def _err(kind, tmp_path, mutate):
    drv, prof, bas = _views(2000, 5)
    drv, prof, bas = mutate(drv, prof, bas)
    _write_views(tmp_path, drv, prof, bas)
    raw = kind
    ref, ref_err, got, got_err = _run_both(raw, drv, prof, bas, tmp_path)
    assert ref_err is not None, "oracle did not fail"
    assert got_err is not None, "engine did not fail"
    from paper_2210_07768_b200.config import StageError
    assert isinstance(got_err, StageError), got_err
    assert got_err.stage == ref_err.stage
    assert type(got_err.__cause__).__name__ in (type(ref_err.cause).__name__,
                                                "LayerExecutionError")
    return ref_err, got_err


def _same(*a):
    return a


def test_type_error_mix_of_str(tmp_path):
    ops = [{"name": "m", "inputs": ["query"], "outputs": ["m"], "pre": [{"fn": "mix"}],
            "body": {"fn": "hash:3"}}]
    ref_err, got_err = _err(_config(512, ops, {"m": 3}), tmp_path, _same)
    assert got_err.__cause__.node == ref_err.node == "m.pre1"
    assert isinstance(got_err.__cause__.__cause__, TypeError)
    assert got_err.batch_index == ref_err.chunk


def test_lone_surrogate_hash_is_encode_error(tmp_path):
    from paper_2210_07768_b200.columns import ColumnImage, Kind

    def mut(drv, prof, bas):
        metas = drv.columns["meta"].to_pylist()
        metas[700] = '{"u": {"city": "\\ud800"}}'
        drv.columns["meta"] = ColumnImage.from_values(Kind.JSON, metas)
        return drv, prof, bas
    ops = [{"name": "c", "inputs": ["cx"], "outputs": ["c"], "body": {"fn": "hash:3"}}]
    ref_err, got_err = _err(_config(512, ops, {"c": 3}, filt="age != -12345"), tmp_path, mut)
    assert isinstance(got_err.__cause__.__cause__, UnicodeEncodeError)


def test_duplicate_instance_ids(tmp_path):
    from paper_2210_07768_b200.columns import ColumnImage, Kind

    def mut(drv, prof, bas):
        ids = drv.columns["instance_id"].to_pylist()
        for i in range(1000, 1100):  # many rows share one id: some survive to the merge
            ids[i] = ids[999]
        drv.columns["instance_id"] = ColumnImage.from_values(Kind.INT64, ids)
        return drv, prof, bas
    ops = [{"name": "c", "inputs": ["query"], "outputs": ["c"], "body": {"fn": "hash:3"}}]
    raw = _config(512, ops, {"c": 3}, filt="age != -12345")
    ref_err, got_err = _err(raw, tmp_path, mut)
    assert got_err.stage == "merge"
    assert got_err.batch_index == ref_err.chunk
    assert str(got_err.__cause__) == str(ref_err.cause)  # the first repeat, signed id


@pytest.mark.parametrize("pairs", [[(1500, 1400), (702, 1400)], [(1993, 12), (1200, 1102)],
                                   [(1300, 1030), (1200, 1210)], [(1400, 1399), (1390, 1380)],
                                   [(14, 7)]])
def test_duplicate_id_message_is_first_repeat(pairs, tmp_path):
    """check_unique_ids reports the first row, in row order, whose id occurred
    before -- also when several ids repeat in the failing chunk (negative ids
    print signed)."""
    ops = [{"name": "c", "inputs": ["query"], "outputs": ["c"], "body": {"fn": "hash:3"}}]
    raw = _config(512, ops, {"c": 3}, filt="age != -12345")
    ref_err, got_err = _err(raw, tmp_path, _set_ids(pairs))
    assert (got_err.stage, got_err.batch_index) == (ref_err.stage, ref_err.chunk)
    assert str(got_err.__cause__) == str(ref_err.cause)


@pytest.mark.parametrize("label", [None, 2, -1])
def test_bad_labels(label, tmp_path):
    from paper_2210_07768_b200.columns import ColumnImage, Kind

    def mut(drv, prof, bas):
        labels = drv.columns["label"].to_pylist()
        for i in range(0, 2000, 97):
            labels[i] = label
        drv.columns["label"] = ColumnImage.from_values(Kind.INT64, labels)
        return drv, prof, bas
    ops = [{"name": "c", "inputs": ["query"], "outputs": ["c"], "body": {"fn": "hash:3"}}]
    ref_err, got_err = _err(_config(512, ops, {"c": 3}, filt="age != -12345"), tmp_path, mut)
    assert got_err.batch_index == ref_err.chunk


def _set_ids(pairs):
    """Mutation: ids[dst] = ids[src] for (dst, src) in pairs."""
    from paper_2210_07768_b200.columns import ColumnImage, Kind

    def mut(drv, prof, bas):
        ids = drv.columns["instance_id"].to_pylist()
        for dst, src in pairs:
            ids[dst] = ids[src]
        drv.columns["instance_id"] = ColumnImage.from_values(Kind.INT64, ids)
        return drv, prof, bas
    return mut


def _set_labels(rows, value):
    from paper_2210_07768_b200.columns import ColumnImage, Kind

    def mut(drv, prof, bas):
        labels = drv.columns["label"].to_pylist()
        for i in rows:
            labels[i] = value
        drv.columns["label"] = ColumnImage.from_values(Kind.INT64, labels)
        return drv, prof, bas
    return mut


def _chain(*muts):
    def mut(*views):
        for m in muts:
            views = m(*views)
        return views
    return mut


# Placement of failures that surface after their row:
# a repeated id fails the merge of the chunk of its SECOND occurrence; a bad
# label fails the merge of the chunk that flushes its mini-batch, or the final
# flush (stage "emit", no batch index); a repeat in the same chunk beats a flush.
PLACEMENT = {  # rows chosen among those that reach the merge in _views(2000, 5)
    "dup_far": _set_ids([(1900, 3)]),                        # chunks 0 and 3
    "dup_three": _set_ids([(1500, 1400), (702, 1400)]),      # 2nd occurrence: row 1400
    "dup_two_ids": _set_ids([(1993, 12), (1200, 1102)]),     # min over ids
    "dup_same_chunk": _set_ids([(600, 601)]),
    "label_straddle": _set_labels([505], None),              # batch completes later
    "label_tail": _set_labels([1998], 5),                    # final partial batch
    "label_null_vs_range": _chain(_set_labels([302], 7), _set_labels([505], None)),
    "label_and_dup": _chain(_set_labels([40], None), _set_ids([(1003, 1000)])),
    "labels_two": _chain(_set_labels([1030], 3), _set_labels([1021], None)),
}


@pytest.mark.parametrize("case", sorted(PLACEMENT))
@pytest.mark.parametrize("batch_size", [512, 100, 1500])
def test_failure_placement_matches_reference(case, batch_size, tmp_path):
    ops = [{"name": "c", "inputs": ["query"], "outputs": ["c"], "body": {"fn": "hash:3"}}]
    raw = _config(batch_size, ops, {"c": 3}, filt="age != -12345")
    ref_err, got_err = _err(raw, tmp_path, PLACEMENT[case])
    assert (got_err.stage, got_err.batch_index) == (ref_err.stage, ref_err.chunk)


def test_failure_placement_across_launches(tmp_path):
    """The same placement when the run is split over several launches."""
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.engine import run_views
    drv, prof, bas = _views(2000, 5)
    drv, prof, bas = _chain(_set_labels([1010], None), _set_ids([(1900, 3)]))(drv, prof, bas)
    _write_views(tmp_path, drv, prof, bas)
    ops = [{"name": "c", "inputs": ["query"], "outputs": ["c"], "body": {"fn": "hash:3"}}]
    raw = _config(100, ops, {"c": 3}, filt="age != -12345")
    ref, ref_err, _, _ = _run_both(raw, drv, prof, bas, tmp_path)
    assert ref_err is not None
    for rows in (300, 700):
        with pytest.raises(Exception) as ei:
            run_views(config_from_dict(raw, tmp_path), {"ev": drv, "pr": prof}, bas,
                      max_rows_per_launch=rows)
        assert (ei.value.stage, ei.value.batch_index) == (ref_err.stage, ref_err.chunk)


def _float_views(n, seed, extra=()):
    from paper_2210_07768_b200.columns import Kind, ViewImage
    rng = random.Random(seed)
    nums = []
    for _ in range(n):
        r = rng.random()
        if r < 0.5:
            nd = rng.choice([1, 3, 7, 12, 16, 17, 19])
            d = "".join(rng.choice("0123456789") for _ in range(nd)).lstrip("0") or "0"
            e = rng.choice([0, rng.randint(-45, 38 - nd)])  # stay inside float32 range
            t = f"{d}e{e}" if rng.random() < 0.4 else (d[:1] + "." + d[1:] if nd > 1 else d)
            nums.append(("-" if rng.random() < 0.3 else "") + t)
        elif r < 0.7:
            nums.append(str(rng.choice([0, 1, -1, 7, 2**53 + 1, 10**20, -(2**70), 16777217])))
        else:
            nums.append(rng.choice(["NaN", "Infinity", "-Infinity", "true", "null", '"1.5"',
                                    "-0", "-0.0", "0.1", "3.4028235e38", "1e-46", "1.17549435e-38"]))
    nums += list(extra)
    docs = ['{"u": {"f": %s, "city": "x"}}' % x for x in nums]
    m = len(docs)
    drv = ViewImage.from_pydict(
        [("instance_id", Kind.INT64), ("label", Kind.INT64), ("user_id", Kind.INT64),
         ("query", Kind.UTF8), ("meta", Kind.JSON), ("age", Kind.INT64)],
        {"instance_id": list(range(1, m + 1)), "label": [0] * m, "user_id": [1] * m,
         "query": ["q"] * m, "meta": docs, "age": [30] * m}, ("user_id",))
    prof = ViewImage.from_pydict([("user_id", Kind.INT64), ("city", Kind.UTF8),
                                  ("score", Kind.FLOAT32)],
                                 {"user_id": [1], "city": ["c"], "score": [0.5]}, ("user_id",))
    bas = ViewImage.from_pydict([("instance_id", Kind.INT64), ("basic_a", Kind.INT64)],
                                {"instance_id": list(range(1, m + 1)), "basic_a": [1] * m},
                                ("instance_id",))
    return drv, prof, bas


def _float_config():
    raw = _config(512, [{"name": "fs", "inputs": ["fx"], "outputs": ["fs"],
                         "body": {"fn": "hash:5"}}], {"fs": 5}, filt="age == 30")
    raw["views"][0]["clean"]["extract"].append(
        {"source": "meta", "path": "u.f", "output": "fx", "kind": "float32"})
    return raw


def test_json_float32_leaves_match_oracle(tmp_path):
    """Correctly rounded decimal -> double -> float32 (canon_f32(float(v)))."""
    drv, prof, bas = _float_views(4000, 21)
    _write_views(tmp_path, drv, prof, bas)
    ref, ref_err, got, got_err = _run_both(_float_config(), drv, prof, bas, tmp_path)
    assert ref_err is None and got_err is None, (ref_err, got_err)
    assert (got.report.digest, got.report.signs) == (ref.digest, ref.signs)
    np.testing.assert_array_equal(got.csr["signs"], np.array(ref.values, np.uint64))


@pytest.mark.parametrize("bad", ["3.5e38", "1e40", str(10**400)])
def test_json_float32_overflow_is_stage_error(bad, tmp_path):
    drv, prof, bas = _float_views(100, 22, extra=[bad])
    _write_views(tmp_path, drv, prof, bas)
    ref, ref_err, got, got_err = _run_both(_float_config(), drv, prof, bas, tmp_path)
    assert ref_err is not None and got_err is not None
    assert type(ref_err.cause).__name__ == "OverflowError"
    assert got_err.stage == ref_err.stage == "clean"
    assert isinstance(got_err.__cause__, OverflowError)


def test_float32_str_repr_matches_oracle(tmp_path):
    """str() of Float32 values (Python repr of the widened double) feeding
    lower / trim / token / concat / lookup -- JSON leaves and a side-view column."""
    import struct
    rng = random.Random(31)
    extra = []
    for _ in range(3000):  # random float32 bit patterns, written as their repr
        x = struct.unpack("<f", struct.pack("<I", rng.getrandbits(32)))[0]
        if x == x and abs(x) != float("inf"):
            extra.append(repr(x))
    extra += ["1e16", "1e15", "0.0001", "0.00001", "123456789", "16777216", "1.5e-7",
              "1e-45", "3.4028234663852886e+38", "-0.0", "0.1", "100"]
    drv, prof, bas = _float_views(3000, 23, extra=extra)
    keys = [repr(struct.unpack("<f", struct.pack("<f", float(x)))[0]) for x in extra[::7]]
    (tmp_path / "fdict.tsv").write_text("".join(f"{k}\t{i + 1}\n" for i, k in enumerate(keys)))
    ops = [
        {"name": "fl", "inputs": ["fx"], "outputs": ["fl"], "pre": [{"fn": "lower"}],
         "body": {"fn": "hash:3"}},
        {"name": "ft", "inputs": ["fx"], "outputs": ["ft"], "pre": [{"fn": "trim"}],
         "body": {"fn": "hash:4"}},
        {"name": "fk", "inputs": ["fx"], "outputs": ["fk"], "pre": [{"fn": "token:.:1"}],
         "body": {"fn": "hash:5"}},
        {"name": "fc", "inputs": ["fx", "score", "cx"], "outputs": ["fc"],
         "body": {"fn": "concat:|"}},
        {"name": "fch", "inputs": ["fc"], "outputs": ["fch"], "body": {"fn": "hash:6"}},
        {"name": "fd", "inputs": ["fx"], "outputs": ["fd"], "pre": [{"fn": "lookup:fdict"}],
         "body": {"fn": "hash:7"}},
    ]
    raw = _config(512, ops, {"fl": 3, "ft": 4, "fk": 5, "fch": 6, "fd": 7}, filt="age == 30",
                  tables={"fdict": {"path": "fdict.tsv", "default": 0}})
    raw["views"][0]["clean"]["extract"].append(
        {"source": "meta", "path": "u.f", "output": "fx", "kind": "float32"})
    _write_views(tmp_path, drv, prof, bas)
    ref, ref_err, got, got_err = _run_both(raw, drv, prof, bas, tmp_path)
    assert ref_err is None and got_err is None, (ref_err, got_err)
    assert (got.report.digest, got.report.signs) == (ref.digest, ref.signs)
    np.testing.assert_array_equal(got.csr["slots"], np.array(ref.slots, np.uint16))
    np.testing.assert_array_equal(got.csr["signs"], np.array(ref.values, np.uint64))


def test_engine_reused_after_a_duplicate_id_run(tmp_path):
    """A run that fails on a repeated instance id leaves its later-occurrence pairs
    dirty; the next run on the same engine clears them on the device
    (fbx_idset_clear reads the previous run's dup flag) and is exact."""
    from paper_2210_07768_b200 import engine as E
    from paper_2210_07768_b200.columns import ColumnImage, Kind
    from paper_2210_07768_b200.config import StageError, config_from_dict
    drv, prof, bas = _views(2000, 5)
    ids = drv.columns["instance_id"].to_pylist()
    bad_ids = list(ids)
    for i in range(1000, 1100):
        bad_ids[i] = bad_ids[999]
    ops = [{"name": "c", "inputs": ["query"], "outputs": ["c"], "body": {"fn": "hash:3"}}]
    raw = _config(512, ops, {"c": 3}, filt="age != -12345")
    _write_views(tmp_path, drv, prof, bas)
    cfg = config_from_dict(raw, tmp_path)
    views = {"ev": drv, "pr": prof}
    eng = E.Engine(E.prepare(cfg, views, bas), views, bas)
    bad = drv.project(list(drv.order))
    bad.columns["instance_id"] = ColumnImage.from_values(Kind.INT64, bad_ids)
    for view, expect_fail in ((bad, True), (drv, False), (bad, True), (drv, False)):
        eng.bind_driver(E.DeviceView(view))
        eng.reserve(view.row_count)
        eng.begin_run(view.row_count)
        eng.launch(0, view.row_count, tile_base=0)
        if expect_fail:
            with pytest.raises(StageError):
                eng.finish()
        else:
            got = eng.finish().counters
            tables, sizes = O.load_tables(raw.get("tables", {}), tmp_path)
            ref = O.run_pipelined(raw, views, bas, tables, sizes)
            assert (got.digest, got.instances, got.signs) == (ref.digest, ref.instances,
                                                              ref.signs)


POOL_OPS = [
    {"name": "t0", "inputs": ["query"], "outputs": ["t0"], "pre": [{"fn": "token: :0"}],
     "body": {"fn": "hash:3"}},
    {"name": "t1", "inputs": ["query"], "outputs": ["t1"], "pre": [{"fn": "token: :1"}],
     "body": {"fn": "hash:4"}},
    {"name": "tx", "inputs": ["cx"], "outputs": ["tx"], "pre": [{"fn": "token:u:0"}],
     "body": {"fn": "hash:5"}},
    {"name": "th", "inputs": ["city"], "outputs": ["th"],   # host-placed: no arena
     "pre": [{"fn": "token:a:1", "footprint_bytes": 1 << 30}], "body": {"fn": "hash:6"}},
    {"name": "cc", "inputs": ["city", "query"], "outputs": ["cc"], "body": {"fn": "concat:+"}},
    {"name": "tc", "inputs": ["cc"], "outputs": ["tc"], "pre": [{"fn": "token:+:1"}],
     "body": {"fn": "hash:7"}},
    {"name": "ta", "inputs": ["age"], "outputs": ["ta"], "pre": [{"fn": "token:1:0"}],
     "body": {"fn": "hash:8"}},
]
POOL_FEATS = {"t0": 3, "t1": 4, "tx": 5, "th": 6, "tc": 7, "ta": 8}


POOL_CASES = [(128, 256, 512, "all"), (1024, 7, 64, "all"), (4096, 256, 512, "all"),
              (4096, 100, 1500, "all"), (3200, 7, 64, "all"), (8960, 1, 40, "all"),
              (4096, 7, 64, "all"), (8 << 20, 256, 512, "all"), (8 << 20, 100, 1500, "all"),
              (1024, 256, 512, "layer2"), (2048, 3, 100, "layer2")]


@pytest.mark.parametrize("pool,lpg,batch_size,ops", POOL_CASES)
def test_pool_bytes_matches_reference(pool, lpg, batch_size, ops, tmp_path):
    """config device.pool_bytes / lanes_per_group: the reference ArenaPool's
    PoolExhausted (mempool.py:114-134) -- same chunk, layer, node, requested and
    remaining bytes -- or the same run when nothing exhausts."""
    drv, prof, bas = _views(2000, 9)
    _write_views(tmp_path, drv, prof, bas)
    dag = POOL_OPS if ops == "all" else [o for o in POOL_OPS if o["name"] in ("cc", "tc")]
    feats = {k: v for k, v in POOL_FEATS.items() if any(o["name"] == k for o in dag)}
    raw = _config(batch_size, dag, feats, filt="age != -12345")
    raw["device"] = {"budget_bytes": 65536, "pool_bytes": pool, "lanes_per_group": lpg}
    ref, ref_err, got, got_err = _run_both(raw, drv, prof, bas, tmp_path)
    if ref_err is None:
        assert got_err is None, got_err
        assert (got.report.digest, got.report.instances, got.report.signs) == \
            (ref.digest, ref.instances, ref.signs)
        return
    assert got_err is not None, "engine did not fail"
    assert (got_err.stage, got_err.batch_index) == (ref_err.stage, ref_err.chunk)
    lay = got_err.__cause__
    assert (lay.layer_index, lay.node) == (ref_err.layer, ref_err.node)
    cause, want = lay.__cause__, ref_err.cause
    assert type(cause).__name__ == type(want).__name__
    if type(want).__name__ == "PoolExhausted":
        assert (cause.requested, cause.remaining) == (want.requested, want.remaining)


def _basic_dup(dst, src):
    from paper_2210_07768_b200.columns import ColumnImage, Kind

    def mut(drv, prof, bas):
        ids = bas.columns["instance_id"].to_pylist()
        ids[dst] = ids[src]
        bas.columns["instance_id"] = ColumnImage.from_values(Kind.INT64, ids)
        return drv, prof, bas
    return mut


@pytest.mark.parametrize("dst,src", [(-1, 0), (5, 6)])
def test_basic_view_duplicate_id_fails_prepare(dst, src, tmp_path):
    """check_unique_ids over the basic view (pipeline.py:975-980): raised by the
    device index build itself -- stage prepare, no batch index."""
    ops = [{"name": "c", "inputs": ["query"], "outputs": ["c"], "body": {"fn": "hash:3"}}]
    raw = _config(512, ops, {"c": 3}, filt="age != -12345")
    ref_err, got_err = _err(raw, tmp_path, _basic_dup(dst, src))
    assert (got_err.stage, got_err.batch_index) == ("prepare", None) == (ref_err.stage,
                                                                         ref_err.chunk)
    assert "basic features" in str(got_err.__cause__)
    assert str(got_err.__cause__) == str(ref_err.cause)


@pytest.mark.parametrize("pairs", [[(1500, 3), (700, 600)], [(700, 600), (1500, 3)],
                                   [(9, 8), (10, 8), (4, 1800)]])
@pytest.mark.parametrize("streamed", [False, True])
def test_basic_view_names_the_first_repeat(pairs, streamed, tmp_path):
    """Several ids repeat in the basic view: the message names the id of the first
    row, in row order, whose id occurred before (viewpipe.py:562-576) -- found by a
    device sort of the id column, whatever order the index build saw them in."""
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.engine import run_pipelined
    ops = [{"name": "c", "inputs": ["query"], "outputs": ["c"], "body": {"fn": "hash:3"}}]
    raw = _config(512, ops, {"c": 3}, filt="age != -12345")
    drv, prof, bas = _views(2000, 5)
    for dst, src in pairs:
        drv, prof, bas = _basic_dup(dst, src)(drv, prof, bas)
    _write_views(tmp_path, drv, prof, bas)
    tables, sizes = O.load_tables({}, tmp_path)
    with pytest.raises(O.OracleError) as ref:
        O.run_pipelined(raw, {"ev": drv, "pr": prof}, bas, tables, sizes)
    cfg = config_from_dict(raw, tmp_path)
    with pytest.raises(Exception) as got:
        if streamed:
            run_pipelined(cfg)
        else:
            run_pipelined(cfg, collect=True)
    assert (got.value.stage, got.value.batch_index) == ("prepare", None)
    assert str(got.value.__cause__) == str(ref.value.cause)


def test_long_strings_grow_the_device_arena(tmp_path):
    """Strings far above the arena's 96 B/row estimate (concat of ~300-byte
    queries, materialised non-ASCII lower, escaped JSON strings): the launch
    overflows the engine's own bump pool, the engine grows it and repeats the
    run -- same result as the oracle, no failure (no fixed per-row cap)."""
    from paper_2210_07768_b200.columns import ColumnImage, Kind
    rng = random.Random(77)
    drv, prof, bas = _views(20000, 8)
    words = ["Ärger", "straße", "ΣΟΦΙΑ", "Mechanical", "keyboard", "İstanbul", "x" * 40]
    qs = [" ".join(rng.choice(words) for _ in range(rng.randrange(20, 40))) for _ in range(20000)]
    drv.columns["query"] = ColumnImage.from_values(Kind.UTF8, qs)
    metas = [json.dumps({"u": {"city": "\u00c9" * rng.randrange(30, 60) + "Q" * 50}})
             for _ in range(20000)]
    drv.columns["meta"] = ColumnImage.from_values(Kind.JSON, metas)
    _write_views(tmp_path, drv, prof, bas)
    ops = [{"name": "cc", "inputs": ["query", "cx"], "outputs": ["cc"], "body": {"fn": "concat:|"}},
           {"name": "cl", "inputs": ["cc"], "outputs": ["cl"], "pre": [{"fn": "lower"}],
            "body": {"fn": "hash:3"}},
           {"name": "t7", "inputs": ["query"], "outputs": ["t7"], "pre": [{"fn": "token: :7"}],
            "body": {"fn": "hash:4"}}]
    raw = _config(512, ops, {"cl": 3, "t7": 4}, filt="age != -12345")
    ref, ref_err, got, got_err = _run_both(raw, drv, prof, bas, tmp_path)
    assert ref_err is None and got_err is None, (ref_err, got_err)
    assert (got.report.digest, got.report.instances, got.report.signs) == \
        (ref.digest, ref.instances, ref.signs)
