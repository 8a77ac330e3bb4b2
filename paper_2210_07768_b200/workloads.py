"""Measurement DAGs of SURVEY.md Appendix B, as reference-schema config dicts.

Each variant replaces ``operators``, ``emit.features`` and ``tables`` of the
generated ``pipeline.json`` (reference ``corpus.py:146-231``); views, the clean
policy, the join and device knobs are kept.  ``lookup_heavy`` needs three
extra dictionary files written beside the corpus (``write_lookup_tables``).
"""

from __future__ import annotations

import copy
import itertools
from pathlib import Path

from .corpus import VOCAB, config_dict, fnv1a64

BASIC_FEATURES = {"basic_a": 40, "basic_b": 41}
BIG = {"footprint_bytes": 1 << 30, "kind": "memory-bound"}


def _op(name, inputs, outputs=None, body=None, pre=(), post=()):
    o = {"name": name, "inputs": list(inputs), "outputs": list(outputs or [name]),
         "body": {"fn": body}}
    if pre:
        o["pre"] = [dict(p) for p in pre]
    if post:
        o["post"] = [dict(p) for p in post]
    return o


def _fig4():
    ops = [
        _op("alpha", ["query"], ["alpha_out"], "hash:1", post=[{"fn": "mix"}]),
        _op("beta", ["query"], ["beta_out"], "hash:2", pre=[{"fn": "lower"}], post=[{"fn": "mix"}]),
        _op("gamma", ["city"], ["gamma_out"], "hash:3",
            pre=[{"fn": "trim", **BIG}], post=[{"fn": "fold"}]),
    ]
    return ops, {"alpha_out": 1, "beta_out": 2, "gamma_out": 3}, {}


def _sign_heavy():
    ops = [_op(f"q_t{i}", ["query"], body=f"hash:{20 + i}", pre=[{"fn": f"token: :{i}"}])
           for i in range(4)]
    ops += [
        _op("q_low", ["query"], body="hash:24", pre=[{"fn": "lower"}]),
        _op("q_full", ["query"], body="hash:25"),
        _op("cx_sig", ["city_x"], body="hash:26"),
        _op("c_sig", ["city"], body="hash:27", pre=[{"fn": "trim"}]),
        _op("age_sig", ["age"], body="hash:28"),
        _op("score_sig", ["score"], body="hash:29"),
        _op("user_sig", ["user_id"], body="hash:30", post=[{"fn": "mix"}]),
    ]
    emit = {f"q_t{i}": 20 + i for i in range(4)}
    emit.update({"q_low": 24, "q_full": 25, "cx_sig": 26, "c_sig": 27, "age_sig": 28,
                 "score_sig": 29, "user_sig": 30})
    return ops, emit, {}


def _cross_heavy():
    t = lambda i, a: {"fn": f"token: :{i}", "arg": a}  # noqa: E731
    ops = [
        _op("x_t0t1", ["query", "query"], body="hash:50", pre=[t(0, 0), t(1, 1)]),
        _op("x_t0c", ["query", "city"], body="hash:51", pre=[t(0, 0)]),
        _op("x_t1cx", ["query", "city_x"], body="hash:52", pre=[t(1, 0)]),
        _op("x_qca", ["query", "city", "age"], body="hash:53"),
        _op("x_t012", ["query", "query", "query"], body="hash:54",
            pre=[t(0, 0), t(1, 1), t(2, 2)]),
        _op("x_cc", ["city", "city_x"], body="concat:|"),
        _op("x_cc_sig", ["x_cc"], body="hash:55", pre=[{"fn": "lower"}]),
        _op("x_su", ["score", "user_id"], ["x_su_mix", "x_su_fold"], "hash:56",
            post=[{"fn": "mix"}, {"fn": "fold"}]),
    ]
    emit = {"x_t0t1": 50, "x_t0c": 51, "x_t1cx": 52, "x_qca": 53, "x_t012": 54,
            "x_cc_sig": 55, "x_su_mix": 56, "x_su_fold": 57}
    return ops, emit, {}


LOOKUP_TABLES = {
    "city_dict": {"path": "city_dict.tsv", "default": 0},
    "user_dict": {"path": "user_dict.tsv", "default": 7},
    "query_dict": {"path": "query_dict.tsv", "default": 0},
    "token_dict": {"path": "token_dict.tsv", "default": 0},
}


def _lookup_heavy():
    lk = lambda t: {"fn": f"lookup:{t}", **BIG}  # noqa: E731
    ops = [
        _op("l_city", ["city"], body="hash:60", pre=[lk("city_dict")]),
        _op("l_cx", ["city_x"], body="hash:61", pre=[lk("city_dict")]),
        _op("l_user", ["user_id"], body="hash:62", pre=[lk("user_dict")]),
        _op("l_query", ["query"], body="hash:63", pre=[lk("query_dict")]),
    ]
    for i in range(4):
        ops.append(_op(f"t{i}", ["query"], [f"tok{i}"], "concat:", pre=[{"fn": f"token: :{i}"}]))
        ops.append(_op(f"l_tok{i}", [f"tok{i}"], body=f"hash:{64 + i}",
                       pre=[lk("token_dict")]))
    emit = {"l_city": 60, "l_cx": 61, "l_user": 62, "l_query": 63}
    emit.update({f"l_tok{i}": 64 + i for i in range(4)})
    return ops, emit, copy.deepcopy(LOOKUP_TABLES)


VARIANTS = {
    "fig4": _fig4,
    "sign_heavy": _sign_heavy,
    "cross_heavy": _cross_heavy,
    "lookup_heavy": _lookup_heavy,
}
DAGS = ("default", "fig4", "sign_heavy", "cross_heavy", "lookup_heavy")


def workload_config(dag: str, batch_size: int = 512, ops_only: bool = False) -> dict:
    """The reference-schema config for one Appendix-B DAG."""
    cfg = config_dict(batch_size, views=2)
    if dag != "default":
        ops, emit, tables = VARIANTS[dag]()
        cfg["operators"] = ops
        cfg["emit"] = {"features": {**emit, **BASIC_FEATURES}}
        cfg["tables"] = tables
    if ops_only:
        cfg["emit"]["features"] = {c: s for c, s in cfg["emit"]["features"].items()
                                   if c not in BASIC_FEATURES}
    return cfg


def lookup_table_entries(users: int, fillers: int = 100_000) -> dict[str, dict[str, int]]:
    """token/user/query dictionaries of Appendix B (``query`` gets ``fillers``)."""
    token = {w: fnv1a64(b"t:" + w.encode()) for w in VOCAB}
    user = {str(u): fnv1a64(b"u:" + str(u).encode()) for u in range(users) if u % 10 != 0}
    query = {}
    for k in range(1, 5):
        for p in itertools.permutations(VOCAB, k):
            q = " ".join(p)
            query[q] = fnv1a64(b"q:" + q.encode())
    for i in range(fillers):
        query[f"f{i}"] = i
    return {"token_dict": token, "user_dict": user, "query_dict": query}


def write_lookup_tables(dest: str | Path, users: int, fillers: int = 100_000) -> None:
    dest = Path(dest)
    for name, entries in lookup_table_entries(users, 0).items():
        with open(dest / f"{name}.tsv", "w", encoding="utf-8") as fh:
            fh.write("".join(f"{k}\t{v}\n" for k, v in entries.items()))
            if name == "query_dict":  # fillers f{i} -> i, streamed (1e7 lines)
                step = 1 << 20
                for lo in range(0, fillers, step):
                    fh.write("".join(f"f{i}\t{i}\n" for i in range(lo, min(lo + step, fillers))))
