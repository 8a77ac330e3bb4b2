"""Seeded synthetic ads-log corpus (measurement input, not the product path).

Restates the reference generator ``corpus.py:52-272`` so that the same
``(rows, users, seed)`` yields byte-identical FBXC views: every draw is made
from one ``random.Random(seed)`` (MT19937, CPython's algorithms) in the
reference's order -- driver rows (``_driver_batch`` :52-108), then the profile
side view (:111-123), then basic payloads (:126-143).  The column images are
built directly (``ViewImage``), so nothing round-trips through files unless
``write`` is asked for.  ``make_corpus_fast`` (C, ``csrc/corpus_gen.c``) is the
bulk path used by the benchmark and is checked against this one in tests.
"""

from __future__ import annotations

import json
import random
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .columns import ColumnImage, Kind, ViewImage, write_view, wrap_u64

GOLDEN = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1

CITIES = ("tokyo", "osaka", "kyoto", "sapporo", "nagoya", "fukuoka", "sendai",
          "hiroshima", "kobe", "yokohama", "unknown")
VOCAB = ("shoes", "running", "coffee", "beans", "noise", "cancelling",
         "headphones", "mechanical", "keyboard", "standing", "desk",
         "espresso", "grinder", "trail", "gravel", "bike")
BROKEN_JSON = ('{"u": {"city": "par', '{"u": [', "not json{", "{,}")
SOURCES = ("app", "web")

DRIVER_SPEC = (("instance_id", Kind.INT64), ("label", Kind.INT64),
               ("user_id", Kind.INT64), ("query", Kind.UTF8),
               ("meta", Kind.JSON), ("age", Kind.INT64))
PROFILE_SPEC = (("user_id", Kind.INT64), ("city", Kind.UTF8), ("score", Kind.FLOAT32))
BASIC_SPEC = (("instance_id", Kind.INT64), ("basic_a", Kind.INT64),
              ("basic_b", Kind.INT64), ("payload", Kind.FLOAT32))


def fnv1a64(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & MASK64
    return h


def instance_id_of(i: int) -> int:
    """u64 id of driver row i (``corpus.py:43-45``): a bijection on u64."""
    return (GOLDEN * (i + 1)) & MASK64


def basic_sign(instance_id: int, tag: bytes) -> int:
    return fnv1a64(instance_id.to_bytes(8, "little") + tag)


def _draw_driver(rows: int, users: int, rng: random.Random) -> dict[str, list]:
    cols: dict[str, list] = {n: [] for n, _ in DRIVER_SPEC}
    rnd, below, pick = rng.random, rng.randrange, rng.choice
    for i in range(rows):
        cols["instance_id"].append(wrap_u64(instance_id_of(i)))
        cols["label"].append(int(rnd() < 0.3))
        cols["user_id"].append(below(users))
        if rnd() < 0.05:
            cols["query"].append(None)
        else:
            cols["query"].append(" ".join(rng.sample(VOCAB, rng.randint(1, 4))))
        r = rnd()
        if r < 0.02:
            meta = pick(BROKEN_JSON)
        elif r < 0.05:
            meta = None
        elif r < 0.15:
            meta = json.dumps({"src": pick(SOURCES)})
        else:
            inner = {"city": pick(CITIES), "tier": rng.randint(0, 3)}
            meta = json.dumps({"u": inner, "src": pick(SOURCES)})
        cols["meta"].append(meta)
        r = rnd()
        cols["age"].append(None if r < 0.10 else
                           rng.randint(121, 190) if r < 0.15 else rng.randint(18, 90))
    return cols


def _draw_profile(users: int, rng: random.Random) -> dict[str, list]:
    cols: dict[str, list] = {n: [] for n, _ in PROFILE_SPEC}
    for u in range(users):
        if rng.random() < 0.03:
            continue
        cols["user_id"].append(u)
        cols["city"].append(None if rng.random() < 0.04 else rng.choice(CITIES))
        cols["score"].append(None if rng.random() < 0.10 else rng.uniform(0.0, 1.0))
    return cols


def _draw_basic(rows: int, rng: random.Random) -> dict[str, list]:
    ids = [instance_id_of(i) for i in range(rows)]
    return {
        "instance_id": [wrap_u64(v) for v in ids],
        "basic_a": [wrap_u64(basic_sign(v, b"a")) for v in ids],
        "basic_b": [wrap_u64(basic_sign(v, b"b")) for v in ids],
        "payload": [rng.uniform(-1.0, 1.0) for _ in range(rows)],
    }


@dataclass
class Corpus:
    """The generated views and tables, in memory."""

    driver: ViewImage
    profile: ViewImage | None
    basic: ViewImage
    city_dict: dict[str, int] | None
    rows: int
    users: int
    seed: int


def make_corpus(rows: int = 20_000, users: int = 2_000, seed: int = 7,
                views: int = 2) -> Corpus:
    """Build the corpus column images (same draws as ``gen_corpus``)."""
    if rows < 0 or users < 1:
        raise ValueError("rows must be >= 0 and users >= 1")
    if views not in (1, 2):
        raise ValueError("views must be 1 or 2")
    rng = random.Random(seed)
    driver = ViewImage.from_pydict(DRIVER_SPEC, _draw_driver(rows, users, rng), ("user_id",))
    profile = None
    if views == 2:
        profile = ViewImage.from_pydict(PROFILE_SPEC, _draw_profile(users, rng), ("user_id",))
    basic = ViewImage.from_pydict(BASIC_SPEC, _draw_basic(rows, rng), ("instance_id",))
    city = {c: fnv1a64(c.encode()) for c in CITIES} if views == 2 else None
    return Corpus(driver, profile, basic, city, rows, users, seed)


def make_corpus_fast(rows: int = 20_000, users: int = 2_000, seed: int = 7,
                     views: int = 2) -> Corpus:
    """``make_corpus`` through the C generator (csrc/corpus_gen.c): the same
    bytes, ~100x faster -- used for the 1M..100M-record benchmark logs."""
    import ctypes

    from .build import build_corpus_gen
    if rows < 0 or users < 1 or views not in (1, 2):
        raise ValueError("bad corpus parameters")
    lib = ctypes.CDLL(str(build_corpus_gen()))

    class Out(ctypes.Structure):
        _fields_ = [(n, ctypes.c_void_p) for n in (
            "id", "label", "user", "age", "id_n", "label_n", "user_n", "query_n", "meta_n",
            "age_n", "query_off", "meta_off", "query", "meta", "p_user", "p_user_n",
            "p_city_n", "p_score_n", "p_city_off", "p_city", "p_score", "b_id", "b_a", "b_b",
            "b_id_n", "b_a_n", "b_b_n", "b_pay_n", "b_pay")] + [("profile_rows", ctypes.c_uint64)]

    nb = (rows + 7) // 8
    ub = (users + 7) // 8
    arr = {
        "id": np.zeros(rows, np.int64), "label": np.zeros(rows, np.int64),
        "user": np.zeros(rows, np.int64), "age": np.zeros(rows, np.int64),
        "query_off": np.zeros(rows + 1, np.uint32), "meta_off": np.zeros(rows + 1, np.uint32),
        "query": np.zeros(rows * 48 + 64, np.uint8), "meta": np.zeros(rows * 64 + 64, np.uint8),
        "p_user": np.zeros(users, np.int64), "p_city_off": np.zeros(users + 1, np.uint32),
        "p_city": np.zeros(users * 16 + 16, np.uint8), "p_score": np.zeros(users, np.float32),
        "b_id": np.zeros(rows, np.int64), "b_a": np.zeros(rows, np.int64),
        "b_b": np.zeros(rows, np.int64), "b_pay": np.zeros(rows, np.float32)}
    for k in ("id_n", "label_n", "user_n", "query_n", "meta_n", "age_n", "b_id_n", "b_a_n",
              "b_b_n", "b_pay_n"):
        arr[k] = np.zeros(nb, np.uint8)
    for k in ("p_user_n", "p_city_n", "p_score_n"):
        arr[k] = np.zeros(ub, np.uint8)
    out = Out(**{k: a.ctypes.data for k, a in arr.items()})
    lib.fbxgen_corpus(ctypes.c_uint64(rows), ctypes.c_uint64(users), ctypes.c_uint64(seed),
                      ctypes.c_int(views), ctypes.byref(out))
    a = arr
    C = ColumnImage
    driver = ViewImage({
        "instance_id": C(Kind.INT64, rows, a["id_n"], a["id"]),
        "label": C(Kind.INT64, rows, a["label_n"], a["label"]),
        "user_id": C(Kind.INT64, rows, a["user_n"], a["user"]),
        "query": C(Kind.UTF8, rows, a["query_n"], a["query"][: a["query_off"][-1]],
                   a["query_off"]),
        "meta": C(Kind.JSON, rows, a["meta_n"], a["meta"][: a["meta_off"][-1]], a["meta_off"]),
        "age": C(Kind.INT64, rows, a["age_n"], a["age"])},
        ("user_id",), tuple(n for n, _ in DRIVER_SPEC))
    profile = None
    if views == 2:
        np_ = int(out.profile_rows)
        pb = (np_ + 7) // 8
        off = a["p_city_off"][: np_ + 1]
        profile = ViewImage({
            "user_id": C(Kind.INT64, np_, a["p_user_n"][:pb].copy(), a["p_user"][:np_]),
            "city": C(Kind.UTF8, np_, a["p_city_n"][:pb].copy(), a["p_city"][: off[-1]], off),
            "score": C(Kind.FLOAT32, np_, a["p_score_n"][:pb].copy(), a["p_score"][:np_])},
            ("user_id",), tuple(n for n, _ in PROFILE_SPEC))
    basic = ViewImage({
        "instance_id": C(Kind.INT64, rows, a["b_id_n"], a["b_id"]),
        "basic_a": C(Kind.INT64, rows, a["b_a_n"], a["b_a"]),
        "basic_b": C(Kind.INT64, rows, a["b_b_n"], a["b_b"]),
        "payload": C(Kind.FLOAT32, rows, a["b_pay_n"], a["b_pay"])},
        ("instance_id",), tuple(n for n, _ in BASIC_SPEC))
    city = {c: fnv1a64(c.encode()) for c in CITIES} if views == 2 else None
    return Corpus(driver, profile, basic, city, rows, users, seed)


def config_dict(batch_size: int = 512, views: int = 2) -> dict:
    """``pipeline.json`` of the generated corpus (``corpus.py:146-231``)."""
    events = {
        "name": "user_events",
        "path": "user_events.fbxc",
        "clean": {
            "fills": {"age": 0, "query": ""},
            "extract": [{"source": "meta", "path": "u.city", "output": "city_x",
                         "kind": "utf8"}],
            "filter": "age <= 120",
        },
    }
    q_sig = {"name": "q_sig", "inputs": ["query"], "outputs": ["q_sig"],
             "pre": [{"fn": "token: :0"}], "body": {"fn": "hash:11"}}
    cross = {"name": "cross_sig", "inputs": ["query", "city_x"],
             "outputs": ["cross_sig", "cross_fold"], "body": {"fn": "hash:13"},
             "post": [{"fn": "mix"}, {"fn": "fold"}]}
    features = {"q_sig": 11, "cross_sig": 13, "cross_fold": 15, "basic_a": 40, "basic_b": 41}
    cfg = {
        "driver": "user_events",
        "views": [events],
        "basic": {"path": "basic.fbxc"},
        "tables": {},
        "operators": [q_sig, cross],
        "emit": {"features": features},
        "batch_size": batch_size,
        "staging_dir": "staging",
        "device": {"budget_bytes": 64 << 10, "pool_bytes": 8 << 20},
    }
    if views == 2:
        cfg["views"].append({"name": "user_profile", "path": "user_profile.fbxc",
                             "clean": {"fills": {"city": "unknown"}}})
        cfg["join"] = {"keys": ["user_id"]}
        cfg["tables"] = {"city_dict": {"path": "city_dict.tsv", "default": 0}}
        cfg["operators"].insert(1, {
            "name": "city_sig", "inputs": ["city"], "outputs": ["city_sig"],
            "pre": [{"fn": "lookup:city_dict", "footprint_bytes": 1 << 20,
                     "kind": "memory-bound"}],
            "body": {"fn": "hash:12"}})
        features["city_sig"] = 12
    return cfg


def write_corpus(corpus: Corpus, dest: str | Path, batch_size: int = 512) -> dict[str, Path]:
    """Write the corpus as the reference's file set (views, dict, config)."""
    dest = Path(dest)
    dest.mkdir(parents=True, exist_ok=True)
    paths = {"user_events": write_view(corpus.driver, dest / "user_events.fbxc")}
    if corpus.profile is not None:
        paths["user_profile"] = write_view(corpus.profile, dest / "user_profile.fbxc")
    paths["basic"] = write_view(corpus.basic, dest / "basic.fbxc")
    views = 2 if corpus.profile is not None else 1
    if corpus.city_dict is not None:
        paths["city_dict"] = dest / "city_dict.tsv"
        paths["city_dict"].write_text(
            "".join(f"{k}\t{v}\n" for k, v in corpus.city_dict.items()), encoding="utf-8")
    paths["config"] = dest / "pipeline.json"
    paths["config"].write_text(json.dumps(config_dict(batch_size, views), indent=2) + "\n",
                               encoding="utf-8")
    return paths


def gen_corpus(dest: str | Path, rows: int = 20_000, users: int = 2_000, seed: int = 7,
               batch_size: int = 512, views: int = 2) -> dict[str, Path]:
    """Same signature and files as the reference ``gen_corpus`` (corpus.py:235)."""
    return write_corpus(make_corpus(rows, users, seed, views), dest, batch_size)
