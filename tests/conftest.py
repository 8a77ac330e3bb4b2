"""Shared fixtures.  `gpu` marks tests that need a B200 (run with -m gpu)."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = ROOT / "tests" / "golden"
REFERENCE = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def goldens():
    return json.loads((GOLDEN / "goldens.json").read_text())


def golden_run(goldens, rows, seed, dag, ops_only=False, views=2):
    for r in goldens["runs"]:
        if (r["rows"], r["seed"], r["dag"], r["ops_only"], r["views"]) == (rows, seed, dag,
                                                                            ops_only, views):
            return r
    raise KeyError((rows, seed, dag, ops_only, views))


_CORPORA = {}


def corpus(rows, users, seed, views=2):
    """In-memory corpus + its files (tables for lookup_heavy) in a temp dir."""
    import tempfile

    from paper_2210_07768_b200.corpus import make_corpus, write_corpus
    from paper_2210_07768_b200.workloads import write_lookup_tables
    key = (rows, users, seed, views)
    if key not in _CORPORA:
        c = make_corpus(rows, users, seed, views)
        d = Path(tempfile.mkdtemp(prefix="fbxcorpus"))
        write_corpus(c, d)
        if views == 2:
            write_lookup_tables(d, users)
        _CORPORA[key] = (c, d)
    return _CORPORA[key]


def reference_available() -> bool:
    return (REFERENCE / "featurebox" / "__init__.py").exists()


# The unmodified reference as installed for the reference arm (pip --target
# baseline/_ref, git-ignored, travels to the GPU box); /root/reference here.
INSTALLED_REFERENCE = ROOT / "baseline" / "_ref"


def reference_package_path() -> Path | None:
    for p in (INSTALLED_REFERENCE, REFERENCE):
        if (p / "featurebox" / "__init__.py").exists():
            return p
    return None
