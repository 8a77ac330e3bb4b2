"""GPU: the row-aligned `_extract_batch` kernel against the reference's own
`_extract_batch` outputs over the cleaned + joined 2k table (tests/golden)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, corpus

pytestmark = pytest.mark.gpu
DAGS = ("default", "fig4", "sign_heavy", "cross_heavy", "lookup_heavy")


@pytest.mark.parametrize("dag", DAGS)
def test_extract_batch_matches_reference(dag):
    from paper_2210_07768_b200.columns import read_view
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.engine import extract_batch
    from paper_2210_07768_b200.workloads import workload_config
    c, d = corpus(2000, 300, 7)
    table = read_view(GOLDEN / "joined_2k.fbxc")
    out = extract_batch(table, config_from_dict(workload_config(dag), d))
    ref = np.load(GOLDEN / f"extract_{dag}.npz")
    cols = [k for k in ref.files if "." not in k]
    assert cols
    for col in cols:
        img = out.columns[col]
        np.testing.assert_array_equal(img.null_mask(), ref[col + ".null"], err_msg=col)
        if col + ".offsets" in ref.files:
            np.testing.assert_array_equal(img.offsets.astype(np.uint64), ref[col + ".offsets"])
            np.testing.assert_array_equal(img.data, ref[col], err_msg=col)
        else:
            np.testing.assert_array_equal(img.data, ref[col], err_msg=col)
    for c0 in table.order:  # input columns pass through untouched
        assert out.columns[c0] is table.columns[c0]
