"""Where a run fails, in the reference's pipeline order.

Every failure is an error key (``fbx::err_key``, fbx_core.cuh):
``chunk(32) | stage(4) | layer(8) | node rank(12) | code(8)`` -- the smallest
key is the failure the reference raises first (chunk by chunk, stage by stage
within a chunk, pipeline.py:1040-1090).  Two failures are only known after the
kernel and are placed here, by the single-GPU engine and by the record-sharded
combine (``sharded.py``) alike:

* a repeated instance id fails the merge of the chunk holding the first row, in
  row order, whose id occurred before (``check_unique_ids``, viewpipe.py:562-576);
* a null / non-0/1 label fails when its mini-batch is flushed: the merge of the
  chunk whose ``_Emitter.add`` fills the batch (pipeline.py:748-777), else the
  final flush (stage "emit").  ``emit_minibatch`` checks every label of a batch
  for null before ``MiniBatch.validate`` checks the range (pipeline.py:357-433),
  so within one batch a null wins over an earlier non-0/1 label.
"""

from __future__ import annotations

import numpy as np

from . import codegen

NONE = (1 << 64) - 1


def key_of(chunk: int, stage: str, sub: int) -> int:
    return (chunk << 32) | (codegen.STAGE[stage] << 28) | sub


def dup_key(row: int, batch_size: int) -> int:
    """check_unique_ids fails in the merge of the row's chunk."""
    return key_of(row // batch_size, "merge", codegen.ERR["dup_id"])


def label_failure(null_pos: int, range_pos: int, batch_size: int):
    """(batch, is_range, position in batch) of the first label failure, from
    the first null label's and the first non-0/1 label's emission positions
    (``NONE`` = none); None without one."""
    bn = null_pos // batch_size if null_pos != NONE else None
    br = range_pos // batch_size if range_pos != NONE else None
    if bn is None and br is None:
        return None
    if br is None or (bn is not None and bn <= br):
        return bn, 0, null_pos % batch_size
    return br, 1, range_pos % batch_size


def label_key(failure, chunk_ends: np.ndarray, chunk0: int, batch_size: int) -> int:
    """Error key of a label failure (``label_failure``): the merge of the first
    chunk whose run-inclusive instance count reaches (batch + 1) * batch_size
    (``chunk_ends``: one count per chunk, the first being chunk ``chunk0``),
    after that chunk's id check; else the final flush."""
    batch, rng, pos = failure
    code = codegen.ERR["label_range" if rng else "null_label"]
    sub = (((1 + rng) & 0xFF) << 20) | ((pos & 0xFFF) << 8) | code
    hit = np.nonzero(np.asarray(chunk_ends) >= (batch + 1) * batch_size)[0]
    if hit.size == 0:
        return key_of(0xFFFFFFFF, "emit", sub)
    return key_of(int(hit[0]) + chunk0, "merge", sub)
