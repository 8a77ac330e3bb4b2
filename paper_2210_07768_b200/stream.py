"""The drop-in ``run_pipelined``'s driver stream: FBXC file -> HBM in bounded memory.

The reference reads the driver view ``batch_size`` rows at a time through a
bounded queue of chunks (``read_driver`` + ``_pump``, pipeline.py:986-1006) and
never holds the whole log.  Here a slice of whole chunks is the unit:

  host reader thread   parallel pread of the slice's column spans (libfbx
                       ``fbx_read_spans``) into one of ``nbuf`` pinned buffers
  copy stream          one H2D of the packed slice into one of ``nbuf`` device
                       buffers
  compute stream       the fused kernel over the slice (the look-back and the
                       counters continue across slices); its CSR lands in a
                       one-slice ring (launch-local offsets), which a trainer
                       reads per slice and the digest sink never needs

Host and device memory are O(slice), whatever the log size (the run-wide
instance-id set of ``check_unique_ids`` and one status word per chunk aside).
"""

from __future__ import annotations

import os
import threading
import time

from . import runtime
from .columns import open_view


class FileRun:
    """One driver file streamed through an ``Engine`` (bounded memory).

    Built from the prepared plan alone, so ``start()`` can begin reading the
    first slices while the side views, the basic features and their indexes
    are still being prepared; ``run(engine)`` then consumes the slices."""

    PARTS = ("nulls", "offsets", "data")

    def __init__(self, prepared, path, columns=None, device="cuda", slice_rows: int = 1 << 19,
                 nbuf: int = 3, threads: int | None = None, rows: tuple[int, int] | None = None):
        import torch
        self.torch = torch
        self.vf = vf = open_view(path)
        chunk = prepared.ir.chunk
        # rows: a record shard [lo, hi) of the log (whole chunks; sharded.py)
        r0, n = (0, vf.row_count) if rows is None else (rows[0], min(rows[1], vf.row_count))
        if (r0 % chunk and r0 != n) or not 0 <= r0 <= n:
            raise ValueError("FileRun: a row range starts at a chunk boundary inside the log")
        self.row_lo, self.row_hi = r0, n
        self.n = n - r0
        if prepared.program.tiles_per_chunk > 1:
            raise ValueError("FileRun: batch_size > 1024 runs device-resident (chunk merge)")
        limit = (1 << 24) // chunk * chunk  # Engine.LAUNCH_ROWS_MAX
        self.slice_rows = S = min(max(chunk, slice_rows // chunk * chunk), max(chunk, limit))
        self.bounds = [(lo, min(lo + S, n)) for lo in range(r0, n, S)]
        # a short last slice: once the reads are done (the call is bound by the page
        # cache -> pinned copy), only its H2D + kernel remain (measured: 5.16 -> 4.89
        # ms per 1M-record run_pipelined; FBX_TAPER=0 turns it off)
        tail = max(chunk, (S // 4) // chunk * chunk)
        if os.environ.get("FBX_TAPER", "1") != "0" and len(self.bounds) >= 2:
            lo, hi = self.bounds[-1]
            cut = (hi - tail) // chunk * chunk
            if cut - lo >= tail:
                self.bounds[-1:] = [(lo, cut), (cut, hi)]
        slots = prepared.program.slots
        kinds = dict(vf.schema)
        self.cols = [c for c, _ in vf.schema
                     if (columns is None or c in columns)
                     and any(f"drv.{c}.{p}" in slots for p in self.PARTS)]
        self.threads = runtime.host_threads() if threads is None else threads
        # boundary offsets of every var-length column at every slice edge: the data
        # span of a slice is [off[lo], off[hi]) (one 4-byte pread per edge)
        edges = [lo for lo, _ in self.bounds] + [n]  # n: the range's end
        self.edge_off: dict[str, list[int]] = {}
        with open(vf.path, "rb") as fh:
            fd = fh.fileno()
            for c in self.cols:
                if kinds[c].var_length:
                    o0 = vf.segments[(c, "offsets")][0]
                    self.edge_off[c] = [int.from_bytes(os.pread(fd, 4, o0 + 4 * r), "little")
                                        for r in edges]
        self.kinds = kinds
        self.layout = [self._pieces(k) for k in range(len(self.bounds))]
        self.cap = max([sum((b - a + 15) // 16 * 16 for _, _, a, b, _ in pcs)
                        for pcs in self.layout] or [16]) + 16
        dev = torch.device(device)
        nb = min(nbuf, max(1, len(self.bounds)))
        self.host = [torch.empty(self.cap, dtype=torch.uint8, pin_memory=True) for _ in range(nb)]
        self.dev = [torch.empty(self.cap + 32, dtype=torch.uint8, device=dev) for _ in range(nb)]
        self.s_h2d = torch.cuda.Stream(dev)
        self.s_comp = torch.cuda.Stream(dev)
        self.h2d_bytes = sum(sum(b - a for _, _, a, b, _ in pcs) for pcs in self.layout)
        K = len(self.bounds)
        self.ready = [threading.Event() for _ in range(K)]
        self.recorded = [threading.Event() for _ in range(K)]
        self.h2d_done = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        self.h2d_start = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        self.comp_done = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        self.comp_start = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        self.failure: list = [None, None]
        self.read_s = 0.0
        self.cancel = threading.Event()
        self.thread = None

    def _pieces(self, k: int):
        """(column, part, start, end, dst) byte spans of slice k within each
        segment, dst 16-B aligned in the packed slice."""
        lo, hi = self.bounds[k]
        vf = self.vf
        out, off = [], 0
        for c in self.cols:
            kind = self.kinds[c]
            sp = {"nulls": (lo // 8, (hi + 7) // 8)}
            if kind.var_length:
                e = self.edge_off[c]
                seg_len = vf.segments[(c, "data")][1]
                sp["offsets"] = (lo * 4, (hi + 1) * 4)
                sp["data"] = (e[k] & ~15, min((e[k + 1] + 15) & ~15, seg_len))
            else:
                w = kind.fixed_width
                sp["data"] = (lo * w, hi * w)
            for p, (a, b) in sp.items():
                out.append((c, p, a, b, off))
                off += (b - a + 15) // 16 * 16
        return out

    def _reader(self):
        """Host thread: read slice k into pinned buffer k % nb, then enqueue its
        H2D on the copy stream -- so the first slices are in HBM before the
        engine exists.  Reuse waits: the pinned buffer for slice k - nb's H2D,
        the device buffer (on the device) for slice k - nb's kernel."""
        torch, nb, vf = self.torch, len(self.host), self.vf
        k = 0
        try:
            for k in range(len(self.bounds)):
                if self.cancel.is_set():
                    return
                if k >= nb:
                    self.h2d_done[k - nb].synchronize()  # the pinned buffer is free again
                t = time.perf_counter()
                pcs = self.layout[k]
                torch.cuda.nvtx.range_push(f"fbx read slice {k}")
                runtime.read_spans(vf.path, self.host[k % nb].data_ptr(),
                                   [vf.segments[(c, p)][0] + a for c, p, a, _, _ in pcs],
                                   [b - a for _, _, a, b, _ in pcs],
                                   [o for *_, o in pcs], self.threads)
                torch.cuda.nvtx.range_pop()
                self.read_s += time.perf_counter() - t
                if k >= nb:
                    self.recorded[k - nb].wait()  # slice k - nb's kernel is enqueued
                    if self.cancel.is_set():
                        return
                buf = k % nb
                nbytes = pcs[-1][4] + (pcs[-1][3] - pcs[-1][2]) if pcs else 0
                with torch.cuda.stream(self.s_h2d):
                    if k >= nb:
                        self.s_h2d.wait_event(self.comp_done[k - nb])  # device buffer reuse
                    self.h2d_start[k].record(self.s_h2d)
                    self.dev[buf][:nbytes].copy_(self.host[buf][:nbytes], non_blocking=True)
                    self.h2d_done[k].record(self.s_h2d)
                self.ready[k].set()
        except BaseException as exc:  # noqa: BLE001 -- re-raised by the host loop
            self.failure[0], self.failure[1] = k, exc
            for e in self.ready[k:]:
                e.set()

    def start(self):
        """Begin reading slices into the pinned ring and copying them to HBM
        (a host thread)."""
        if self.thread is None:
            cur = self.torch.cuda.current_stream(self.dev[0].device)
            self.s_h2d.wait_stream(cur)  # the staging buffers' allocation
            self.thread = threading.Thread(target=self._reader, name="fbx-read", daemon=True)
            self.thread.start()

    def stop(self):
        self.cancel.set()
        for e in self.recorded:
            e.set()
        if self.thread is not None:
            self.thread.join()

    def run(self, eng) -> dict:
        """Stream every slice through ``eng`` (reserved with ``ring=True`` and a
        begun run); returns the timing / byte counters of the stream (the
        engine's state holds the results)."""
        torch = self.torch
        nb = len(self.host)
        self.start()
        cur = torch.cuda.current_stream(eng.device)
        self.s_comp.wait_stream(cur)  # the engine's prepare work (index builds, run reset)
        launch_s = 0.0
        launches = 0
        tiles_before = 0
        done = 0
        try:
            for k, (lo, hi) in enumerate(self.bounds):
                self.ready[k].wait()
                if self.failure[1] is not None and self.failure[0] <= k:
                    raise _ReadFailure(self.failure[0], self.failure[1])
                buf = k % nb
                pcs = self.layout[k]
                base = self.dev[buf].data_ptr()
                for c, p, a, _, o in pcs:
                    eng._set(f"drv.{c}.{p}", base + o - a)
                with torch.cuda.stream(self.s_comp):
                    self.s_comp.wait_event(self.h2d_done[k])
                    self.comp_start[k].record(self.s_comp)
                    t = time.perf_counter()
                    tiles = eng.launch(lo, hi, self.s_comp.cuda_stream, tile_base=tiles_before)
                    launches += 1 + eng.ring_after_launch(self.s_comp.cuda_stream)
                    launch_s += time.perf_counter() - t
                    self.comp_done[k].record(self.s_comp)
                self.recorded[k].set()
                tiles_before += tiles
                done = k + 1
        except _ReadFailure as exc:
            # the slices before the failed one ran: their failures may come first
            self.stop()
            exc.timings = self._timings(cur, done, launches, launch_s)
            raise
        finally:
            self.stop()
        return self._timings(cur, done, launches, launch_s)

    def _timings(self, cur, done: int, launches: int, launch_s: float) -> dict:
        self.s_comp.synchronize()
        self.s_h2d.synchronize()
        cur.wait_stream(self.s_comp)
        ev = list(zip(self.h2d_start, self.h2d_done))[:done]
        comp = list(zip(self.comp_start, self.comp_done))[:done]
        return {"launches": launches, "launch_s": launch_s, "read_s": self.read_s,
                "h2d_s": sum(a.elapsed_time(b) for a, b in ev) / 1e3,
                "kernel_s": sum(a.elapsed_time(b) for a, b in comp) / 1e3,
                "h2d_bytes": sum(sum(b - a for _, _, a, b, _ in self.layout[k])
                                 for k in range(done)),
                "slices": done}


class _ReadFailure(Exception):
    def __init__(self, index: int, cause: BaseException):
        super().__init__(str(cause))
        self.index, self.cause = index, cause
