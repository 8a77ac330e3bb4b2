"""ctypes binding of libfbx.so (include/fbx.h).

ctypes releases the GIL for the duration of every foreign call, so a host
thread driving one engine never blocks other Python threads.  The library is
built in-tree (``build.py``); a missing library is an error, never a
fallback.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import threading
from pathlib import Path

import numpy as np

from .build import LIB, build_library

_lock = threading.Lock()
_lib = None

FBX_MAX_PARAM_SLOTS = 384
STATE_FIELDS = ("error_key", "error_detail", "emit_range_pos", "emit_range_label",
                "emit_null_pos", "pool_flagged", "tile_ticket", "pool_head", "pool_overflow",
                "digest", "instances", "signs", "malformed", "filtered", "joined", "side_rows",
                "dup_seen", "pad")
STATE_BYTES = 8 * len(STATE_FIELDS)

EXPORTS = ("fbx_version", "fbx_error_message", "fbx_compile", "fbx_free", "fbx_program_load",
           "fbx_program_unload", "fbx_program_kernel", "fbx_kernel_attributes",
           "fbx_kernel_set_max_dynamic_smem", "fbx_launch", "fbx_state_reset",
           "fbx_dict_build", "fbx_l2_flush", "fbx_exclusive_scan_u32", "fbx_gather_strings",
           "fbx_dup_resolve", "fbx_state_snapshot",
           "fbx_pool_reset", "fbx_crc32", "fbx_crc32_scratch_words", "fbx_idset_clear",
           "fbx_pool_account", "fbx_memset_async", "fbx_read_spans",
           "fbx_merge_subtiles", "fbx_select_rows", "fbx_take", "fbx_pack_nulls",
           "fbx_sort_keys", "fbx_join_count", "fbx_join_fill", "fbx_first_repeat",
           "fbx_unpack_nulls", "fbx_spans", "fbx_idset_entries", "fbx_seen_before")


class FbxError(RuntimeError):
    pass


def lib() -> ctypes.CDLL:
    """Load (building first if the in-tree library is missing) libfbx.so."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB.exists():
                build_library()
            L = ctypes.CDLL(str(LIB))
            vp, sz, c = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
            L.fbx_version.restype = ctypes.c_char_p
            L.fbx_error_message.restype = ctypes.c_char_p
            L.fbx_error_message.argtypes = [ctypes.c_void_p]
            L.fbx_compile.argtypes = [ctypes.c_char_p, ctypes.c_char_p,
                                      ctypes.POINTER(ctypes.c_char_p), c,
                                      ctypes.POINTER(vp), ctypes.POINTER(sz),
                                      ctypes.c_char_p, sz]
            L.fbx_free.argtypes = [vp]
            L.fbx_program_load.argtypes = [vp, sz, ctypes.POINTER(vp)]
            L.fbx_program_unload.argtypes = [vp]
            L.fbx_program_kernel.argtypes = [vp, ctypes.c_char_p, ctypes.POINTER(vp)]
            L.fbx_kernel_attributes.argtypes = [vp, ctypes.POINTER(c), ctypes.POINTER(c),
                                                ctypes.POINTER(c)]
            L.fbx_kernel_set_max_dynamic_smem.argtypes = [vp, c]
            L.fbx_launch.argtypes = [vp, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, vp, vp]
            L.fbx_state_reset.argtypes = [vp, vp, sz, vp]
            L.fbx_dict_build.argtypes = [vp, ctypes.c_ulonglong, vp, vp, vp,
                                         ctypes.c_ulonglong, vp, vp]
            L.fbx_l2_flush.argtypes = [vp, sz, vp]
            L.fbx_exclusive_scan_u32.argtypes = [vp, vp, ctypes.c_ulonglong, vp]
            L.fbx_gather_strings.argtypes = [vp, vp, vp, ctypes.c_ulonglong, vp, vp]
            L.fbx_dup_resolve.argtypes = [vp, vp, ctypes.c_ulonglong, vp, vp]
            L.fbx_state_snapshot.argtypes = [vp, vp, vp]
            L.fbx_pool_reset.argtypes = [vp, vp]
            L.fbx_idset_clear.argtypes = [vp, sz, vp, sz, vp, vp]
            L.fbx_memset_async.argtypes = [vp, c, sz, vp]
            u, ull = ctypes.c_uint, ctypes.c_ulonglong
            L.fbx_pool_account.argtypes = [vp, vp, ull, u, u, vp, u, vp, u, vp, vp, u, ull, ull,
                                           vp, vp, vp, vp]
            L.fbx_crc32.argtypes = [vp, ctypes.c_ulonglong, vp, vp, vp]
            L.fbx_read_spans.argtypes = [ctypes.c_char_p, vp, vp, vp, vp, ctypes.c_uint,
                                         ctypes.c_uint]
            L.fbx_merge_subtiles.argtypes = [vp, ctypes.c_uint, ctypes.c_ulonglong,
                                             ctypes.c_ulonglong, ctypes.c_ulonglong,
                                             ctypes.c_uint] + [vp] * 12 + [vp]
            ull = ctypes.c_ulonglong
            L.fbx_select_rows.argtypes = [vp, ull, vp, vp, vp]
            L.fbx_take.argtypes = [vp, ctypes.c_uint, vp, ull, vp, vp]
            L.fbx_pack_nulls.argtypes = [vp, vp, ull, vp, vp]
            L.fbx_sort_keys.argtypes = [vp, vp, ull, vp, vp, vp, vp, vp, vp, vp]
            L.fbx_join_count.argtypes = [vp, vp, ull, vp, ull, vp, vp, vp]
            L.fbx_join_fill.argtypes = [vp, ull, vp, vp, vp, vp, ull, vp, vp, vp]
            L.fbx_first_repeat.argtypes = [vp, vp, ull, vp, vp]
            L.fbx_unpack_nulls.argtypes = [vp, ull, vp, vp]
            L.fbx_spans.argtypes = [vp, vp, ull, vp, vp, vp]
            L.fbx_idset_entries.argtypes = [vp, vp, vp, ull, vp, vp, vp, vp]
            L.fbx_seen_before.argtypes = [vp, vp, ull, vp, ull, vp, vp]
            L.fbx_crc32_scratch_words.argtypes = [ctypes.c_ulonglong]
            L.fbx_crc32_scratch_words.restype = ctypes.c_ulonglong
            for name in EXPORTS:
                getattr(L, name).restype = getattr(L, name).restype or c
            L.fbx_version.restype = ctypes.c_char_p
            L.fbx_error_message.restype = ctypes.c_char_p
            L.fbx_error_message.argtypes = [ctypes.c_void_p]
            L.fbx_free.restype = None
            _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib().fbx_error_message(None).decode(errors="replace")
        raise FbxError(f"{what} failed ({rc}): {msg}")


_CUBIN_CACHE: dict[str, bytes] = {}


def compile_source(source: str, name: str = "plan.cu", options: tuple[str, ...] = ()) -> bytes:
    """NVRTC -> sm_100a cubin (host-only).  Cached per process and on disk."""
    opts = ("-arch=sm_100a", "-std=c++17", "-lineinfo", "-diag-suppress=177,550", *options,
            *os.environ.get("FBX_NVRTC_OPTS", "").split())  # A/B experiments only
    patch = os.environ.get("FBX_SOURCE_PATCH")
    if patch:  # A/B experiments only: a script's patch(source) -> source
        ns: dict = {}
        exec(compile(Path(patch).read_text(), patch, "exec"), ns)
        source = ns["patch"](source)
    dump = os.environ.get("FBX_DUMP_SOURCE")
    if dump:  # profiling aid: keep the generated plan so ncu can import it by name
        Path(dump).write_text(source)
        name = str(Path(dump).resolve())
    key = hashlib.sha256((name + "\0" + source + "\0" + "\0".join(opts)).encode()).hexdigest()
    if key in _CUBIN_CACHE:
        return _CUBIN_CACHE[key]
    cache_dir = Path(os.environ.get("FBX_CACHE", Path.home() / ".cache" / "fbx_b200"))
    cpath = cache_dir / f"{key}.cubin"
    if cpath.exists():
        data = cpath.read_bytes()
        if data[:4] == b"\x7fELF":  # else a damaged entry: recompile
            _CUBIN_CACHE[key] = data
            return data
    L = lib()
    arr = (ctypes.c_char_p * len(opts))(*[o.encode() for o in opts])
    img = ctypes.c_void_p()
    n = ctypes.c_size_t()
    log = ctypes.create_string_buffer(1 << 16)
    rc = L.fbx_compile(source.encode(), name.encode(), arr, len(opts), ctypes.byref(img),
                       ctypes.byref(n), log, len(log))
    if rc != 0:
        raise FbxError(f"plan compilation failed: {L.fbx_error_message(None).decode(errors='replace')}")
    data = ctypes.string_at(img, n.value)
    L.fbx_free(img)
    _CUBIN_CACHE[key] = data
    try:
        cache_dir.mkdir(parents=True, exist_ok=True)
        tmp = cpath.with_suffix(f".{os.getpid()}.tmp")  # ranks compile concurrently
        tmp.write_bytes(data)
        tmp.replace(cpath)
    except OSError:
        pass
    return data


class Program:
    """A loaded plan module and its kernels."""

    def __init__(self, cubin: bytes):
        self._cubin = ctypes.create_string_buffer(cubin, len(cubin))
        h = ctypes.c_void_p()
        _check(lib().fbx_program_load(self._cubin, len(cubin), ctypes.byref(h)), "program load")
        self.handle = h
        self.kernels: dict[str, ctypes.c_void_p] = {}

    def kernel(self, name: str) -> ctypes.c_void_p:
        if name not in self.kernels:
            k = ctypes.c_void_p()
            _check(lib().fbx_program_kernel(self.handle, name.encode(), ctypes.byref(k)),
                   f"kernel {name}")
            self.kernels[name] = k
        return self.kernels[name]

    def attributes(self, name: str) -> dict:
        regs, thr, smem = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(lib().fbx_kernel_attributes(self.kernel(name), ctypes.byref(regs),
                                           ctypes.byref(thr), ctypes.byref(smem)), "attributes")
        return {"registers": regs.value, "max_threads": thr.value, "static_smem": smem.value}

    def set_dynamic_smem(self, name: str, nbytes: int):
        _check(lib().fbx_kernel_set_max_dynamic_smem(self.kernel(name), int(nbytes)),
               "set dynamic smem")

    def launch(self, name: str, grid: int, block: int, smem: int, stream: int,
               params: np.ndarray):
        assert params.dtype == np.uint64 and params.size == FBX_MAX_PARAM_SLOTS
        _check(lib().fbx_launch(self.kernel(name), int(grid), int(block), int(smem),
                                ctypes.c_void_p(stream), params.ctypes.data_as(ctypes.c_void_p)),
               f"launch {name}")


def state_reset(d_state: int, d_status: int, n_tiles: int, stream: int):
    _check(lib().fbx_state_reset(ctypes.c_void_p(d_state), ctypes.c_void_p(d_status),
                                 int(n_tiles), ctypes.c_void_p(stream)), "state reset")


def state_snapshot(d_state: int, h_mapped: int, stream: int):
    _check(lib().fbx_state_snapshot(ctypes.c_void_p(d_state), ctypes.c_void_p(h_mapped),
                                    ctypes.c_void_p(stream)), "state snapshot")


def idset_clear(d_ids: int, n: int, d_pairs: int, npairs: int, d_state: int, stream: int):
    _check(lib().fbx_idset_clear(ctypes.c_void_p(d_ids), int(n), ctypes.c_void_p(d_pairs),
                                 int(npairs), ctypes.c_void_p(d_state), ctypes.c_void_p(stream)),
           "id-set clear")


def pool_reset(d_state: int, stream: int):
    _check(lib().fbx_pool_reset(ctypes.c_void_p(d_state), ctypes.c_void_p(stream)), "pool reset")


def crc32(d_buf: int, n: int, d_scratch: int, d_out: int, stream: int):
    _check(lib().fbx_crc32(ctypes.c_void_p(d_buf), n, ctypes.c_void_p(d_scratch),
                           ctypes.c_void_p(d_out), ctypes.c_void_p(stream)), "crc32")


def crc32_scratch_words(n: int) -> int:
    return int(lib().fbx_crc32_scratch_words(n))


def dict_build(d_slots: int, capacity: int, d_blob: int, d_offs: int, d_vals: int, n: int,
               d_dup: int, stream: int):
    _check(lib().fbx_dict_build(ctypes.c_void_p(d_slots), capacity, ctypes.c_void_p(d_blob),
                                ctypes.c_void_p(d_offs), ctypes.c_void_p(d_vals), n,
                                ctypes.c_void_p(d_dup), ctypes.c_void_p(stream)), "dict build")


def l2_flush(d_buf: int, nbytes: int, stream: int):
    _check(lib().fbx_l2_flush(ctypes.c_void_p(d_buf), int(nbytes), ctypes.c_void_p(stream)),
           "l2 flush")


def dup_resolve(d_winner: int, d_later: int, n_slots: int, d_out: int, stream: int):
    _check(lib().fbx_dup_resolve(ctypes.c_void_p(d_winner), ctypes.c_void_p(d_later),
                                 int(n_slots), ctypes.c_void_p(d_out), ctypes.c_void_p(stream)),
           "dup resolve")


def memset_async(d_ptr: int, value: int, nbytes: int, stream: int):
    _check(lib().fbx_memset_async(ctypes.c_void_p(d_ptr), value, int(nbytes),
                                  ctypes.c_void_p(stream)), "memset")


def pool_account(d_flag: int, d_chunk: int, n_tiles: int, spc: int, tile_rows: int,
                 d_keys: int, kw: int, d_sizes: int, ni: int, d_joined: int, d_nodes: int,
                 n_nodes: int, lanes_per_group: int, capacity: int, d_rank: int, d_sum: int,
                 d_state: int, stream: int):
    vp = ctypes.c_void_p
    _check(lib().fbx_pool_account(vp(d_flag), vp(d_chunk), n_tiles, spc, tile_rows, vp(d_keys),
                                  kw, vp(d_sizes), ni, vp(d_joined), vp(d_nodes), n_nodes,
                                  lanes_per_group, capacity, vp(d_rank), vp(d_sum), vp(d_state),
                                  vp(stream)), "pool account")


def exclusive_scan_u32(d_in: int, d_out: int, n: int, stream: int):
    _check(lib().fbx_exclusive_scan_u32(ctypes.c_void_p(d_in), ctypes.c_void_p(d_out), n,
                                        ctypes.c_void_p(stream)), "scan")


def gather_strings(d_ptrs: int, d_lens: int, d_offsets: int, n: int, d_out: int, stream: int):
    _check(lib().fbx_gather_strings(ctypes.c_void_p(d_ptrs), ctypes.c_void_p(d_lens),
                                    ctypes.c_void_p(d_offsets), n, ctypes.c_void_p(d_out),
                                    ctypes.c_void_p(stream)), "gather strings")


def host_threads() -> int:
    """Reader threads for the host ingest (fbx_read_spans): FBX_READ_THREADS, else
    every core this process may run on, up to 32.  Each reader writes its pieces
    back from its cache (clwb) so the H2D that follows runs at the pinned rate;
    measured per 1M-record run_pipelined on the 16-core box: 8 readers 6.1 ms,
    12 5.1-5.5 ms, 16 4.9-5.1 ms (without the write-back 16 readers were slower
    than 8: the DMA snooped their dirty lines)."""
    env = os.environ.get("FBX_READ_THREADS")
    if env:
        return max(1, int(env))
    try:
        n = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        n = os.cpu_count() or 1
    cap = os.environ.get("FEATUREBOX_THREADS", "")  # the reference's host-thread cap
    if cap.isdigit() and int(cap) >= 1:
        n = min(n, int(cap))
    return max(1, min(32, n))


def read_spans(path, dst: int, file_off, length, dst_off, threads: int | None = None):
    """Parallel pread of FBXC spans into host memory at ``dst`` (fbx_read_spans);
    raises FbxError (FBX_E_IO) on open / read failures and truncated files."""
    fo = np.ascontiguousarray(file_off, dtype=np.uint64)
    ln = np.ascontiguousarray(length, dtype=np.uint64)
    do = np.ascontiguousarray(dst_off, dtype=np.uint64)
    n = int(fo.size)
    if not (ln.size == do.size == n):
        raise ValueError("read_spans: span arrays differ in length")
    vp = ctypes.c_void_p
    _check(lib().fbx_read_spans(str(path).encode(), vp(dst), fo.ctypes.data_as(vp),
                                ln.ctypes.data_as(vp), do.ctypes.data_as(vp), n,
                                host_threads() if threads is None else int(threads)),
           "read spans")


def merge_subtiles(d_tile_start: int, spc: int, n_tiles: int, n: int, s0: int, max_len: int,
                   ins: tuple, outs: tuple, d_scratch: int, d_bad: int, stream: int):
    """fbx_merge_subtiles: ins / outs = (ids, labels, offsets, slots, signs) pointers."""
    vp = ctypes.c_void_p
    _check(lib().fbx_merge_subtiles(vp(d_tile_start), spc, n_tiles, n, s0, max_len,
                                    *[vp(x) for x in ins], *[vp(x) for x in outs], vp(d_scratch),
                                    vp(d_bad), vp(stream)), "merge sub-tiles")


def call(name: str, *args):
    """A libfbx table operation (include/fbx.h); pointers and sizes as ints."""
    _check(getattr(lib(), name)(*args), name)
