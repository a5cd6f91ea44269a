"""Thin ctypes binding of libmbe.so (include/mbe.h) — argument marshalling only.

Every step of the search runs in the library's CUDA kernels.  There is no CPU
fallback: if libmbe.so is missing or no CUDA device is usable, the calls raise.
Function names mirror the C ABI: mbe_load_csr, mbe_enumerate, mbe_free,
mbe_get_info, mbe_strerror, mbe_last_error_detail.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import threading
from typing import List, Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MBE_LIB_PATH: load an alternative build of the same library (A/B timing of build variants)
LIB_PATH = os.environ.get("MBE_LIB_PATH") or os.path.join(_HERE, "libmbe.so")

MBE_OK, MBE_EINVAL, MBE_ENOMEM, MBE_ECUDA, MBE_EOVERFLOW, MBE_ERANGE, MBE_EDIST, MBE_EINTERNAL = 0, -1, -2, -3, -4, -5, -6, -7
MBE_NO_STEAL, MBE_STATS, MBE_NO_ANTICHAIN, MBE_NO_TWIN, MBE_STEAL_ONE, MBE_STEAL_HALF = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20
MBE_ARENA_GROW = 0x40
MBE_NO_RS = 0x80
MBE_ORDER = {"ascending": 0, "input": 1, "descending": 2}

EXPORTED_SYMBOLS = ("mbe_load_csr", "mbe_enumerate", "mbe_get_info", "mbe_free", "mbe_release_workspaces",
                    "mbe_strerror", "mbe_last_error_detail", "mbe_format_listing", "mbe_counter_create",
                    "mbe_counter_ipc_handle", "mbe_counter_open", "mbe_counter_ptr", "mbe_counter_reset",
                    "mbe_counter_read", "mbe_counter_close")

_u32, _i32, _u64, _dbl, _vp = ctypes.c_uint32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
_p64, _p32 = ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32)


class mbe_config(ctypes.Structure):
    _fields_ = [("struct_size", _u32), ("ctas_per_sm", _u32), ("threads_per_cta", _u32),
                ("bitmap_threshold", _u32), ("candidate_side", _i32), ("flags", _u32), ("rank", _u32),
                ("world", _u32), ("claim_counter", _vp), ("arena_bytes", _u64), ("stream", _vp),
                ("per_root", _p64), ("watchdog_ms", _u32), ("defer_min", _u32), ("order", _u32)]


class mbe_output(ctypes.Structure):
    _fields_ = [("cap_records", _u64), ("cap_ids", _u64), ("rec_off", _p64), ("rec_n1", _p32), ("rec_n2", _p32),
                ("ids", _p32)]


class mbe_result(ctypes.Structure):
    _fields_ = [("count", _u64), ("hash", _u64), ("tasks", _u64), ("pruned", _u64), ("steals", _u64),
                ("records_written", _u64), ("truncated", _u32), ("candidate_side", _i32), ("kernel_ms", _dbl),
                ("wall_ms", _dbl), ("alg_bytes", _u64), ("list_tasks", _u64), ("bitmap_tasks", _u64),
                ("frames", _u64), ("n_warps", _u32), ("max_depth", _u32), ("phase_cycles", _u64 * 16),
                ("max_task_cycles", _u64 * 3), ("roots_out_ms", _dbl), ("max_phase_cycles", _u64 * 16),
                ("roots_claimed", _u64), ("claim_chunks", _u32), ("attempts", _u32), ("busy_hist", _u32 * 20),
                ("busy_ms_min", _dbl), ("busy_ms_mean", _dbl), ("busy_ms_max", _dbl),
                ("alg_bytes_list", _u64), ("alg_bytes_bitrow", _u64), ("alg_bytes_write", _u64),
                ("workspace_bytes", _u64)]


class mbe_graph_info(ctypes.Structure):
    _fields_ = [("n1", _u32), ("n2", _u32), ("n_edges", _u64), ("max_deg1", _u32), ("max_deg2", _u32),
                ("device", _i32), ("h2d_bytes", _u64)]


_lock = threading.Lock()
_lib = None


class MBEError(RuntimeError):
    def __init__(self, code: int, where: str):
        lib = load_library()
        msg = lib.mbe_strerror(code).decode()
        detail = lib.mbe_last_error_detail().decode()
        super().__init__(f"{where}: {msg} ({code}){': ' + detail if detail else ''}")
        self.code = code


def load_library():
    """dlopen libmbe.so; raises if it has not been built (no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"libmbe.so not built at {LIB_PATH}: run `python -m paper_2401_05039_b200.build` "
                                   "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            lib.mbe_load_csr.argtypes = [_u32, _u32, _p64, _p32, ctypes.c_int, _u32,
                                         ctypes.POINTER(ctypes.c_void_p)]
            lib.mbe_load_csr.restype = ctypes.c_int
            lib.mbe_enumerate.argtypes = [_vp, ctypes.POINTER(mbe_config), ctypes.POINTER(mbe_result),
                                          ctypes.POINTER(mbe_output)]
            lib.mbe_enumerate.restype = ctypes.c_int
            lib.mbe_get_info.argtypes = [_vp, ctypes.POINTER(mbe_graph_info)]
            lib.mbe_get_info.restype = ctypes.c_int
            lib.mbe_free.argtypes = [_vp]
            lib.mbe_free.restype = None
            lib.mbe_release_workspaces.argtypes = []
            lib.mbe_release_workspaces.restype = None
            lib.mbe_strerror.argtypes = [ctypes.c_int]
            lib.mbe_strerror.restype = ctypes.c_char_p
            lib.mbe_last_error_detail.argtypes = []
            lib.mbe_last_error_detail.restype = ctypes.c_char_p
            lib.mbe_format_listing.argtypes = [ctypes.POINTER(mbe_output), _u64, ctypes.c_char_p, _u64,
                                               ctypes.POINTER(ctypes.c_uint64)]
            lib.mbe_format_listing.restype = ctypes.c_int
            lib.mbe_counter_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
            lib.mbe_counter_create.restype = ctypes.c_int
            lib.mbe_counter_ipc_handle.argtypes = [_vp, ctypes.c_char_p]
            lib.mbe_counter_ipc_handle.restype = ctypes.c_int
            lib.mbe_counter_open.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
            lib.mbe_counter_open.restype = ctypes.c_int
            lib.mbe_counter_ptr.argtypes = [_vp]
            lib.mbe_counter_ptr.restype = _vp
            lib.mbe_counter_reset.argtypes = [_vp, _vp]
            lib.mbe_counter_reset.restype = ctypes.c_int
            lib.mbe_counter_read.argtypes = [_vp]
            lib.mbe_counter_read.restype = _u64
            lib.mbe_counter_close.argtypes = [_vp]
            lib.mbe_counter_close.restype = None
            _lib = lib
    return _lib


@dataclasses.dataclass
class Result:
    count: int
    hash: int
    tasks: int
    pruned: int
    steals: int
    candidate_side: int
    kernel_ms: float
    wall_ms: float
    alg_bytes: int
    list_tasks: int
    bitmap_tasks: int
    frames: int
    n_warps: int
    max_depth: int
    records_written: int = 0
    truncated: bool = False
    phase_cycles: tuple = ()
    max_task_cycles: tuple = ()
    roots_out_ms: float = -1.0
    max_phase_cycles: tuple = ()
    roots_claimed: int = 0
    claim_chunks: int = 0
    attempts: int = 1
    busy_hist: tuple = ()
    busy_ms: tuple = ()  # (min, mean, max) task time per warp, MBE_STATS
    alg_parts: tuple = ()  # (list, bit-row, frame writes) algorithmic bytes, MBE_STATS
    workspace_bytes: int = 0  # device workspace of the launch (all warps)


def mbe_strerror(code: int) -> str:
    return load_library().mbe_strerror(code).decode()


def mbe_last_error_detail() -> str:
    return load_library().mbe_last_error_detail().decode()


def mbe_load_csr(n1: int, n2: int, row_ptr, col_idx, device: int = 0, flags: int = 0, ingest_threads: int = 0) -> int:
    """Copy a HOST row-CSR (original ids) to the device; returns an opaque handle.
    ingest_threads: host threads of the ingest (flags bits 0-7; 0 = auto)."""
    flags = (flags & ~0xFF) | (ingest_threads & 0xFF)
    lib = load_library()
    rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
    ci = np.ascontiguousarray(col_idx, dtype=np.uint32)
    if ci.size == 0:
        ci = np.zeros(1, dtype=np.uint32)
    h = ctypes.c_void_p()
    rc = lib.mbe_load_csr(int(n1), int(n2), rp.ctypes.data_as(_p64), ci.ctypes.data_as(_p32), int(device),
                          int(flags), ctypes.byref(h))
    if rc != MBE_OK:
        raise MBEError(rc, "mbe_load_csr")
    return h.value


def make_config(ctas_per_sm: int = 0, threads_per_cta: int = 0, bitmap_threshold: int = 0, candidate_side: int = 0,
                flags: int = 0, rank: int = 0, world: int = 1, claim_counter: int = 0, arena_bytes: int = 0,
                stream: int = 0, per_root=None, watchdog_ms: int = 0, defer_min: int = 0, order=0) -> mbe_config:
    c = mbe_config()
    c.struct_size = ctypes.sizeof(mbe_config)
    c.ctas_per_sm = ctas_per_sm
    c.threads_per_cta = threads_per_cta
    c.bitmap_threshold = bitmap_threshold
    c.candidate_side = candidate_side
    c.flags = flags
    c.rank = rank
    c.world = world
    c.claim_counter = claim_counter or None
    c.arena_bytes = arena_bytes
    c.stream = stream or None
    c.per_root = per_root.ctypes.data_as(_p64) if per_root is not None else None
    c.watchdog_ms = watchdog_ms
    c.defer_min = defer_min
    c.order = MBE_ORDER[order] if isinstance(order, str) else int(order)
    return c


def mbe_enumerate(handle: int, config: Optional[mbe_config] = None, output: Optional[mbe_output] = None) -> Result:
    lib = load_library()
    res = mbe_result()
    rc = lib.mbe_enumerate(ctypes.c_void_p(handle), ctypes.byref(config) if config is not None else None,
                           ctypes.byref(res), ctypes.byref(output) if output is not None else None)
    if rc != MBE_OK:
        raise MBEError(rc, "mbe_enumerate")
    return Result(int(res.count), int(res.hash), int(res.tasks), int(res.pruned), int(res.steals),
                  int(res.candidate_side), float(res.kernel_ms), float(res.wall_ms), int(res.alg_bytes),
                  int(res.list_tasks), int(res.bitmap_tasks), int(res.frames), int(res.n_warps),
                  int(res.max_depth), int(res.records_written), bool(res.truncated),
                  tuple(int(v) for v in res.phase_cycles), tuple(int(v) for v in res.max_task_cycles),
                  float(res.roots_out_ms), tuple(int(v) for v in res.max_phase_cycles), int(res.roots_claimed),
                  int(res.claim_chunks), int(res.attempts), tuple(int(v) for v in res.busy_hist),
                  (float(res.busy_ms_min), float(res.busy_ms_mean), float(res.busy_ms_max)),
                  (int(res.alg_bytes_list), int(res.alg_bytes_bitrow), int(res.alg_bytes_write)),
                  int(res.workspace_bytes))


def mbe_format_listing(output: mbe_output, n_records: int) -> bytes:
    """Canonical listing text (include/mbe.h mbe_format_listing): size query, then format."""
    lib = load_library()
    need = ctypes.c_uint64(0)
    rc = lib.mbe_format_listing(ctypes.byref(output), n_records, None, 0, ctypes.byref(need))
    if rc not in (MBE_OK, MBE_EOVERFLOW):
        raise MBEError(rc, "mbe_format_listing")
    buf = ctypes.create_string_buffer(max(need.value, 1))
    rc = lib.mbe_format_listing(ctypes.byref(output), n_records, buf, need.value, ctypes.byref(need))
    if rc != MBE_OK:
        raise MBEError(rc, "mbe_format_listing")
    return buf.raw[:need.value]


def make_output(cap_records: int, cap_ids: int):
    """(mbe_output, keep-alive arrays rec_off, rec_n1, rec_n2, ids) over numpy host buffers."""
    rec_off = np.zeros(max(cap_records, 1), dtype=np.uint64)
    n1 = np.zeros(max(cap_records, 1), dtype=np.uint32)
    n2 = np.zeros(max(cap_records, 1), dtype=np.uint32)
    ids = np.zeros(max(cap_ids, 1), dtype=np.uint32)
    out = mbe_output()
    out.cap_records, out.cap_ids = cap_records, cap_ids
    out.rec_off, out.rec_n1, out.rec_n2 = rec_off.ctypes.data_as(_p64), n1.ctypes.data_as(_p32), n2.ctypes.data_as(_p32)
    out.ids = ids.ctypes.data_as(_p32)
    return out, (rec_off, n1, n2, ids)


def mbe_get_info(handle: int) -> dict:
    info = mbe_graph_info()
    rc = load_library().mbe_get_info(ctypes.c_void_p(handle), ctypes.byref(info))
    if rc != MBE_OK:
        raise MBEError(rc, "mbe_get_info")
    return {f: getattr(info, f) for f, _ in info._fields_}


def mbe_free(handle: int) -> None:
    if handle:
        load_library().mbe_free(ctypes.c_void_p(handle))


def mbe_release_workspaces() -> None:
    load_library().mbe_release_workspaces()


class ClaimCounter:
    """Cross-process claim counter (include/mbe.h mbe_counter_*): created by one rank, opened by the
    others from its 64-byte CUDA IPC handle; ``ptr`` goes into mbe_config.claim_counter."""

    def __init__(self, device: int = 0, handle: Optional[bytes] = None):
        lib = load_library()
        h = ctypes.c_void_p()
        if handle is None:
            rc = lib.mbe_counter_create(int(device), ctypes.byref(h))
            where = "mbe_counter_create"
        else:
            if len(handle) != 64:
                raise ValueError("IPC handle must be 64 bytes")
            rc = lib.mbe_counter_open(int(device), handle, ctypes.byref(h))
            where = "mbe_counter_open"
        if rc != MBE_OK:
            raise MBEError(rc, where)
        self.c = h.value
        self.owner = handle is None

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        rc = load_library().mbe_counter_ipc_handle(ctypes.c_void_p(self.c), buf)
        if rc != MBE_OK:
            raise MBEError(rc, "mbe_counter_ipc_handle")
        return buf.raw

    @property
    def ptr(self) -> int:
        return load_library().mbe_counter_ptr(ctypes.c_void_p(self.c)) or 0

    def reset(self, stream: int = 0) -> None:
        rc = load_library().mbe_counter_reset(ctypes.c_void_p(self.c), ctypes.c_void_p(stream or None))
        if rc != MBE_OK:
            raise MBEError(rc, "mbe_counter_reset")

    def read(self) -> int:
        return int(load_library().mbe_counter_read(ctypes.c_void_p(self.c)))

    def close(self) -> None:
        if self.c:
            load_library().mbe_counter_close(ctypes.c_void_p(self.c))
            self.c = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MBEGraph:
    """RAII wrapper: a graph resident on one GPU."""

    def __init__(self, n1: int, n2: int, row_ptr, col_idx, device: int = 0, ingest_threads: int = 0):
        self.n1, self.n2 = int(n1), int(n2)
        self.handle = mbe_load_csr(n1, n2, row_ptr, col_idx, device, ingest_threads=ingest_threads)

    @classmethod
    def from_graph(cls, g, device: int = 0, ingest_threads: int = 0) -> "MBEGraph":
        return cls(g.n1, g.n2, g.row_ptr, g.col_idx, device, ingest_threads)

    def info(self) -> dict:
        return mbe_get_info(self.handle)

    def enumerate(self, **cfg) -> Result:
        return mbe_enumerate(self.handle, make_config(**cfg))

    def enumerate_per_root(self, candidate_side: int = 0, **cfg) -> Tuple[Result, np.ndarray]:
        """Result plus per level-1-subtree (count, hash, tasks, pruned) by candidate ORIGINAL id."""
        side = candidate_side or (2 if self.n2 < self.n1 else 1)
        n = self.n1 if side == 1 else self.n2
        pr = np.zeros((max(n, 1), 4), dtype=np.uint64)
        r = mbe_enumerate(self.handle, make_config(candidate_side=side, per_root=pr, **cfg))
        return r, pr[:n]

    def enumerate_list(self, cap_records: int = 1 << 20, cap_ids: int = 1 << 24, **cfg
                       ) -> Tuple[Result, List[Tuple[tuple, tuple]]]:
        """Bounded listing: (result, [(A side-1 ids, B side-2 ids), ...])."""
        out, (rec_off, n1, n2, ids) = make_output(cap_records, cap_ids)
        r = mbe_enumerate(self.handle, make_config(**cfg), out)
        recs = []
        for k in range(r.records_written):
            o, a, b = int(rec_off[k]), int(n1[k]), int(n2[k])
            recs.append((tuple(int(v) for v in ids[o:o + a]), tuple(int(v) for v in ids[o + a:o + a + b])))
        return r, recs

    def enumerate_text(self, cap_records: int = 1 << 20, cap_ids: int = 1 << 24, **cfg) -> Tuple[Result, bytes]:
        """Bounded listing as canonical text (mbe_format_listing)."""
        out, keep = make_output(cap_records, cap_ids)
        r = mbe_enumerate(self.handle, make_config(**cfg), out)
        text = mbe_format_listing(out, r.records_written)
        del keep
        return r, text

    def close(self):
        if self.handle:
            mbe_free(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
