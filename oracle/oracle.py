"""ctypes wrapper of oracle/mbea_oracle.cpp (TEST INFRASTRUCTURE ONLY).

Takes the row-CSR arrays produced by paper_2401_05039_b200.inputs (the only
module both sides share) and runs the plain Algorithm 1 oracle.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mbea_oracle.cpp")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile liboracle.so with g++ (plain -O2; no product code involved)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", _SRC, "-o", tmp])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build_oracle())
            u32, u64, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
            p64, p32 = ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32)
            lib.oracle_mbea.argtypes = [u32, u32, p64, p32, i32, i32, i32, i32, p64]
            lib.oracle_mbea.restype = i32
            lib.oracle_mbea_roots.argtypes = [u32, u32, p64, p32, i32, i32, i32, p32, u64, p64]
            lib.oracle_mbea_roots.restype = i32
            lib.oracle_mbea_list.argtypes = [u32, u32, p64, p32, i32, i32, p32, u64]
            lib.oracle_mbea_list.restype = ctypes.c_int64
            lib.oracle_mbea_plain.argtypes = [u32, u32, p64, p32, i32, i32, p64]
            lib.oracle_mbea_plain.restype = i32
            lib.oracle_mix64.argtypes = [u64]
            lib.oracle_mix64.restype = u64
            _lib = lib
    return _lib


_ORDERS = {"ascending": 0, "input": 1, "descending": 2}


@dataclasses.dataclass
class OracleResult:
    count: int
    hash: int
    tasks: int
    pruned: int
    bad: int
    threads: int


def _arrays(g):
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.uint64)
    ci = np.ascontiguousarray(g.col_idx, dtype=np.uint32)
    if ci.size == 0:
        ci = np.zeros(1, dtype=np.uint32)
    return rp, ci


def _p64(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def _p32(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def mbea(g, candidate_side: int = 0, order: str = "ascending", threads: int = 0,
         check: bool = False) -> OracleResult:
    """Full enumeration: count, hash, search-tree tasks / pruned tasks."""
    lib = _load()
    rp, ci = _arrays(g)
    out = np.zeros(6, dtype=np.uint64)
    rc = lib.oracle_mbea(g.n1, g.n2, _p64(rp), _p32(ci), candidate_side, _ORDERS[order],
                         threads, 1 if check else 0, _p64(out))
    if rc:
        raise ValueError(f"oracle_mbea: error {rc}")
    return OracleResult(*[int(v) for v in out])


def mbea_plain(g, candidate_side: int = 0, order: str = "ascending") -> OracleResult:
    """Sequential literal MBEA(V, ∅, P, ∅) with closure checks (small graphs)."""
    lib = _load()
    rp, ci = _arrays(g)
    out = np.zeros(6, dtype=np.uint64)
    rc = lib.oracle_mbea_plain(g.n1, g.n2, _p64(rp), _p32(ci), candidate_side,
                               _ORDERS[order], _p64(out))
    if rc:
        raise ValueError(f"oracle_mbea_plain: error {rc}")
    return OracleResult(*[int(v) for v in out])


def mbea_roots(g, roots, candidate_side: int = 0, order: str = "ascending", threads: int = 0) -> np.ndarray:
    """Per-root (count, hash, tasks, pruned) for candidate-side ORIGINAL ids ``roots``."""
    lib = _load()
    rp, ci = _arrays(g)
    roots = np.ascontiguousarray(roots, dtype=np.uint32)
    out = np.zeros((max(len(roots), 1), 4), dtype=np.uint64)
    rc = lib.oracle_mbea_roots(g.n1, g.n2, _p64(rp), _p32(ci), candidate_side,
                               _ORDERS[order], threads, _p32(roots), len(roots), _p64(out))
    if rc:
        raise ValueError(f"oracle_mbea_roots: error {rc}")
    return out[: len(roots)]


def mbea_list(g, candidate_side: int = 0, order: str = "ascending"):
    """Set of maximal bicliques as frozenset of (tuple(A side-1 ids), tuple(B side-2 ids))."""
    lib = _load()
    rp, ci = _arrays(g)
    cap = 1 << 16
    while True:
        buf = np.zeros(cap, dtype=np.uint32)
        n = lib.oracle_mbea_list(g.n1, g.n2, _p64(rp), _p32(ci), candidate_side,
                                 _ORDERS[order], _p32(buf), cap)
        if n < 0:
            raise ValueError(f"oracle_mbea_list: error {n}")
        if n <= cap:
            break
        cap = int(n)
    out = []
    k = 0
    while k < n:
        a, b = int(buf[k]), int(buf[k + 1])
        A = tuple(int(v) for v in buf[k + 2: k + 2 + a])
        B = tuple(int(v) for v in buf[k + 2 + a: k + 2 + a + b])
        out.append((A, B))
        k += 2 + a + b
    return out


def mix64(z: int) -> int:
    return int(_load().oracle_mix64(z & 0xFFFFFFFFFFFFFFFF))
