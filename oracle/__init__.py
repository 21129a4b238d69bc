"""CPU oracle for the GConn hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
reference arm may import this package, and only as the checker or the
measured CPU baseline — never as the product path.  It wraps
gconn_oracle.c, a plain-C restatement of the reference connlab algorithms
(file:line citations in the C source), whose parity is pinned by
tests/test_oracle.py against fixtures produced by the reference itself.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "libgconn_oracle.so"
_lib = None


def build() -> Path:
    subprocess.run(["sh", str(HERE / "build.sh")], check=True, capture_output=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        h = C.CDLL(str(LIB))
        P = C.c_void_p
        h.or_gen_rmat.argtypes = [C.c_int, C.c_int64, P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, P, P]
        h.or_build_csr.argtypes = [C.c_int64, P, P, C.c_int64, P, P]
        h.or_build_csr.restype = C.c_int64
        h.or_components.argtypes = [C.c_int64, P, P, P]
        h.or_components.restype = C.c_int64
        h.or_check_forest.argtypes = [C.c_int64, P, P, P, P, P, P, P]
        h.or_incremental_replay.argtypes = [C.c_int64, P, P, P, C.c_int64, C.c_int64, P, P]
        _lib = h
    return _lib


def _p(a):
    return a.ctypes.data if a.size else None


def pcg_state(seed: int):
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return (s >> 64) & m, s & m, (inc >> 64) & m, inc & m


def gen_rmat(scale, edge_factor, a=0.5, b=0.1, c=0.1, seed=0):
    """graphs.py:210-245 restated in C; returns (n, edges int64 (m, 2))."""
    n = 1 << scale
    m = edge_factor * n
    base = (C.c_double * 4)(a, b, c, 1.0 - a - b - c)
    src = np.zeros(m, dtype=np.int64)
    dst = np.zeros(m, dtype=np.int64)
    lib().or_gen_rmat(scale, m, base, *pcg_state(seed), _p(src), _p(dst))
    return n, np.column_stack((src, dst))


def build_csr(n, edges):
    """graphs.py:90-121 restated in C; returns (offsets int64, targets int32)."""
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int64).reshape(-1, 2))
    src = np.ascontiguousarray(e[:, 0])
    dst = np.ascontiguousarray(e[:, 1])
    off = np.zeros(n + 1, dtype=np.int64)
    tgt = np.zeros(max(2 * len(e), 1), dtype=np.int32)
    m = lib().or_build_csr(n, _p(src), _p(dst), len(e), _p(off), tgt.ctypes.data)
    if m < 0:
        raise ValueError(f"edge {-m - 1} has an endpoint outside [0, {n})")
    return off, tgt[:m].copy()


def components(n, off, tgt):
    """Canonical component-minimum labels (validate.py:74-122); returns (labels, count)."""
    off = np.ascontiguousarray(off, dtype=np.int64)
    tgt = np.ascontiguousarray(tgt, dtype=np.int32)
    lab = np.zeros(max(n, 1), dtype=np.int32)
    c = lib().or_components(n, _p(off), _p(tgt), lab.ctypes.data)
    return lab[:n].astype(np.int64), int(c)


def check_forest(n, off, tgt, fu, fv, oracle_labels) -> dict:
    """The four clauses of validate.py:178-244."""
    off = np.ascontiguousarray(off, dtype=np.int64)
    tgt = np.ascontiguousarray(tgt, dtype=np.int32)
    fu = np.ascontiguousarray(fu, dtype=np.int32)
    fv = np.ascontiguousarray(fv, dtype=np.int32)
    o = np.ascontiguousarray(oracle_labels, dtype=np.int32)
    out = np.zeros(4, dtype=np.int32)
    wit = np.zeros(2, dtype=np.int64)
    lib().or_check_forest(n, _p(off), _p(tgt), _p(fu), _p(fv), _p(o), out.ctypes.data, wit.ctypes.data)
    names = ["edges_exist", "acyclic", "count", "components_match"]
    rep = {"passed": bool(out.all()), "clauses": {k: {"ok": bool(v)} for k, v in zip(names, out)},
           "witness": wit.tolist()}
    return rep


def incremental_replay(cap, us, vs, isq, batch):
    """SequentialUF (validate.py:125-155) with batch barriers (driver.py:695-708)."""
    us = np.ascontiguousarray(us, dtype=np.int32)
    vs = np.ascontiguousarray(vs, dtype=np.int32)
    isq = np.ascontiguousarray(isq, dtype=np.uint8)
    bits = np.zeros(max(len(us), 1), dtype=np.uint8)
    lab = np.zeros(max(cap, 1), dtype=np.int32)
    lib().or_incremental_replay(cap, _p(us), _p(vs), _p(isq), len(us), batch, bits.ctypes.data,
                                lab.ctypes.data)
    return bits[:len(us)].astype(bool), lab[:cap].astype(np.int64)


_UNION = {"async": 0, "rem_cas": 4}
_FIND = {"naive": 0, "split": 1, "halve": 2, "compress": 3}
_SPLICE = {"none": 0, "split": 1, "halve": 2, "splice": 3}


def max_threads() -> int:
    h = lib()
    h.or_max_threads.restype = C.c_int
    return int(h.or_max_threads())


def static_uf(n, off, tgt, sample="kout", k=2, union="rem_cas", find="halve", splice="splice",
              threads=0):
    """CPU port of the union-find static pipeline (driver.py:454-500) — the
    bench.py CPU baseline.  Returns (labels int32, stats dict, (t_sample, t_finish, t_finalize))."""
    h = lib()
    h.or_static_uf.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                               C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    off = np.ascontiguousarray(off, dtype=np.int64)
    tgt = np.ascontiguousarray(tgt, dtype=np.int32)
    P = np.empty(max(n, 1), dtype=np.int32)
    st = np.zeros(8, dtype=np.int64)
    tm = np.zeros(3, dtype=np.float64)
    h.or_static_uf(n, _p(off), _p(tgt), {"none": 0, "kout": 1}[sample], k, _UNION[union], _FIND[find],
                   _SPLICE[splice], threads, P.ctypes.data, st.ctypes.data, tm.ctypes.data)
    return P[:n], {"insp_sample": int(st[0]), "insp_finish": int(st[1]), "l_max": int(st[2]),
                   "components": int(st[3]), "active": int(st[4])}, tuple(tm.tolist())
