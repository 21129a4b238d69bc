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


_UNION = {"async": 0, "rem_cas": 4, "sv": 6, "lt": 7}
_FIND = {"naive": 0, "split": 1, "halve": 2, "compress": 3}
_SPLICE = {"none": 0, "split": 1, "halve": 2, "splice": 3}
_SAMPLE = {"none": 0, "kout": 1, "bfs": 3}
# minbased.py:58-79 LT_VARIANTS: name -> (connect, update, shortcut, alter)
_LT = {"cusa": (0, 0, 0, 1), "crsa": (0, 1, 0, 1), "pusa": (1, 0, 0, 1), "prsa": (1, 1, 0, 1),
       "pus": (1, 0, 0, 0), "prs": (1, 1, 0, 0), "eusa": (2, 0, 0, 1), "eus": (2, 0, 0, 0),
       "cufa": (0, 0, 1, 1), "crfa": (0, 1, 1, 1), "pufa": (1, 0, 1, 1), "prfa": (1, 1, 1, 1),
       "puf": (1, 0, 1, 0), "prf": (1, 1, 1, 0), "eufa": (2, 0, 1, 1), "euf": (2, 0, 1, 0)}


class _OrSpec(C.Structure):
    _fields_ = [("sample", C.c_int32), ("kout_k", C.c_int32), ("finish", C.c_int32), ("find", C.c_int32),
                ("splice", C.c_int32), ("lt_connect", C.c_int32), ("lt_update", C.c_int32),
                ("lt_shortcut", C.c_int32), ("lt_alter", C.c_int32), ("pad", C.c_int32),
                ("bfs_source", C.c_int64)]


def max_threads() -> int:
    h = lib()
    h.or_max_threads.restype = C.c_int
    return int(h.or_max_threads())


def parse(text: str) -> dict:
    """A connlab spec string (driver.py:197-276) for the spec subset the port
    covers: samplers none / kout / bfs; union-find async / rem_cas with
    their find and splice rules, sv, and every lt_<variant>."""
    parts = text.split("+")
    sample, finish = parts[0], parts[1]
    d = {"sample": sample, "finish": finish, "find": "naive", "splice": "splice"}
    if finish == "async":
        d["find"] = parts[2] if len(parts) > 2 else "naive"
        d["splice"] = "none"
    elif finish == "rem_cas":
        d["find"] = parts[2] if len(parts) > 2 else "naive"
        d["splice"] = parts[3] if len(parts) > 3 else "splice"
    elif finish.startswith("lt_"):
        d["lt"] = finish[3:]
        d["finish"] = "lt"
    elif finish != "sv":
        raise ValueError(f"the C port does not cover finish '{finish}'")
    if sample not in _SAMPLE:
        raise ValueError(f"the C port does not cover sampler '{sample}'")
    return d


def pipeline(n, off, tgt, spec: str, threads=0, forest=False, k=2, bfs_source=-1):
    """CPU port of _pipeline / spanning_forest (driver.py:454-536): returns
    (labels int32, stats dict, (t_sample, t_finish, t_finalize)[, (fu, fv)])."""
    h = lib()
    h.or_pipeline.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.POINTER(_OrSpec), C.c_int, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    d = parse(spec)
    sp = _OrSpec()
    sp.sample = _SAMPLE[d["sample"]]
    sp.kout_k = k
    sp.finish = _UNION[d["finish"]]
    sp.find = _FIND[d["find"]]
    sp.splice = _SPLICE[d["splice"]]
    if d["finish"] == "lt":
        sp.lt_connect, sp.lt_update, sp.lt_shortcut, sp.lt_alter = _LT[d["lt"]]
    sp.bfs_source = bfs_source
    if d["sample"] == "bfs" and bfs_source < 0 and n and len(tgt):
        raise ValueError("BFS sampling needs the source vertex (driver.bfs_source semantics)")
    off = np.ascontiguousarray(off, dtype=np.int64)
    tgt = np.ascontiguousarray(tgt, dtype=np.int32)
    P = np.empty(max(n, 1), dtype=np.int32)
    fu = np.empty(max(n, 1), dtype=np.int32) if forest else None
    fv = np.empty(max(n, 1), dtype=np.int32) if forest else None
    st = np.zeros(8, dtype=np.int64)
    tm = np.zeros(3, dtype=np.float64)
    h.or_pipeline(n, _p(off), _p(tgt), C.byref(sp), threads, P.ctypes.data,
                  fu.ctypes.data if forest else None, fv.ctypes.data if forest else None,
                  st.ctypes.data, tm.ctypes.data)
    stats = {"insp_sample": int(st[0]), "insp_finish": int(st[1]), "l_max": int(st[2]),
             "components": int(st[3]), "active": int(st[4]), "lmax_count": int(st[5]),
             "rounds": int(st[6]), "bfs_levels": int(st[7])}
    out = (P[:n], stats, tuple(tm.tolist()))
    if forest:
        out = out + ((fu[:n], fv[:n]),)
    return out


def static_uf(n, off, tgt, sample="kout", k=2, union="rem_cas", find="halve", splice="splice",
              threads=0):
    """The union-find static pipeline (the bench.py reference arm): returns
    (labels int32, stats dict, (t_sample, t_finish, t_finalize))."""
    text = f"{sample}+{union}+{find}" + (f"+{splice}" if union == "rem_cas" else "")
    return pipeline(n, off, tgt, text, threads, k=k)


def incr_insert(cap, P, us, vs, union="async", find="halve", splice="none", threads=0) -> float:
    """One insert-only batch (driver.py:620-649) into the parent array P
    (cap slots, sentinel cap); returns the seconds it took."""
    h = lib()
    h.or_incr_insert.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                 C.c_int, C.c_int, C.c_void_p]
    us = np.ascontiguousarray(us, dtype=np.int32)
    vs = np.ascontiguousarray(vs, dtype=np.int32)
    sec = C.c_double(0)
    h.or_incr_insert(cap, P.ctypes.data, _p(us), _p(vs), len(us), _UNION[union], _FIND[find], _SPLICE[splice],
                     threads, C.byref(sec))
    return sec.value
