"""Validation helpers of the reference API (validate.py:74-298), B200-side.

``check_forest`` keeps the reference's four clauses and report format
(validate.py:178-244) but evaluates them with libgconn kernels, so it
finishes in milliseconds at BASELINE sizes (the reference's per-edge Python
loops take ~25 s at n = 2^22):

  (a) edges_exist      — binary search of every recorded edge in its CSR row
  (b) acyclic          — union the recorded edges into fresh sets; an edge
                         that does not merge two trees closes a cycle
  (c) count            — populated slots = n - #components(oracle)
  (d) components_match — forest components vs the oracle partition

``partition_equal``, ``canonical_labels`` and ``sampling_stats`` are the
reference's host-side census definitions restated over numpy.
``oracle_components`` / ``oracle_components_unionfind`` return canonical
labels from two independent device routes (label-propagation rounds and
sequential-order-free union-find) for cross-checking; the test-suite's
ground truth remains the C oracle under ``oracle/``.
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _native as N
from .api import _csr, _require_cuda, _stream, _workspace, host_int64, static_connectivity_device
from .errors import MalformedInputError
from .graph import Graph
from .spec import parse_spec


def _torch():
    import torch
    return torch


# ------------------------------------------------------------- host census

def partition_equal(a, b) -> bool:
    """validate.py:158-172: same partition irrespective of label values."""
    a = np.asarray(a, dtype=np.int64)
    b = np.asarray(b, dtype=np.int64)
    if a.shape != b.shape:
        return False
    if len(a) == 0:
        return True
    pairs = (a << np.int64(32)) | (b & np.int64(0xFFFFFFFF))
    return len(np.unique(a)) == len(np.unique(pairs)) == len(np.unique(b))


def canonical_labels(labels) -> np.ndarray:
    """validate.py:251-259: each class relabelled by its minimum member."""
    labels = np.asarray(labels, dtype=np.int64)
    n = len(labels)
    if n == 0:
        return labels.copy()
    mins = np.full(n, n, dtype=np.int64)
    np.minimum.at(mins, labels, np.arange(n, dtype=np.int64))
    return mins[labels]


def sampling_stats(g: Graph, post_sample_labels, oracle=None) -> tuple[float, float]:
    """validate.py:267-298: (cov, ic) census of post-sampling labels; with an
    oracle, asserts that the sampled partition refines it."""
    labels = np.asarray(post_sample_labels, dtype=np.int64)
    n = g.n
    if n == 0:
        return 1.0, 0.0
    counts = np.bincount(labels, minlength=n)
    mode = int(counts.argmax())
    cov = counts[mode] / n
    if g.m == 0:
        ic = 0.0
    else:
        src = np.repeat(np.arange(n, dtype=np.int64), g.degrees)
        ic = float(np.count_nonzero(labels[src] != labels[g.targets])) / g.m
    if oracle is not None:
        oracle = np.asarray(oracle, dtype=np.int64)
        order = np.argsort(labels, kind="stable")
        ls, os_ = labels[order], oracle[order]
        same_class = ls[1:] == ls[:-1]
        if np.any(same_class & (os_[1:] != os_[:-1])):
            raise AssertionError("post-sampling labels merge distinct true components")
    return float(cov), float(ic)


# ------------------------------------------------------------ device routes

def oracle_components(g: Graph) -> np.ndarray:
    """Canonical component labels by label-propagation rounds (no union-find
    on this route; validate.py:74-98 uses a BFS flood for the same reason)."""
    labels, _ = static_connectivity_device(g, parse_spec("none+lp"), metrics=False)
    return host_int64(labels)


def oracle_components_unionfind(g: Graph) -> np.ndarray:
    """Canonical labels by asynchronous union-find with full compression
    (validate.py:101-122's second, independent route)."""
    labels, _ = static_connectivity_device(g, parse_spec("none+async+compress"), metrics=False)
    return host_int64(labels)


def _forest_pairs(forest):
    """(us, vs) int32 CUDA tensors from ForestEdges / DeviceForest / a list."""
    torch = _torch()
    fu = getattr(forest, "fu", None)
    if fu is not None and isinstance(fu, torch.Tensor):
        keep = forest.fu >= 0
        return forest.fu[keep].to("cuda", torch.int32), forest.fv[keep].to("cuda", torch.int32)
    edges = forest.edges if hasattr(forest, "edges") else forest
    pairs = np.array([e for e in edges if e is not None], dtype=np.int64).reshape(-1, 2)
    t = torch.from_numpy(pairs.astype(np.int32)).to("cuda")
    return t[:, 0].contiguous(), t[:, 1].contiguous()


def check_forest(g: Graph, forest, oracle) -> dict:
    """validate.py:178-244: the four forest clauses with witnesses."""
    _require_cuda()
    torch = _torch()
    n = g.n
    us, vs = _forest_pairs(forest)
    k = int(us.numel())
    report: dict = {"passed": True, "clauses": {}}

    def clause(name, ok, witness=None):
        entry = {"ok": bool(ok)}
        if not ok:
            entry["witness"] = witness
            report["passed"] = False
        report["clauses"][name] = entry

    lib = N.lib()
    # (a) every recorded edge exists in E
    csr, keep = _csr(g)
    miss = torch.zeros(1, dtype=torch.int64, device="cuda")
    N.check(lib.gc_edges_exist(C.byref(csr), us.data_ptr() if k else None, vs.data_ptr() if k else None, k,
                               miss.data_ptr(), _stream()))
    mi = int(miss.item()) if k else -1  # UINT64_MAX reads back as -1
    ok_a = mi < 0
    clause("edges_exist", ok_a, None if ok_a else (int(us[mi].item()), int(vs[mi].item())))

    # (b) acyclic: recorded edges unioned in order into fresh sets
    if k and (us.min().item() < 0 or vs.min().item() < 0 or us.max().item() >= n or vs.max().item() >= n):
        raise MalformedInputError("forest endpoint outside [0, n)")
    spec = N.Spec()
    spec.finish = N.FINISH["async"]
    spec.find = N.FIND["halve"]
    mu = torch.empty(max(k, 1), dtype=torch.int32, device="cuda")
    mv = torch.empty(max(k, 1), dtype=torch.int32, device="cuda")

    def merges(p: int):
        """Union the first p recorded edges into fresh sets: (parent, #merging)."""
        par = torch.arange(max(n, 1), dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        if p:
            N.check(lib.gc_union_edges_list(par.data_ptr(), n, us.data_ptr(), vs.data_ptr(), p, C.byref(spec),
                                            None, mu.data_ptr(), mv.data_ptr(), cnt.data_ptr(), _stream()))
        return par, int(cnt.item())

    parent, merged = merges(k)
    witness = None
    if merged != k:
        # the reference's witness is the first edge (slot order) whose
        # endpoints the earlier edges already join: the shortest cyclic
        # prefix, found by bisection over prefix lengths
        lo, hi = 1, k  # prefix hi is cyclic, prefix lo - 1 is not
        while lo < hi:
            mid = (lo + hi) // 2
            if merges(mid)[1] != mid:
                hi = mid
            else:
                lo = mid + 1
        witness = (int(us[lo - 1].item()), int(vs[lo - 1].item()))
        # the reference stops its union loop at that edge (validate.py:219-226),
        # so clause (d) sees the components of the acyclic prefix only
        parent, _ = merges(lo - 1)
    clause("acyclic", merged == k, witness)

    # (c) populated slot count = n - component count
    orc = np.asarray(oracle, dtype=np.int64)
    component_count = len(np.unique(orc)) if n else 0
    expected = n - component_count
    clause("count", k == expected, {"populated": k, "expected": expected})

    # (d) forest components match the oracle partition
    if n:
        ws = _workspace(4 * n + 8192)
        N.check(lib.gc_label_finalization(parent.data_ptr(), n, ws.data_ptr(), ws.numel(), _stream()))
        orc_d = torch.from_numpy(orc.astype(np.int32)).to("cuda")
        N.check(lib.gc_canonical_labels(orc_d.data_ptr(), n, ws.data_ptr(), ws.numel(), _stream()))
        diff = torch.nonzero(parent[:n] != orc_d).flatten()
        same = diff.numel() == 0
        clause("components_match", same, None if same else {"vertex": int(diff[0].item())})
    else:
        clause("components_match", True)
    return report


def report_to_json(report: dict) -> str:
    return json.dumps(report, indent=2, sort_keys=True)
