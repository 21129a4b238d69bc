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

``canonical_labels``, ``partition_equal`` and ``sampling_stats`` keep the
reference's definitions and run as device passes (``gc_canonical_labels``,
``gc_label_census``: a histogram mode, a crossing-edge count and a
refinement check against an oracle labelling).  ``oracle_components`` /
``oracle_components_unionfind`` are two host routes that share no code with
libgconn (scipy's traversal; numpy min-hooking + pointer jumping), so
checking the device against them is a real check; the test-suite's ground
truth remains the C oracle under ``oracle/`` and the reference fixtures.
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _native as N
from .api import _csr, _require_cuda, _stream, _workspace, host_int64
from .errors import MalformedInputError
from .graph import Graph


def _torch():
    import torch
    return torch


# ---------------------------------------------------------- device census

def _dense_ids(labels) -> np.ndarray:
    """Any labelling as int32 ids in [0, n) inducing the same partition (the
    device kernels index with label values; the reference accepts any
    int64 values)."""
    a = np.asarray(labels, dtype=np.int64).reshape(-1)
    n = len(a)
    if n == 0 or (a.min() >= 0 and a.max() < n):
        return a.astype(np.int32)
    _, inv = np.unique(a, return_inverse=True)
    return inv.astype(np.int32)


def _canonical_device(labels):
    """gc_canonical_labels on a dense int32 device copy (values become each
    class's minimum member)."""
    torch = _torch()
    dense = _dense_ids(labels)
    n = len(dense)
    t = torch.from_numpy(dense).to("cuda")
    if n:
        ws = _workspace(4 * n + 8192)
        N.check(N.lib().gc_canonical_labels(t.data_ptr(), n, ws.data_ptr(), ws.numel(), _stream()))
    return t


def canonical_labels(labels) -> np.ndarray:
    """validate.py:251-259: relabel every class by its minimum member
    (device: one atomic-min pass per class, then a gather)."""
    _require_cuda()
    return host_int64(_canonical_device(labels))


def partition_equal(a, b) -> bool:
    """validate.py:158-170: do two labellings induce the same partition?
    Two labellings are the same partition exactly when their canonical
    (minimum-member) forms are equal element for element."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        return False
    if a.size == 0:
        return True
    _require_cuda()
    torch = _torch()
    return bool(torch.equal(_canonical_device(a), _canonical_device(b)))


def label_census(g: Graph, labels, oracle=None) -> dict:
    """gc_label_census: the most frequent label and its count, the
    label-crossing directed edges, and (with an oracle) the first vertex
    whose class is not inside one oracle class (or -1)."""
    _require_cuda()
    torch = _torch()
    lab = torch.from_numpy(_dense_ids(labels) if not hasattr(labels, "data_ptr") else labels.cpu().numpy()
                           .astype(np.int32)).to("cuda")
    if lab.numel() != g.n:
        raise MalformedInputError(f"labels must have length n={g.n}")
    orc = None
    if oracle is not None:
        orc = torch.from_numpy(_dense_ids(oracle)).to("cuda")
    csr, keep = _csr(g)
    ws = _workspace(4 * g.n + 8192)
    out = (C.c_int64 * 4)()
    N.check(N.lib().gc_label_census(C.byref(csr), lab.data_ptr() if g.n else None,
                                    orc.data_ptr() if orc is not None and g.n else None, out, ws.data_ptr(),
                                    ws.numel(), _stream()))
    return {"mode": int(out[0]), "mode_count": int(out[1]), "crossing": int(out[2]),
            "first_unrefined": int(out[3])}


def sampling_stats(g: Graph, post_sample_labels, oracle=None) -> tuple[float, float]:
    """validate.py:267-298: (cov, ic) of post-sampling labels — cov = the
    most frequent label's share of the vertices, ic = the share of directed
    edges whose endpoints carry different labels; with an oracle labelling,
    raises AssertionError unless the sampled partition refines it."""
    if g.n == 0:
        return 1.0, 0.0
    c = label_census(g, post_sample_labels, oracle)
    if oracle is not None and c["first_unrefined"] >= 0:
        raise AssertionError("post-sampling labels merge distinct true components "
                             f"(vertex {c['first_unrefined']})")
    cov = c["mode_count"] / g.n
    ic = c["crossing"] / g.m if g.m else 0.0
    return float(cov), float(ic)


# ---------------------------------------------------------- oracle routes

def oracle_components(g: Graph) -> np.ndarray:
    """validate.py:74-98: canonical component labels from a route that
    shares nothing with libgconn — scipy's graph traversal on the host CSR
    (the reference floods with BFS for the same reason), then the
    minimum-member relabelling."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components
    n = g.n
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    off, tgt = g.offsets, g.targets
    a = csr_matrix((np.ones(len(tgt), dtype=np.int8), tgt, off), shape=(n, n))
    _, comp = connected_components(a, directed=False)
    first = np.full(comp.max() + 1, n, dtype=np.int64)
    order = np.arange(n - 1, -1, -1, dtype=np.int64)  # descending: the last write per class is its minimum
    first[comp[order]] = order
    return first[comp]


def oracle_components_unionfind(g: Graph) -> np.ndarray:
    """validate.py:101-122's second, independent route: host-side min-label
    hooking + pointer jumping over the CSR (numpy), to the fixpoint."""
    n = g.n
    lab = np.arange(n, dtype=np.int64)
    if n == 0 or g.m == 0:
        return lab
    src = np.repeat(np.arange(n, dtype=np.int64), g.degrees)
    dst = g.targets.astype(np.int64)
    while True:
        lo = np.minimum(lab[src], lab[dst])
        before = lab.copy()
        np.minimum.at(lab, lab[src], lo)
        np.minimum.at(lab, lab[dst], lo)
        while True:  # jump every vertex to its root
            nxt = lab[lab]
            if np.array_equal(nxt, lab):
                break
            lab = nxt
        if np.array_equal(lab, before):
            return lab


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
