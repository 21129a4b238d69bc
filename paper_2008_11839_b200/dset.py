"""DisjointSets and the batch union seam on the device (reference dset.py:346-416).

``DisjointSets`` keeps the reference constructor and probes — ``union``,
``find_root``, ``same_set``, ``record``, ``labels_array`` — over an int32
parent array in HBM.  ``union_edge_list`` is the reference's batch seam
(dset.py:402-416): one libgconn launch applies the configured union rule to
every pair concurrently (``gc_union_edges``), so ``workers`` only exists for
signature compatibility.  Single-pair calls are correct but pay one launch
each; batch through ``union_edge_list`` for throughput.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .api import _require_cuda, _stream, host_int64, jtb_ranks
from .errors import ConfigError, MalformedInputError
from .spec import AlgorithmSpec, FinishKind, SampleKind, UnionConfig, UnionOp, valid_combination

_JTB_RANK_SEED = 0x1234  # dset.py:343


def _torch():
    import torch
    return torch


def _as_device_i32(x, n: int):
    """Endpoints as a contiguous int32 CUDA tensor.  Host inputs are range
    checked here; device tensors by gc_union_edges itself (MalformedInputError
    either way, before any union runs)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        if x.dtype.is_floating_point or x.dtype is torch.bool:
            raise MalformedInputError(f"endpoints must be integer ids, not {x.dtype}")
        if x.dtype is torch.int64 and x.numel():
            lo, hi = torch.aminmax(x)
            if int(lo) < 0 or int(hi) >= n:  # narrowing to int32 would wrap
                raise MalformedInputError(f"endpoint outside [0, {n})")
        t = x.reshape(-1).to("cuda", torch.int32)
    else:
        a = np.asarray(x, dtype=np.int64).reshape(-1)
        if a.size and (a.min() < 0 or a.max() >= n):
            raise MalformedInputError(f"endpoint outside [0, {n})")
        t = torch.from_numpy(a.astype(np.int32)).to("cuda")
    return t.contiguous()


class DisjointSets:
    """Shared union-find state plus the configured rule (dset.py:346-399).

    ``forest``, when given, is a length-n list that receives the original
    (u, v) pair at slot r when root r is hooked away; on the device the slots
    live in two int32 arrays and are copied into the list after every batch.
    ``threaded`` is accepted for compatibility: device CAS is always atomic.
    """

    def __init__(self, n, cfg: UnionConfig, threaded=False, seed=_JTB_RANK_SEED, forest=None):
        if not valid_combination(cfg):
            raise ConfigError(f"unsupported union-find combination: {cfg}")
        _require_cuda()
        torch = _torch()
        self.n = int(n)
        self.cfg = cfg
        self.forest = forest
        self.p = torch.arange(self.n, dtype=torch.int32, device="cuda")
        self._aux = None
        if cfg.union is UnionOp.HOOKS:
            self._aux = torch.full((max(self.n, 1),), self.n, dtype=torch.int32, device="cuda")
        elif cfg.union is UnionOp.REM_LOCK:
            self._aux = torch.zeros(max(self.n, 1), dtype=torch.int32, device="cuda")
        self._spec = N.Spec()
        self._spec.sample = N.SAMPLE[SampleKind.NONE.value]
        self._spec.finish = N.FINISH[cfg.union.value]
        self._spec.find = N.FIND[cfg.find.value]
        self._spec.splice = N.SPLICE[cfg.splice.value]
        self._ranks = None
        if cfg.union is UnionOp.JTB:
            self._ranks = jtb_ranks(self.n, seed).clone()
            self._spec.jtb_ranks = self._ranks.data_ptr()
        self._fu = self._fv = None
        if forest is not None:
            if len(forest) != self.n:
                raise MalformedInputError("forest must have one slot per vertex")
            if cfg.splice.value == "splice":
                raise ConfigError("atomic splice is not root-based: no forest recording")
            self._fu = torch.full((max(self.n, 1),), -1, dtype=torch.int32, device="cuda")
            self._fv = torch.full((max(self.n, 1),), -1, dtype=torch.int32, device="cuda")

    # ------------------------------------------------------------ batch seam
    def union_batch(self, us, vs) -> None:
        us = _as_device_i32(us, self.n)
        vs = _as_device_i32(vs, self.n)
        if us.numel() != vs.numel():
            raise MalformedInputError("us and vs differ in length")
        k = int(us.numel())
        if k == 0:
            return
        N.check(N.lib().gc_union_edges(
            self.p.data_ptr(), self.n, us.data_ptr(), vs.data_ptr(), k, C.byref(self._spec),
            self._aux.data_ptr() if self._aux is not None else None,
            self._fu.data_ptr() if self._fu is not None else None,
            self._fv.data_ptr() if self._fv is not None else None, _stream()))
        self._sync_forest()

    def _sync_forest(self) -> None:
        if self.forest is None:
            return
        fu = self._fu[:self.n].cpu().numpy()
        fv = self._fv[:self.n].cpu().numpy()
        for r in np.flatnonzero(fu >= 0):
            self.forest[int(r)] = (int(fu[r]), int(fv[r]))

    # ---------------------------------------------------------- single ops
    def union(self, u: int, v: int) -> bool:
        """dset.py:381-382: True iff this call merged two sets.  A lone union
        merges exactly when the endpoints were in different sets before it."""
        if not (0 <= u < self.n and 0 <= v < self.n):
            raise MalformedInputError(f"endpoint outside [0, {self.n})")
        before = self.same_set(u, v)
        self.union_batch([u], [v])
        return not before

    def _find(self, xs, kind: str):
        torch = _torch()
        xs = _as_device_i32(xs, self.n)
        roots = torch.empty_like(xs)
        if xs.numel():
            N.check(N.lib().gc_find_batch(self.p.data_ptr(), self.n, xs.data_ptr(), xs.numel(),
                                          N.FIND[kind], roots.data_ptr(), _stream()))
        return roots

    def find_root(self, u: int) -> int:
        """dset.py:384-385: the root, applying the configured compaction."""
        find = self.cfg.find.value
        return int(self._find([u], find)[0].item())

    def same_set(self, u: int, v: int) -> bool:
        """dset.py:387-389: read-only connectivity probe (no compression writes)."""
        r = self._find([u, v], "naive").cpu().numpy()
        return bool(r[0] == r[1])

    def record(self, slot: int, u: int, v: int) -> None:
        if self.forest is not None:
            self.forest[slot] = (u, v)
            self._fu[slot] = u
            self._fv[slot] = v

    def labels_array(self):
        """dset.py:395-399: np.int64 root of every vertex (read-only walk)."""
        torch = _torch()
        if self.n == 0:
            return np.zeros(0, dtype=np.int64)
        roots = torch.empty(self.n, dtype=torch.int32, device="cuda")
        N.check(N.lib().gc_find_batch(self.p.data_ptr(), self.n, None, self.n, N.FIND["naive"],
                                      roots.data_ptr(), _stream()))
        return host_int64(roots)


def union_edge_list(ds: DisjointSets, us, vs, workers=1) -> None:
    """dset.py:402-416: apply ds.union over parallel endpoint lists — one
    concurrent device launch (``workers`` is accepted and ignored)."""
    ds.union_batch(us, vs)


def spec_for(cfg: UnionConfig) -> AlgorithmSpec:
    """The unsampled static spec that runs ``cfg`` as its finish."""
    return AlgorithmSpec(sample=SampleKind.NONE, finish=FinishKind(cfg.union.value), cfg=cfg)
