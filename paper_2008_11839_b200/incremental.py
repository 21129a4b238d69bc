"""Batch-incremental connectivity (reference driver.py:544-725).

``incremental(init, spec, batches, ...)`` keeps connlab's signature and
semantics (insert sub-phase, barrier, query sub-phase; lazy sentinel
initialisation; racy mode; ``on_batch`` state hook).  ``IncrementalConnectivity``
is the columnar device-resident form the throughput path uses: batches are
(u, v) tensors instead of per-op Python objects (SURVEY hard part 9).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .api import LoweredSpec, RunStats, _require_cuda, _stream, host_int64
from .errors import ConfigError
from .graph import Graph
from .spec import AlgorithmSpec, FinishKind, SpliceOp, format_spec


def _torch():
    import torch
    return torch


@dataclass(frozen=True)
class Insert:
    u: int
    v: int


@dataclass(frozen=True)
class Query:
    u: int
    v: int


def _check_incremental(spec: AlgorithmSpec, racy: bool) -> None:
    if not spec.incremental_capable():
        raise ConfigError(f"incremental needs a root-based finish; '{format_spec(spec)}' is not supported")
    if racy:
        if not spec.is_union_finish():
            raise ConfigError("racy mode interleaves single ops and only works with union-find finishes")
        if spec.cfg.splice is SpliceOp.SPLICE_ATOMIC:
            raise ConfigError("the splice rule moves non-roots across trees mid-union; interleaved "
                              "queries would observe torn components - use the batched (non-racy) mode")


class IncrementalConnectivity:
    """Device-resident incremental state over `capacity` vertex slots."""

    def __init__(self, spec: AlgorithmSpec, capacity: int, racy: bool = False):
        _check_incremental(spec, racy)
        _require_cuda()
        self.spec = spec
        self.capacity = int(capacity)
        self.racy = racy
        lowered = LoweredSpec(spec, None, max(self.capacity, 1))
        self._lowered = lowered
        self._h = C.c_void_p()
        N.check(N.lib().gc_incr_create(self.capacity, C.byref(lowered.s), _stream(), C.byref(self._h)))
        self.stats = N.Stats()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.lib().gc_incr_destroy(h)
            except Exception:
                pass
            self._h = None

    def reserve(self, batch_len: int) -> None:
        """Pre-size the round finishes' per-batch buffers (gc_incr_reserve)."""
        N.check(N.lib().gc_incr_reserve(self._h, int(batch_len)))

    def insert(self, us, vs, sync: bool = True) -> None:
        """Insert-only batch (columnar device tensors, int32).  sync=False
        (union-find specs): enqueue only; later queries / labels order after
        it, and the caller keeps us / vs alive until then."""
        n = int(us.numel())
        fn = N.lib().gc_incr_insert if sync else N.lib().gc_incr_insert_async
        N.check(fn(self._h, us.data_ptr() if n else None, vs.data_ptr() if n else None, n, C.byref(self.stats)))

    def insert_list(self, us, vs):
        """Insert-only batch that also returns the edges that merged two trees
        (the exchange unit of the sharded driver; root-based rules only)."""
        torch = _torch()
        n = int(us.numel())
        ou = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        ov = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        if n:
            N.check(N.lib().gc_incr_insert_list(self._h, us.data_ptr(), vs.data_ptr(), n, ou.data_ptr(),
                                                ov.data_ptr(), cnt.data_ptr(), C.byref(self.stats)))
        c = int(cnt.item())
        return ou[:c], ov[:c]

    def query(self, us, vs):
        """Query-only batch; returns a uint8 CUDA tensor of connected bits."""
        torch = _torch()
        n = int(us.numel())
        bits = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
        N.check(N.lib().gc_incr_query(self._h, us.data_ptr() if n else None,
                                      vs.data_ptr() if n else None, n, bits.data_ptr(),
                                      C.byref(self.stats)))
        return bits[:n]

    def batch(self, us, vs, is_query):
        """Mixed batch in reference order; returns uint8 bits (1 = connected query)."""
        torch = _torch()
        n = int(us.numel())
        bits = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
        if n:
            N.check(N.lib().gc_incr_batch(self._h, us.data_ptr(), vs.data_ptr(), is_query.data_ptr(), n,
                                          bits.data_ptr(), int(self.racy), C.byref(self.stats)))
        return bits[:n]

    def state(self):
        """Copy of the live state with the sentinel convention (driver.py:656, 710)."""
        torch = _torch()
        slots = self.capacity if self.spec.is_union_finish() else self.capacity + 1
        out = torch.empty(max(slots, 1), dtype=torch.int32, device="cuda")
        N.check(N.lib().gc_incr_state(self._h, out.data_ptr()))
        return out[:slots]

    def labels(self):
        """(finalized int32 labels tensor, component count of initialised vertices)."""
        torch = _torch()
        out = torch.empty(max(self.capacity, 1), dtype=torch.int32, device="cuda")
        comps = C.c_int64(0)
        N.check(N.lib().gc_incr_labels(self._h, out.data_ptr(), C.byref(comps)))
        return out[: self.capacity], int(comps.value)


def incremental(init, spec: AlgorithmSpec, batches, workers=1, capacity=None, racy=False,
                on_batch=None):
    """driver.py:567-725: returns (np.int64 labels, [np.bool_ bits per batch], RunStats)."""
    _check_incremental(spec, racy)
    torch = _torch()
    batches = [list(b) for b in batches]
    cap = capacity or 0
    if init is not None:
        cap = max(cap, init.n)
    for b in batches:
        for op in b:
            cap = max(cap, op.u + 1, op.v + 1)
    inc = IncrementalConnectivity(spec, cap, racy=racy)
    stats = RunStats()
    if spec.finish is FinishKind.JTB:
        stats.notes.append("reference-approximate")
    # the initial graph is an untimed insert-only prologue (driver.py:651-654)
    if init is not None and init.m:
        ue = init.undirected_edges()
        inc.insert(torch.from_numpy(ue[:, 0].astype(np.int32)).to("cuda"),
                   torch.from_numpy(ue[:, 1].astype(np.int32)).to("cuda"))
        inc.stats = N.Stats()
    results = []
    for bi, batch in enumerate(batches):
        k = len(batch)
        us = np.fromiter((op.u for op in batch), dtype=np.int32, count=k)
        vs = np.fromiter((op.v for op in batch), dtype=np.int32, count=k)
        isq = np.fromiter((isinstance(op, Query) for op in batch), dtype=np.uint8, count=k)
        if k:
            bits = inc.batch(torch.from_numpy(us).to("cuda"), torch.from_numpy(vs).to("cuda"),
                             torch.from_numpy(isq).to("cuda"))
            results.append(bits.cpu().numpy().astype(bool))
        else:
            results.append(np.zeros(0, dtype=bool))
        if on_batch is not None:
            on_batch(bi, host_int64(inc.state()))
    labels, comps = inc.labels()
    st = inc.stats
    stats.phase_times = {"insert": st.t_sample_ms / 1e3, "query": st.t_finish_ms / 1e3}
    stats.edge_inspections = {"insert": int(st.insp_finish)} if st.insp_finish else {}
    stats.rounds = int(st.rounds)
    stats.component_count = comps
    return host_int64(labels), results, stats
