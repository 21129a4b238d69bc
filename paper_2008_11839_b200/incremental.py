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
from .errors import ConfigError, MalformedInputError
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


class PackedBits:
    """Query results as one bit per op, packed LSB-first into 32-bit words
    on the device (gc_incr_query / gc_incr_batch write one __ballot_sync word
    per 32 ops): ``words`` is the int32 CUDA tensor, ``numpy()`` unpacks to
    the reference's per-op bool array (driver.py:658-668) on the host."""

    def __init__(self, words, n: int):
        self.words = words
        self.n = int(n)

    def __len__(self) -> int:
        return self.n

    def numpy(self) -> np.ndarray:
        if self.n == 0:
            return np.zeros(0, dtype=bool)
        raw = self.words.cpu().numpy().view(np.uint8)
        return np.unpackbits(raw, bitorder="little")[: self.n].astype(bool)

    def tolist(self) -> list:
        return self.numpy().tolist()


class LiveState:
    """The live incremental state handed to ``on_batch`` (driver.py:710-711
    passes the live parent list / label array, not a copy): a zero-copy view
    of the handle's device array with the sentinel convention.  It exposes
    ``__cuda_array_interface__`` (``torch.as_tensor(state, device="cuda")``
    aliases it) and converts to a host int64 array only when read as numpy
    (``np.asarray(state)``, indexing).  Valid during the callback; later
    batches mutate it.  Writes through the view change the live parent
    array, as in the reference; a write that splits a component (rather
    than merging) would leave the union-find rules' giant-filter bitmap marking
    vertices as connected that no longer are — run such a stream with
    ``GC_INCR_GIANT=0``."""

    def __init__(self, ptr: int, slots: int, owner):
        self._ptr = int(ptr or 0)
        self._slots = int(slots)
        self._owner = owner  # keeps the handle alive while the view exists

    @property
    def __cuda_array_interface__(self):
        # writable, as the reference hands the live (mutable) state; torch
        # rejects read-only device arrays
        return {"shape": (self._slots,), "typestr": "<i4", "data": (self._ptr, False), "version": 3,
                "strides": None}

    def tensor(self):
        torch = _torch()
        if self._slots == 0:
            return torch.empty(0, dtype=torch.int32, device="cuda")
        return torch.as_tensor(self, device="cuda")

    def __len__(self) -> int:
        return self._slots

    def __array__(self, dtype=None, copy=None):
        out = self.tensor().cpu().numpy().astype(np.int64)
        return out if dtype is None else out.astype(dtype)

    def __getitem__(self, idx):
        return np.asarray(self)[idx]

    def tolist(self) -> list:
        return np.asarray(self).tolist()


def _ids(x, what: str):
    """Endpoint arrays as contiguous int32 CUDA tensors on the current device
    (a strided or int64 tensor would otherwise be reinterpreted by the ABI)."""
    torch = _torch()
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
    if t.dim() != 1:
        raise ValueError(f"{what} must be one-dimensional")
    if t.dtype not in (torch.int8, torch.int16, torch.int32, torch.int64, torch.uint8):
        raise TypeError(f"{what} must hold integer vertex ids, not {t.dtype}")
    if t.dtype is torch.int64 and t.numel():
        lo, hi = torch.aminmax(t)
        if int(lo) < 0 or int(hi) >= 2 ** 31:  # narrowing would wrap into valid ids
            raise MalformedInputError(f"{what}: vertex id outside [0, 2^31)")
    return t.to("cuda", torch.int32).contiguous()


class IncrementalConnectivity:
    """Device-resident incremental state over `capacity` vertex slots.

    Every entry point runs on the caller's current CUDA stream.  Endpoints
    are coerced to contiguous int32 device tensors; an endpoint outside
    [0, capacity) raises MalformedInputError (the op itself is skipped on
    the device, so the state is never written out of bounds)."""

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
        self._stream = _stream().value
        self.stats = N.Stats()

    def _on_current_stream(self):
        cur = _stream()
        if cur.value != self._stream:
            N.check(N.lib().gc_incr_set_stream(self._h, cur))
            self._stream = cur.value

    def _pair(self, us, vs):
        us, vs = _ids(us, "us"), _ids(vs, "vs")
        if us.numel() != vs.numel():
            raise ValueError("us and vs must have the same length")
        self._on_current_stream()
        return us, vs

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.lib().gc_incr_destroy(h)
            except Exception:
                pass
            self._h = None

    def reserve(self, batch_len: int) -> None:
        """Pre-size the per-batch buffers (gc_incr_reserve): the round finishes' COO, the
        giant filter's compacted batch."""
        N.check(N.lib().gc_incr_reserve(self._h, int(batch_len)))

    def insert(self, us, vs, sync: bool = True) -> None:
        """Insert-only batch (columnar, int32 ids).  sync=False (union-find
        specs): enqueue only on the current stream; later calls order after
        it, and a malformed endpoint is reported by the next synchronising
        call.  The kernel runs on the current stream, so the caching allocator
        cannot hand the (possibly coerced) id buffers to later work before it
        has read them."""
        us, vs = self._pair(us, vs)
        n = int(us.numel())
        fn = N.lib().gc_incr_insert if sync else N.lib().gc_incr_insert_async
        N.check(fn(self._h, us.data_ptr() if n else None, vs.data_ptr() if n else None, n, C.byref(self.stats)))

    def insert_list(self, us, vs):
        """Insert-only batch that also returns the edges that merged two trees
        (the exchange unit of the sharded driver; root-based rules only)."""
        torch = _torch()
        us, vs = self._pair(us, vs)
        n = int(us.numel())
        ou = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        ov = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        if n:
            N.check(N.lib().gc_incr_insert_list(self._h, us.data_ptr(), vs.data_ptr(), n, ou.data_ptr(),
                                                ov.data_ptr(), cnt.data_ptr(), C.byref(self.stats)))
        c = int(cnt.item())
        return ou[:c], ov[:c]

    def query(self, us, vs) -> PackedBits:
        """Query-only batch; returns the connected bits packed 32 per word."""
        torch = _torch()
        us, vs = self._pair(us, vs)
        n = int(us.numel())
        words = torch.zeros(max((n + 31) // 32, 1), dtype=torch.int32, device="cuda")
        if n:
            N.check(N.lib().gc_incr_query(self._h, us.data_ptr(), vs.data_ptr(), n, words.data_ptr(),
                                          C.byref(self.stats)))
        return PackedBits(words, n)

    def batch(self, us, vs, is_query) -> PackedBits:
        """Mixed batch in reference order; returns packed bits (1 = connected query)."""
        torch = _torch()
        us, vs = self._pair(us, vs)
        n = int(us.numel())
        isq = torch.as_tensor(is_query).to("cuda", torch.uint8).contiguous()
        if isq.numel() != n:
            raise ValueError("is_query must have one flag per op")
        words = torch.zeros(max((n + 31) // 32, 1), dtype=torch.int32, device="cuda")
        if n:
            N.check(N.lib().gc_incr_batch(self._h, us.data_ptr(), vs.data_ptr(), isq.data_ptr(), n,
                                          words.data_ptr(), int(self.racy), C.byref(self.stats)))
        return PackedBits(words, n)

    def state(self):
        """Copy of the live state with the sentinel convention (driver.py:656, 710)."""
        torch = _torch()
        self._on_current_stream()
        slots = self.capacity if self.spec.is_union_finish() else self.capacity + 1
        out = torch.empty(max(slots, 1), dtype=torch.int32, device="cuda")
        N.check(N.lib().gc_incr_state(self._h, out.data_ptr()))
        return out[:slots]

    def live_state(self) -> LiveState:
        """The live device state itself (no copy), as on_batch receives it."""
        self._on_current_stream()
        ptr = C.c_void_p()
        slots = C.c_int64(0)
        N.check(N.lib().gc_incr_state_view(self._h, C.byref(ptr), C.byref(slots)))
        return LiveState(ptr.value, slots.value, self)

    def labels(self):
        """(finalized int32 labels tensor, component count of initialised vertices)."""
        torch = _torch()
        self._on_current_stream()
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
            results.append(bits.numpy())
        else:
            results.append(np.zeros(0, dtype=bool))
        if on_batch is not None:
            on_batch(bi, inc.live_state())
    labels, comps = inc.labels()
    st = inc.stats
    stats.phase_times = {"insert": st.t_sample_ms / 1e3, "query": st.t_finish_ms / 1e3}
    stats.edge_inspections = {"insert": int(st.insp_finish)} if st.insp_finish else {}
    stats.rounds = int(st.rounds)
    stats.component_count = comps
    return host_int64(labels), results, stats
