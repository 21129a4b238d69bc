"""Multi-GPU connectivity: one process per GPU, torch.distributed
for the plumbing (NCCL over NVLink on B200; gloo for the CPU tests).

The reference has no multi-GPU path; the designs
here follow the survey:

* **Edge-sharded static CC / spanning forest.**  Rows of the CSR are split
  into edge-balanced blocks.  Each rank runs the unsampled union-find
  pipeline on its block (the `t < u` rule of the finish presents every
  undirected edge on exactly one rank), producing a local forest F_r and a
  parent array.  Forests merge tree-wise in log2(P) rounds: the partner's
  forest edges are unioned into the receiver's state and the edges that merge
  two trees are added to its forest (``gc_union_edges_list``).  Rank 0 ends
  with a spanning forest of the union and broadcasts the canonical labels.
  Sampled specs are not sound per shard (a per-shard L_max may skip an edge
  between two different local giants, SURVEY §8e caveat) and are rejected.
* **Batch-sharded incremental.**  Every rank keeps a full replica.  Each
  batch's inserts are split 1/P; a rank unions its part recording the edges
  that merged trees (a spanning forest of the part w.r.t. its replica),
  all-gathers those lists and unions the foreign ones.  All replicas then
  induce the same partition, so queries are answered locally after the
  exchange — the reference's insert -> barrier -> query order
  (driver.py:695-708).  Communication is 8 bytes per merging edge.

The local compute goes through an ``Engine``; ``GpuEngine`` is libgconn.
Tests plug a CPU engine to exercise the collective logic with gloo.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError
from .spec import AlgorithmSpec, SampleKind, format_spec


def _torch():
    import torch
    return torch


def _dist():
    import torch.distributed as dist
    return dist


# ------------------------------------------------------------------ sharding

def shard_bounds(offsets, world: int) -> list[tuple[int, int]]:
    """Contiguous row blocks [lo, hi) with (nearly) equal directed-edge counts."""
    off = np.asarray(offsets.cpu() if hasattr(offsets, "cpu") else offsets, dtype=np.int64)
    n = len(off) - 1
    m = int(off[-1])
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(off, (m * r) // world, side="left")))
    cuts.append(n)
    cuts = [min(max(c, 0), n) for c in cuts]
    for i in range(1, len(cuts)):
        cuts[i] = max(cuts[i], cuts[i - 1])
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


def shard_graph(g, lo: int, hi: int):
    """The graph restricted to rows [lo, hi): same vertex set, other rows empty."""
    from .graph import Graph
    torch = _torch()
    if g.on_device:
        off, tgt = g.device_arrays()
        idx = torch.arange(g.n + 1, device=off.device).clamp_(lo, hi)
        off_s = off[idx] - off[lo]
        tgt_s = tgt[off[lo]:off[hi]]
        return Graph(g.n, off_s.contiguous(), tgt_s.contiguous())
    off, tgt = g.offsets, g.targets
    idx = np.clip(np.arange(g.n + 1), lo, hi)
    return Graph(g.n, off[idx] - off[lo], tgt[off[lo]:off[hi]])


# -------------------------------------------------------------------- engine

class GpuEngine:
    """Local compute on this rank's GPU through libgconn."""

    device = "cuda"

    def local_forest(self, shard, spec):
        from .api import spanning_forest_device
        df, _st, parent = spanning_forest_device(shard, spec, want_parent=True)
        keep = df.fu >= 0
        return parent, df.fu[keep].contiguous(), df.fv[keep].contiguous()

    def union_list(self, parent, us, vs, spec):
        import ctypes as C
        from . import _native as N
        from .api import LoweredSpec, _stream
        torch = _torch()
        k = int(us.numel())
        out_u = torch.empty(max(k, 1), dtype=torch.int32, device="cuda")
        out_v = torch.empty(max(k, 1), dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        if k:
            low = LoweredSpec(spec, None, parent.numel())
            aux = None
            if spec.cfg.union.value in ("hooks", "rem_lock"):
                aux = torch.full((parent.numel(),), parent.numel() if spec.cfg.union.value == "hooks" else 0,
                                 dtype=torch.int32, device="cuda")
            N.check(N.lib().gc_union_edges_list(parent.data_ptr(), parent.numel(), us.data_ptr(), vs.data_ptr(),
                                                k, C.byref(low.s), aux.data_ptr() if aux is not None else None,
                                                out_u.data_ptr(), out_v.data_ptr(), cnt.data_ptr(), _stream()))
        c = int(cnt.item())
        return out_u[:c], out_v[:c]

    def finalize(self, parent):
        import ctypes as C
        from . import _native as N
        from .api import _stream, _workspace
        lab = parent.clone()
        n = lab.numel()
        if n:
            ws = _workspace(4 * n + 8192)
            N.check(N.lib().gc_label_finalization(lab.data_ptr(), n, ws.data_ptr(), ws.numel(), _stream()))
        return lab

    def incr_create(self, spec, capacity):
        from .incremental import IncrementalConnectivity
        return IncrementalConnectivity(spec, capacity)

    def incr_insert_list(self, h, us, vs):
        return h.insert_list(us, vs)

    def incr_insert(self, h, us, vs):
        h.insert(us, vs)

    def incr_query(self, h, us, vs):
        return h.query(us, vs)

    def incr_labels(self, h):
        return h.labels()


# ------------------------------------------------------------- collectives

def _comm_device(group=None):
    dist = _dist()
    return "cuda" if dist.get_backend(group) == "nccl" else "cpu"


def _send_pairs(us, vs, dst, group=None):
    torch = _torch()
    dist = _dist()
    dev = _comm_device(group)
    k = torch.tensor([us.numel()], dtype=torch.int64, device=dev)
    dist.send(k, dst, group=group)
    if us.numel():
        dist.send(torch.stack([us, vs]).to(dev, torch.int32).contiguous(), dst, group=group)


def _recv_pairs(src, group=None):
    torch = _torch()
    dist = _dist()
    dev = _comm_device(group)
    k = torch.zeros(1, dtype=torch.int64, device=dev)
    dist.recv(k, src, group=group)
    kk = int(k.item())
    buf = torch.empty((2, kk), dtype=torch.int32, device=dev)
    if kk:
        dist.recv(buf, src, group=group)
    return buf[0], buf[1]


def all_gather_pairs(us, vs, group=None):
    """All-gather variable-length (u, v) lists: counts first, then padded data."""
    torch = _torch()
    dist = _dist()
    dev = _comm_device(group)
    world = dist.get_world_size(group)
    k = torch.tensor([us.numel()], dtype=torch.int64, device=dev)
    ks = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(ks, k, group=group)
    counts = [int(x.item()) for x in ks]
    kmax = max(counts) if counts else 0
    if kmax == 0:
        return [(us[:0], vs[:0]) for _ in range(world)]
    mine = torch.full((2, kmax), -1, dtype=torch.int32, device=dev)
    if us.numel():
        mine[:, :us.numel()] = torch.stack([us, vs]).to(dev, torch.int32)
    bufs = [torch.empty((2, kmax), dtype=torch.int32, device=dev) for _ in range(world)]
    dist.all_gather(bufs, mine, group=group)
    return [(b[0, :c], b[1, :c]) for b, c in zip(bufs, counts)]


# -------------------------------------------------------- sharded static / forest

@dataclass
class ShardedResult:
    labels: object          # canonical labels (every rank)
    forest_u: object        # global spanning forest edges (every rank)
    forest_v: object
    components: int
    merge_rounds: int
    exchanged_edges: int    # forest edges sent over the interconnect by all ranks


def _check_sharded_spec(spec: AlgorithmSpec):
    if spec.sample is not SampleKind.NONE or not spec.is_union_finish() or not spec.is_root_based():
        raise ConfigError(f"sharded connectivity needs an unsampled root-based union-find spec; "
                          f"'{format_spec(spec)}' is not (per-shard sampling is unsound, SURVEY 8e)")


def sharded_spanning_forest(g_shard, spec: AlgorithmSpec, group=None, engine=None) -> ShardedResult:
    """Edge-sharded spanning forest + labels.  ``g_shard`` is this rank's
    row block (``shard_graph``); every rank calls collectively."""
    _check_sharded_spec(spec)
    torch = _torch()
    dist = _dist()
    engine = engine or GpuEngine()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    parent, fu, fv = engine.local_forest(g_shard, spec)
    dev_local = parent.device
    step, rounds, sent = 1, 0, 0
    active = True
    while step < world:
        if active:
            if rank % (2 * step) == step:
                _send_pairs(fu, fv, rank - step, group)
                sent += fu.numel()
                active = False
            elif rank % (2 * step) == 0 and rank + step < world:
                ou, ov = _recv_pairs(rank + step, group)
                mu, mv = engine.union_list(parent, ou.to(dev_local), ov.to(dev_local), spec)
                fu = torch.cat([fu, mu])
                fv = torch.cat([fv, mv])
        step *= 2
        rounds += 1
    # rank 0 holds the global forest and parent array: broadcast results
    n = g_shard.n
    dev = _comm_device(group)
    labels = engine.finalize(parent) if rank == 0 else torch.empty(n, dtype=torch.int32, device=dev_local)
    lab_c = labels.to(dev)
    dist.broadcast(lab_c, 0, group=group)
    k = torch.tensor([fu.numel() if rank == 0 else 0], dtype=torch.int64, device=dev)
    dist.broadcast(k, 0, group=group)
    kk = int(k.item())
    fbuf = torch.stack([fu, fv]).to(dev, torch.int32) if rank == 0 else torch.empty((2, kk), dtype=torch.int32,
                                                                                     device=dev)
    if kk:
        dist.broadcast(fbuf, 0, group=group)
    tot = torch.tensor([sent], dtype=torch.int64, device=dev)
    dist.all_reduce(tot, group=group)
    labels = lab_c.to(dev_local)
    comps = int((labels == torch.arange(n, device=labels.device, dtype=labels.dtype)).sum().item())
    return ShardedResult(labels, fbuf[0].to(dev_local), fbuf[1].to(dev_local), comps, rounds, int(tot.item()))


def sharded_static_connectivity(g_shard, spec: AlgorithmSpec, group=None, engine=None):
    """Edge-sharded static connectivity: canonical labels on every rank."""
    res = sharded_spanning_forest(g_shard, spec, group, engine)
    return res.labels, res


# ------------------------------------------------------- sharded incremental

class ShardedIncremental:
    """Batch-sharded incremental connectivity with a full replica per rank."""

    def __init__(self, spec: AlgorithmSpec, capacity: int, group=None, engine=None):
        if not (spec.is_union_finish() and spec.is_root_based()):
            raise ConfigError(f"sharded incremental needs a root-based union-find spec; "
                              f"'{format_spec(spec)}' is not")
        dist = _dist()
        self.spec, self.capacity, self.group = spec, int(capacity), group
        self.engine = engine or GpuEngine()
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.h = self.engine.incr_create(spec, self.capacity)
        self.exchanged = 0

    def _slice(self, k: int) -> tuple[int, int]:
        return (k * self.rank) // self.world, (k * (self.rank + 1)) // self.world

    def insert(self, us, vs, local: bool = False):
        """Insert a batch.  With ``local=False`` every rank passes the whole
        batch and takes its 1/P slice; with ``local=True`` the arrays already
        are this rank's part."""
        if not local:
            lo, hi = self._slice(int(us.numel()))
            us, vs = us[lo:hi], vs[lo:hi]
        mu, mv = self.engine.incr_insert_list(self.h, us, vs)
        lists = all_gather_pairs(mu, mv, self.group)
        for r, (ou, ov) in enumerate(lists):
            self.exchanged += int(ou.numel())
            if r != self.rank and ou.numel():
                self.engine.incr_insert(self.h, ou.to(mu.device), ov.to(mu.device))

    def query(self, us, vs):
        """Queries after the batch barrier: every replica induces the same
        partition, so each rank answers locally."""
        return self.engine.incr_query(self.h, us, vs)

    def labels(self):
        return self.engine.incr_labels(self.h)
