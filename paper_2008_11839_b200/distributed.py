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
* **Sampled specs (k-out / HB): two-phase exchange.**  A per-shard L_max is
  not sound (it may skip an edge between two different local giants, SURVEY
  §8e caveat), so each rank samples its rows, the sampled merging edges are
  all-gathered and unioned everywhere, and only then is the (now global and
  identical) L_max taken and the finish run over each rank's active rows,
  followed by a second all-gather (``sharded_two_phase``).
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

import os
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError
from .spec import AlgorithmSpec, KOutMode, SampleKind, format_spec


def _torch():
    import torch
    return torch


def _dist():
    import torch.distributed as dist
    return dist


# ------------------------------------------------------------------ sharding

def shard_bounds(offsets, world: int, by: str = "edges") -> list[tuple[int, int]]:
    """Contiguous row blocks [lo, hi) with (nearly) equal directed-edge counts
    (``by="edges"``: the unsampled finish walks every edge) or equal row
    counts (``by="rows"``: k-out / HB sampling costs the same per row
    whatever its degree, so edge-balanced blocks would leave the ranks that
    hold the many low-degree rows with most of the work)."""
    off = np.asarray(offsets.cpu() if hasattr(offsets, "cpu") else offsets, dtype=np.int64)
    n = len(off) - 1
    m = int(off[-1])
    cuts = [0]
    for r in range(1, world):
        if by == "rows":
            cuts.append((n * r) // world)
        else:
            cuts.append(int(np.searchsorted(off, (m * r) // world, side="left")))
    cuts.append(n)
    cuts = [min(max(c, 0), n) for c in cuts]
    for i in range(1, len(cuts)):
        cuts[i] = max(cuts[i], cuts[i - 1])
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


def shard_balance(spec: AlgorithmSpec) -> str:
    """The shard_bounds balance for a spec (rows for the per-row samplers)."""
    return "rows" if spec.sample in (SampleKind.KOUT, SampleKind.HB) else "edges"


def shard_graph(g, lo: int, hi: int):
    """The graph restricted to rows [lo, hi): same vertex set, other rows empty."""
    from .graph import Graph
    torch = _torch()
    if g.on_device:
        off, tgt = g.device_arrays()
        idx = torch.arange(g.n + 1, device=off.device).clamp_(lo, hi)
        off_s = off[idx] - off[lo]
        tgt_s = tgt[off[lo]:off[hi]]
        out = Graph(g.n, off_s.contiguous(), tgt_s.contiguous())
    else:
        off, tgt = g.offsets, g.targets
        idx = np.clip(np.arange(g.n + 1), lo, hi)
        out = Graph(g.n, off[idx] - off[lo], tgt[off[lo]:off[hi]])
    out.row_block = (int(lo), int(hi))  # the kernels walk only these rows
    return out


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

    def union_pairs(self, parent, us, vs, spec):
        """Union without recording (gc_union_edges): any rule, root-based or not."""
        import ctypes as C
        from . import _native as N
        from .api import LoweredSpec, _stream
        torch = _torch()
        k = int(us.numel())
        if not k:
            return
        low = LoweredSpec(spec, None, parent.numel())
        aux = None
        if spec.cfg.union.value in ("hooks", "rem_lock"):
            aux = torch.full((parent.numel(),), parent.numel() if spec.cfg.union.value == "hooks" else 0,
                             dtype=torch.int32, device="cuda")
        N.check(N.lib().gc_union_edges(parent.data_ptr(), parent.numel(), us.data_ptr(), vs.data_ptr(), k,
                                       C.byref(low.s), aux.data_ptr() if aux is not None else None, None, None,
                                       _stream()))

    def _shard_call(self, fn, shard, spec, parent, record=True):
        import ctypes as C
        from . import _native as N
        from .api import LoweredSpec, _csr, _stream, _workspace
        torch = _torch()
        n = shard.n
        low = LoweredSpec(spec, shard, n)
        csr, keep = _csr(shard)
        lib = N.lib()
        ws = _workspace(lib.gc_workspace_size(n, shard.m, C.byref(low.s)))
        st = N.Stats()
        lo, hi = getattr(shard, "row_block", (0, n))
        if not record:
            N.check(getattr(lib, fn)(C.byref(csr), C.byref(low.s), lo, hi, parent.data_ptr(), None, None, None,
                                     C.byref(st), ws.data_ptr(), ws.numel(), _stream()))
            return None, None, st
        out_u = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        out_v = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        N.check(getattr(lib, fn)(C.byref(csr), C.byref(low.s), lo, hi, parent.data_ptr(), out_u.data_ptr(),
                                 out_v.data_ptr(), cnt.data_ptr(), C.byref(st), ws.data_ptr(), ws.numel(),
                                 _stream()))
        c = int(cnt.item())
        return out_u[:c], out_v[:c], st

    def shard_sample(self, shard, spec, record=True):
        """gc_shard_sample: identity parent + the sampler over this block's rows
        (record=False: no merge list, for the compact summary exchange)."""
        torch = _torch()
        parent = torch.empty(max(shard.n, 1), dtype=torch.int32, device="cuda")
        mu, mv, st = self._shard_call("gc_shard_sample", shard, spec, parent, record)
        return parent, mu, mv, int(st.insp_sample)

    def shard_finish(self, shard, spec, parent):
        """gc_shard_finish: L_max + active gather + finish over this block's rows."""
        mu, mv, st = self._shard_call("gc_shard_finish", shard, spec, parent)
        return mu, mv, {"insp_finish": int(st.insp_finish), "l_max": int(st.l_max),
                        "lmax_count": int(st.lmax_count), "n_active": int(st.n_active)}

    def shard_summary(self, parent, hint=None, pairs=True):
        """gc_shard_summary: (bitmap int32 words, class label, remainder pairs or None)."""
        from . import _native as N
        from .api import _stream, _workspace
        torch = _torch()
        n = parent.numel()
        words = torch.zeros(max((n + 31) // 32, 1), dtype=torch.int32, device="cuda")
        label = torch.zeros(1, dtype=torch.int64, device="cuda")
        out_u = out_v = cnt = None
        if pairs:
            out_u = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
            out_v = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
            cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        ws = _workspace(N.lib().gc_shard_summary_workspace(n))
        ptr = (lambda t: t.data_ptr() if t is not None else None)
        N.check(N.lib().gc_shard_summary(parent.data_ptr(), n, ptr(hint), words.data_ptr(), label.data_ptr(),
                                         ptr(out_u), ptr(out_v), ptr(cnt), ws.data_ptr(), ws.numel(), _stream()))
        if not pairs:
            return words, label, None, None
        c = int(cnt.item())
        return words, label, out_u[:c], out_v[:c]

    def shard_absorb(self, parent, words_all, labels_all):
        """gc_shard_absorb (round A); returns rank 0's class representative (device)."""
        from . import _native as N
        from .api import _stream, _workspace
        torch = _torch()
        n = parent.numel()
        rep = torch.zeros(1, dtype=torch.int32, device="cuda")
        ws = _workspace(4 * n + 8192)
        words_all = words_all.contiguous()
        labels_all = labels_all.contiguous()
        N.check(N.lib().gc_shard_absorb(parent.data_ptr(), n, words_all.data_ptr(), labels_all.data_ptr(),
                                        int(labels_all.numel()), rep.data_ptr(), ws.data_ptr(), ws.numel(),
                                        _stream()))
        return rep

    def shard_join(self, parent, words_all, labels_all, us, vs, spec):
        """gc_shard_join over all ranks' summaries (words_all: nranks x words)."""
        import ctypes as C
        from . import _native as N
        from .api import LoweredSpec, _stream, _workspace
        n = parent.numel()
        low = LoweredSpec(spec, None, n)
        ws = _workspace(5 * n + 8192)
        words_all = words_all.contiguous()
        labels_all = labels_all.contiguous()
        k = int(us.numel())
        N.check(N.lib().gc_shard_join(parent.data_ptr(), n, words_all.data_ptr(), labels_all.data_ptr(),
                                      int(labels_all.numel()), us.data_ptr() if k else None,
                                      vs.data_ptr() if k else None, k, C.byref(low.s), ws.data_ptr(), ws.numel(),
                                      _stream()))

    # distributed BFS (gc_dbfs_*): state = dict of device buffers.  The state
    # is bound to the stream current at dbfs_init, and the per-level calls
    # reuse cached pointers / CSR descriptors (they run a few times per level,
    # where host overhead is most of their cost).
    def dbfs_init(self, n, source):
        from . import _native as N
        from .api import _stream
        torch = _torch()
        words = max((n + 31) // 32, 1)
        st = {"n": n,
              "F": torch.zeros(words, dtype=torch.int32, device="cuda"),
              "V": torch.zeros(words, dtype=torch.int32, device="cuda"),
              "M": torch.zeros(words, dtype=torch.int32, device="cuda"),
              "N": torch.zeros(words, dtype=torch.int32, device="cuda"),
              "par": torch.empty(max(n, 1), dtype=torch.int32, device="cuda"),
              "ids": torch.empty(max(n, 1), dtype=torch.int32, device="cuda"),
              # [count, bad flag]: the advance reads both with one device read
              "cnt": torch.zeros(2, dtype=torch.int64, device="cuda"),
              "stream": _stream(), "lib": N.lib()}
        st["ptr"] = {k: st[k].data_ptr() for k in ("F", "V", "M", "N", "par", "ids", "cnt")}
        N.check(st["lib"].gc_dbfs_init(n, source, st["ptr"]["F"], st["ptr"]["V"], st["ptr"]["par"], st["stream"]))
        return st

    @staticmethod
    def _dbfs_csr(shard):
        c = getattr(shard, "_dbfs_csr", None)
        if c is None:
            import ctypes as C
            from .api import _csr
            csr, keep = _csr(shard)
            lo, hi = getattr(shard, "row_block", (0, shard.n))
            c = shard._dbfs_csr = (C.byref(csr), lo, hi, csr, keep)
        return c

    def dbfs_marks(self, shard, st):
        from . import _native as N
        ref, lo, hi = self._dbfs_csr(shard)[:3]
        p = st["ptr"]
        N.check(st["lib"].gc_dbfs_marks(ref, lo, hi, p["F"], p["V"], p["M"], p["ids"], p["cnt"], st["stream"]))
        return st["ids"][:int(st["cnt"][0].item())]

    def dbfs_merge_marks(self, st, ids):
        from . import _native as N
        ids = ids.to("cuda", dtype=__import__("torch").int32).contiguous()
        if ids.numel():
            N.check(st["lib"].gc_dbfs_merge_marks(st["n"], ids.data_ptr(), ids.numel(), st["ptr"]["M"],
                                                  st["ptr"]["cnt"] + 8, st["stream"]))

    def dbfs_claim(self, shard, st, marks, foreign=None):
        """foreign: the other ranks' mark ids, merged in the same call."""
        from . import _native as N
        ref, lo, hi = self._dbfs_csr(shard)[:3]
        p = st["ptr"]
        if foreign is not None and foreign.numel():
            foreign = foreign.to("cuda", dtype=__import__("torch").int32).contiguous()
            N.check(st["lib"].gc_dbfs_merge_claim(ref, lo, hi, p["F"], p["V"], p["M"], foreign.data_ptr(),
                                                  foreign.numel(), p["cnt"] + 8, p["par"], p["N"], p["cnt"],
                                                  st["stream"]))
        else:
            N.check(st["lib"].gc_dbfs_claim(ref, lo, hi, p["F"], p["V"], p["M"] if marks else None, p["par"],
                                            p["N"], p["cnt"], st["stream"]))
        return st["N"]

    def dbfs_advance(self, st):
        from . import _native as N
        p = st["ptr"]
        N.check(st["lib"].gc_dbfs_advance(st["n"], p["V"], p["F"], p["N"], p["cnt"], st["stream"]))
        count, bad = st["cnt"].tolist()
        if bad:
            from .errors import MalformedInputError
            raise MalformedInputError("a merged frontier mark lies outside [0, n)")
        return int(count)

    def dbfs_finish(self, shard, st):
        import ctypes as C
        from . import _native as N
        from .api import _csr, _stream, _workspace
        torch = _torch()
        n = st["n"]
        csr, _keep = _csr(shard)
        lo, hi = getattr(shard, "row_block", (0, n))
        labels = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        fu = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        fv = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        insp = torch.zeros(1, dtype=torch.int64, device="cuda")
        ws = _workspace(64)
        N.check(N.lib().gc_dbfs_finish(C.byref(csr), lo, hi, st["V"].data_ptr(), st["par"].data_ptr(),
                                       labels.data_ptr(), fu.data_ptr(), fv.data_ptr(), st["cnt"].data_ptr(),
                                       insp.data_ptr(), ws.data_ptr(), ws.numel(), _stream()))
        k = int(st["cnt"][0].item())
        return labels[:n], fu[:k], fv[:k], int(insp.item())

    def row_degrees(self, shard, ids):
        """Degrees of the given vertices in this rank's rows (0 elsewhere)."""
        torch = _torch()
        off, _tgt = shard.device_arrays()
        ids = torch.as_tensor(ids, dtype=torch.int64, device=off.device)
        return (off[ids + 1] - off[ids]).to(torch.int64)

    def finalize(self, parent, inplace=False):
        """Canonical labels (gc_label_finalization); inplace=True reuses the
        parent buffer (the sharded drivers no longer need it afterwards)."""
        import ctypes as C
        from . import _native as N
        from .api import _stream, _workspace
        lab = parent if inplace else parent.clone()
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
    counts = torch.cat(ks).tolist()  # one device read for all the counts
    kmax = max(counts) if counts else 0
    if kmax == 0:
        return [(us[:0], vs[:0]) for _ in range(world)]
    mine = torch.full((2, kmax), -1, dtype=torch.int32, device=dev)
    if us.numel():
        mine[:, :us.numel()] = torch.stack([us, vs]).to(dev, torch.int32)
    bufs = [torch.empty((2, kmax), dtype=torch.int32, device=dev) for _ in range(world)]
    dist.all_gather(bufs, mine, group=group)
    return [(b[0, :c], b[1, :c]) for b, c in zip(bufs, counts)]


def all_gather_ids(ids, group=None):
    """All-gather variable-length int32 id lists (counts, then padded data)."""
    torch = _torch()
    dist = _dist()
    dev = _comm_device(group)
    world = dist.get_world_size(group)
    k = torch.tensor([ids.numel()], dtype=torch.int64, device=dev)
    ks = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(ks, k, group=group)
    counts = torch.cat(ks).tolist()  # one device read for all the counts
    kmax = max(counts) if counts else 0
    if kmax == 0:
        return [ids[:0] for _ in range(world)]
    mine = torch.full((kmax,), -1, dtype=torch.int32, device=dev)
    if ids.numel():
        mine[:ids.numel()] = ids.to(dev, torch.int32)
    bufs = [torch.empty(kmax, dtype=torch.int32, device=dev) for _ in range(world)]
    dist.all_gather(bufs, mine, group=group)
    return [b[:c] for b, c in zip(bufs, counts)]


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


def _check_two_phase_spec(spec: AlgorithmSpec):
    if not spec.is_union_finish():
        raise ConfigError(f"sharded connectivity needs a union-find finish; '{format_spec(spec)}' is not")
    if spec.sample not in (SampleKind.NONE, SampleKind.KOUT, SampleKind.HB, SampleKind.BFS):
        raise ConfigError(f"sharded sampling supports none / kout / hb / bfs, not '{spec.sample.value}' "
                          "(LDD has no distributed form)")
    if spec.sample is SampleKind.KOUT and spec.kout_mode is not KOutMode.FIRST_K:
        raise ConfigError("sharded k-out needs FIRST_K: random offsets are drawn over the whole graph")


# ------------------------------------------------------- distributed BFS

# Beamer's switch (as the single-GPU sampler, traverse.cu): bottom-up once
# the frontier is more than 1/alpha of the unreached vertices, back to
# top-down below n/beta frontier vertices
DBFS_ALPHA = int(os.environ.get("GC_DBFS_ALPHA", "14"))
DBFS_BETA = int(os.environ.get("GC_DBFS_BETA", "24"))


def global_bfs_source(g_shard, spec: AlgorithmSpec, group=None, engine=None) -> int:
    """sampling.py:130-132 over a row-sharded graph: the highest-degree vertex
    of the seeded probe set (ties: the smaller id), degrees summed over the
    ranks that own the probes' rows."""
    torch = _torch()
    dist = _dist()
    engine = engine or GpuEngine()
    n = g_shard.n
    probes = np.unique(np.random.default_rng(spec.seed).integers(0, n, size=spec.bfs_probes))
    deg = engine.row_degrees(g_shard, probes).to(_comm_device(group), torch.int64)
    dist.all_reduce(deg, group=group)
    d = deg.cpu().numpy()
    return int(probes[int(np.argmax(d))])


@dataclass
class DistributedBfs:
    labels: object      # reached set -> its minimum id, others identity (every rank)
    tree_u: object      # the whole BFS tree (every rank): (parent, v) per reached v != source;
    tree_v: object      # with gather_tree=False only the (parent, v) of this rank's rows
    insp_sample: int    # sum of the reached vertices' degrees (sampling.py:141-144)
    levels: int
    reached: int
    exchanged_ids: int  # top-down mark ids all-gathered over all levels


def distributed_bfs(g_shard, spec: AlgorithmSpec, group=None, engine=None,
                    gather_tree: bool = True) -> DistributedBfs:
    """BFS sampling (sampling.py:120-172) as a level-synchronous traversal over
    row-sharded CSR.  The frontier and visited bitmaps are
    replicated; the owner of a vertex decides its parent (the first frontier
    vertex of its ascending row, the reference's smallest-discoverer rule),
    so only bits cross the interconnect: per level, the top-down marks as id
    lists (narrow frontiers, merged here as one batch) and the next-frontier
    bitmap as an all-reduce SUM (the ranks' claimed bits are disjoint, so the
    sum is the union).  gather_tree=False keeps each rank's tree edges local
    (one pair per reached vertex: all-gathering them moves 8 B per vertex)."""
    torch = _torch()
    dist = _dist()
    engine = engine or GpuEngine()
    n = g_shard.n
    if n == 0:
        z = torch.zeros(0, dtype=torch.int32)
        return DistributedBfs(z, z, z, 0, 0, 0, 0)
    m_tot = torch.tensor([g_shard.m], dtype=torch.int64, device=_comm_device(group))
    dist.all_reduce(m_tot, group=group)
    if int(m_tot.item()) == 0:  # sampling.py:128-129: nothing to traverse
        lab = torch.arange(n, dtype=torch.int32, device=engine.device)
        z = torch.zeros(0, dtype=torch.int32, device=engine.device)
        return DistributedBfs(lab, z, z, 0, 0, 0, 0)
    src = global_bfs_source(g_shard, spec, group, engine)
    st = engine.dbfs_init(n, src)
    dev = _comm_device(group)
    nf, reached, levels, bottom_up, sent = 1, 1, 0, False, 0
    while nf:
        want_bu = nf * DBFS_ALPHA > n - reached if not bottom_up else nf >= n // DBFS_BETA
        bottom_up = want_bu
        if bottom_up:
            nxt = engine.dbfs_claim(g_shard, st, marks=False)
        else:
            ids = engine.dbfs_marks(g_shard, st)
            rank = dist.get_rank(group)
            foreign = []
            for r, ou in enumerate(all_gather_ids(ids, group)):
                sent += int(ou.numel())
                if r != rank and ou.numel():
                    foreign.append(ou.to(ids.device))
            merged = (torch.cat(foreign) if len(foreign) > 1 else foreign[0]) if foreign else None
            nxt = engine.dbfs_claim(g_shard, st, marks=True, foreign=merged)
        buf = nxt.to(dev)
        dist.all_reduce(buf, group=group)  # disjoint bits: SUM == OR
        if buf is not nxt:
            nxt.copy_(buf.to(nxt.device))
        nf = engine.dbfs_advance(st)
        reached += nf
        levels += 1
    labels, fu, fv, insp = engine.dbfs_finish(g_shard, st)
    tot = torch.tensor([insp], dtype=torch.int64, device=dev)
    dist.all_reduce(tot, group=group)
    if gather_tree:
        tree = all_gather_pairs(fu, fv, group)
        tu = torch.cat([t[0].to(labels.device) for t in tree])
        tv = torch.cat([t[1].to(labels.device) for t in tree])
    else:
        tu, tv = fu.to(labels.device), fv.to(labels.device)
    return DistributedBfs(labels, tu, tv, int(tot.item()), levels, reached, sent)


@dataclass
class TwoPhaseResult:
    labels: object          # canonical labels (identical on every rank)
    forest_u: object        # this rank's spanning forest of the whole graph (forest_slices: its slice)
    forest_v: object        # (None for non-root-based specs)
    components: int
    insp_sample: int        # whole-graph inspection counts (sum over ranks)
    insp_finish: int
    l_max: int
    lmax_count: int
    n_active: int
    exchanged_edges: int    # merging edges all-gathered, both phases


def _exchange_and_merge(parent, mu, mv, spec, engine, group, rank):
    """All-gather every rank's merge list; union the foreign ones.  Returns
    the edges that merged trees here (own + foreign) and the total exchanged.
    Root-based rules exchange real merging edges (a forest); the others
    (Rem with the atomic splice) exchange root transitions (v, P[v]), which
    carry the partition but are not graph edges."""
    torch = _torch()
    fu, fv = [mu], [mv]
    total = 0
    record = spec.is_root_based()
    # the foreign lists are unioned as one batch (one launch and one range
    # check instead of one per rank)
    gu, gv = [], []
    for r, (ou, ov) in enumerate(all_gather_pairs(mu, mv, group)):
        total += int(ou.numel())
        if r != rank and ou.numel():
            gu.append(ou.to(parent.device))
            gv.append(ov.to(parent.device))
    if gu:
        ou, ov = torch.cat(gu), torch.cat(gv)
        if record:
            au, av = engine.union_list(parent, ou, ov, spec)
            fu.append(au)
            fv.append(av)
        else:
            engine.union_pairs(parent, ou, ov, spec)
    return torch.cat(fu), torch.cat(fv), total


def _gather_words(words, label, group):
    torch = _torch()
    dist = _dist()
    dev = _comm_device(group)
    world = dist.get_world_size(group)
    wl = [torch.empty_like(words, device=dev) for _ in range(world)]
    dist.all_gather(wl, words.to(dev), group=group)
    ll = [torch.empty(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(ll, label.to(dev), group=group)
    return torch.stack(wl), torch.cat(ll)


def _exchange_summary(parent, spec, engine, group):
    """Phase-1 exchange for labels-only runs (csrc/shard.cu): round A
    all-gathers each rank's local giant as an n-bit bitmap and absorbs all
    of them locally; round B all-gathers the dominant class's bitmap plus the
    few remaining non-singleton vertices as pairs, and every rank rebuilds
    the same exact join.  Returns the number of remainder pairs exchanged."""
    torch = _torch()
    words, label, _, _ = engine.shard_summary(parent, pairs=False)
    wa, la = _gather_words(words, label, group)
    rep = engine.shard_absorb(parent, wa.to(parent.device), la.to(parent.device))
    words, label, ru, rv = engine.shard_summary(parent, hint=rep, pairs=True)
    wb, lb = _gather_words(words, label, group)
    pairs = all_gather_pairs(ru, rv, group)
    us = torch.cat([p[0] for p in pairs]).to(parent.device)
    vs = torch.cat([p[1] for p in pairs]).to(parent.device)
    engine.shard_join(parent, wb.to(parent.device), lb.to(parent.device), us, vs, spec)
    return int(us.numel())


def sharded_two_phase(g_shard, spec: AlgorithmSpec, group=None, engine=None,
                      forest: bool = True, forest_slices: bool = False) -> TwoPhaseResult:
    """The two-phase pipeline over edge-sharded row blocks.

    The skip of the finish is only sound for ONE global post-sample labelling
    and ONE global L_max (a per-shard L_max could skip an edge
    between two different local giants), so the sampled partitions are
    merged before L_max is taken:

      1. every rank samples its own rows, recording the merging edges;
      2. all-gather them, union the foreign ones: every replica now induces
         the global sampled partition, so compression gives identical labels,
         L_max and active sets on every rank with no further collective;
      3. every rank runs the finish over the active vertices of its rows,
         recording merging edges; all-gather + union again;
      4. finalise locally — identical canonical labels everywhere.

    Each rank's kept merging edges form a spanning forest of the whole graph.

    With ``forest=False`` (labels only) step 2 exchanges a compact summary
    instead of the sampled merging edges (``_exchange_summary``): two rounds
    of n-bit class bitmaps plus the few vertices outside the dominant class
    as pairs, instead of one pair per sampled row; BFS sampling then keeps
    its tree edges local (the labels need only the replicated bitmaps).

    ``forest_slices=True`` (BFS sampling) returns the forest distributed
    instead of replicated: each rank's BFS tree edges of its own rows, plus
    on rank 0 the merging edges of the finish; the union over the ranks is
    a spanning forest.  It saves the all-gather of the BFS tree (8 bytes
    per reached vertex per rank).
    """
    _check_two_phase_spec(spec)
    dist = _dist()
    engine = engine or GpuEngine()
    rank = dist.get_rank(group)
    summary = not forest and spec.sample not in (SampleKind.NONE, SampleKind.BFS)
    torch = _torch()
    if spec.sample is SampleKind.BFS:
        # the distributed traversal leaves the same global labels on every
        # rank (no partition exchange); its tree is the sampled forest
        gather = forest and not forest_slices
        bfs = distributed_bfs(g_shard, spec, group, engine, gather_tree=gather)
        parent, insp_s = bfs.labels.contiguous(), bfs.insp_sample
        # gathered tree edges were exchanged once: count them like merging edges
        f1u, f1v, x1 = bfs.tree_u, bfs.tree_v, int(bfs.tree_u.numel()) if gather else 0
    elif not summary:
        parent, mu, mv, insp_s = engine.shard_sample(g_shard, spec, record=True)
        f1u, f1v, x1 = _exchange_and_merge(parent, mu, mv, spec, engine, group, rank)
    else:
        parent, mu, mv, insp_s = engine.shard_sample(g_shard, spec, record=False)
        x1 = _exchange_summary(parent, spec, engine, group)
        f1u = f1v = torch.empty(0, dtype=torch.int32, device=parent.device)
    mu, mv, info = engine.shard_finish(g_shard, spec, parent)
    f2u, f2v, x2 = _exchange_and_merge(parent, mu, mv, spec, engine, group, rank)
    torch = _torch()
    labels = engine.finalize(parent, inplace=True)
    n = g_shard.n
    dev = _comm_device(group)
    tot = torch.tensor([0 if spec.sample is SampleKind.BFS else insp_s, info["insp_finish"]], dtype=torch.int64,
                       device=dev)
    dist.all_reduce(tot, group=group)
    if spec.sample is SampleKind.BFS:
        tot[0] = insp_s  # already the sum over ranks
    labels = labels[:n]
    comps = int((labels == torch.arange(n, device=labels.device, dtype=labels.dtype)).sum().item())
    keep = forest and spec.is_root_based()
    if keep and forest_slices and spec.sample is SampleKind.BFS and rank != 0:
        f2u, f2v = f2u[:0], f2v[:0]  # rank 0 carries the merge forest
    fu = torch.cat([f1u, f2u]) if keep else None
    fv = torch.cat([f1v, f2v]) if keep else None
    return TwoPhaseResult(labels, fu, fv, comps, int(tot[0].item()), int(tot[1].item()), info["l_max"],
                          info["lmax_count"], info["n_active"], x1 + x2)


# gc_shard_absorb / gc_shard_join combine at most this many ranks' bitmap
# summaries (kMaxRanks in csrc/shard.cu); wider groups exchange edges instead
MAX_SUMMARY_RANKS = 8


def sharded_static_connectivity(g_shard, spec: AlgorithmSpec, group=None, engine=None):
    """Edge-sharded static connectivity: canonical labels on every rank.
    Unsampled root-based specs merge forests tree-wise; every other
    union-find spec (sampled, or Rem with the atomic splice) runs the
    two-phase exchange, with the compact bitmap summary up to
    MAX_SUMMARY_RANKS ranks and the merging-edge exchange beyond."""
    if spec.sample is SampleKind.NONE and spec.is_union_finish() and spec.is_root_based():
        res = sharded_spanning_forest(g_shard, spec, group, engine)
    else:
        wide = _dist().get_world_size(group) > MAX_SUMMARY_RANKS
        res = sharded_two_phase(g_shard, spec, group, engine, forest=wide)
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


# ------------------------------------------- single-process communicator

class DeviceComm:
    """The C-ABI communicator (``gc_comm_init``): one process drives one rank
    per listed device — NCCL over NVLink / NVSwitch when the devices are
    distinct, a loopback communicator (ranks share the device, collectives
    are device copies) when the list repeats one device.  The same two-phase
    pipeline as ``sharded_two_phase``, orchestrated natively, for callers
    that cannot run one process per GPU."""

    def __init__(self, devices):
        import ctypes as C
        from . import _native as N
        devs = list(int(d) for d in devices)
        if not devs:
            raise ValueError("a communicator needs at least one device")
        arr = (C.c_int * len(devs))(*devs)
        h = C.c_void_p()
        N.check(N.lib().gc_comm_init(len(devs), arr, C.byref(h)))
        self._h, self.devices = h, devs

    @property
    def size(self) -> int:
        from . import _native as N
        return int(N.lib().gc_comm_size(self._h))

    @property
    def loopback(self) -> bool:
        from . import _native as N
        return bool(N.lib().gc_comm_is_loopback(self._h))

    def close(self):
        from . import _native as N
        if self._h:
            N.lib().gc_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _shards(self, g, spec, balance=None):
        """Row blocks of a device graph, one per rank (each copied to the
        rank's device), with the lowered spec (its BFS source computed on the
        whole graph, sampling.py:130-132)."""
        import ctypes as C
        from . import _native as N
        from .api import LoweredSpec, _csr
        torch = _torch()
        if not g.on_device:
            g = g.cuda()
        low = LoweredSpec(spec, g, g.n)
        bounds = shard_bounds(g.offsets if g._h_off is not None else g._d_off, self.size,
                              balance or shard_balance(spec))
        csrs = (N.Csr * self.size)()
        keep = []
        for r, (lo, hi) in enumerate(bounds):
            with torch.cuda.device(self.devices[r]):
                sh = shard_graph(g, lo, hi)
                off, tgt = sh.device_arrays()
                off = off.to(f"cuda:{self.devices[r]}")
                tgt = tgt.to(f"cuda:{self.devices[r]}")
                keep += [off, tgt]
                csrs[r].n, csrs[r].m = g.n, int(tgt.numel())
                csrs[r].offsets = off.data_ptr()
                csrs[r].targets = tgt.data_ptr() if tgt.numel() else None
        lo = (C.c_int64 * self.size)(*[b[0] for b in bounds])
        hi = (C.c_int64 * self.size)(*[b[1] for b in bounds])
        return csrs, lo, hi, low, keep

    def static_connectivity(self, g, spec):
        """Canonical labels on every rank (list of device tensors) + stats."""
        import ctypes as C
        from . import _native as N
        torch = _torch()
        csrs, lo, hi, low, keep = self._shards(g, spec)
        labels = [torch.empty(max(g.n, 4), dtype=torch.int32, device=f"cuda:{d}") for d in self.devices]
        ptrs = (C.c_void_p * self.size)(*[t.data_ptr() for t in labels])
        st = N.Stats()
        N.check(N.lib().gc_comm_static_cc(self._h, csrs, lo, hi, C.byref(low.s), ptrs, C.byref(st)))
        return [t[:g.n] for t in labels], st

    def spanning_forest(self, g, spec):
        """(labels per rank, [(fu, fv)] per rank: a spanning forest of the
        whole graph on every rank, stats)."""
        import ctypes as C
        from . import _native as N
        torch = _torch()
        csrs, lo, hi, low, keep = self._shards(g, spec)
        n = g.n
        mk = (lambda d: torch.empty(max(n, 4), dtype=torch.int32, device=f"cuda:{d}"))
        labels = [mk(d) for d in self.devices]
        fu = [mk(d) for d in self.devices]
        fv = [mk(d) for d in self.devices]
        P = C.c_void_p * self.size
        cnt = (C.c_int64 * self.size)()
        st = N.Stats()
        N.check(N.lib().gc_comm_spanning_forest(self._h, csrs, lo, hi, C.byref(low.s),
                                                P(*[t.data_ptr() for t in labels]), P(*[t.data_ptr() for t in fu]),
                                                P(*[t.data_ptr() for t in fv]), cnt, C.byref(st)))
        return ([t[:n] for t in labels], [(fu[r][:cnt[r]], fv[r][:cnt[r]]) for r in range(self.size)], st)
