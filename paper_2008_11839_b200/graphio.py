"""Graph files and the remaining reference generators (graphs.py:124-308).

* GCN1 binary CSR (magic "GCN1", u64 n, u64 m, u64 offsets[n+1], u32
  targets[m], little endian) — graphs.py:170-190.  ``load_graph_binary``
  reads the file straight into pinned host buffers and, with
  ``device=True``, issues the host->device copy of each chunk as soon as it
  is read, so disk reads overlap the PCIe transfer.
* ``gen_ba`` / ``gnp_graph`` — the reference's small deterministic
  generators (numpy ``default_rng`` streams, so outputs are identical).
"""
from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .errors import ConfigError, MalformedInputError
from .generators import build_csr
from .graph import EdgeList, Graph

BINARY_MAGIC = b"GCN1"
_CHUNK = 64 << 20  # bytes per read / copy chunk


def _torch():
    import torch
    return torch


# ------------------------------------------------------------------ edges

def graph_to_edge_list(g: Graph) -> EdgeList:
    """graphs.py:124-126: one pair per undirected edge, u < v."""
    return EdgeList(g.n, g.undirected_edges())


# ---------------------------------------------------------------- binary

def save_graph_binary(g: Graph, path) -> None:
    """graphs.py:170-177."""
    with open(path, "wb") as fh:
        fh.write(BINARY_MAGIC)
        fh.write(struct.pack("<QQ", g.n, g.m))
        fh.write(np.asarray(g.offsets).astype("<u8").tobytes())
        fh.write(np.asarray(g.targets).astype("<u4").tobytes())


def is_binary_graph(path) -> bool:
    with open(path, "rb") as fh:
        return fh.read(4) == BINARY_MAGIC


def _read_into(fh, dst_np: np.ndarray, dev=None, src_t=None) -> int:
    """Fill a pinned host array chunk by chunk; after each chunk, enqueue its
    async copy to the matching slice of ``dev``.  Returns bytes read."""
    view = memoryview(dst_np).cast("B")
    total = 0
    step = max(_CHUNK // dst_np.itemsize, 1) * dst_np.itemsize
    while total < len(view):
        got = fh.readinto(view[total:total + step])
        if not got:
            break
        if dev is not None and got % dst_np.itemsize == 0:
            a, b = total // dst_np.itemsize, (total + got) // dst_np.itemsize
            dev[a:b].copy_(src_t[a:b], non_blocking=True)
        total += got
    return total


def load_graph_binary(path, device: bool = False) -> Graph:
    """graphs.py:180-190.  The arrays land in pinned host memory; with
    ``device=True`` the device copy streams in behind the file reads and the
    Graph is returned device-resident (host views stay available)."""
    torch = _torch()
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != BINARY_MAGIC:
            raise MalformedInputError(f"{path}: bad magic {magic!r}")
        head = fh.read(16)
        if len(head) != 16:
            raise MalformedInputError(f"{path}: truncated binary graph")
        n, m = struct.unpack("<QQ", head)
        if n >= 2 ** 31:
            raise MalformedInputError(f"{path}: vertex count {n} outside [0, 2^31)")
        pin = torch.cuda.is_available()
        off_t = torch.empty(n + 1, dtype=torch.int64, pin_memory=pin)
        tgt_t = torch.empty(m, dtype=torch.int32, pin_memory=pin)
        d_off = d_tgt = None
        if device:
            d_off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
            d_tgt = torch.empty(m, dtype=torch.int32, device="cuda")
        # u64 / u32 little endian == int64 / int32 on this host for valid graphs
        got_o = _read_into(fh, off_t.numpy(), d_off, off_t)
        got_t = _read_into(fh, tgt_t.numpy(), d_tgt, tgt_t)
    if got_o != 8 * (n + 1) or got_t != 4 * m:
        raise MalformedInputError(f"{path}: truncated binary graph")
    if device:
        torch.cuda.current_stream().synchronize()
        g = Graph(n, d_off, d_tgt)
        g._h_off, g._h_tgt = off_t, tgt_t
        return g
    return Graph(n, off_t, tgt_t)


def load_graph(path, device: bool = False) -> Graph:
    """graphs.py:198-202 for the binary CSR format.  Text edge lists
    (graphs.py:129-167) are file plumbing outside the accelerated path
    (SURVEY §2): parse them with connlab and hand the arrays to Graph."""
    if not is_binary_graph(path):
        raise MalformedInputError(f"{path}: not a GCN1 binary graph (text edge lists are read by "
                                  "connlab.graphs.load_edge_list; pass its arrays to Graph / build_csr)")
    return load_graph_binary(path, device=device)


# ------------------------------------------------------------- generators

def gen_ba(n: int, attach: int, seed: int = 0) -> EdgeList:
    """graphs.py:248-276: preferential attachment over a degree-weighted
    endpoint pool; same numpy stream, same edges."""
    if attach < 1:
        raise ConfigError(f"attach must be >= 1, got {attach}")
    if n <= attach:
        raise ConfigError(f"need n > attach, got n={n}, attach={attach}")
    rng = np.random.default_rng(seed)
    out = np.empty(((n - attach) * attach, 2), dtype=np.int64)
    pool: list[int] = []
    targets = list(range(attach))
    row = 0
    for source in range(attach, n):
        out[row:row + attach, 0] = source
        out[row:row + attach, 1] = targets
        row += attach
        pool.extend(targets)
        pool.extend([source] * attach)
        chosen: set[int] = set()
        while len(chosen) < attach:
            chosen.add(pool[int(rng.integers(len(pool)))])
        targets = sorted(chosen)
    return EdgeList(n, out)


def gnp_graph(n: int, p: float, seed: int = 0) -> Graph:
    """graphs.py:304-308: Erdos-Renyi G(n, p) over the upper triangle."""
    rng = np.random.default_rng(seed)
    u, v = np.triu_indices(n, k=1)
    keep = rng.random(len(u)) < p
    return build_csr(EdgeList(n, np.column_stack((u[keep], v[keep]))))
