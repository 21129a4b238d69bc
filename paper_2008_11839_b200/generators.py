"""CSR normalisation and synthetic graph families (reference graphs.py:90-121,
210-320).

``build_csr`` and the large generators run on the GPU: ``gen_rmat``
reproduces numpy's PCG64 stream, so the device edge list equals the
reference's ``gen_rmat(scale, edge_factor, seed=...)`` bit for bit, and
``gen_uniform_pairs`` equals ``default_rng(seed).integers(0, n, size=(k, 2))``
for power-of-two n.  The small deterministic families build their edge lists
with numpy (they are tiny) and normalise through the device ``build_csr``.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .errors import ConfigError, MalformedInputError
from .graph import VERTEX_LIMIT, EdgeList, Graph


def _torch():
    import torch
    return torch


def _stream():
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _pcg_state(seed: int):
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return (s >> 64) & m, s & m, (inc >> 64) & m, inc & m


def build_csr(el: EdgeList, keep_host: bool = True) -> Graph:
    """Symmetrize, drop self-loops, dedupe, sort rows (graphs.py:90-121), on device."""
    torch = _torch()
    n = int(el.n)
    if n < 0 or n >= VERTEX_LIMIT:
        raise MalformedInputError(f"vertex count {n} outside [0, 2^31)")
    edges = el.edges
    k = len(el)
    if isinstance(edges, np.ndarray) and k:
        if edges.min() < 0 or edges.max() >= n:
            bad = edges[(edges[:, 0] >= n) | (edges[:, 1] >= n) | (edges < 0).any(axis=1)][0]
            raise MalformedInputError(f"edge {tuple(int(x) for x in bad)} has endpoint outside [0, {n})")
    if not torch.cuda.is_available():
        raise N.NativeError("build_csr runs on the GPU (no CUDA device found)")
    lib = N.lib()
    if isinstance(edges, np.ndarray):
        dev = torch.from_numpy(np.ascontiguousarray(edges)).to("cuda")
    else:
        dev = edges.to("cuda")
    src = dev[:, 0].contiguous()
    dst = dev[:, 1].contiguous()
    off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    tgt = torch.empty(max(2 * k, 1), dtype=torch.int32, device="cuda")
    ws = torch.empty(max(int(lib.gc_build_csr_workspace(n, k)), 256), dtype=torch.uint8, device="cuda")
    m = C.c_int64(0)
    N.check(lib.gc_build_csr(n, src.data_ptr() if k else None, dst.data_ptr() if k else None, k,
                             off.data_ptr() if n else None, tgt.data_ptr(), C.byref(m), ws.data_ptr(),
                             ws.numel(), _stream()))
    del ws
    if n == 0:
        off = torch.zeros(1, dtype=torch.int64, device="cuda")
    tgt = tgt[: m.value].clone()
    g = Graph(n, off, tgt)
    if keep_host and n <= (1 << 22):
        g._host()
    return g


def gen_rmat(scale: int, edge_factor: int, a: float = 0.5, b: float = 0.1, c: float = 0.1,
             seed: int = 0, device: bool = False) -> EdgeList:
    """RMAT with per-level +-10% noise (graphs.py:210-245), generated on the
    GPU with the reference's exact PCG64 stream.  Returns a device EdgeList
    when device=True, else a numpy one."""
    if scale < 1:
        raise ConfigError(f"scale must be >= 1, got {scale}")
    if a + b + c > 1.0 + 1e-12:
        raise ConfigError(f"quadrant probabilities sum to {a + b + c:.4f} > 1")
    torch = _torch()
    d = 1.0 - a - b - c
    n = 1 << scale
    m = edge_factor * n
    base = (C.c_double * 4)(a, b, c, d)
    sh, sl, ih, il = _pcg_state(seed)
    src = torch.empty(max(m, 1), dtype=torch.int64, device="cuda")
    dst = torch.empty(max(m, 1), dtype=torch.int64, device="cuda")
    N.check(N.lib().gc_gen_rmat(scale, m, base, sh, sl, ih, il, src.data_ptr(), dst.data_ptr(),
                                _stream()))
    e = torch.stack([src[:m], dst[:m]], dim=1)
    return EdgeList(n, e if device else e.cpu().numpy())


def gen_uniform_pairs(log2n: int, num_pairs: int, seed: int = 1, device: bool = True) -> EdgeList:
    """default_rng(seed).integers(0, 2^log2n, size=(num_pairs, 2)) on device
    (the uniform-random family of tests/helpers.py:33-37)."""
    torch = _torch()
    n = 1 << log2n
    sh, sl, ih, il = _pcg_state(seed)
    src = torch.empty(max(num_pairs, 1), dtype=torch.int64, device="cuda")
    dst = torch.empty(max(num_pairs, 1), dtype=torch.int64, device="cuda")
    N.check(N.lib().gc_gen_uniform_pow2(log2n, num_pairs, sh, sl, ih, il, src.data_ptr(),
                                        dst.data_ptr(), _stream()))
    e = torch.stack([src[:num_pairs], dst[:num_pairs]], dim=1)
    return EdgeList(n, e if device else e.cpu().numpy())


def grid3d_edges(side: int) -> EdgeList:
    """6-neighbour side^3 grid with natural row-major ids, on device."""
    torch = _torch()
    n = side ** 3
    idx = torch.arange(n, dtype=torch.int64, device="cuda").reshape(side, side, side)
    parts = [torch.stack([idx[:-1].reshape(-1), idx[1:].reshape(-1)], 1),
             torch.stack([idx[:, :-1].reshape(-1), idx[:, 1:].reshape(-1)], 1),
             torch.stack([idx[:, :, :-1].reshape(-1), idx[:, :, 1:].reshape(-1)], 1)]
    return EdgeList(n, torch.cat(parts, 0))


def path_graph(n: int) -> Graph:
    e = np.column_stack((np.arange(n - 1), np.arange(1, n))) if n > 1 else np.empty((0, 2))
    return build_csr(EdgeList(n, e))


def star_graph(n: int, center: int = 0) -> Graph:
    leaves = np.array([v for v in range(n) if v != center], dtype=np.int64)
    return build_csr(EdgeList(n, np.column_stack((np.full(len(leaves), center), leaves))))


def clique_graph(n: int) -> Graph:
    u, v = np.triu_indices(n, k=1)
    return build_csr(EdgeList(n, np.column_stack((u, v))))


def grid_graph(rows: int, cols: int) -> Graph:
    idx = np.arange(rows * cols).reshape(rows, cols)
    e = np.vstack((np.column_stack((idx[:, :-1].ravel(), idx[:, 1:].ravel())),
                   np.column_stack((idx[:-1, :].ravel(), idx[1:, :].ravel()))))
    return build_csr(EdgeList(rows * cols, e))


def disjoint_union(parts: list[Graph]) -> Graph:
    chunks, base = [], 0
    for g in parts:
        if g.m:
            chunks.append(g.undirected_edges() + base)
        base += g.n
    e = np.vstack(chunks) if chunks else np.empty((0, 2), dtype=np.int64)
    return build_csr(EdgeList(base, e))
