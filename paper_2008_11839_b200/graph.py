"""Graph containers (reference graphs.py:28-121) with device residency.

``Graph`` keeps the reference's symmetrized-CSR contract — int64 offsets[n+1],
int32 targets[m] sorted per row, no self-loops or duplicates, ``m`` counts
directed entries — but its arrays can live on the host (numpy or pinned
torch), on the GPU (torch CUDA tensors), or both.  Kernels always read the
device copy; host views are materialised lazily for callers that index them.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import MalformedInputError

VERTEX_LIMIT = 2 ** 31


def _torch():
    import torch
    return torch


@dataclass
class EdgeList:
    """COO pairs over [0, n) (graphs.py:28-40); duplicates / self-loops allowed."""

    n: int
    edges: object  # (k, 2) int64: numpy array or torch tensor (host or CUDA)

    def __post_init__(self):
        torch = _torch()
        if isinstance(self.edges, torch.Tensor):
            self.edges = self.edges.to(torch.int64).reshape(-1, 2)
        else:
            self.edges = np.asarray(self.edges, dtype=np.int64).reshape(-1, 2)

    def __len__(self) -> int:
        return int(self.edges.shape[0])


class Graph:
    """Symmetrized CSR; ``m`` counts directed entries (graphs.py:43-87)."""

    def __init__(self, n: int, offsets, targets):
        torch = _torch()
        self.n = int(n)
        self._h_off = self._h_tgt = None
        self._d_off = self._d_tgt = None
        if isinstance(offsets, torch.Tensor) and offsets.is_cuda:
            self._d_off = offsets.to(torch.int64).contiguous()
            self._d_tgt = targets.to(torch.int32).contiguous()
            self.m = int(self._d_tgt.numel())
        else:
            if isinstance(offsets, torch.Tensor):
                self._h_off = offsets.to(torch.int64).contiguous()
                self._h_tgt = targets.to(torch.int32).contiguous()
            else:
                self._h_off = np.ascontiguousarray(offsets, dtype=np.int64)
                self._h_tgt = np.ascontiguousarray(targets, dtype=np.int32)
            self.m = int(len(self._h_tgt))
        if self.n < 0 or self.n >= VERTEX_LIMIT:
            raise MalformedInputError(f"vertex count {self.n} outside [0, 2^31)")

    # ----------------------------------------------------------- host views
    def _host(self):
        if self._h_off is None:
            self._h_off = self._d_off.cpu().numpy()
            self._h_tgt = self._d_tgt.cpu().numpy()
        off, tgt = self._h_off, self._h_tgt
        torch = _torch()
        if isinstance(off, torch.Tensor):
            off, tgt = off.numpy(), tgt.numpy()
        return off, tgt

    @property
    def offsets(self) -> np.ndarray:
        return self._host()[0]

    @property
    def targets(self) -> np.ndarray:
        return self._host()[1]

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets)

    def degree(self, v: int) -> int:
        off = self.offsets
        return int(off[v + 1] - off[v])

    def neighbors(self, v: int) -> np.ndarray:
        off, tgt = self._host()
        return tgt[off[v]:off[v + 1]]

    def undirected_edges(self) -> np.ndarray:
        """(u, v) with u < v, one per undirected edge (graphs.py:79-84)."""
        off, tgt = self._host()
        src = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(off))
        dst = tgt.astype(np.int64)
        keep = src < dst
        return np.column_stack((src[keep], dst[keep]))

    # --------------------------------------------------------- device views
    def device_arrays(self, stream=None):
        """(offsets int64, targets int32) CUDA tensors, uploaded once and cached."""
        torch = _torch()
        if self._d_off is None:
            off, tgt = self._h_off, self._h_tgt
            if not isinstance(off, torch.Tensor):
                off, tgt = torch.from_numpy(off), torch.from_numpy(tgt)
            self._d_off = off.to("cuda", non_blocking=True)
            self._d_tgt = tgt.to("cuda", non_blocking=True)
        return self._d_off, self._d_tgt

    def upload(self):
        """Fresh device copy of the host arrays (used for end-to-end timing)."""
        torch = _torch()
        off, tgt = self._h_off, self._h_tgt
        if off is None:
            return self.device_arrays()
        if not isinstance(off, torch.Tensor):
            off, tgt = torch.from_numpy(off), torch.from_numpy(tgt)
        return off.to("cuda", non_blocking=True), tgt.to("cuda", non_blocking=True)

    @property
    def on_device(self) -> bool:
        return self._d_off is not None

    def cuda(self) -> "Graph":
        d_off, d_tgt = self.device_arrays()
        g = Graph(self.n, d_off, d_tgt)
        g._h_off, g._h_tgt = self._h_off, self._h_tgt
        if hasattr(self, "row_block"):  # a sharded row block stays one
            g.row_block = self.row_block
        return g

    def drop_host(self) -> None:
        if self._d_off is not None:
            self._h_off = self._h_tgt = None

    def __repr__(self) -> str:
        return f"Graph(n={self.n}, m={self.m}, device={self.on_device})"
