"""Shared helpers for the -m gpu parity tests."""
from __future__ import annotations

import numpy as np

from paper_2008_11839_b200 import Graph


def graph_of(golden, name) -> Graph:
    n, off, tgt, _ = golden.graphs[name]
    return Graph(n, off, tgt)
