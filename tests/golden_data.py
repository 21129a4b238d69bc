"""Loader for the reference-generated fixtures in tests/golden/ (see
tests/golden/make_golden.py).  Test infrastructure only."""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

G = Path(__file__).resolve().parent / "golden"


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()[:16]


class Golden:
    def __init__(self):
        z = np.load(G / "small_suite.npz")
        self.graphs = {}
        for key in z.files:
            if key.endswith("__n"):
                name = key[:-3]
                self.graphs[name] = (int(z[key][0]), z[name + "__off"], z[name + "__tgt"],
                                     z[name + "__oracle"])
        self.spec_stats = json.loads((G / "spec_stats.json").read_text())
        self.rmat = json.loads((G / "rmat.json").read_text())
        self.incr = json.loads((G / "incremental.json").read_text())

    def names(self):
        return sorted(self.graphs)
