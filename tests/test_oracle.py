"""Pin the C oracle against the reference-generated fixtures (CPU only)."""
import numpy as np
import pytest

import oracle
from golden_data import h


def test_oracle_components_match_reference(golden):
    for name, (n, off, tgt, ref) in golden.graphs.items():
        lab, c = oracle.components(n, off, tgt)
        assert np.array_equal(lab, ref), name
        assert c == len(np.unique(ref)) if n else c == 0


def test_oracle_build_csr_matches_reference(golden):
    for name, (n, off, tgt, _) in golden.graphs.items():
        ue = []
        for u in range(n):
            for t in tgt[off[u]:off[u + 1]]:
                if u < t:
                    ue.append((u, t))
        # shuffled, duplicated, with self-loops: normalisation must undo it
        e = np.array(ue + ue[:3] + [(0, 0)] if n else [], dtype=np.int64).reshape(-1, 2)
        e = e[np.random.default_rng(0).permutation(len(e))]
        o2, t2 = oracle.build_csr(n, e[:, ::-1] if len(e) else e)
        assert np.array_equal(o2, off) and np.array_equal(t2, tgt), name


def test_oracle_rmat_matches_reference(golden):
    n, e = oracle.gen_rmat(7, 4, seed=2)
    assert e.tolist() == golden.rmat["s7_ef4_seed2_edges"]
    for key in ["s10_ef8_seed3", "s12_ef8_seed1", "s16_ef8_seed1"]:
        sc, ef, seed = (int(x[1:]) if x[0] == "s" and x[1:].isdigit() else None for x in key.split("_")[:1]), None, None
        scale = int(key.split("_")[0][1:])
        ef = int(key.split("_")[1][2:])
        seed = int(key.split("_")[2][4:])
        n, e = oracle.gen_rmat(scale, ef, seed=seed)
        pin = golden.rmat[key]
        assert h(e) == pin["edges_hash"], key
        off, tgt = oracle.build_csr(n, e)
        assert len(tgt) == pin["m"] and h(off) == pin["offsets_hash"] and h(tgt) == pin["targets_hash"]
        lab, c = oracle.components(n, off, tgt)
        assert c == pin["components"] and h(lab) == pin["oracle_hash"], key


def test_rmat_frozen_shape():
    # test_graphs.py:105-118: gen_rmat(7, 4, seed=2) -> m=710, 4 comps, largest 125
    n, e = oracle.gen_rmat(7, 4, seed=2)
    off, tgt = oracle.build_csr(n, e)
    lab, c = oracle.components(n, off, tgt)
    assert len(tgt) == 710 and c == 4 and np.bincount(lab).max() == 125


def test_check_forest_clauses():
    # triangle + isolate (test_driver.py:202-209)
    off, tgt = oracle.build_csr(4, np.array([(0, 1), (1, 2), (2, 0)]))
    lab, _ = oracle.components(4, off, tgt)
    fu = np.array([-1, 0, 1, -1]); fv = np.array([-1, 1, 2, -1])
    assert oracle.check_forest(4, off, tgt, fu, fv, lab)["passed"]
    bad = oracle.check_forest(4, off, tgt, np.array([-1, 0, 0, 2]), np.array([-1, 1, 2, 1]), lab)
    assert not bad["clauses"]["acyclic"]["ok"] and not bad["clauses"]["count"]["ok"]
    missing = oracle.check_forest(4, off, tgt, np.array([-1, 0, 1, -1]), np.array([-1, 1, 3, -1]), lab)
    assert not missing["clauses"]["edges_exist"]["ok"]


def test_incremental_replay_golden(golden):
    g = golden.incr["golden"]
    us = [0, 0, 0, 1, 0]; vs = [1, 1, 2, 2, 2]; q = [0, 1, 1, 0, 1]
    # batches of 3 then 2 -> replay per batch boundary
    b1, l1 = oracle.incremental_replay(5, us[:3], vs[:3], q[:3], 3)
    assert b1.tolist() == g["bits"][0]
    r = golden.incr["random"]
    ops = r["ops"]
    us = np.array([o[1] for o in ops]); vs = np.array([o[2] for o in ops])
    isq = np.array([o[0] == "q" for o in ops], dtype=np.uint8)
    bits, lab = oracle.incremental_replay(r["capacity"], us, vs, isq, r["batch"])
    exp = r["results"]["none+async+halve"]
    flat = [b for bb in exp["bits"] for b in bb]
    assert bits.tolist() == flat
    # canonical labels: uninitialised singletons keep their own id
    assert lab.tolist() == exp["labels"]
