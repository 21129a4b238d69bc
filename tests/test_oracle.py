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


# ---- the C/OpenMP pipeline port (bench reference arm, bench_configs CPU
# baselines) pinned against the reference's own statistics -----------------

def _bfs_source(n, off, seed=1, probes=64):
    """sampling.py:130-132"""
    pr = np.unique(np.random.default_rng(seed).integers(0, n, size=probes))
    return int(pr[np.argmax(np.diff(off)[pr])])


PORT_SPECS = ["none+async+naive", "none+async+halve", "none+async+compress", "none+rem_cas+naive+splice",
              "none+rem_cas+halve+split", "kout+rem_cas+halve+splice", "kout+async+halve", "none+sv",
              "kout+sv", "bfs+sv", "bfs+async+halve", "bfs+rem_cas+split+halve"] + \
             [f"{s}+lt_{v}" for s in ("none", "kout") for v in oracle._LT]


@pytest.mark.parametrize("threads", [1, 4])
def test_port_matches_reference_stats_small_suite(golden, threads):
    """Labels hash, component count, rounds, sample / finish inspections and
    cov equal the reference's workers=1 statistics (spec_stats.json) on
    every suite graph, single- and multi-threaded."""
    for name, (n, off, tgt, orc) in golden.graphs.items():
        for text in PORT_SPECS:
            ref = golden.spec_stats[name].get(text)
            if ref is None:
                continue
            src = _bfs_source(n, off) if text.startswith("bfs") and n and len(tgt) else -1
            lab, st, _ = oracle.pipeline(n, off, tgt, text, threads=threads, bfs_source=src)
            assert np.array_equal(lab, orc), (name, text)
            got = {"components": st["components"], "rounds": st["rounds"],
                   "insp_sample": st["insp_sample"], "insp_finish": st["insp_finish"]}
            assert got == {k: ref[k] for k in got}, (name, text)
            cov = st["lmax_count"] / n if n else 1.0
            assert cov == pytest.approx(ref["cov"], rel=1e-12), (name, text)


def test_port_matches_reference_s16_pins(golden):
    """BASELINE config 1 (RMAT s16 ef8 seed 1): every pinned spec the port
    covers reproduces the reference's labels and statistics."""
    pin = golden.rmat["s16_ef8_seed1"]
    n, e = oracle.gen_rmat(16, 8, seed=1)
    off, tgt = oracle.build_csr(n, e)
    covered = 0
    for text, ref in pin["specs"].items():
        try:
            oracle.parse(text)
        except ValueError:
            continue
        covered += 1
        src = _bfs_source(n, off) if text.startswith("bfs") else -1
        lab, st, _ = oracle.pipeline(n, off, tgt, text, bfs_source=src)
        assert h(lab) == ref["labels"], text
        got = {"components": st["components"], "rounds": st["rounds"], "insp_sample": st["insp_sample"],
               "insp_finish": st["insp_finish"]}
        assert got == {k: ref[k] for k in got}, text
        assert st["lmax_count"] / n == pytest.approx(ref["cov"], rel=1e-12), text
    assert covered >= 10


def test_port_forest_clauses(golden):
    """spanning_forest with bfs / none / k-out samplers + union-find: the
    port's forest passes the four clauses with exactly n - c edges."""
    for name, (n, off, tgt, orc) in golden.graphs.items():
        for text in ["bfs+async+halve", "none+async+halve", "kout+rem_cas+halve+split"]:
            src = _bfs_source(n, off) if text.startswith("bfs") and n and len(tgt) else -1
            lab, st, _, (fu, fv) = oracle.pipeline(n, off, tgt, text, threads=4, forest=True, bfs_source=src)
            rep = oracle.check_forest(n, off, tgt, fu, fv, orc)
            assert rep["passed"], (name, text, rep)


def test_port_bfs_forest_matches_reference(golden):
    """BFS forests are deterministic in the reference (min-parent, re-rooted
    at the component minimum): bfs+sv's forest hash (the rounds finish adds
    nothing on suite graphs whose BFS component is everything) equals the
    reference's where the finish records no edges."""
    checked = 0
    for name, (n, off, tgt, orc) in golden.graphs.items():
        ref = golden.spec_stats[name].get("bfs+sv")
        if not ref or "forest" not in ref or ref["insp_finish"] != 0:
            continue
        src = _bfs_source(n, off) if n and len(tgt) else -1
        _, _, _, (fu, fv) = oracle.pipeline(n, off, tgt, "bfs+async+halve", forest=True, bfs_source=src)
        pairs = [(int(a), int(b)) if a >= 0 else None for a, b in zip(fu, fv)]
        flat = np.array([x for p in pairs for x in (p if p else (-1, -1))], dtype=np.int64)
        assert h(flat) == ref["forest"], name
        checked += 1
    assert checked >= 1


def test_port_incremental_insert_matches_replay(golden):
    r = golden.incr["random"]
    cap = r["capacity"]
    ops = r["ops"]
    us = np.array([o[1] for o in ops if o[0] == "i"], dtype=np.int32)
    vs = np.array([o[2] for o in ops if o[0] == "i"], dtype=np.int32)
    P = np.full(cap, cap, dtype=np.int32)
    for b0 in range(0, len(us), 37):
        oracle.incr_insert(cap, P, us[b0:b0 + 37], vs[b0:b0 + 37], "async", "halve", threads=4)
    _, lab = oracle.incremental_replay(cap, us, vs, np.zeros(len(us), dtype=np.uint8), len(us))
    got = np.where(P == cap, np.arange(cap), P)
    for v in range(cap):  # chase to roots
        while got[got[v]] != got[v]:
            got[v] = got[got[v]]
    got = np.array([got[v] for v in range(cap)])
    assert got.tolist() == lab.tolist()
