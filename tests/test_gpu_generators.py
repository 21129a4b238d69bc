"""Device generators / CSR build vs the reference fixtures and the C oracle."""
import numpy as np
import pytest

import oracle
from golden_data import h
from paper_2008_11839_b200 import EdgeList, MalformedInputError, build_csr, gen_rmat, gen_uniform_pairs

pytestmark = pytest.mark.gpu


def test_gen_rmat_bit_exact(golden):
    el = gen_rmat(7, 4, seed=2)
    assert el.edges.tolist() == golden.rmat["s7_ef4_seed2_edges"]
    for key in ["s10_ef8_seed3", "s12_ef8_seed1", "s16_ef8_seed1"]:
        parts = key.split("_")
        scale, ef, seed = int(parts[0][1:]), int(parts[1][2:]), int(parts[2][4:])
        el = gen_rmat(scale, ef, seed=seed, device=True)
        pin = golden.rmat[key]
        assert h(el.edges.cpu().numpy()) == pin["edges_hash"], key
        g = build_csr(el, keep_host=True)
        assert g.m == pin["m"] and h(g.offsets) == pin["offsets_hash"] and h(g.targets) == pin["targets_hash"]


def test_build_csr_matches_golden(golden):
    for name, (n, off, tgt, _) in golden.graphs.items():
        src = np.repeat(np.arange(n), np.diff(off))
        e = np.column_stack((src, tgt))
        e = np.vstack([e, e[:5]]) if len(e) else e.reshape(-1, 2)
        g = build_csr(EdgeList(n, e[np.random.default_rng(1).permutation(len(e))]))
        assert np.array_equal(g.offsets, off) and np.array_equal(g.targets, tgt), name


def test_build_csr_rejects_out_of_range():
    with pytest.raises(MalformedInputError):
        build_csr(EdgeList(3, np.array([[0, 3]])))


def test_uniform_pairs_match_numpy():
    el = gen_uniform_pairs(12, 5000, seed=3, device=False)
    ref = np.random.default_rng(3).integers(0, 1 << 12, size=(5000, 2), dtype=np.int64)
    assert np.array_equal(el.edges, ref)


def test_rmat_s20_vs_oracle():
    el = gen_rmat(18, 8, seed=5, device=True)
    n, e = oracle.gen_rmat(18, 8, seed=5)
    assert np.array_equal(el.edges.cpu().numpy(), e)
