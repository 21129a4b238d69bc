"""Spanning-forest parity: the four check_forest clauses (validate.py:178-244)
for every root-based spec; bit-identical forests for the deterministic
recorders (SV / LT minimum edge index, BFS first discoverer)."""
import numpy as np
import pytest

import oracle
from golden_data import h
from gpu_util import graph_of
from paper_2008_11839_b200 import (ConfigError, enumerate_specs, format_spec, parse_spec,
                                   spanning_forest, spanning_forest_device)

pytestmark = pytest.mark.gpu


def test_forest_all_root_based_specs(golden):
    specs = [s for s in enumerate_specs() if s.is_root_based()]
    for name in golden.names():
        n, off, tgt, orc = golden.graphs[name]
        g = graph_of(golden, name)
        for spec in specs:
            df, st = spanning_forest_device(g, spec)
            fu = df.fu.cpu().numpy(); fv = df.fv.cpu().numpy()
            rep = oracle.check_forest(n, off, tgt, fu, fv, orc)
            assert rep["passed"], (name, format_spec(spec), rep)
            ref = golden.spec_stats[name][format_spec(spec)]
            assert int((fu >= 0).sum()) == ref["forest_count"]
            assert st.component_count == n - ref["forest_count"]
            if "forest" in ref:
                flat = np.stack([fu, fv], 1).reshape(-1)
                assert h(flat) == ref["forest"], (name, format_spec(spec))


@pytest.mark.parametrize("text", ["none+lp", "none+stergiou", "none+lt_cusa", "none+rem_cas+naive+splice"])
def test_forest_rejects_non_root_based(text, golden):
    with pytest.raises(ConfigError):
        spanning_forest(graph_of(golden, "path4"), parse_spec(text))


def test_forest_triangle(golden):
    fe, st = spanning_forest(graph_of(golden, "triangle_iso"), parse_spec("none+async+halve"))
    assert len(fe) == 2 and st.component_count == 2


def _bfs_min_parent_forest(n, off, tgt, src):
    """numpy restatement of the reference BFS forest (sampling.py:139-171):
    level-synchronous BFS from src; a vertex's parent is its first
    discoverer, which for the ascending frontier order of the reference is
    its smallest neighbour one level up; then the tree is re-rooted at the
    component minimum.  Returns (fu, fv) slots for the BFS component
    (other slots -2 = not compared) and the component mask."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import breadth_first_order
    A = sp.csr_matrix((np.ones(len(tgt), np.int8), tgt, off), shape=(n, n))
    order, pred = breadth_first_order(A, src, directed=True, return_predecessors=True)
    level = np.full(n, -1, np.int64)
    level[src] = 0
    for v in order[1:]:
        level[v] = level[pred[v]] + 1
    row = np.repeat(np.arange(n), np.diff(off))
    up = (level[row] >= 1) & (level[tgt] == level[row] - 1)
    cand = np.where(up, tgt.astype(np.int64), np.iinfo(np.int64).max)
    par = np.full(n, -1, np.int64)
    nz = np.diff(off) > 0
    mins = np.minimum.reduceat(cand, off[:-1][nz]) if nz.any() else np.zeros(0, np.int64)
    par[np.nonzero(nz)[0]] = mins
    comp = level >= 0
    par[~comp] = -1
    par[src] = -1
    fu = np.full(n, -2, np.int64)
    fv = np.full(n, -2, np.int64)
    fu[comp] = par[comp]
    fv[comp] = np.where(par[comp] >= 0, np.nonzero(comp)[0], -1)
    mn = int(np.nonzero(comp)[0].min())
    assert (par[comp & (level >= 1)] >= 0).all() and (par[comp] < n).all()
    cur = mn
    fu[cur] = fv[cur] = -1
    while cur != src:  # reverse the path mn -> ... -> src (levels strictly drop)
        p = int(par[cur])
        fu[p], fv[p] = cur, p
        cur = p
    return fu, fv, comp


@pytest.mark.parametrize("log2n", [14, 18])
def test_bfs_forest_matches_min_parent_tree(log2n):
    """Uniform random graphs (tests/helpers.py:33-37 family) large enough for
    wide top-down levels (frontier >= 256 at these sizes: bitmap mark +
    parent pull) and bottom-up levels: the BFS-component slots must equal
    the reference's BFS tree exactly; the rest (union-find finish) is
    checked by the four clauses."""
    from paper_2008_11839_b200 import build_csr, check_forest, gen_uniform_pairs, spanning_forest_device
    from paper_2008_11839_b200.api import bfs_source
    g = build_csr(gen_uniform_pairs(log2n, 4 << log2n, seed=5, device=True))
    spec = parse_spec("bfs+async+halve")
    src = bfs_source(g, spec.bfs_probes, spec.seed)
    ef_u, ef_v, comp = _bfs_min_parent_forest(g.n, g.offsets, g.targets, src)
    df, st = spanning_forest_device(g, spec)
    fu = df.fu.cpu().numpy().astype(np.int64)
    fv = df.fv.cpu().numpy().astype(np.int64)
    assert np.array_equal(fu[comp], ef_u[comp])
    assert np.array_equal(fv[comp], ef_v[comp])
    ref, _ = oracle.components(g.n, g.offsets, g.targets)
    assert check_forest(g, df, ref)["passed"]


def test_bfs_source_picked_on_device(golden):
    """Device-only graphs pick the BFS source in the seed kernel from the probe
    list (sampling.py:130-132); the forests must equal the host-picked ones
    (and the reference's hashes where the golden file pins them)."""
    import dataclasses
    from paper_2008_11839_b200 import gen_rmat, build_csr
    # deterministic finishes (SV / LT record the minimum edge index), so the
    # whole forest is a function of the source
    specs = [parse_spec(t) for t in ("bfs+sv", "bfs+lt_prs")]
    specs.append(dataclasses.replace(parse_spec("bfs+sv"), bfs_probes=1000, seed=7))
    for name in golden.names():
        n, off, tgt, orc = golden.graphs[name]
        for spec in specs:
            g_host = graph_of(golden, name)
            g_dev = graph_of(golden, name).cuda()
            g_dev.drop_host()
            a, _ = spanning_forest_device(g_host, spec)
            b, _ = spanning_forest_device(g_dev, spec)
            assert np.array_equal(a.fu.cpu().numpy(), b.fu.cpu().numpy()), (name, format_spec(spec))
            assert np.array_equal(a.fv.cpu().numpy(), b.fv.cpu().numpy()), (name, format_spec(spec))
    # a device-generated graph against its host-backed copy
    g = build_csr(gen_rmat(14, 8, seed=3, device=True), keep_host=False)
    gh = g.cuda()
    gh._h_off = g._d_off.cpu().numpy()
    gh._h_tgt = g._d_tgt.cpu().numpy()
    spec = parse_spec("bfs+sv")
    a, _, pa = spanning_forest_device(gh, spec, want_parent=True)
    b, _, pb = spanning_forest_device(g, spec, want_parent=True)
    assert np.array_equal(a.fu.cpu().numpy(), b.fu.cpu().numpy())
    assert np.array_equal(pa.cpu().numpy(), pb.cpu().numpy())
