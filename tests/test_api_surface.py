"""The rest of the reference's public API (connlab/__init__.py:12-82):
DisjointSets + union_edge_list, validate.py helpers, graph files and the
small generators — checked against fixtures produced by the reference
(tests/golden/make_golden_api.py)."""
import json

import numpy as np
import pytest

from golden_data import G, h
from paper_2008_11839_b200 import (DisjointSets, EdgeList, FindOp, ForestEdges, Graph, MalformedInputError,
                                   SpliceOp, UnionConfig, UnionOp, all_valid_configs, canonical_labels,
                                   check_forest, gen_ba, is_binary_graph, load_graph, partition_equal,
                                   sampling_stats, union_edge_list)

API = json.loads((G / "api.json").read_text())


# ----------------------------------------------------------------- CPU side

def test_gen_ba_matches_reference():
    for key, want in API["gen_ba"].items():
        n, att, seed = (int(x) for x in key.split(","))
        el = gen_ba(n, att, seed=seed)
        assert el.n == want["n"] and len(el) == want["k"] and h(el.edges) == want["hash"], key
        assert (el.edges[:, 1] < el.edges[:, 0]).all()


def test_text_edge_lists_are_out_of_scope(tmp_path):
    """Text edge lists (graphs.py:129-167) are file plumbing off the
    accelerated path: load_graph takes GCN1 files only and says
    where text files are read."""
    p = tmp_path / "tiny.txt"
    p.write_text("# n 4\n0 2\n3 1\n")
    assert not is_binary_graph(p)
    with pytest.raises(MalformedInputError, match="not a GCN1 binary graph"):
        load_graph(p)


@pytest.mark.gpu
def test_census_helpers_match_reference():
    from paper_2008_11839_b200 import build_csr  # noqa: F401  (GPU not needed below)
    assert partition_equal([0, 0, 2, 3], [5, 5, 1, 0])
    assert not partition_equal([0, 0, 2, 3], [5, 5, 5, 0])
    assert canonical_labels([3, 3, 1, 1, 3]).tolist() == [0, 0, 2, 2, 0]
    # census golden (test_validate.py:106-110): path-4, labels [0,0,2,3]
    g = Graph(4, np.array([0, 1, 3, 5, 6]), np.array([1, 0, 2, 1, 3, 2]))
    cov, ic = sampling_stats(g, [0, 0, 2, 3])
    assert cov == 0.5 and ic == pytest.approx(4 / 6)


@pytest.mark.gpu
def test_sampling_stats_cases():
    # the fixture graph is gen_ba(300, 2, seed=3) symmetrised by the reference
    el = gen_ba(300, 2, seed=3)
    e = el.edges
    u = np.concatenate([e[:, 0], e[:, 1]])
    v = np.concatenate([e[:, 1], e[:, 0]])
    order = np.lexsort((v, u))
    u, v = u[order], v[order]
    keep = np.ones(len(u), bool)
    keep[1:] = (u[1:] != u[:-1]) | (v[1:] != v[:-1])
    u, v = u[keep], v[keep]
    off = np.zeros(301, np.int64)
    np.add.at(off, u + 1, 1)
    g = Graph(300, np.cumsum(off), v)
    for case in API["sampling_stats"]["cases"]:
        cov, ic = sampling_stats(g, case["labels"])
        assert cov == case["cov"] and ic == case["ic"]


# ----------------------------------------------------------------- GPU side

@pytest.mark.gpu
def test_find_traces_every_rule():
    for f in FindOp:
        union = UnionOp.JTB if f is FindOp.TWO_TRY else UnionOp.ASYNC
        ds = DisjointSets(4, UnionConfig(union, f, SpliceOp.NONE))
        import torch
        ds.p.copy_(torch.tensor([0, 0, 1, 2], dtype=torch.int32))
        want = API["find_traces"][f.value]
        assert ds.find_root(3) == want["root"], f
        assert ds.p.cpu().tolist() == want["p"], f


@pytest.mark.gpu
def test_disjoint_sets_every_config():
    edges = np.array(API["ds_edges"], dtype=np.int64)
    for cfg in all_valid_configs():
        ds = DisjointSets(200, cfg)
        union_edge_list(ds, edges[:, 0], edges[:, 1], workers=4)
        lab = ds.labels_array()
        assert h(canonical_labels(lab)) == API["ds_labels"], cfg
        assert ds.same_set(int(edges[0, 0]), int(edges[0, 1]))


@pytest.mark.gpu
def test_disjoint_sets_single_unions_and_forest():
    cfg = UnionConfig(UnionOp.REM_CAS, FindOp.HALVE, SpliceOp.SPLIT_ONE)
    forest = [None] * 6
    ds = DisjointSets(6, cfg, forest=forest)
    assert ds.union(1, 2) is True
    assert ds.union(2, 1) is False
    assert ds.union(4, 5) is True
    assert ds.union(5, 1) is True
    assert not ds.same_set(0, 1) and ds.same_set(4, 2)
    assert sum(e is not None for e in forest) == 3
    assert ds.labels_array().tolist() == [0, 1, 1, 3, 1, 1]


@pytest.mark.gpu
def test_check_forest_reports_match_reference():
    for gname, cases in API["check_forest"].items():
        gd = cases["graph"]
        g = Graph(gd["n"], np.array(gd["off"]), np.array(gd["tgt"]))
        for cname, case in cases.items():
            if cname == "graph":
                continue
            edges = [tuple(e) if e is not None else None for e in case["edges"]]
            rep = json.loads(json.dumps(check_forest(g, ForestEdges(edges), np.array(gd["oracle"]))))
            assert rep == case["report"], (gname, cname, rep)


@pytest.mark.gpu
def test_binary_graph_roundtrip(tmp_path):
    from paper_2008_11839_b200 import gen_rmat, build_csr, load_graph, load_graph_binary, save_graph_binary
    g = build_csr(gen_rmat(12, 8, seed=3))
    p = tmp_path / "g.gcn1"
    save_graph_binary(g, p)
    assert is_binary_graph(p)
    for dev in (False, True):
        g2 = load_graph(p, device=dev)
        assert g2.n == g.n and np.array_equal(g2.offsets, g.offsets) and np.array_equal(g2.targets, g.targets)
    g3 = load_graph_binary(p, device=True)
    off, tgt = g3.device_arrays()
    assert np.array_equal(off.cpu().numpy(), g.offsets) and np.array_equal(tgt.cpu().numpy(), g.targets)
    p.write_bytes(p.read_bytes()[:-3])
    with pytest.raises(MalformedInputError, match="truncated"):
        load_graph_binary(p)


def _ba_graph_host(n, att, seed):
    el = gen_ba(n, att, seed=seed)
    e = el.edges
    u = np.concatenate([e[:, 0], e[:, 1]])
    v = np.concatenate([e[:, 1], e[:, 0]])
    order = np.lexsort((v, u))
    u, v = u[order], v[order]
    keep = np.ones(len(u), bool)
    keep[1:] = (u[1:] != u[:-1]) | (v[1:] != v[:-1])
    u, v = u[keep], v[keep]
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, u + 1, 1)
    return Graph(n, np.cumsum(off), v)


def test_make_stream_order_matches_reference():
    from paper_2008_11839_b200.sweep import CSV_COLUMNS, chunk, make_stream, make_stream_columnar
    assert CSV_COLUMNS == API["csv_columns"]
    assert chunk(list(range(5)), 2) == [[0, 1], [2, 3], [4]] and chunk([1, 2], 0) == [[1, 2]]
    g = _ba_graph_host(300, 2, 3)
    for ratio, want in API["make_stream"].items():
        ratio = int(ratio)
        us, vs, isq = make_stream_columnar(g, ratio, seed=1, device=False)
        arr = np.stack([us, vs, isq], axis=1).astype(np.int64)
        assert len(arr) == want["len"] and h(arr) == want["hash"], ratio
        ops = make_stream(g, ratio, seed=1)
        arr2 = np.array([[op.u, op.v, int(type(op).__name__ == "Query")] for op in ops], dtype=np.int64)
        assert h(arr2) == want["hash"]


_SWEEP_KEYS = ["graph", "spec", "sample", "finish", "find", "splice", "workers", "batch_size", "ratio", "cov",
               "ic", "inspections_sample", "inspections_finish", "rounds", "components"]


@pytest.mark.gpu
def test_sweep_rows_match_reference():
    from paper_2008_11839_b200 import parse_spec
    from paper_2008_11839_b200.sweep import rows_to_csv_text, small_suite, sweep_incremental, sweep_static
    suite = [x for x in small_suite() if x[0] in ("comps_30", "rmat_s7_ef4", "grid_12x12", "ba_120_a3")]
    specs = [parse_spec(t) for t in ("kout+rem_cas+halve+splice", "hb+sv", "none+lt_prs", "bfs+async+halve")]
    rows = sweep_static(suite, specs, [1], repeats=1)
    got = [{k: str(r[k]) for k in _SWEEP_KEYS} for r in rows]
    assert got == API["sweep_static"]
    ispecs = [parse_spec(t) for t in ("none+async+halve", "none+sv")]
    rows = sweep_incremental(suite[:2], ispecs, batch_sizes=[64, 256], ratios=[1, 10])
    got = [{k: str(r[k]) for k in _SWEEP_KEYS} for r in rows]
    assert got == API["sweep_incremental"]
    assert rows_to_csv_text(rows).splitlines()[0] == ",".join(API["csv_columns"])
    static_rows = sweep_static(suite[:1], specs[:1], [1], repeats=1)
    text = rows_to_csv_text(static_rows, roofline=True)
    assert text.splitlines()[0].endswith("alg_bytes,hbm_gbs,hbm_frac")
    assert float(static_rows[0]["hbm_frac"]) > 0


def test_binary_graph_host_roundtrip_and_errors(tmp_path):
    """GCN1 files (graphs.py:170-190) on the host path: no GPU needed."""
    from paper_2008_11839_b200 import load_graph_binary, save_graph_binary
    g = _ba_graph_host(300, 2, 3)
    p = tmp_path / "g.gcn1"
    save_graph_binary(g, p)
    raw = p.read_bytes()
    assert raw[:4] == b"GCN1" and len(raw) == 4 + 16 + 8 * (g.n + 1) + 4 * g.m
    assert is_binary_graph(p)
    g2 = load_graph_binary(p)
    assert g2.n == g.n and np.array_equal(g2.offsets, g.offsets) and np.array_equal(g2.targets, g.targets)
    (tmp_path / "bad.gcn1").write_bytes(b"GCN2" + raw[4:])
    with pytest.raises(MalformedInputError, match="bad magic"):
        load_graph_binary(tmp_path / "bad.gcn1")
    (tmp_path / "short.gcn1").write_bytes(raw[:40])
    with pytest.raises(MalformedInputError, match="truncated"):
        load_graph_binary(tmp_path / "short.gcn1")


@pytest.mark.gpu
def test_census_refinement_and_oracle_routes():
    """sampling_stats' refinement assertion (validate.py:290-297) and the two
    host oracle routes against the C oracle."""
    import oracle
    from paper_2008_11839_b200 import oracle_components, oracle_components_unionfind
    from paper_2008_11839_b200.validate import label_census
    n, e = oracle.gen_rmat(10, 8, seed=3)
    off, tgt = oracle.build_csr(n, e)
    ref, comps = oracle.components(n, off, tgt)
    g = Graph(n, off, tgt)
    assert np.array_equal(oracle_components(g), ref)
    assert np.array_equal(oracle_components_unionfind(g), ref)
    fine = np.arange(n)
    assert sampling_stats(g, fine, ref)[0] == pytest.approx(1 / n)
    sampling_stats(g, ref, ref)  # the partition refines itself
    bad = ref.copy()
    iso = np.flatnonzero(np.diff(off) == 0)
    assert len(iso) >= 1
    bad[iso[0]] = ref[np.flatnonzero(np.diff(off) > 0)[0]]  # glue an isolate onto a component
    with pytest.raises(AssertionError, match="merge distinct"):
        sampling_stats(g, bad, ref)
    c = label_census(g, ref)
    assert c["crossing"] == 0 and c["mode_count"] == np.bincount(ref).max()
