"""Concurrency stress and edge cases on the GPU.

The fixture suite (test_gpu_static.py) pins every statistic on small graphs,
where little contention arises.  Here every one of the 204 specs runs on an
RMAT scale-18 graph (262k vertices, ~4M directed entries — heavy contention
on the hub parents) and is checked bit-exact against the C oracle; the
order-independent statistics (Appendix A of SURVEY.md: post-sample labels
are the component minima of the sampled edges whatever the interleaving)
must agree across every union-find finish of one sampler; and the headline
spec is replayed many times to catch rare races."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rmat18():
    from paper_2008_11839_b200 import build_csr, gen_rmat
    g = build_csr(gen_rmat(18, 8, seed=7, device=True))
    ref, comps = oracle.components(g.n, g.offsets, g.targets)
    return g, ref, comps


def test_every_spec_rmat18(rmat18):
    from paper_2008_11839_b200 import enumerate_specs, format_spec, static_connectivity
    g, ref, comps = rmat18
    stats_by_sampler = {}
    for spec in enumerate_specs():
        labels, st = static_connectivity(g, spec)
        text = format_spec(spec)
        assert np.array_equal(labels, ref), text
        assert st.component_count == comps, text
        if spec.is_union_finish():
            key = (st.edge_inspections.get("sample", 0), st.edge_inspections.get("finish", 0), st.cov)
            stats_by_sampler.setdefault(spec.sample.value, set()).add(key)
    for sampler, keys in stats_by_sampler.items():
        # JTB links by rank, not by id, but its partition (hence every count) is the same
        assert len(keys) == 1, (sampler, keys)


def test_replay_headline_spec_many_times(rmat18):
    from paper_2008_11839_b200 import StaticConnectivity, parse_spec
    g, ref, comps = rmat18
    plan = StaticConnectivity(g, parse_spec("kout+rem_cas+halve+splice"))
    first = None
    for _ in range(40):
        labels, st = plan.run()
        lab = labels.cpu().numpy().astype(np.int64)
        assert np.array_equal(lab, ref)
        key = (st.edge_inspections.get("sample"), st.edge_inspections.get("finish"), st.cov, st.component_count)
        first = first or key
        assert key == first


def test_forest_every_root_based_union_rule_rmat18(rmat18):
    from paper_2008_11839_b200 import enumerate_specs, format_spec, spanning_forest_device
    g, ref, comps = rmat18
    for spec in enumerate_specs():
        if not (spec.is_union_finish() and spec.is_root_based()) or spec.sample.value not in ("none", "kout"):
            continue
        df, st = spanning_forest_device(g, spec)
        rep = oracle.check_forest(g.n, g.offsets, g.targets, df.fu.cpu().numpy(), df.fv.cpu().numpy(), ref)
        assert rep["passed"], (format_spec(spec), rep)


def test_empty_and_single_vertex_graphs():
    from paper_2008_11839_b200 import (DisjointSets, FindOp, Graph, SpliceOp, UnionConfig, UnionOp, enumerate_specs,
                                       incremental, parse_spec, spanning_forest, static_connectivity)
    for n in (0, 1, 2):
        g = Graph(n, np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int32))
        for spec in enumerate_specs():
            labels, st = static_connectivity(g, spec)
            assert labels.tolist() == list(range(n))
            assert st.component_count == n
        fe, st = spanning_forest(g, parse_spec("bfs+async+halve"))
        assert len(fe) == 0 and st.component_count == n
    labels, bits, _ = incremental(None, parse_spec("none+async+halve"), [[]], capacity=3)
    assert labels.tolist() == [0, 1, 2] and bits[0].tolist() == []
    ds = DisjointSets(0, UnionConfig(UnionOp.ASYNC, FindOp.HALVE, SpliceOp.NONE))
    assert ds.labels_array().tolist() == []


def test_hub_rows_and_duplicate_input():
    """A vertex adjacent to everything (warp-cooperative rows), duplicate and
    self-loop input pairs (build_csr drops them)."""
    from paper_2008_11839_b200 import EdgeList, build_csr, parse_spec, static_connectivity
    n = 5000
    rng = np.random.default_rng(3)
    e = np.concatenate([np.stack([np.zeros(n - 1, np.int64), np.arange(1, n)], 1),
                        rng.integers(0, n, size=(20000, 2)),
                        np.stack([np.arange(n), np.arange(n)], 1)])  # self loops
    e = np.concatenate([e, e[:3000]])  # duplicates
    g = build_csr(EdgeList(n, e))
    off, tgt = g.offsets, g.targets
    assert np.all(np.diff(off) >= 0) and len(tgt) == off[-1]
    ref, comps = oracle.components(n, off, tgt)
    assert comps == 1
    for text in ("none+rem_cas+naive+splice", "kout+async+halve", "hb+hooks+split", "none+sv", "none+lt_prs",
                 "bfs+early+compress", "ldd+lt_crfa", "none+jtb+twotry"):
        labels, st = static_connectivity(g, parse_spec(text))
        assert np.array_equal(labels, ref), text


def test_malformed_csr_is_rejected_not_faulted():
    """Out-of-range targets / broken offsets raise MalformedInputError before
    any kernel reads them (the GPU context stays usable)."""
    from paper_2008_11839_b200 import Graph, MalformedInputError, parse_spec, static_connectivity
    spec = parse_spec("kout+rem_cas+halve+splice")
    bad_tgt = Graph(4, np.array([0, 1, 2, 3, 4]), np.array([1, 0, 3, 9], dtype=np.int32))
    with pytest.raises(MalformedInputError, match="target"):
        static_connectivity(bad_tgt, spec)
    bad_off = Graph(4, np.array([0, 2, 1, 3, 4]), np.array([1, 0, 3, 2], dtype=np.int32))
    with pytest.raises(MalformedInputError, match="offsets"):
        static_connectivity(bad_off, spec)
    ok = Graph(4, np.array([0, 1, 2, 3, 4]), np.array([1, 0, 3, 2], dtype=np.int32))
    labels, _ = static_connectivity(ok, spec)
    assert labels.tolist() == [0, 0, 2, 2]
