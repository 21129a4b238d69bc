"""Incremental parity (driver.py:567-725) against reference goldens and the
SequentialUF oracle."""
import numpy as np
import pytest

import oracle
from paper_2008_11839_b200 import ConfigError, Insert, Query, incremental, parse_spec, path_graph

pytestmark = pytest.mark.gpu


def test_golden_bits(golden):
    g = golden.incr["golden"]
    batches = [[Insert(0, 1), Query(0, 1), Query(0, 2)], [Insert(1, 2), Query(0, 2)]]
    labels, results, st = incremental(None, parse_spec("none+async+halve"), batches, capacity=5)
    assert [b.tolist() for b in results] == g["bits"]
    assert labels.tolist() == g["labels"]
    assert st.component_count == g["components"]
    assert set(st.phase_times) == {"insert", "query"}


def test_random_stream_all_incremental_specs(golden):
    r = golden.incr["random"]
    ops = [Insert(u, v) if k == "i" else Query(u, v) for k, u, v in r["ops"]]
    batches = [ops[i:i + r["batch"]] for i in range(0, len(ops), r["batch"])]
    for text, exp in r["results"].items():
        labels, results, st = incremental(None, parse_spec(text), batches, capacity=r["capacity"])
        assert [b.tolist() for b in results] == exp["bits"], text
        assert labels.tolist() == exp["labels"], text
        assert st.component_count == exp["components"], text
        assert st.rounds == exp["rounds"], text
        assert st.edge_inspections.get("insert", 0) == exp["insp"], text


def test_every_incremental_spec_vs_sequential_oracle():
    rng = np.random.default_rng(4)
    cap = 300
    ops = []
    for _ in range(3000):
        u, v = int(rng.integers(0, cap)), int(rng.integers(0, cap))
        ops.append(Insert(u, v) if rng.random() < 0.3 else Query(u, v))
    batches = [ops[i:i + 128] for i in range(0, len(ops), 128)]
    us = np.array([o.u for o in ops]); vs = np.array([o.v for o in ops])
    isq = np.array([isinstance(o, Query) for o in ops], dtype=np.uint8)
    bits, lab = oracle.incremental_replay(cap, us, vs, isq, 128)
    from paper_2008_11839_b200 import enumerate_specs, format_spec
    for spec in enumerate_specs():
        if spec.sample.value != "none" or not spec.incremental_capable():
            continue
        labels, results, _ = incremental(None, spec, batches, capacity=cap)
        assert np.concatenate(results).tolist() == bits.tolist(), format_spec(spec)
        assert labels.tolist() == lab.tolist(), format_spec(spec)


def test_starts_from_graph():
    g = path_graph(6)
    batches = [[Query(0, 5), Insert(6, 0), Query(6, 5)]]
    labels, results, _ = incremental(g, parse_spec("none+sv"), batches, capacity=7)
    assert results[0].tolist() == [True, False, True]
    assert labels.tolist() == [0] * 7


def test_racy_mode_soundness():
    g = path_graph(50)
    ops = [Insert(i + 50, i + 51) for i in range(30)] + [Query(i, i + 1) for i in range(40)]
    labels, results, _ = incremental(g, parse_spec("none+async+halve"), [ops], capacity=81, racy=True)
    bits, lab = oracle.incremental_replay(81, np.r_[np.arange(49), [o.u for o in ops]],
                                          np.r_[np.arange(1, 50), [o.v for o in ops]],
                                          np.r_[np.zeros(49), [isinstance(o, Query) for o in ops]].astype(np.uint8),
                                          10 ** 6)
    assert labels.tolist() == lab.tolist()
    for pos, op in enumerate(ops):
        if results[0][pos]:
            assert isinstance(op, Query)


@pytest.mark.parametrize("text,racy", [("none+lp", False), ("none+lt_pusa", False), ("none+sv", True),
                                       ("none+rem_cas+naive+splice", True)])
def test_rejections(text, racy):
    with pytest.raises(ConfigError):
        incremental(None, parse_spec(text), [[Insert(0, 1)]], capacity=4, racy=racy)


def test_lazy_capacity():
    labels, _, st = incremental(None, parse_spec("none+async+naive"), [[Insert(97, 99)]])
    assert len(labels) == 100 and labels[97] == labels[99] == 97 and labels[98] == 98
    assert st.component_count == 1


@pytest.mark.parametrize("text", ["none+async+halve", "none+rem_cas+halve+split", "none+sv"])
def test_async_insert_stream(text):
    """insert(sync=False) enqueues union-find batches back to back; labels and
    queries order after them (round finishes fall back to the synchronous form)."""
    import torch
    from paper_2008_11839_b200 import IncrementalConnectivity, build_csr, gen_rmat
    g = build_csr(gen_rmat(14, 8, seed=3, device=True))
    ref, comps = oracle.components(g.n, g.offsets, g.targets)
    ue = g.undirected_edges()
    us = torch.from_numpy(ue[:, 0].astype(np.int32)).cuda()
    vs = torch.from_numpy(ue[:, 1].astype(np.int32)).cuda()
    inc = IncrementalConnectivity(parse_spec(text), g.n)
    inc.reserve(50_000)
    for b0 in range(0, us.numel(), 50_000):
        inc.insert(us[b0:b0 + 50_000], vs[b0:b0 + 50_000], sync=False)
    labels, _ = inc.labels()
    lab = labels.cpu().numpy().astype(np.int64)
    touched = np.diff(g.offsets) > 0
    assert np.array_equal(lab[touched], ref[touched])


@pytest.mark.parametrize("text", ["none+async+halve", "none+async+split"])
def test_giant_filter_stream(text):
    """The giant filter (async rules): an RMAT stream inserted twice, so the
    second pass runs in the filter's compact mode (every insert's endpoints
    are marked), with queries answered from the marks and by root chases;
    labels, query bits and merging-edge lists checked against the oracle."""
    import torch
    from paper_2008_11839_b200 import IncrementalConnectivity, build_csr, gen_rmat
    g = build_csr(gen_rmat(14, 8, seed=5, device=True))
    ref, comps = oracle.components(g.n, g.offsets, g.targets)
    ue = g.undirected_edges()
    rng = np.random.default_rng(6)
    ue = ue[rng.permutation(len(ue))]
    us = torch.from_numpy(ue[:, 0].astype(np.int32)).cuda()
    vs = torch.from_numpy(ue[:, 1].astype(np.int32)).cuda()
    inc = IncrementalConnectivity(parse_spec(text), g.n)
    inc.reserve(8192)
    touched = np.diff(g.offsets) > 0
    for rep in range(2):
        merged = 0
        for b0 in range(0, us.numel(), 8192):
            mu, mv = inc.insert_list(us[b0:b0 + 8192], vs[b0:b0 + 8192])
            merged += int(mu.numel())
            # merging edges join distinct reference components only once
            assert np.array_equal(ref[mu.cpu().numpy()], ref[mv.cpu().numpy()])
        # first pass: a spanning forest of the touched vertices; second: nothing merges
        assert merged == (int(touched.sum()) - (comps - int((~touched).sum())) if rep == 0 else 0)
    # queries: every edge (connected) and random pairs
    qu = np.concatenate([ue[:5000, 0], rng.integers(0, g.n, 5000)]).astype(np.int32)
    qv = np.concatenate([ue[:5000, 1], rng.integers(0, g.n, 5000)]).astype(np.int32)
    bits = inc.query(torch.from_numpy(qu).cuda(), torch.from_numpy(qv).cuda()).numpy()
    exp = (ref[qu] == ref[qv]) & touched[qu] & touched[qv]
    exp |= qu == qv
    assert np.array_equal(bits, exp)
    labels, _ = inc.labels()
    lab = labels.cpu().numpy().astype(np.int64)
    assert np.array_equal(lab[touched], ref[touched])
    # a mixed batch in compact mode: re-inserted edges (all filtered) + queries
    mix_u = np.concatenate([ue[:3000, 0], qu[:3000]]).astype(np.int32)
    mix_v = np.concatenate([ue[:3000, 1], qv[:3000]]).astype(np.int32)
    isq = np.concatenate([np.zeros(3000, bool), np.ones(3000, bool)])
    order = rng.permutation(6000)
    bits = inc.batch(torch.from_numpy(mix_u[order]).cuda(), torch.from_numpy(mix_v[order]).cuda(),
                     isq[order]).numpy()
    assert np.array_equal(bits, isq[order] & np.concatenate([np.zeros(3000, bool), exp[:3000]])[order])
    # compact mode with a malformed endpoint: the compaction drops it and
    # raises the sticky flag; the batch's good inserts still apply
    from paper_2008_11839_b200 import MalformedInputError
    bad_u = torch.from_numpy(np.concatenate([ue[:9000, 0], [g.n + 5]]).astype(np.int32)).cuda()
    bad_v = torch.from_numpy(np.concatenate([ue[:9000, 1], [0]]).astype(np.int32)).cuda()
    with pytest.raises(MalformedInputError):
        inc.insert(bad_u, bad_v)
    q = inc.query(bad_u[:100], bad_v[:100]).numpy()
    assert q.all()
