"""Static connectivity parity on the GPU against reference-generated fixtures.

Labels must equal the reference's canonical labels bit for bit; rounds,
inspection counts, cov / ic and component counts must equal the reference's
workers=1 statistics (driver.py:492-499) for every one of the 204 specs.
"""
import numpy as np
import pytest

from gpu_util import graph_of
from golden_data import h
from paper_2008_11839_b200 import (ConfigError, Graph, enumerate_specs, finish_phase, format_spec,
                                   label_finalization, parse_spec, static_connectivity)

pytestmark = pytest.mark.gpu


def _check(golden, name, spec, labels, st, check_ic=True):
    ref = golden.spec_stats[name][format_spec(spec)]
    n, off, tgt, oracle = golden.graphs[name]
    assert np.array_equal(labels, oracle), (name, format_spec(spec))
    assert h(labels) == ref["labels"]
    got = {"rounds": st.rounds, "insp_sample": st.edge_inspections.get("sample", 0),
           "insp_finish": st.edge_inspections.get("finish", 0), "components": st.component_count}
    exp = {k: ref[k] for k in got}
    assert got == exp, (name, format_spec(spec))
    assert st.cov == pytest.approx(ref["cov"], abs=0, rel=1e-12), (name, format_spec(spec))
    if check_ic:
        assert st.ic == pytest.approx(ref["ic"], abs=0, rel=1e-12), (name, format_spec(spec))


@pytest.mark.parametrize("sample", ["none", "kout", "hb", "bfs"])
def test_all_specs_small_suite(golden, sample):
    specs = [s for s in enumerate_specs() if s.sample.value == sample]
    for name in golden.names():
        g = graph_of(golden, name)
        for spec in specs:
            labels, st = static_connectivity(g, spec)
            _check(golden, name, spec, labels, st)


def test_component_minimum_labels():
    from paper_2008_11839_b200 import clique_graph, disjoint_union, path_graph, star_graph
    g = disjoint_union([path_graph(40), star_graph(25), clique_graph(8)])
    for text in ["none+async+halve", "kout+rem_cas+halve+splice", "hb+sv", "bfs+lt_prs", "ldd+sv",
                 "ldd+lt_prs", "ldd(0.5)+rem_cas+halve+splice"]:
        labels, st = static_connectivity(g, parse_spec(text))
        assert labels.tolist() == [0] * 40 + [40] * 25 + [65] * 8, text
        assert st.component_count == 3


def test_ldd_on_suite(golden):
    for name in golden.names():
        g = graph_of(golden, name)
        for text in ["ldd+sv", "ldd+lt_prs", "ldd+lt_crfa", "ldd+rem_cas+halve+splice", "ldd+lp",
                     "ldd(0.05)+stergiou"]:
            labels, st = static_connectivity(g, parse_spec(text))
            assert np.array_equal(labels, golden.graphs[name][3]), (name, text)


def test_label_finalization():
    assert label_finalization([0, 0, 1]).tolist() == [0, 0, 0]
    assert label_finalization([0, 1, 2]).tolist() == [0, 1, 2]
    assert label_finalization([3, 3, 3, 3]).tolist() == [0, 0, 0, 0]
    assert label_finalization([]).tolist() == []


def test_finish_phase():
    from paper_2008_11839_b200 import path_graph
    g = path_graph(6)
    out = finish_phase(g, [0, 0, 0, 3, 4, 5], l_max=0, spec=parse_spec("none+async+halve"))
    assert label_finalization(out).tolist() == [0] * 6
    out = finish_phase(path_graph(4), [0, 0, 0, 0], l_max=0, spec=parse_spec("none+async+halve"))
    assert out.tolist() == [0, 0, 0, 0]
    for text in ["none+sv", "none+lt_prs", "none+lp", "none+stergiou", "none+rem_cas+split+halve"]:
        out = finish_phase(g, [0, 0, 0, 3, 4, 5], l_max=0, spec=parse_spec(text))
        assert label_finalization(out).tolist() == [0] * 6, text


def test_config1_rmat_s16_stats(golden):
    from paper_2008_11839_b200 import build_csr, gen_rmat
    pin = golden.rmat["s16_ef8_seed1"]
    g = build_csr(gen_rmat(16, 8, seed=1, device=True), keep_host=False)
    assert g.m == pin["m"]
    for text, ref in pin["specs"].items():
        labels, st = static_connectivity(g, parse_spec(text))
        assert h(labels) == ref["labels"], text
        got = {"rounds": st.rounds, "insp_sample": st.edge_inspections.get("sample", 0),
               "insp_finish": st.edge_inspections.get("finish", 0), "components": st.component_count}
        assert got == {k: ref[k] for k in got}, text
        assert st.cov == pytest.approx(ref["cov"], rel=1e-12) and st.ic == pytest.approx(ref["ic"], rel=1e-12)


def test_plan_replay_matches_direct(golden):
    from paper_2008_11839_b200 import StaticConnectivity
    for name in ["rmat_s10_ef8", "ba_120_a3", "comps_30", "edgeless4", "star64"]:
        g = graph_of(golden, name)
        for text in ["kout+rem_cas+halve+splice", "none+async+halve", "hb+jtb+twotry", "none+lt_prs",
                     "bfs+sv"]:
            plan = StaticConnectivity(g, parse_spec(text))
            for _ in range(3):  # first run captures, later runs replay the CUDA graph
                labels, st = plan.run()
                # plans skip the untimed ic census (metrics are off on the replay path)
                _check(golden, name, parse_spec(text), labels.cpu().numpy(), st, check_ic=False)
