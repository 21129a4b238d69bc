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
