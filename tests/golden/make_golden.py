"""Generate the golden fixtures by running the REFERENCE (connlab) in the
build container.

/root/reference does not exist on the GPU box, so everything the GPU-side
parity tests need from the reference is captured here as small files:

  small_suite.npz   CSR arrays of the reference's 12-graph correctness suite
                    (bench.py:81-97) plus extra shapes, and their oracle labels
  spec_stats.json   per (graph, spec): labels hash, rounds, inspections,
                    cov/ic, component count — reference workers=1 runs
  rmat.json         gen_rmat shape/hash pins (test_graphs.py:105-118 and the
                    config-1 input)
  incremental.json  incremental golden bits (test_driver.py:232-243) and a
                    seeded random stream with its expected bits

Run:  python tests/golden/make_golden.py   (needs /root/reference)
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import connlab  # noqa: E402
from connlab import (EdgeList, Insert, Query, build_csr, enumerate_specs,  # noqa: E402
                     format_spec, incremental, parse_spec, spanning_forest,
                     static_connectivity)
from connlab.bench import small_suite  # noqa: E402
from connlab.graphs import (clique_graph, disjoint_union, gen_rmat, path_graph,  # noqa: E402
                            star_graph)
from connlab.validate import SequentialUF, oracle_components  # noqa: E402


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()[:16]


def extra_graphs():
    g = []
    g.append(("p40_s25_c8", disjoint_union([path_graph(40), star_graph(25), clique_graph(8)])))
    g.append(("star50_path2", disjoint_union([star_graph(50), path_graph(2)])))
    g.append(("star64", star_graph(64)))
    g.append(("path8", path_graph(8)))
    g.append(("path4", path_graph(4)))
    g.append(("triangle_iso", build_csr(EdgeList(4, np.array([(0, 1), (1, 2), (2, 0)])))))
    g.append(("crossed", build_csr(EdgeList(4, np.array([(0, 2), (1, 3), (2, 3)])))))
    g.append(("star30_clique6", disjoint_union([star_graph(30), clique_graph(6)])))
    g.append(("edgeless4", build_csr(EdgeList(4, np.empty((0, 2), dtype=np.int64)))))
    rng = np.random.default_rng(11)
    g.append(("rand120_400", build_csr(EdgeList(120, rng.integers(0, 120, size=(400, 2))))))
    g.append(("rmat_s10_ef8", build_csr(gen_rmat(10, 8, seed=3))))
    return g


def main():
    graphs = small_suite() + extra_graphs()
    arrays = {}
    stats = {}
    for name, g in graphs:
        arrays[f"{name}__n"] = np.array([g.n])
        arrays[f"{name}__off"] = g.offsets
        arrays[f"{name}__tgt"] = g.targets
        o = oracle_components(g)
        arrays[f"{name}__oracle"] = o
    specs = enumerate_specs()
    for name, g in graphs:
        rows = {}
        for spec in specs:
            lab, st = static_connectivity(g, spec, workers=1)
            rows[format_spec(spec)] = {
                "labels": h(lab),
                "rounds": st.rounds,
                "insp_sample": st.edge_inspections.get("sample", 0),
                "insp_finish": st.edge_inspections.get("finish", 0),
                "cov": st.cov,
                "ic": st.ic,
                "components": st.component_count,
            }
            if spec.is_root_based():
                fe, fst = spanning_forest(g, spec, workers=1)
                rows[format_spec(spec)]["forest_count"] = len(fe)
                if spec.finish.value in ("sv", "lt") and spec.sample.value in ("none", "bfs"):
                    # deterministic forests (min edge index / first discoverer)
                    flat = [x for e in fe.edges for x in (e if e else (-1, -1))]
                    rows[format_spec(spec)]["forest"] = h(flat)
        stats[name] = rows
        print(name, g.n, g.m, file=sys.stderr)
    np.savez_compressed(OUT / "small_suite.npz", **arrays)
    (OUT / "spec_stats.json").write_text(json.dumps(stats, sort_keys=True))

    # RMAT pins: test_graphs.py:105-118 and the config-1 input
    rm = {}
    el = gen_rmat(7, 4, seed=2)
    rm["s7_ef4_seed2_edges"] = el.edges.tolist()
    g = build_csr(el)
    rm["s7_ef4_seed2"] = {"m": g.m, "offsets_hash": h(g.offsets), "targets_hash": h(g.targets)}
    for scale, ef, seed in [(10, 8, 3), (12, 8, 1), (16, 8, 1)]:
        el = gen_rmat(scale, ef, seed=seed)
        g = build_csr(el)
        o = oracle_components(g)
        key = f"s{scale}_ef{ef}_seed{seed}"
        rm[key] = {"edges_hash": h(el.edges), "m": g.m, "offsets_hash": h(g.offsets),
                   "targets_hash": h(g.targets), "components": int(len(np.unique(o))),
                   "oracle_hash": h(o)}
        if scale == 16:
            rows = {}
            for text in ["none+rem_cas+naive+splice", "none+async+compress", "kout+rem_cas+halve+splice",
                         "none+sv", "kout+sv", "hb+sv", "bfs+sv", "none+lt_prs", "none+lt_crfa",
                         "none+stergiou", "none+lp", "kout+lt_prsa", "hb+async+halve", "bfs+async+halve",
                         "kout+lp", "hb+stergiou"]:
                lab, st = static_connectivity(g, parse_spec(text))
                rows[text] = {"labels": h(lab), "rounds": st.rounds,
                              "insp_sample": st.edge_inspections.get("sample", 0),
                              "insp_finish": st.edge_inspections.get("finish", 0),
                              "cov": st.cov, "ic": st.ic, "components": st.component_count}
                print(text, rows[text], file=sys.stderr)
            rm[key]["specs"] = rows
    (OUT / "rmat.json").write_text(json.dumps(rm, sort_keys=True))

    # incremental pins
    inc = {}
    batches = [[Insert(0, 1), Query(0, 1), Query(0, 2)], [Insert(1, 2), Query(0, 2)]]
    lab, res, st = incremental(None, parse_spec("none+async+halve"), batches, capacity=5)
    inc["golden"] = {"labels": lab.tolist(), "bits": [b.tolist() for b in res],
                     "components": st.component_count}
    rng = np.random.default_rng(4)
    ops = []
    for _ in range(400):
        u, v = int(rng.integers(0, 60)), int(rng.integers(0, 60))
        ops.append(("i" if rng.random() < 0.6 else "q", u, v))
    bl = [ops[i:i + 32] for i in range(0, len(ops), 32)]
    conv = [[Insert(u, v) if k == "i" else Query(u, v) for k, u, v in b] for b in bl]
    res_by = {}
    for text in ["none+async+halve", "none+rem_cas+halve+split", "none+sv", "none+lt_prs",
                 "none+hooks+naive", "none+jtb+twotry", "none+lt_crfa"]:
        lab, res, st = incremental(None, parse_spec(text), conv, capacity=64)
        res_by[text] = {"labels": lab.tolist(), "bits": [b.tolist() for b in res],
                        "components": st.component_count, "rounds": st.rounds,
                        "insp": st.edge_inspections.get("insert", 0)}
    inc["random"] = {"ops": ops, "batch": 32, "capacity": 64, "results": res_by}
    (OUT / "incremental.json").write_text(json.dumps(inc, sort_keys=True))


if __name__ == "__main__":
    main()
