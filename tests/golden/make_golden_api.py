"""Golden fixtures for the API-completeness surface (DisjointSets probes,
validate.py helpers, graph files / generators), produced by running the
REFERENCE (connlab) in the build container.

  api.json   gen_ba / gnp_graph hashes, find traces of every find rule,
             check_forest reports for valid and corrupted forests,
             sampling_stats census values

Run:  python tests/golden/make_golden_api.py   (needs /root/reference)
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

from connlab import (DisjointSets, FindOp, SpliceOp, UnionConfig, UnionOp, build_csr,  # noqa: E402
                     check_forest, gen_ba, parse_spec, spanning_forest, static_connectivity)
from connlab.driver import ForestEdges  # noqa: E402
from connlab.graphs import disjoint_union, gnp_graph, grid_graph, path_graph, star_graph  # noqa: E402
from connlab.validate import oracle_components, sampling_stats  # noqa: E402


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()[:16]


def main():
    out = {}
    out["gen_ba"] = {}
    for n, att, seed in [(100, 3, 1), (500, 4, 7), (64, 1, 0)]:
        el = gen_ba(n, att, seed=seed)
        out["gen_ba"][f"{n},{att},{seed}"] = {"n": el.n, "k": len(el.edges), "hash": h(el.edges)}
    out["gnp"] = {}
    for n, p, seed in [(60, 0.08, 9), (40, 0.1, 3)]:
        g = gnp_graph(n, p, seed=seed)
        out["gnp"][f"{n},{p},{seed}"] = {"m": g.m, "off": h(g.offsets), "tgt": h(g.targets)}

    # find traces on P = [0, 0, 1, 2], u = 3 (test_dset.py:77-90)
    out["find_traces"] = {}
    for f in FindOp:
        union = UnionOp.JTB if f is FindOp.TWO_TRY else UnionOp.ASYNC
        ds = DisjointSets(4, UnionConfig(union, f, SpliceOp.NONE))
        ds.p[:] = [0, 0, 1, 2]
        r = ds.find_root(3)
        out["find_traces"][f.value] = {"root": r, "p": list(ds.p)}

    # DisjointSets union sequences: labels_array after a fixed edge list
    g = build_csr(gen_ba(200, 2, seed=5))
    ue = g.undirected_edges()
    out["ds_edges"] = ue.tolist()
    out["ds_labels"] = h(oracle_components(g))

    # check_forest reports
    graphs = {"grid": grid_graph(6, 7), "mixed": disjoint_union([path_graph(9), star_graph(6), grid_graph(3, 3)])}
    out["check_forest"] = {}
    for gname, g in graphs.items():
        orc = oracle_components(g)
        fe, _ = spanning_forest(g, parse_spec("none+sv"))
        edges = list(fe.edges)
        filled = [i for i, e in enumerate(edges) if e is not None]
        empty = [i for i, e in enumerate(edges) if e is None]
        cases = {"valid": list(edges)}
        bad = list(edges)
        bad[filled[0]] = None
        cases["missing_one"] = bad
        bad = list(edges)
        u, v = bad[filled[1]]
        bad[filled[1]] = (u, (v + 17) % g.n if (v + 17) % g.n != u else (v + 18) % g.n)
        cases["not_an_edge"] = bad
        bad = list(edges)
        u, v = edges[filled[2]]
        bad[empty[0]] = (v, u)  # duplicate of an edge: closes a 2-cycle
        cases["cycle"] = bad
        out["check_forest"][gname] = {}
        for cname, ed in cases.items():
            rep = check_forest(g, ForestEdges(ed), orc)
            out["check_forest"][gname][cname] = {
                "edges": [list(e) if e is not None else None for e in ed],
                "report": rep}
        out["check_forest"][gname]["graph"] = {"n": g.n, "off": g.offsets.tolist(), "tgt": g.targets.tolist(),
                                               "oracle": orc.tolist()}

    # sampling_stats census
    g = build_csr(gen_ba(300, 2, seed=3))
    labs, st = static_connectivity(g, parse_spec("kout+async+halve"))
    out["sampling_stats"] = {"graph_seed": 3, "cases": []}
    rng = np.random.default_rng(0)
    for trial in range(3):
        lab = rng.integers(0, 5, size=g.n) * (trial + 1) % g.n
        cov, ic = sampling_stats(g, lab)
        out["sampling_stats"]["cases"].append({"labels": lab.tolist(), "cov": cov, "ic": ic})
    # make_stream op order (bench.py:179-193) on a small graph
    from connlab.bench import CSV_COLUMNS, make_stream
    from connlab.driver import Query
    g = build_csr(gen_ba(300, 2, seed=3))
    out["make_stream"] = {}
    for ratio in (0, 1, 10):
        ops = make_stream(g, ratio, seed=1)
        arr = np.array([[op.u, op.v, int(isinstance(op, Query))] for op in ops], dtype=np.int64)
        out["make_stream"][str(ratio)] = {"len": len(ops), "hash": h(arr)}
    out["csv_columns"] = CSV_COLUMNS
    # sweep rows (bench.py:131-240) without the timing columns
    from connlab.bench import small_suite, sweep_incremental, sweep_static
    keep = ["graph", "spec", "sample", "finish", "find", "splice", "workers", "batch_size", "ratio", "cov",
            "ic", "inspections_sample", "inspections_finish", "rounds", "components"]
    suite = [x for x in small_suite() if x[0] in ("comps_30", "rmat_s7_ef4", "grid_12x12", "ba_120_a3")]
    specs = [parse_spec(t) for t in ("kout+rem_cas+halve+splice", "hb+sv", "none+lt_prs", "bfs+async+halve")]
    rows = sweep_static(suite, specs, [1], repeats=1)
    out["sweep_static"] = [{k: str(r[k]) for k in keep} for r in rows]
    ispecs = [parse_spec(t) for t in ("none+async+halve", "none+sv")]
    rows = sweep_incremental(suite[:2], ispecs, batch_sizes=[64, 256], ratios=[1, 10])
    out["sweep_incremental"] = [{k: str(r[k]) for k in keep} for r in rows]
    (OUT / "api.json").write_text(json.dumps(out, sort_keys=True))
    print("wrote", OUT / "api.json")


if __name__ == "__main__":
    main()
