#!/usr/bin/env python
"""Measure every BASELINE.json config on one B200 (bench.py carries the
headline config 2).  Each config: build the input on the GPU, run once
untimed and check it against the C oracle (bit-exact labels / forest clauses
/ query bits), then time `--reps` runs with CUDA events and report the median.
One JSON line per measurement; also written to --out.

  python bench_configs.py [--configs 1,3,4,5] [--reps 5] [--out profiles/configs_r1.jsonl]
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0  # B200_PROFILING.md fallback


def ev_time(fn, reps, warm=2):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return statistics.median(ts), ts


def host_csr(g):
    return g._d_off.cpu().numpy(), g._d_tgt.cpu().numpy()


SPECS = None  # --specs filter


def want(specs):
    return [t for t in specs if SPECS is None or t in SPECS]


def emit(out, rec):
    line = json.dumps(rec)
    print(line, flush=True)
    if out:
        with open(out, "a") as f:
            f.write(line + "\n")


def alg_bytes_static(n, insp_sample, insp_finish, sampled, rounds, forest_edges=0):
    """B = 4 E_insp + 8 (n+1) + 4 n P (+ 8 (n - c) forest
    slots); P = 4 label passes unsampled, 7 sampled, + 3 per finish round."""
    passes = (7 if sampled else 4) + 3 * int(rounds or 0)
    return 4 * (insp_sample + insp_finish) + 8 * (n + 1) + 4 * n * passes + 8 * forest_edges


def roofline_fields(alg, seconds):
    gbs = alg / seconds / 1e9
    return {"alg_bytes": int(alg), "hbm_gbs": gbs, "hbm_frac": gbs / hbm_peak()}


def cpu_line(out, tag, spec, seconds, units, unit, threads, sample, extra=None):
    rec = {"config": tag, "cpu_baseline": True, "kind": "port", "cores": threads, "spec": spec,
           "seconds": seconds, unit: units / seconds, "sample": sample}
    if extra:
        rec.update(extra)
    emit(out, rec)


def cpu_static(out, tag, g, off, tgt, ref, specs, forest=False, bfs_source=-1):
    """The C/OpenMP port of the reference pipeline (oracle/gconn_oracle.c,
    test infrastructure) on all host threads, same graph, labels checked."""
    import numpy as np
    import oracle
    threads = oracle.max_threads()
    for text in specs:
        res = oracle.pipeline(g.n, off, tgt, text, threads, forest=forest, bfs_source=bfs_source)
        lab, st, tm = res[0], res[1], res[2]
        ok = bool(np.array_equal(lab.astype(np.int64), ref))
        cpu_line(out, tag, text, sum(tm), g.m / 2, "edges_per_s", threads, "the whole workload",
                 {"labels_bit_exact": ok, "rounds": st["rounds"], "insp_sample": st["insp_sample"],
                  "insp_finish": st["insp_finish"]})


def static_config(tag, g, specs, reps, out, cpu_spec=None, extra=None):
    import numpy as np
    import oracle
    from paper_2008_11839_b200 import StaticConnectivity, parse_spec, static_connectivity_device
    off, tgt = host_csr(g)
    t0 = time.perf_counter()
    ref, comps = oracle.components(g.n, off, tgt)
    t_oracle = time.perf_counter() - t0
    for text in want(specs):
        spec = parse_spec(text)
        labels, st = static_connectivity_device(g, spec, metrics=True)
        ok = bool(np.array_equal(labels.cpu().numpy().astype(np.int64), ref))
        plan = StaticConnectivity(g, spec)
        med, ts = ev_time(lambda: plan.run(), reps)
        _, st2 = plan.run()
        rec = {"config": tag, "spec": text, "n": g.n, "m_directed": g.m, "seconds": med,
               "edges_per_s": (g.m / 2) / med, "labels_bit_exact": ok, "components": comps,
               "rounds": st.rounds, "insp_sample": st.edge_inspections.get("sample", 0),
               "insp_finish": st.edge_inspections.get("finish", 0), "cov": st.cov, "ic": st.ic,
               "phase_ms": {k: v * 1e3 for k, v in st2.phase_times.items()},
               "kernel_ms": {"sample": st2.kernel_ms_sample, "finish": st2.kernel_ms_finish},
               "oracle_seconds": t_oracle}
        rec.update(roofline_fields(alg_bytes_static(g.n, rec["insp_sample"], rec["insp_finish"],
                                                    spec.sample.value != "none", st.rounds), med))
        if extra:
            rec.update(extra)
        emit(out, rec)
    if cpu_spec:
        cpu_static(out, tag, g, off, tgt, ref, cpu_spec)


def config1(args):
    from paper_2008_11839_b200 import build_csr, gen_rmat
    g = build_csr(gen_rmat(16, 8, seed=1, device=True), keep_host=False)
    # Rem-CAS + full compression is rejected by the reference (dset.py:68-73):
    # run its parser default rem_cas+naive+splice and the full-compression
    # link companion async+compress
    static_config("1: static RMAT s16 ef8", g, ["none+rem_cas+naive+splice", "none+async+compress",
                                                 "kout+rem_cas+halve+splice"], args.reps, args.out,
                  cpu_spec=["none+rem_cas+naive+splice", "kout+rem_cas+halve+splice"])


def config3(args):
    import torch
    from paper_2008_11839_b200 import EdgeList, build_csr, grid3d_edges
    side = args.grid_side
    el = grid3d_edges(side)
    g = build_csr(el, keep_host=False)
    # LDD's shift rate has no reference default: sweep it, named in the spec string
    specs = ["ldd+sv", "ldd+lt_prs", "ldd+lt_crfa", "none+sv", "none+lt_prs", "none+lt_crfa", "kout+sv",
             "bfs+sv"] + [f"ldd({b})+sv" for b in (0.1, 0.3, 0.5, 0.8)]
    # the port has no LDD (absent from the reference): its CPU baseline is
    # the oracle-checkable companions
    cpu = ["none+sv", "none+lt_prs", "kout+sv"] if args.cpu else None
    static_config(f"3: 3-D grid {side}^3 natural ids", g, specs, args.reps, args.out, cpu_spec=cpu)
    if args.no_permuted:
        return
    # randomly relabelled copy: exercises the high-diameter behaviour
    n = side ** 3
    perm = torch.randperm(n, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    e = el.edges.to("cuda")
    g2 = build_csr(EdgeList(n, perm[e]), keep_host=False)
    static_config(f"3: 3-D grid {side}^3 permuted ids", g2,
                  ["ldd+sv", "ldd+lt_prs", "none+sv", "none+lt_prs", "kout+sv"]
                  + [f"ldd({b})+sv" for b in (0.1, 0.3, 0.5, 0.8)], args.reps, args.out, cpu_spec=cpu)


def config4(args):
    import numpy as np
    import torch
    import oracle
    from paper_2008_11839_b200 import IncrementalConnectivity, build_csr, gen_rmat, parse_spec
    scale = args.incr_scale
    g = build_csr(gen_rmat(scale, 8, seed=1, device=True), keep_host=False)
    n = g.n
    off, tgt = g._d_off, g._d_tgt
    src = torch.repeat_interleave(torch.arange(n, device="cuda", dtype=torch.int32), off[1:] - off[:-1])
    keep = src < tgt
    us, vs = src[keep], tgt[keep]
    del src, keep
    perm = torch.randperm(us.numel(), device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    us, vs = us[perm].contiguous(), vs[perm].contiguous()
    del perm
    total = us.numel()
    bs = args.batch
    offh, tgth = host_csr(g)
    ref, comps = oracle.components(n, offh, tgth)
    # incremental counts only initialised vertices (driver.py:719-724): the
    # isolated vertices of the CSR are never touched by an insert
    comps_init = comps - int((np.diff(offh) == 0).sum())
    g_deg_host = offh
    del tgth
    for text in want(["none+async+halve", "none+rem_cas+halve+split", "none+sv", "none+lt_prs"]):
        spec = parse_spec(text)
        best = None
        for rep in range(args.reps_incr):
            inc = IncrementalConnectivity(spec, n)
            inc.reserve(bs)  # buffer allocation outside the timed batches
            torch.cuda.synchronize()
            t = 0.0
            if spec.is_union_finish():
                # union-find inserts are enqueued back to back on the stream
                # (insert(sync=False)); the whole stream is timed on the device
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                for b0 in range(0, total, bs):
                    inc.insert(us[b0:b0 + bs], vs[b0:b0 + bs], sync=False)
                e1.record()
                e1.synchronize()
                t = e0.elapsed_time(e1) / 1e3
            else:
                for b0 in range(0, total, bs):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    inc.insert(us[b0:b0 + bs], vs[b0:b0 + bs])
                    e1.record()
                    e1.synchronize()
                    t += e0.elapsed_time(e1) / 1e3
            best = t if best is None else min(best, t)
            if rep == 0:
                labels, c = inc.labels()
                ok = bool(np.array_equal(labels.cpu().numpy().astype(np.int64), ref)) and c == comps_init
            del inc
        # B = 16 |ins| + 16 |qry| + 4 hooks + ceil(|ops| / 8); the
        # hooks (successful unions) of an insert-only stream number
        # (initialised vertices) - (their components)
        inited = int((np.diff(g_deg_host) > 0).sum())
        hooks = inited - comps_init
        alg = 16 * total + 4 * hooks + (total + 7) // 8
        tag4 = f"4: incremental RMAT s{scale} ef8, {bs}-edge insert batches"
        emit(args.out, {"config": tag4, "spec": text,
                        "n": n, "inserts": total, "batches": (total + bs - 1) // bs, "seconds": best,
                        "ops_per_s": total / best, "labels_bit_exact": ok, "components": comps_init,
                        "alg_bytes": alg, "hbm_gbs": alg / best / 1e9,
                        "hbm_frac": alg / best / 1e9 / hbm_peak()})
        if args.cpu and text in ("none+async+halve", "none+rem_cas+halve+split"):
            # bounded sample: the first two batches of the same
            # stream into an empty s26-capacity parent array, C/OpenMP port
            threads = oracle.max_threads()
            P = np.full(n, n, dtype=np.int32)
            nb = min(2, (total + bs - 1) // bs)
            secs, done = 0.0, 0
            for b0 in range(0, nb * bs, bs):
                hu = us[b0:b0 + bs].cpu().numpy()
                hv = vs[b0:b0 + bs].cpu().numpy()
                parts = text.split("+")
                secs += oracle.incr_insert(n, P, hu, hv, parts[1], parts[2],
                                           parts[3] if len(parts) > 3 else "none", threads)
                done += len(hu)
            cpu_line(args.out, tag4, text, secs, done, "ops_per_s", threads,
                     f"the first {nb} batches ({done} inserts) of the stream")


def config5(args):
    import numpy as np
    import oracle
    from paper_2008_11839_b200 import build_csr, gen_uniform_pairs, parse_spec, spanning_forest_device
    lg = args.uniform_log2n
    n = 1 << lg
    g = build_csr(gen_uniform_pairs(lg, 4 * n, seed=1), keep_host=False)
    off, tgt = host_csr(g)
    ref, comps = oracle.components(n, off, tgt)
    tag5 = f"5: spanning forest uniform 2^{lg} deg 8"
    for text in want(["bfs+async+halve", "kout+async+halve", "none+async+halve"]):
        spec = parse_spec(text)
        df, st = spanning_forest_device(g, spec)
        rep = oracle.check_forest(n, off, tgt, df.fu.cpu().numpy(), df.fv.cpu().numpy(), ref)
        med, _ = ev_time(lambda: spanning_forest_device(g, spec), args.reps)
        rec = {"config": tag5, "spec": text, "n": n,
               "m_directed": g.m, "seconds": med, "edges_per_s": (g.m / 2) / med,
               "forest_clauses": rep["clauses"], "forest_ok": rep["passed"],
               "components": comps, "forest_edges": n - st.component_count,
               "insp_sample": st.edge_inspections.get("sample", 0),
               "insp_finish": st.edge_inspections.get("finish", 0),
               "phase_ms": {k: v * 1e3 for k, v in st.phase_times.items()}}
        rec.update(roofline_fields(alg_bytes_static(n, rec["insp_sample"], rec["insp_finish"],
                                                    spec.sample.value != "none", 0, n - st.component_count), med))
        emit(args.out, rec)
    if args.cpu:
        from paper_2008_11839_b200.api import bfs_source
        threads = oracle.max_threads()
        spec = parse_spec("bfs+async+halve")
        src = bfs_source(g, spec.bfs_probes, spec.seed)
        for text in ["bfs+async+halve", "none+async+halve"]:
            lab, st, tm, (fu, fv) = oracle.pipeline(n, off, tgt, text, threads, forest=True, bfs_source=src)
            ok = oracle.check_forest(n, off, tgt, fu, fv, ref)["passed"]
            cpu_line(args.out, tag5, text, sum(tm), g.m / 2, "edges_per_s", threads, "the whole workload",
                     {"forest_ok": ok, "labels_bit_exact": bool(np.array_equal(lab.astype(np.int64), ref))})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,3,4,5")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--reps-incr", type=int, default=2)
    ap.add_argument("--grid-side", type=int, default=256)
    ap.add_argument("--incr-scale", type=int, default=26)
    ap.add_argument("--batch", type=int, default=10_000_000)
    ap.add_argument("--uniform-log2n", type=int, default=27)
    ap.add_argument("--out", default=None)
    ap.add_argument("--specs", default=None, help="comma list: only these specs")
    ap.add_argument("--no-permuted", action="store_true")
    ap.add_argument("--cpu", type=int, default=1, help="1: time the C/OpenMP port beside each config")
    args = ap.parse_args()
    global SPECS
    if args.specs:
        SPECS = set(args.specs.split(","))
    import torch
    torch.cuda.set_device(0)
    for c in args.configs.split(","):
        {"1": config1, "3": config3, "4": config4, "5": config5}[c.strip()](args)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
