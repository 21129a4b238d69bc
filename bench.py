#!/usr/bin/env python
"""Benchmark: GConn static connectivity on B200 (BASELINE.json configs[1]).

Workload (one "step"): static connectivity with k-out sampling + union-find
Rem-CAS + path halving + splice (`kout+rem_cas+halve+splice`) on the RMAT
scale-24 average-degree-16 graph (edge_factor 8, seed 1, the reference's
gen_rmat distribution reproduced bit-for-bit on the GPU), inputs resident in
HBM.  metric = undirected edges / second = (m_dir / 2) / step time, the
reference's throughput definition (bench.py:167).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): the edge-sharded two-phase pipeline on
an RMAT graph of scale 24 + log2(N) (weak scaling: each rank owns about one
scale-24 graph's edges), merged with all-gathers over NCCL; value = the
graph's undirected edges / max-over-ranks step time (see run_sharded).

--impl reference times the reference algorithm's CPU restatement (oracle/,
a C port of connlab's _pipeline with OpenMP on all host threads) on the same
config; only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SPEC = "kout+rem_cas+halve+splice"
METRIC = "connectivity edges/sec (static & incremental) on RMAT at 1/2/4/8 B200"
UNIT = "edges/s"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML every ~2 ms while
    the timed region runs (the recipe's nvidia-smi clocks line, at a rate
    that also covers sub-second timed regions).  Falls back to nvidia-smi."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, cuda_index: int, period_s: float = 0.002):
        self.cuda_index = cuda_index
        self.period = period_s
        self.samples = []  # (sm_mhz, max_mhz, reasons-bitmask)
        self.stop = threading.Event()
        self.t = None
        self.nvml = None
        self.proc = None
        self.smi_lines = []

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            p = torch.cuda.get_device_properties(self.cuda_index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.cuda_index)

    def _poll(self):
        nv, h = self.nvml
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, mx, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        try:
            self.nvml = self._handle()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < 2.0:
                time.sleep(0.001)
        except Exception:
            self.nvml = None
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--id={self.cuda_index}",
                     "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                     "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                     "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "20"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=lambda: self.smi_lines.extend(
                    ln.strip() for ln in self.proc.stdout), daemon=True)
                self.t.start()
            except FileNotFoundError:
                self.proc = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.t is not None:
            self.t.join(timeout=5)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        if self.nvml is not None:
            nv = self.nvml[0]
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            for s, m, r in self.samples:
                sm.append(float(s))
                mx = max(mx, float(m))
                reasons.update(k for k, b in bits.items() if r & b)
            src = "nvml"
        else:
            for ln in self.smi_lines:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx = max(mx, float(parts[1]))
                except ValueError:
                    continue
                reasons.update(nm for nm, f in zip(self.NAMES, parts[2:6]) if f.lower() == "active")
            src = "nvidia-smi"
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm), "source": src}


L2_NOTE = ("inputs (offsets + targets, 1.2 GB at scale 24) exceed the 126 MB L2; the GPU arm also "
           "writes a 256 MiB buffer between timed steps (outside the step events)")


def bench_config(scale: int, ef: int, seed: int, n: int, m: int, ws: int) -> dict:
    """The workload description both arms print (identical dicts, so the
    driver can match the reference arm's line to ours)."""
    shards = f", {ws} row blocks" if ws > 1 else ""
    return {"workload": f"static CC {SPEC} on RMAT scale-{scale} ef{ef} (avg degree 16) seed {seed}{shards}",
            "spec": SPEC, "n": n, "m_directed": m, "undirected_edges": m // 2, "l2": L2_NOTE}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_graph(scale: int, ef: int, seed: int):
    from paper_2008_11839_b200 import build_csr, gen_rmat
    el = gen_rmat(scale, ef, seed=seed, device=True)
    g = build_csr(el, keep_host=False)
    del el
    return g


def run_sharded(args):
    """N > 1: the edge-sharded two-phase pipeline on one graph.

    Weak scaling: the RMAT scale grows by log2(N) so every rank owns about
    one scale-24 graph's worth of edges.  Every rank generates the same graph
    (deterministic stream), keeps only its edge-balanced row block, and each
    step runs `sharded_two_phase`: local sampling over its rows, all-gather
    of a compact summary of the sampled partition (local giant as an n-bit
    bitmap + the non-giant remainder as pairs), the finish over its active
    rows, an all-gather of the finish's merging edges, local finalisation.  The step time is CUDA events on the
    rank's stream (host-side collective waits included), max over ranks."""
    import math

    import numpy as np
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local % ndev)
    backend = os.environ.get("GC_DIST_BACKEND", "nccl")
    kw = {} if "RANK" in os.environ else {"rank": 0, "world_size": 1, "store": dist.HashStore()}
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local % ndev), **kw)
    else:
        dist.init_process_group(backend, **kw)
    from paper_2008_11839_b200 import parse_spec
    from paper_2008_11839_b200.distributed import shard_balance, shard_bounds, shard_graph, sharded_two_phase

    spec = parse_spec(SPEC)
    scale = args.scale + int(math.ceil(math.log2(ws)))
    g = make_graph(scale, args.edge_factor, args.seed)
    n, m = g.n, g.m
    lo, hi = shard_bounds(g._d_off, ws, shard_balance(spec))[rank]
    shard = shard_graph(g, lo, hi)
    parity = None
    res = sharded_two_phase(shard, spec, forest=False)
    if rank == 0 and not args.skip_check:
        import oracle
        ref, comps = oracle.components(n, g._d_off.cpu().numpy(), g._d_tgt.cpu().numpy())
        ok = bool(np.array_equal(res.labels.cpu().numpy().astype(np.int64), ref)) and res.components == comps
        parity = {"labels_bit_exact": ok, "components": comps, "insp_sample": res.insp_sample,
                  "insp_finish": res.insp_finish, "cov": res.lmax_count / n}
        if not ok:
            print(json.dumps({"error": "parity failure", "parity": parity}), file=sys.stderr)
            sys.exit(3)
    del g
    torch.cuda.empty_cache()
    from paper_2008_11839_b200 import Graph
    from paper_2008_11839_b200 import _native as N
    from paper_2008_11839_b200.api import host_int64
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        sharded_two_phase(shard, spec, forest=False)
    torch.cuda.synchronize()
    dist.barrier()
    lib = N.lib()
    l0 = lib.gc_launch_count()
    times, exchanged = [], 0
    with ClockSampler(local % ndev) as clk:
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = sharded_two_phase(shard, spec, forest=False)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            exchanged = r.exchanged_edges
    torch.cuda.synchronize()
    launches = lib.gc_launch_count() - l0
    dist.barrier()
    dev = "cuda" if backend == "nccl" else "cpu"
    tmax = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    total_ms = float(tmax.item())
    ms_per_step = total_ms / args.steps
    value = (m / 2) * args.steps / (total_ms / 1e3)
    # end to end: every rank copies its row block in from pinned host memory,
    # runs the sharded pipeline and reads the labels back (int64, pinned);
    # wall clock per step, max over ranks
    e2e = None
    if args.e2e_steps > 0:
        off_h = shard._d_off.cpu().pin_memory()
        tgt_h = shard._d_tgt.cpu().pin_memory()
        def host_shard():
            hg = Graph(n, off_h, tgt_h)
            hg.row_block = shard.row_block
            return hg
        sharded_two_phase(host_shard().cuda(), spec, forest=False)
        et = []
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            r = sharded_two_phase(host_shard().cuda(), spec, forest=False)
            host_int64(r.labels)
            torch.cuda.synchronize()
            et.append(time.perf_counter() - t0)
        tm = torch.tensor([statistics.median(et)], dtype=torch.float64, device=dev)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        e2e_t = float(tm.item())
        e2e = {"value": (m / 2) / e2e_t, "unit": UNIT,
               "h2d_bytes_per_step": int(off_h.numel() * 8 + tgt_h.numel() * 4), "d2h_bytes_per_step": 8 * n,
               "seconds_per_step": e2e_t,
               "timing": "wall clock per rank (pinned H2D of its row block, sharded pipeline, int64 labels "
                         "D2H), max over ranks; bytes are rank 0's"}
    peak, peak_kind = peaks()
    step_bytes = 4 * (res.insp_sample + res.insp_finish) + 8 * (n + 1) + 4 * n * 7
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
                "config": bench_config(scale, args.edge_factor, args.seed, n, m, ws),
                "parallelism": f"edge-sharded x{ws} ({backend}), two-phase: giant-bitmap + remainder "
                               "all-gather, then finish merging edges",
                "exchanged_pairs_per_step": exchanged,
                "exchanged_bitmap_bytes_per_step": ws * ((n + 31) // 32) * 4,
                "e2e": e2e, "gpu_launches": launches, "launches_per_step": launches / args.steps,
                "roofline": {"bound": "hbm", "achieved": step_bytes / (ms_per_step / 1e3) / 1e9 / ws,
                             "peak": peak, "unit": "GB/s",
                             "frac": step_bytes / (ms_per_step / 1e3) / 1e9 / ws / peak, "traffic": None,
                             "kernel": "whole sharded step (per-GPU share of the SURVEY 8(d) bytes)",
                             "peak_source": peak_kind},
                "cpu_baseline": None, "parity": parity, "clocks": clk.summary()}
        print(json.dumps(line))
    dist.destroy_process_group()


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2008_11839_b200 import (Graph, StaticConnectivity, parse_spec, static_connectivity,
                                       static_connectivity_device)
    from paper_2008_11839_b200 import _native as N

    spec = parse_spec(SPEC)
    g = make_graph(args.scale, args.edge_factor, args.seed)
    n, m = g.n, g.m
    torch.cuda.synchronize()

    # ---- untimed parity check against the CPU oracle (rank 0)
    parity = None
    labels, st0 = static_connectivity_device(g, spec, metrics=True)
    if rank == 0 and not args.skip_check:
        import oracle
        off_h = g._d_off.cpu().numpy()
        tgt_h = g._d_tgt.cpu().numpy()
        ref, comps = oracle.components(n, off_h, tgt_h)
        ok = bool(np.array_equal(labels.cpu().numpy().astype(np.int64), ref)) and st0.component_count == comps
        parity = {"labels_bit_exact": ok, "components": comps, "cov": st0.cov, "ic": st0.ic,
                  "insp_sample": st0.edge_inspections.get("sample", 0),
                  "insp_finish": st0.edge_inspections.get("finish", 0)}
        if not ok:
            print(json.dumps({"error": "parity failure", "parity": parity}), file=sys.stderr)
            sys.exit(3)
    del labels

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    stream = torch.cuda.current_stream()

    plan = StaticConnectivity(g, spec)  # graph-captured pipeline, replayed per step
    if rank == 0 and not args.skip_check:
        # the timed path is the captured plan: check one replay as well
        plan.run()  # first run captures
        plab, pst = plan.run()
        pok = bool(np.array_equal(plab.cpu().numpy().astype(np.int64), ref)) and pst.component_count == comps
        parity["plan_labels_bit_exact"] = pok
        if not pok:
            print(json.dumps({"error": "parity failure on the plan replay", "parity": parity}), file=sys.stderr)
            sys.exit(3)

    def step():
        _, st = plan.run()
        return st

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    lib = N.lib()
    l0 = lib.gc_launch_count()
    times, ksamp, kfin, kstats = [], [], [], None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()  # evict L2 between timed steps (outside the events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st = step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            ksamp.append(st.kernel_ms_sample)
            kfin.append(st.kernel_ms_finish)
            kstats = st
    torch.cuda.synchronize()
    launches = lib.gc_launch_count() - l0
    if ws > 1:
        dist.barrier()
    total_ms = sum(times)
    tmax = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    total_ms = float(tmax.item())
    ms_per_step = total_ms / args.steps
    value = ws * (m / 2) * args.steps / (total_ms / 1e3)

    # ---- end-to-end: public API with host (pinned) buffers, H2D + D2H inside
    e2e = None
    if args.e2e_steps > 0:
        off_h = g._d_off.cpu().pin_memory()
        tgt_h = g._d_tgt.cpu().pin_memory()
        host_g = Graph(n, off_h, tgt_h)
        static_connectivity(host_g, spec)  # warm the path
        torch.cuda.synchronize()
        et = []
        for _ in range(args.e2e_steps):
            hg = Graph(n, off_h, tgt_h)  # fresh container: no cached device copy
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            lab, _ = static_connectivity(hg, spec)
            torch.cuda.synchronize()
            et.append(time.perf_counter() - t0)
        e2e_t = statistics.median(et)
        e2e = {"value": ws * (m / 2) / e2e_t, "unit": UNIT, "h2d_bytes_per_step": 8 * (n + 1) + 4 * m,
               "d2h_bytes_per_step": 8 * n, "seconds_per_step": e2e_t,
               "timing": "wall clock around static_connectivity(host Graph) incl. pinned H2D, D2H, int64 labels"}

    # ---- roofline of the dominant kernel (k-out union over the sampled rows)
    peak, peak_kind = peaks()
    e_s = kstats.edge_inspections.get("sample", 0)
    e_f = kstats.edge_inspections.get("finish", 0)
    kout_bytes = 8 * (n + 1) + 4 * e_s + 8 * n  # offsets + sampled targets + parent read/write
    kms = statistics.mean(ksamp)
    achieved = kout_bytes / (kms / 1e3) / 1e9
    step_bytes = 4 * (e_s + e_f) + 8 * (n + 1) + 4 * n * 7  # SURVEY 8(d), P = 7 with sampling
    traffic, traffic_src = args.traffic, "--traffic"
    tj = ROOT / "profiles" / "traffic.json"
    if traffic is None and tj.exists():
        t = json.loads(tj.read_text())
        traffic, traffic_src = t["traffic_bytes"], f"profiles/traffic.json ({t['source']})"
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": "k_union_rows<Rule<REM_CAS,HALVE,SPLICE>> (k-out sampling)",
                "kernel_ms": kms, "kernel_bytes": kout_bytes, "peak_source": peak_kind,
                "step_alg_bytes": step_bytes,
                "step_frac": step_bytes / (ms_per_step / 1e3) / 1e9 / peak,
                "kernel_share_of_step": kms / ms_per_step,
                # the measured DRAM bytes (ncu) over the live kernel time: how
                # close the kernel runs to the HBM floor of the traffic the CSR
                # layout forces (each 8-byte row head costs a 64-byte burst)
                "traffic_frac": (traffic / (kms / 1e3) / 1e9 / peak) if traffic else None}

    cpu = None
    if rank == 0 and args.cpu_baseline:
        cpu = cpu_baseline(g)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
                "config": bench_config(args.scale, args.edge_factor, args.seed, n, m, ws),
                "parallelism": f"replicas{ws}" if ws > 1 else "single-gpu",
                "e2e": e2e, "gpu_launches": launches, "launches_per_step": launches / args.steps,
                "roofline": roofline, "cpu_baseline": cpu, "parity": parity,
                "clocks": clk.summary()}
        print(json.dumps(line))
    if ws > 1:
        dist.destroy_process_group()


def cpu_baseline(g):
    """The reference algorithm's C port (oracle/) on this box's host cores."""
    import oracle
    off = g._d_off.cpu().numpy()
    tgt = g._d_tgt.cpu().numpy()
    threads = oracle.max_threads()
    _, st, tm = oracle.static_uf(g.n, off, tgt, "kout", 2, "rem_cas", "halve", "splice", threads)
    t = sum(tm)
    return {"value": (g.m / 2) / t, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"one full run of the same workload (n={g.n}, m={g.m}) — "
                      f"sample {tm[0]:.3f}s finish {tm[1]:.3f}s finalize {tm[2]:.3f}s",
            "seconds": t}


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    import math

    import oracle
    # the same workload as our arm at this N (weak scaling: scale 24 + log2 N)
    scale = args.scale + (int(math.ceil(math.log2(ws))) if ws > 1 else 0)
    n, e = oracle.gen_rmat(scale, args.edge_factor, seed=args.seed)
    off, tgt = oracle.build_csr(n, e)
    del e
    m = len(tgt)
    threads = oracle.max_threads()
    for _ in range(args.warmup):
        lab, st, _ = oracle.static_uf(n, off, tgt, "kout", 2, "rem_cas", "halve", "splice", threads)
    parity = None
    if not args.skip_check:
        # the arm itself is checked: its labels against the sequential
        # union-find oracle (validate.py:101-122), as our arm's are
        import numpy as np
        ref, comps = oracle.components(n, off, tgt)
        parity = {"labels_bit_exact": bool(np.array_equal(lab, ref)) and st["components"] == comps,
                  "components": comps, "insp_sample": st["insp_sample"], "insp_finish": st["insp_finish"],
                  "cov": st["lmax_count"] / n if n else 1.0}
    times = []
    for _ in range(args.steps):
        _, st, tm = oracle.static_uf(n, off, tgt, "kout", 2, "rem_cas", "halve", "splice", threads)
        times.append(sum(tm))
    t = sum(times)
    value = (m / 2) * args.steps / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": bench_config(scale, args.edge_factor, args.seed, n, m, ws),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": "the full workload per step: C/OpenMP restatement of connlab "
                                       "_pipeline (oracle/gconn_oracle.c or_pipeline, pinned to the "
                                       "reference's own labels and statistics by tests/test_oracle.py); "
                                       "the reference itself is pure Python and takes ~45 s per run "
                                       "at this size"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "parity": parity}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--edge-factor", type=int, default=8)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--skip-check", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="run the edge-sharded path even at N=1 (used for tests)")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the dominant kernel (profiles/)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif dist_env()[0] > 1 or args.sharded:
        run_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
