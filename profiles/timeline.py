"""Kernel timeline of one warm run through torch.profiler (CUPTI activity
records: real concurrency, no serialisation, unlike an ncu launch list).
Prints each kernel's start offset, duration and the idle gap before it, then
the busy/idle totals — the gaps are host synchronisation and launch latency.

  python profiles/timeline.py grid256:ldd+sv [warm_reps]
  python profiles/timeline.py bfs_uniform27
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2008_11839_b200 import (build_csr, gen_rmat, gen_uniform_pairs, grid3d_edges, parse_spec,  # noqa: E402
                                   spanning_forest_device, static_connectivity_device)


def workload(name):
    if name.startswith("forest_uniform27"):  # forest_uniform27[:spec]
        g = build_csr(gen_uniform_pairs(27, 4 << 27, seed=1), keep_host=False)
        sp = parse_spec(name.split(":")[1] if ":" in name else "bfs+async+halve")
        return lambda: spanning_forest_device(g, sp)
    if name.startswith("static_uniform27"):  # static_uniform27:spec
        g = build_csr(gen_uniform_pairs(27, 4 << 27, seed=1), keep_host=False)
        sp = parse_spec(name.split(":")[1])
        return lambda: static_connectivity_device(g, sp, metrics=False)
    if name == "bfs_uniform27":
        g = build_csr(gen_uniform_pairs(27, 4 << 27, seed=1), keep_host=False)
        return lambda: spanning_forest_device(g, parse_spec("bfs+async+halve"))
    if name.startswith("grid256"):
        g = build_csr(grid3d_edges(256), keep_host=False)
        sp = parse_spec(name.split(":")[1])
        return lambda: static_connectivity_device(g, sp, metrics=False)
    if name.startswith("incrp"):  # incrp26:spec[:batches] — config 4's randomly permuted stream (incr_giant_probe)
        parts = name[5:].split(":")
        scale, spec = parts[0], parts[1]
        nb = int(parts[2]) if len(parts) > 2 else 12
        from paper_2008_11839_b200 import IncrementalConnectivity
        g = build_csr(gen_rmat(int(scale), 8, seed=1, device=True), keep_host=False)
        off, tgt = g._d_off, g._d_tgt
        src = torch.repeat_interleave(torch.arange(g.n, device="cuda", dtype=torch.int32), off[1:] - off[:-1])
        keep = src < tgt
        us, vs = src[keep].contiguous(), tgt[keep].contiguous()
        perm = torch.randperm(us.numel(), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
        us, vs = us[perm].contiguous(), vs[perm].contiguous()
        del src, keep, perm
        sp = parse_spec(spec)

        def run():
            inc = IncrementalConnectivity(sp, g.n)
            inc.reserve(10_000_000)
            for b0 in range(0, min(us.numel(), nb * 10_000_000), 10_000_000):
                inc.insert(us[b0:b0 + 10_000_000], vs[b0:b0 + 10_000_000])
        return run
    if name.startswith("incr"):  # incr24:none+sv — 10M-insert batches of RMAT s24's undirected edges
        scale, spec = name[4:].split(":")
        from paper_2008_11839_b200 import IncrementalConnectivity
        g = build_csr(gen_rmat(int(scale), 8, seed=1, device=True), keep_host=False)
        off, tgt = g._d_off, g._d_tgt
        src = torch.repeat_interleave(torch.arange(g.n, device="cuda", dtype=torch.int32), off[1:] - off[:-1])
        keep = src < tgt
        us, vs = src[keep].contiguous(), tgt[keep].contiguous()
        sp = parse_spec(spec)

        def run():
            inc = IncrementalConnectivity(sp, g.n)
            for b0 in range(0, us.numel(), 10_000_000):
                inc.insert(us[b0:b0 + 10_000_000], vs[b0:b0 + 10_000_000])
        return run
    if name.startswith("plan"):  # plan24:spec — the captured StaticConnectivity plan (bench.py's step)
        scale, spec = name[4:].split(":")
        from paper_2008_11839_b200 import StaticConnectivity
        g = build_csr(gen_rmat(int(scale), 8, seed=1, device=True), keep_host=False)
        plan = StaticConnectivity(g, parse_spec(spec))
        return lambda: plan.run()
    if name.startswith("rmat"):
        scale, spec = name[4:].split(":")
        g = build_csr(gen_rmat(int(scale), 8, seed=1, device=True), keep_host=False)
        sp = parse_spec(spec)
        return lambda: static_connectivity_device(g, sp, metrics=False)
    raise SystemExit(f"unknown workload {name}")


def main():
    run = workload(sys.argv[1])
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
        run()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        run()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.device_resource_id is not None]
    ev = [e for e in ev if e.time_range.elapsed_us() >= 0]
    ev.sort(key=lambda e: e.time_range.start)
    if not ev:
        raise SystemExit("no device events")
    t0 = ev[0].time_range.start
    busy = idle = 0.0
    end = t0
    for e in ev:
        s, d = e.time_range.start, e.time_range.elapsed_us()
        gap = max(0.0, s - end)
        idle += gap
        busy += d
        end = max(end, s + d)
        print(f"{s - t0:10.1f} {d:9.1f} gap {gap:8.1f}  {e.name[:80]}")
    print(f"span {end - t0:.1f} us  busy {busy:.1f} us  idle {idle:.1f} us  events {len(ev)}")


if __name__ == "__main__":
    main()
