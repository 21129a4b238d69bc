"""Per-batch insert times of config 4 (RMAT s26, 54 x 10M inserts) for one
union-find spec; run once with GC_INCR_GIANT=1 and once with =0.
  python profiles/incr_giant_probe.py [spec]"""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2008_11839_b200 import build_csr, gen_rmat, parse_spec, IncrementalConnectivity  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "none+async+halve"
as_list = "--list" in sys.argv  # insert_list (records merging edges, as the sharded driver)
sort_mode = next((a.split("=")[1] for a in sys.argv if a.startswith("--sort=")), "")  # experiment: batch order
g = build_csr(gen_rmat(26, 8, seed=1, device=True), keep_host=False)
off, tgt = g._d_off, g._d_tgt
src = torch.repeat_interleave(torch.arange(g.n, device="cuda", dtype=torch.int32), off[1:] - off[:-1])
keep = src < tgt
us, vs = src[keep].contiguous(), tgt[keep].contiguous()
perm = torch.randperm(us.numel(), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
us, vs = us[perm].contiguous(), vs[perm].contiguous()
del src, keep, perm
for rep in range(2):
    inc = IncrementalConnectivity(parse_spec(spec), g.n)
    inc.reserve(10_000_000)
    torch.cuda.synchronize()
    ts = []
    batches = []
    for b0 in range(0, us.numel(), 10_000_000):
        bu, bv = us[b0:b0 + 10_000_000], vs[b0:b0 + 10_000_000]
        if sort_mode == "u":  # by u (untimed): P[u] reads local
            o = torch.argsort(bu)
            bu, bv = bu[o].contiguous(), bv[o].contiguous()
        elif sort_mode.startswith("ushift"):  # by u >> k (2^k-vertex windows of P)
            o = torch.argsort(bu >> int(sort_mode[6:]), stable=True)
            bu, bv = bu[o].contiguous(), bv[o].contiguous()
        batches.append((bu, bv))
    for bu, bv in batches:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if as_list:
            inc.insert_list(bu, bv)
        else:
            inc.insert(bu, bv, sync=False)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    if rep:
        print(json.dumps({"spec": spec, "list": as_list, "sort": sort_mode, "total_ms": sum(ts), "batch_ms": [round(t, 4) for t in ts]}))
    del inc
