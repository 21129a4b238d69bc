import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2008_11839_b200 import build_csr, gen_rmat, parse_spec, IncrementalConnectivity
g = build_csr(gen_rmat(26, 8, seed=1, device=True), keep_host=False)
off, tgt = g._d_off, g._d_tgt
src = torch.repeat_interleave(torch.arange(g.n, device="cuda", dtype=torch.int32), off[1:] - off[:-1])
keep = src < tgt
us, vs = src[keep].contiguous(), tgt[keep].contiguous()
perm = torch.randperm(us.numel(), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
us, vs = us[perm].contiguous(), vs[perm].contiguous()
for text in ["none+sv", "none+sv"]:
    inc = IncrementalConnectivity(parse_spec(text), g.n)
    torch.cuda.synchronize()
    ts = []
    for b0 in range(0, us.numel(), 10_000_000):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(); inc.insert(us[b0:b0 + 10_000_000], vs[b0:b0 + 10_000_000]); e1.record(); e1.synchronize()
        ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3, inc.stats.rounds if hasattr(inc, "stats") else -1))
    print(text, "total", round(sum(t[0] for t in ts), 2), "wall", round(sum(t[1] for t in ts), 2))
    print([round(t[0], 2) for t in ts[:12]], [round(t[0], 2) for t in ts[-6:]])
    del inc
