"""Single-GPU static step (the bench's plan replay, L2 flushed between runs)
at RMAT scale s, for comparing the sharded model's weak-scaling graphs with
one GPU on the same graph.
  python profiles/single_scale.py 24 25 26 27"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2008_11839_b200 import build_csr, gen_rmat, parse_spec  # noqa: E402
from paper_2008_11839_b200.api import StaticConnectivity  # noqa: E402

spec = parse_spec("kout+rem_cas+halve+splice")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for s in (int(x) for x in sys.argv[1:]):
    g = build_csr(gen_rmat(s, 8, seed=1, device=True), keep_host=False)
    plan = StaticConnectivity(g, spec)
    for _ in range(3):
        plan.run()
    ts = []
    for r in range(10):
        flush.fill_(r)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.run()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    print(json.dumps({"scale": s, "n": g.n, "m_directed": g.m, "step_ms": ms,
                      "edges_per_s": (g.m / 2) / (ms / 1e3)}), flush=True)
    del plan, g
    torch.cuda.empty_cache()
