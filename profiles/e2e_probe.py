"""Break the end-to-end static_connectivity call into its parts on the GPU
(H2D of the pinned CSR, the pipeline, D2H of the labels, host conversion)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_11839_b200 import Graph, build_csr, gen_rmat, parse_spec, static_connectivity  # noqa: E402
from paper_2008_11839_b200.api import static_connectivity_device  # noqa: E402


def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best, r


g = build_csr(gen_rmat(24, 8, seed=1, device=True), keep_host=False)
off_h = g._d_off.cpu().pin_memory()
tgt_h = g._d_tgt.cpu().pin_memory()
spec = parse_spec("kout+rem_cas+halve+splice")
nb = off_h.numel() * 8 + tgt_h.numel() * 4
s, _ = t(lambda: (off_h.to("cuda", non_blocking=True), tgt_h.to("cuda", non_blocking=True)))
print(f"h2d pinned {nb/1e9:.3f} GB: {s*1e3:.2f} ms = {nb/s/1e9:.1f} GB/s")
d_off, d_tgt = off_h.cuda(), tgt_h.cuda()
dg = Graph(g.n, d_off, d_tgt)
s, (lab, st) = t(lambda: static_connectivity_device(dg, spec, metrics=True))
print(f"device pipeline metrics=True: {s*1e3:.2f} ms")
s, _ = t(lambda: static_connectivity_device(dg, spec, metrics=False))
print(f"device pipeline metrics=False: {s*1e3:.2f} ms")
s, h = t(lambda: lab.cpu())
print(f"labels.cpu() pageable int32: {s*1e3:.2f} ms")
s, _ = t(lambda: h.numpy().astype(np.int64))
print(f"astype int64 host: {s*1e3:.2f} ms")
pin = torch.empty(g.n, dtype=torch.int64, pin_memory=True)
s, _ = t(lambda: pin.copy_(lab.to(torch.int64), non_blocking=True))
print(f"int64 on device + D2H pinned: {s*1e3:.2f} ms")
for _ in range(2):
    hg = Graph(g.n, off_h, tgt_h)
    s, _ = t(lambda: static_connectivity(Graph(g.n, off_h, tgt_h), spec), reps=1)
    print(f"static_connectivity(host graph) e2e: {s*1e3:.2f} ms")
