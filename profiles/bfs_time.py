"""Time the BFS-sampled spanning forest on the config-5 graph (uniform 2^27,
4n pairs): median of CUDA-event times after warm-up."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2008_11839_b200 import build_csr, gen_uniform_pairs, parse_spec, spanning_forest_device  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
g = build_csr(gen_uniform_pairs(lg, 4 << lg, seed=1), keep_host=False)
for text in sys.argv[2:] or ["bfs+async+halve"]:
    sp = parse_spec(text)
    for _ in range(2):
        spanning_forest_device(g, sp)
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        spanning_forest_device(g, sp)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(text, "forest ms", round(statistics.median(ts), 3))
