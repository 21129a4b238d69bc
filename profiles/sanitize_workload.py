"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
every sampler x a spread of finishes, forests, incremental (plain and racy),
DisjointSets probes, check_forest, the sharded building blocks."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_11839_b200 import (DisjointSets, FindOp, IncrementalConnectivity, SpliceOp, UnionConfig,  # noqa: E402
                                   UnionOp, build_csr, check_forest, gen_rmat, gen_uniform_pairs, parse_spec, spanning_forest_device,
                                   static_connectivity)
from paper_2008_11839_b200.distributed import GpuEngine, shard_bounds, shard_graph  # noqa: E402

g = build_csr(gen_rmat(10, 8, seed=3, device=True))
ref = None
for text in ["none+rem_cas+naive+splice", "kout+rem_cas+halve+splice", "hb+hooks+compress", "bfs+async+halve",
             "ldd+sv", "none+lt_prs", "kout+lt_crfa", "none+stergiou", "hb+lp", "kout+jtb+twotry",
             "none+rem_lock+split+halve", "bfs+early+split"]:
    lab, st = static_connectivity(g, parse_spec(text))
    ref = lab if ref is None else ref
    assert np.array_equal(lab, ref), text
for text in ["bfs+async+halve", "none+sv", "kout+rem_cas+split+split", "none+lt_prf"]:
    df, st = spanning_forest_device(g, parse_spec(text))
    assert check_forest(g, df, ref)["passed"], text
# a frontier above the wide top-down threshold (2^16): bitmap mark + parent pull
gu = build_csr(gen_uniform_pairs(18, 4 << 18, seed=1, device=True))
refu = static_connectivity(gu, parse_spec("none+async+halve"))[0]
df, st = spanning_forest_device(gu, parse_spec("bfs+async+halve"))
assert check_forest(gu, df, refu)["passed"]
ue = g.undirected_edges()
us = torch.from_numpy(ue[:, 0].astype(np.int32)).cuda()
vs = torch.from_numpy(ue[:, 1].astype(np.int32)).cuda()
for text, racy in [("none+async+halve", False), ("none+rem_cas+halve+split", True), ("none+sv", False)]:
    inc = IncrementalConnectivity(parse_spec(text), g.n, racy=racy)
    isq = torch.zeros(us.numel(), dtype=torch.uint8, device="cuda")
    isq[::7] = 1
    inc.batch(us, vs, isq)
    inc.labels()
# the incremental giant filter: a second pass over the same edges runs in
# compact mode; insert_list flags merges by index
inc = IncrementalConnectivity(parse_spec("none+async+halve"), g.n)
inc.reserve(2048)
for rep in range(2):
    for b0 in range(0, us.numel(), 2048):
        inc.insert_list(us[b0:b0 + 2048], vs[b0:b0 + 2048])
for b0 in range(0, us.numel(), 2048):
    inc.insert(us[b0:b0 + 2048], vs[b0:b0 + 2048], sync=False)
inc.query(us[:1000], vs[:1000])
inc.labels()
ds = DisjointSets(g.n, UnionConfig(UnionOp.REM_CAS, FindOp.HALVE, SpliceOp.SPLIT_ONE))
ds.union_batch(us, vs)
ds.labels_array()
eng = GpuEngine()
spec = parse_spec("kout+rem_cas+halve+splice")
for lo, hi in shard_bounds(g.offsets, 2):
    sh = shard_graph(g.cuda(), lo, hi)
    parent, _, _, _ = eng.shard_sample(sh, spec, record=False)
    w, lab1, _, _ = eng.shard_summary(parent, pairs=False)
    rep = eng.shard_absorb(parent, torch.stack([w, w]), torch.cat([lab1, lab1]))
    w2, lab2, ru, rv = eng.shard_summary(parent, hint=rep, pairs=True)
    eng.shard_join(parent, torch.stack([w2, w2]), torch.cat([lab2, lab2]), ru, rv, spec)
    eng.shard_finish(sh, spec, parent)
torch.cuda.synchronize()
print("sanitize workload ok")
