"""Small driver for ncu captures: run one workload `--reps` times.

  python profiles/run_workload.py bfs_uniform27|grid256:<spec>|gridperm256:<spec>|kout_s24|incr_s24|incr_s26
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2008_11839_b200 import (IncrementalConnectivity, build_csr, gen_rmat, gen_uniform_pairs,  # noqa: E402
                                   grid3d_edges, parse_spec, spanning_forest_device,
                                   static_connectivity_device)


def main():
    name = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    if name == "bfs_uniform27":
        g = build_csr(gen_uniform_pairs(27, 4 << 27, seed=1), keep_host=False)
        for _ in range(reps):
            spanning_forest_device(g, parse_spec("bfs+async+halve"))
    elif name.startswith("grid256") or name.startswith("gridperm256"):
        spec = name.split(":")[1]
        el = grid3d_edges(256)
        if name.startswith("gridperm"):
            from paper_2008_11839_b200 import EdgeList
            n = 256 ** 3
            perm = torch.randperm(n, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
            el = EdgeList(n, perm[el.edges.to("cuda")])
        g = build_csr(el, keep_host=False)
        for _ in range(reps):
            static_connectivity_device(g, parse_spec(spec), metrics=False)
    elif name == "kout_s24":
        g = build_csr(gen_rmat(24, 8, seed=1, device=True), keep_host=False)
        for _ in range(reps):
            static_connectivity_device(g, parse_spec("kout+rem_cas+halve+splice"), metrics=False)
    elif name == "incr_s24":
        g = build_csr(gen_rmat(24, 8, seed=1, device=True), keep_host=False)
        off, tgt = g._d_off, g._d_tgt
        src = torch.repeat_interleave(torch.arange(g.n, device="cuda", dtype=torch.int32), off[1:] - off[:-1])
        keep = src < tgt
        us, vs = src[keep].contiguous(), tgt[keep].contiguous()
        for _ in range(reps):
            inc = IncrementalConnectivity(parse_spec("none+async+halve"), g.n)
            for b0 in range(0, us.numel(), 10_000_000):
                inc.insert(us[b0:b0 + 10_000_000], vs[b0:b0 + 10_000_000])
    elif name == "incr_s26":
        # config 4 as bench_configs.py runs it: permuted undirected edges of
        # RMAT s26, 10M-insert batches enqueued back to back
        g = build_csr(gen_rmat(26, 8, seed=1, device=True), keep_host=False)
        off, tgt = g._d_off, g._d_tgt
        src = torch.repeat_interleave(torch.arange(g.n, device="cuda", dtype=torch.int32), off[1:] - off[:-1])
        keep = src < tgt
        us, vs = src[keep], tgt[keep]
        del src, keep
        perm = torch.randperm(us.numel(), device="cuda", generator=torch.Generator("cuda").manual_seed(1))
        us, vs = us[perm].contiguous(), vs[perm].contiguous()
        del perm
        for _ in range(reps):
            inc = IncrementalConnectivity(parse_spec("none+async+halve"), g.n)
            for b0 in range(0, us.numel(), 10_000_000):
                inc.insert(us[b0:b0 + 10_000_000], vs[b0:b0 + 10_000_000], sync=False)
            torch.cuda.synchronize()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
