"""Multi-GPU model for the sharded two-phase pipeline, measured on ONE GPU.

This environment exposes a single B200, so the P-rank run is replayed in one
process: every rank's device work (sample its row block, summarise, join all
summaries, finish its active rows, merge the finish edges, finalise) runs on
the GPU one rank after another and is timed with CUDA events per stage; the
collectives are replaced by in-memory concatenation and costed from the
bytes they would move at the measured NVLink peer bandwidth (770 GB/s per
direction, B200_PROFILING.md).  Predicted step = max over ranks of the
device time + the collective time.  Labels are checked against the C oracle.

  python profiles/shard_model.py [--ranks 1,2,4,8] [--scale0 24] [--reps 3]
"""
import argparse
import json
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_11839_b200 import build_csr, gen_rmat, parse_spec  # noqa: E402
from paper_2008_11839_b200.distributed import GpuEngine, shard_balance, shard_bounds, shard_graph  # noqa: E402

NVLINK = 770e9  # bytes/s per direction, measured peer copy (B200_PROFILING.md)


class Timer:
    def __init__(self):
        self.t = {}

    def __call__(self, name, fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        e1.synchronize()
        self.t[name] = self.t.get(name, 0.0) + e0.elapsed_time(e1)
        return out


def build(P, scale0, strong=False):
    scale = scale0 if strong else scale0 + int(math.ceil(math.log2(P)))
    g = build_csr(gen_rmat(scale, 8, seed=1, device=True), keep_host=False)
    by = shard_balance(parse_spec("kout+rem_cas+halve+splice"))
    return scale, g, [shard_graph(g, lo, hi) for lo, hi in shard_bounds(g._d_off, P, by)]


def run(P, scale, g, shards, check):
    spec = parse_spec("kout+rem_cas+halve+splice")
    n, m = g.n, g.m
    eng = GpuEngine()
    timers = [Timer() for _ in range(P)]
    # phase 1: sample + summary on every rank
    states = []
    for r in range(P):
        T = timers[r]
        parent, _, _, _ = T("sample", lambda: eng.shard_sample(shards[r], spec, record=False))
        words, label, _, _ = T("summaryA", lambda: eng.shard_summary(parent, pairs=False))
        states.append([parent, words, label])
    wa = torch.stack([s[1] for s in states])
    la = torch.cat([s[2] for s in states])
    for r in range(P):
        T = timers[r]
        parent = states[r][0]
        rep = T("absorb", lambda: eng.shard_absorb(parent, wa, la))
        words, label, ru, rv = T("summaryB", lambda: eng.shard_summary(parent, hint=rep, pairs=True))
        states[r] += [words, label, ru, rv]
    words_all = torch.stack([s[3] for s in states])
    labels_all = torch.cat([s[4] for s in states])
    us = torch.cat([s[5] for s in states])
    vs = torch.cat([s[6] for s in states])
    # what each rank receives: two rounds of bitmaps + the remainder pairs
    bytes1 = wa.numel() * 4 + words_all.numel() * 4 + us.numel() * 8 + 16 * P
    fin = []
    for r in range(P):
        T = timers[r]
        parent = states[r][0]
        T("join", lambda: eng.shard_join(parent, words_all, labels_all, us, vs, spec))
        mu, mv, _ = T("finish", lambda: eng.shard_finish(shards[r], spec, parent))
        fin.append((mu, mv))
    fu = torch.cat([f[0] for f in fin])
    fv = torch.cat([f[1] for f in fin])
    bytes2 = fu.numel() * 8
    labels = None
    for r in range(P):
        T = timers[r]
        parent = states[r][0]
        fq = [fin[q] for q in range(P) if q != r and fin[q][0].numel()]
        if fq:  # the foreign lists as one batch, as _exchange_and_merge does
            ou, ov = torch.cat([f[0] for f in fq]), torch.cat([f[1] for f in fq])
            T("merge2", lambda: eng.union_pairs(parent, ou, ov, spec))
        lab = T("finalize", lambda: eng.finalize(parent, inplace=True))
        if r == 0:
            labels = lab
    ok = None
    if check:
        import oracle
        ref, _ = oracle.components(n, g._d_off.cpu().numpy(), g._d_tgt.cpu().numpy())
        ok = bool(np.array_equal(labels.cpu().numpy().astype(np.int64), ref))
    dev = [sum(T.t.values()) for T in timers]
    comm_ms = (bytes1 + bytes2) / NVLINK * 1e3 if P > 1 else 0.0
    step = max(dev) + comm_ms
    return {"ranks": P, "scale": int(math.log2(n)), "n": n, "m_directed": m, "labels_ok": ok,
            "device_ms_max": max(dev), "comm_ms_model": comm_ms, "step_ms_model": step,
            "edges_per_s_model": (m / 2) / (step / 1e3),
            "stage_ms_rank0": {k: round(v, 4) for k, v in timers[0].t.items()},
            "bytes_phase1_per_rank": bytes1, "bytes_phase2_per_rank": bytes2, "remainder_pairs": int(us.numel())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--scale0", type=int, default=24)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--strong", action="store_true", help="same graph for every P (strong scaling)")
    a = ap.parse_args()
    for P in (int(x) for x in a.ranks.split(",")):
        scale, g, shards = build(P, a.scale0, a.strong)
        ok = run(P, scale, g, shards, a.check)["labels_ok"]  # warm-up (allocator, caches) + check
        best = None
        for _ in range(a.reps):
            r = run(P, scale, g, shards, False)
            if best is None or r["step_ms_model"] < best["step_ms_model"]:
                best = r
        best["labels_ok"] = ok
        print(json.dumps(best), flush=True)
        del g, shards
        torch.cuda.empty_cache()




def run_incremental(P, scale, batch, check):
    """Batch-sharded incremental (ShardedIncremental) replayed on one GPU:
    per batch every rank inserts its 1/P slice recording merging edges, the
    merges are exchanged (costed at NVLink rate) and every rank inserts the
    foreign ones; batch time = max over ranks + exchange."""
    from paper_2008_11839_b200 import IncrementalConnectivity
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
    spec = parse_spec("none+async+halve")
    reps = [IncrementalConnectivity(spec, n) for _ in range(P)]
    for rp in reps:
        rp.reserve(batch)  # buffer allocation outside the timed batches
    total_ms, comm_bytes = 0.0, 0
    per_batch = []
    for b0 in range(0, us.numel(), batch):
        bu, bv = us[b0:b0 + batch], vs[b0:b0 + batch]
        k = bu.numel()
        t_rank = [0.0] * P
        merges = []
        for r in range(P):
            lo, hi = (k * r) // P, (k * (r + 1)) // P
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            mu, mv = reps[r].insert_list(bu[lo:hi], bv[lo:hi])
            e1.record()
            e1.synchronize()
            t_rank[r] += e0.elapsed_time(e1)
            merges.append((mu, mv))
        if P > 1:
            for r in range(P):
                fu = torch.cat([m[0] for q, m in enumerate(merges) if q != r])
                fv = torch.cat([m[1] for q, m in enumerate(merges) if q != r])
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                if fu.numel():
                    reps[r].insert(fu, fv)
                e1.record()
                e1.synchronize()
                t_rank[r] += e0.elapsed_time(e1)
            nbytes = sum(m[0].numel() for m in merges) * 8
            comm_bytes += nbytes
            total_ms += max(t_rank) + nbytes / NVLINK * 1e3
            per_batch.append((round(max(t_rank), 4), int(sum(m[0].numel() for m in merges))))
        else:
            total_ms += t_rank[0]
            per_batch.append((round(t_rank[0], 4), int(merges[0][0].numel())))
    ok = None
    if check:
        import oracle
        ref, _ = oracle.components(n, off.cpu().numpy(), tgt.cpu().numpy())
        lab, _ = reps[0].labels()
        lab = lab.cpu().numpy().astype(np.int64)
        deg = np.diff(off.cpu().numpy())
        ok = bool(np.array_equal(lab[deg > 0], ref[deg > 0]))
    return {"mode": "incremental", "ranks": P, "scale": scale, "n": n, "inserts": int(us.numel()), "batch": batch,
            "labels_ok": ok, "step_ms_model": total_ms, "inserts_per_s_model": us.numel() / (total_ms / 1e3),
            "exchanged_bytes": comm_bytes, "batch_ms_merges": per_batch}


def run_bfs_forest(P, log2n, check):
    """Config 5 sharded (sharded_two_phase with BFS sampling, spanning
    forest, bfs+async+halve on uniform 2^log2n, strong scaling: the same
    graph split over P row blocks), replayed on one GPU.  Per BFS level: each
    rank's marks / merge / claim / advance timed with CUDA events, the mark
    lists all-gathered and the next-frontier bitmaps all-reduced (costed at
    NVLink rate); then each rank's tree edges all-gathered, its finish over
    its active rows, the merging edges exchanged and unioned, finalise.
    Step = sum over levels of (max over ranks + collectives) + the same for
    the later phases."""
    from paper_2008_11839_b200 import gen_uniform_pairs
    from paper_2008_11839_b200.distributed import DBFS_ALPHA, DBFS_BETA
    spec = parse_spec("bfs+async+halve")
    g = build_csr(gen_uniform_pairs(log2n, 4 << log2n, seed=1, device=True), keep_host=False)
    n, m = g.n, g.m
    shards = [shard_graph(g, lo, hi) for lo, hi in shard_bounds(g._d_off, P, "edges")]
    eng = GpuEngine()
    for sh in shards:  # the once-per-graph CSR validation, outside the timing
        eng._dbfs_csr(sh)
    words_bytes = ((n + 31) // 32) * 4

    def ev(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        e1.synchronize()
        return out, e0.elapsed_time(e1)

    # BFS source: highest-degree probe (sampling.py:130-132), global degrees
    probes = np.unique(np.random.default_rng(spec.seed).integers(0, n, size=spec.bfs_probes))
    deg = (g._d_off[torch.as_tensor(probes + 1, device="cuda")] - g._d_off[torch.as_tensor(probes, device="cuda")])
    src = int(probes[int(torch.argmax(deg).item())])
    sts = [eng.dbfs_init(n, src) for _ in range(P)]
    torch.cuda.synchronize()
    total_ms, comm_ms = 0.0, 0.0
    nf, reached, bottom_up, levels = 1, 1, False, 0
    while nf:
        bottom_up = nf * DBFS_ALPHA > n - reached if not bottom_up else nf >= n // DBFS_BETA
        t = [0.0] * P
        tt = {k: [0.0] * P for k in ("marks", "merge", "claim", "advance")}
        nxt = []
        if bottom_up:
            for r in range(P):
                out, dt = ev(lambda: eng.dbfs_claim(shards[r], sts[r], marks=False))
                t[r] += dt
                tt["claim"][r] += dt
                nxt.append(out)
        else:
            ids = []
            for r in range(P):
                out, dt = ev(lambda: eng.dbfs_marks(shards[r], sts[r]).clone())
                t[r] += dt
                tt["marks"][r] += dt
                ids.append(out)
            sent = sum(int(x.numel()) for x in ids)
            comm_ms += sent * 4 / NVLINK * 1e3 if P > 1 else 0.0
            for r in range(P):
                # the foreign lists merged as one batch (distributed_bfs)
                foreign = [ids[q] for q in range(P) if q != r and ids[q].numel()]
                fl = torch.cat(foreign) if foreign else None
                out, dt = ev(lambda: eng.dbfs_claim(shards[r], sts[r], marks=True, foreign=fl))
                t[r] += dt
                tt["claim"][r] += dt
                nxt.append(out)
        # all-reduce of the disjoint next-frontier bitmaps (SUM == OR)
        acc = nxt[0].clone()
        for q in range(1, P):
            acc += nxt[q]
        for r in range(P):
            nxt[r].copy_(acc)
        if P > 1:
            comm_ms += 2 * (P - 1) / P * words_bytes / NVLINK * 1e3
        nfs = []
        for r in range(P):
            out, dt = ev(lambda: eng.dbfs_advance(sts[r]))
            t[r] += dt
            tt["advance"][r] += dt
            nfs.append(out)
        nf = nfs[0]
        reached += nf
        levels += 1
        total_ms += max(t)
        if os.environ.get("BFS_MODEL_TRACE"):
            print(f"level {levels} {'bu' if bottom_up else 'td'} next {nf} max_rank_ms {max(t):.3f} "
                  f"{ {k: round(max(v), 3) for k, v in tt.items()} }", file=sys.stderr)
    levels_ms = total_ms
    fin = []
    t = [0.0] * P
    for r in range(P):
        out, dt = ev(lambda: eng.dbfs_finish(shards[r], sts[r]))
        t[r] += dt
        fin.append(out)
    total_ms += max(t)
    dbfs_finish_ms = max(t)
    tree_pairs = sum(int(f[1].numel()) for f in fin)
    level_comm_ms = comm_ms
    # replicated forest output: the BFS tree all-gathered (forest_slices=True
    # keeps each rank's tree edges local and skips it)
    tree_comm_ms = tree_pairs * 8 * (P - 1) / P / NVLINK * 1e3 if P > 1 else 0.0
    parents = [f[0].contiguous() for f in fin]
    del sts
    # finish over each rank's active rows, merge exchange, finalise
    t = [0.0] * P
    merges = []
    for r in range(P):
        out, dt = ev(lambda: eng.shard_finish(shards[r], spec, parents[r]))
        t[r] += dt
        merges.append(out)
    mbytes = sum(int(x[0].numel()) for x in merges) * 8
    if P > 1:
        comm_ms += mbytes / NVLINK * 1e3
    labels = None
    for r in range(P):
        fq = [merges[q] for q in range(P) if q != r and merges[q][0].numel()]
        if fq:
            ou, ov = torch.cat([f[0] for f in fq]), torch.cat([f[1] for f in fq])
            _, dt = ev(lambda: eng.union_list(parents[r], ou, ov, spec))
            t[r] += dt
        lab, dt = ev(lambda: eng.finalize(parents[r], inplace=True))
        t[r] += dt
        if r == 0:
            labels = lab
    total_ms += max(t)
    ok = None
    if check:
        import oracle
        ref, _ = oracle.components(n, g._d_off.cpu().numpy(), g._d_tgt.cpu().numpy())
        ok = bool(np.array_equal(labels.cpu().numpy().astype(np.int64), ref))
    step = total_ms + comm_ms + tree_comm_ms
    return {"mode": "bfs_forest", "ranks": P, "log2n": log2n, "n": n, "m_directed": m, "labels_ok": ok,
            "levels": levels, "device_ms": total_ms, "levels_ms": levels_ms, "dbfs_finish_ms": dbfs_finish_ms,
            "finish_merge_finalize_ms": total_ms - levels_ms - dbfs_finish_ms, "level_comm_ms": level_comm_ms,
            "tree_comm_ms": tree_comm_ms, "step_ms_model_slices": total_ms + comm_ms, "comm_ms_model": comm_ms, "step_ms_model": step,
            "edges_per_s_model": (m / 2) / (step / 1e3),
            "edges_per_s_model_slices": (m / 2) / ((total_ms + comm_ms) / 1e3), "tree_pairs": tree_pairs}


def main_bfs():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bfs", action="store_true")
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--log2n", type=int, default=27)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    for P in (int(x) for x in a.ranks.split(",")):
        run_bfs_forest(P, a.log2n, False)  # warm-up
        print(json.dumps(run_bfs_forest(P, a.log2n, a.check)), flush=True)
        torch.cuda.empty_cache()


def main_incremental():
    ap = argparse.ArgumentParser()
    ap.add_argument("--incremental", action="store_true")
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--batch", type=int, default=10_000_000)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    for P in (int(x) for x in a.ranks.split(",")):
        run_incremental(P, a.scale, a.batch, False)  # warm-up
        print(json.dumps(run_incremental(P, a.scale, a.batch, a.check)), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    if "--incremental" in sys.argv:
        main_incremental()
    elif "--bfs" in sys.argv:
        main_bfs()
    else:
        main()
