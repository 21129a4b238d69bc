"""The sharded drivers on the GPU engine (libgconn).  One GPU is visible, so
(1) the P-rank tree merge is replayed in-process shard by shard, and (2) two
real ranks share cuda:0 over gloo (collectives staged through host memory)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
from golden_data import Golden

pytestmark = pytest.mark.gpu


def _merge_in_process(g, spec, world):
    from paper_2008_11839_b200.distributed import GpuEngine, shard_bounds, shard_graph
    eng = GpuEngine()
    states = []
    for lo, hi in shard_bounds(g.offsets, world):
        states.append(list(eng.local_forest(shard_graph(g, lo, hi), spec)))
    step = 1
    while step < world:
        for r in range(0, world, 2 * step):
            if r + step < world:
                parent, fu, fv = states[r]
                _, ou, ov = states[r + step]
                mu, mv = eng.union_list(parent, ou, ov, spec)
                states[r] = [parent, torch.cat([fu, mu]), torch.cat([fv, mv])]
        step *= 2
    parent, fu, fv = states[0]
    return eng.finalize(parent), fu, fv


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_tree_merge_on_gpu(world):
    from paper_2008_11839_b200 import Graph, build_csr, gen_rmat, parse_spec
    gold = Golden()
    graphs = [(name,) + gold.graphs[name] for name in ["rmat_s10_ef8", "comps_30", "two_comp", "grid_12x12"]]
    g16 = build_csr(gen_rmat(16, 8, seed=1, device=True))
    o16, _ = oracle.components(g16.n, g16.offsets, g16.targets)
    graphs.append(("rmat_s16", g16.n, g16.offsets, g16.targets, o16))
    for spec_text in ["none+async+halve", "none+rem_cas+split+halve", "none+hooks+compress", "none+jtb+naive"]:
        spec = parse_spec(spec_text)
        for name, n, off, tgt, orc in graphs:
            labels, fu, fv = _merge_in_process(Graph(n, off, tgt), spec, world)
            lab = labels.cpu().numpy().astype(np.int64)
            from paper_2008_11839_b200 import label_finalization
            assert np.array_equal(label_finalization(lab), orc), (name, spec_text, world)
            su = np.full(n, -1, np.int32); sv = np.full(n, -1, np.int32)
            su[:fu.numel()] = fu.cpu().numpy(); sv[:fv.numel()] = fv.cpu().numpy()
            rep = oracle.check_forest(n, off, tgt, su, sv, orc)
            assert rep["passed"], (name, spec_text, world, rep)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _two_rank_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2008_11839_b200 import build_csr, gen_rmat, parse_spec
        from paper_2008_11839_b200.distributed import ShardedIncremental, shard_bounds, shard_graph, \
            sharded_spanning_forest
        g = build_csr(gen_rmat(14, 8, seed=3, device=True))
        lo, hi = shard_bounds(g.offsets, world)[rank]
        res = sharded_spanning_forest(shard_graph(g.cuda(), lo, hi), parse_spec("none+async+halve"))
        # incremental: the graph's edges in 8 batches, then queries
        ue = g.undirected_edges()
        inc = ShardedIncremental(parse_spec("none+async+halve"), g.n)
        for part in np.array_split(np.arange(len(ue)), 8):
            inc.insert(torch.from_numpy(ue[part, 0].astype(np.int32)).cuda(),
                       torch.from_numpy(ue[part, 1].astype(np.int32)).cuda())
        lab, comps = inc.labels()
        q.put((rank, (res.labels.cpu().numpy(), res.forest_u.cpu().numpy(), res.forest_v.cpu().numpy(),
                      lab.cpu().numpy(), comps)))
    finally:
        dist.destroy_process_group()


def test_two_ranks_share_one_gpu():
    import torch.multiprocessing as mp
    from paper_2008_11839_b200 import build_csr, gen_rmat
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_two_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    g = build_csr(gen_rmat(14, 8, seed=3, device=True))
    orc, comps = oracle.components(g.n, g.offsets, g.targets)
    iso = int((np.diff(g.offsets) == 0).sum())
    for r in range(2):
        labels, fu, fv, ilab, icomps = res[r]
        assert np.array_equal(labels.astype(np.int64), orc)
        su = np.full(g.n, -1, np.int32); sv = np.full(g.n, -1, np.int32)
        su[:len(fu)] = fu; sv[:len(fv)] = fv
        assert oracle.check_forest(g.n, g.offsets, g.targets, su, sv, orc)["passed"]
        assert np.array_equal(ilab.astype(np.int64), orc)
        assert icomps == comps - iso


def _two_phase_gpu_worker(rank, world, port, specs, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2008_11839_b200 import build_csr, gen_rmat, parse_spec
        from paper_2008_11839_b200.distributed import shard_bounds, shard_graph, sharded_two_phase
        g = build_csr(gen_rmat(15, 8, seed=5, device=True))
        lo, hi = shard_bounds(g.offsets, world)[rank]
        out = {}
        for text in specs:
            r = sharded_two_phase(shard_graph(g.cuda(), lo, hi), parse_spec(text.lstrip("~")),
                                  forest=not text.startswith("~"))
            out[text] = (r.labels.cpu().numpy(), None if r.forest_u is None else r.forest_u.cpu().numpy(),
                         None if r.forest_v is None else r.forest_v.cpu().numpy(), r.insp_sample, r.insp_finish,
                         r.lmax_count, r.n_active)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_two_phase_sampled_ranks_share_one_gpu(world):
    """Sampled specs over row shards on the GPU engine: labels bit-exact and
    inspection counts / cov / active set equal to the single-GPU pipeline."""
    import torch.multiprocessing as mp
    from paper_2008_11839_b200 import build_csr, gen_rmat, parse_spec, static_connectivity_device
    # "~spec": labels only through the compact giant-bitmap summary exchange
    specs = ["kout+rem_cas+halve+splice", "kout+async+halve", "hb+rem_cas+split+halve", "none+hooks+compress",
             "~kout+rem_cas+halve+splice", "~hb+jtb+twotry", "~kout+hooks+compress",
             # distributed level-synchronous BFS sampling (gc_dbfs_*)
             "bfs+async+halve", "~bfs+rem_cas+halve+splice"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_two_phase_gpu_worker, args=(r, world, port, specs, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    g = build_csr(gen_rmat(15, 8, seed=5, device=True))
    orc, comps = oracle.components(g.n, g.offsets, g.targets)
    for text in specs:
        _, st = static_connectivity_device(g, parse_spec(text.lstrip("~")))
        for r in range(world):
            labels, fu, fv, i_s, i_f, lcnt, nact = res[r][text]
            assert np.array_equal(labels.astype(np.int64), orc), (text, r)
            assert i_s == st.edge_inspections.get("sample", 0), (text, r)
            assert i_f == st.edge_inspections.get("finish", 0), (text, r)
            assert lcnt / g.n == st.cov and nact == st.active, (text, r)
            if fu is not None:
                su = np.full(g.n, -1, np.int32); sv = np.full(g.n, -1, np.int32)
                su[:len(fu)] = fu; sv[:len(fv)] = fv
                assert oracle.check_forest(g.n, g.offsets, g.targets, su, sv, orc)["passed"], (text, r)


def _two_giants_graph():
    """Two disjoint RMAT s13 halves: with two row blocks each rank's local
    giant lies in a different component, so the absorb takes its general
    multi-class path (the single-class fast path does not apply)."""
    import torch
    from paper_2008_11839_b200 import EdgeList, build_csr, gen_rmat
    a = gen_rmat(13, 8, seed=7, device=True).edges.to("cuda")
    b = gen_rmat(13, 8, seed=8, device=True).edges.to("cuda") + (1 << 13)
    return build_csr(EdgeList(1 << 14, torch.cat([a, b])))


def _two_giants_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2008_11839_b200 import parse_spec
        from paper_2008_11839_b200.distributed import shard_bounds, shard_graph, sharded_two_phase
        g = _two_giants_graph()
        lo, hi = shard_bounds(g.offsets, world, "rows")[rank]
        r = sharded_two_phase(shard_graph(g.cuda(), lo, hi), parse_spec("kout+rem_cas+halve+splice"), forest=False)
        q.put((rank, (r.labels.cpu().numpy(), r.insp_sample, r.insp_finish, r.lmax_count, r.n_active)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_summary_exchange_disjoint_giants(world):
    import torch.multiprocessing as mp
    from paper_2008_11839_b200 import parse_spec, static_connectivity_device
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_two_giants_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    g = _two_giants_graph()
    orc, _ = oracle.components(g.n, g.offsets, g.targets)
    _, st = static_connectivity_device(g, parse_spec("kout+rem_cas+halve+splice"))
    for r in range(world):
        labels, i_s, i_f, lcnt, nact = res[r]
        assert np.array_equal(labels.astype(np.int64), orc), r
        assert i_s == st.edge_inspections.get("sample", 0) and i_f == st.edge_inspections.get("finish", 0), r
        assert lcnt / g.n == st.cov and nact == st.active, r


def _dbfs_uniform_worker(rank, world, port, log2n, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2008_11839_b200 import build_csr, gen_uniform_pairs, parse_spec
        from paper_2008_11839_b200.distributed import shard_bounds, shard_graph, sharded_two_phase
        n = 1 << log2n
        g = build_csr(gen_uniform_pairs(log2n, 4 * n, seed=1), keep_host=False)
        lo, hi = shard_bounds(g._d_off, world)[rank]
        r = sharded_two_phase(shard_graph(g, lo, hi), parse_spec("bfs+async+halve"), forest=True)
        # the same run with the forest returned as per-rank slices
        s = sharded_two_phase(shard_graph(g, lo, hi), parse_spec("bfs+async+halve"), forest=True,
                              forest_slices=True)
        q.put((rank, (r.labels.cpu().numpy(), r.forest_u.cpu().numpy(), r.forest_v.cpu().numpy(), r.insp_sample,
                      r.insp_finish, r.lmax_count, r.n_active, s.labels.cpu().numpy(), s.forest_u.cpu().numpy(),
                      s.forest_v.cpu().numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_bfs_forest_config5_shape(world):
    """Config 5 scaled (uniform 2^20, 4n pairs, bfs+async+halve spanning
    forest): the distributed BFS sampler + sharded finish give the oracle
    labels, a forest passing the four clauses on every rank, and the
    single-GPU pipeline's inspection counts / cov / active set."""
    import torch.multiprocessing as mp
    from paper_2008_11839_b200 import build_csr, gen_uniform_pairs, parse_spec, spanning_forest_device
    log2n = 20
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dbfs_uniform_worker, args=(r, world, port, log2n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    n = 1 << log2n
    g = build_csr(gen_uniform_pairs(log2n, 4 * n, seed=1))
    orc, comps = oracle.components(n, g.offsets, g.targets)
    _, st = spanning_forest_device(g, parse_spec("bfs+async+halve"))
    slices_u, slices_v = [], []
    for r in range(world):
        labels, fu, fv, i_s, i_f, lcnt, nact, slab, slu, slv = res[r]
        assert np.array_equal(slab.astype(np.int64), orc), r
        slices_u.append(slu)
        slices_v.append(slv)
        assert np.array_equal(labels.astype(np.int64), orc), r
        assert i_s == st.edge_inspections.get("sample", 0) and i_f == st.edge_inspections.get("finish", 0), r
        assert lcnt / n == st.cov and nact == st.active, r
        assert len(fu) == n - comps
        su = np.full(n, -1, np.int32); sv = np.full(n, -1, np.int32)
        su[:len(fu)] = fu; sv[:len(fv)] = fv
        assert oracle.check_forest(n, g.offsets, g.targets, su, sv, orc)["passed"], r
    # the slices' union is one spanning forest
    fu, fv = np.concatenate(slices_u), np.concatenate(slices_v)
    assert len(fu) == n - comps
    su = np.full(n, -1, np.int32); sv = np.full(n, -1, np.int32)
    su[:len(fu)] = fu; sv[:len(fv)] = fv
    assert oracle.check_forest(n, g.offsets, g.targets, su, sv, orc)["passed"]
