"""The largest vertex count the ABI accepts (2^31 - 1 ids; the incremental
capacity one below, its sentinel being the capacity itself).

A sparse graph over the whole id range: 2^20 random edges among vertices
drawn from the bottom and the top 2^21 ids, a path through 0 and n - 1, the
rest isolated.  Every per-vertex array (offsets 17 GB, labels, bitmaps,
LDD's unpacked claim state — n exceeds the packed key's 2^24) spans the
full range, so 32-bit index arithmetic anywhere on the path would show up as
a fault or a wrong label.  Expected labels come from the oracle run on the
graph compacted to its touched vertices (compaction keeps id order, so
component minima map back unchanged); untouched vertices are their own
component."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

N_MAX = (1 << 31) - 1


@pytest.fixture(scope="module")
def huge():
    import torch
    from paper_2008_11839_b200 import EdgeList, build_csr
    free, _ = torch.cuda.mem_get_info()
    if free < (100 << 30):
        pytest.skip("needs ~100 GB of free device memory")
    rng = np.random.default_rng(11)
    pool = np.concatenate([rng.integers(0, 1 << 21, size=1 << 19), rng.integers(N_MAX - (1 << 21), N_MAX, size=1 << 19),
                           [0, N_MAX - 1]])
    e = pool[rng.integers(0, len(pool), size=(1 << 20, 2))]
    e = np.concatenate([e, [[0, N_MAX - 1], [N_MAX - 1, N_MAX - 2], [1, 0], [0, N_MAX - 2]]])
    touched = np.unique(e)
    ce = np.searchsorted(touched, e)
    coff, ctgt = oracle.build_csr(len(touched), ce)
    clab, ccomps = oracle.components(len(touched), coff, ctgt)
    exp_t = touched[clab]
    g = build_csr(EdgeList(N_MAX, torch.from_numpy(e).cuda()), keep_host=False)
    return g, e, touched, exp_t, ccomps, (coff, ctgt, clab)


def _check_labels(labels, touched, exp_t):
    import torch
    n = labels.numel()
    assert n == N_MAX
    t = torch.from_numpy(touched).cuda()
    assert torch.equal(labels[t].to(torch.int64), torch.from_numpy(exp_t).cuda())
    moved = torch.nonzero(labels != torch.arange(n, dtype=torch.int32, device="cuda")).flatten().cpu().numpy()
    assert np.array_equal(moved, touched[exp_t != touched])


@pytest.mark.parametrize("text", ["kout+rem_cas+halve+splice", "none+async+halve", "hb+rem_cas+split+halve",
                                  "ldd+sv", "bfs+sv", "none+sv", "kout+lt_prs"])
def test_static_at_max_vertex_count(huge, text):
    from paper_2008_11839_b200 import parse_spec, static_connectivity_device
    g, e, touched, exp_t, ccomps, _ = huge
    labels, st = static_connectivity_device(g, parse_spec(text))
    _check_labels(labels, touched, exp_t)
    assert st.component_count == N_MAX - len(touched) + ccomps, text


def test_forest_at_max_vertex_count(huge):
    import torch
    from paper_2008_11839_b200 import parse_spec, spanning_forest_device
    g, e, touched, exp_t, ccomps, (coff, ctgt, clab) = huge
    df, st = spanning_forest_device(g, parse_spec("bfs+async+halve"))
    keep = torch.nonzero(df.fu >= 0).flatten()
    fu, fv = df.fu[keep].cpu().numpy(), df.fv[keep].cpu().numpy()
    assert len(fu) == len(touched) - ccomps
    # the forest's endpoints are touched vertices; checked on the compacted graph
    cu, cv = np.searchsorted(touched, fu), np.searchsorted(touched, fv)
    assert np.array_equal(touched[cu], fu) and np.array_equal(touched[cv], fv)
    slots_u = np.full(len(touched), -1, np.int32)
    slots_v = np.full(len(touched), -1, np.int32)
    slots_u[: len(cu)], slots_v[: len(cv)] = cu, cv
    assert oracle.check_forest(len(touched), coff, ctgt, slots_u, slots_v, clab)["passed"]


def test_incremental_at_max_capacity(huge):
    import torch
    from paper_2008_11839_b200 import IncrementalConnectivity, parse_spec
    g, e, touched, exp_t, ccomps, _ = huge
    cap = N_MAX - 1  # the sentinel value is the capacity
    keep = (e < cap).all(axis=1)
    ek = e[keep]
    tk = np.unique(ek)
    cek = np.searchsorted(tk, ek)
    coff, ctgt = oracle.build_csr(len(tk), cek)
    clab, kcomps = oracle.components(len(tk), coff, ctgt)
    us = torch.from_numpy(ek[:, 0].astype(np.int32)).cuda()
    vs = torch.from_numpy(ek[:, 1].astype(np.int32)).cuda()
    for text in ["none+async+halve", "none+rem_cas+halve+split"]:
        inc = IncrementalConnectivity(parse_spec(text), cap)
        b = (len(ek) + 3) // 4
        for b0 in range(0, len(ek), b):
            inc.insert(us[b0:b0 + b], vs[b0:b0 + b])
        bits = inc.query(torch.tensor([0, 2], dtype=torch.int32).cuda(),
                         torch.tensor([cap - 1, cap - 3], dtype=torch.int32).cuda())
        assert bits.numpy().tolist()[0] == 1
        labels, comps = inc.labels()
        assert comps == kcomps, text
        t = torch.from_numpy(tk).cuda()
        assert torch.equal(labels[t].to(torch.int64), torch.from_numpy(tk[clab]).cuda()), text
        assert int((labels != torch.arange(cap, dtype=torch.int32, device="cuda")).sum()) == \
            int((tk[clab] != tk).sum()), text
        del inc, labels
