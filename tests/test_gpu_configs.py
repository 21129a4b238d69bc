"""Parity at every BASELINE.json config shape, scaled to sizes the oracle
finishes in seconds (configs 1 and 2 are pinned at full size elsewhere:
RMAT s16 against the reference's own statistics in test_gpu_static.py, RMAT
s24 in bench.py's untimed check).

* config 3 — LDD + SV / LT on 3-D grids (64^3 and 96^3, natural and randomly
  permuted ids).  LDD is absent from the reference (driver.py:65-69), so its
  intermediate partition is pinned the way SURVEY §8c prescribes: the final
  labels equal the oracle's, the post-sample labels REFINE the oracle
  partition (validate.py:290-297: no sampled class spans two true
  components) and are each cluster's minimum member, and cov / ic equal the
  census recomputed on the host from those labels.  The oracle-checkable
  companions (none+sv, none+lt_prs, bfs+sv) must match the C port's
  statistics, which tests/test_oracle.py pins to the reference's own.
* config 4 — incremental insert batches on a make_stream(ratio=0) stream of
  RMAT s16 (5 batches), labels against SequentialUF; a mixed
  insert / query stream (ratio 10) against the replayed query bits.
* config 5 — spanning forest with bfs+async+halve on uniform 2^20 (4n
  i.i.d. pairs): the four check_forest clauses, and sample / finish
  inspections, cov and the component count equal the C port's.
"""
import numpy as np
import pytest

import oracle
from paper_2008_11839_b200 import (Graph, IncrementalConnectivity, parse_spec, spanning_forest_device,
                                   static_connectivity, static_connectivity_device)

pytestmark = pytest.mark.gpu


def _grid_pairs(side):
    idx = np.arange(side ** 3, dtype=np.int64).reshape(side, side, side)
    parts = [np.stack([idx[:-1].ravel(), idx[1:].ravel()], 1),
             np.stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()], 1),
             np.stack([idx[:, :, :-1].ravel(), idx[:, :, 1:].ravel()], 1)]
    return np.concatenate(parts)


_GRIDS = {}


def _grid(side, permuted):
    key = (side, permuted)
    if key not in _GRIDS:
        n = side ** 3
        e = _grid_pairs(side)
        if permuted:
            perm = np.random.default_rng(side).permutation(n)
            e = perm[e]
        off, tgt = oracle.build_csr(n, e)
        ref, comps = oracle.components(n, off, tgt)
        _GRIDS[key] = (n, off, tgt, ref, comps)
    return _GRIDS[key]


def _bfs_source(n, off, seed=1, probes=64):
    pr = np.unique(np.random.default_rng(seed).integers(0, n, size=probes))
    return int(pr[np.argmax(np.diff(off)[pr])])


def _census(off, tgt, post):
    n = len(post)
    cov = np.bincount(post, minlength=n).max() / n
    src = np.repeat(np.arange(n), np.diff(off))
    ic = np.count_nonzero(post[src] != post[tgt]) / len(tgt)
    return cov, ic


@pytest.mark.parametrize("side,permuted", [(64, False), (64, True), (96, False), (96, True)])
@pytest.mark.parametrize("text", ["ldd+sv", "ldd+lt_prs", "ldd(0.5)+sv"])
def test_config3_ldd_grid(side, permuted, text):
    n, off, tgt, ref, comps = _grid(side, permuted)
    g = Graph(n, off, tgt)
    labels, st, post = static_connectivity_device(g, parse_spec(text), post_sample=True)
    lab = labels.cpu().numpy().astype(np.int64)
    post = post.cpu().numpy().astype(np.int64)
    assert np.array_equal(lab, ref), text
    assert st.component_count == comps
    # each LDD cluster is labelled by its minimum member ...
    assert (post <= np.arange(n)).all() and (post[post] == post).all()
    # ... and never spans two true components (validate.py:290-297)
    assert np.array_equal(ref[post], ref)
    cov, ic = _census(off, tgt, post)
    assert st.cov == pytest.approx(cov, rel=1e-12) and st.ic == pytest.approx(ic, rel=1e-12)
    # the finish sees exactly the vertices outside the most frequent label
    assert st.active == n - int(np.bincount(post, minlength=n).max())
    assert st.edge_inspections.get("sample", 0) > 0


@pytest.mark.parametrize("side,permuted", [(64, False), (96, True)])
@pytest.mark.parametrize("text", ["none+sv", "none+lt_prs", "bfs+sv", "kout+sv", "none+lt_crfa"])
def test_config3_companions_match_port(side, permuted, text):
    n, off, tgt, ref, comps = _grid(side, permuted)
    g = Graph(n, off, tgt)
    labels, st = static_connectivity(g, parse_spec(text))
    assert np.array_equal(labels, ref), text
    src = _bfs_source(n, off) if text.startswith("bfs") else -1
    _, pst, _ = oracle.pipeline(n, off, tgt, text, bfs_source=src)
    got = {"rounds": st.rounds, "insp_sample": st.edge_inspections.get("sample", 0),
           "insp_finish": st.edge_inspections.get("finish", 0), "components": st.component_count}
    exp = {"rounds": pst["rounds"], "insp_sample": pst["insp_sample"], "insp_finish": pst["insp_finish"],
           "components": pst["components"]}
    assert got == exp, text
    assert st.cov == pytest.approx(pst["lmax_count"] / n, rel=1e-12), text


def _rmat(scale):
    n, e = oracle.gen_rmat(scale, 8, seed=1)
    off, tgt = oracle.build_csr(n, e)
    return n, off, tgt


@pytest.mark.parametrize("text", ["none+async+halve", "none+rem_cas+halve+split", "none+sv", "none+lt_prs"])
def test_config4_stream_batches(text):
    """make_stream(ratio=0) semantics (bench.py:179-193): permuted
    undirected edges, chunked into 5 batches, capacity n."""
    import torch
    n, off, tgt = _rmat(16)
    src = np.repeat(np.arange(n), np.diff(off))
    keep = src < tgt
    ue = np.stack([src[keep], tgt[keep]], 1)
    ue = ue[np.random.default_rng(1).permutation(len(ue))]
    us = torch.from_numpy(ue[:, 0].astype(np.int32)).cuda()
    vs = torch.from_numpy(ue[:, 1].astype(np.int32)).cuda()
    inc = IncrementalConnectivity(parse_spec(text), n)
    b = (len(ue) + 4) // 5
    for b0 in range(0, len(ue), b):
        inc.insert(us[b0:b0 + b], vs[b0:b0 + b], sync=False)
    labels, comps = inc.labels()
    _, rep = oracle.incremental_replay(n, ue[:, 0], ue[:, 1], np.zeros(len(ue), np.uint8), b)
    assert labels.cpu().numpy().astype(np.int64).tolist() == rep.tolist(), text
    touched = np.zeros(n, bool)
    touched[ue.ravel()] = True
    assert comps == len(np.unique(rep[touched]))


@pytest.mark.parametrize("text", ["none+async+halve", "none+rem_cas+halve+split", "none+sv"])
def test_config4_mixed_stream_bits(text):
    """make_stream(ratio=10): every 10th op a random-pair query; the packed
    query bits of each batch equal the SequentialUF replay's."""
    import torch
    n, off, tgt = _rmat(14)
    src = np.repeat(np.arange(n), np.diff(off))
    keep = src < tgt
    ue = np.stack([src[keep], tgt[keep]], 1)
    rng = np.random.default_rng(3)
    ue = ue[rng.permutation(len(ue))]
    q = rng.integers(0, n, size=(len(ue) // 10, 2))
    us = np.concatenate([ue[:, 0], q[:, 0]]).astype(np.int32)
    vs = np.concatenate([ue[:, 1], q[:, 1]]).astype(np.int32)
    isq = np.concatenate([np.zeros(len(ue), np.uint8), np.ones(len(q), np.uint8)])
    order = rng.permutation(len(us))
    us, vs, isq = us[order], vs[order], isq[order]
    batch = 20_000
    bits_ref, lab_ref = oracle.incremental_replay(n, us, vs, isq, batch)
    inc = IncrementalConnectivity(parse_spec(text), n)
    got = []
    for b0 in range(0, len(us), batch):
        sl = slice(b0, b0 + batch)
        got.append(inc.batch(torch.from_numpy(us[sl]).cuda(), torch.from_numpy(vs[sl]).cuda(),
                             torch.from_numpy(isq[sl]).cuda()).numpy())
    got = np.concatenate(got)
    assert np.array_equal(got, bits_ref), text
    assert got[isq == 0].sum() == 0  # inserts read 0
    labels, _ = inc.labels()
    assert labels.cpu().numpy().astype(np.int64).tolist() == lab_ref.tolist()


def test_config5_bfs_forest_uniform():
    """spanning_forest(bfs+async+halve) on uniform 2^20 with 4n pairs."""
    log2n = 20
    n = 1 << log2n
    e = np.random.default_rng(1).integers(0, n, size=(4 * n, 2))
    off, tgt = oracle.build_csr(n, e)
    ref, comps = oracle.components(n, off, tgt)
    g = Graph(n, off, tgt)
    df, st = spanning_forest_device(g, parse_spec("bfs+async+halve"))
    fu, fv = df.fu.cpu().numpy(), df.fv.cpu().numpy()
    rep = oracle.check_forest(n, off, tgt, fu, fv, ref)
    assert rep["passed"], rep
    assert int((fu >= 0).sum()) == n - comps
    _, pst, _ = oracle.pipeline(n, off, tgt, "bfs+async+halve", bfs_source=_bfs_source(n, off))
    assert st.edge_inspections.get("sample", 0) == pst["insp_sample"]
    assert st.edge_inspections.get("finish", 0) == pst["insp_finish"]
    assert st.cov == pytest.approx(pst["lmax_count"] / n, rel=1e-12)
    assert st.component_count == comps


def test_incremental_malformed_endpoint_is_reported():
    import torch
    from paper_2008_11839_b200 import MalformedInputError
    inc = IncrementalConnectivity(parse_spec("none+async+halve"), 100)
    us = torch.tensor([1, 2, 150], dtype=torch.int32, device="cuda")
    vs = torch.tensor([2, 3, 4], dtype=torch.int32, device="cuda")
    with pytest.raises(MalformedInputError):
        inc.insert(us, vs)
    # the bad op was skipped; the good ones applied and the flag cleared
    bits = inc.query(torch.tensor([1], device="cuda"), torch.tensor([3], device="cuda"))
    assert bits.numpy().tolist() == [True]
    inc.insert(us, vs, sync=False)  # reported by the next synchronising call
    with pytest.raises(MalformedInputError):
        inc.labels()
    with pytest.raises(MalformedInputError):
        inc.insert(torch.tensor([-1], dtype=torch.int64), torch.tensor([0], dtype=torch.int64))


def test_live_state_view():
    """on_batch gets the live device state (driver.py:710-711), no copy."""
    import torch
    from paper_2008_11839_b200 import Insert, Query, incremental
    seen = []

    def hook(bi, state):
        t = torch.as_tensor(state, device="cuda")
        seen.append((bi, len(state), np.asarray(state).tolist(), t.data_ptr()))

    batches = [[Insert(0, 1), Query(0, 1)], [Insert(2, 3), Insert(1, 2), Query(0, 3)]]
    labels, results, _ = incremental(None, parse_spec("none+async+halve"), batches, capacity=5, on_batch=hook)
    assert [r.tolist() for r in results] == [[False, True], [False, False, True]]
    assert seen[0][2][:2] == [0, 0] and seen[0][2][2:] == [5, 5, 5]  # sentinel = capacity
    assert seen[0][3] == seen[1][3]  # the same live buffer both times
    assert labels.tolist() == [0, 0, 0, 0, 4]


def test_finish_phase_rejects_out_of_range_labels():
    from paper_2008_11839_b200 import MalformedInputError, finish_phase, path_graph
    with pytest.raises(MalformedInputError):
        finish_phase(path_graph(4), [0, 0, 9, 3], l_max=0, spec=parse_spec("none+async+halve"))


_CUT_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
from test_gpu_configs import _grid
from paper_2008_11839_b200 import Graph, parse_spec, static_connectivity_device
out = {}
for side, permuted in [(64, False), (64, True)]:
    n, off, tgt, ref, comps = _grid(side, permuted)
    g = Graph(n, off, tgt)
    for text in ["ldd+sv", "ldd+lt_prs", "ldd+lt_crfa", "ldd(0.1)+stergiou"]:
        labels, st = static_connectivity_device(g, parse_spec(text))
        out[f"{side}{permuted}{text}"] = [st.rounds, st.edge_inspections.get("finish", 0),
                                          st.component_count, int(labels.sum().item())]
print(json.dumps(out))
"""


def test_config3_ldd_cut_edges_match_gather():
    """The labels-only rounds finish after LDD takes its working COO from the
    sampler's cut edges (GC_LDD_CUT); the rounds, counted finish inspections,
    components and labels must equal the gather path's (GC_LDD_CUT=0), run in
    a second process because the knob is read once."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = []
    for cut in ("1", "0"):
        env = dict(os.environ, GC_LDD_CUT=cut)
        r = subprocess.run([sys.executable, "-c", _CUT_SCRIPT, root], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert res[0] == res[1]
