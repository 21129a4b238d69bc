"""Every alternative kernel path a runtime knob selects (DESIGN.md "Runtime
knobs") gives the oracle's results.  The knobs are read once per process, so
each set runs the battery below in its own interpreter:

* static connectivity on RMAT s14 (k-out, hook-based, BFS and unsampled
  specs; labels bit-exact, the C port's inspection counts) and on a
  permuted 48^3 grid (LDD + SV / LT: labels, post-sample refinement);
* the BFS spanning forest of a uniform 2^16 graph (the four clauses);
* a 12-batch incremental insert stream on RMAT s15 with every union-find
  rule the giant filter serves, plus insert_list, and a mixed insert / query
  stream (labels and query bits against SequentialUF).
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

_BATTERY = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
import oracle
from test_gpu_configs import _grid, _bfs_source
from paper_2008_11839_b200 import (Graph, IncrementalConnectivity, StaticConnectivity, parse_spec,
                                   spanning_forest_device, static_connectivity, static_connectivity_device)

n, e = oracle.gen_rmat(14, 8, seed=3)
off, tgt = oracle.build_csr(n, e)
ref, comps = oracle.components(n, off, tgt)
g = Graph(n, off, tgt)
for text in ["kout+rem_cas+halve+splice", "kout+async+compress", "hb+rem_cas+split+halve",
             "none+async+halve", "none+rem_lock+halve+splice", "bfs+sv", "kout+lt_prs", "ldd+sv"]:
    labels, st = static_connectivity(g, parse_spec(text))
    assert np.array_equal(labels, ref), text
    assert st.component_count == comps, text
    if text.startswith(("kout", "ldd")):  # the plan (captured graph, or enqueued under GC_NO_GRAPH)
        plan = StaticConnectivity(g, parse_spec(text))
        for _ in range(2):
            assert np.array_equal(plan.run()[0].cpu().numpy().astype(np.int64), ref), text
    try:
        oracle.parse(text)
    except ValueError:  # outside the C port's spec subset (LDD / HB samplers, Rem-Lock): labels only
        continue
    src = _bfs_source(n, off) if text.startswith("bfs") else -1
    _, pst, _ = oracle.pipeline(n, off, tgt, text, bfs_source=src)
    assert st.edge_inspections.get("sample", 0) == pst["insp_sample"], text
    assert st.edge_inspections.get("finish", 0) == pst["insp_finish"], text


gn, goff, gtgt, gref, gcomps = _grid(48, True)
gg = Graph(gn, goff, gtgt)
for text in ["ldd+sv", "ldd+lt_prs", "ldd(0.5)+lt_crfa", "ldd+async+halve"]:
    labels, st, post = static_connectivity_device(gg, parse_spec(text), post_sample=True)
    lab = labels.cpu().numpy().astype(np.int64)
    post = post.cpu().numpy().astype(np.int64)
    assert np.array_equal(lab, gref), text
    assert (post <= np.arange(gn)).all() and (post[post] == post).all(), text
    assert np.array_equal(gref[post], gref), text

un = 1 << 16
ue = np.random.default_rng(5).integers(0, un, size=(4 * un, 2))
uoff, utgt = oracle.build_csr(un, ue)
uref, ucomps = oracle.components(un, uoff, utgt)
df, st = spanning_forest_device(Graph(un, uoff, utgt), parse_spec("bfs+async+halve"))
fu, fv = df.fu.cpu().numpy(), df.fv.cpu().numpy()
assert oracle.check_forest(un, uoff, utgt, fu, fv, uref)["passed"]

n, e = oracle.gen_rmat(15, 8, seed=4)
off, tgt = oracle.build_csr(n, e)
src = np.repeat(np.arange(n), np.diff(off))
keep = src < tgt
ue = np.stack([src[keep], tgt[keep]], 1)
ue = ue[np.random.default_rng(6).permutation(len(ue))]
us = torch.from_numpy(ue[:, 0].astype(np.int32)).cuda()
vs = torch.from_numpy(ue[:, 1].astype(np.int32)).cuda()
b = (len(ue) + 11) // 12
_, rep = oracle.incremental_replay(n, ue[:, 0], ue[:, 1], np.zeros(len(ue), np.uint8), b)
for text in ["none+async+halve", "none+async+split", "none+rem_cas+halve+split", "none+rem_lock+naive+splice",
             "none+hooks+halve", "none+early+split"]:
    # merging-edge lists need a root-based rule (no atomic splice)
    for listed in (False, True) if not text.endswith("+splice") else (False,):
        inc = IncrementalConnectivity(parse_spec(text), n)
        merged = 0
        for b0 in range(0, len(ue), b):
            if listed:
                mu, mv = inc.insert_list(us[b0:b0 + b], vs[b0:b0 + b])
                merged += int(mu.numel())
            else:
                inc.insert(us[b0:b0 + b], vs[b0:b0 + b], sync=False)
        labels, c = inc.labels()
        assert labels.cpu().numpy().astype(np.int64).tolist() == rep.tolist(), (text, listed)
        touched = np.zeros(n, bool)
        touched[ue.ravel()] = True
        if listed:
            assert merged == int(touched.sum()) - len(np.unique(rep[touched])), text

rng = np.random.default_rng(7)
q = rng.integers(0, n, size=(len(ue) // 10, 2))
mus = np.concatenate([ue[:, 0], q[:, 0]]).astype(np.int32)
mvs = np.concatenate([ue[:, 1], q[:, 1]]).astype(np.int32)
isq = np.concatenate([np.zeros(len(ue), np.uint8), np.ones(len(q), np.uint8)])
order = rng.permutation(len(mus))
mus, mvs, isq = mus[order], mvs[order], isq[order]
bits_ref, lab_ref = oracle.incremental_replay(n, mus, mvs, isq, 30_000)
for text in ["none+async+halve", "none+rem_cas+halve+split"]:
    inc = IncrementalConnectivity(parse_spec(text), n)
    got = []
    for b0 in range(0, len(mus), 30_000):
        sl = slice(b0, b0 + 30_000)
        got.append(inc.batch(torch.from_numpy(mus[sl]).cuda(), torch.from_numpy(mvs[sl]).cuda(),
                             torch.from_numpy(isq[sl]).cuda()).numpy())
    assert np.array_equal(np.concatenate(got), bits_ref), text
print("ok")
"""

_KNOBS = [
    {},
    {"GC_LDD_PACKED": "0"},
    {"GC_LDD_PERSIST": "0", "GC_BFS_PERSIST": "0"},
    {"GC_INCR_GIANT": "0"},
    {"GC_INCR_LAZY": "0"},
    {"GC_COO_MLP": "0"},
    {"GC_COO_MLP": "8"},
    {"GC_FIN_LIST": "0", "GC_FIN_TMA": "0", "GC_MODE_COOP": "0"},
    {"GC_NO_GRAPH": "1", "GC_LDD_CUT": "0", "GC_BFS_WIDE_MIN": "1073741824"},
    {"GC_BFS_TRACE": "1", "GC_LDD_TRACE": "1", "GC_BFS_ALPHA": "4", "GC_BFS_WIDE_MIN": "256"},
    {"GC_L2_WINDOW": "1"},
    {"GC_L2_WINDOW": "1", "GC_NO_GRAPH": "1"},
]


@pytest.mark.parametrize("knobs", _KNOBS, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()) or "default")
def test_knob_paths_match_oracle(knobs):
    root = str(Path(__file__).resolve().parent.parent)
    env = dict(os.environ, **knobs)
    r = subprocess.run([sys.executable, "-c", _BATTERY, root], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, json.dumps(knobs) + "\n" + r.stderr[-3000:]
    assert r.stdout.strip().splitlines()[-1] == "ok"
