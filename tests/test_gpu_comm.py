"""The single-process multi-device C ABI (gc_comm_*, csrc/comm.cu).  One GPU
is visible, so the multi-rank orchestration runs as a loopback communicator
(every rank on cuda:0, collectives as device copies) and the NCCL transport
as a one-device communicator; both against the oracle and the single-GPU
pipeline's statistics."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

SPECS = ["kout+rem_cas+halve+splice", "none+async+halve", "hb+rem_cas+split+halve", "kout+hooks+compress",
         "bfs+async+halve", "none+rem_cas+naive+splice"]


def _graph():
    from paper_2008_11839_b200 import build_csr, gen_rmat
    return build_csr(gen_rmat(14, 8, seed=3, device=True))


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_comm_static_labels_and_stats(devices):
    from paper_2008_11839_b200 import parse_spec, static_connectivity_device
    from paper_2008_11839_b200.distributed import DeviceComm
    g = _graph()
    orc, comps = oracle.components(g.n, g.offsets, g.targets)
    comm = DeviceComm(devices)
    assert comm.size == len(devices) and comm.loopback == (len(devices) > 1)
    for text in SPECS:
        spec = parse_spec(text)
        labels, st = comm.static_connectivity(g, spec)
        _, ref = static_connectivity_device(g, spec)
        for r, lab in enumerate(labels):
            assert np.array_equal(lab.cpu().numpy().astype(np.int64), orc), (text, r)
        assert st.insp_sample == ref.edge_inspections.get("sample", 0), text
        assert st.insp_finish == ref.edge_inspections.get("finish", 0), text
        assert st.lmax_count / g.n == ref.cov and st.n_active == ref.active, text
    comm.close()


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0, 0]])
def test_comm_spanning_forest(devices):
    from paper_2008_11839_b200 import parse_spec
    from paper_2008_11839_b200.distributed import DeviceComm
    g = _graph()
    orc, comps = oracle.components(g.n, g.offsets, g.targets)
    comm = DeviceComm(devices)
    for text in ["bfs+async+halve", "kout+async+halve", "none+rem_cas+halve+split"]:
        labels, forests, _ = comm.spanning_forest(g, parse_spec(text))
        for r, ((fu, fv), lab) in enumerate(zip(forests, labels)):
            assert np.array_equal(lab.cpu().numpy().astype(np.int64), orc), (text, r)
            assert fu.numel() == g.n - comps, (text, r)
            su = np.full(g.n, -1, np.int32); sv = np.full(g.n, -1, np.int32)
            su[:fu.numel()] = fu.cpu().numpy(); sv[:fv.numel()] = fv.cpu().numpy()
            assert oracle.check_forest(g.n, g.offsets, g.targets, su, sv, orc)["passed"], (text, r)
    comm.close()


def test_comm_rejects_bad_configs():
    from paper_2008_11839_b200 import ConfigError, parse_spec
    from paper_2008_11839_b200.distributed import DeviceComm
    comm = DeviceComm([0, 0])
    with pytest.raises(ConfigError):
        comm.static_connectivity(_graph(), parse_spec("none+sv"))
    with pytest.raises(ConfigError):
        comm.spanning_forest(_graph(), parse_spec("kout+rem_cas+halve+splice"))
    comm.close()
