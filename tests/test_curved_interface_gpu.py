"""GPU parity of the general non-conforming interface: two curved
(vertex-lattice) boxes joined through Eq. 7's SIPG terms at the fine-face GLL nodes, with the owner
coarse element and x_hat^- of each node from Algorithm 3 on the GPU (sem_face_match) and one
table-driven kernel per step adding the face terms to both boxes' residuals -- vs the oracle's literal
face matrices (bounding-box search + Newton inverse map) on the same seeded geometry and states."""
import math

import numpy as np
import pytest

from sem_inputs import BC_ABSORBING, curved_interface_config, random_state

from parity import TOL, compare, gpu_run, oracle_run, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


CASES = {
    "non-nested 6:4, jittered, N 4/3": dict(jitter=0.15, seed=3),
    "non-nested 6:4, affine, N 3/3": dict(jitter=0.0, degree_f=3, degree_c=3),
    "nested 6:3, curved faces, N 5/2": dict(nc=(3, 3, 2), jitter=0.2, nested_jitter=True, degree_f=5, degree_c=2, seed=2),
    "two materials, jittered, absorbing top": dict(jitter=0.15, seed=6, c_f=1130.0, bc_top=BC_ABSORBING),
}


@pytest.mark.parametrize("name", list(CASES))
def test_general_interface_random_state(name):
    rec = curved_interface_config(**CASES[name])
    if "two materials" in name:
        from sem_inputs.workloads import cfl_dt
        rec["boxes"][0]["rho"] = 1140.0
        rec["dt"] = cfl_dt(rec["boxes"], 0.25)
    st = random_state(rec, seed=11)
    for n in (1, 3, 20):
        nm = oracle_run(rec, n, state=st)
        sim = gpu_run(rec, n, state=st)
        for b in range(2):   # the increment isolates the operator from the (exactly copied) initial field
            d_gpu = sim.pressure(b) - st[b][0]
            d_orc = nm.sys.split(nm.p)[b] - st[b][0]
            assert rel_l2(d_gpu, d_orc) < 1e-10, (name, n, b, rel_l2(d_gpu, d_orc))
        for k, v in compare(sim, nm).items():
            assert v < TOL, (name, n, k, v)
        sim.close()


def test_general_interface_pulse_long_run():
    """A Gaussian pulse crossing the jittered non-nested interface for 300 steps (absorbing top)."""
    rec = curved_interface_config(jitter=0.15, seed=8, bc_top=BC_ABSORBING)
    from oracle.operators import System
    xyz = System(rec).node_coords()
    c = np.array([75e-6, 75e-6, 40e-6])
    p0 = np.exp(-np.sum(((xyz - c) / 25e-6) ** 2, axis=1))
    s = System(rec)
    st = [(pb, np.zeros_like(pb)) for pb in s.split(p0)]
    nm = oracle_run(rec, 300, state=st)
    sim = gpu_run(rec, 300, state=st, chunks=[100, 101, 99])
    assert np.abs(nm.sys.split(nm.p)[1]).max() > 1e-3      # the pulse crossed the interface
    for k, v in compare(sim, nm).items():
        assert v < TOL, (k, v)


def _structured(rec):
    """The same boxes without vertex lattices: structured boxes whose lattices do not nest (6 : 4) --
    sem_dg_interface_build moves them to the element-scatter path and the general interface."""
    for b in rec["boxes"]:
        b.pop("vertices", None)
    return rec


def test_non_nested_structured_boxes_random_state():
    rec = _structured(curved_interface_config(jitter=0.0, seed=3))
    st = random_state(rec, seed=17)
    for n in (1, 4, 25):
        nm = oracle_run(rec, n, state=st)
        sim = gpu_run(rec, n, state=st)
        for k, v in compare(sim, nm).items():
            assert v < TOL, (n, k, v)
        sim.close()


def test_non_nested_structured_boxes_with_pmut():
    """A PMUT transmitting on the fine box of a non-nested (6 : 4) two-box mesh, 300 steps."""
    rec = _structured(curved_interface_config(jitter=0.0, pmut=True, bc_top=BC_ABSORBING))
    nm = oracle_run(rec, 300)
    sim = gpu_run(rec, 300)
    assert np.abs(nm.q).max() > 1e-13 and np.abs(nm.sys.split(nm.p)[1]).max() > 1e-3
    for k, v in compare(sim, nm).items():
        assert v < TOL, (k, v)
