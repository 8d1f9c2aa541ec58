"""GPU parity of PMUTs on a curved (vertex-lattice) box (SURVEY 8(f) item 3 with Eqs. 11-12): the
coupling is tabulated per membrane node with the trilinear face's |J_s| and the nodes' physical
positions (not the separable affine factors) and the force enters the element-scatter residual --
vs the oracle's face-quadrature coupling table on the same seeded geometry."""
import numpy as np
import pytest

from sem_inputs import curved_pmut_config, random_state

from parity import TOL, compare, gpu_run, oracle_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_curved_pmut_tx():
    rec = curved_pmut_config()
    nm = oracle_run(rec, rec["n_steps"])
    sim = gpu_run(rec, rec["n_steps"], chunks=[100, 99, 101])
    r = compare(sim, nm)
    assert np.abs(nm.p).max() > 1.0 and np.abs(nm.q).max() > 1e-13
    for k, v in r.items():
        assert v < TOL, (k, v, r)


def test_curved_pmut_rx_random_state():
    """RX from t = 0 (open circuit, Eq. 3) excited by a rough random pressure field: the projection
    (Eq. 12) and the force (Eq. 11) both carry the tabulated weights."""
    rec = curved_pmut_config(rx=True, n_steps=60)
    st = random_state(rec, seed=21)
    for n in (1, 5, 60):
        nm = oracle_run(rec, n, state=st)
        sim = gpu_run(rec, n, state=st)
        r = compare(sim, nm)
        assert n == 1 or np.abs(nm.q).max() > 0.0      # q^1 = 0 (pdd^0 = qdd^0 = 0), driven after
        for k, v in r.items():
            assert v < TOL, (n, k, v, r)
        sim.close()
