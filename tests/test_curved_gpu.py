"""GPU parity of curved (trilinear vertex-lattice) boxes: the element-scatter path
(curved_residual / curved_update kernels, metric terms recomputed from the vertices) vs the oracle's
brute-force element matrices on the same seeded geometry and states."""
import numpy as np
import pytest

from sem_inputs import BC_ABSORBING, BC_RIGID, curved_config, random_state

from parity import TOL, compare, gpu_run, oracle_run, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("N,nel,top,seed", [(3, (4, 3, 5), BC_ABSORBING, 1), (4, (3, 3, 3), BC_RIGID, 2),
                                            (5, (2, 3, 2), BC_ABSORBING, 3), (2, (5, 4, 3), BC_RIGID, 4)])
def test_curved_random_state(N, nel, top, seed):
    rec = curved_config(nel=nel, degree=N, extent=tuple(1e-4 * n for n in nel), bc_top=top, seed=seed)
    st = random_state(rec, seed=seed)
    for n in (1, 3, 20):
        nm = oracle_run(rec, n, state=st)
        sim = gpu_run(rec, n, state=st)
        d_gpu = sim.pressure(0) - st[0][0]
        d_orc = nm.p - st[0][0]
        assert rel_l2(d_gpu, d_orc) < 1e-10, (n, rel_l2(d_gpu, d_orc))
        for k, v in compare(sim, nm).items():
            assert v < TOL, (n, k, v)
        sim.close()


def test_curved_smooth_long_run():
    rec = curved_config(nel=(3, 3, 4), degree=4, extent=(3e-4, 3e-4, 4e-4), bc_top=BC_ABSORBING, seed=5)
    from oracle.operators import System
    xyz = System(rec).node_coords()
    p0 = np.exp(-np.sum(((xyz - np.array([1.5e-4, 1.5e-4, 1.5e-4])) / 6e-5) ** 2, axis=1))
    st = [(p0, np.zeros_like(p0))]
    nm = oracle_run(rec, 300, state=st)
    sim = gpu_run(rec, 300, state=st, chunks=[100, 101, 99])
    for k, v in compare(sim, nm).items():
        assert v < TOL, (k, v)
