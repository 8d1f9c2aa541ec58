"""The paper's Section 6.2 scenario at desk scale: a PMUT transmits
a tone burst, switches to open-circuit reception at t_bar (Eq. 3) and receives the echo of
a rigid obstacle (Neumann surfaces, reading R27).  GPU (obstacle box on the element-scatter path with
the PMUT forcing in its nodal update) vs the oracle: the pressure field, the modal state and the
received-voltage time series within 1e-11; the echo is visible in the voltage."""
import numpy as np
import pytest

from sem_inputs import obstacle_pmut_config

from parity import TOL, compare, rel_l2

pytestmark = pytest.mark.gpu

CHUNK = 40


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _gpu_series(rec):
    from paper_2603_06267_b200 import Simulation
    sim = Simulation(rec)
    v = []
    for _ in range(rec["n_steps"] // CHUNK):
        sim.step(CHUNK)
        v.append(sim.modal()[2].copy())
    return sim, np.array(v)


def _oracle_series(rec):
    from threadpoolctl import threadpool_limits
    from oracle.newmark import Newmark
    from oracle.operators import System
    nm = Newmark(System(rec))
    v = []
    with threadpool_limits(1):
        for _ in range(rec["n_steps"] // CHUNK):
            nm.run(CHUNK)
            v.append(nm.v_rx().copy())
    return nm, np.array(v)


def test_pmut_obstacle_tx_rx_echo():
    rec = obstacle_pmut_config()
    sim, v_gpu = _gpu_series(rec)
    nm, v_orc = _oracle_series(rec)
    r = compare(sim, nm)
    r["v_series"] = rel_l2(v_gpu, v_orc, 1e-6)
    for k, val in r.items():
        assert val < TOL, (k, val, r)
    # physics: the same run without the obstacle (a plain structured box) receives no echo: the two
    # voltage series agree until the round trip 2 * 300 um / c = 0.4 us and part after it
    free, v_free = _gpu_series(obstacle_pmut_config(with_obstacle=False))
    t = rec["dt"] * CHUNK * np.arange(1, len(v_gpu) + 1)
    early = t < 0.3e-6
    late = t > 0.5e-6
    assert np.allclose(v_gpu[early], v_free[early], rtol=0, atol=1e-12 * np.abs(v_free).max())
    d_late = np.abs(v_gpu[late] - v_free[late]).max()
    assert d_late > 1e-3 * np.abs(v_free[late]).max(), (d_late, np.abs(v_free[late]).max())
    sim.close()
    free.close()


def test_cylinder_circular_pmut_obstacle_tx_rx_echo():
    """Section 6.2 in its own geometry: cylinder column (mapped box, rigid wall, absorbing top), circular membrane
    with caller-defined mode shapes, a rounded rigid slab 300 um above it; TX burst, then RX of the echo."""
    from sem_inputs import cylinder_obstacle_config
    rec = cylinder_obstacle_config()
    rec["n_steps"] = (rec["n_steps"] // CHUNK) * CHUNK
    sim, v_gpu = _gpu_series(rec)
    nm, v_orc = _oracle_series(rec)
    r = compare(sim, nm)
    r["v_series"] = rel_l2(v_gpu, v_orc, 1e-6)
    for k, val in r.items():
        assert val < TOL, (k, val, r)
    free_rec = cylinder_obstacle_config(with_obstacle=False)
    free_rec["n_steps"] = rec["n_steps"]
    free, v_free = _gpu_series(free_rec)
    t = rec["dt"] * CHUNK * np.arange(1, len(v_gpu) + 1)
    early, late = t < 0.3e-6, t > 0.5e-6
    assert np.allclose(v_gpu[early], v_free[early], rtol=0, atol=1e-12 * np.abs(v_free).max())
    d_late = np.abs(v_gpu[late] - v_free[late]).max()
    assert d_late > 1e-3 * np.abs(v_free[late]).max(), (d_late, np.abs(v_free[late]).max())
    sim.close()
    free.close()
