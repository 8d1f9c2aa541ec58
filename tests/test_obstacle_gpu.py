"""GPU parity of rigid obstacles (`sem_box_set_obstacle`): solid elements skipped
by the element-scatter path (residual kernel, assembled mass / ABC diagonal), obstacle-interior nodes
held at 0, vs the oracle's System without those elements (pinned in tests/test_oracle_obstacle.py)."""
import numpy as np
import pytest

from sem_inputs import BC_ABSORBING, BC_RIGID, obstacle_config, random_state

from parity import TOL, compare, gpu_run, oracle_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("N,nel,lo,hi,amp,seed", [
    (3, (6, 6, 4), (2, 2, 1), (4, 4, 3), 0.0, None),     # block in the middle, affine box
    (5, (4, 3, 3), (1, 0, 1), (3, 2, 2), 0.0, None),     # obstacle touching the -y box face
    (2, (7, 5, 4), (3, 1, 0), (5, 4, 2), 0.12, 3),       # curved box, obstacle on the floor
    (4, (3, 3, 4), (0, 0, 3), (3, 3, 4), 0.1, None),     # solid top layer under the absorbing face
])
def test_obstacle_random_state(N, nel, lo, hi, amp, seed):
    rec = obstacle_config(nel=nel, degree=N, solid_lo=lo, solid_hi=hi, curved_amp=amp, seed=seed)
    st = random_state(rec, seed=11)
    for n in (1, 4, 25):
        nm = oracle_run(rec, n, state=st)
        sim = gpu_run(rec, n, state=st)
        for k, v in compare(sim, nm).items():
            assert v < TOL, (n, k, v)
        p = sim.pressure(0)
        assert np.all(p[~nm.sys.active] == 0.0)
        sim.close()


def test_obstacle_wall_decouples_on_gpu():
    N, nel = 3, (7, 2, 2)
    rec = obstacle_config(nel=nel, degree=N, solid_lo=(3, 0, 0), solid_hi=(4, 2, 2), bc=[BC_RIGID] * 6)
    nn = tuple(N * e + 1 for e in nel)
    gx = np.tile(np.arange(nn[0]), nn[1] * nn[2])
    rng = np.random.default_rng(2)
    p0 = np.where(gx <= 3 * N, rng.standard_normal(gx.size), 0.0)
    v0 = np.where(gx <= 3 * N, 1e7 * rng.standard_normal(gx.size), 0.0)
    sim = gpu_run(rec, 80, state=[(p0, v0)])
    p = sim.pressure(0)
    assert np.all(p[gx >= 4 * N] == 0.0)
    assert np.max(np.abs(p[gx <= 3 * N])) > 0.1
    sim.close()


def test_obstacle_long_run_absorbing():
    rec = obstacle_config(nel=(5, 5, 4), degree=4, solid_lo=(2, 2, 1), solid_hi=(3, 3, 3),
                          bc=[BC_RIGID] * 4 + [BC_RIGID, BC_ABSORBING])
    from oracle.operators import System
    xyz = System(rec).node_coords()
    c = np.array([0.25e-4, 0.25e-4, 0.5e-4])
    p0 = np.exp(-np.sum(((xyz - c) / 2.5e-5) ** 2, axis=1))
    st = [(p0, np.zeros_like(p0))]
    nm = oracle_run(rec, 250, state=st)
    sim = gpu_run(rec, 250, state=st, chunks=[100, 150])
    for k, v in compare(sim, nm).items():
        assert v < TOL, (k, v)
    sim.close()


def test_obstacle_errors():
    from paper_2603_06267_b200 import SemError, Simulation, sem_box_set_obstacle
    rec = obstacle_config(nel=(3, 3, 3), degree=3, solid_lo=(1, 1, 1), solid_hi=(2, 2, 2))
    sim = Simulation(rec)
    with pytest.raises(SemError, match="STATE|already"):
        sem_box_set_obstacle(sim.ctx, 0, np.zeros(27, dtype=bool))          # second obstacle
    sim.close()
    plain = obstacle_config(nel=(3, 3, 3), degree=3, solid_lo=(0, 0, 0), solid_hi=(0, 0, 0))
    plain["boxes"][0].pop("solid")
    sim = Simulation(plain)
    with pytest.raises(SemError):
        sem_box_set_obstacle(sim.ctx, 0, np.zeros(26, dtype=bool))          # wrong size
    with pytest.raises(SemError):
        sem_box_set_obstacle(sim.ctx, 0, np.ones(27, dtype=bool))           # no fluid left
    sim.close()
    from sem_inputs import config
    rec0 = config(0)
    sim = Simulation(rec0)                                                   # box 0 carries the PMUTs
    with pytest.raises(SemError, match="STATE|PMUT"):
        sem_box_set_obstacle(sim.ctx, 0, np.zeros(64, dtype=bool))
    sim.close()
