"""GPU parity: libsem (CUDA, sm_100a) vs the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): relative L2 <= 1e-11 on every box's pressure field and on the modal
amplitudes after the configured number of steps (reading R21 floor for near-zero modal amplitudes).
"""
import numpy as np
import pytest

from sem_inputs import cavity_config, config, conforming_cut_config, random_state, small_config

from parity import TOL, compare, gpu_run, oracle_run, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_cfg0_full():
    rec = config(0)
    nm = oracle_run(rec, rec["n_steps"])
    sim = gpu_run(rec, rec["n_steps"])
    r = compare(sim, nm)
    assert np.abs(nm.p).max() > 1.0 and np.abs(nm.q).max() > 1e-12     # non-trivial run
    for k, v in r.items():
        assert v < TOL, (k, v, r)


@pytest.mark.parametrize("name", ["cfg1s", "cfg2s", "cfg3s", "cfg4s"])
def test_small_configs_full_run(name):
    rec = small_config(name)
    nm = oracle_run(rec, rec["n_steps"])
    sim = gpu_run(rec, rec["n_steps"])
    r = compare(sim, nm)
    for k, v in r.items():
        assert v < TOL, (k, v, r)


@pytest.mark.parametrize("name", ["cfg0", "cfg1s", "cfg2s", "cfg4s"])
def test_random_state_operator_parity(name):
    """Seeded random p^0, p'^0 (rough fields exercise every stencil entry and the penalty)."""
    rec = config(0) if name == "cfg0" else small_config(name)
    st = random_state(rec, seed=7)
    for n in (1, 2, 5):
        nm = oracle_run(rec, n, state=st)
        sim = gpu_run(rec, n, state=st)
        r = compare(sim, nm)
        # the increment p^n - p^0 isolates the operator from the (exactly copied) initial field
        for b in range(len(sim.ndof)):
            d_gpu = sim.pressure(b) - st[b][0]
            d_orc = nm.sys.split(nm.p)[b] - st[b][0]
            assert rel_l2(d_gpu, d_orc) < 1e-12 * 100, (name, n, b)
        for k, v in r.items():
            assert v < TOL, (name, n, k, v)
        sim.close()


def test_tx_then_rx_switch():
    """TX burst until t_bar, open-circuit RX feedback after it (Eq. 3):
    cfg 0 with t_bar mid-run and a capacitance small enough for the feedback to matter."""
    rec = config(0)
    pm = rec["pmut"]
    pm["rx"] = True
    pm["amp_v"] = 5.0
    pm["t_switch"] = 250.5 * rec["dt"]
    w1 = 2 * np.pi * pm["freq_hz"][0, 0]
    pm["capacitance"] = pm["eta"][0] ** 2 / (pm["modal_mass"][0] * 0.2 * w1 * w1)
    nm = oracle_run(rec, 400)
    sim = gpu_run(rec, 400)
    r = compare(sim, nm)
    assert np.abs(nm.q).max() > 1e-12
    for k, v in r.items():
        assert v < TOL, (k, v, r)


def test_literal_coupling_flag():
    rec = config(0, coupling="literal")
    nm = oracle_run(rec, 300)
    sim = gpu_run(rec, 300)
    for k, v in compare(sim, nm).items():
        assert v < TOL, (k, v)


@pytest.mark.parametrize("N,nel", [(1, (3, 5, 2)), (2, (2, 3, 4)), (3, (11, 3, 2)), (6, (2, 1, 3)),
                                   (7, (1, 2, 1)), (8, (2, 2, 1)),
                                   # several x tiles (TXE = 2 x 30 nodes for N = 2, 3, 5; 56 for N = 4; 48
                                   # for N = 8) with a ragged last tile, or the TXE + 1 last tile
                                   (3, (45, 3, 2)), (2, (60, 2, 2)), (5, (25, 2, 1)), (4, (31, 2, 2)),
                                   (8, (13, 1, 1))])
def test_degrees_and_ragged_tiles(N, nel):
    """Every compiled degree; NX not a multiple of 32, NY not of 8, single-element directions, several x
    tiles with ragged or one-node-wider last tiles."""
    rec = cavity_config(nel=nel, degree=N, extent=(1.1e-4 * nel[0], 0.9e-4 * nel[1], 1.3e-4 * nel[2]))
    rec["boxes"][0]["bc"] = [1, 0, 0, 1, 0, 1]           # mixed absorbing / rigid faces
    st = random_state(rec, seed=N)
    nm = oracle_run(rec, 40, state=st)
    sim = gpu_run(rec, 40, state=st)
    for k, v in compare(sim, nm).items():
        assert v < TOL, (k, v)


@pytest.mark.parametrize("ratio,nh", [(1, 5), (2, 3), (3, 2)])
def test_interface_ratios(ratio, nh):
    rec = conforming_cut_config(nel_xy=6, nz_lo=2, nz_hi=3, degree=5, degree_hi=nh, ratio=ratio, h=25e-6,
                                bc_top=1)
    st = random_state(rec, seed=11)
    nm = oracle_run(rec, 30, state=st)
    sim = gpu_run(rec, 30, state=st)
    for k, v in compare(sim, nm).items():
        assert v < TOL, (k, v)


def test_graph_and_direct_launch_bitwise_equal():
    from paper_2603_06267_b200 import SEM_F_NO_GRAPH
    rec = small_config("cfg2s")
    a = gpu_run(rec, 37, chunks=[1, 2, 5, 29])
    b = gpu_run(rec, 37, flags=SEM_F_NO_GRAPH)
    c = gpu_run(rec, 37)
    for box in range(2):
        assert np.array_equal(a.pressure(box), b.pressure(box))
        assert np.array_equal(a.pressure(box), c.pressure(box))
    assert np.array_equal(a.modal()[0], b.modal()[0])


def test_error_paths():
    from paper_2603_06267_b200 import SemError, Simulation
    rec = config(0)
    bad = config(0)
    bad["boxes"][0]["degree"] = 9
    with pytest.raises(SemError):
        Simulation(bad)
    ov = config(1)
    ov["pmut"]["centers"][1] = ov["pmut"]["centers"][0] + np.array([50e-6, 0.0])
    with pytest.raises(SemError, match="overlap"):
        Simulation(ov)
    it = small_config("cfg2s")
    ex = it["boxes"][1]["extent"]
    it["boxes"][1]["extent"] = (ex[0] * 2 / 3, ex[1], ex[2])   # interface faces do not coincide
    with pytest.raises(SemError, match="UNMATCHED"):
        Simulation(it)
    sim = Simulation(rec)
    with pytest.raises(SemError):
        sim.write_state(0, np.zeros(5), np.zeros(5))


@pytest.mark.parametrize("ratio,nh", [(2, 3), (1, 5)])
def test_two_material_interface_random_state(ratio, nh):
    """c+ != c- across Gamma_I (the paper's lens material rho = 1140, c = 1130 under water):
    exercises the per-side c^2 of the average flux and the coarse side's c-^2 / c+^2 factor, and the
    harmonic-mean penalty, from a rough random state."""
    from sem_inputs.workloads import cfl_dt
    rec = conforming_cut_config(nel_xy=6, nz_lo=2, nz_hi=3, degree=5, degree_hi=nh, ratio=ratio, h=25e-6,
                                bc_top=1)
    rec["boxes"][0]["c"], rec["boxes"][0]["rho"] = 1130.0, 1140.0
    rec["dt"] = cfl_dt(rec["boxes"])
    st = random_state(rec, seed=13)
    for n in (1, 3, 30):
        nm = oracle_run(rec, n, state=st)
        sim = gpu_run(rec, n, state=st)
        for k, v in compare(sim, nm).items():
            assert v < TOL, (n, k, v)
        sim.close()


def test_state_rewrite_mid_run():
    """The volume kernel hands the next step's interface its face traces; a state written between steps
    (sem_write_state) invalidates them, and the next step reads the planes again."""
    rec = conforming_cut_config(nel_xy=6, nz_lo=2, nz_hi=3, degree=5, degree_hi=3, ratio=2, h=25e-6, bc_top=1)
    from paper_2603_06267_b200 import Simulation
    sim = Simulation(rec)
    for b, (p, v) in enumerate(random_state(rec, seed=22)):
        sim.write_state(b, p, v)
    sim.step(17)
    st = random_state(rec, seed=23)
    for b, (p, v) in enumerate(st):
        sim.write_state(b, p, v)
    sim.step(11)
    nm = oracle_run(rec, 11, state=st)
    for k, v in compare(sim, nm).items():
        assert v < TOL, (k, v)
    sim.close()
