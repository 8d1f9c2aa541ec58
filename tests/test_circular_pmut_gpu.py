"""GPU parity of a circular membrane (r_p = 65 um) with caller-defined mode shapes
(sem_pmut_desc.shape_fn, reading R33: clamped circular plate modes standing in for the paper's FEM
eigenmodes) on a curved box: TX run, RX from a random state, and the error paths."""
import numpy as np
import pytest

from sem_inputs import circular_pmut_config, config, random_state

from parity import TOL, compare, gpu_run, oracle_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_circular_pmut_tx():
    rec = circular_pmut_config()
    nm = oracle_run(rec, rec["n_steps"])
    sim = gpu_run(rec, rec["n_steps"], chunks=[100, 99, 101])
    r = compare(sim, nm)
    assert np.abs(nm.p).max() > 1.0 and np.abs(nm.q).max() > 1e-13
    assert np.abs(nm.q[0, 2]) > 0.0       # the second axisymmetric mode is driven too
    for k, v in r.items():
        assert v < TOL, (k, v, r)


def test_circular_pmut_rx_random_state():
    rec = circular_pmut_config(rx=True, n_steps=60)
    st = random_state(rec, seed=23)
    for n in (1, 5, 60):
        nm = oracle_run(rec, n, state=st)
        sim = gpu_run(rec, n, state=st)
        r = compare(sim, nm)
        assert n == 1 or np.abs(nm.q).max() > 0.0
        if n == 60:
            assert np.abs(nm.q[0, 1]) > 0.0   # the cos(theta) mode sees the rough field
        for k, v in r.items():
            assert v < TOL, (n, k, v, r)
        sim.close()


def test_shape_fn_needs_a_curved_box():
    from paper_2603_06267_b200.sem import SemError, Simulation
    rec = config(0)
    rec["pmut"]["shape_fn"] = lambda k, m, xr, yr: 1.0
    with pytest.raises(SemError):
        Simulation(rec)


def test_cylinder_domain_circular_pmut():
    """The cylinder column of P:L1225 (one box mapped onto the disc, rigid wall, absorbing top) with the
    circular membrane transmitting, then receiving its own field (TX -> RX switch)."""
    from sem_inputs import cylinder_pmut_config
    rec = cylinder_pmut_config(n_steps=400)
    rec["pmut"]["rx"] = True
    rec["pmut"]["t_switch"] = 250 * rec["dt"]
    nm = oracle_run(rec, rec["n_steps"])
    sim = gpu_run(rec, rec["n_steps"], chunks=[150, 101, 149])
    r = compare(sim, nm)
    assert np.abs(nm.p).max() > 1.0 and np.abs(nm.q).max() > 1e-13
    for k, v in r.items():
        assert v < TOL, (k, v, r)


def test_cylinder_fine_lattice_offcentre_membrane():
    """A 16 x 16 mapped lattice moves the face nodes near the corners by more than two elements: the
    coupling table must pick a membrane's nodes by their physical positions (a small off-centre disc
    towards the mapped corner), not from the affine lattice."""
    from sem_inputs import clamped_disc_shape, cylinder_pmut_config
    rec = cylinder_pmut_config(nel=(16, 16, 2), degree=3, height=40e-6, n_steps=80, cfl=0.1)
    R, r = 90e-6, 15e-6
    modes = ((0, 1), (1, 1), (0, 2))
    rec["pmut"]["centers"] = np.array([[R + 0.55 * R, R + 0.55 * R]])
    rec["pmut"]["side"] = 2 * r
    rec["pmut"]["shape_fn"] = clamped_disc_shape(r, modes)
    nm = oracle_run(rec, rec["n_steps"])
    sim = gpu_run(rec, rec["n_steps"])
    r_ = compare(sim, nm)
    assert np.abs(nm.q).max() > 0.0 and np.abs(nm.p).max() > 0.0
    for k, v in r_.items():
        assert v < TOL, (k, v, r_)


def test_cylinder_two_boxes_circular_pmut_through_the_interface():
    """Fine inner box with the circular membrane under a coarse outer box, both on the same polygonal
    cylinder, joined by the general non-conforming interface (Algorithm 3 on curved nested faces): the
    burst crosses the interface within the run."""
    from sem_inputs import cylinder_two_box_config
    rec = cylinder_two_box_config()
    nm = oracle_run(rec, rec["n_steps"])
    sim = gpu_run(rec, rec["n_steps"], chunks=[200, 99, 201])
    assert np.abs(nm.q).max() > 1e-13 and np.abs(nm.sys.split(nm.p)[1]).max() > 1e-2
    for k, v in compare(sim, nm).items():
        assert v < TOL, (k, v)
