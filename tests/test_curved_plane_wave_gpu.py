"""GPU parity of the incident plane wave (reading R13, config 4's source) on curved boxes: the load is
tabulated per top-face node from the vertex lattice (trilinear face weights, physical positions)."""
import numpy as np
import pytest

from sem_inputs import BC_ABSORBING, curved_config, cylinder_two_box_config, plane_wave_source

from parity import TOL, compare, gpu_run, oracle_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("N,az", [(4, 0.0), (3, 130.0), (5, -60.0)])
def test_curved_box_plane_wave(N, az):
    rec = curved_config(nel=(4, 3, 3), degree=N, extent=(2.0e-4, 1.5e-4, 1.5e-4), bc_top=BC_ABSORBING, seed=5,
                        n_steps=300)
    # the top layer's interior vertices also move in-plane (the face stays planar)
    b = rec["boxes"][0]
    nx, ny, nz = b["nel"]
    V = b["vertices"].reshape(nz + 1, ny + 1, nx + 1, 3)
    J = np.random.default_rng(7).uniform(-0.15, 0.15, size=(ny + 1, nx + 1, 2)) * 5.0e-5
    J[0] = J[-1] = 0.0
    J[:, 0] = J[:, -1] = 0.0
    V[-1, :, :, :2] += J
    b["vertices"] = V.reshape(-1, 3)
    rec["plane_wave"] = plane_wave_source(0, deg=20.0, azimuth_deg=az)
    rec["plane_wave"]["t0_s"] = 1.5 * rec["plane_wave"]["sigma_s"]      # the pulse enters within the run
    nm = oracle_run(rec, rec["n_steps"])
    sim = gpu_run(rec, rec["n_steps"], chunks=[100, 1, 199])
    assert np.abs(nm.p).max() > 10.0
    for k, v in compare(sim, nm).items():
        assert v < TOL, (k, v)


def test_cylinder_two_boxes_receive_a_plane_wave():
    """Config 4's scenario on the cylinder: the wave enters through the coarse box's absorbing top,
    crosses the general interface and the circular membrane receives it (RX from t = 0)."""
    rec = cylinder_two_box_config(n_steps=700)
    rec["pmut"]["rx"] = True
    rec["pmut"]["t_switch"] = 0.0
    rec["pmut"]["amp_v"] = 0.0
    rec["plane_wave"] = plane_wave_source(1, deg=20.0, azimuth_deg=30.0)
    rec["plane_wave"]["t0_s"] = 1.5 * rec["plane_wave"]["sigma_s"]
    nm = oracle_run(rec, rec["n_steps"])
    sim = gpu_run(rec, rec["n_steps"], chunks=[300, 400])
    assert np.abs(nm.sys.split(nm.p)[0]).max() > 1.0 and np.abs(nm.q).max() > 0.0
    for k, v in compare(sim, nm).items():
        assert v < TOL, (k, v)


def test_mixed_structured_and_curved_boxes_rejected():
    from paper_2603_06267_b200.sem import SemError, Simulation
    rec = cylinder_two_box_config()
    del rec["boxes"][1]["vertices"]
    rec["interface"] = None
    rec["boxes"][0]["bc"][5] = 0
    rec["boxes"][1]["bc"][4] = 0
    rec["plane_wave"] = plane_wave_source(0)
    rec["boxes"][0]["bc"][5] = BC_ABSORBING
    with pytest.raises(SemError):
        Simulation(rec)
