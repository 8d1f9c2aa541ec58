"""GPU parity of the Gauss-Legendre interface rule (quad_rule 1, reading R9's flag): iface_fine_lg /
iface_lg_normalise / iface_gather_{y,x}_lg vs the oracle's literal SIPG face matrices assembled at
the fine faces' LG points (pinned in tests/test_oracle_interface_lg.py)."""
import pytest

from sem_inputs import conforming_cut_config, random_state, small_config

from parity import TOL, compare, gpu_run, oracle_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _lg(rec):
    rec["interface"] = dict(rec["interface"], quad="lg")
    return rec


@pytest.mark.parametrize("name", ["cfg2s", "cfg4s"])
def test_small_config_lg_full_run(name):
    rec = _lg(small_config(name))
    n = rec["n_steps"]
    nm = oracle_run(rec, n)
    sim = gpu_run(rec, n)
    for k, v in compare(sim, nm).items():
        assert v < TOL, (name, k, v)
    sim.close()


@pytest.mark.parametrize("nel_xy,N,Nh,R", [(6, 5, 3, 2), (4, 4, 4, 1), (6, 3, 2, 3), (4, 2, 5, 2)])
def test_lg_random_state(nel_xy, N, Nh, R):
    rec = _lg(conforming_cut_config(nel_xy=nel_xy, nz_lo=2, nz_hi=2, degree=N, degree_hi=Nh, ratio=R,
                                    h=25e-6, bc_top=1))
    st = random_state(rec, seed=N + 10 * R)
    for n in (1, 15):
        nm = oracle_run(rec, n, state=st)
        sim = gpu_run(rec, n, state=st)
        for k, v in compare(sim, nm).items():
            assert v < TOL, (n, k, v)
        sim.close()
    # the rule matters: the GLL-rule run is far from the LG oracle
    g = dict(rec, interface=dict(rec["interface"], quad="gll"))
    sim = gpu_run(g, 15, state=st)
    assert max(compare(sim, nm).values()) > 1e-9
    sim.close()


def test_lg_rule_errors():
    from paper_2603_06267_b200 import SEM_F_EMULATE_SLABS, SemError, Simulation
    rec = small_config("cfg2s")
    rec["interface"] = dict(rec["interface"], quad="lg")
    with pytest.raises(SemError, match="PARTITION"):
        Simulation(rec, world=2, flags=SEM_F_EMULATE_SLABS)
    from paper_2603_06267_b200 import sem_dg_interface_build
    rec2 = small_config("cfg2s")
    rec2.pop("interface")
    rec2["pmut"] = None
    sim = Simulation(rec2)
    with pytest.raises(SemError, match="ARG"):
        sem_dg_interface_build(sim.ctx, 0, 1, 10.0, 2)
    sim.close()
