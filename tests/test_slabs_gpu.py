"""y-slab decomposition (the multi-GPU path) verified on one GPU: SEM_F_EMULATE_SLABS keeps every
slab of a world-size-W decomposition in one context and replaces the per-step NCCL exchange by a
device copy, so the cut-plane partial rows, the coarse SIPG partial sums, the fix-up kernel, the
membrane-preserving PMUT assignment and the slab readouts all run exactly as on W GPUs.
"""
import numpy as np
import pytest

from sem_inputs import cavity_config, config, conforming_cut_config, random_state, small_config

from crops import crop_record
from parity import TOL, compare, oracle_run, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _sim(rec, world, state=None, steps=0):
    from paper_2603_06267_b200 import SEM_F_EMULATE_SLABS, Simulation
    sim = Simulation(rec, world=world, flags=SEM_F_EMULATE_SLABS)
    if state is not None:
        for b, (p, v) in enumerate(state):
            sim.write_state(b, p, v)
    if steps:
        sim.step(steps)
    return sim


@pytest.mark.parametrize("name,world", [("cfg1s", 2), ("cfg2s", 2), ("cfg3s", 2), ("cfg4s", 2)])
def test_small_configs_slabs(name, world):
    rec = small_config(name)
    nm = oracle_run(rec, rec["n_steps"])
    sim = _sim(rec, world, steps=rec["n_steps"])
    for k, v in compare(sim, nm).items():
        assert v < TOL, (name, world, k, v)


@pytest.mark.parametrize("world", [2, 3, 4, 6])
def test_random_state_cavity_slabs(world):
    rec = cavity_config(nel=(3, 12, 2), degree=5, extent=(6e-5, 12 * 2e-5, 4e-5))
    rec["boxes"][0]["bc"] = [0, 1, 1, 1, 1, 0]
    st = random_state(rec, seed=world)
    nm = oracle_run(rec, 25, state=st)
    sim = _sim(rec, world, state=st, steps=25)
    for k, v in compare(sim, nm).items():
        assert v < TOL, (world, k, v)


@pytest.mark.parametrize("world", [2, 3])
def test_random_state_interface_slabs(world):
    rec = conforming_cut_config(nel_xy=12, nz_lo=2, nz_hi=2, degree=5, degree_hi=3, ratio=2, h=25e-6, bc_top=1)
    st = random_state(rec, seed=7 + world)
    nm = oracle_run(rec, 20, state=st)
    sim = _sim(rec, world, state=st, steps=20)
    for k, v in compare(sim, nm).items():
        assert v < TOL, (world, k, v)


def test_partition_errors():
    from paper_2603_06267_b200 import SemError
    from paper_2603_06267_b200 import SEM_F_EMULATE_SLABS, Simulation
    with pytest.raises(SemError, match="PARTITION"):   # an explicit equal plan: y = 300 um crosses the membrane
        Simulation(config(0), world=2, flags=SEM_F_EMULATE_SLABS, slab_y0=[0, 2, 4])
    with pytest.raises(SemError, match="PARTITION"):   # a cut that is not a coarse element boundary
        Simulation(small_config("cfg2s"), world=2, flags=SEM_F_EMULATE_SLABS, slab_y0=[0, 5, 12])
    with pytest.raises(SemError, match="PARTITION"):
        _sim(small_config("cfg2s"), 5)         # 12 elements are not divisible by 5
    with pytest.raises(SemError, match="PARTITION"):
        _sim(small_config("cfg2s"), 3)         # cuts at y = 100, 200 um cross membranes


def test_fullsize_cfg3_eight_slabs_crops():
    """Config 3 at full size split into 8 y-slabs (cuts every 48 fine elements = 1.2 mm, in membrane
    gaps), sampled against the oracle on crops that straddle a cut."""
    from oracle.newmark import Newmark
    from oracle.operators import System
    from sem_inputs.counter_rng import cb_uniform
    rec = config(3)
    dt = rec["dt"]
    ps, vs, seed = 1.0, 1e-3 / dt, 99
    sim = _sim(rec, 8)
    for b in range(2):
        sim.fill_random_state(b, seed, ps, vs)
    rng = np.random.default_rng(3)
    crops = []
    for win in [(0, 18, 36, 54), (186, 204, 180, 198)]:      # straddle the y cuts at 48 and 192
        crop, info = crop_record(rec, win)
        picks = []
        for b, bx in enumerate(crop["boxes"]):
            idx = np.nonzero(info["valid"][b])[0]
            picks.append(np.unique(rng.choice(idx, size=3000, replace=False)))
        crops.append((crop, info, picks))
    sim.step(1)
    p1 = [[sim.pressure_at(b, info["maps"][b][pk]) for b, pk in enumerate(picks)] for _, info, picks in crops]
    sim.step(1)
    p2 = [[sim.pressure_at(b, info["maps"][b][pk]) for b, pk in enumerate(picks)] for _, info, picks in crops]
    q2, qd2, _ = sim.modal()
    sim.close()
    for ci, (crop, info, picks) in enumerate(crops):
        s = System(crop)
        nm = Newmark(s)
        nm.set_state(np.concatenate([ps * cb_uniform(seed, b, 0, info["maps"][b]) for b in range(2)]),
                     np.concatenate([vs * cb_uniform(seed, b, 1, info["maps"][b]) for b in range(2)]))
        nm.step()
        o1 = s.split(nm.p)
        nm.step()
        o2 = s.split(nm.p)
        for b, pk in enumerate(picks):
            assert rel_l2(p2[ci][b] - p1[ci][b], o2[b][pk] - o1[b][pk]) < TOL, (ci, b)
        ok = np.array(info["pmut_valid"], bool)
        k = info["pmut_full_index"]
        assert rel_l2(q2[k[ok]], nm.q[ok]) < TOL
        assert rel_l2(qd2[k[ok]], nm.qd[ok]) < TOL


@pytest.mark.parametrize("world", [4, 8])
def test_config1_uneven_membrane_preserving_slabs(world):
    """Config 1 at 4 / 8 slabs: equal cuts would split membranes, so sem_slab_plan picks uneven cuts in
    the membrane gaps; the emulated decomposition at full size vs the oracle."""
    from paper_2603_06267_b200.sem import sem_slab_plan
    rec = config(1)
    plan = sem_slab_plan(rec["boxes"], world, rec["pmut"])
    assert len(set(np.diff(plan))) > 1                    # really uneven
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        nm = oracle_run(rec, 200)
    sim = _sim(rec, world, steps=200)
    for k, v in compare(sim, nm).items():
        assert v < TOL, (world, k, v)
    sim.close()


def test_config0_two_uneven_slabs():
    rec = config(0)
    nm = oracle_run(rec, rec["n_steps"])
    sim = _sim(rec, 2, steps=rec["n_steps"])
    for k, v in compare(sim, nm).items():
        assert v < TOL, (k, v)
