"""Full-size sampled parity: BASELINE configs 1-4 at their real sizes, in the launch configuration
bench.py times, against the oracle on lateral crops (tests/crops.py).

The state is a seeded random field filled on the device by `sem_fill_random_state` (counter-based
generator, sem_inputs/counter_rng.py), so no 4 GB host arrays are needed; the oracle reproduces the
same field on its crop.  Two steps are compared: p^1 = p^0 + dt p'^0 (exact), p^2 whose increment
p^2 - p^1 = dt p'^0 + dt^2 p''^1 exercises every operator term (volume rows, SIPG, ABC, PMUT force,
plane wave) at the sampled nodes; the modal state q^2, q'^2 of every PMUT inside a crop is compared
as well.
"""
import numpy as np
import pytest

from sem_inputs import config
from sem_inputs.counter_rng import cb_uniform

from crops import crop_record
from parity import TOL, rel_l2

pytestmark = pytest.mark.gpu

SEED = 20261019


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _windows(rec):
    b0 = rec["boxes"][0]
    nel = b0["nel"][0]
    if len(rec["boxes"]) == 2:          # configs 2-4: 6 fine elements per PMUT pitch cell
        w = 18
        mid = (nel // 2 // 6 - 1) * 6
        return [(0, w, 0, w), (nel - w, nel, nel - w, nel), (mid, mid + w, mid, mid + w)]
    return [(0, 16, 0, 16), (8, 24, 8, 24)]   # config 1: cells of 4 elements starting at element 4


def _sample(valid, n_random, rng, planes=None, nxy=None):
    idx = np.nonzero(valid)[0]
    pick = rng.choice(idx, size=min(n_random, len(idx)), replace=False)
    if planes is not None:
        for z in planes:
            sl = np.arange(z * nxy, (z + 1) * nxy)
            pick = np.concatenate([pick, sl[valid[sl]]])
    return np.unique(pick)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_fullsize_two_steps_on_crops(cfg):
    from oracle.newmark import Newmark
    from oracle.operators import System
    from paper_2603_06267_b200 import Simulation

    rec = config(cfg)
    dt = rec["dt"]
    ps, vs = 1.0, 1e-3 / dt
    sim = Simulation(rec)
    for b in range(len(rec["boxes"])):
        sim.fill_random_state(b, SEED, ps, vs)
    rng = np.random.default_rng(cfg)
    crops = []
    for win in _windows(rec):
        crop, info = crop_record(rec, win)
        picks = []
        for b, bx in enumerate(crop["boxes"]):
            N = bx["degree"]
            nx, ny, nz = (N * n + 1 for n in bx["nel"])
            planes = [0, N, nz - 1 - N, nz - 1] if len(rec["boxes"]) == 2 else [0, nz - 1]
            picks.append(_sample(info["valid"][b], 1500, rng, planes, nx * ny))
        crops.append((win, crop, info, picks))
    # device: fill check, then p^1 and p^2 at the sampled nodes, modal state after 2 steps
    gpu = []
    for win, crop, info, picks in crops:
        for b, pick in enumerate(picks):
            ids = info["maps"][b][pick]
            p0 = sim.pressure_at(b, ids)
            assert np.array_equal(p0, ps * cb_uniform(SEED, b, 0, ids)), "counter RNG differs"
    sim.step(1)
    p1 = [[sim.pressure_at(b, info["maps"][b][pick]) for b, pick in enumerate(picks)]
          for _, _, info, picks in crops]
    sim.step(1)
    p2 = [[sim.pressure_at(b, info["maps"][b][pick]) for b, pick in enumerate(picks)]
          for _, _, info, picks in crops]
    q2 = qd2 = None
    if rec.get("pmut") is not None:
        q2, qd2, _ = sim.modal()
    sim.close()

    for ci, (win, crop, info, picks) in enumerate(crops):
        s = System(crop)
        nm = Newmark(s)
        p0s, v0s = [], []
        for b in range(len(crop["boxes"])):
            ids = info["maps"][b]
            p0s.append(ps * cb_uniform(SEED, b, 0, ids))
            v0s.append(vs * cb_uniform(SEED, b, 1, ids))
        nm.set_state(np.concatenate(p0s), np.concatenate(v0s))
        nm.step()
        o1 = s.split(nm.p)
        nm.step()
        o2 = s.split(nm.p)
        for b, pick in enumerate(picks):
            r1 = o1[b][pick]
            assert rel_l2(p1[ci][b], r1) < 1e-15, (cfg, win, b)
            inc_g = p2[ci][b] - p1[ci][b]
            inc_o = o2[b][pick] - r1
            err = rel_l2(inc_g, inc_o)
            assert err < TOL, (cfg, win, b, err)
            assert rel_l2(p2[ci][b], o2[b][pick]) < TOL
        if q2 is not None and len(info["pmut_full_index"]):
            full_k = info["pmut_full_index"]
            ok = np.array(info["pmut_valid"], bool)
            if ok.any():
                assert rel_l2(q2[full_k[ok]], nm.q[ok]) < TOL, (cfg, win)
                assert rel_l2(qd2[full_k[ok]], nm.qd[ok]) < TOL, (cfg, win)
