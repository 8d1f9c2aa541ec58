"""Pins for curved (trilinear, non-affine) boxes in the oracle:
mass = volume, K 1 = 0, <x, K x> = c^2 Vol, the linear patch test at interior nodes (exact: the
cofactor form |J| J^-T of a trilinear map is polynomial), symmetry / PSD and exact discrete energy."""
import numpy as np
import pytest

from oracle.newmark import Newmark
from oracle.operators import System
from sem_inputs import curved_config


@pytest.mark.parametrize("N", [3, 4, 5])
def test_curved_operator_invariants(N):
    rec = curved_config(nel=(3, 2, 3), degree=N, extent=(3e-4, 2e-4, 3e-4), seed=4)
    s = System(rec)
    vol = np.prod(rec["boxes"][0]["extent"])
    c2 = rec["boxes"][0]["c"] ** 2
    assert abs(s.M.sum() - vol) < 1e-13 * vol
    K1 = s.apply_K(np.ones(s.ndof))
    scale = c2 * vol / 1e-4 ** 2
    assert np.abs(K1).max() < 1e-12 * scale
    xyz = s.node_coords()
    for d in range(3):
        p = xyz[:, d]
        assert abs(p @ s.apply_K(p) - c2 * vol) < 1e-12 * c2 * vol
    # linear patch test: interior rows of K (a.x) vanish
    a = np.array([0.3, -1.2, 0.7])
    p = xyz @ a
    r = s.apply_K(p)
    L = np.asarray(rec["boxes"][0]["extent"])
    interior = np.all((xyz > 1e-9 * L) & (xyz < L * (1 - 1e-9)), axis=1)
    assert np.abs(r[interior]).max() < 1e-11 * np.abs(r).max()
    rng = np.random.default_rng(1)
    u, v = rng.standard_normal((2, s.ndof))
    Ku, Kv = s.apply_K(u), s.apply_K(v)
    assert abs(u @ Kv - v @ Ku) < 1e-12 * abs(u @ Ku)
    assert u @ Ku > 0


def test_curved_energy_conserved():
    rec = curved_config(nel=(2, 3, 2), degree=4, extent=(2e-4, 3e-4, 2e-4), seed=7)
    s = System(rec)
    nm = Newmark(s)
    nm.set_state(np.random.default_rng(2).standard_normal(s.ndof), np.zeros(s.ndof))
    ps = [nm.p.copy()]
    for _ in range(300):
        nm.step()
        ps.append(nm.p.copy())
    dt = rec["dt"]
    E = []
    for n in range(1, 300):
        v = (ps[n + 1] - ps[n]) / dt
        E.append(0.5 * v @ (s.M * v) + 0.5 * ps[n + 1] @ s.apply_K(ps[n]))
    E = np.array(E)
    assert E.min() > 0 and np.max(np.abs(E - E[0])) < 1e-11 * E[0]
