"""Pins for the oracle's interface on general non-conforming meshes: curved
(trilinear) interface faces and lattices that do not nest.  The face matrices are the literal SIPG form
of Eq. 7 at the fine-face GLL nodes (reading R9) with x_hat^- from the Newton inverse map
(P:L934-938).

With nested faces (each coarse face tiled exactly by fine faces, also when curved) the quadrature is
exact for the consistency terms of linear fields, so the linear patch test holds and a DG cut converges
spectrally to the conforming mesh.  With non-nested lattices (6 : 4) a fine face straddles coarse
element edges, the coarse basis is only piecewise polynomial on it and the fine-face rule is inexact
(the method's own quadrature choice): the patch test fails there and accuracy is algebraic; the
pins are then the invariants (constants in the kernel, symmetry, positive jump energy, exact discrete
energy) and convergence towards the conforming mesh."""
import math

import numpy as np
import pytest

from oracle.newmark import Newmark
from oracle.operators import System
from sem_inputs import curved_interface_config

C2 = 1500.0 ** 2


def _inner(xyz, L, H):
    """Nodes off the outer box boundary (both sides of the interface plane included)."""
    x, y, z = xyz.T
    e = 1e-9 * L
    return (x > e) & (x < L - e) & (y > e) & (y < L - e) & (z > e) & (z < H - e)


def _extent(rec):
    return rec["boxes"][0]["extent"][0], rec["boxes"][0]["extent"][2] + rec["boxes"][1]["extent"][2]


@pytest.mark.parametrize("degs,jit", [((4, 3), 0.0), ((3, 3), 0.2), ((5, 2), 0.2)])
def test_nested_curved_linear_patch(degs, jit):
    """6 : 3 lattices, interface faces curved but nested: M^-1 K p = 0 off the outer boundary for linear
    p (zero jump, the consistency term cancels the volume flux) -- at the interface nodes too."""
    rec = curved_interface_config(nc=(3, 3, 2), degree_f=degs[0], degree_c=degs[1], jitter=jit,
                                  nested_jitter=True, seed=2)
    s = System(rec)
    xyz = s.node_coords()
    L, H = _extent(rec)
    inner = _inner(xyz, L, H)
    z0 = rec["boxes"][0]["extent"][2]
    assert np.sum(inner & (np.abs(xyz[:, 2] - z0) < 1e-12)) > 20
    x, y, z = xyz.T
    p = 1.0 + 2e3 * x - 3e3 * y + 4e3 * z
    a = s.apply_K(p) / s.M
    assert np.max(np.abs(a[inner])) < 1e-9 * C2 * 4e3 / 25e-6, np.max(np.abs(a[inner]))


def _mode_run(nc, N, jit, dt=None, steps=None):
    rec = curved_interface_config(nc=(nc, nc, 2), degree_f=N, degree_c=N, jitter=jit, nested_jitter=jit > 0,
                                  seed=4)
    if dt:
        rec["dt"] = dt
    s = System(rec)
    xyz = s.node_coords()
    L, H = _extent(rec)
    p0 = np.cos(math.pi * xyz[:, 0] / L) * np.cos(math.pi * xyz[:, 2] / H)
    nm = Newmark(s)
    nm.set_state(p0, np.zeros(s.ndof))
    om = 1500 * math.pi * math.hypot(1 / L, 1 / H)
    n = steps or int(round(0.5 * math.pi / om / rec["dt"]))
    nm.run(n)
    return rec["dt"], n, nm.p[:s.offsets[1]]       # the fine box's lattice is the same in both runs


@pytest.mark.parametrize("jit", [0.0, 0.2])
def test_nested_cut_converges_spectrally(jit):
    """Cavity mode through a 2 : 1 (nested, optionally curved) interface vs the same fine mesh cut
    conformingly (6 : 6): the difference after a quarter period shrinks spectrally in N (affine) and
    fast (curved: the GLL rule on trilinear elements is not exact)."""
    d = []
    for N in (2, 4):
        dt, n, a = _mode_run(3, N, jit)
        _, _, b = _mode_run(6, N, jit, dt, n)
        d.append(np.abs(a - b).max())
    if jit == 0.0:
        assert d[1] < d[0] / 100 and d[1] < 1e-4, d
    else:
        assert d[1] < d[0] / 10 and d[1] < 1e-3, d


def test_non_nested_converges():
    """6 : 4 (non-nested) vs 6 : 6: the difference shrinks from N = 2 to N = 5 (algebraically)."""
    d = []
    for N in (2, 5):
        dt, n, a = _mode_run(4, N, 0.0)
        _, _, b = _mode_run(6, N, 0.0, dt, n)
        d.append(np.abs(a - b).max())
    assert d[1] < d[0] / 5, d


def test_non_nested_curved_invariants():
    """Jittered non-nested interface faces: constants in the kernel, symmetric, positive jump energy."""
    rec = curved_interface_config(jitter=0.15, seed=3)
    s = System(rec)
    op_scale = s.gamma_F / (s.M.min() / (25e-6 ** 2))
    a = s.apply_K(np.ones(s.ndof)) / s.M
    assert np.max(np.abs(a)) < 1e-13 * op_scale
    rng = np.random.default_rng(5)
    for _ in range(3):
        u, v = rng.standard_normal((2, s.ndof))
        Ku, Kv = s.apply_K(u), s.apply_K(v)
        assert abs(u @ Kv - v @ Ku) < 1e-12 * np.linalg.norm(u) * np.linalg.norm(Kv)
    step = np.where(np.arange(s.ndof) < s.offsets[1], 1.0, 0.0)
    assert step @ s.apply_interface(step) > 0


def test_non_nested_curved_energy_conserved():
    """Closed rigid two-box system with the jittered non-nested interface: the exact discrete energy
    of the leapfrog is constant -- fails for any asymmetric interface term."""
    rec = curved_interface_config(jitter=0.15, seed=5)
    s = System(rec)
    nm = Newmark(s)
    nm.set_state(np.random.default_rng(2).standard_normal(s.ndof), np.zeros(s.ndof))
    ps = [nm.p.copy()]
    for _ in range(200):
        nm.step()
        ps.append(nm.p.copy())
    dt = rec["dt"]
    E = []
    for n in range(1, 200):
        v = (ps[n + 1] - ps[n]) / dt
        E.append(0.5 * v @ (s.M * v) + 0.5 * ps[n + 1] @ s.apply_K(ps[n]))
    E = np.array(E)
    assert E.min() > 0 and np.max(np.abs(E - E[0])) < 1e-11 * E[0]
