"""Pins for oracle.operators against closed forms and invariants (Eqs. 6-12)."""
import math

import numpy as np
import pytest

from oracle.mesh import REF_VERTS
from oracle.operators import System, element_mass, element_stiffness, penalty_gamma
from sem_inputs import cavity_config, conforming_cut_config, config, small_config


def _leggauss_volume(verts, n=3):
    """Independent volume of a trilinear hex: Gauss-Legendre (not GLL) quadrature of det J,
    with the Jacobian written out from the vertex differences."""
    x, w = np.polynomial.legendre.leggauss(n)
    vol = 0.0
    for i, xi in enumerate(x):
        for j, eta in enumerate(x):
            for k, ze in enumerate(x):
                J = np.zeros((3, 3))
                for v in range(8):
                    s = REF_VERTS[v]
                    f = [(1 + s[0] * xi), (1 + s[1] * eta), (1 + s[2] * ze)]
                    J[:, 0] += verts[v] * s[0] * f[1] * f[2] / 8
                    J[:, 1] += verts[v] * s[1] * f[0] * f[2] / 8
                    J[:, 2] += verts[v] * s[2] * f[0] * f[1] / 8
                vol += w[i] * w[j] * w[k] * np.linalg.det(J)
    return vol


DISTORTED = (REF_VERTS + 1) / 2 * np.array([2.0, 1.0, 1.5]) + \
    np.array([[0, 0, 0], [0.1, 0.05, 0], [0.05, -0.1, 0.02], [0.2, 0.1, -0.1],
              [0, 0.1, 0.05], [-0.05, 0, 0.1], [0.1, 0.1, 0.1], [0.05, -0.05, 0.2]])


@pytest.mark.parametrize("N", [2, 3, 5])
def test_element_matrices_distorted(N):
    c = 1.7
    K = element_stiffness(DISTORTED, N, c)
    M = element_mass(DISTORTED, N)
    vol = _leggauss_volume(DISTORTED)
    assert abs(M.sum() - vol) < 1e-13 * vol                   # sum M = volume
    assert np.max(np.abs(K @ np.ones(len(M)))) < 1e-12 * np.abs(K).max()   # K 1 = 0
    assert np.allclose(K, K.T, rtol=0, atol=1e-13 * np.abs(K).max())
    # nodal coordinates of the element -> p = x: <p, K p> = c^2 int |grad x|^2 = c^2 Vol
    from oracle.gll import gll
    from oracle.mesh import map_point
    xg, _ = gll(N)
    n1 = N + 1
    loc = np.array([(a, b, cc) for cc in range(n1) for b in range(n1) for a in range(n1)])
    X = map_point(DISTORTED, xg[loc])
    for d in range(3):
        assert abs(X[:, d] @ K @ X[:, d] - c * c * vol) < 1e-12 * c * c * vol
    ev = np.linalg.eigvalsh(K)
    assert ev.min() > -1e-12 * ev.max()


def test_mass_and_abc_sums():
    s = System(config(0))
    assert abs(s.M.sum() - 0.6e-3 ** 3) < 1e-14 * 0.6e-3 ** 3
    assert abs(s.C.sum() - 1500 * 0.6e-3 ** 2) < 1e-14 * 1500 * 0.6e-3 ** 2
    # C lives only on the +z face
    xyz = s.node_coords()
    assert np.all(s.C[xyz[:, 2] < 0.6e-3 - 1e-12] == 0)
    two = System(small_config("cfg2s"))
    vol = sum(np.prod(b["extent"]) for b in two.rec["boxes"])
    assert abs(two.M.sum() - vol) < 1e-13 * vol


def _quadratic(xyz):
    x, y, z = xyz[:, 0], xyz[:, 1], xyz[:, 2]
    L = 1e-4
    p = (x * x - 2 * y * y + 3 * z * z + x * y - y * z) / L ** 2 + 2 * x / L - z / L + 0.3
    lap = (2 - 4 + 6) / L ** 2
    return p, lap


def _interior(s, xyz, tol=1e-12):
    keep = np.ones(len(xyz), bool)
    for bi, b in enumerate(s.boxes):
        sl = slice(s.offsets[bi], s.offsets[bi + 1])
        lo, hi = b.origin, b.origin + b.extent
        for d in range(3):
            for face, val in ((2 * d, lo[d]), (2 * d + 1, hi[d])):
                if b.bc[face] == 2:   # interface faces are not outer boundary
                    continue
                on = np.abs(xyz[sl, d] - val) < tol * max(1.0, abs(val)) + 1e-15
                keep[sl][on] = False
                kk = keep[sl]
                kk[on] = False
                keep[sl] = kk
    return keep


def test_volume_patch_and_invariants():
    rec = cavity_config(nel=(3, 2, 2), degree=4, extent=(3e-4, 2.2e-4, 1.8e-4))
    s = System(rec)
    xyz = s.node_coords()
    c2 = s.boxes[0].c ** 2
    one = np.ones(s.ndof)
    Kp1 = s.apply_K(one)
    scale = c2 / (1e-4 / 4) ** 2 * np.max(s.M)
    assert np.max(np.abs(Kp1)) < 1e-12 * scale
    p, lap = _quadratic(xyz)
    inner = _interior(s, xyz)
    a = s.apply_K(p) / s.M
    assert np.max(np.abs(a[inner] + c2 * lap)) < 1e-9 * c2 * lap   # (M^-1 K p) = -c^2 lap p
    # symmetry / PSD on random vectors
    rng = np.random.default_rng(0)
    for _ in range(3):
        u, v = rng.standard_normal((2, s.ndof))
        Ku, Kv = s.apply_K(u), s.apply_K(v)
        assert abs(u @ Kv - v @ Ku) < 1e-12 * np.linalg.norm(u) * np.linalg.norm(Kv)
        assert u @ Ku > 0
    # linear field: <x, K x> = c^2 Vol
    vol = np.prod(rec["boxes"][0]["extent"])
    assert abs(xyz[:, 0] @ s.apply_K(xyz[:, 0]) - c2 * vol) < 1e-12 * c2 * vol


def test_penalty_arithmetic():
    # SPEC S:L252-254
    cbar = 2 * 1481 * 1130 / (1481 + 1130)
    assert abs(cbar - 1281.9) < 0.05
    assert abs(penalty_gamma(1.0, 1.0, 2, 3, 1e-5, 4e-5, 10.0) - 9e6) < 1e-6
    assert abs(penalty_gamma(1481.0, 1130.0, 1, 1, 1.0, 1.0, 1.0) - cbar ** 2) < 1e-6
    # config 2-4 value (reading R7): 10 * 1500^2 * 25 / 25e-6
    s = System(small_config("cfg2s"))
    assert abs(s.gamma_F - 2.25e13) < 1e-14 * 2.25e13


@pytest.fixture(scope="module")
def two_box():
    return System(conforming_cut_config(nel_xy=4, nz_lo=2, nz_hi=2, degree=5, degree_hi=3, ratio=2,
                                        h=25e-6))


def test_interface_patch_tests(two_box):
    s = two_box
    xyz = s.node_coords()
    c2 = 1500.0 ** 2
    # penalty-dominated operator scale (round-off relative to ||M^-1 K|| ||p||)
    op_scale = s.gamma_F / (s.M.min() / (25e-6 ** 2))
    # constant
    a = s.apply_K(np.ones(s.ndof)) / s.M
    assert np.max(np.abs(a)) < 1e-13 * op_scale
    inner = _interior(s, xyz)
    # linear: zero residual at every non-boundary node, including both interface sides
    x, y, z = xyz.T
    p = 1.0 + 2e3 * x - 3e3 * y + 4e3 * z
    a = s.apply_K(p) / s.M
    assert np.max(np.abs(a[inner])) < 1e-13 * op_scale * np.abs(p).max()
    assert np.max(np.abs(a[inner])) < 1e-8 * c2 * 4e3 / 25e-6     # vs. the flux scale c^2 |grad p| / h
    # quadratic: M^-1 K p = -c^2 lap p at interior and interface nodes (quadrature exact, R9)
    p, lap = _quadratic(xyz)
    a = s.apply_K(p) / s.M
    err = np.abs(a[inner] + c2 * lap)
    assert np.max(err) < 1e-13 * op_scale * np.abs(p).max()
    assert np.max(err) < 1e-8 * c2 * lap                             # observed ~1e-10 relative
    # and the interface nodes really are in the checked set
    zi = 2 * 25e-6
    assert np.sum(inner & (np.abs(xyz[:, 2] - zi) < 1e-12)) > 2 * 9


def test_interface_symmetric_psd(two_box):
    s = two_box
    rng = np.random.default_rng(1)
    for _ in range(3):
        u, v = rng.standard_normal((2, s.ndof))
        Ku, Kv = s.apply_K(u), s.apply_K(v)
        assert abs(u @ Kv - v @ Ku) < 1e-12 * np.linalg.norm(u) * np.linalg.norm(Kv)
        assert u @ Ku > -1e-10 * np.linalg.norm(u) * np.linalg.norm(Ku)
    # jump penalty: a field discontinuous across Gamma_I has strictly positive interface energy
    xyz = s.node_coords()
    step = np.where(np.arange(s.ndof) < s.offsets[1], 1.0, 0.0)
    assert step @ s.apply_interface(step) > 0
    assert abs(step @ s.apply_volume(step)) < 1e-6 * (step @ s.apply_interface(step))


def test_coupling_table_closed_form():
    rec = small_config("cfg3s")                       # aligned membranes, N=5, 6 modes
    s = System(rec)
    a = rec["pmut"]["side"]
    tol = {(1, 1): 1e-12, (1, 3): 1e-7, (3, 1): 1e-7, (3, 3): 1e-7, (1, 5): 5e-6, (5, 1): 5e-6}
    for k, (idx, vals) in enumerate(s.B):
        for m, (mm, nn) in enumerate(rec["pmut"]["mode_mn"]):
            exact = 4 * a * a / (mm * nn * math.pi ** 2)
            assert abs(vals[m].sum() - exact) < tol[(int(mm), int(nn))] * exact
        # 21x21 face lattice per membrane; the edge rows carry S = 0 up to sin(m pi) round-off
        assert np.sum(np.abs(vals[0]) > 1e-20) == 19 * 19 and len(idx) <= 21 * 21
    # reciprocity: <f(e_km), p> = kappa * (B p)_km
    rng = np.random.default_rng(2)
    p = rng.standard_normal(s.ndof)
    G = s.pmut_project(p)
    for k, m in [(0, 0), (2, 4), (3, 1)]:
        e = np.zeros_like(G)
        e[k, m] = 1.0
        assert abs(s.pmut_force(e) @ p - s.kappa * G[k, m]) < 1e-12 * abs(s.kappa * G[k, m])
    assert abs(s.kappa - 1000 * 1500 ** 2) < 1e-3          # kappa = rho c^2 = 2.25e9 Pa
