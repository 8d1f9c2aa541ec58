"""Pins for caller-defined mode shapes in the oracle's coupling table (reading R33; Eqs. 11-12 with
U_{k,m} an input): B_{k,m,j} = sum_F w_q |J_s| S_{k,m}(x_j) must reproduce closed-form
integrals of the shape -- exactly for a polynomial on a membrane aligned with element boundaries (GLL
exactness), including its first moments (which fix the sign and the x / y order of the arguments the
shape is called with), and up to the quadrature error for the clamped circular plate of P:L1097."""
import math

import numpy as np
from scipy.special import iv, jv

from oracle.operators import System
from sem_inputs import circular_pmut_config, clamped_disc_shape, curved_pmut_config


def test_polynomial_shape_integrates_exactly():
    # 6 x 6 face elements of 25 um, N = 4; membrane = the 4 x 4 central elements (side 100 um)
    rec = curved_pmut_config(amp=0.0, floor_jitter=0.0)
    a = 100e-6
    cfs = (0.0, 0.8, -1.7)

    def shape(k, m, xr, yr):      # vanishes on the square's edge; degree 3 in x, 4 in y
        u, v = 2 * xr / a, 2 * yr / a
        return (1 - u * u) * (1 - v * v) * (1 + cfs[m] * u + 0.5 * cfs[m] * v * v)

    rec["pmut"]["side"] = a
    rec["pmut"]["shape_fn"] = shape
    s = System(rec)
    xyz = s.node_coords()
    cx, cy = rec["pmut"]["centers"][0]
    one = np.ones(s.ndof)
    G0 = s.pmut_project(one)[0]
    Gx = s.pmut_project(xyz[:, 0] - cx)[0]
    Gy = s.pmut_project(xyz[:, 1] - cy)[0]
    for m, c in enumerate(cfs):
        # int (1-u^2)(1 + c u) (a/2) du = 2a/3;  int (1-v^2)(1 + c/2 v^2) (a/2) dv = (a/2)(4/3 + (c/2)(4/15))
        i0 = (2 * a / 3) * (a / 2) * (4 / 3) + (2 * a / 3) * (a / 2) * (0.5 * c) * (4 / 15)
        # x moment: only the c u term survives: (a/2)^2 c int (1-u^2) u^2 du = (a^2/4) c (4/15), times (a/2)(4/3)
        ix = (a * a / 4) * c * (4 / 15) * (a / 2) * (4 / 3)
        assert abs(G0[m] - i0) < 1e-13 * a * a, (m, G0[m], i0)
        assert abs(Gx[m] - ix) < 1e-13 * a ** 3, (m, Gx[m], ix)
        assert abs(Gy[m]) < 1e-13 * a ** 3


def test_clamped_disc_modes_and_their_integrals():
    R = 65e-6
    modes = ((0, 1), (1, 1), (0, 2))
    f = clamped_disc_shape(R, modes)
    # textbook eigenvalues of the clamped circular plate (lambda_01, lambda_11, lambda_02)
    assert np.allclose(f.lam, (3.19622, 4.61090, 6.30644), atol=1e-5)
    # clamped: S = dS/dr = 0 at r = R; unit peak
    for m in range(3):
        assert abs(f(0, m, R, 0.0)) < 1e-14
        assert abs(f(0, m, R * (1 - 1e-6), 0.0)) < 1e-10
        assert f(0, m, 0.0, 1.0001 * R) == 0.0
    assert abs(f(0, 0, 0.0, 0.0) - 1.0) < 1e-12 and abs(f(0, 1, 0.3 * R, 0.0) + f(0, 1, -0.3 * R, 0.0)) < 1e-15
    assert abs(f(0, 1, 0.0, 0.4 * R)) < 1e-15      # cos(theta) nodal line on the y axis
    rec = circular_pmut_config(amp=0.0, floor_jitter=0.0, degree=5)
    s = System(rec)
    G = s.pmut_project(np.ones(s.ndof))[0]
    for m, (n, _) in enumerate(modes):
        l = f.lam[m]
        exact = 0.0 if n else 2 * math.pi * R * R * f.scale[m] * (jv(1, l) - jv(0, l) / iv(0, l) * iv(1, l)) / l
        assert abs(G[m] - exact) < 2e-3 * math.pi * R * R, (m, G[m], exact)
    assert abs(G[0]) > 0.25 * math.pi * R * R


def test_cylinder_domain_geometry_and_stability():
    """The cylinder column of P:L1225 as one mapped box: the lumped mass sums to the volume of the
    extruded polygon through the mapped boundary vertices (shoelace area x height, exact for the
    trilinear map), the absorbing top's ABC diagonal to c x that area, K 1 = 0, and the record's time step
    is inside the leapfrog stability limit of this mesh."""
    from sem_inputs import cylinder_pmut_config
    rec = cylinder_pmut_config(n_steps=120)
    b = rec["boxes"][0]
    nx, ny, nz = b["nel"]
    V = b["vertices"].reshape(nz + 1, ny + 1, nx + 1, 3)[0, :, :, :2]
    ring = np.concatenate([V[0, :-1], V[:-1, -1], V[-1, :0:-1], V[:0:-1, 0]])       # counter-clockwise boundary
    area = 0.5 * abs(np.sum(ring[:, 0] * np.roll(ring[:, 1], -1) - np.roll(ring[:, 0], -1) * ring[:, 1]))
    R = 0.5 * b["extent"][0]
    assert np.allclose(np.hypot(ring[:, 0] - R, ring[:, 1] - R), R, rtol=1e-12)      # wall vertices on the circle
    assert 0.93 * math.pi * R * R < area < math.pi * R * R
    s = System(rec)
    H = b["extent"][2]
    assert abs(s.M.sum() - area * H) < 1e-12 * area * H
    assert abs(s.C.sum() - b["c"] * area) < 1e-12 * b["c"] * area
    assert np.abs(s.apply_K(np.ones(s.ndof))).max() < 1e-10 * b["c"] ** 2 * area * H / (H / nz) ** 2
    # stability of the record's time step: dt < 2 / sqrt(lambda_max(M^-1 K)) (power iteration), margin >= 1.5
    v = np.random.default_rng(0).standard_normal(s.ndof)
    for _ in range(150):
        w = s.apply_K(v) / s.M
        lam = np.linalg.norm(w) / np.linalg.norm(v)
        v = w / np.linalg.norm(w)
    assert rec["dt"] * math.sqrt(lam) / 2 < 0.67, rec["dt"] * math.sqrt(lam) / 2


def test_cylinder_two_box_geometry_and_stability():
    """Fine inner + coarse outer box on the same polygonal cylinder (bilinear subdivision): both lumped
    masses sum to shoelace area x height, the SIPG interface leaves constants alone (K 1 = 0: every fine
    quadrature node found its coarse owner and the jump of a constant vanishes), dt inside the stability
    limit of the coupled operator."""
    from sem_inputs import cylinder_two_box_config
    rec = cylinder_two_box_config()
    s = System(rec)
    M0, M1 = s.split(s.M)
    for b, Mb in zip(rec["boxes"], (M0, M1)):
        nx, ny, nz = b["nel"]
        V = b["vertices"].reshape(nz + 1, ny + 1, nx + 1, 3)[0, :, :, :2]
        ring = np.concatenate([V[0, :-1], V[:-1, -1], V[-1, :0:-1], V[:0:-1, 0]])
        area = 0.5 * abs(np.sum(ring[:, 0] * np.roll(ring[:, 1], -1) - np.roll(ring[:, 0], -1) * ring[:, 1]))
        assert abs(Mb.sum() - area * b["extent"][2]) < 1e-12 * area * b["extent"][2]
    c2 = rec["boxes"][0]["c"] ** 2
    K1 = s.apply_K(np.ones(s.ndof))
    v = np.random.default_rng(0).standard_normal(s.ndof)
    Kv = s.apply_K(v)
    assert np.abs(K1).max() < 1e-11 * np.abs(Kv).max()
    for _ in range(150):
        w = s.apply_K(v) / s.M
        lam = np.linalg.norm(w) / np.linalg.norm(v)
        v = w / np.linalg.norm(w)
    assert rec["dt"] * math.sqrt(lam) / 2 < 0.67, rec["dt"] * math.sqrt(lam) / 2


def test_cylinder_obstacle_fluid_volume():
    """Section 6.2's cylinder with its rounded rigid slab: the lumped mass (fluid only) sums to the column's
    volume minus the slab's -- both extruded polygons (shoelace areas of the mapped boundary rings)."""
    from sem_inputs import cylinder_obstacle_config

    def shoelace(ring):
        return 0.5 * abs(np.sum(ring[:, 0] * np.roll(ring[:, 1], -1) - np.roll(ring[:, 0], -1) * ring[:, 1]))

    rec = cylinder_obstacle_config(n_steps=1)
    b = rec["boxes"][0]
    nx, ny, nz = b["nel"]
    V = b["vertices"].reshape(nz + 1, ny + 1, nx + 1, 3)[0, :, :, :2]
    outer = np.concatenate([V[0, :-1], V[:-1, -1], V[-1, :0:-1], V[:0:-1, 0]])
    B = V[1:ny, 1:nx]                                     # vertices of the 6 x 6 central element block
    inner = np.concatenate([B[0, :-1], B[:-1, -1], B[-1, :0:-1], B[:0:-1, 0]])
    hz = b["extent"][2] / nz
    vol = shoelace(outer) * b["extent"][2] - shoelace(inner) * hz
    s = System(rec)
    assert abs(s.M.sum() - vol) < 1e-12 * vol
    assert 0.55 < shoelace(inner) / shoelace(outer) < 0.8   # (6/8)^2-ish of the section: ~5/6 of the diameter
