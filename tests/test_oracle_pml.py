"""Pins for oracle.pml (Eq. 1 PML; readings R23-R25) against closed forms,
exact polynomial identities and the qualitative absorption property (SPEC acceptance 6)."""
import math

import numpy as np
import pytest

from oracle.newmark import Newmark
from oracle.operators import System
from oracle.pml import Pml, coefficients, damping_profile, zeta_tilde
from sem_inputs import pml_config


def test_zeta_tilde_and_profile_closed_forms():
    # paper's array run: PML thickness = one wavelength lambda_w = c / f = 1481 / 2.5e6 = 592.4 um
    # (P:L1308), so c / l = f = 2.5e6 1/s and zt = 2.5e6 ln(1/R); SPEC S:L326 quotes ~2.3023e7 for R=1e-4
    zt = zeta_tilde(1481.0, 592.4e-6, 1e-4)
    assert abs(zt - 2.5e6 * 4 * math.log(10.0)) < 1e-12 * zt
    assert abs(zt - 2.3023e7) < 2e-4 * zt
    assert abs(zeta_tilde(1500.0, 2e-4, 1e-4) - 0.5 * zeta_tilde(1500.0, 1e-4, 1e-4)) < 1e-9 * zt
    ell = 1e-4
    assert damping_profile(0.0, ell, zt) == 0.0
    assert damping_profile(-3e-5, ell, zt) == 0.0
    assert abs(damping_profile(ell, ell, zt) - zt) < 1e-12 * zt
    assert abs(damping_profile(ell / 2, ell, zt) - zt / 2) < 1e-12 * zt
    # C^1 at the inner plane: z(d) = zt (2 pi^2 / 3)(d/l)^3 + O(d^5)  (Taylor of s - sin(2 pi s)/(2 pi))
    for s in (1e-2, 5e-3):
        d = s * ell
        assert abs(damping_profile(d, ell, zt) / (zt * (2 * math.pi ** 2 / 3) * s ** 3) - 1) < 1e-3
    d = np.linspace(0, ell, 201)
    assert np.all(np.diff(damping_profile(d, ell, zt)) >= 0)        # monotone in the layer


def test_coefficients_are_the_stretching_polynomial():
    """(i w + z1)(i w + z2)(i w + z3) = (i w)^3 + alpha (i w)^2 + beta (i w) + gamma: alpha, beta, gamma
    are the coefficients of the polynomial with roots -z_i (numpy.poly); Z3_i = gamma / z_i and
    Z2_i = alpha - 2 z_i = (sum of the other two) - z_i."""
    rng = np.random.default_rng(5)
    for _ in range(5):
        z = rng.uniform(0.1, 3.0, 3) * 1e7
        a, b, g, Z1, Z2, Z3 = coefficients(z)
        ref = np.poly(-z)
        assert np.allclose([a, b, g], ref[1:], rtol=1e-13, atol=0)
        assert np.allclose(Z3, g / z, rtol=1e-13)
        assert np.allclose(Z1, -z)
        for i in range(3):
            others = [j for j in range(3) if j != i]
            assert abs(Z2[i] - (z[others].sum() - z[i])) < 1e-12 * a
    # one-axis layer: Z3 = 0, beta = gamma = 0
    a, b, g, Z1, Z2, Z3 = coefficients(np.array([2.0, 0.0, 0.0]))
    assert (a, b, g) == (2.0, 0.0, 0.0) and np.all(Z3 == 0) and list(Z2) == [-2.0, 2.0, 2.0]


def _full_pml_system(N=4, nel=(2, 2, 2)):
    # layers on -z and +z, half the box each: every element touches z > 0 (Phi lives everywhere)
    rec = pml_config(nel=nel, degree=N, extent=(2e-4, 2.4e-4, 2.2e-4), layers=(0, 0, 0, 0, 1, 1),
                     layer_el=nel[2] // 2)
    s = System(rec)
    return rec, s, Pml(s, rec["pml"])


@pytest.mark.parametrize("N", [3, 4, 5])
def test_element_gradient_exact_for_polynomials(N):
    rec, s, pml = _full_pml_system(N)
    assert len(pml.elems) == s.boxes[0].nelem
    xyz = s.node_coords()
    x, y, z = xyz.T * 1e4
    f = x ** N + 2 * y ** (N - 1) * z + x * y * z
    g = np.stack([N * x ** (N - 1) + y * z, 2 * (N - 1) * y ** (N - 2) * z + x * z, 2 * y ** (N - 1) + x * y], axis=1) * 1e4
    G = pml.element_gradient(f)
    for k in range(len(pml.elems)):
        ref = g[pml.conn[k]]
        assert np.max(np.abs(G[k] - ref)) < 1e-11 * np.max(np.abs(g))


@pytest.mark.parametrize("N", [3, 4])
def test_weak_divergence_is_lumped_divergence(N):
    """For Phi = (x^2 y, y^2 z, z^2 x) (GLL-exact products), sum_e int Phi . grad psi_i = -M_ii (div Phi)(x_i)
    at interior nodes (element-boundary terms cancel, lumped mass exact for (div Phi) psi_i)."""
    rec, s, pml = _full_pml_system(N)
    xyz = s.node_coords() * 1e4
    phi = np.stack([xyz[:, 0] ** 2 * xyz[:, 1], xyz[:, 1] ** 2 * xyz[:, 2], xyz[:, 2] ** 2 * xyz[:, 0]], axis=1)
    div = (2 * xyz[:, 0] * xyz[:, 1] + 2 * xyz[:, 1] * xyz[:, 2] + 2 * xyz[:, 2] * xyz[:, 0]) * 1e4
    phi_e = np.stack([phi[pml.conn[k]] for k in range(len(pml.elems))])
    rB = pml.weak_divergence(phi_e)
    b = s.boxes[0]
    lo, hi = xyz.min(axis=0), xyz.max(axis=0)
    interior = np.all((xyz > lo + 1e-9) & (xyz < hi - 1e-9), axis=1)
    err = np.abs(-rB[interior] / s.M[interior] - div[interior])
    assert interior.sum() > 10
    assert err.max() < 1e-11 * np.abs(div).max()


def test_phi_update_frozen_gradient_closed_form():
    """Layer along x only (Z3 = 0) and a frozen linear p = g.x: Phi_x' = -z Phi_x - c^2 z g_x,
    Phi_y' = c^2 z g_y, Phi_z' = c^2 z g_z (Eq. 1 line 2 with Z2 = (-z, z, z)):
    Phi_x = -c^2 g_x (1 - e^{-z t}),  Phi_{y,z} = c^2 z g_{y,z} t.  Crank-Nicolson: second order, exact
    for the undamped components."""
    errs = []
    for scale in (1.0, 0.5):
        rec = pml_config(nel=(2, 1, 1), degree=3, extent=(2e-4, 1e-4, 1e-4), layers=(0, 1, 0, 0, 0, 0),
                         layer_el=1)
        s = System(rec)
        pml = Pml(s, rec["pml"])
        xyz = s.node_coords()
        gvec = np.array([3.0, -2.0, 1.5]) * 1e4
        p = xyz @ gvec
        dt = 2e-9 * scale
        nsteps = int(round(4e-8 / dt))
        for _ in range(nsteps):
            pml.advance(p, dt)
        t = nsteps * dt
        c2 = s.boxes[0].c ** 2
        err = 0.0
        for k in range(len(pml.elems)):
            z = pml.zeta[pml.conn[k], 0]
            ref_x = -c2 * gvec[0] * (1 - np.exp(-z * t))
            ref_y = c2 * z * gvec[1] * t
            ref_z = c2 * z * gvec[2] * t
            scale_ref = c2 * abs(gvec[0])
            err = max(err, np.max(np.abs(pml.phi[k][:, 0] - ref_x)) / scale_ref)
            assert np.max(np.abs(pml.phi[k][:, 1] - ref_y)) <= 1e-12 * (np.max(np.abs(ref_y)) + scale_ref)
            assert np.max(np.abs(pml.phi[k][:, 2] - ref_z)) <= 1e-12 * (np.max(np.abs(ref_z)) + scale_ref)
        assert np.max(np.abs(pml.zeta[:, 1:])) == 0.0
        errs.append(err)
    assert errs[0] < 1e-3
    assert 3.5 < errs[0] / errs[1] < 4.5


def _column_run(top_layer, abc):
    rec = pml_config(nel=(1, 1, 16), degree=4, extent=(50e-6, 50e-6, 800e-6), layers=(0, 0, 0, 0, 0, int(top_layer)),
                     layer_el=4, abc_on_pml=abc)
    s = System(rec)
    nm = Newmark(s)
    xyz = s.node_coords()
    p0 = np.exp(-((xyz[:, 2] - 200e-6) / 40e-6) ** 2)
    nm.set_state(p0, np.zeros_like(p0))
    nm.run(int(2 * 800e-6 / 1500 / rec["dt"]))
    return np.abs(nm.p[xyz[:, 2] < 400e-6]).max()


def test_pml_absorbs_normal_incidence():
    """SPEC acceptance 6 (qualitative reproduction of the paper's PML figure): a pulse in a rigid
    column; after two transits the field below the layer is <= 1e-2 of the initial peak with a PML
    (rigid wall behind it), >= 0.3 with a bare rigid top."""
    assert _column_run(True, abc=False) < 1e-2
    assert _column_run(False, abc=False) > 0.3


def test_zero_thickness_is_the_acoustic_system():
    """No layer -> no PML element, alpha = beta = gamma = 0: Algorithm 1 unchanged, bit for bit."""
    rec = pml_config(nel=(2, 2, 2), degree=3, extent=(1e-4, 1e-4, 1e-4), layers=(0,) * 6)
    base = dict(rec)
    base["pml"] = None
    rng = np.random.default_rng(2)
    a, b = Newmark(System(rec)), Newmark(System(base))
    p0 = rng.standard_normal(a.sys.ndof)
    a.set_state(p0, 0 * p0)
    b.set_state(p0, 0 * p0)
    a.run(20)
    b.run(20)
    assert len(a.pml.elems) == 0
    assert np.array_equal(a.p, b.p)
