"""Pins of the oracle's Gauss-Legendre interface quadrature (reading R9's flag: the (N_in+1)^2 LG points
of each fine face instead of its GLL nodes; Fig. 7's "LG" nodes).  Pinned by what the two
rules' exactness degrees fix:
  * for fields both rules integrate exactly (a global linear p: the jump vanishes and the flux is
    constant) the LG and GLL interface operators agree to rounding;
  * for v^T K_Gamma p with p = v = (x/Lx)^5 on the fine side only (z-independent, so only the penalty
    term gamma int x^10 survives), the 6-point LG rule reproduces the closed form gamma Lx Ly / 11
    (exact up to degree 11) while the 6-point GLL rule (exact up to degree 9) does not;
  * constants are in the kernel and the operator is symmetric for either rule.
"""
import numpy as np
import pytest

from oracle.operators import System
from sem_inputs import conforming_cut_config


def _rec(rule, nel_xy=4, degree=5, degree_hi=3, ratio=2):
    rec = conforming_cut_config(nel_xy=nel_xy, nz_lo=1, nz_hi=1, degree=degree, degree_hi=degree_hi,
                                ratio=ratio, h=25e-6)
    rec["interface"] = dict(rec["interface"], quad=rule)
    return rec


def _coords(s):
    return np.concatenate([b.node_coords() for b in s.boxes])


@pytest.mark.parametrize("ratio,dh", [(2, 3), (1, 5)])
def test_lg_equals_gll_on_linear_fields(ratio, dh):
    sg, sl = System(_rec("gll", degree_hi=dh, ratio=ratio)), System(_rec("lg", degree_hi=dh, ratio=ratio))
    xyz = _coords(sg)
    p = 1.0 + 3e3 * xyz[:, 0] - 2e3 * xyz[:, 1] + 5e3 * xyz[:, 2]
    rg, rl = sg.apply_interface(p), sl.apply_interface(p)
    # the jump of a linear field is zero only to rounding and is multiplied by gamma ~ 1e13 / m
    assert np.max(np.abs(rl - rg)) <= 1e-10 * np.max(np.abs(rg))
    assert np.max(np.abs(rg)) > 0.0


def test_lg_exact_penalty_integral_gll_not():
    out = {}
    for rule in ("gll", "lg"):
        s = System(_rec(rule, nel_xy=1, degree_hi=5, ratio=1))     # one fine face: x^10 on [0, Lx]
        xyz = _coords(s)
        Lx = s.boxes[0].extent[0]
        Ly = s.boxes[0].extent[1]
        nF = s.boxes[0].ndof
        v = np.zeros(s.ndof)
        v[:nF] = (xyz[:nF, 0] / Lx) ** 5
        val = v @ s.apply_interface(v)
        out[rule] = abs(val / (s.gamma_F * Lx * Ly / 11.0) - 1.0)
    assert out["lg"] < 1e-12, out
    assert out["gll"] > 1e-6, out


@pytest.mark.parametrize("rule", ["gll", "lg"])
def test_constants_in_kernel_and_symmetry(rule):
    s = System(_rec(rule, nel_xy=2))
    assert np.max(np.abs(s.apply_interface(np.ones(s.ndof)))) < 1e-6 * s.gamma_F * 1e-12
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal(s.ndof), rng.standard_normal(s.ndof)
    x, y = a @ s.apply_interface(b), b @ s.apply_interface(a)
    assert abs(x - y) <= 1e-12 * max(abs(x), abs(y))
