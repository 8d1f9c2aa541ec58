"""The oracle against the worked examples in tests/golden/ (each case cites its source; expected values
are closed-form expressions, see the fixture's "about")."""
import json
import math
import os

import numpy as np
import pytest

from oracle.gll import gll
from oracle.mesh import REF_VERTS
from oracle.operators import element_mass, element_stiffness, penalty_gamma
from oracle.pml import coefficients, damping_profile, zeta_tilde

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")
CASES = {c["id"]: c for c in json.load(open(GOLDEN))["cases"]}


def ev(expr):
    return float(eval(str(expr), {"__builtins__": {}}, {"sqrt": math.sqrt, "pi": math.pi, "log": math.log}))


def close(x, expr, tol):
    e = ev(expr)
    return abs(x - e) <= tol * max(abs(e), 1.0)


def cube(lo, hi):
    return np.asarray(lo, float)[None, :] + (REF_VERTS + 1.0) / 2.0 * (np.asarray(hi, float) - np.asarray(lo, float))[None, :]


@pytest.mark.parametrize("cid", ["gll_1", "gll_2", "gll_3", "gll_4", "gll_5"])
def test_gll_rules(cid):
    c = CASES[cid]
    x, w = gll(c["N"])
    for got, exp in zip(x, c["nodes"]):
        assert close(got, exp, c["tol"]), (cid, got, exp)
    for got, exp in zip(w, c["weights"]):
        assert close(got, exp, c["tol"]), (cid, got, exp)


def test_gll_exact_moment():
    c = CASES["gll_2_xi2"]
    x, w = gll(2)
    assert close(float(w @ x ** 2), c["expected"], c["tol"])


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
def test_mass_and_stiffness_examples(N):
    v = cube((0, 0, 0), (1, 1, 1))
    c = CASES["mass_unit_cube"]
    assert close(float(element_mass(v, N).sum()), c["expected"], c["tol"])
    c = CASES["mass_2x1x1"]
    tot = element_mass(v, N).sum() + element_mass(cube((1, 0, 0), (2, 1, 1)), N).sum()
    assert close(float(tot), c["expected"], c["tol"])
    c = CASES["stiffness_x_energy"]
    K = element_stiffness(v, N, 1.0)
    x, _ = gll(N)
    n1 = N + 1
    px = np.array([(x[i % n1] + 1) / 2 for i in range(n1 ** 3)])   # the x coordinate of each node
    assert close(float(px @ K @ px), c["expected"], c["tol"])


def test_abc_face_sum():
    from oracle.operators import System
    from sem_inputs import BC_ABSORBING, BC_RIGID, cavity_config
    c = CASES["abc_face_sum"]
    side = math.sqrt(c["A"])
    rec = cavity_config(nel=(2, 2, 1), degree=3, extent=(side, side, side / 2), c=c["c"])
    rec["boxes"][0]["bc"] = [BC_RIGID] * 5 + [BC_ABSORBING]
    assert close(float(System(rec).C.sum()), c["expected"], c["tol"])


def test_penalty_examples():
    c = CASES["penalty_equal_speeds"]
    g = penalty_gamma(c["c"], c["c"], c["r"][0], c["r"][1], c["h"][0], c["h"][1], c["alpha"])
    assert close(g, c["expected"], c["tol"])
    c = CASES["penalty_cbar"]
    cbar = math.sqrt(penalty_gamma(c["c"][0], c["c"][1], 1, 1, 1.0, 1.0, 1.0))
    assert close(cbar, c["expected"], c["tol"])
    c = CASES["penalty_value"]
    assert close(penalty_gamma(1.0, 1.0, 2, 3, 1e-5, 4e-5, 10.0), c["expected"], c["tol"])


def test_pml_examples():
    c = CASES["pml_zeta_tilde"]
    zt = zeta_tilde(1481.0, 592.4e-6, 1e-4)
    assert close(zt, c["expected"], c["tol"])
    c = CASES["pml_profile"]
    ell = 592.4e-6
    for d, exp in zip((0.0, ell / 2, ell), c["expected"]):
        assert close(float(damping_profile(d, ell, zt)) / zt, exp, c["tol"])
    for cid in ("pml_coefficients_s00", "pml_coefficients_sss"):
        c = CASES[cid]
        s = c["s"]
        z = np.array([s, 0.0, 0.0]) if cid.endswith("s00") else np.array([s, s, s])
        a, b, g, Z1, Z2, Z3 = coefficients(z)
        assert close(float(a), c["alpha"], c["tol"]) and close(float(b), c["beta"], c["tol"])
        assert close(float(g), c["gamma"], c["tol"])
        for got, exp in zip(Z2, c["Z2"]):
            assert close(float(got), exp, c["tol"])
        for key, arr in (("Z1", Z1), ("Z3", Z3)):
            for got, exp in zip(arr, c.get(key, [])):
                assert close(float(got), exp, c["tol"])
