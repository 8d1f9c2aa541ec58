"""Pins for oracle.gll against closed forms (GLL rule, Lagrange basis)."""
import math

import numpy as np
import pytest

from oracle.gll import basis_matrix, deriv_matrix, gll, legendre


def test_gll_closed_forms():
    # N=1: nodes +-1, weights 1; N=2: nodes -1,0,1, weights 1/3, 4/3, 1/3
    x, w = gll(1)
    assert np.allclose(x, [-1, 1], atol=0) and np.allclose(w, [1, 1], rtol=1e-15)
    x, w = gll(2)
    assert np.allclose(x, [-1, 0, 1], atol=1e-16)
    assert np.allclose(w, [1 / 3, 4 / 3, 1 / 3], rtol=1e-15)
    # N=3: interior nodes +-1/sqrt(5), weights 1/6, 5/6 (textbook)
    x, w = gll(3)
    assert np.allclose(x, [-1, -1 / math.sqrt(5), 1 / math.sqrt(5), 1], rtol=1e-15)
    assert np.allclose(w, [1 / 6, 5 / 6, 5 / 6, 1 / 6], rtol=1e-15)
    # N=4: interior +-sqrt(3/7), 0; weights 1/10, 49/90, 32/45
    x, w = gll(4)
    assert np.allclose(x, [-1, -math.sqrt(3 / 7), 0, math.sqrt(3 / 7), 1], rtol=1e-15, atol=1e-16)
    assert np.allclose(w, [0.1, 49 / 90, 32 / 45, 49 / 90, 0.1], rtol=1e-14)


@pytest.mark.parametrize("n", range(1, 9))
def test_gll_exactness(n):
    x, w = gll(n)
    assert abs(w.sum() - 2) < 1e-14
    assert np.allclose(x, -x[::-1], atol=1e-15)
    for k in range(0, 2 * n):                      # exact up to degree 2N-1
        exact = 2.0 / (k + 1) if k % 2 == 0 else 0.0
        assert abs(w @ x ** k - exact) < 1e-14
    if n >= 1:                                      # and NOT exact for x^(2N) (it is GLL, not GL)
        k = 2 * n
        assert abs(w @ x ** k - 2.0 / (k + 1)) > 1e-6
    # interior nodes are roots of P_N'
    _, dp = legendre(n, x[1:-1])
    assert np.all(np.abs(dp) < 1e-12)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8])
def test_lagrange_basis(n):
    x, _ = gll(n)
    B = basis_matrix(x, x)
    assert np.array_equal(B, np.eye(n + 1))       # cardinal at nodes, exactly
    D = deriv_matrix(x, x)
    assert np.allclose(D @ np.ones(n + 1), 0, atol=1e-12)
    assert np.allclose(D @ x, 1, atol=1e-12)
    # derivative exact for a degree-N polynomial at arbitrary points
    rng = np.random.default_rng(n)
    coef = rng.standard_normal(n + 1)
    poly = np.polynomial.Polynomial(coef)
    t = rng.uniform(-1, 1, 7)
    assert np.allclose(deriv_matrix(x, t) @ poly(x), poly.deriv()(t), atol=1e-11)
    assert np.allclose(basis_matrix(x, t) @ poly(x), poly(t), atol=1e-12)
    # partition of unity off-node
    assert np.allclose(basis_matrix(x, t).sum(axis=1), 1, atol=1e-13)
