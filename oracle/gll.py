"""Gauss-Legendre-Lobatto rule and Lagrange basis (oracle; test infrastructure only).

P:L581 "Lagrangian basis functions", "diagonal mass matrix ... evaluated
with reduced integration": the SEM uses the (N+1)-point GLL rule as both the
interpolation nodes and the quadrature.  Nodes are -1, +1 and the roots of P_N'
(Newton, tol 1e-15); weights 2 / (N (N+1) P_N(x_j)^2).
"""
from __future__ import annotations

import math
from functools import lru_cache

import numpy as np


def legendre(n: int, x):
    """P_n(x) and P_n'(x) by the three-term recurrence (Bonnet)."""
    x = np.asarray(x, dtype=np.float64)
    p0, p1 = np.ones_like(x), x.copy()
    d0, d1 = np.zeros_like(x), np.ones_like(x)
    if n == 0:
        return p0, d0
    for k in range(1, n):
        p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1)
        d2 = d0 + (2 * k + 1) * p1
        p0, p1, d0, d1 = p1, p2, d1, d2
    return p1, d1


@lru_cache(maxsize=None)
def gll(n: int):
    """(nodes, weights) of the n+1 point GLL rule on [-1, 1], ascending."""
    if not 1 <= n <= 16:
        raise ValueError("degree must be in 1..16")
    x = np.empty(n + 1)
    x[0], x[n] = -1.0, 1.0
    for j in range(1, n):
        xi = -math.cos(math.pi * j / n)
        for _ in range(100):
            p, dp = legendre(n, xi)
            # Legendre ODE: (1-x^2) P'' = 2 x P' - n(n+1) P
            d2p = (2 * xi * dp - n * (n + 1) * p) / (1 - xi * xi)
            step = float(dp / d2p)
            xi -= step
            if abs(step) < 1e-15:
                break
        x[j] = xi
    p, _ = legendre(n, x)
    w = 2.0 / (n * (n + 1) * p * p)
    return x, w


def lagrange(nodes, j: int, x):
    """ell_j(x) = prod_{k != j} (x - x_k) / (x_j - x_k)   (product formula)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.ones_like(x)
    for k, xk in enumerate(nodes):
        if k != j:
            out = out * (x - xk) / (nodes[j] - xk)
    return out


def lagrange_deriv(nodes, j: int, x):
    """ell_j'(x) = sum_{m != j} 1/(x_j - x_m) prod_{k != j, m} (x - x_k)/(x_j - x_k)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    for m, xm in enumerate(nodes):
        if m == j:
            continue
        term = np.full_like(x, 1.0 / (nodes[j] - xm))
        for k, xk in enumerate(nodes):
            if k != j and k != m:
                term = term * (x - xk) / (nodes[j] - xk)
        out = out + term
    return out


def basis_matrix(nodes, x):
    """B[q, j] = ell_j(x_q)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    return np.stack([lagrange(nodes, j, x) for j in range(len(nodes))], axis=1)


def deriv_matrix(nodes, x):
    """D[q, j] = ell_j'(x_q)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    return np.stack([lagrange_deriv(nodes, j, x) for j in range(len(nodes))], axis=1)
