"""Perfectly matched layer of Eq. (1) for the oracle (TEST INFRASTRUCTURE ONLY).

PAPER.md (P:L<line>):
* Eq. (1):  p_tt + alpha p_t + beta p = div(c^2 grad p) + div Phi - gamma psi,
                        Phi_t = Z1 Phi + c^2 Z2 grad p + c^2 Z3 grad psi,   psi_t = p.
* alpha = z1 + z2 + z3, beta = z1 z2 + z2 z3 + z3 z1, gamma = z1 z2 z3,
              Z1 = diag(-z_i), Z2 = diag(alpha - 2 z_i), Z3 = diag(z2 z3, z3 z1, z1 z2).
* z_i(x_i) = zt_i ((|x_i| - h_i)/l_i - sin(2 pi (|x_i| - h_i)/l_i)/(2 pi)) inside the layer
              h_i <= |x_i| <= h_i + l_i, 0 elsewhere;  zt_i = (c / l_i) log(1/R).
* "a similar scheme is employed when a PML boundary is introduced" -- the placement of the
  auxiliary updates in Algorithm 1 is not given.  Readings (R23-R25):

  R23 (layers of a box): a PML of thickness l on box face f occupies the l-thick slab of the box next
      to f; the distance into the layer d = (distance from the layer's inner plane), so
      z_i = zt (d/l - sin(2 pi d/l)/(2 pi)) for 0 <= d <= l (the paper's |x_i| - h_i).  The face keeps
      its own boundary condition (the paper's Gamma_ABC at the outer PML boundary: ABC).
  R24 (spaces and weak form): psi is a continuous nodal GLL field like p; Phi is element-local
      (discontinuous, one 3-vector per element GLL node, like the element-wise gradient it is driven
      by).  div Phi enters the weak form integrated by parts, -sum_e int_e Phi . grad v, with the
      outer-boundary term int Phi.n v dropped (natural condition on the total flux
      (c^2 grad p + Phi).n).  GLL quadrature throughout (reduced integration).
  R25 (time levels): Algorithm 1 unchanged for p; psi and Phi live at half steps:
          psi^{n+3/2} = psi^{n+1/2} + dt p^{n+1},                  psi^{n+1} = (psi^{n+1/2} + psi^{n+3/2})/2,
          Phi^{n+3/2} = [(1 - dt z/2) Phi^{n+1/2} + dt c^2 (Z2 grad p^{n+1} + Z3 grad psi^{n+1})] / (1 + dt z/2),
          Phi^{n+1} = (Phi^{n+1/2} + Phi^{n+3/2})/2   (Crank-Nicolson on Z1, explicit because diagonal),
      and the acoustic solve of Algorithm 1 gains the PML terms at the predictor velocity
      (like C pdot^{n+1}):
          pdd^{n+1} = M^-1 (f - K p^{n+1} - C pd^{n+1} - B^T Phi^{n+1}) - alpha pd^{n+1} - beta p^{n+1} - gamma psi^{n+1}
      with (B^T Phi)_i = sum_e sum_q w_q |J_q| Phi(e, q) . grad phi_i(x_q).  psi^{1/2} = Phi^{1/2} = 0.
"""
from __future__ import annotations

import math

import numpy as np

from .gll import gll


def zeta_tilde(c, ell, R):
    """zt = (c / l) log(1/R)."""
    if not (0.0 < R < 1.0):
        raise ValueError("reflection coefficient must be in (0, 1)")
    return c / ell * math.log(1.0 / R)


def damping_profile(d, ell, zt):
    """z(d) = zt (d/l - sin(2 pi d / l) / (2 pi)) for 0 <= d <= l, 0 for d <= 0.
    d is the distance into the layer (the paper's |x_i| - h_i)."""
    d = np.asarray(d, dtype=np.float64)
    s = np.clip(d / ell, 0.0, 1.0)
    return np.where(d > 0.0, zt * (s - np.sin(2.0 * math.pi * s) / (2.0 * math.pi)), 0.0)


def coefficients(z):
    """alpha, beta, gamma and the diagonals of Z1, Z2, Z3 from z = (..., 3)."""
    z = np.asarray(z, dtype=np.float64)
    z1, z2, z3 = z[..., 0], z[..., 1], z[..., 2]
    alpha = z1 + z2 + z3
    beta = z1 * z2 + z2 * z3 + z3 * z1
    gamma = z1 * z2 * z3
    Z1 = -z
    Z2 = alpha[..., None] - 2.0 * z
    Z3 = np.stack([z2 * z3, z3 * z1, z1 * z2], axis=-1)
    return alpha, beta, gamma, Z1, Z2, Z3


def box_zeta(box, thickness, R):
    """Nodal z_i (ndof_box, 3) of a box with PML layers of the given per-face thickness (R23)."""
    xyz = box.node_coords()
    z = np.zeros_like(xyz)
    for f in range(6):
        ell = float(thickness[f])
        if ell <= 0.0:
            continue
        d_ax, side = f // 2, f % 2
        lo, hi = box.origin[d_ax], box.origin[d_ax] + box.extent[d_ax]
        dist = (xyz[:, d_ax] - (hi - ell)) if side else ((lo + ell) - xyz[:, d_ax])
        z[:, d_ax] += damping_profile(dist, ell, zeta_tilde(box.c, ell, R))
    return z


class Pml:
    """PML auxiliaries of one box: nodal coefficients, element-local Phi, and one R25 update."""

    def __init__(self, system, spec):
        from .operators import _lattice_pts, _shape_key, ref_gradients
        from .mesh import jacobian

        self.sys = system
        bi = int(spec["box"])
        box = system.boxes[bi]
        thick = np.asarray(spec["thickness"], dtype=np.float64)
        for d in range(3):
            if thick[2 * d] + thick[2 * d + 1] > box.extent[d] * (1 + 1e-12):
                raise ValueError("PML layers overlap")
        self.box, self.bi, self.c = box, bi, box.c
        off = int(system.offsets[bi])
        zb = box_zeta(box, thick, float(spec["R"]))
        n = system.ndof
        self.zeta = np.zeros((n, 3))
        self.zeta[off:off + box.ndof] = zb
        self.alpha, self.beta, self.gamma, _, _, _ = coefficients(self.zeta)
        conn = box.connectivity() + off
        el = np.nonzero(np.any(self.zeta[conn].sum(axis=2) > 0.0, axis=1))[0]   # elements touching z > 0
        self.elems = el
        self.conn = conn[el]
        # element gradient (G[q, i, d] = d_d phi_i(x_q)) and weak-divergence (W[q] = w_q |J_q|) operators
        # by brute force at the element's GLL nodes; identical element shapes share them
        x, w, a, b, c = _lattice_pts(box.N)
        xi = np.stack([x[a], x[b], x[c]], axis=1)
        wq = w[a] * w[b] * w[c]
        _, ghat = ref_gradients(box.N, xi)
        cache = {}
        self.G, self.W = [], []
        for e in el:
            v = box.vertices(e)
            k = _shape_key(v)
            if k not in cache:
                J = jacobian(v, xi)
                G = np.einsum("qid,qde->qie", ghat, np.linalg.inv(J))
                cache[k] = (G, wq * np.abs(np.linalg.det(J)))
            self.G.append(cache[k][0])
            self.W.append(cache[k][1])
        nl = (box.N + 1) ** 3
        self.psi = np.zeros(n)                           # psi^{n+1/2}
        self.phi = np.zeros((len(el), nl, 3))            # Phi^{n+1/2} per element node

    def advance(self, p1, dt):
        """One R25 update at t^{n+1}: returns (B^T Phi^{n+1}, psi^{n+1}) and commits the half-step state."""
        psi_new = self.psi + dt * p1
        psi_mid = 0.5 * (self.psi + psi_new)
        rB = np.zeros(self.sys.ndof)
        c2 = self.c * self.c
        for k in range(len(self.elems)):
            ids = self.conn[k]
            G, W = self.G[k], self.W[k]
            gp = np.einsum("qid,i->qd", G, p1[ids])          # grad p^{n+1} at the element's nodes
            gs = np.einsum("qid,i->qd", G, psi_mid[ids])     # grad psi^{n+1}
            z = self.zeta[ids]
            _, _, _, _, Z2, Z3 = coefficients(z)
            old = self.phi[k]
            new = ((1.0 - 0.5 * dt * z) * old + dt * c2 * (Z2 * gp + Z3 * gs)) / (1.0 + 0.5 * dt * z)
            mid = 0.5 * (old + new)
            self.phi[k] = new
            rB[ids] += np.einsum("q,qid,qd->i", W, G, mid)    # sum_q w_q |J| Phi . grad phi_i
        self.psi = psi_new
        return rB, psi_mid

    def weak_divergence(self, phi_elem):
        """(B^T Phi)_i for a given element-local field phi_elem (n_pml_el, n_loc, 3) (for pins)."""
        rB = np.zeros(self.sys.ndof)
        for k in range(len(self.elems)):
            rB[self.conn[k]] += np.einsum("q,qid,qd->i", self.W[k], self.G[k], phi_elem[k])
        return rB

    def element_gradient(self, f):
        """Element-local gradient of a nodal field at every PML element node (n_pml_el, n_loc, 3)."""
        return np.stack([np.einsum("qid,i->qd", self.G[k], f[self.conn[k]]) for k in range(len(self.elems))])
