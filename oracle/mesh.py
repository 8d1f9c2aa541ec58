"""Structured hexahedral boxes for the oracle (test infrastructure only).

P:L413-420: T_h = T_in U T_out of hexahedra, each the image of [-1,1]^3 under a
trilinear map X_K with positive Jacobian; face sets F^I (interface) and F^B
(Neumann / ABC / PMUT).  P:L539-547: V_a^{r_a} is continuous inside each region
(one global id per lattice point of a box), discontinuous across Gamma_I (the two
boxes are numbered separately and never merged).

Global ids inside a box are lexicographic, x fastest:
    id(gx, gy, gz) = gx + NX * (gy + NY * gz),  NX = N*nel_x + 1, ...
which is the output layout of ``sem_read_pressure``; element (ex, ey, ez) local
node (a, b, c) is lattice point (N ex + a, N ey + b, N ez + c).
"""
from __future__ import annotations

import itertools

import numpy as np

from .gll import gll

# reference vertices of [-1,1]^3 in the order v = i + 2 j + 4 k
REF_VERTS = np.array([[2 * i - 1, 2 * j - 1, 2 * k - 1]
                      for k in (0, 1) for j in (0, 1) for i in (0, 1)], dtype=np.float64)


def trilinear_shape(xi):
    """N_v(xi) for the 8 vertices, xi of shape (..., 3) -> (..., 8)."""
    xi = np.asarray(xi, dtype=np.float64)
    s = 1.0 + xi[..., None, :] * REF_VERTS          # (..., 8, 3)
    return np.prod(s, axis=-1) / 8.0


def trilinear_grad(xi):
    """dN_v/dxi_d, shape (..., 8, 3)."""
    xi = np.asarray(xi, dtype=np.float64)
    s = 1.0 + xi[..., None, :] * REF_VERTS          # (..., 8, 3)
    g = np.empty(s.shape)
    for d in range(3):
        others = [e for e in range(3) if e != d]
        g[..., d] = REF_VERTS[:, d] * s[..., others[0]] * s[..., others[1]] / 8.0
    return g


def map_point(verts, xi):
    """X_K(xi) = sum_v N_v(xi) X_v.  verts (8,3), xi (...,3)."""
    return trilinear_shape(xi) @ verts


def jacobian(verts, xi):
    """J[i, j] = dX_i / dxi_j at xi, shape (..., 3, 3)."""
    g = trilinear_grad(xi)                         # (..., 8, 3)
    return np.einsum("vi,...vj->...ij", verts, g)


def inverse_map(verts, x, tol=1e-14, maxit=50):
    """Newton for X_K(xi) = x (x_hat_q^- = X_{K^-}^{-1}(x_q))."""
    xi = np.zeros(3)
    for _ in range(maxit):
        r = x - map_point(verts, xi)
        dxi = np.linalg.solve(jacobian(verts, xi), r)
        xi = xi + dxi
        if np.max(np.abs(dxi)) < tol:
            break
    return xi


class Box:
    """One structured hex box of degree-N GLL elements."""

    def __init__(self, desc):
        self.desc = desc
        self.N = int(desc["degree"])
        self.nel = tuple(int(v) for v in desc["nel"])
        self.origin = np.asarray(desc["origin"], dtype=np.float64)
        self.extent = np.asarray(desc["extent"], dtype=np.float64)
        self.c = float(desc["c"])
        self.rho = float(desc["rho"])
        self.bc = list(desc["bc"])
        self.nodes1d, self.weights1d = gll(self.N)
        self.nn = tuple(self.N * n + 1 for n in self.nel)
        self.ndof = self.nn[0] * self.nn[1] * self.nn[2]
        self.nelem = self.nel[0] * self.nel[1] * self.nel[2]
        self.h = self.extent / np.asarray(self.nel, dtype=np.float64)
        v = desc.get("vertices")
        self.vlat = None if v is None else np.asarray(v, dtype=np.float64).reshape(-1, 3)
        if self.vlat is not None and len(self.vlat) != (self.nel[0] + 1) * (self.nel[1] + 1) * (self.nel[2] + 1):
            raise ValueError("vertex lattice size mismatch")
        # obstacle: "solid" elements are removed from the fluid domain Omega, so
        # their faces towards the fluid are Neumann (rigid) surfaces: the natural boundary condition of
        # the weak form (Eq. 4 with no boundary term) -- nothing is assembled for them.
        sol = desc.get("solid")
        self.solid = np.zeros(self.nelem, dtype=bool)
        if sol is not None:
            sol = np.asarray(sol)
            if sol.dtype == bool:
                if sol.shape != (self.nelem,):
                    raise ValueError("solid mask size mismatch")
                self.solid = sol.copy()
            else:
                self.solid[sol.astype(np.int64)] = True

    # --- lattice / numbering -------------------------------------------------
    def gid(self, gx, gy, gz):
        return gx + self.nn[0] * (gy + self.nn[1] * gz)

    def elem_index(self, ex, ey, ez):
        return ex + self.nel[0] * (ey + self.nel[1] * ez)

    def elem_coords(self, e):
        ex = e % self.nel[0]
        ey = (e // self.nel[0]) % self.nel[1]
        ez = e // (self.nel[0] * self.nel[1])
        return ex, ey, ez

    def local_lattice(self):
        """(a, b, c) for local node i = a + (N+1)(b + (N+1) c)."""
        n1 = self.N + 1
        return np.array([(a, b, c) for c in range(n1) for b in range(n1) for a in range(n1)])

    def connectivity(self):
        """conn[e, i] = global id of local node i of element e (e = ex + nel_x (ey + nel_y ez))."""
        loc = self.local_lattice()
        e = np.arange(self.nelem)
        ex, ey, ez = self.elem_coords(e)
        return self.gid(self.N * ex[:, None] + loc[None, :, 0], self.N * ey[:, None] + loc[None, :, 1],
                        self.N * ez[:, None] + loc[None, :, 2]).astype(np.int64)

    def vertices(self, e):
        """The 8 physical vertices of element e (order v = i + 2j + 4k).  A box with a "vertices"
        lattice [(nel_x+1)(nel_y+1)(nel_z+1), 3] (x fastest) is a logically structured, geometrically
        trilinear (curved) mesh; otherwise the vertices are the affine lattice."""
        ex, ey, ez = self.elem_coords(e)
        if self.vlat is not None:
            nx, ny = self.nel[0] + 1, self.nel[1] + 1
            idx = [(ex + i) + nx * ((ey + j) + ny * (ez + k)) for k in (0, 1) for j in (0, 1) for i in (0, 1)]
            return self.vlat[idx]
        lo = self.origin + self.h * np.array([ex, ey, ez], dtype=np.float64)
        return lo[None, :] + (REF_VERTS + 1.0) / 2.0 * self.h[None, :]

    def node_coords(self):
        """Physical coordinates of every global node, via the trilinear map of an owning element."""
        xyz = np.empty((self.ndof, 3))
        loc = self.local_lattice()
        xi = self.nodes1d[loc]                      # (n_loc, 3)
        conn = self.connectivity()
        for e in range(self.nelem):
            xyz[conn[e]] = map_point(self.vertices(e), xi)
        return xyz

    def boundary_faces(self, face):
        """Elements touching box face ``face`` (0..5 = -x,+x,-y,+y,-z,+z), ascending ids."""
        d, side = face // 2, face % 2
        ec = self.elem_coords(np.arange(self.nelem))[d]
        return list(np.nonzero(ec == (self.nel[d] - 1 if side else 0))[0])

    def fluid_boundary_faces(self, face):
        """boundary_faces(face) without the solid (obstacle) elements."""
        return [e for e in self.boundary_faces(face) if not self.solid[e]]


def face_local_nodes(N, face):
    """Local node ids (a + (N+1)(b + (N+1)c)) on element face ``face`` and their 2D (s,t) indices."""
    n1 = N + 1
    d, side = face // 2, face % 2
    fixed = N if side else 0
    tang = [e for e in range(3) if e != d]
    ids, st = [], []
    for t, s in itertools.product(range(n1), range(n1)):
        abc = [0, 0, 0]
        abc[d] = fixed
        abc[tang[0]] = s
        abc[tang[1]] = t
        ids.append(abc[0] + n1 * (abc[1] + n1 * abc[2]))
        st.append((s, t))
    return np.array(ids), np.array(st), tang
