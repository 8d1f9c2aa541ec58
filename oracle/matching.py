"""Algorithm 3 (face matching on the non-conforming interface) for the oracle
(TEST INFRASTRUCTURE ONLY).

The interface faces F are defined by the quadrature nodes of the finer side: for every
fine face dK+ and every quadrature node x_q = X_{K+}(xhat_q+) the coarse face dK- that
contains x_q is searched (Algorithm 3):

    for dK+ on Gamma_I:  for x_q, q = 1..N_q:  for dK- on Gamma_I:
        if |n+ + n-| < tol  and  V_{K-} in C_r(x_q):                  (normal filter, one-vertex radius
            xhat_q- = X_{K-}^{-1}(x_q)  (Newton-Raphson)        filter, r = max(diam dK-, diam dK+)
            if xhat_q- in [-1, 1]^3:  K- is the neighbour               + eps)

Readings (R26): the quadrature nodes are the fine face's GLL nodes (reading R9); n+- are the
outward unit normals at the face centres; V_{K-} is the face's first vertex (lowest local vertex
index); "in [-1,1]^3" is tested with a 1e-9 tolerance and the first matching coarse face in index
order is taken (a node on a coarse edge belongs to the lowest-index face containing it).
"""
from __future__ import annotations

import numpy as np

from .gll import gll
from .mesh import REF_VERTS, inverse_map, jacobian, map_point

FACE_VERTS = [[v for v in range(8) if ((REF_VERTS[v, f // 2] > 0) == bool(f % 2))] for f in range(6)]


def face_center_normal(verts, face):
    """Outward unit normal of local face ``face`` of the trilinear element at the face centre."""
    d, side = face // 2, face % 2
    xi = np.zeros(3)
    xi[d] = 1.0 if side else -1.0
    J = jacobian(verts, xi)
    t = [e for e in range(3) if e != d]
    n = np.cross(J[:, t[0]], J[:, t[1]])
    n /= np.linalg.norm(n)
    c = map_point(verts, xi)
    if (c - verts.mean(axis=0)) @ n < 0:
        n = -n
    return n


def face_diameter(verts, face):
    fv = verts[FACE_VERTS[face]]
    return max(np.linalg.norm(a - b) for a in fv for b in fv)


def face_quad_points(verts, face, N):
    """Physical GLL nodes x_q = X_K(xhat_q) of the face (s fastest), and the reference points."""
    x, _ = gll(N)
    d, side = face // 2, face % 2
    t = [e for e in range(3) if e != d]
    pts, ref = [], []
    for b in range(N + 1):
        for a in range(N + 1):
            xi = np.zeros(3)
            xi[d] = 1.0 if side else -1.0
            xi[t[0]], xi[t[1]] = x[a], x[b]
            ref.append(xi)
            pts.append(map_point(verts, xi))
    return np.array(pts), np.array(ref)


def match_faces(fine, coarse, N, tol=1e-6, eps=1e-12):
    """Algorithm 3 literally.  fine / coarse: lists of (verts (8,3), local face).  Returns
    owner[f, q] (index into ``coarse``, -1 if unmatched) and xi[f, q, :] (xhat_q- in the owner)."""
    cn = [face_center_normal(v, f) for v, f in coarse]
    cd = [face_diameter(v, f) for v, f in coarse]
    cV = [v[FACE_VERTS[f][0]] for v, f in coarse]
    nq = (N + 1) ** 2
    owner = np.full((len(fine), nq), -1, dtype=np.int64)
    xis = np.zeros((len(fine), nq, 3))
    for i, (vf, ff) in enumerate(fine):
        npl = face_center_normal(vf, ff)
        df = face_diameter(vf, ff)
        pts, _ = face_quad_points(vf, ff, N)
        for q in range(nq):
            for j, (vc, fc) in enumerate(coarse):
                r = max(cd[j], df) + eps
                if np.linalg.norm(npl + cn[j]) < tol and np.linalg.norm(cV[j] - pts[q]) < r:
                    xi = inverse_map(vc, pts[q])
                    if np.max(np.abs(xi)) <= 1.0 + 1e-9:
                        owner[i, q] = j
                        xis[i, q] = xi
                        break
    return owner, xis
