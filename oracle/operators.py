"""Discrete operators of Eqs. (6)-(12) by brute-force quadrature (oracle; test infrastructure only).

* Volume stiffness (Eq. 7, first sum):
      K_e[i, j] = sum_q w_q |det J_q| c^2 (grad phi_i . grad phi_j)(xi_q)
  on the (N+1)^3 GLL rule, grad phi = grad_hat phi . J^{-1}, from the trilinear map of each
  element.  Elements of identical shape share one cached K_e (still computed by quadrature).
* Mass (Eq. 6): lumped M_ii = sum_e w_i |det J(xi_i)| (reduced integration).
* ABC (Eq. 8): C_ii = sum_{F in F_ABC} c w_s w_t |J_s|  (GLL-collocated, diagonal).
* PMUT coupling (Eqs. 11-12): B_{k,m,j} = sum_{F on gamma_k} w_s w_t |J_s| S_{k,m}(x_j)
  with U_{k,m}.n = -S_{k,m} on the -z face (reading R4), so
      int p U.n = -B p      and     f = -kappa sum_m qdd_m int U_m.n psi = +kappa B^T qdd.
* SIPG interface (Eq. 7, three Gamma_I sums), written out per fine face F:
      K_F[i, j] = sum_q W_q [ -{c^2 grad phi_j}.[[phi_i]] - {c^2 grad phi_i}.[[phi_j]]
                              + gamma_F [[phi_i]].[[phi_j]] ]
  with [[u]] = u+ n+ + u- n-, {v} = (v+ + v-)/2, quadrature at the fine face's GLL
  nodes x_q (reading R9), x_hat_q^- by Newton on the coarse trilinear map after a
  bounding-box filter (the spirit of Algorithm 3's radius filter), and
      gamma_F = alpha cbar^2 max(r+, r-)^2 / min(h+, h-),  cbar = harmonic mean of c,
  h = smallest element edge (reading R7).
"""
from __future__ import annotations

import math

import numpy as np

from .gll import basis_matrix, deriv_matrix, gll
from .mesh import Box, face_local_nodes, inverse_map, jacobian, map_point

BC_ABSORBING, BC_INTERFACE = 1, 2


def _lattice_pts(N):
    x, w = gll(N)
    n1 = N + 1
    c, b, a = np.meshgrid(np.arange(n1), np.arange(n1), np.arange(n1), indexing="ij")
    a, b, c = a.ravel(), b.ravel(), c.ravel()
    return x, w, a, b, c


def ref_gradients(N, xi_pts):
    """Reference basis values and gradients of the (N+1)^3 tensor basis at arbitrary points.
    xi_pts (nq, 3) -> phi (nq, n_loc), ghat (nq, n_loc, 3); local i = a + (N+1)(b + (N+1)c)."""
    x, _ = gll(N)
    n1 = N + 1
    L = [basis_matrix(x, xi_pts[:, d]) for d in range(3)]     # (nq, n1)
    D = [deriv_matrix(x, xi_pts[:, d]) for d in range(3)]
    nq = xi_pts.shape[0]

    def tens(fx, fy, fz):
        return np.einsum("qc,qb,qa->qcba", fz, fy, fx).reshape(nq, n1 ** 3)

    phi = tens(L[0], L[1], L[2])
    ghat = np.stack([tens(D[0], L[1], L[2]), tens(L[0], D[1], L[2]), tens(L[0], L[1], D[2])], axis=-1)
    return phi, ghat


def element_stiffness(verts, N, c):
    """K_e by brute-force GLL quadrature on the trilinear element with vertices ``verts``."""
    x, w, a, b, cc = _lattice_pts(N)
    xi = np.stack([x[a], x[b], x[cc]], axis=1)
    wq = w[a] * w[b] * w[cc]
    _, ghat = ref_gradients(N, xi)
    J = jacobian(verts, xi)                                   # (nq, 3, 3)
    Jinv = np.linalg.inv(J)
    det = np.abs(np.linalg.det(J))
    gphys = np.einsum("qid,qde->qie", ghat, Jinv)
    return np.einsum("q,qie,qje->ij", wq * det * c * c, gphys, gphys)


def element_mass(verts, N):
    """Lumped element mass: w_q |det J(xi_q)| at the collocated node q."""
    x, w, a, b, cc = _lattice_pts(N)
    xi = np.stack([x[a], x[b], x[cc]], axis=1)
    return w[a] * w[b] * w[cc] * np.abs(np.linalg.det(jacobian(verts, xi)))


def face_quadrature(verts, N, face, rule="gll"):
    """Per face quadrature point: local id (GLL rule: the collocated face node; LG: None), reference
    point, physical point, weight w_s w_t |J_s|, outward normal.  rule "gll": the face's (N+1)^2 GLL
    nodes (reading R9); "lg": the (N+1)^2 Gauss-Legendre points of the same face (R9's flag, Fig. 7's
    "LG" nodes)."""
    x, w = gll(N)
    ids, st, tang = face_local_nodes(N, face)
    if rule == "lg":
        x, w = np.polynomial.legendre.leggauss(N + 1)
    elif rule != "gll":
        raise ValueError(f"unknown face rule {rule!r}")
    d, side = face // 2, face % 2
    xi = np.zeros((len(ids), 3))
    xi[:, d] = 1.0 if side else -1.0
    xi[:, tang[0]] = x[st[:, 0]]
    xi[:, tang[1]] = x[st[:, 1]]
    J = jacobian(verts, xi)
    cr = np.cross(J[:, :, tang[0]], J[:, :, tang[1]])
    js = np.linalg.norm(cr, axis=1)
    n = cr / js[:, None]
    pts = map_point(verts, xi)
    centroid = verts.mean(axis=0)
    sgn = np.sign(np.einsum("qd,qd->q", n, pts - centroid[None, :]))
    n = n * sgn[:, None]
    return (ids if rule == "gll" else None), xi, pts, w[st[:, 0]] * w[st[:, 1]] * js, n


def _shape_key(verts):
    return tuple(np.round((verts - verts[0]) / max(np.ptp(verts), 1e-300) * 1e12).astype(np.int64).ravel())


def penalty_gamma(c_plus, c_minus, r_in, r_out, h_in, h_out, alpha):
    """gamma_F = alpha cbar^2 max(r_in, r_out)^2 / min(h_in, h_out), cbar = 2 c+ c- / (c+ + c-)."""
    cbar = 2.0 * c_plus * c_minus / (c_plus + c_minus)
    return alpha * cbar * cbar * max(r_in, r_out) ** 2 / min(h_in, h_out)


def mode_shape(pm, k, m, x, y):
    """S_{k,m}(x, y) = sin(m pi x'/a) sin(n pi y'/a) on the square membrane, 0 outside (reading R19).
    With pm["shape_fn"] (an input: the paper's U_{k,m} are FEM eigenmodes; reading R33)
    S_{k,m}(x, y) = shape_fn(k, m, x - cx, y - cy) inside the membrane's bounding square, 0 outside."""
    a = pm["side"]
    cx, cy = pm["centers"][k]
    mm, nn = pm["mode_mn"][m]
    xl = x - (cx - a / 2)
    yl = y - (cy - a / 2)
    inside = (xl >= 0) & (xl <= a) & (yl >= 0) & (yl <= a)
    if pm.get("shape_fn") is not None:
        s = np.array([pm["shape_fn"](k, m, float(xv - cx), float(yv - cy)) for xv, yv in zip(x, y)], dtype=np.float64)
        return np.where(inside, s, 0.0)
    return np.where(inside, np.sin(mm * math.pi * xl / a) * np.sin(nn * math.pi * yl / a), 0.0)


class System:
    """Assembled (matrix-free by element) DG-SEM system of Eqs. (9)-(12) for one workload record."""

    def __init__(self, rec):
        self.rec = rec
        self.boxes = [Box(b) for b in rec["boxes"]]
        self.offsets = np.cumsum([0] + [b.ndof for b in self.boxes])
        self.ndof = int(self.offsets[-1])
        self._build_volume()
        # nodes of the fluid (every node when there is no obstacle): the others have no mass, no
        # stiffness row and stay 0
        self.active = self.M > 0
        self._build_abc()
        self._build_pmut(rec.get("pmut"))
        self._build_interface(rec.get("interface"))
        self._build_plane_wave(rec.get("plane_wave"))

    # ----------------------------------------------------------------- volume
    def _build_volume(self):
        self.vol = []
        self.M = np.zeros(self.ndof)
        for bi, box in enumerate(self.boxes):
            conn = box.connectivity() + self.offsets[bi]
            cache = {}
            keys = np.empty(box.nelem, dtype=np.int64)
            for e in range(box.nelem):
                if box.solid[e]:          # obstacle element: not part of the fluid (nothing assembled)
                    keys[e] = -1
                    continue
                v = box.vertices(e)
                k = _shape_key(v)
                if k not in cache:
                    cache[k] = (len(cache), element_stiffness(v, box.N, box.c), element_mass(v, box.N))
                keys[e] = cache[k][0]
            mats = sorted(cache.values(), key=lambda m: m[0])
            for kid, Ke, Me in mats:
                sel = np.nonzero(keys == kid)[0]
                np.add.at(self.M, conn[sel].ravel(), np.tile(Me, len(sel)))
                self.vol.append((conn[sel], Ke))

    def apply_volume(self, p):
        """r = sum_e P_e^T K_e P_e p: element products, then one scatter-add of every element's
        contributions (a single bincount: one pass over the global vector however many shape groups)."""
        idx, val = [], []
        for conn, Ke in self.vol:
            idx.append(conn.ravel())
            val.append((p[conn] @ Ke.T).ravel())
        if not idx:
            return np.zeros(self.ndof)
        return np.bincount(np.concatenate(idx), np.concatenate(val), minlength=self.ndof)

    # ------------------------------------------------------------------- ABC
    def _build_abc(self):
        self.C = np.zeros(self.ndof)
        for bi, box in enumerate(self.boxes):
            for face in range(6):
                if box.bc[face] != BC_ABSORBING:
                    continue
                conn = box.connectivity() + self.offsets[bi]
                for e in box.fluid_boundary_faces(face):
                    ids, _, _, wq, _ = face_quadrature(box.vertices(e), box.N, face)
                    np.add.at(self.C, conn[e, ids], box.c * wq)

    # ------------------------------------------------------------------ PMUTs
    def _build_pmut(self, pm):
        self.pm = pm
        if pm is None:
            return
        box = self.boxes[pm["box"]]
        off = self.offsets[pm["box"]]
        conn = box.connectivity() + off
        face = pm["face"]
        n_p, n_m = len(pm["centers"]), len(pm["mode_mn"])
        acc = [dict() for _ in range(n_p)]
        cen = np.asarray(pm["centers"], dtype=np.float64)
        half = 0.5 * pm["side"]
        for e in box.boundary_faces(face):
            ids, _, pts, wq, _ = face_quadrature(box.vertices(e), box.N, face)
            g = conn[e, ids]
            # only membranes whose square meets the face's bounding box can have S != 0 on it
            lo, hi = pts[:, :2].min(axis=0), pts[:, :2].max(axis=0)
            near = np.nonzero(np.all((cen + half >= lo) & (cen - half <= hi), axis=1))[0]
            for k in near:
                for m in range(n_m):
                    s = mode_shape(pm, k, m, pts[:, 0], pts[:, 1])
                    for j, val in zip(g[s != 0], (wq * s)[s != 0]):
                        acc[k].setdefault(int(j), np.zeros(n_m))[m] += val
        self.B = []
        for k in range(n_p):
            idx = np.array(sorted(acc[k]), dtype=np.int64)
            vals = np.stack([acc[k][j] for j in idx], axis=1) if len(idx) else np.zeros((n_m, 0))
            self.B.append((idx, vals))
        self.kappa = box.rho * box.c ** 2            # kappa = rho c^2

    def pmut_project(self, p):
        """G[k, m] = sum_j B_{k,m,j} p_j   (so int_gamma_k p U_{k,m}.n = -G)."""
        return np.stack([vals @ p[idx] for idx, vals in self.B])

    def pmut_force(self, qdd):
        """f_i = -kappa sum_{k,m} qdd_{k,m} int U_{k,m}.n psi_i = +kappa sum B_{k,m,i} qdd_{k,m}  (Eq. 11)."""
        f = np.zeros(self.ndof)
        for (idx, vals), qk in zip(self.B, qdd):
            f[idx] += self.kappa * (qk @ vals)
        return f

    # -------------------------------------------------------------- interface
    def _build_interface(self, itf):
        self.iface = []
        self.gamma_F = None
        if itf is None:
            return
        fb, cb = itf["fine_box"], itf["coarse_box"]
        F, Cx = self.boxes[fb], self.boxes[cb]
        connF = F.connectivity() + self.offsets[fb]
        connC = Cx.connectivity() + self.offsets[cb]
        gam = penalty_gamma(F.c, Cx.c, F.N, Cx.N, float(F.h.min()), float(Cx.h.min()), itf["alpha"])
        self.gamma_F = gam
        cands = Cx.boundary_faces(4)                              # coarse -z faces
        cverts = np.stack([Cx.vertices(e) for e in cands])         # (nc, 8, 3)
        lo, hi = cverts.min(axis=1), cverts.max(axis=1)
        tol = 1e-9 * float(np.max(Cx.h))
        groups = {}
        rule = itf.get("quad", "gll")
        for e in F.boundary_faces(5):                             # fine +z faces
            vF = F.vertices(e)
            _, xiq, pts, wq, nrm = face_quadrature(vF, F.N, 5, rule)
            owners, xim = [], []
            for q in range(len(xiq)):
                inbox = np.nonzero(np.all((pts[q] >= lo - tol) & (pts[q] <= hi + tol), axis=1))[0]
                found = None
                for ci in inbox:                                  # lowest id first (tie-break)
                    xi = inverse_map(cverts[ci], pts[q])
                    if np.max(np.abs(xi)) <= 1 + 1e-9:
                        found = (ci, xi)
                        break
                if found is None:
                    raise RuntimeError("orphan interface quadrature point")
                owners.append(found[0])
                xim.append(found[1])
            uniq = sorted(set(owners))
            # identical relative geometry => identical face matrix (cache; still computed literally)
            key = (_shape_key(vF),
                   tuple(tuple(np.round((cverts[u] - vF[0]) / tol).astype(np.int64).ravel()) for u in uniq),
                   tuple(uniq.index(o) for o in owners))
            dofs = np.concatenate([connF[e]] + [connC[cands[u]] for u in uniq])
            if key not in groups:
                KF = self._face_matrix(F, Cx, vF, [cverts[u] for u in uniq], owners, uniq, np.array(xim),
                                       xiq, wq, nrm, gam)
                groups[key] = (KF, [])
            groups[key][1].append(dofs)
        for KF, dl in groups.values():
            self.iface.append((np.stack(dl), KF))

    @staticmethod
    def _face_matrix(F, Cx, vF, cvs, owners, uniq, xim, xi_p, wq, nrm, gam):
        nF = (F.N + 1) ** 3
        nC = (Cx.N + 1) ** 3
        nd = nF + nC * len(uniq)
        # fine side: basis values / gradients at the reference points xi_p of the quadrature points
        phiF, ghF = ref_gradients(F.N, xi_p)
        JF = np.linalg.inv(jacobian(vF, xi_p))
        gF = np.einsum("qid,qde->qie", ghF, JF)
        KF = np.zeros((nd, nd))
        for q in range(len(xi_p)):
            phi = np.zeros(nd)
            dn = np.zeros(nd)          # c^2 grad phi . n+  (own side's c)
            sgn = np.zeros(nd)
            phi[:nF] = phiF[q]
            dn[:nF] = F.c ** 2 * gF[q] @ nrm[q]
            sgn[:nF] = 1.0
            u = uniq.index(owners[q])
            xq = xim[q][None, :]
            phiC, ghC = ref_gradients(Cx.N, xq)
            gC = np.einsum("qid,qde->qie", ghC, np.linalg.inv(jacobian(cvs[u], xq)))
            sl = slice(nF + u * nC, nF + (u + 1) * nC)
            phi[sl] = phiC[0]
            dn[sl] = Cx.c ** 2 * gC[0] @ nrm[q]
            sgn[sl] = -1.0                                # [[phi]] = phi+ n+ + phi- n-, n- = -n+
            jump = sgn * phi                               # [[phi_i]] . n+
            avg = 0.5 * dn                                 # {c^2 grad phi_i} . n+
            KF += wq[q] * (-np.outer(jump, avg) - np.outer(avg, jump) + gam * np.outer(jump, jump))
        return KF

    def apply_interface(self, p):
        idx, val = [], []
        for dofs, KF in self.iface:
            idx.append(dofs.ravel())
            val.append((p[dofs] @ KF.T).ravel())
        if not idx:
            return np.zeros(self.ndof)
        return np.bincount(np.concatenate(idx), np.concatenate(val), minlength=self.ndof)

    def apply_K(self, p):
        r = self.apply_volume(p)
        if self.iface:
            r += self.apply_interface(p)
        return r

    # ------------------------------------------------------------ plane wave
    def _build_plane_wave(self, pw):
        self.pw = pw
        if pw is None:
            return
        box = self.boxes[pw["box"]]
        conn = box.connectivity() + self.offsets[pw["box"]]
        face = pw["face"]
        w = {}
        xyz = {}
        nrm = None
        for e in box.boundary_faces(face):
            ids, _, pts, wq, n = face_quadrature(box.vertices(e), box.N, face)
            nrm = n[0]
            for j, p_, ww in zip(conn[e, ids], pts, wq):
                w[int(j)] = w.get(int(j), 0.0) + ww
                xyz[int(j)] = p_
        self.pw_idx = np.array(sorted(w), dtype=np.int64)
        self.pw_w = np.array([w[j] for j in self.pw_idx])
        self.pw_xyz = np.stack([xyz[j] for j in self.pw_idx])
        kd = np.asarray(pw["direction"], dtype=np.float64)
        # reference point: the face corner the wavefront reaches first (min k.x), reading R13
        corners = np.array([[x, y, self.pw_xyz[0, 2]] for x in (self.pw_xyz[:, 0].min(), self.pw_xyz[:, 0].max())
                            for y in (self.pw_xyz[:, 1].min(), self.pw_xyz[:, 1].max())])
        # a lateral crop of a larger box (tests) passes the full box's reference corner explicitly
        self.pw_xref = (np.asarray(pw["x_ref"], dtype=np.float64) if pw.get("x_ref") is not None
                        else corners[np.argmin(corners @ kd)])
        self.pw_k = kd
        self.pw_n = nrm
        self.pw_c = box.c

    def plane_wave_load(self, t):
        """b_j = int c A s'(tau(x)) (1 - n.k) psi_j  -- total-field first-order ABC with incident
        plane wave p_inc = A s(t - k.(x - x_ref)/c) (reading R13)."""
        b = np.zeros(self.ndof)
        if self.pw is None:
            return b
        pw = self.pw
        tau = t - (self.pw_xyz - self.pw_xref) @ self.pw_k / self.pw_c
        u = tau - pw["t0_s"]
        sig = pw["sigma_s"]
        om = 2 * math.pi * pw["f0_hz"]
        env = np.exp(-u * u / (2 * sig * sig))
        ds = env * (-u / (sig * sig) * np.sin(om * u) + om * np.cos(om * u))
        b[self.pw_idx] = self.pw_c * pw["amp_pa"] * ds * (1.0 - float(self.pw_n @ self.pw_k)) * self.pw_w
        return b

    # ------------------------------------------------------------- utilities
    def split(self, v):
        return [v[self.offsets[i]:self.offsets[i + 1]] for i in range(len(self.boxes))]

    def node_coords(self):
        return np.concatenate([b.node_coords() for b in self.boxes])
