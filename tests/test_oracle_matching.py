"""Pins for oracle.matching (Algorithm 3; reading R26): the structured 2:1 closed form
and, on jittered (trilinear) interfaces, an independent point-in-quadrilateral test plus the round trip
X_{K-}(xhat-) = x_q."""
import numpy as np
import pytest

from oracle.gll import gll
from oracle.matching import FACE_VERTS, face_quad_points, match_faces
from oracle.mesh import map_point
from sem_inputs import interface_faces


@pytest.mark.parametrize("N,R", [(5, 2), (3, 3)])
def test_structured_closed_form(N, R):
    """Unperturbed R:1 lattice: fine node x = (i + (xi_a + 1)/2) h_f lies in coarse element
    floor(x / h_c) (the lower-index element on a shared edge) at xhat- = (2 r + xi_a + 1)/R - 1
    (r = fine element offset inside the coarse one); the same in y; xhat-_z = -1."""
    nfx, nfy, hf = 2 * R, R, 25e-6
    fine, coarse = interface_faces(nfx, nfy, R, hf)
    own, xi = match_faces(fine, coarse, N)
    x, _ = gll(N)
    ncx = nfx // R
    for f, (v, _) in enumerate(fine):
        i, j = f % nfx, f // nfx
        for q in range(own.shape[1]):
            a, b = q % (N + 1), q // (N + 1)
            ex, ry, ey = i // R, j % R, j // R
            rx = i % R
            if a == 0 and rx == 0 and ex > 0:          # on a coarse edge: lower-index element
                ex, rx, xa = ex - 1, R - 1, 1.0
            else:
                xa = x[a]
            if b == 0 and ry == 0 and ey > 0:
                ey, ry, xb = ey - 1, R - 1, 1.0
            else:
                xb = x[b]
            assert own[f, q] == ex + ncx * ey, (f, q)
            ref = [(2 * rx + xa + 1) / R - 1, (2 * ry + xb + 1) / R - 1, -1.0]
            assert np.max(np.abs(xi[f, q] - ref)) < 1e-12


def _in_quad(p, quad):
    """2D point-in-convex-quadrilateral (boundary inclusive) by edge cross products."""
    s = []
    for k in range(4):
        a, b = quad[k], quad[(k + 1) % 4]
        s.append((b[0] - a[0]) * (p[1] - a[1]) - (b[1] - a[1]) * (p[0] - a[0]))
    s = np.array(s)
    scale = np.max(np.abs(quad)) ** 2
    return bool(np.all(s >= -1e-9 * scale) or np.all(s <= 1e-9 * scale))


def test_jittered_interface_containment_and_round_trip():
    fine, coarse = interface_faces(6, 4, 2, 25e-6, jitter=0.15, seed=3)
    N = 4
    own, xi = match_faces(fine, coarse, N)
    assert np.all(own >= 0)
    for f, (v, face) in enumerate(fine):
        pts, _ = face_quad_points(v, face, N)
        for q in range(len(pts)):
            vc, fc = coarse[own[f, q]]
            assert np.linalg.norm(map_point(vc, xi[f, q]) - pts[q]) < 1e-12 * 25e-6 * 10
            fv = vc[FACE_VERTS[fc]][[0, 1, 3, 2]][:, :2]            # counter-clockwise corners
            assert _in_quad(pts[q][:2], fv)
            # no lower-index coarse face contains the point (first match in index order)
            for j in range(own[f, q]):
                vj, fj = coarse[j]
                if _in_quad(pts[q][:2], vj[FACE_VERTS[fj]][[0, 1, 3, 2]][:, :2]):
                    # allowed only if the point is on the shared boundary; then j would have matched
                    pytest.fail(f"lower-index face {j} also contains node {f},{q}")
