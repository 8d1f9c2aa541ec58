"""Pins for the incident plane wave on a vertex-lattice (curved) box in the oracle (reading R13 with the
trilinear faces' weights and node positions): on the AFFINE vertex lattice the load vector equals the
structured box's, node by node (whose delay law, trace speeds and first-hit corner are pinned in
test_oracle_time.py); on a laterally jittered top face the load still integrates the same field --
sum_j b_j(t) = c A (1 - n.k) int_face s'(tau(x)) dA up to quadrature error -- and its total weight is the
face area exactly."""
import math

import numpy as np

from oracle.operators import System
from sem_inputs import BC_ABSORBING, curved_config, plane_wave_source


def _rec(amp, seed=None, degree=4):
    rec = curved_config(nel=(4, 3, 2), degree=degree, extent=(2.0e-4, 1.5e-4, 1.0e-4), amp=amp, bc_top=BC_ABSORBING,
                        seed=seed)
    rec["plane_wave"] = plane_wave_source(0, deg=25.0, azimuth_deg=130.0)
    return rec


def test_affine_vertex_lattice_matches_structured_box():
    rc = _rec(0.0)
    rs = _rec(0.0)
    del rs["boxes"][0]["vertices"]
    sc, ss = System(rc), System(rs)
    assert np.allclose(sc.pw_xref, ss.pw_xref, rtol=0, atol=1e-18)
    for t in (0.2e-6, 0.6e-6, 0.9e-6):
        bc, bs = sc.plane_wave_load(t), ss.plane_wave_load(t)
        assert np.abs(bs).max() > 0.0
        assert np.abs(bc - bs).max() < 1e-12 * np.abs(bs).max()


def test_jittered_top_face_weights_and_integral():
    rec = _rec(0.0, degree=6)
    # move the interior vertices of the top layer in-plane (the face stays planar and keeps its rectangle)
    b = rec["boxes"][0]
    nx, ny, nz = b["nel"]
    V = b["vertices"].reshape(nz + 1, ny + 1, nx + 1, 3)
    J = np.random.default_rng(3).uniform(-0.2, 0.2, size=(ny + 1, nx + 1, 2)) * 5.0e-5
    J[0] = J[-1] = 0.0
    J[:, 0] = J[:, -1] = 0.0
    V[-1, :, :, :2] += J
    b["vertices"] = V.reshape(-1, 3)
    s = System(rec)
    area = b["extent"][0] * b["extent"][1]
    assert abs(s.pw_w.sum() - area) < 1e-12 * area
    ref = System(_rec(0.0, degree=6))
    pw = rec["plane_wave"]
    for t in (0.5e-6, 0.8e-6):
        tot, tot_ref = s.plane_wave_load(t).sum(), ref.plane_wave_load(t).sum()
        scale = b["c"] * pw["amp_pa"] * 2 * math.pi * pw["f0_hz"] * area
        assert abs(tot - tot_ref) < 2e-4 * scale, (tot, tot_ref, scale)
