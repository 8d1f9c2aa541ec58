"""Workload records for BASELINE.json configs 0-4 and their reduced test variants.

Everything here is a *parameter* of a run (geometry, material, drive, seeds), as
listed in BASELINE.json ``configs`` and fixed where the configs are silent by the
readings in DESIGN.md section "Readings" (R-numbers).  Units are SI throughout.

Record layout (plain dicts / numpy arrays, no method arithmetic):

``boxes``      list of {origin[3], extent[3], nel[3], degree, c, rho, bc[6]}
               bc order: -x, +x, -y, +y, -z, +z  (BC_RIGID / BC_ABSORBING / BC_INTERFACE)
``interface``  None or {fine_box, coarse_box, alpha}
``pmut``       None or {box, face, centers[n,2], side, mode_mn[M,2], freq_hz[n,M],
               modal_mass[M], damping[M], eta[M], rx, t_switch, capacitance,
               amp_v, f0_hz, n_cycles, delay_s[n]}
``plane_wave`` None or {box, face, amp_pa, f0_hz, sigma_s, t0_s, direction[3]}
``dt``, ``n_steps``, ``coupling`` ('predicted' | 'literal'), ``seed``
"""
from __future__ import annotations

import math

import numpy as np

BC_RIGID, BC_ABSORBING, BC_INTERFACE = 0, 1, 2
FACE_NAMES = ("-x", "+x", "-y", "+y", "-z", "+z")

UM = 1e-6
C_WATER, RHO_WATER = 1500.0, 1000.0

# BASELINE.json config 0: PMUT element parameters shared by all configs.
MEMBRANE_SIDE = 100 * UM
PITCH = 150 * UM
MODES_3 = ((1, 1), (1, 3), (3, 1))
FREQS_3 = (3.0e6, 15.0e6, 15.0e6)
# config 3: six modes.  Shapes for modes 5-6 are reading R15.
MODES_6 = ((1, 1), (1, 3), (3, 1), (3, 3), (1, 5), (5, 1))
FREQS_6 = (3.0e6, 15.0e6, 15.0e6, 27.0e6, 33.0e6, 33.0e6)
MODAL_MASS = 1e-10      # kg
DAMPING = 0.01
ETA = 1e-6              # N/V (= C/m)
DRIVE_V, DRIVE_F0, DRIVE_CYCLES = 5.0, 3.0e6, 3
CFL = 0.3
STEER_DEG = 20.0        # reading R11 (linear steering angle, configs 1-2)
RX_CAPACITANCE = 1e-10  # reading R14
PENALTY_ALPHA = 10.0    # config 2: "penalty coefficient 10*N^2/h"


def _box(origin, extent, nel, degree, bc, c=C_WATER, rho=RHO_WATER):
    return {"origin": tuple(float(v) for v in origin), "extent": tuple(float(v) for v in extent),
            "nel": tuple(int(v) for v in nel), "degree": int(degree), "c": float(c),
            "rho": float(rho), "bc": list(bc)}


def cfl_dt(boxes, cfl=CFL):
    """Reading R8: dt = cfl * min_box h_min / (c N^2)."""
    best = math.inf
    for b in boxes:
        h = min(e / n for e, n in zip(b["extent"], b["nel"]))
        best = min(best, h / (b["c"] * b["degree"] ** 2))
    return cfl * best


def _scatter(n_pmut, seed, rel=0.01):
    """Reading R16: one N(0,1) draw per PMUT (row-major, x fastest), applied to all its modes."""
    return 1.0 + rel * np.random.default_rng(seed).standard_normal(n_pmut)


def _grid_centers(n_side, pitch, offset):
    c = offset + pitch * np.arange(n_side)
    xx, yy = np.meshgrid(c, c, indexing="xy")       # x fastest in the flattened order
    return np.stack([xx.ravel(), yy.ravel()], axis=1)


def _pmut(centers, modes, freqs, scatter, delay, *, rx=False, amp=DRIVE_V, box=0, face=4):
    n = len(centers)
    m = len(modes)
    f = np.asarray(freqs, float)[None, :] * (np.ones(n) if scatter is None else scatter)[:, None]
    return {"box": box, "face": face, "centers": np.asarray(centers, float).reshape(n, 2),
            "side": MEMBRANE_SIDE, "mode_mn": np.asarray(modes, np.int32).reshape(m, 2),
            "freq_hz": f, "modal_mass": np.full(m, MODAL_MASS), "damping": np.full(m, DAMPING),
            "eta": np.full(m, ETA), "rx": bool(rx), "t_switch": 0.0 if rx else math.inf,
            "capacitance": RX_CAPACITANCE, "amp_v": 0.0 if rx else amp, "f0_hz": DRIVE_F0,
            "n_cycles": DRIVE_CYCLES, "delay_s": np.asarray(delay, float).reshape(n)}


def _steer_delay(centers, c=C_WATER, deg=STEER_DEG):
    """Reading R11: tau_k = (x_k - min x) sin(theta) / c."""
    x = centers[:, 0]
    return (x - x.min()) * math.sin(math.radians(deg)) / c


def _focus_delay(centers, focus, c=C_WATER):
    """Reading R12: tau_k = (max_j |x_j - F| - |x_k - F|) / c (farthest element fires first)."""
    pts = np.concatenate([centers, np.zeros((len(centers), 1))], axis=1)
    d = np.linalg.norm(pts - np.asarray(focus)[None, :], axis=1)
    return (d.max() - d) / c


def _two_box(n_side, fine_nz, coarse_nz, *, nf=5, nc=3, hf=25 * UM):
    """Configs 2-4 layout (reading R17/R18): fine N=5 primary z in [0, fine_nz*hf],
    coarse N=3 secondary above it, lateral size n_side * pitch, 2:1 in h."""
    L = n_side * PITCH
    nfx = int(round(L / hf))
    hc = 2 * hf
    fine = _box((0, 0, 0), (L, L, fine_nz * hf), (nfx, nfx, fine_nz), nf,
                [BC_RIGID] * 4 + [BC_RIGID, BC_INTERFACE])
    coarse = _box((0, 0, fine_nz * hf), (L, L, coarse_nz * hc), (nfx // 2, nfx // 2, coarse_nz), nc,
                  [BC_RIGID] * 4 + [BC_INTERFACE, BC_ABSORBING])
    return [fine, coarse]


def _finish(rec):
    rec.setdefault("interface", None)
    rec.setdefault("pmut", None)
    rec.setdefault("plane_wave", None)
    rec.setdefault("coupling", "predicted")
    rec["dt"] = cfl_dt(rec["boxes"]) if rec.get("dt") is None else float(rec["dt"])
    return rec


def _plane_wave(box, *, amp=1e3, f0=3.0e6, deg=20.0):
    """Reading R13: Gaussian-modulated sine s(tau)=exp(-(tau-t0)^2/(2 sigma^2)) sin(2 pi f0 (tau-t0)),
    sigma = 1/(2 f0), t0 = 4 sigma, direction (sin th, 0, -cos th), entering through +z of ``box``."""
    sigma = 1.0 / (2.0 * f0)
    th = math.radians(deg)
    return {"box": box, "face": 5, "amp_pa": amp, "f0_hz": f0, "sigma_s": sigma, "t0_s": 4 * sigma,
            "direction": (math.sin(th), 0.0, -math.cos(th))}


def config(i: int, **over):
    """BASELINE.json configs[i] as a workload record."""
    if i == 0:
        boxes = [_box((0, 0, 0), (600 * UM,) * 3, (4, 4, 4), 4, [BC_RIGID] * 5 + [BC_ABSORBING])]
        pm = _pmut([[300 * UM, 300 * UM]], MODES_3, FREQS_3, None, [0.0])
        rec = {"name": "cfg0", "boxes": boxes, "pmut": pm, "n_steps": 400, "seed": 0}
    elif i == 1:
        boxes = [_box((0, 0, 0), (900 * UM, 900 * UM, 1200 * UM), (24, 24, 32), 4,
                      [BC_RIGID] * 5 + [BC_ABSORBING])]
        cen = _grid_centers(4, PITCH, 225 * UM)
        pm = _pmut(cen, MODES_3, FREQS_3, _scatter(16, 0), _steer_delay(cen))
        rec = {"name": "cfg1", "boxes": boxes, "pmut": pm, "n_steps": 2000, "seed": 0}
    elif i == 2:
        boxes = _two_box(16, 24, 80)
        cen = _grid_centers(16, PITCH, 75 * UM)
        pm = _pmut(cen, MODES_3, FREQS_3, _scatter(256, 0), _steer_delay(cen))
        rec = {"name": "cfg2", "boxes": boxes, "pmut": pm, "n_steps": 3000, "seed": 0,
               "interface": {"fine_box": 0, "coarse_box": 1, "alpha": PENALTY_ALPHA}}
    elif i == 3:
        boxes = _two_box(64, 24, 80)
        cen = _grid_centers(64, PITCH, 75 * UM)
        focus = (4.8e-3, 4.8e-3, 4.0e-3)
        pm = _pmut(cen, MODES_6, FREQS_6, _scatter(4096, 0), _focus_delay(cen, focus))
        rec = {"name": "cfg3", "boxes": boxes, "pmut": pm, "n_steps": 2000, "seed": 0,
               "interface": {"fine_box": 0, "coarse_box": 1, "alpha": PENALTY_ALPHA}}
    elif i == 4:
        boxes = _two_box(32, 24, 80)
        cen = _grid_centers(32, PITCH, 75 * UM)
        pm = _pmut(cen, MODES_3, FREQS_3, _scatter(1024, 4), np.zeros(1024), rx=True)
        rec = {"name": "cfg4", "boxes": boxes, "pmut": pm, "n_steps": 4000, "seed": 4,
               "interface": {"fine_box": 0, "coarse_box": 1, "alpha": PENALTY_ALPHA},
               "plane_wave": _plane_wave(1)}
    else:
        raise ValueError(f"no config {i}")
    rec.update(over)
    return _finish(rec)


def crop_config(i: int, n_side: int, **over):
    """A lateral crop of configs 2-4: n_side x n_side PMUTs with the config's full depth, N, h,
    interface, modes and drive law (the bounded CPU sample of bench.py's cpu_baseline)."""
    if i not in (2, 3, 4):
        raise ValueError("crop only for the two-box configs 2-4")
    full = config(i)
    boxes = _two_box(n_side, full["boxes"][0]["nel"][2], full["boxes"][1]["nel"][2])
    cen = _grid_centers(n_side, PITCH, 75 * UM)
    pmf = full["pmut"]
    modes = [tuple(m) for m in pmf["mode_mn"]]
    freqs = FREQS_6 if i == 3 else FREQS_3
    if i == 3:
        half = n_side * PITCH / 2
        pm = _pmut(cen, modes, freqs, _scatter(n_side * n_side, full["seed"]), _focus_delay(cen, (half, half, 4.0e-3)))
    elif i == 2:
        pm = _pmut(cen, modes, freqs, _scatter(n_side * n_side, full["seed"]), _steer_delay(cen))
    else:
        pm = _pmut(cen, modes, freqs, _scatter(n_side * n_side, full["seed"]), np.zeros(n_side * n_side), rx=True)
    rec = {"name": f"cfg{i}crop{n_side}", "boxes": boxes, "pmut": pm, "n_steps": full["n_steps"],
           "seed": full["seed"], "interface": full["interface"], "plane_wave": full["plane_wave"]}
    rec.update(over)
    return _finish(rec)


def config_names():
    return [f"cfg{i}" for i in range(5)]


def small_config(name: str, **over):
    """Reduced variants with the structure of configs 1-4 (same N, h, interface, PMUT physics)
    at sizes the oracle finishes in seconds.  Used by parity tests only."""
    if name == "cfg1s":   # config 1 physics, 2x2 array, N=4, h=37.5um, unaligned membranes
        boxes = [_box((0, 0, 0), (450 * UM, 450 * UM, 300 * UM), (12, 12, 8), 4,
                      [BC_RIGID] * 5 + [BC_ABSORBING])]
        cen = _grid_centers(2, PITCH, 150 * UM)
        pm = _pmut(cen, MODES_3, FREQS_3, _scatter(4, 0), _steer_delay(cen))
        rec = {"name": name, "boxes": boxes, "pmut": pm, "n_steps": 300, "seed": 0}
    elif name == "cfg2s":  # config 2 layout, 2x2 array, N5/N3 2:1 interface
        boxes = _two_box(2, 4, 4)
        cen = _grid_centers(2, PITCH, 75 * UM)
        pm = _pmut(cen, MODES_3, FREQS_3, _scatter(4, 0), _steer_delay(cen))
        rec = {"name": name, "boxes": boxes, "pmut": pm, "n_steps": 300, "seed": 0,
               "interface": {"fine_box": 0, "coarse_box": 1, "alpha": PENALTY_ALPHA}}
    elif name == "cfg3s":  # config 3 physics: 6 modes, focus law
        boxes = _two_box(2, 4, 4)
        cen = _grid_centers(2, PITCH, 75 * UM)
        focus = (150 * UM, 150 * UM, 4.0e-3)
        pm = _pmut(cen, MODES_6, FREQS_6, _scatter(4, 0), _focus_delay(cen, focus))
        rec = {"name": name, "boxes": boxes, "pmut": pm, "n_steps": 300, "seed": 0,
               "interface": {"fine_box": 0, "coarse_box": 1, "alpha": PENALTY_ALPHA}}
    elif name == "cfg4s":  # config 4 physics: RX feedback + plane-wave boundary source
        boxes = _two_box(2, 4, 3)
        cen = _grid_centers(2, PITCH, 75 * UM)
        pm = _pmut(cen, MODES_3, FREQS_3, _scatter(4, 4), np.zeros(4), rx=True)
        pw = _plane_wave(1)
        pw["t0_s"] = 0.0  # pulse centred at t=0 so the short run sees the full waveform's rise
        rec = {"name": name, "boxes": boxes, "pmut": pm, "n_steps": 400, "seed": 4,
               "interface": {"fine_box": 0, "coarse_box": 1, "alpha": PENALTY_ALPHA},
               "plane_wave": pw}
    else:
        raise ValueError(f"no small config {name}")
    rec.update(over)
    return _finish(rec)


def small_config_names():
    return ["cfg1s", "cfg2s", "cfg3s", "cfg4s"]


def cavity_config(nel=(3, 3, 3), degree=4, extent=(1e-3, 1e-3, 1e-3), c=C_WATER, n_steps=100, cfl=0.3):
    """Closed rigid box, no PMUT, no ABC: for cavity eigenmode and energy pins."""
    boxes = [_box((0, 0, 0), extent, nel, degree, [BC_RIGID] * 6, c=c)]
    rec = {"name": "cavity", "boxes": boxes, "n_steps": n_steps, "seed": 0}
    rec["dt"] = cfl_dt(boxes, cfl)
    return _finish(rec)


PML_R = 1e-4           # reflection coefficient of the PML profile (R in [1e-5, 1e-4])


def pml_config(nel=(4, 4, 6), degree=4, extent=(0.4e-3, 0.4e-3, 0.6e-3), layers=(0, 0, 0, 0, 0, 1),
               layer_el=2, R=PML_R, abc_on_pml=True, c=C_WATER, n_steps=100, cfl=0.3):
    """One box with PML layers (oracle/pml.py readings R23-R25): ``layers`` flags
    the faces (-x,+x,-y,+y,-z,+z) that carry a layer ``layer_el`` elements thick; those faces are
    absorbing (the paper's Gamma_ABC behind the PML) if ``abc_on_pml``, the others rigid."""
    h = [e / n for e, n in zip(extent, nel)]
    thick = [float(layers[f]) * layer_el * h[f // 2] for f in range(6)]
    bc = [BC_ABSORBING if (layers[f] and abc_on_pml) else BC_RIGID for f in range(6)]
    boxes = [_box((0, 0, 0), extent, nel, degree, bc, c=c)]
    rec = {"name": "pml", "boxes": boxes, "n_steps": n_steps, "seed": 0,
           "pml": {"box": 0, "thickness": thick, "R": float(R)}}
    rec["dt"] = cfl_dt(boxes, cfl)
    return _finish(rec)


def conforming_cut_config(nel_xy=3, nz_lo=2, nz_hi=2, degree=4, h=1e-4 / 3, alpha=PENALTY_ALPHA,
                          n_steps=100, cfl=0.3, ratio=1, degree_hi=None, bc_top=BC_RIGID):
    """Two boxes stacked in z with a DG interface between them.  ratio=1 and degree_hi=None gives
    a conforming mesh cut by the interface (pin: equals the single CG box up to discretisation)."""
    dh = degree if degree_hi is None else degree_hi
    lo = _box((0, 0, 0), (nel_xy * h, nel_xy * h, nz_lo * h), (nel_xy, nel_xy, nz_lo), degree,
              [BC_RIGID] * 5 + [BC_INTERFACE])
    hh = ratio * h
    hi = _box((0, 0, nz_lo * h), (nel_xy * h, nel_xy * h, nz_hi * hh),
              (nel_xy // ratio, nel_xy // ratio, nz_hi), dh, [BC_RIGID] * 4 + [BC_INTERFACE, bc_top])
    rec = {"name": "cut", "boxes": [lo, hi], "n_steps": n_steps, "seed": 0,
           "interface": {"fine_box": 0, "coarse_box": 1, "alpha": alpha}}
    rec["dt"] = cfl_dt(rec["boxes"], cfl)
    return _finish(rec)


def n_nodes(box):
    return tuple(box["degree"] * n + 1 for n in box["nel"])


def box_dof(box):
    nx, ny, nz = n_nodes(box)
    return nx * ny * nz


def total_dof(rec):
    return sum(box_dof(b) for b in rec["boxes"])


def random_state(rec, seed=1234, scale_v=None):
    """Seeded random (p, pdot) per box for operator-level tests (lexicographic x-fastest)."""
    rng = np.random.default_rng(seed)
    out = []
    for b in rec["boxes"]:
        n = box_dof(b)
        p = rng.standard_normal(n)
        v = rng.standard_normal(n) * (1.0 / rec["dt"] * 1e-3 if scale_v is None else scale_v)
        out.append((p, v))
    return out


def interface_faces(nfx=4, nfy=3, R=2, hf=25e-6, z0=0.0, jitter=0.0, seed=0):
    """Face sets of a 2:1 (R:1) non-conforming interface for the face-matching algorithm (Algorithm 3):
    fine elements nfx x nfy of edge hf below the plane z = z0 (their +z faces, local face 5) and coarse
    elements (nfx/R) x (nfy/R) of edge R hf above it (their -z faces, local face 4).  Interior vertices
    of the plane are moved in-plane by U(-jitter, jitter) * edge (seeded), so the maps are trilinear
    (non-affine) while both face sets still tile the same planar region.  Returns (fine, coarse):
    lists of (verts (8, 3) in the order v = i + 2 j + 4 k, local face)."""
    rng = np.random.default_rng(seed)
    ncx, ncy = nfx // R, nfy // R

    def plane_lattice(nx, ny, h):
        X, Y = np.meshgrid(np.arange(nx + 1) * h, np.arange(ny + 1) * h, indexing="ij")
        J = rng.uniform(-jitter, jitter, size=(2, nx + 1, ny + 1)) * h
        J[:, 0, :] = J[:, -1, :] = 0.0
        J[:, :, 0] = J[:, :, -1] = 0.0
        return X + J[0], Y + J[1]

    fx, fy = plane_lattice(nfx, nfy, hf)
    cx, cy = plane_lattice(ncx, ncy, R * hf)
    fine, coarse = [], []
    for j in range(nfy):
        for i in range(nfx):
            v = np.zeros((8, 3))
            for k in range(8):
                a, b, c = k & 1, (k >> 1) & 1, k >> 2
                if c == 1:      # top = interface plane (jittered)
                    v[k] = [fx[i + a, j + b], fy[i + a, j + b], z0]
                else:
                    v[k] = [(i + a) * hf, (j + b) * hf, z0 - hf]
            fine.append((v, 5))
    for j in range(ncy):
        for i in range(ncx):
            v = np.zeros((8, 3))
            for k in range(8):
                a, b, c = k & 1, (k >> 1) & 1, k >> 2
                if c == 0:      # bottom = interface plane (jittered)
                    v[k] = [cx[i + a, j + b], cy[i + a, j + b], z0]
                else:
                    v[k] = [(i + a) * R * hf, (j + b) * R * hf, z0 + R * hf]
            coarse.append((v, 4))
    return fine, coarse


def curved_config(nel=(3, 3, 3), degree=4, extent=(3e-4, 3e-4, 3e-4), amp=0.12, bc_top=BC_RIGID, c=C_WATER,
                  n_steps=100, cfl=0.25, seed=None):
    """One logically structured box whose vertex lattice is displaced by the smooth bulge
    u(x) = amp h (sin(pi x/Lx) sin(pi y/Ly) sin(pi z/Lz)) (1, 0.7, -0.5) (boundary vertices fixed, so
    the box faces stay planar) -- trilinear, non-affine elements.  With ``seed``
    the interior vertices get an extra U(-amp/2, amp/2) h jitter.  Faces rigid except the top (bc_top)."""
    L = np.asarray(extent, dtype=np.float64)
    h = L / np.asarray(nel)
    gx, gy, gz = [np.arange(n + 1) * hh for n, hh in zip(nel, h)]
    Z, Y, X = np.meshgrid(gz, gy, gx, indexing="ij")
    pts = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    bump = np.sin(np.pi * pts[:, 0] / L[0]) * np.sin(np.pi * pts[:, 1] / L[1]) * np.sin(np.pi * pts[:, 2] / L[2])
    hmin = float(h.min())
    pts = pts + amp * hmin * bump[:, None] * np.array([1.0, 0.7, -0.5])[None, :]
    if seed is not None:
        interior = np.all((pts > 1e-12 * L) & (pts < L * (1 - 1e-12)), axis=1)
        jit = np.random.default_rng(seed).uniform(-0.5 * amp, 0.5 * amp, size=pts.shape) * hmin
        pts[interior] += jit[interior]
    boxes = [_box((0, 0, 0), extent, nel, degree, [BC_RIGID] * 5 + [bc_top], c=c)]
    boxes[0]["vertices"] = pts
    rec = {"name": "curved", "boxes": boxes, "n_steps": n_steps, "seed": 0}
    rec["dt"] = cfl_dt(boxes, cfl)
    return _finish(rec)



def solid_block(nel, lo, hi):
    """Element indices (ex + nel_x (ey + nel_y ez)) of the block lo <= (ex, ey, ez) < hi."""
    ex, ey, ez = np.meshgrid(*[np.arange(a, b) for a, b in zip(lo, hi)], indexing="ij")
    return np.sort((ex + nel[0] * (ey + nel[1] * ez)).ravel()).astype(np.int64)


def obstacle_config(nel=(6, 6, 4), degree=3, h=25e-6, solid_lo=(2, 2, 1), solid_hi=(4, 4, 3), bc=None,
                    curved_amp=0.0, c=C_WATER, n_steps=100, cfl=0.25, seed=None):
    """One box with a rigid obstacle: the elements of the index block
    solid_lo <= (ex, ey, ez) < solid_hi are removed from the fluid, their faces towards the fluid are
    Neumann (rigid) surfaces.  bc: six face tags (default: rigid, absorbing top).  curved_amp > 0 puts
    the box on curved_config's displaced vertex lattice (with ``seed``: jittered)."""
    extent = tuple(h * n for n in nel)
    if curved_amp > 0.0:
        rec = curved_config(nel=nel, degree=degree, extent=extent, amp=curved_amp, c=c, n_steps=n_steps,
                            cfl=cfl, seed=seed)
    else:
        rec = {"name": "obstacle", "boxes": [_box((0, 0, 0), extent, nel, degree, [BC_RIGID] * 6, c=c)],
               "n_steps": n_steps, "seed": 0}
        rec["dt"] = cfl_dt(rec["boxes"], cfl)
        rec = _finish(rec)
    rec["name"] = "obstacle"
    rec["boxes"][0]["bc"] = list(bc) if bc is not None else [BC_RIGID] * 5 + [BC_ABSORBING]
    rec["boxes"][0]["solid"] = solid_block(nel, solid_lo, solid_hi)
    return rec


def obstacle_pmut_config(n_cycles=1, n_steps=2160, with_obstacle=True):
    """The paper's Section 6.2 scenario at desk scale: one PMUT on the bottom face
    transmits a tone burst, switches to open-circuit reception (Eq. 3) at t_bar = the burst's end, and
    receives the echo of a rigid obstacle -- a 250 x 250 x 25 um solid slab (the paper's obstacle
    thickness h_2 = 25 um; it spans 5/6 of the box width as r_obs / r = 1700 / 2000 does) 300 um above
    the membrane.  Water, N = 3, h = 25 um, 12 x 12 x 16 elements;
    absorbing lateral and top faces (the paper's absorbing outer boundary), rigid bottom around the
    membrane.  Config-0 membrane physics (100 um square, 3 modes); n_cycles = 1 keeps the burst
    (1/3 us) shorter than the echo delay (0.4 us).  RX capacitance: reading R14."""
    h, nel = 25 * UM, (12, 12, 16)
    boxes = [_box((0, 0, 0), tuple(h * n for n in nel), nel, 3,
                  [BC_ABSORBING] * 4 + [BC_RIGID, BC_ABSORBING])]
    pm = _pmut([[150 * UM, 150 * UM]], MODES_3, FREQS_3, None, [0.0])
    pm["n_cycles"] = int(n_cycles)
    pm["rx"] = True
    pm["amp_v"] = DRIVE_V
    pm["t_switch"] = n_cycles / DRIVE_F0
    rec = {"name": "obstacle_pmut", "boxes": boxes, "pmut": pm, "n_steps": int(n_steps), "seed": 0}
    rec = _finish(rec)
    if with_obstacle:
        rec["boxes"][0]["solid"] = solid_block(nel, (1, 1, 12), (11, 11, 13))
    return rec


def curved_interface_config(nf=(6, 6, 2), nc=(4, 4, 2), degree_f=4, degree_c=3, hf=25e-6, jitter=0.15, seed=0,
                            bc_top=BC_RIGID, c_f=C_WATER, c_c=C_WATER, alpha=PENALTY_ALPHA, n_steps=100, cfl=0.25,
                            coarse_height=75e-6, nested_jitter=False, pmut=False):
    """Two curved (vertex-lattice) boxes stacked in z, joined by a general non-conforming DG interface
    (the interface quadrature of P:L912-938 with Algorithm 3's matching,
    P:L1062-1080, on trilinear faces).  The fine box has nf elements of degree degree_f and edge hf, the
    coarse box above it nc elements of degree degree_c over the same lateral extent L = nf[0] hf, so the
    lattices need not nest (6 : 4 is a 1.5 : 1 ratio); the coarse box is coarse_height tall.  The interior vertices of the interface plane move
    in-plane by U(-jitter, jitter) x edge, independently on the two sides (seeded), so the two face sets
    tile the same plane without matching; every other vertex stays on the affine lattice.  With
    nested_jitter (nf a multiple of nc) only the coarse vertices are drawn and the fine interface
    vertices are the coarse faces' bilinear maps at the sub-lattice points: curved faces that nest.  Faces rigid
    except the coarse top (bc_top).  pmut: one config-0 membrane (TX) centred on the fine box's floor."""
    rng = np.random.default_rng(seed)
    L = nf[0] * hf
    hc = L / nc[0]
    hcz = coarse_height / nc[2]
    z0 = nf[2] * hf

    def lattice(nel, h, zb, jitter_layer):
        nx, ny, nz = (n + 1 for n in nel)
        Z, Y, X = np.meshgrid(zb + np.arange(nz) * h[2], np.arange(ny) * h[1], np.arange(nx) * h[0], indexing="ij")
        pts = np.stack([X, Y, Z], axis=-1)            # [nz][ny][nx][3]
        if jitter > 0.0:
            J = rng.uniform(-jitter, jitter, size=(ny, nx, 2)) * np.array(h[:2])
            J[0, :, :] = J[-1, :, :] = 0.0
            J[:, 0, :] = J[:, -1, :] = 0.0
            pts[jitter_layer, :, :, :2] += J
        return pts.reshape(-1, 3)

    fine = _box((0, 0, 0), (L, L, z0), nf, degree_f, [BC_RIGID] * 5 + [BC_INTERFACE], c=c_f)
    coarse = _box((0, 0, z0), (L, L, coarse_height), nc, degree_c, [BC_RIGID] * 4 + [BC_INTERFACE, bc_top], c=c_c)
    fine["vertices"] = lattice(nf, (hf, hf, hf), 0.0, nf[2])
    coarse["vertices"] = lattice(nc, (hc, hc, hcz), z0, 0)
    if nested_jitter:
        R = nf[0] // nc[0]
        if nf[0] != R * nc[0] or nf[1] != R * nc[1]:
            raise ValueError("nested_jitter needs nf = R nc laterally")
        cv = coarse["vertices"].reshape(nc[2] + 1, nc[1] + 1, nc[0] + 1, 3)[0]     # interface layer
        fv = fine["vertices"].reshape(nf[2] + 1, nf[1] + 1, nf[0] + 1, 3)
        for j in range(nf[1] + 1):
            for i in range(nf[0] + 1):
                I, Jc = min(i // R, nc[0] - 1), min(j // R, nc[1] - 1)
                u, v = i / R - I, j / R - Jc
                fv[nf[2], j, i] = ((1 - u) * (1 - v) * cv[Jc, I] + u * (1 - v) * cv[Jc, I + 1] +
                                   (1 - u) * v * cv[Jc + 1, I] + u * v * cv[Jc + 1, I + 1])
        fine["vertices"] = fv.reshape(-1, 3)
    rec = {"name": "curved_iface", "boxes": [fine, coarse], "n_steps": n_steps, "seed": seed,
           "interface": {"fine_box": 0, "coarse_box": 1, "alpha": alpha}}
    if pmut:   # one config-0 membrane centred on the fine box's floor (TX burst)
        rec["pmut"] = _pmut([[L / 2, L / 2]], MODES_3, FREQS_3, None, [0.0])
    rec["dt"] = cfl_dt(rec["boxes"], cfl)
    return _finish(rec)


def curved_pmut_config(nel=(6, 6, 4), degree=4, h=25e-6, amp=0.12, floor_jitter=0.12, seed=9, rx=False,
                       n_steps=300, cfl=0.25):
    """A PMUT on a curved box (SURVEY 8(f) item 3 with the PMUT coupling of Eqs. 11-12): curved_config's
    bulged, jittered vertex lattice whose z = 0 layer (the membrane face) also moves in-plane by
    U(-floor_jitter, floor_jitter) x h (interior vertices; the face stays planar), so the face weights
    |J_s| and the node positions the mode shapes are evaluated at are not those of the affine lattice.
    One config-0 membrane (100 um square, 3 modes) centred on the floor; TX burst, or RX from t = 0."""
    extent = tuple(h * n for n in nel)
    rec = curved_config(nel=nel, degree=degree, extent=extent, amp=amp, bc_top=BC_ABSORBING, n_steps=n_steps,
                        cfl=cfl, seed=seed)
    rec["name"] = "curved_pmut"
    v = rec["boxes"][0]["vertices"].reshape(nel[2] + 1, nel[1] + 1, nel[0] + 1, 3)
    J = np.random.default_rng(seed + 1).uniform(-floor_jitter, floor_jitter, size=(nel[1] + 1, nel[0] + 1, 2)) * h
    J[0, :, :] = J[-1, :, :] = 0.0
    J[:, 0, :] = J[:, -1, :] = 0.0
    v[0, :, :, :2] += J
    rec["boxes"][0]["vertices"] = v.reshape(-1, 3)
    cx, cy = extent[0] / 2, extent[1] / 2
    rec["pmut"] = _pmut([[cx, cy]], MODES_3, FREQS_3, None, [0.0], rx=rx)
    return rec


def clamped_disc_shape(radius, modes=((0, 1), (1, 1), (0, 2))):
    """Mode shapes of a clamped circular plate of radius `radius` -- an INPUT of the method (the paper
    takes U_{k,m} from a 3D FEM eigen-analysis of the membrane; this textbook family
    stands in for it on the circular membranes of P:L1097, reading R33): for (n, s)
      S(r, theta) = cos(n theta) [J_n(l r/R) - J_n(l)/I_n(l) I_n(l r/R)] / max,  r <= R, else 0,
    l = the s-th positive root of J_n(l) I_{n+1}(l) + I_n(l) J_{n+1}(l) (S = dS/dr = 0 at r = R).
    Returns shape_fn(k, m, x_rel, y_rel) -> float for oracle and C ABI alike."""
    from scipy.optimize import brentq
    from scipy.special import iv, jv

    lam, scale = [], []
    for n, s in modes:
        f = lambda l, n=n: jv(n, l) * iv(n + 1, l) + iv(n, l) * jv(n + 1, l)
        grid = np.linspace(0.5, 40.0, 4000)
        v = f(grid)
        roots = [brentq(f, grid[i], grid[i + 1], xtol=1e-15) for i in range(len(grid) - 1) if v[i] * v[i + 1] < 0]
        l = roots[s - 1]
        rr = np.linspace(0.0, 1.0, 2001)
        prof = jv(n, l * rr) - jv(n, l) / iv(n, l) * iv(n, l * rr)
        lam.append(l)
        scale.append(1.0 / np.abs(prof).max())

    def shape_fn(k, m, xr, yr):
        r = math.hypot(xr, yr) / radius
        if r > 1.0:
            return 0.0
        n, l = modes[m][0], lam[m]
        ang = math.cos(n * math.atan2(yr, xr)) if n else 1.0
        return float(scale[m] * ang * (jv(n, l * r) - jv(n, l) / iv(n, l) * iv(n, l * r)))

    shape_fn.lam = tuple(lam)
    shape_fn.scale = tuple(scale)
    return shape_fn


def circular_pmut_config(radius=65 * UM, nel=(6, 6, 4), degree=4, h=25e-6, rx=False, n_steps=300, **kw):
    """curved_pmut_config's box (bulged, jittered vertex lattice, in-plane jitter on the membrane face)
    carrying one CIRCULAR membrane of radius r_p = 65 um with clamped_disc_shape's modes
    (reading R33) instead of the square sines; `side` is the bounding square 2 r_p."""
    rec = curved_pmut_config(nel=nel, degree=degree, h=h, rx=rx, n_steps=n_steps, **kw)
    rec["name"] = "circular_pmut"
    modes = ((0, 1), (1, 1), (0, 2))
    rec["pmut"]["side"] = 2.0 * radius
    rec["pmut"]["mode_mn"] = np.asarray(modes, np.int32)
    rec["pmut"]["shape_fn"] = clamped_disc_shape(radius, modes)
    return rec


def cylinder_pmut_config(domain_radius=90 * UM, radius=65 * UM, nel=(6, 6, 4), degree=4, height=100 * UM, rx=False,
                         n_steps=300, cfl=0.25):
    """A cylindrical water column (the cylinder domains of P:L1225) as ONE logically structured box: the
    square vertex lattice [-1, 1]^2 is mapped onto the disc by (x, y) -> (x sqrt(1 - y^2/2),
    y sqrt(1 - x^2/2)) R in every z layer (an extruded cylinder whose rigid wall is the polygon through
    the mapped boundary vertices; the four corner elements have one 180 deg - 90 deg/nel angle, so the
    lattice stays coarse; dt = cfl min(0.75 h, h_z) / (c N^2) is half the stability limit, pinned in the tests), absorbing top, one circular membrane r_p = 65 um
     with clamped_disc_shape's modes centred on the floor."""
    h = 2.0 * domain_radius / nel[0]
    rec = curved_pmut_config(nel=nel, degree=degree, h=h, amp=0.0, floor_jitter=0.0, rx=rx, n_steps=n_steps, cfl=cfl)
    rec["name"] = "cylinder_pmut"
    b = rec["boxes"][0]
    ext = (2.0 * domain_radius, 2.0 * domain_radius * nel[1] / nel[0], height)
    gx, gy, gz = [np.linspace(0.0, e, n + 1) for e, n in zip(ext, nel)]
    Z, Y, X = np.meshgrid(gz, gy, gx, indexing="ij")
    u = X / domain_radius - 1.0
    v = Y / (0.5 * ext[1]) - 1.0
    b["extent"] = ext
    b["vertices"] = np.stack([(1.0 + u * np.sqrt(1.0 - 0.5 * v * v)) * domain_radius,
                              (1.0 + v * np.sqrt(1.0 - 0.5 * u * u)) * 0.5 * ext[1], Z], axis=-1).reshape(-1, 3)
    hz = height / nel[2]
    rec["dt"] = cfl * min(0.75 * h, hz) / (b["c"] * degree ** 2)
    modes = ((0, 1), (1, 1), (0, 2))
    rec["pmut"]["centers"] = np.array([[domain_radius, 0.5 * ext[1]]])
    rec["pmut"]["side"] = 2.0 * radius
    rec["pmut"]["mode_mn"] = np.asarray(modes, np.int32)
    rec["pmut"]["shape_fn"] = clamped_disc_shape(radius, modes)
    return rec


def cylinder_two_box_config(domain_radius=90 * UM, radius=65 * UM, nc=(4, 4, 2), ratio=2, nfz=3, degree_f=4,
                            degree_c=3, coarse_height=90 * UM, n_steps=500, cfl=0.35, alpha=PENALTY_ALPHA):
    """The paper's array geometry in a cylinder: a fine inner box carrying a
    circular membrane (r_p = 65 um, clamped_disc_shape, reading R33) under a coarse outer box, both
    mapped onto the same polygonal cylinder, joined by the general non-conforming interface.  The coarse
    lateral vertex lattice is cylinder_pmut_config's square -> disc map; the fine one (ratio x finer) is
    its bilinear subdivision, so every fine face lies in one coarse face (curved faces that nest) and
    both boxes have the same polygonal wall.  Rigid wall and floor, absorbing top."""
    ncx, ncy, ncz = nc
    nf = (ratio * ncx, ratio * ncy, nfz)
    hc = 2.0 * domain_radius / ncx
    hf = hc / ratio
    z0 = nfz * hf
    g = np.linspace(-1.0, 1.0, ncx + 1)
    gy = np.linspace(-1.0, 1.0, ncy + 1)
    V, U = np.meshgrid(gy, g, indexing="ij")
    cl = np.stack([(1.0 + U * np.sqrt(1.0 - 0.5 * V * V)) * domain_radius,
                   (1.0 + V * np.sqrt(1.0 - 0.5 * U * U)) * domain_radius], axis=-1)       # [ncy+1][ncx+1][2]
    fl = np.empty((nf[1] + 1, nf[0] + 1, 2))
    for j in range(nf[1] + 1):
        for i in range(nf[0] + 1):
            I, Jc = min(i // ratio, ncx - 1), min(j // ratio, ncy - 1)
            u, v = i / ratio - I, j / ratio - Jc
            fl[j, i] = ((1 - u) * (1 - v) * cl[Jc, I] + u * (1 - v) * cl[Jc, I + 1] + (1 - u) * v * cl[Jc + 1, I] +
                        u * v * cl[Jc + 1, I + 1])

    def extrude(lat, zs):
        out = np.empty((len(zs),) + lat.shape[:2] + (3,))
        out[..., :2] = lat[None]
        out[..., 2] = np.asarray(zs)[:, None, None]
        return out.reshape(-1, 3)

    L = 2.0 * domain_radius
    fine = _box((0, 0, 0), (L, L, z0), nf, degree_f, [BC_RIGID] * 5 + [BC_INTERFACE])
    coarse = _box((0, 0, z0), (L, L, coarse_height), nc, degree_c, [BC_RIGID] * 4 + [BC_INTERFACE, BC_ABSORBING])
    fine["vertices"] = extrude(fl, np.arange(nfz + 1) * hf)
    coarse["vertices"] = extrude(cl, z0 + np.arange(ncz + 1) * (coarse_height / ncz))
    rec = {"name": "cylinder_two_box", "boxes": [fine, coarse], "n_steps": n_steps, "seed": 0,
           "interface": {"fine_box": 0, "coarse_box": 1, "alpha": alpha}}
    modes = ((0, 1), (1, 1), (0, 2))
    rec["pmut"] = _pmut([[domain_radius, domain_radius]], modes, FREQS_3, None, [0.0])
    rec["pmut"]["side"] = 2.0 * radius
    rec["pmut"]["shape_fn"] = clamped_disc_shape(radius, modes)
    rec["dt"] = cfl * min(0.6 * hf / degree_f ** 2, 0.6 * hc / degree_c ** 2, coarse_height / ncz / degree_c ** 2) / C_WATER
    return _finish(rec)


def plane_wave_source(box, *, amp=1e3, f0=3.0e6, deg=20.0, azimuth_deg=0.0):
    """Reading R13's incident wave record for any box (config 4's source; tests attach it to curved
    boxes): direction (sin th cos az, sin th sin az, -cos th) entering through +z."""
    pw = _plane_wave(box, amp=amp, f0=f0, deg=deg)
    th, az = math.radians(deg), math.radians(azimuth_deg)
    pw["direction"] = (math.sin(th) * math.cos(az), math.sin(th) * math.sin(az), -math.cos(th))
    return pw


def cylinder_obstacle_config(n_cycles=1, n_steps=2050, cfl=0.2, with_obstacle=True):
    """Section 6.2 in its own geometry (cylinder domain P:L1225) at desk scale: a
    cylindrical water column (one box mapped square -> disc, R = 150 um, 8 x 8 x 16 elements, N = 3,
    rigid wall and floor, absorbing top) with one CIRCULAR membrane (r_p = 65 um, clamped_disc_shape,
    reading R33) that transmits a one-cycle burst, switches to open-circuit reception at the burst's end
    and receives the echo of a rigid slab one element (25 um = h_2) thick 300 um above it; the slab is
    the mapped image of the 6 x 6 central lattice elements, i.e. a rounded disc spanning about 5/6 of the
    diameter as r_obs / r = 1700 / 2000 does."""
    R, nel, hz, degree = 150 * UM, (8, 8, 16), 25 * UM, 3
    rec = cylinder_pmut_config(domain_radius=R, nel=nel, degree=degree, height=hz * nel[2], rx=False, n_steps=n_steps,
                               cfl=cfl)
    rec["name"] = "cylinder_obstacle"
    # rigid wall, absorbing top: the explicit ABC term needs dt C_ii / M_ii < 2, and C_ii / M_ii is large at
    # the four near-degenerate wall corners of the mapped lattice (an absorbing wall there diverges at this dt)
    pm = rec["pmut"]
    pm["n_cycles"] = int(n_cycles)
    pm["rx"] = True
    pm["amp_v"] = DRIVE_V
    pm["t_switch"] = n_cycles / DRIVE_F0
    if with_obstacle:
        rec["boxes"][0]["solid"] = solid_block(nel, (1, 1, 12), (7, 7, 13))
    return rec
