"""Pins for oracle.newmark (Algorithm 1) against closed forms and invariants."""
import math

import numpy as np
import pytest

from oracle.newmark import Newmark, drive
from oracle.operators import System
from sem_inputs import cavity_config, config, conforming_cut_config, small_config


def _history(nm, n):
    out = [nm.p.copy()]
    for _ in range(n):
        nm.step()
        out.append(nm.p.copy())
    return out


def test_leapfrog_identity_closed_box():
    """p^{n+1} - 2 p^n + p^{n-1} = -dt^2 M^{-1} K p^n with C = 0, f = 0."""
    rec = cavity_config(nel=(2, 2, 3), degree=3)
    s = System(rec)
    nm = Newmark(s)
    rng = np.random.default_rng(3)
    nm.set_state(rng.standard_normal(s.ndof), rng.standard_normal(s.ndof) / rec["dt"] * 1e-2)
    ps = _history(nm, 12)
    dt = rec["dt"]
    for n in range(2, 12):
        lhs = ps[n + 1] - 2 * ps[n] + ps[n - 1]
        rhs = -dt * dt * s.apply_K(ps[n]) / s.M
        assert np.linalg.norm(lhs - rhs) < 1e-12 * np.linalg.norm(rhs) + 1e-14 * np.linalg.norm(ps[n])


@pytest.mark.parametrize("kind", ["single", "interface"])
def test_discrete_energy_conserved(kind):
    """E^{n+1/2} = 1/2 v^T M v + 1/2 p^{n+1}^T K p^n, v = (p^{n+1}-p^n)/dt, is exactly conserved by
    leapfrog in a closed lossless box (with or without the SIPG interface)."""
    if kind == "single":
        rec = cavity_config(nel=(2, 3, 2), degree=4)
    else:
        rec = conforming_cut_config(nel_xy=2, nz_lo=2, nz_hi=2, degree=5, degree_hi=3, ratio=2, h=25e-6)
    s = System(rec)
    nm = Newmark(s)
    rng = np.random.default_rng(4)
    nm.set_state(rng.standard_normal(s.ndof), np.zeros(s.ndof))
    ps = _history(nm, 400)
    dt = rec["dt"]
    E = []
    for n in range(1, 400):
        v = (ps[n + 1] - ps[n]) / dt
        E.append(0.5 * v @ (s.M * v) + 0.5 * ps[n + 1] @ s.apply_K(ps[n]))
    E = np.array(E)
    assert E.min() > 0
    assert np.max(np.abs(E - E[0])) < 1e-11 * E[0]


def _mode(xyz, L, l=1, m=0, n=0):
    return (np.cos(l * math.pi * xyz[:, 0] / L[0]) * np.cos(m * math.pi * xyz[:, 1] / L[1])
            * np.cos(n * math.pi * xyz[:, 2] / L[2]))


def test_cavity_eigenmode_spectral_convergence():
    """Rayleigh quotient of the interpolated rigid-box mode -> c^2 k^2 spectrally in N."""
    L = np.array([0.6e-3, 0.6e-3, 0.6e-3])
    c = 1500.0
    k2 = (math.pi / L[0]) ** 2 + (math.pi / L[2]) ** 2
    errs = []
    for N in (2, 3, 4, 5, 6):
        s = System(cavity_config(nel=(2, 2, 2), degree=N, extent=tuple(L)))
        p = _mode(s.node_coords(), L, 1, 0, 1)
        lam = p @ s.apply_K(p) / (p @ (s.M * p))
        errs.append(abs(lam - c * c * k2) / (c * c * k2))
    errs = np.array(errs)
    assert np.all(np.diff(np.log10(errs)) < -0.9)           # at least 8x per degree
    assert errs[-1] < 1e-6


def test_cavity_mode_time_series():
    """Config-0 box, (1,0,0) mode at f = c/(2 L) = 1.25 MHz: the discrete evolution is
    cos(w_h t) p0 with 2(1 - cos w_h dt) = dt^2 lambda_h (lambda_h the Rayleigh quotient)."""
    rec = cavity_config(nel=(4, 4, 4), degree=4, extent=(0.6e-3,) * 3)
    rec["dt"] = config(0)["dt"]
    s = System(rec)
    xyz = s.node_coords()
    p0 = _mode(xyz, [0.6e-3] * 3)
    lam = p0 @ s.apply_K(p0) / (p0 @ (s.M * p0))
    dt = rec["dt"]
    wh = math.acos(1 - dt * dt * lam / 2) / dt
    assert abs(wh / (2 * math.pi) - 1.25e6) < 1e-4 * 1.25e6
    nm = Newmark(s)
    nm.set_state(p0, np.zeros_like(p0))
    # Algorithm 1 with pdd^0 = 0 (R20) starts from p^1 = p^0 (not the cos-shifted value); compare
    # against the exact discrete recursion's solution  p^n = p0 (cos(w n dt) + A sin(w n dt))
    # where A makes p^1 = p^0:  cos(w dt) + A sin(w dt) = 1.
    A = (1 - math.cos(wh * dt)) / math.sin(wh * dt)
    for n in range(1, 401):
        nm.step()
        if n % 100 == 0:
            ref = p0 * (math.cos(wh * n * dt) + A * math.sin(wh * n * dt))
            assert np.linalg.norm(nm.p - ref) < 1e-5 * np.linalg.norm(p0)


def test_conforming_cut_matches_single_box():
    """A conforming mesh cut by the DG interface (same N, h both sides) reproduces the single CG
    box up to discretisation error that shrinks spectrally in N."""
    diffs = []
    for N in (3, 5):
        h = 1e-4
        cut = conforming_cut_config(nel_xy=2, nz_lo=2, nz_hi=2, degree=N, ratio=1, h=h)
        one = cavity_config(nel=(2, 2, 4), degree=N, extent=(2 * h, 2 * h, 4 * h))
        dt = min(cut["dt"], one["dt"])
        cut["dt"] = one["dt"] = dt
        L = [2 * h, 2 * h, 4 * h]
        sc, so = System(cut), System(one)
        res = []
        for s in (sc, so):
            xyz = s.node_coords()
            nm = Newmark(s)
            nm.set_state(_mode(xyz, L, 0, 0, 1), np.zeros(s.ndof))
            nm.run(int(round(0.25 * 4 * h / 1500 / dt)))
            res.append((xyz, nm.p.copy()))
        (xc, pc), (xo, po) = res
        # compare at the single box's nodes: the cut's lower box holds z <= 2h exactly
        lo = sc.offsets[1]
        key = {tuple(np.round(x / h * 1e9).astype(np.int64)): i for i, x in enumerate(xo)}
        idx = np.array([key[tuple(np.round(x / h * 1e9).astype(np.int64))] for x in xc[:lo]])
        diffs.append(np.max(np.abs(pc[:lo] - po[idx])) / np.max(np.abs(po)))
    assert diffs[1] < diffs[0] / 10
    assert diffs[1] < 1e-4


def _oscillator_record(dt_scale=1.0, amp=0.0):
    rec = config(0)
    rec["boxes"][0]["rho"] = 0.0            # kappa = rho c^2 = 0: PMUTs decoupled from the fluid
    rec["dt"] *= dt_scale
    rec["pmut"]["amp_v"] = amp
    rec["pmut"]["delay_s"] = np.zeros(len(rec["pmut"]["delay_s"]))
    return rec


@pytest.mark.parametrize("zeta", [0.0, 0.01])
def test_unloaded_pmut_free_decay(zeta):
    """q(t) = q0 e^{-zeta w t} (cos w_d t + zeta/sqrt(1-zeta^2) sin w_d t).  Undamped (the paper's
    Eq. 2): second order.  With the config's damping evaluated at the predictor velocity (R3, like
    C pd^{n+1} at P:L625) the damping term is first order in dt."""
    errs = []
    for scale in (0.25, 0.125):
        rec = _oscillator_record(scale)
        rec["pmut"]["damping"] = np.full(3, zeta)
        nm = Newmark(System(rec))
        nm.q[:] = 1e-9
        # consistent initial acceleration for a non-zero initial displacement (reading R20);
        # Algorithm 1's qdd^0 = 0 is consistent only for the zero initial state
        nm.qdd[:] = -(2 * math.pi * rec["pmut"]["freq_hz"]) ** 2 * 1e-9
        w = 2 * math.pi * rec["pmut"]["freq_hz"]
        z = rec["pmut"]["damping"][None, :]
        wd = w * np.sqrt(1 - z * z)
        err = 0.0
        for _ in range(int(round(2e-7 / rec["dt"]))):
            nm.step()
            t = nm.n * rec["dt"]
            ref = 1e-9 * np.exp(-z * w * t) * (np.cos(wd * t) + z / np.sqrt(1 - z * z) * np.sin(wd * t))
            err = max(err, np.max(np.abs(nm.q - ref)) / 1e-9)
        assert np.all(nm.p == 0)
        errs.append(err)
    assert errs[0] < 5e-3
    if zeta == 0.0:
        assert 3.5 < errs[0] / errs[1] < 5.5                 # second order
    else:
        assert 1.8 < errs[0] / errs[1] < 4.5                 # first order in the damping term


@pytest.mark.parametrize("zeta", [0.0, 0.01])
def test_unloaded_pmut_hann_duhamel(zeta):
    """Forced response to the Hann burst = Duhamel integral of eta phi(t)/M_m (O(dt^2) undamped)."""
    errs = []
    for scale in (0.5, 0.25):
        rec = _oscillator_record(scale, amp=5.0)
        pm = rec["pmut"]
        pm["damping"] = np.full(3, zeta)
        nm = Newmark(System(rec))
        T = 1.2e-6
        nm.run(int(round(T / rec["dt"])))
        t = nm.n * rec["dt"]
        k = 0
        ref = []
        s = np.linspace(0, t, 200001)
        om0 = 2 * math.pi * pm["f0_hz"]
        tp = s
        win = (tp <= pm["n_cycles"] / pm["f0_hz"])
        phi = np.where(win, pm["amp_v"] * np.sin(om0 * tp) * 0.5 * (1 - np.cos(om0 * tp / pm["n_cycles"])), 0)
        for m in range(3):
            w = 2 * math.pi * pm["freq_hz"][k, m]
            z = pm["damping"][m]
            wd = w * math.sqrt(1 - z * z)
            h = np.exp(-z * w * (t - s)) * np.sin(wd * (t - s)) / wd
            F = pm["eta"][m] * phi / pm["modal_mass"][m]
            ref.append(np.trapezoid(h * F, s))
        ref = np.array(ref)
        errs.append(np.max(np.abs(nm.q[k] - ref)) / np.max(np.abs(ref)))
    assert errs[0] < 2e-2
    lo = 3.5 if zeta == 0.0 else 1.8
    assert lo < errs[0] / errs[1] < 5.5


def test_rx_feedback_coupled_modes_closed_form():
    """Open-circuit RX feedback (Eq. 3 second line): with kappa = 0, zeta = 0 and
    phi = (1/C) sum_n eta q_n, the modes obey q'' = -A q with A = diag(w^2) - (eta^2/(M_m C)) 1 1^T,
    so q(t) = V cos(sqrt(Lambda) t) V^-1 q0 (q'(0) = 0).  C is chosen so the feedback is ~30% of
    w_1^2 (the config's C = 1e-10 F would shift w^2 by 3e-7 only); the scheme is second order."""
    errs = []
    for scale in (0.25, 0.125):
        rec = _oscillator_record(scale)
        pm = rec["pmut"]
        pm["damping"] = np.zeros(3)
        pm["rx"], pm["t_switch"] = True, 0.0
        w = 2 * math.pi * pm["freq_hz"][0]
        Mm, eta = pm["modal_mass"][0], pm["eta"][0]
        pm["capacitance"] = eta * eta / (Mm * 0.3 * w[0] ** 2)
        A = np.diag(w ** 2) - (eta * eta / (Mm * pm["capacitance"])) * np.ones((3, 3))
        lam, V = np.linalg.eigh(A)
        assert np.all(lam > 0)
        q0 = np.array([1e-9, 0.5e-9, -0.3e-9])
        nm = Newmark(System(rec))
        nm.q[0] = q0
        nm.qdd[0] = -A @ q0                  # consistent initial acceleration (reading R20)
        err = 0.0
        for _ in range(int(round(1e-6 / rec["dt"]))):
            nm.step()
            t = nm.n * rec["dt"]
            ref = V @ (np.cos(np.sqrt(lam) * t) * (V.T @ q0))
            err = max(err, np.max(np.abs(nm.q[0] - ref)) / 1e-9)
        assert np.all(nm.p == 0)
        # the received voltage is the feedback itself
        assert abs(nm.v_rx()[0] - eta * nm.q[0].sum() / pm["capacitance"]) <= 1e-12 * abs(nm.v_rx()[0]) + 1e-30
        errs.append(err)
    assert errs[0] < 2e-2
    assert 3.5 < errs[0] / errs[1] < 4.5                     # second order


def test_drive_window():
    pm = config(1)["pmut"]
    tau = pm["delay_s"]
    T = pm["n_cycles"] / pm["f0_hz"]
    t = np.linspace(-1e-7, 2e-6, 3001)
    v = np.array([drive(pm, ti) for ti in t])           # (nt, n_pmut)
    for k in range(len(tau)):
        off = (t < tau[k]) | (t > tau[k] + T)
        assert np.all(v[off, k] == 0)
        assert np.max(np.abs(v[:, k])) <= pm["amp_v"]
        assert np.max(np.abs(v[:, k])) > 0.8 * pm["amp_v"]


def test_abc_normal_incidence():
    """First-order ABC (Eq. 8): an up-going plane pulse leaves through the top face; the energy
    left in the column after it has passed is a small fraction of the incident energy."""
    h = 50e-6
    rec = cavity_config(nel=(1, 1, 24), degree=4, extent=(h, h, 24 * h))
    rec["boxes"][0]["bc"][5] = 1
    s = System(rec)
    xyz = s.node_coords()
    z = xyz[:, 2]
    c = 1500.0
    w = 3 * h
    z0 = 8 * h
    G = np.exp(-((z - z0) / w) ** 2)
    dG = -2 * (z - z0) / w ** 2 * G
    nm = Newmark(s)
    nm.set_state(G, -c * dG)                            # p = G(z - c t): up-going
    E0 = nm.energy()
    nm.run(int(round((24 * h - z0 + 4 * w) / c / rec["dt"])))
    assert nm.energy() < 1e-2 * E0


def test_plane_wave_source_normal_incidence():
    """Total-field ABC with incident data (reading R13) at normal incidence into a rigid-bottom
    column: mid-column p follows A s(t - (z_top - z)/c), doubling at the rigid bottom."""
    h = 50e-6
    nz = 24
    rec = cavity_config(nel=(1, 1, nz), degree=4, extent=(h, h, nz * h))
    rec["boxes"][0]["bc"][5] = 1
    f0 = 3e6
    sig = 1 / (2 * f0)
    rec["plane_wave"] = {"box": 0, "face": 5, "amp_pa": 1e3, "f0_hz": f0, "sigma_s": sig, "t0_s": 4 * sig,
                         "direction": (0.0, 0.0, -1.0)}
    s = System(rec)
    xyz = s.node_coords()
    c = 1500.0
    top = nz * h
    zm = 16 * h
    im = np.argmin(np.abs(xyz[:, 2] - zm) + np.abs(xyz[:, 0]) + np.abs(xyz[:, 1]))
    ib = np.argmin(np.abs(xyz[:, 2]) + np.abs(xyz[:, 0]) + np.abs(xyz[:, 1]))
    nm = Newmark(s)
    dt = rec["dt"]

    def src(t):
        u = t - 4 * sig
        return 1e3 * np.exp(-u * u / (2 * sig * sig)) * np.sin(2 * math.pi * f0 * u)

    t_echo = (top + zm) / c                              # reflection from the bottom returns to zm
    mid, bot, ref_mid, ref_bot = [], [], [], []
    n_end = int(round(((top) / c + 8 * sig) / dt))
    for _ in range(n_end):
        nm.step()
        t = nm.n * dt
        if t < t_echo - 4 * sig:
            mid.append(nm.p[im])
            ref_mid.append(src(t - (top - zm) / c))
        bot.append(nm.p[ib])
        ref_bot.append(2 * src(t - top / c))
    mid, ref_mid, bot, ref_bot = map(np.array, (mid, ref_mid, bot, ref_bot))
    assert np.max(np.abs(mid - ref_mid)) < 0.03 * 1e3
    assert abs(np.max(np.abs(bot)) - np.max(np.abs(ref_bot))) < 0.03 * 2e3
    assert np.max(np.abs(bot - ref_bot)) < 0.06 * 2e3


def test_literal_coupling_diverges_predicted_bounded():
    """Evidence for reading R2 on config 0: Algorithm 1 read literally (g(p^n, phi^n)) grows
    without bound at the configured modal mass; the predicted ordering stays bounded."""
    rec = config(0)
    s = System(rec)
    amp = {}
    for cp in ("literal", "predicted"):
        nm = Newmark(s, coupling=cp).run(1200)
        amp[cp] = np.abs(nm.q).max()
    assert amp["literal"] > 1e3 * amp["predicted"]
    assert amp["predicted"] < 1e-9


def _oblique_column(x_ref=None):
    """Laterally wide, one-element-thick box, rigid bottom and sides, total-field ABC top with an
    incident plane pulse at 20 deg (reading R13).  Returns (system, time axis, histories at three
    observation points, their coordinates)."""
    h, nel_x, nz = 50e-6, 80, 24
    rec = cavity_config(nel=(nel_x, 1, nz), degree=3, extent=(nel_x * h, h, nz * h), cfl=0.45)
    rec["boxes"][0]["bc"][5] = 1
    f0 = 5e6
    sig = 1 / (2 * f0)
    th = math.radians(20.0)
    rec["plane_wave"] = {"box": 0, "face": 5, "amp_pa": 1e3, "f0_hz": f0, "sigma_s": sig, "t0_s": 4 * sig,
                         "direction": (math.sin(th), 0.0, -math.cos(th)), "x_ref": x_ref}
    s = System(rec)
    xyz = s.node_coords()
    top = nz * h
    # observation points (x, depth below the top): far enough from the source corner, the downstream
    # wall and the rigid bottom that no diffracted or reflected wave reaches them inside the window
    obs = [(1.9e-3, 0.6e-3), (2.4e-3, 0.6e-3), (2.4e-3, 0.4e-3)]
    ids = [int(np.argmin(np.abs(xyz[:, 0] - X) + np.abs(xyz[:, 2] - (top - d)) + np.abs(xyz[:, 1])))
           for X, d in obs]
    dt = rec["dt"]
    n = int((7 * sig + (2.6e-3 * math.sin(th) + 0.6e-3 * math.cos(th)) / 1500.0) / dt)
    nm = Newmark(s)
    hist = []
    for _ in range(n):
        nm.step()
        hist.append(nm.p[ids])
    return s, dt * np.arange(1, n + 1), np.array(hist), xyz[ids], (f0, sig, th, top)


def test_plane_wave_source_oblique_incidence():
    """Reading R13 away from normal incidence (k = (sin 20, 0, -cos 20)): the injected field is the
    plane wave A s(t - k.(x - x_ref)/c) itself (the total-field ABC data makes the incident wave satisfy
    the boundary condition exactly, so nothing is reflected at the top), which fixes
      * the waveform and amplitude at interior points (the (1 - n.k) factor),
      * the delay law's sign: arrivals along x are later by dx sin(th)/c (trace speed c/sin th),
      * the depth trace: arrivals deeper by dz are later by dz cos(th)/c (trace speed c/cos th),
      * x_ref = the top corner the wavefront reaches first: with the other corner the absolute timing
        is off by L_x sin(th)/c and the waveform check fails."""
    s, t, hist, pts, (f0, sig, th, top) = _oblique_column()
    c = 1500.0
    kd = np.array([math.sin(th), 0.0, -math.cos(th)])
    xref = np.array([0.0, 0.0, top])
    assert np.allclose(s.pw_xref, xref)

    def src(u):
        u = u - 4 * sig
        return 1e3 * np.exp(-u * u / (2 * sig * sig)) * np.sin(2 * math.pi * f0 * u)

    for j in range(3):
        ref = src(t - (pts[j] - xref) @ kd / c)
        assert np.max(np.abs(hist[:, j])) > 0.8e3
        assert np.max(np.abs(hist[:, j] - ref)) < 0.03e3, j

    def centroid(v):   # energy-centroid arrival time of a pulse
        return float(np.sum(t * v * v) / np.sum(v * v))

    ta = [centroid(hist[:, j]) for j in range(3)]
    dx = pts[1][0] - pts[0][0]
    assert abs((ta[1] - ta[0]) - dx * math.sin(th) / c) < 0.02 * dx * math.sin(th) / c
    depth_delay = (pts[2][2] - pts[1][2]) * math.cos(th) / c
    assert abs((ta[1] - ta[2]) - depth_delay) < 0.02 * abs(depth_delay)

    # the other top corner as x_ref: the same delay law, shifted by L_x sin(th)/c -> visibly wrong
    s2, t2, hist2, pts2, _ = _oblique_column(x_ref=(4e-3, 0.0, top))
    ref = src(t2 - (pts2[1] - xref) @ kd / c)
    assert np.max(np.abs(hist2[:, 1] - ref)) > 0.5e3
