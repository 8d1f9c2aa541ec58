"""Algorithm 1 (Newmark gamma=1/2, beta=0) for Eqs. (9)-(12), literally (oracle; test infrastructure only).

P:L605-633, three vectors per field:

    q^{n+1}   = q^n + dt qd^n + dt^2/2 qdd^n            (PMUT predictor, L615)
    qd^{n+1}  = qd^n + dt/2 qdd^n                        (L617)
    qdd^{n+1} = -W q^{n+1} + g(p, phi)                   (PMUT solve, L619)
    qd^{n+1} += dt/2 qdd^{n+1}                           (corrector, L621)
    p^{n+1}   = p^n + dt pd^n + dt^2/2 pdd^n             (acoustic predictor, L623)
    pd^{n+1}  = pd^n + dt/2 pdd^n                        (L624)
    pdd^{n+1} = M^{-1} (f(qdd^{n+1}) - K p^{n+1} - C pd^{n+1})   (L625)
    pd^{n+1} += dt/2 pdd^{n+1}                           (L626)

Readings:
  R1  S loop bodies n = 0..S-1; the result is p^S at t = S dt.
  R2  coupling='predicted' (default): the PMUT solve consumes p^{n+1} (the acoustic predictor,
      which does not depend on qdd^{n+1}) and phi^{n+1}; coupling='literal' consumes p^n, phi^n
      exactly as printed at L619.
  R3  the modal ODE carries the config's modal mass M_m and damping zeta:
      qdd = -w^2 q - 2 zeta w qd* + (int p U.n + eta phi) / M_m, qd* the predictor velocity.
  R13 configs with a plane-wave source add b(t^{n+1}) to f.
  R20 pdd^0 = 0 (L609-610) also for non-zero initial (p, pd) used by tests.
"""
from __future__ import annotations

import math

import numpy as np


def drive(pm, t):
    """phi_{k,0}(t): TX tone burst A sin(2 pi f0 t') (1 - cos(2 pi f0 t'/n_c))/2 for
    t' = t - tau_k in [0, n_c/f0], else 0 (reading R10; parity unpinned: config constant)."""
    tp = t - pm["delay_s"]
    T = pm["n_cycles"] / pm["f0_hz"]
    om = 2 * math.pi * pm["f0_hz"]
    on = (tp >= 0) & (tp <= T)
    return np.where(on, pm["amp_v"] * np.sin(om * tp) * 0.5 * (1 - np.cos(om * tp / pm["n_cycles"])), 0.0)


def voltage(pm, t, q):
    """phi_k(t) (Eq. 3 second line): drive for t <= t_bar, (1/C) sum_m eta_m q_m after."""
    if t <= pm["t_switch"]:
        return drive(pm, t)
    return (q * pm["eta"][None, :]).sum(axis=1) / pm["capacitance"]


def _div_mass(r, M):
    """M^-1 r for the lumped mass; nodes outside the fluid (M = 0, obstacle interiors) get 0."""
    out = np.zeros_like(r)
    np.divide(r, M, out=out, where=M > 0)
    return out


class Newmark:
    """State and loop of Algorithm 1 for a ``operators.System``."""

    def __init__(self, system, coupling=None):
        self.sys = system
        rec = system.rec
        self.dt = float(rec["dt"])
        self.coupling = coupling or rec.get("coupling", "predicted")
        n = system.ndof
        self.p = np.zeros(n)
        self.pd = np.zeros(n)
        self.pdd = np.zeros(n)
        self.n = 0
        # PML auxiliaries (Eq. 1 lines 2-3; readings R23-R25 in oracle/pml.py)
        self.pml = None
        if rec.get("pml") is not None:
            from .pml import Pml
            self.pml = Pml(system, rec["pml"])
        pm = system.pm
        if pm is not None:
            shape = pm["freq_hz"].shape
            self.q = np.zeros(shape)
            self.qd = np.zeros(shape)
            self.qdd = np.zeros(shape)
            self.omega = 2 * math.pi * pm["freq_hz"]
            self.zeta = pm["damping"][None, :]
            self.mass = pm["modal_mass"][None, :]
            self.eta = pm["eta"][None, :]

    def set_state(self, p, pd):
        """Initial p^0, pd^0 (tests); pdd^0 = 0 (R20)."""
        self.p = np.array(p, dtype=np.float64)
        self.pd = np.array(pd, dtype=np.float64)
        self.pdd = np.zeros_like(self.p)

    def _pmut_solve(self, q1, qd1, p_used, t_used, q_used):
        s = self.sys
        pm = s.pm
        load = -s.pmut_project(p_used)                      # int p U.n = -B p (R4)
        phi = voltage(pm, t_used, q_used)[:, None]
        return (-self.omega ** 2 * q1 - 2 * self.zeta * self.omega * qd1
                + (load + self.eta * phi) / self.mass)

    def step(self):
        s, dt = self.sys, self.dt
        tn, tn1 = self.n * dt, (self.n + 1) * dt
        have_pmut = s.pm is not None
        p1 = self.p + dt * self.pd + 0.5 * dt * dt * self.pdd
        pd1 = self.pd + 0.5 * dt * self.pdd
        f = np.zeros(s.ndof)
        if have_pmut:
            q1 = self.q + dt * self.qd + 0.5 * dt * dt * self.qdd
            qd1 = self.qd + 0.5 * dt * self.qdd
            if self.coupling == "literal":
                qdd1 = self._pmut_solve(q1, qd1, self.p, tn, self.q)
            else:
                qdd1 = self._pmut_solve(q1, qd1, p1, tn1, q1)
            qd1 = qd1 + 0.5 * dt * qdd1
            f += s.pmut_force(qdd1)
        f += s.plane_wave_load(tn1)
        inactive = ~s.active                                  # obstacle interiors (no fluid element)
        if inactive.any():
            p1[inactive] = 0.0
            pd1[inactive] = 0.0
        if self.pml is None:
            pdd1 = _div_mass(f - s.apply_K(p1) - s.C * pd1, s.M)
        else:   # R25: PML terms at the predictor velocity, psi^{n+1} and Phi^{n+1}
            rB, psi1 = self.pml.advance(p1, dt)
            pm_ = self.pml
            pdd1 = (_div_mass(f - s.apply_K(p1) - s.C * pd1 - rB, s.M)
                    - pm_.alpha * pd1 - pm_.beta * p1 - pm_.gamma * psi1)
        pd1 = pd1 + 0.5 * dt * pdd1
        self.p, self.pd, self.pdd = p1, pd1, pdd1
        if have_pmut:
            self.q, self.qd, self.qdd = q1, qd1, qdd1
        self.n += 1

    def run(self, n_steps):
        for _ in range(n_steps):
            self.step()
        return self

    def v_rx(self):
        """phi_k at t^n (received voltage for RX, drive for TX)."""
        return voltage(self.sys.pm, self.n * self.dt, self.q)

    def energy(self):
        """E = 1/2 pd^T M pd + 1/2 p^T K p (continuous-in-time energy of Eq. 9 without sources)."""
        return 0.5 * self.pd @ (self.sys.M * self.pd) + 0.5 * self.p @ self.sys.apply_K(self.p)


def run_record(rec, n_steps=None, coupling=None, state=None):
    """Convenience: build the system, optionally set (p, pd), run, return the Newmark object."""
    from .operators import System
    nm = Newmark(System(rec), coupling=coupling)
    if state is not None:
        nm.set_state(np.concatenate([s[0] for s in state]), np.concatenate([s[1] for s in state]))
    return nm.run(rec["n_steps"] if n_steps is None else n_steps)
