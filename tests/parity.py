"""Shared helpers of the GPU parity tests (tests only)."""
import math

import numpy as np

TOL = 1e-11   # BASELINE.json north_star: relative L2 <= 1e-11 on pressure and modal amplitudes


def rel_l2(x, ref, s_phys=0.0):
    """Reading R21: ||x - ref|| / max(||ref||, sqrt(n) s_phys)."""
    x = np.asarray(x, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    den = max(np.linalg.norm(ref), math.sqrt(ref.size) * s_phys)
    if den == 0.0:
        return float(np.linalg.norm(x))
    return float(np.linalg.norm(x - ref) / den)


def oracle_run(rec, n_steps, state=None, coupling=None):
    from oracle.newmark import Newmark
    from oracle.operators import System
    nm = Newmark(System(rec), coupling=coupling)
    if state is not None:
        nm.set_state(np.concatenate([s[0] for s in state]), np.concatenate([s[1] for s in state]))
    return nm.run(n_steps)


def gpu_run(rec, n_steps, state=None, flags=0, chunks=None, world=1):
    from paper_2603_06267_b200 import Simulation
    sim = Simulation(rec, flags=flags, world=world)
    if state is not None:
        for b, (p, v) in enumerate(state):
            sim.write_state(b, p, v)
    if chunks is None:
        sim.step(n_steps)
    else:
        done = 0
        for c in chunks:
            sim.step(c)
            done += c
        assert done == n_steps
    return sim


def compare(sim, nm, s_phys_q=1e-9):
    """Per-box pressure relL2 and modal relL2 (floor-guarded, R21)."""
    out = {}
    for b in range(len(sim.ndof)):
        ref = nm.sys.split(nm.p)[b]
        out[f"p{b}"] = rel_l2(sim.pressure(b), ref)
    if nm.sys.pm is not None:
        q, qd, v = sim.modal()
        out["q"] = rel_l2(q, nm.q, s_phys_q)
        out["qd"] = rel_l2(qd, nm.qd, s_phys_q / nm.dt * 1e-3)
        out["v"] = rel_l2(v, nm.v_rx(), 1e-6)
    return out
