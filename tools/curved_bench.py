"""Throughput of the curved-box (element-scatter) path vs the structured path on the same box, and of
the same (affine) box with a rigid obstacle (a centred block of 1/3 x 1/3 x 1/3 of the elements).
python tools/curved_bench.py [nel_x nel_y nel_z degree steps] -> one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_06267_b200 import Simulation, sem_kernel_time, sem_set_profiling  # noqa: E402
from sem_inputs import BC_ABSORBING, curved_config, solid_block  # noqa: E402

a = [int(v) for v in sys.argv[1:]] or [96, 96, 24, 5, 20]
nel, N, steps = tuple(a[:3]), a[3], a[4]
rec = curved_config(nel=nel, degree=N, extent=tuple(25e-6 * n for n in nel), bc_top=BC_ABSORBING, seed=None)
out = {"what": "curved box (element scatter, metric recomputed) vs the same box structured", "nel": nel, "degree": N}
for name in ("curved", "structured", "obstacle"):
    r = dict(rec)
    r["boxes"] = [dict(rec["boxes"][0])]
    if name != "curved":
        r["boxes"][0]["vertices"] = None
    if name == "obstacle":
        r["boxes"][0]["solid"] = solid_block(nel, [n // 3 for n in nel], [n - n // 3 for n in nel])
    t0 = time.perf_counter()
    sim = Simulation(r)
    setup = time.perf_counter() - t0
    sim.fill_random_state(0, 3, 1.0, 1e3)
    sim.step(3)
    sim.sync()
    sem_set_profiling(sim.ctx, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sim.step(steps)
    sim.sync()
    e1.record()
    torch.cuda.synchronize()
    vol_ms, n = sem_kernel_time(sim.ctx, 0)
    ndof = sim.ndof[0]
    out[name] = {"dof": ndof, "setup_s": setup, "ms_per_step": vol_ms / max(n, 1),
                 "gdof_per_s": ndof / (vol_ms / max(n, 1) / 1e3) / 1e9}
    if name == "obstacle":
        out[name]["solid_elements"] = int(len(r["boxes"][0]["solid"]))
        out[name]["note"] = "DOF counts the whole lattice (obstacle interiors included)"
    sim.close()
out["ratio_structured_over_curved"] = out["structured"]["gdof_per_s"] / out["curved"]["gdof_per_s"]
print(json.dumps(out))
