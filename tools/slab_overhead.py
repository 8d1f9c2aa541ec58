"""Cost of the y-slab decomposition measured on one GPU (SEM_F_EMULATE_SLABS: all G slabs in one
context, exchange by device copies): ms/step of cfg 3 for G = 1, 2, 4, 8 slabs processed back to
back.  The G-slab time divided by G approximates one rank's compute per step at G GPUs (the NCCL
exchange of ~3 MB per neighbour runs on a second stream beside the volume kernel)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06267_b200 import SEM_F_EMULATE_SLABS, SEM_F_NO_GRAPH, Simulation  # noqa: E402
from sem_inputs import config  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ci = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rec = config(ci)
from paper_2603_06267_b200.sem import sem_slab_plan  # noqa: E402
out = {"what": f"cfg{ci} y-slab decomposition emulated on one GPU", "steps": steps}
base = None
for G in (1, 2, 4, 8):
    out.setdefault("plans", {})[f"G{G}"] = sem_slab_plan(rec["boxes"], G, rec.get("pmut"))
    flags = SEM_F_EMULATE_SLABS if G > 1 else 0
    sim = Simulation(rec, world=G, flags=flags)
    sim.step(3)
    sim.sync()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sim.step(steps)
    sim.sync()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    base = ms if base is None else base
    out[f"G{G}"] = {"ms_per_step_all_slabs": ms, "ms_per_slab_step": ms / G,
                    "overhead_vs_1": ms / base - 1.0}
    sim.close()
print(json.dumps(out))
