"""Full-length parity of one BASELINE config: GPU (libsem) vs the CPU oracle after the configured number
of steps (the north star's bar: relative L2 <= 1e-11 on every box's pressure and on the modal
amplitudes).  python tools/full_run_parity.py [config] [steps] -> one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

from parity import compare, gpu_run, oracle_run  # noqa: E402
from sem_inputs import config  # noqa: E402

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rec = config(ci)
n = int(sys.argv[2]) if len(sys.argv) > 2 else rec["n_steps"]
t0 = time.perf_counter()
sim = gpu_run(rec, n)
sim.sync()
t_gpu = time.perf_counter() - t0
t0 = time.perf_counter()
nm = oracle_run(rec, n)
t_orc = time.perf_counter() - t0
r = compare(sim, nm)
out = {"config": f"cfg{ci}", "steps": n, "dof": int(sum(sim.ndof)), "relL2": r,
       "max_relL2": max(r.values()), "pass_1e-11": bool(max(r.values()) <= 1e-11),
       "oracle_max_abs_p": float(np.abs(nm.p).max()), "oracle_max_abs_q": float(np.abs(nm.q).max()),
       "gpu_wall_s": t_gpu, "oracle_wall_s": t_orc}
print(json.dumps(out))
