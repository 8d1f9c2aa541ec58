"""Full-length parity for configs whose oracle run exceeds a GPU-box call: the GPU run and the oracle
run are made separately (the oracle on any host), each saving the pressure at the same seeded uniform
sample of nodes per box plus the modal state; --compare reports the sampled relative L2 errors.

  python tools/full_run_sampled.py gpu    CFG OUT.npz [steps]
  python tools/full_run_sampled.py oracle CFG OUT.npz [steps]
  python tools/full_run_sampled.py compare GPU.npz ORACLE.npz
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from sem_inputs import config, total_dof  # noqa: E402
from sem_inputs.workloads import box_dof  # noqa: E402

N_SAMPLE = 1_000_000


def sample_ids(rec):
    rng = np.random.default_rng(2026)
    return [np.sort(rng.choice(box_dof(b), size=min(N_SAMPLE, box_dof(b)), replace=False)) for b in rec["boxes"]]


def main():
    mode = sys.argv[1]
    if mode == "compare":
        a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
        out = {}
        for k in a.files:
            if k.startswith("p") or k in ("q", "qd"):
                x, r = a[k].ravel(), b[k].ravel()
                out[k] = float(np.linalg.norm(x - r) / max(np.linalg.norm(r), 1e-300))
        out["max"] = max(out.values())
        out["pass_1e-11"] = bool(out["max"] <= 1e-11)
        out["note"] = f"relative L2 over a seeded uniform sample of {N_SAMPLE} nodes per box (all of q)"
        print(json.dumps(out))
        return
    ci, path = int(sys.argv[2]), sys.argv[3]
    rec = config(ci)
    n = int(sys.argv[4]) if len(sys.argv) > 4 else rec["n_steps"]
    ids = sample_ids(rec)
    t0 = time.perf_counter()
    save = {"steps": n}
    if mode == "gpu":
        from parity import gpu_run
        sim = gpu_run(rec, n)
        for b in range(len(rec["boxes"])):
            save[f"p{b}"] = sim.pressure_at(b, ids[b])
        q, qd, _ = sim.modal()
        save["q"], save["qd"] = q, qd
    else:
        from parity import oracle_run
        nm = oracle_run(rec, n)
        for b, pb in enumerate(nm.sys.split(nm.p)):
            save[f"p{b}"] = pb[ids[b]]
        save["q"], save["qd"] = nm.q, nm.qd
    save["wall_s"] = time.perf_counter() - t0
    np.savez(path, **save)
    print(json.dumps({"mode": mode, "config": ci, "steps": n, "dof": total_dof(rec), "wall_s": save["wall_s"]}))


if __name__ == "__main__":
    main()
