"""Measure GPU Algorithm 3 (sem_face_match) on config 3's interface: 384 x 384 fine faces (N = 5,
36 nodes each = 5.3M quadrature nodes) against 192 x 192 coarse faces, structured and jittered;
the oracle's literal loop timed on a small sample for context.  Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2603_06267_b200 import sem_face_match  # noqa: E402
from sem_inputs import interface_faces  # noqa: E402

out = {"what": "Algorithm 3 face matching (P:L1062-1080) on cfg3's interface", "degree": 5}
for name, jit in (("structured", 0.0), ("jittered", 0.15)):
    fine, coarse = interface_faces(384, 384, 2, 25e-6, z0=0.6e-3, jitter=jit, seed=5)
    sem_face_match(fine[:64], coarse, 5)                     # warm-up (context, module load)
    t0 = time.perf_counter()
    owner, xi, ms = sem_face_match(fine, coarse, 5)
    wall = time.perf_counter() - t0
    n = owner.size
    out[name] = {"fine_faces": len(fine), "coarse_faces": len(coarse), "nodes": n, "unmatched": int((owner < 0).sum()),
                 "device_ms": ms, "nodes_per_s": n / (ms / 1e3), "call_wall_s": wall}
from oracle.matching import match_faces  # noqa: E402
fine, coarse = interface_faces(16, 16, 2, 25e-6, z0=0.6e-3, jitter=0.15, seed=5)
t0 = time.perf_counter()
match_faces(fine, coarse, 5)
dt = time.perf_counter() - t0
out["oracle_sample"] = {"fine_faces": len(fine), "coarse_faces": len(coarse), "seconds": dt,
                        "nodes_per_s": len(fine) * 36 / dt}
out["paper_context"] = "P:L1447: 318,698 interfaces, 315 CPU processes: ~160,000 s naive -> ~630 s optimised (setup)"
print(json.dumps(out))
