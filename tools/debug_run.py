"""Every kernel family on small cases, for the bounds-checked build (SEM_LIB=.../libsem_debug.so):
PMUT (cfg 0), 2:1 interface (fused and generic, both quadrature rules), RX + plane wave (cfg 4s), PML
(also under 2 slabs), curved box, obstacle, emulated slab decompositions (even and uneven), face
matching, the general interface, PMUTs on curved and obstacle boxes, the two-box cylinder (caller-defined
shapes, plane wave on a curved box).  Prints "debug run ok"."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_06267_b200 import LIB_PATH, SEM_F_EMULATE_SLABS, Simulation, sem_face_match  # noqa: E402
from sem_inputs import (conforming_cut_config, config, curved_config, curved_interface_config,  # noqa: E402
                        curved_pmut_config, interface_faces, obstacle_config, obstacle_pmut_config, pml_config,
                        random_state, small_config, cylinder_two_box_config, plane_wave_source)

print("library:", LIB_PATH)
cases = [(config(0), {}), (small_config("cfg2s"), {}), (small_config("cfg4s"), {}),
         (dict(small_config("cfg2s"), interface=dict(small_config("cfg2s")["interface"], quad="lg")), {}),
         (conforming_cut_config(nel_xy=6, nz_lo=2, nz_hi=2, degree=3, degree_hi=2, ratio=3, h=25e-6), {}),
         (pml_config(nel=(3, 3, 4), degree=3), {}), (curved_config(nel=(3, 2, 2), degree=4, seed=2), {}),
         (obstacle_config(nel=(4, 4, 3), degree=2, solid_lo=(1, 1, 1), solid_hi=(3, 3, 2)), {}),
         (small_config("cfg2s"), {"world": 2, "flags": SEM_F_EMULATE_SLABS}),
         (curved_interface_config(jitter=0.15, seed=3), {}), (curved_pmut_config(), {}),
         (obstacle_pmut_config(), {}), (config(1), {"world": 4, "flags": SEM_F_EMULATE_SLABS}),
         (pml_config(nel=(3, 6, 3), degree=3, layers=(1, 1, 1, 1, 0, 1), layer_el=1), {"world": 2, "flags": SEM_F_EMULATE_SLABS})]
cyl = cylinder_two_box_config()          # circular membrane (shape_fn), general interface, plane wave on a curved box
cyl["plane_wave"] = plane_wave_source(1, deg=20.0, azimuth_deg=30.0)
cases.append((cyl, {}))
for rec, kw in cases:
    sim = Simulation(rec, **kw)
    st = random_state(rec, seed=1)
    for b, (p, v) in enumerate(st):
        sim.write_state(b, p, v)
    sim.step(4)
    sim.sync()
    for b in range(len(rec["boxes"])):
        sim.pressure(b)
    sim.close()
fine, coarse = interface_faces(4, 4, 2, 25e-6, jitter=0.1, seed=1)
sem_face_match(fine, coarse, 4)
print("debug run ok")
