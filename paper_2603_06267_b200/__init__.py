"""B200-native FP64 time step of the coupled PMUT-array / DG-SEM acoustic model (arxiv 2603.06267).

The product is ``lib/libsem.so`` (C ABI in ``include/sem.h``, CUDA sources in ``csrc/``); this
package is its thin ctypes binding.  Importing it without the built library raises ImportError:
there is no CPU fallback.
"""
from .sem import (  # noqa: F401
    EXPORTED, LIB_PATH, SEM_F_COUPLING_LITERAL, SEM_F_EMULATE_SLABS, SEM_F_NAN_CHECK, SEM_F_NO_GRAPH, SemError,
    Simulation, sem_nccl_unique_id,
    sem_dg_interface_build, sem_destroy, sem_fill_random_state, sem_kernel_time, sem_last_launch_count,
    sem_mesh_create, sem_plane_wave_source, sem_pmut_attach, sem_query, sem_read_modal, sem_read_pressure,
    sem_read_pressure_at, sem_set_profiling, sem_step, sem_sync, sem_write_state, sem_pml_attach, sem_face_match,
    sem_box_set_vertices, sem_box_set_obstacle,
)
