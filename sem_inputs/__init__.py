"""Seeded synthetic workloads for the PMUT-array / DG-SEM time step.

This module is the ONLY code shared by the CUDA path (its tests / bench) and the
CPU oracle.  It holds no arithmetic of the method itself: it turns the
BASELINE.json configurations (and DESIGN.md's documented readings of them) into
plain parameter records -- box geometry, PMUT placement, drive delays, modal
frequency scatter drawn from ``numpy.random.default_rng(seed)``, the time step
from the CFL rule, and seeded random fields for operator-level tests.
"""
from .workloads import (  # noqa: F401
    BC_RIGID, BC_ABSORBING, BC_INTERFACE, FACE_NAMES,
    config, config_names, small_config, small_config_names,
    random_state, n_nodes, box_dof, total_dof, cavity_config, conforming_cut_config, pml_config,
    interface_faces, curved_config, obstacle_config, solid_block, obstacle_pmut_config,
    curved_interface_config, curved_pmut_config, clamped_disc_shape, circular_pmut_config, cylinder_pmut_config, cylinder_two_box_config, cylinder_obstacle_config, plane_wave_source,
)
