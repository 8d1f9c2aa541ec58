"""CPU oracle for the coupled PMUT-array / DG-SEM acoustic time step (arxiv 2603.06267).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2603_06267_b200``) never imports it, and
this package never imports the product path: the two share no code except the
seeded workload generator ``sem_inputs`` (which holds no method arithmetic).

What it computes, in the paper's order and notation (PAPER.md = P:L<line>):

* ``gll``        GLL nodes / weights and the Lagrange basis by the product
                 formula (reduced integration).
* ``mesh``       structured hexahedral boxes: trilinear maps X_K,
                 CG numbering inside a box, boxes not merged (DG).
* ``operators``  element matrices by brute-force GLL quadrature of Eq. (7)'s
                 volume term, lumped M (Eq. 6), ABC matrix C (Eq. 8), PMUT
                 coupling table (Eqs. 11-12) and the literal SIPG face matrix of
                 Eq. (7)'s three interface sums with gamma_F.
* ``newmark``    Algorithm 1 literally: three vectors per field,
                 predictor / solve / corrector, with the coupling-time-level flag
                 of DESIGN.md reading R2.
* ``pml``        the perfectly matched layer of Eq. (1):
                 damping profile, coefficients, element-local Phi, weak divergence,
                 and the auxiliary update of readings R23-R25.

Every function is pinned by ``tests/test_oracle_*.py`` against closed forms,
invariants or brute force.  Functions marked
"parity unpinned" below are pinned only through documented constants:
the drive / delay / scatter / plane-wave readings R10-R16 (no paper values).
"""
