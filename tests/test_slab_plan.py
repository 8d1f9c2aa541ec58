"""Host-only slab planner (sem_slab_plan, no GPU): membrane-preserving y-slabs, equal
when admissible, otherwise the admissible cuts nearest to the equal ones (config 1 at 4 and 8 GPUs, whose
equal cuts would split membranes: SURVEY 8(e))."""
import numpy as np
import pytest

from sem_inputs import config


@pytest.fixture(scope="module")
def plan():
    from paper_2603_06267_b200.build import build
    build()
    from paper_2603_06267_b200.sem import sem_slab_plan
    return sem_slab_plan


def _check(rec, cuts, world):
    b0 = rec["boxes"][0]
    nel = b0["nel"][1]
    assert cuts[0] == 0 and cuts[-1] == nel and len(cuts) == world + 1
    assert all(b > a for a, b in zip(cuts, cuts[1:]))
    hy = b0["extent"][1] / nel
    pm = rec["pmut"]
    for k in cuts[1:-1]:
        y = b0["origin"][1] + k * hy
        for c in pm["centers"]:
            assert not (c[1] - pm["side"] / 2 <= y <= c[1] + pm["side"] / 2)     # no membrane is split
        for b in rec["boxes"][1:]:
            assert (k * b["nel"][1]) % nel == 0                                   # a coarse element boundary


@pytest.mark.parametrize("ci", [2, 3, 4])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_two_box_configs_equal_slabs(plan, ci, world):
    rec = config(ci)
    cuts = plan(rec["boxes"], world, rec["pmut"])
    nel = rec["boxes"][0]["nel"][1]
    assert cuts == [nel * r // world for r in range(world + 1)]
    _check(rec, cuts, world)


def test_config1_uneven_slabs(plan):
    rec = config(1)
    # the admissible cuts (element boundaries in the membrane gaps) are 1-4, 8, 12, 16, 20-23 (x 37.5 um);
    # the planner minimises the largest slab: 8 elements at 4 GPUs, 4 at 8 GPUs (the best possible)
    c4 = plan(rec["boxes"], 4, rec["pmut"])
    _check(rec, c4, 4)
    assert max(np.diff(c4)) == 8
    c8 = plan(rec["boxes"], 8, rec["pmut"])
    _check(rec, c8, 8)
    assert max(np.diff(c8)) == 4
    assert plan(rec["boxes"], 2, rec["pmut"]) == [0, 12, 24]


def test_infeasible_plan_rejected(plan):
    from paper_2603_06267_b200.sem import SemError
    rec = config(1)
    with pytest.raises(SemError):
        plan(rec["boxes"], 20, rec["pmut"])     # more slabs than membrane gaps allow
