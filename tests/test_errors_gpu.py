"""Error behaviour of the C ABI (include/sem.h): every documented failure returns its status code
(SemError.status) instead of crashing; no CPU fallback anywhere."""
import numpy as np
import pytest

from sem_inputs import BC_ABSORBING, cavity_config, config, conforming_cut_config, curved_config

pytestmark = pytest.mark.gpu

SEM_E_ARG, SEM_E_STATE, SEM_E_NONFINITE, SEM_E_UNMATCHED = -1, -4, -5, -7


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _status(fn):
    from paper_2603_06267_b200 import SemError
    with pytest.raises(SemError) as ei:
        fn()
    return ei.value.status


def test_nonfinite_detected_with_step_index():
    """An unstable time step (10x the CFL limit) blows up; SEM_F_NAN_CHECK reports SEM_E_NONFINITE."""
    from paper_2603_06267_b200 import SEM_F_NAN_CHECK, SemError, Simulation
    rec = cavity_config(nel=(2, 2, 2), degree=4)
    rec["dt"] *= 10.0
    sim = Simulation(rec, flags=SEM_F_NAN_CHECK)
    sim.fill_random_state(0, 1, 1.0, 0.0)
    with pytest.raises(SemError) as ei:
        for _ in range(200):
            sim.step(50)
    assert ei.value.status == SEM_E_NONFINITE and "step" in str(ei.value)
    sim.close()


def test_bad_degree_rejected():
    from paper_2603_06267_b200 import Simulation
    rec = cavity_config(nel=(2, 2, 2), degree=4)
    rec["boxes"][0]["degree"] = 9
    assert _status(lambda: Simulation(rec)) != 0


def test_write_state_size_checked():
    from paper_2603_06267_b200 import Simulation
    rec = cavity_config(nel=(2, 2, 2), degree=3)
    sim = Simulation(rec)
    n = sim.ndof[0]
    assert _status(lambda: sim.write_state(0, np.zeros(n - 1), np.zeros(n - 1))) == SEM_E_ARG
    sim.close()


def test_pml_layers_overlap_rejected():
    from paper_2603_06267_b200 import Simulation
    rec = cavity_config(nel=(2, 2, 2), degree=3, extent=(1e-4, 1e-4, 1e-4))
    rec["pml"] = {"box": 0, "thickness": [6e-5, 6e-5, 0, 0, 0, 0], "R": 1e-4}
    assert _status(lambda: Simulation(rec)) == SEM_E_ARG
    rec["pml"] = {"box": 0, "thickness": [2e-5, 0, 0, 0, 0, 0], "R": 1.5}
    assert _status(lambda: Simulation(rec)) == SEM_E_ARG


def test_curved_box_refuses_pml():
    """Curved boxes carry PMUTs (tabulated coupling) and the general interface, not a PML."""
    from paper_2603_06267_b200 import Simulation
    rec = curved_config(nel=(4, 4, 4), degree=4, extent=(0.6e-3,) * 3, bc_top=BC_ABSORBING)
    rec["pml"] = {"box": 0, "thickness": [0.15e-3, 0, 0, 0, 0, 0], "R": 1e-4}
    assert _status(lambda: Simulation(rec)) == SEM_E_STATE


def test_interface_lattice_mismatch():
    from paper_2603_06267_b200 import Simulation
    rec = conforming_cut_config(nel_xy=4, nz_lo=2, nz_hi=2, degree=5, degree_hi=3, ratio=2, h=25e-6)
    rec["boxes"][1]["extent"] = (rec["boxes"][1]["extent"][0] * 1.1,) + tuple(rec["boxes"][1]["extent"][1:])
    assert _status(lambda: Simulation(rec)) == SEM_E_UNMATCHED


def test_nccl_loadable_unique_id():
    """The multi-GPU path dlopens NCCL (the libnccl.so.2 torch ships): a unique id can be created."""
    import torch.distributed  # noqa: F401  (the same process state bench.py runs in)
    from paper_2603_06267_b200 import sem_nccl_unique_id
    uid = sem_nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128 and any(uid)


def test_caller_allocator_torch_pool():
    """sem_mesh_desc dev_alloc / dev_free: the context's arrays come from torch's caching allocator,
    the results are bit-identical to the cudaMalloc context's and the memory returns on destroy."""
    import numpy as np
    import torch

    from paper_2603_06267_b200 import Simulation
    from sem_inputs import small_config
    rec = small_config("cfg2s")
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    a = Simulation(rec, torch_memory=True)
    held = torch.cuda.memory_allocated() - base
    a.step(40)
    pa = [a.pressure(b) for b in range(2)]
    qa = a.modal()[0]
    a.close()
    torch.cuda.synchronize()
    assert held > 0 and torch.cuda.memory_allocated() == base
    b = Simulation(rec)
    b.step(40)
    for k in range(2):
        assert np.array_equal(pa[k], b.pressure(k))
    assert np.array_equal(qa, b.modal()[0])
    b.close()
