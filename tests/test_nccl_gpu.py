"""Real NCCL y-slab run (one rank per GPU) vs the single-GPU emulation of the same decomposition.

The NCCL transport and the emulation (SEM_F_EMULATE_SLABS: every slab in one context, device copies
in place of ncclSend/ncclRecv) run the same kernels on the same slab data in the same order, so the
results must be bitwise equal; rank 0's readback gathers the slabs through NCCL.  Skipped below 2
visible GPUs (NCCL cannot run two ranks on one device; emulated ranks that wait on one another on one
GPU are not a substitute, B200_PROFILING.md).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STEPS = 60


def _need_two():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")


def _rank_main(rank, world, port, out_dir, name, graph):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    from paper_2603_06267_b200 import SEM_F_NO_GRAPH, Simulation
    from paper_2603_06267_b200.sem import sem_nccl_unique_id
    idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        idt.copy_(torch.frombuffer(bytearray(sem_nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(idt, 0)
    rec = _record(name)
    sim = Simulation(rec, device=rank, rank=rank, world=world, nccl_unique_id=bytes(idt.cpu().numpy().tobytes()),
                     flags=0 if graph else SEM_F_NO_GRAPH)
    sim.step(STEPS)
    ps = [sim.pressure(b) for b in range(len(rec["boxes"]))]   # collective: rank 0 assembles
    q, qd, v = sim.modal()
    if rank == 0:
        np.savez(os.path.join(out_dir, "nccl.npz"), *ps, q=q, qd=qd, v=v)
    sim.close()
    dist.destroy_process_group()


def _record(name):
    from sem_inputs import config, small_config
    return config(0) if name == "cfg0" else small_config(name)


@pytest.mark.parametrize("graph", [True, False])
@pytest.mark.parametrize("name", ["cfg2s", "cfg4s", "cfg0"])   # cfg0: an uneven plan [0, 1, 4] (R30)
def test_nccl_two_ranks_bitwise_equals_emulation(tmp_path, name, graph):
    _need_two()
    import torch.multiprocessing as mp
    from paper_2603_06267_b200 import SEM_F_EMULATE_SLABS, Simulation
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mp.start_processes(_rank_main, args=(2, port, str(tmp_path), name, graph), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(tmp_path / "nccl.npz")
    rec = _record(name)
    emu = Simulation(rec, world=2, flags=SEM_F_EMULATE_SLABS)
    emu.step(STEPS)
    for b in range(len(rec["boxes"])):
        assert np.array_equal(got[f"arr_{b}"], emu.pressure(b)), b
    q, qd, v = emu.modal()
    assert np.array_equal(got["q"], q) and np.array_equal(got["qd"], qd)
    emu.close()
