"""Multi-rank host logic on CPU (world size 2, gloo): the y-slab decomposition that libsem's NCCL path
implements, checked without a GPU.

* `sem_slab_plan` (host-only C-ABI entry) applies the partition rules: equal y-slabs, cuts in the
  membrane gaps, cuts on coarse-element boundaries of the 2:1 interface.
* Two gloo ranks each build the oracle operator of their own slab with natural (rigid) cut faces,
  exchange ONE cut plane of partial results (K p and the lumped mass) and add the neighbour's part:
  every node of each slab then equals the global operator, and every slab-local PMUT projection
  equals the global one.  This is the identity the per-step exchange of the GPU path relies on
  (cut node row = own-side row + neighbour's partial).
"""
import os
import socket

import numpy as np
import pytest

from sem_inputs import config, small_config
from sem_inputs.counter_rng import cb_uniform


def _plan(rec, world):
    from paper_2603_06267_b200.sem import sem_slab_plan
    return sem_slab_plan(rec["boxes"], world, rec.get("pmut"))


def test_slab_plan_rules():
    from paper_2603_06267_b200.sem import SemError
    for i in (2, 3, 4):
        rec = config(i)
        for g in (1, 2, 4, 8):
            x0 = _plan(rec, g)
            nel = rec["boxes"][0]["nel"][1]
            assert x0 == [nel // g * r for r in range(g + 1)]
    assert _plan(config(1), 2) == [0, 12, 24]
    # equal cuts would split membranes: uneven membrane-preserving plans (tests/test_slab_plan.py)
    assert _plan(config(0), 2) == [0, 1, 4]
    for rec, g in ((small_config("cfg2s"), 3), (small_config("cfg2s"), 5)):
        with pytest.raises(SemError, match="PARTITION"):
            _plan(rec, g)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name):
    import torch
    import torch.distributed as dist
    from crops import crop_record
    from oracle.operators import System

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        rec = small_config(name)
        x0 = _plan(rec, world)
        nb = len(rec["boxes"])
        seed = 5
        # global reference (small enough for every rank to build)
        gs = System(rec)
        gp = np.concatenate([cb_uniform(seed, b, 0, np.arange(gs.boxes[b].ndof)) for b in range(nb)])
        gK = gs.split(gs.apply_K(gp))
        gM = gs.split(gs.M)
        gG = gs.pmut_project(gp) if gs.pm is not None else None
        # this rank's slab with natural cut faces
        win = (0, rec["boxes"][0]["nel"][0], x0[rank], x0[rank + 1])
        crop, info = crop_record(rec, win, margin_fine=0)
        ss = System(crop)
        sp = np.concatenate([cb_uniform(seed, b, 0, info["maps"][b]) for b in range(nb)])
        sK = ss.split(ss.apply_K(sp))
        sM = ss.split(ss.M)
        for b in range(nb):
            N = crop["boxes"][b]["degree"]
            nx = N * crop["boxes"][b]["nel"][0] + 1
            ny = N * crop["boxes"][b]["nel"][1] + 1
            lat = np.arange(len(info["maps"][b]))
            gy = (lat // nx) % ny
            # the cut row shared with the neighbour: last row (rank 0) / first row (rank 1)
            cut_row = ny - 1 if rank == 0 else 0
            mine = torch.from_numpy(np.stack([sK[b][gy == cut_row], sM[b][gy == cut_row]]))
            other = [torch.zeros_like(mine) for _ in range(world)]
            dist.all_gather(other, mine)                      # the one-plane exchange
            nbr = other[1 - rank].numpy()
            K_tot = sK[b].copy()
            M_tot = sM[b].copy()
            K_tot[gy == cut_row] += nbr[0]
            M_tot[gy == cut_row] += nbr[1]
            ref_K = gK[b][info["maps"][b]]
            ref_M = gM[b][info["maps"][b]]
            scale = np.abs(ref_K).max()
            assert np.max(np.abs(K_tot - ref_K)) < 1e-12 * scale, (rank, b)
            assert np.max(np.abs(M_tot - ref_M)) < 1e-14 * np.abs(ref_M).max(), (rank, b)
            # without the exchange the cut column is wrong (the test has teeth)
            assert np.max(np.abs(sK[b] - ref_K)) > 1e-6 * scale
        if gG is not None and len(info["pmut_full_index"]):
            sG = ss.pmut_project(sp)
            assert np.allclose(sG, gG[info["pmut_full_index"]], rtol=1e-13, atol=0)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg2s", "cfg1s"])
def test_slab_split_two_ranks_gloo(name):
    import torch.multiprocessing as mp
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    mp.spawn(_worker, args=(2, _free_port(), name), nprocs=2, join=True)
