"""Benchmark of the B200 DG-SEM / PMUT leapfrog step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

A "step" is one pass of the whole hot path (Algorithm 1): modal ROM update, SIPG
interface flux, fused volume stiffness + ABC + PMUT forcing + kick-drift on every acoustic node of
both boxes.  Workload: BASELINE.json configs[3] (64x64 PMUT array, 526,755,050 FP64 DOF; the
largest config and the one the north-star's roofline / scaling targets name), synthetic inputs
(sem_inputs), state resident in HBM (12.6 GB > L2, so no flush is needed between steps).

Prints ONE JSON line on rank 0.  For N > 1 the ranks run the y-slab decomposition: under torchrun, or
spawned by this script itself (torch.distributed.run on 127.0.0.1) when WORLD_SIZE is unset.

Timing: the CUDA-graph path users get (profiling off): exactly K steps, timed as 5 repeats of ~K/5 steps
(each bracketed by barrier + synchronize, max over ranks), median ms per step; per-kernel times for the
roofline come from a separate profiling pass over K more steps (direct launches with CUDA events on the
launching stream).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "acoustic GDOF-updates/s per leapfrog step (FP64)"
UNIT = "GDOF/s"
BYTES_PER_DOF = 32.0          # SURVEY 8(d)'s algorithmic bytes: read p, w; write p, w (FP64) -- the roofline's unit
KERNEL_BYTES_PER_DOF = 24.0   # what the two-level volume kernel moves: read p^{n+1}, p^n; write p^{n+2} (DESIGN 1)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "samples": len(sm),
                "reasons": sorted(reasons)}


SPEC_HBM_GBS = 8000.0         # B200 HBM3e spec (~8 TB/s) named by BASELINE.json north_star
N_REPEATS = 5                 # median of 5 timed runs


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _spawn_ranks(n):
    """`python bench.py --gpus N` outside torchrun: re-launch this script as N local ranks (one per GPU)
    under torch.distributed.run on 127.0.0.1; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def cpu_baseline(steps, warmup=1, patch=4):
    """The oracle as it stands (numpy, FP64) on a bounded sample of the config-3 workload: a
    patch x patch PMUT lateral crop with the full config-3 depth, N, h, interface and modes."""
    import numpy as np  # noqa: F401
    from oracle.newmark import Newmark
    from oracle.operators import System
    from sem_inputs.workloads import crop_config
    try:
        from threadpoolctl import threadpool_info
        cores = max([t.get("num_threads", 1) for t in threadpool_info()] or [1])
    except Exception:
        cores = os.cpu_count()
    rec = crop_config(3, patch)
    sys_ = System(rec)
    nm = Newmark(sys_)
    nm.run(warmup)
    t0 = time.perf_counter()
    nm.run(steps)
    dt = time.perf_counter() - t0
    val = sys_.ndof * steps / dt / 1e9
    return {"value": val, "unit": UNIT, "cores": cores, "cpu_model": _cpu_model(), "host_cpus": os.cpu_count(),
            "kind": "oracle", "ms_per_step": dt / steps * 1e3,
            "sample": f"config-3 crop: {patch}x{patch} PMUTs ({rec['boxes'][0]['nel']} fine + "
                      f"{rec['boxes'][1]['nel']} coarse elements, {sys_.ndof} DOF), {steps} timed steps "
                      f"after {warmup} warm-up, {dt:.1f} s"}


def workload_config(rec, cfg, world):
    """The bench line's "config" (shared by both arms: the reference arm reports on the same workload)."""
    import numpy as np
    ndof_total = sum(int(np.prod([b["degree"] * n + 1 for n in b["nel"]])) for b in rec["boxes"])
    return {"workload": f"cfg{cfg}", "dof": ndof_total,
            "boxes": [f"{b['nel'][0]}x{b['nel'][1]}x{b['nel'][2]} N={b['degree']}" for b in rec["boxes"]],
            "n_pmut": len(rec["pmut"]["centers"]) if rec.get("pmut") else 0,
            "n_modes": len(rec["pmut"]["mode_mn"]) if rec.get("pmut") else 0,
            "dt": rec["dt"], "l2": "state 24 B/DOF resident = %.1f GB > 126 MB L2; no flush needed"
            % (24 * ndof_total / 1e9), "parallelism": f"y-slabs x{world}"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from sem_inputs import config
    cb = cpu_baseline(args.steps, args.warmup, patch=args.ref_patch)
    out = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms_per_step"], "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(config(args.config), args.config, world),
           "cpu_baseline": cb,
           "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=150)
    ap.add_argument("--ref-patch", type=int, default=4)
    ap.add_argument("--pml", type=int, default=0,
                    help="PML layers of this many elements on the lateral and top faces of the last box "
                         "(SURVEY 8(f) item 1; not part of BASELINE.json's configs)")
    ap.add_argument("--iface-quad", default="gll", choices=["gll", "lg"],
                    help="interface quadrature: the fine faces' GLL nodes (reading R9, BASELINE) or their "
                         "Gauss-Legendre points (R9's flag)")
    args = ap.parse_args()
    assert args.warmup >= 3 or os.environ.get("BENCH_ALLOW_SHORT"), "timing rules: warmup >= 3"

    if args.impl == "reference":
        # the oracle arm runs on rank 0 only (other torchrun ranks exit 0 without work)
        return run_reference(args, int(os.environ.get("RANK", "0")), args.gpus)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    import numpy as np
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2603_06267_b200.sem import (SEM_F_NO_GRAPH, Simulation, sem_kernel_time, sem_last_launch_count,
                                           sem_nccl_unique_id, sem_read_modal, sem_read_pressure_ptr,
                                           sem_set_profiling, sem_write_state_ptr)
    from sem_inputs import config

    rec = config(args.config)
    if args.iface_quad != "gll" and rec.get("interface") is not None:
        rec["interface"] = dict(rec["interface"], quad=args.iface_quad)
    if args.pml:
        bl = rec["boxes"][-1]
        hl = [e / n for e, n in zip(bl["extent"], bl["nel"])]
        th = [args.pml * hl[f // 2] if f != 4 else 0.0 for f in range(6)]
        bl["bc"] = [1 if th[f] > 0 else bl["bc"][f] for f in range(6)]     # ABC behind the layer
        rec["pml"] = {"box": len(rec["boxes"]) - 1, "thickness": th, "R": 1e-4}
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    nccl_id = None
    flags = 0
    if world > 1:
        # y-slab decomposition: libsem's own NCCL communicator for the per-step
        # cut-plane exchange; the id is created on rank 0 and broadcast through torch.distributed
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(sem_nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())
        if os.environ.get("BENCH_NCCL_NO_GRAPH"):
            flags |= SEM_F_NO_GRAPH     # NCCL send/recv are otherwise captured in the step graph
    sim = Simulation(rec, device=local, stream=stream.cuda_stream, rank=rank, world=world, nccl_unique_id=nccl_id,
                     flags=flags)
    ndof_total = sum(sim.ndof)      # global node count (every rank holds one y-slab of it)

    # ---- device-resident timed region: the CUDA-graph path users get (profiling off); exactly K steps,
    #      timed as N_REPEATS repeats of ~K/N_REPEATS steps, each bracketed by barrier + synchronize;
    #      max over ranks per repeat; the step time is the median over repeats of ms per step
    sim.step(args.warmup)
    sim.sync()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nrep = max(1, min(N_REPEATS, args.steps))
    chunks = [args.steps // nrep + (1 if r < args.steps % nrep else 0) for r in range(nrep)]
    reps, launches = [], 0
    for n in chunks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        sim.step(n)
        launches += sem_last_launch_count(sim.ctx)
        e1.record(stream)
        torch.cuda.synchronize()
        r = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([r], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            r = float(t.item())
        reps.append(r)
    clk = clocks.stop()
    ms = statistics.median([r / n for r, n in zip(reps, chunks)]) * args.steps
    # ---- per-kernel pass (same K steps, direct launches with CUDA events around each kernel group on
    #      the launching stream): the roofline's kernel time and the step shares
    sem_set_profiling(sim.ctx, 1)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    sim.step(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_prof = e0.elapsed_time(e1)
    vol_ms, vol_n = sem_kernel_time(sim.ctx, 0)
    ifc_ms, ifc_n = sem_kernel_time(sim.ctx, 1)
    mod_ms, mod_n = sem_kernel_time(sim.ctx, 2)
    pml_ms, pml_n = sem_kernel_time(sim.ctx, 3)
    sem_set_profiling(sim.ctx, 0)
    ms_step = ms / args.steps
    value = ndof_total * args.steps / (ms / 1e3) / 1e9     # strong scaling: fixed global problem

    peak, peak_kind = _peaks()
    vol_step_ms = vol_ms / max(vol_n, 1)
    achieved = BYTES_PER_DOF * ndof_total / world / (vol_step_ms / 1e3) / 1e9   # this rank's slab
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_cfg{args.config}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("bytes_per_step")
        except Exception:
            traffic = None

    # ---- end to end through the C ABI with host buffers ------------------------------------------
    e2e = None
    if not args.no_e2e:
        if world == 1:   # pinned host buffers of the full boxes
            hp = [torch.zeros(n, dtype=torch.float64).pin_memory() for n in sim.ndof]
            hv = [torch.zeros(n, dtype=torch.float64).pin_memory() for n in sim.ndof]
            ho = [torch.empty(n, dtype=torch.float64).pin_memory() for n in sim.ndof]
        else:
            # the ABI takes global arrays but a rank only touches its own slab (rank 0 the whole readback):
            # lazily allocated pageable buffers, so N ranks do not pin N copies of the full field
            hp = [torch.from_numpy(np.zeros(n)) for n in sim.ndof]
            hv = [torch.from_numpy(np.zeros(n)) for n in sim.ndof]
            ho = [torch.from_numpy(np.empty(n)) for n in sim.ndof]
        nm = sim.n_pmut_modes
        qh = np.empty(nm)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for b in range(len(sim.ndof)):
            sem_write_state_ptr(sim.ctx, b, hp[b].data_ptr(), hv[b].data_ptr(), sim.ndof[b])
        sim.step(args.steps)
        launches_e2e = sem_last_launch_count(sim.ctx)
        for b in range(len(sim.ndof)):
            sem_read_pressure_ptr(sim.ctx, b, ho[b].data_ptr(), sim.ndof[b])   # collective: rank 0 assembles
        if nm:
            sem_read_modal(sim.ctx, nm)
        torch.cuda.synchronize()
        t_e2e = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        h2d = 16.0 * ndof_total
        d2h = 8.0 * ndof_total + 16.0 * nm
        e2e = {"value": ndof_total * args.steps / t_e2e / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
               "note": "write_state (H2D p0, p'0; pinned host buffers at N=1, pageable slab-touching "
                       "buffers at N>1) + sem_step(K) + read_pressure/read_modal (D2H), host wall clock", "gpu_launches": launches_e2e}

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(rec, args.config, world),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "vol_kernel (both boxes, per step)",
                     "bytes_per_step_algorithmic": BYTES_PER_DOF * ndof_total,
                     "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                     "frac_spec_8tbs": achieved / SPEC_HBM_GBS,
                     "bytes_per_dof_algorithmic": BYTES_PER_DOF,
                     "bytes_per_dof_kernel": KERNEL_BYTES_PER_DOF,
                     "frac_kernel_bytes": achieved * KERNEL_BYTES_PER_DOF / BYTES_PER_DOF / peak,
                     "bytes_note": "achieved uses SURVEY 8(d)'s 32 B/DOF (read p, w; write p, w); the two-level "
                                   "kernel recomputes w = (p^{n+1} - p^n)/dt and moves 24 B/DOF, so its own "
                                   "bandwidth fraction is frac_kernel_bytes (DESIGN.md section 1)",
                     "step_frac": BYTES_PER_DOF * ndof_total / world / (ms_step / 1e3) / 1e9 / peak,
                     "share_of_step": vol_ms / ms_prof if ms_prof > 0 else None,
                     "timing": "kernel times from a separate profiling pass of the same K steps (direct "
                               "launches, CUDA events on the launching stream)",
                     "interface_ms_per_step": ifc_ms / max(ifc_n, 1), "modal_ms_per_step": mod_ms / max(mod_n, 1)},
        "gpu_launches": launches,
        "repeats_ms": reps,
        "repeat_steps": chunks,
        "timed_path": f"CUDA graph (sem_step): the K steps timed in {nrep} repeats, median ms per step",
        "clocks": clk,
        "e2e": e2e,
    }
    if args.pml:
        out["config"]["pml"] = {"elements_per_layer": args.pml, "box": rec["pml"]["box"], "R": rec["pml"]["R"],
                                "faces": "lateral + top", "element_kernel_ms_per_step": pml_ms / max(pml_n, 1)}
    if args.iface_quad != "gll":
        out["config"]["iface_quad"] = args.iface_quad
    if rank == 0 and world == 1 and not args.no_cpu_baseline:   # the contract: rank 0 at N = 1 only
        out["cpu_baseline"] = cpu_baseline(args.cpu_steps)
    if rank == 0:
        print(json.dumps(out), flush=True)
    sim.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
