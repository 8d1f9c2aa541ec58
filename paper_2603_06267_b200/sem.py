"""ctypes binding of libsem (include/sem.h): argument marshalling only.

Every step of the method runs in the CUDA library; this module converts Python / numpy
arguments to the C structs of ``sem.h`` and raises ``SemError`` on a non-zero status.  There is
no CPU fallback: importing this module fails loudly if ``lib/libsem.so`` is missing.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SEM_LIB") or os.path.join(_HERE, "lib", "libsem.so")

SEM_F_COUPLING_LITERAL = 1 << 0
SEM_F_NAN_CHECK = 1 << 1
SEM_F_NO_GRAPH = 1 << 2
SEM_F_EMULATE_SLABS = 1 << 3

_STATUS = {0: "SEM_OK", -1: "SEM_E_ARG", -2: "SEM_E_CUDA", -3: "SEM_E_NCCL", -4: "SEM_E_STATE",
           -5: "SEM_E_NONFINITE", -6: "SEM_E_PARTITION", -7: "SEM_E_UNMATCHED", -8: "SEM_E_OOM"}


class SemError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")


class BoxDesc(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("extent", C.c_double * 3), ("nel", C.c_int * 3),
                ("degree", C.c_int), ("c", C.c_double), ("rho", C.c_double), ("bc", C.c_int * 6)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class MeshDesc(C.Structure):
    _fields_ = [("n_boxes", C.c_int), ("boxes", C.POINTER(BoxDesc)), ("dt", C.c_double),
                ("device", C.c_int), ("stream", C.c_void_p), ("rank", C.c_int), ("world", C.c_int),
                ("nccl_unique_id", C.c_void_p), ("flags", C.c_int),
                ("dev_alloc", ALLOC_FN), ("dev_free", FREE_FN), ("alloc_user", C.c_void_p),
                ("slab_y0", C.POINTER(C.c_longlong))]


def torch_allocator(device=0):
    """(dev_alloc, dev_free) ctypes callbacks on torch's caching allocator (sem_mesh_desc); keep the
    returned pair alive as long as the context."""
    import torch

    def _alloc(nbytes, _user):
        return torch.cuda.caching_allocator_alloc(int(nbytes), device)

    def _free(ptr, _user):
        torch.cuda.caching_allocator_delete(int(ptr))

    return ALLOC_FN(_alloc), FREE_FN(_free)


class FaceSet(C.Structure):
    _fields_ = [("n", C.c_int), ("verts", C.POINTER(C.c_double)), ("face", C.POINTER(C.c_int))]


SHAPE_FN = C.CFUNCTYPE(C.c_double, C.c_int, C.c_int, C.c_double, C.c_double, C.c_void_p)


class PmutDesc(C.Structure):
    _fields_ = [("box", C.c_int), ("face", C.c_int), ("n_pmut", C.c_int), ("n_modes", C.c_int),
                ("center", C.POINTER(C.c_double)), ("side", C.c_double), ("mode_mn", C.POINTER(C.c_int)),
                ("freq_hz", C.POINTER(C.c_double)), ("modal_mass", C.POINTER(C.c_double)),
                ("damping_ratio", C.POINTER(C.c_double)), ("eta", C.POINTER(C.c_double)),
                ("rx", C.c_int), ("t_switch", C.c_double), ("capacitance", C.c_double),
                ("amp_v", C.c_double), ("f0_hz", C.c_double), ("n_cycles", C.c_int),
                ("delay_s", C.POINTER(C.c_double)), ("shape_fn", SHAPE_FN), ("shape_user", C.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsem.so not built ({LIB_PATH}); run __graft_entry__.build() -- "
                          "there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sig = {
        "sem_mesh_create": [C.POINTER(MeshDesc), C.POINTER(P)],
        "sem_nccl_unique_id": [C.c_void_p],
        "sem_slab_plan": [C.POINTER(BoxDesc), C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_longlong)],
        "sem_pmut_attach": [P, C.POINTER(PmutDesc)],
        "sem_dg_interface_build": [P, C.c_int, C.c_int, C.c_double, C.c_int],
        "sem_plane_wave_source": [P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                  C.POINTER(C.c_double)],
        "sem_pml_attach": [P, C.c_int, C.POINTER(C.c_double), C.c_double],
        "sem_box_set_vertices": [P, C.c_int, C.POINTER(C.c_double), C.c_size_t],
        "sem_box_set_obstacle": [P, C.c_int, C.POINTER(C.c_ubyte), C.c_size_t],
        "sem_face_match": [C.c_int, C.POINTER(FaceSet), C.POINTER(FaceSet), C.c_int, C.c_double,
                           C.POINTER(C.c_longlong), C.POINTER(C.c_double), C.POINTER(C.c_double)],
        "sem_step": [P, C.c_int],
        "sem_sync": [P],
        "sem_read_pressure": [P, C.c_int, C.POINTER(C.c_double), C.c_size_t],
        "sem_read_pressure_at": [P, C.c_int, C.POINTER(C.c_longlong), C.c_size_t, C.POINTER(C.c_double)],
        "sem_read_modal": [P, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_size_t],
        "sem_write_state": [P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_size_t],
        "sem_fill_random_state": [P, C.c_int, C.c_ulonglong, C.c_double, C.c_double],
        "sem_query": [P, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong), C.POINTER(C.c_double)],
        "sem_set_profiling": [P, C.c_int],
        "sem_kernel_time": [P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_longlong)],
        "sem_last_launch_count": [P, C.POINTER(C.c_longlong)],
        "sem_last_error": [P],
        "sem_destroy": [P],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.sem_last_error.restype = C.c_char_p
    lib.sem_destroy.restype = None
    return lib


LIB = _load()
EXPORTED = ("sem_mesh_create", "sem_nccl_unique_id", "sem_slab_plan", "sem_pmut_attach", "sem_dg_interface_build",
            "sem_plane_wave_source", "sem_pml_attach", "sem_face_match", "sem_box_set_vertices",
            "sem_box_set_obstacle", "sem_step", "sem_sync", "sem_read_pressure", "sem_read_pressure_at", "sem_read_modal",
            "sem_write_state", "sem_fill_random_state", "sem_query", "sem_set_profiling", "sem_kernel_time",
            "sem_last_launch_count", "sem_last_error", "sem_destroy")


def _check(ctx, st):
    if st != 0:
        msg = LIB.sem_last_error(ctx)
        raise SemError(st, msg.decode() if msg else "")


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ---- thin wrappers with the C names -------------------------------------------------------------
def _box_array(boxes):
    arr = (BoxDesc * len(boxes))()
    for i, b in enumerate(boxes):
        arr[i].origin[:] = [float(v) for v in b["origin"]]
        arr[i].extent[:] = [float(v) for v in b["extent"]]
        arr[i].nel[:] = [int(v) for v in b["nel"]]
        arr[i].degree = int(b["degree"])
        arr[i].c = float(b["c"])
        arr[i].rho = float(b["rho"])
        arr[i].bc[:] = [int(v) for v in b["bc"]]
    return arr


def sem_slab_plan(boxes, world, pm=None):
    """Host-only partition plan: box-0 element index where each of the `world` slabs starts."""
    arr = _box_array(boxes)
    x0 = (C.c_longlong * (world + 1))()
    pd, keep = (None, None) if pm is None else _pmut_desc(pm)
    st = LIB.sem_slab_plan(arr, len(boxes), int(world), C.cast(C.byref(pd), C.c_void_p) if pd is not None else None,
                           x0)
    if st != 0:
        raise SemError(st, "sem_slab_plan rejected the partition")
    return list(x0)


def sem_mesh_create(boxes, dt, device=0, stream=None, rank=0, world=1, nccl_unique_id=None, flags=0,
                    allocator=None, slab_y0=None):
    """allocator: optional (dev_alloc, dev_free) pair of ctypes callbacks (see torch_allocator);
    slab_y0: optional slab plan [world + 1] (sem_slab_plan)."""
    arr = _box_array(boxes)
    d = MeshDesc(len(boxes), arr, float(dt), int(device), C.c_void_p(stream) if stream else None, int(rank),
                 int(world), C.cast(C.c_char_p(nccl_unique_id), C.c_void_p) if nccl_unique_id else None, int(flags))
    if allocator is not None:
        d.dev_alloc, d.dev_free = allocator
    if slab_y0 is not None:
        plan = (C.c_longlong * len(slab_y0))(*[int(v) for v in slab_y0])
        d.slab_y0 = C.cast(plan, C.POINTER(C.c_longlong))
    out = C.c_void_p()
    st = LIB.sem_mesh_create(C.byref(d), C.byref(out))
    if st != 0:
        raise SemError(st, "sem_mesh_create failed (descriptor rejected or CUDA unavailable)")
    return out


def sem_nccl_unique_id():
    """128-byte ncclUniqueId (rank 0; broadcast it to the other ranks)."""
    buf = C.create_string_buffer(128)
    st = LIB.sem_nccl_unique_id(C.cast(buf, C.c_void_p))
    if st != 0:
        raise SemError(st, "sem_nccl_unique_id failed (libnccl.so.2 not loadable?)")
    return buf.raw


def _pmut_desc(pm):
    K, M = len(pm["centers"]), len(pm["mode_mn"])
    keep = dict(center=np.ascontiguousarray(pm["centers"], np.float64).ravel(),
                mode=np.ascontiguousarray(pm["mode_mn"], np.int32).ravel(),
                freq=np.ascontiguousarray(pm["freq_hz"], np.float64).ravel(),
                mass=np.ascontiguousarray(pm["modal_mass"], np.float64),
                damp=np.ascontiguousarray(pm["damping"], np.float64),
                eta=np.ascontiguousarray(pm["eta"], np.float64),
                delay=np.ascontiguousarray(pm["delay_s"], np.float64))
    d = PmutDesc(int(pm["box"]), int(pm["face"]), K, M, _dptr(keep["center"]), float(pm["side"]),
                 keep["mode"].ctypes.data_as(C.POINTER(C.c_int)), _dptr(keep["freq"]), _dptr(keep["mass"]),
                 _dptr(keep["damp"]), _dptr(keep["eta"]), int(bool(pm["rx"])),
                 float(pm["t_switch"]) if math.isfinite(pm["t_switch"]) else 1e300,
                 float(pm["capacitance"]), float(pm["amp_v"]), float(pm["f0_hz"]), int(pm["n_cycles"]),
                 _dptr(keep["delay"]))
    if pm.get("shape_fn") is not None:     # caller-defined mode shapes (sem.h, reading R33): passed through
        fn = pm["shape_fn"]
        keep["shape_fn"] = SHAPE_FN(lambda k, m, xr, yr, _user: float(fn(k, m, xr, yr)))
        d.shape_fn = keep["shape_fn"]
    return d, keep


def sem_pmut_attach(ctx, pm):
    d, keep = _pmut_desc(pm)
    _check(ctx, LIB.sem_pmut_attach(ctx, C.byref(d)))


def sem_dg_interface_build(ctx, fine_box, coarse_box, penalty_alpha, quad_rule=0):
    _check(ctx, LIB.sem_dg_interface_build(ctx, fine_box, coarse_box, float(penalty_alpha), quad_rule))


def sem_plane_wave_source(ctx, box, face, amp_pa, f0_hz, sigma_s, t0_s, direction):
    d = (C.c_double * 3)(*[float(v) for v in direction])
    _check(ctx, LIB.sem_plane_wave_source(ctx, box, face, amp_pa, f0_hz, sigma_s, t0_s, d))


def sem_box_set_vertices(ctx, box, verts):
    v = np.ascontiguousarray(verts, np.float64).reshape(-1, 3)
    _check(ctx, LIB.sem_box_set_vertices(ctx, int(box), _dptr(v), v.shape[0]))


def sem_box_set_obstacle(ctx, box, solid):
    """solid: bool / 0-1 mask of the box's nel_x nel_y nel_z elements, x fastest (include/sem.h)."""
    m = np.ascontiguousarray(solid, np.uint8).ravel()
    _check(ctx, LIB.sem_box_set_obstacle(ctx, int(box), m.ctypes.data_as(C.POINTER(C.c_ubyte)), m.size))


def sem_pml_attach(ctx, box, thickness, R):
    t = (C.c_double * 6)(*[float(v) for v in thickness])
    _check(ctx, LIB.sem_pml_attach(ctx, int(box), t, float(R)))


def sem_face_match(fine, coarse, degree, normal_tol=1e-6, device=0):
    """Algorithm 3 on the GPU.  fine / coarse: lists of (verts (8,3), local face).  Returns
    (owner [n_fine, (degree+1)^2] int64, xi [n_fine, (degree+1)^2, 3], device ms)."""
    def faceset(fs):
        v = np.ascontiguousarray(np.stack([f[0] for f in fs]) if fs else np.zeros((0, 8, 3)), np.float64)
        fc = np.ascontiguousarray([int(f[1]) for f in fs], np.int32)
        return FaceSet(len(fs), _dptr(v), fc.ctypes.data_as(C.POINTER(C.c_int))), (v, fc)
    fset, keep_f = faceset(fine)
    cset, keep_c = faceset(coarse)
    nq = (degree + 1) ** 2
    owner = np.empty((len(fine), nq), np.int64)
    xi = np.empty((len(fine), nq, 3), np.float64)
    ms = C.c_double(0.0)
    st = LIB.sem_face_match(int(device), C.byref(fset), C.byref(cset), int(degree), float(normal_tol),
                            owner.ctypes.data_as(C.POINTER(C.c_longlong)), _dptr(xi), C.byref(ms))
    if st not in (0, -7):
        raise SemError(st, "sem_face_match failed")
    return owner, xi, ms.value


def sem_step(ctx, n_steps):
    _check(ctx, LIB.sem_step(ctx, int(n_steps)))


def sem_sync(ctx):
    _check(ctx, LIB.sem_sync(ctx))


def sem_read_pressure(ctx, box, out):
    _check(ctx, LIB.sem_read_pressure(ctx, box, _dptr(out), out.size))
    return out


def sem_read_pressure_at(ctx, box, ids):
    ids = np.ascontiguousarray(ids, np.int64)
    out = np.empty(len(ids))
    _check(ctx, LIB.sem_read_pressure_at(ctx, box, ids.ctypes.data_as(C.POINTER(C.c_longlong)), len(ids),
                                         _dptr(out)))
    return out


def sem_read_modal(ctx, n):
    q, qd, v = np.empty(n), np.empty(n), None
    _check(ctx, LIB.sem_read_modal(ctx, _dptr(q), _dptr(qd), None, n))
    return q, qd


def sem_read_voltage(ctx, n, n_pmut):
    v = np.empty(n_pmut)
    _check(ctx, LIB.sem_read_modal(ctx, None, None, _dptr(v), n))
    return v


def sem_write_state(ctx, box, p, pdot):
    p = np.ascontiguousarray(p, np.float64)
    pdot = np.ascontiguousarray(pdot, np.float64)
    _check(ctx, LIB.sem_write_state(ctx, box, _dptr(p), _dptr(pdot), p.size))


def sem_write_state_ptr(ctx, box, p_ptr, pdot_ptr, n):
    """Host pointers (e.g. pinned torch tensors' data_ptr())."""
    _check(ctx, LIB.sem_write_state(ctx, box, C.cast(C.c_void_p(p_ptr), C.POINTER(C.c_double)),
                                    C.cast(C.c_void_p(pdot_ptr), C.POINTER(C.c_double)), n))


def sem_read_pressure_ptr(ctx, box, ptr, n):
    _check(ctx, LIB.sem_read_pressure(ctx, box, C.cast(C.c_void_p(ptr), C.POINTER(C.c_double)), n))


def sem_fill_random_state(ctx, box, seed, p_scale, v_scale):
    _check(ctx, LIB.sem_fill_random_state(ctx, box, int(seed), float(p_scale), float(v_scale)))


def sem_query(ctx):
    nd, st, t = C.c_longlong(), C.c_longlong(), C.c_double()
    _check(ctx, LIB.sem_query(ctx, C.byref(nd), C.byref(st), C.byref(t)))
    return nd.value, st.value, t.value


def sem_set_profiling(ctx, on):
    _check(ctx, LIB.sem_set_profiling(ctx, int(bool(on))))


def sem_kernel_time(ctx, which):
    ms, n = C.c_double(), C.c_longlong()
    _check(ctx, LIB.sem_kernel_time(ctx, which, C.byref(ms), C.byref(n)))
    return ms.value, n.value


def sem_last_launch_count(ctx):
    n = C.c_longlong()
    _check(ctx, LIB.sem_last_launch_count(ctx, C.byref(n)))
    return n.value


def sem_destroy(ctx):
    LIB.sem_destroy(ctx)


# ---- convenience object over a workload record --------------------------------------------------
class Simulation:
    """One context built from a ``sem_inputs`` workload record (boxes, PMUTs, interface, source)."""

    def __init__(self, rec, device=0, stream=None, flags=0, rank=0, world=1, nccl_unique_id=None,
                 torch_memory=False, slab_y0=None):
        self.rec = rec
        if rec.get("coupling", "predicted") == "literal":
            flags |= SEM_F_COUPLING_LITERAL
        # torch_memory: the context's device arrays come from torch's caching allocator
        self._allocator = torch_allocator(device) if torch_memory else None
        if slab_y0 is None and world > 1:   # equal slabs when admissible, else the uneven plan
            slab_y0 = sem_slab_plan(rec["boxes"], world, rec.get("pmut"))
        self.ctx = sem_mesh_create(rec["boxes"], rec["dt"], device, stream, rank, world, nccl_unique_id, flags,
                                   self._allocator, slab_y0)
        self.nn = [tuple(b["degree"] * n + 1 for n in b["nel"]) for b in rec["boxes"]]
        self.ndof = [a * b * c for a, b, c in self.nn]
        try:
            for bi, b in enumerate(rec["boxes"]):
                if b.get("vertices") is not None:
                    sem_box_set_vertices(self.ctx, bi, b["vertices"])
                if b.get("solid") is not None:
                    sol = np.asarray(b["solid"])
                    if sol.dtype != bool:
                        mask = np.zeros(int(np.prod(b["nel"])), dtype=bool)
                        mask[sol.astype(np.int64)] = True
                        sol = mask
                    sem_box_set_obstacle(self.ctx, bi, sol)
            if rec.get("pmut") is not None:
                sem_pmut_attach(self.ctx, rec["pmut"])
            if rec.get("interface") is not None:
                it = rec["interface"]
                rule = {"gll": 0, "lg": 1}[it.get("quad", "gll")]
                sem_dg_interface_build(self.ctx, it["fine_box"], it["coarse_box"], it["alpha"], rule)
            if rec.get("pml") is not None:
                pl = rec["pml"]
                sem_pml_attach(self.ctx, pl["box"], pl["thickness"], pl["R"])
            if rec.get("plane_wave") is not None:
                pw = rec["plane_wave"]
                sem_plane_wave_source(self.ctx, pw["box"], pw["face"], pw["amp_pa"], pw["f0_hz"], pw["sigma_s"],
                                      pw["t0_s"], pw["direction"])
        except Exception:
            self.close()
            raise

    @property
    def n_pmut_modes(self):
        pm = self.rec.get("pmut")
        return 0 if pm is None else len(pm["centers"]) * len(pm["mode_mn"])

    def step(self, n):
        sem_step(self.ctx, n)

    def sync(self):
        sem_sync(self.ctx)

    def pressure(self, box):
        return sem_read_pressure(self.ctx, box, np.empty(self.ndof[box]))

    def pressure_at(self, box, ids):
        return sem_read_pressure_at(self.ctx, box, ids)

    def modal(self):
        n = self.n_pmut_modes
        q, qd = sem_read_modal(self.ctx, n)
        v = sem_read_voltage(self.ctx, n, len(self.rec["pmut"]["centers"]))
        shape = self.rec["pmut"]["freq_hz"].shape
        return q.reshape(shape), qd.reshape(shape), v

    def write_state(self, box, p, pdot):
        sem_write_state(self.ctx, box, p, pdot)

    def fill_random_state(self, box, seed, p_scale, v_scale):
        sem_fill_random_state(self.ctx, box, seed, p_scale, v_scale)

    def query(self):
        return sem_query(self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            sem_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
