"""The C-ABI library loads and exports every entry point include/sem.h declares (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sem.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:sem_status|const char\*|void)\s+(sem_[a-z_]+)\s*\(", txt, re.M)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2603_06267_b200.build import build
    return build()


def test_header_declares_boundary_calls():
    names = _declared()
    for need in ("sem_mesh_create", "sem_pmut_attach", "sem_dg_interface_build", "sem_step",
                 "sem_read_pressure", "sem_read_modal", "sem_destroy", "sem_last_error"):
        assert need in names


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sem_[a-z_]+)$", out, re.M))
    assert set(_declared()) <= exported


def test_binding_wraps_every_symbol(lib_path):
    import paper_2603_06267_b200 as pkg
    assert set(_declared()) <= set(pkg.EXPORTED)


def test_library_is_sm100a(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_null_safety(lib_path):
    lib = ctypes.CDLL(lib_path)
    lib.sem_last_error.restype = ctypes.c_char_p
    lib.sem_last_error.argtypes = [ctypes.c_void_p]
    assert lib.sem_last_error(None) == b"null context"
    lib.sem_step.argtypes = [ctypes.c_void_p, ctypes.c_int]
    assert lib.sem_step(None, 1) == -1          # SEM_E_ARG without touching the device
    lib.sem_destroy.argtypes = [ctypes.c_void_p]
    lib.sem_destroy(None)
