"""Device-side bounds checks (libsem_debug.so, -DSEM_DEBUG_CHECKS; the pool offers no
compute-sanitizer): every kernel family on small cases in a subprocess that loads the checked build.
A failed check traps and the run fails."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_bounds_checked_build_runs_clean():
    lib = os.path.join(ROOT, "paper_2603_06267_b200", "lib", "libsem_debug.so")
    assert os.path.exists(lib), "run __graft_entry__.build() first (it builds libsem_debug.so too)"
    env = dict(os.environ, SEM_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "debug_run.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "debug run ok" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])
    assert "debug check failed" not in r.stdout + r.stderr
    assert "libsem_debug.so" in r.stdout
