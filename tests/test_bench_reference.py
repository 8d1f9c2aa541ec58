"""bench.py's reference arm (the oracle on the host cores) runs without a GPU and prints
the contract's JSON line; with --gpus N outside torchrun it reports N (rank 0 alone runs it)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "3", "--gpus", "2", "--ref-patch", "2"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 2
    assert d["metric"].startswith("acoustic GDOF-updates/s") and d["unit"] == "GDOF/s" and d["higher_is_better"]
    assert d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["cpu_model"]
    assert d["config"]["workload"] == "cfg3" and d["config"]["dof"] == 526755050
