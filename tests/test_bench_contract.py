"""bench.py's JSON contract: the reference arm runs on the CPU (C1, the
reference's own CPU-runnable config) and prints one line with the keys the
driver reads; the GPU arm's line is checked on the B200."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    from oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"], 600)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["unit"] == "GTEPS" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run(["--config", "c1", "--steps", "3", "--warmup", "3", "--no-cpu"], 1200)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["dtype"] == "f64"
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert 0 < r["frac"] < 1
    assert d["e2e"]["d2h_bytes_per_step"] > 0 and d["clocks"]["samples"] > 0


def test_reference_arm_imports_no_product_code():
    """--impl reference must time the reference alone: nothing of the product
    package (nor its libtpa_gpu.so) is loaded in that process."""
    from oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    code = (
        "import runpy, sys\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '1', '--warmup', '0']\n"
        "try:\n"
        "    runpy.run_path('bench.py', run_name='__main__')\n"
        "except SystemExit:\n"
        "    pass\n"
        "bad = [m for m in sys.modules if m.startswith('paper_1708_02574_b200')]\n"
        "maps = open('/proc/self/maps').read()\n"
        "assert not bad and 'libtpa_gpu' not in maps, bad\n"
        "print('clean')\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "clean" in r.stdout, r.stderr[-2000:]
