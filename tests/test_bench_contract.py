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


@pytest.mark.gpu
def test_two_rank_launch_walks_the_partitioned_path():
    """The driver's N > 1 launch line with two ranks, both on cuda:0
    (TPA_BENCH_SAME_DEVICE=1: gloo group, the product's CUDA IPC exchange
    between the two processes).  Not a measurement: it checks that the
    multi-rank path runs end to end and prints rank 0's single line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, TPA_BENCH_SAME_DEVICE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--config", "c2", "--steps", "2", "--warmup", "3", "--no-cpu"],
                       capture_output=True, text=True, timeout=1200, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert "ipc" in d["parallelism"] and d["preprocess_sweeps"] == 116


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
