"""The reference's OWN unit tests (proj/tests/{graph,cpi,tpa,metrics,analysis,
persistence}_test.cpp, 76 test cases, compiled unchanged by integration/Makefile
against a self-written doctest-compatible header).

* CPU build = the reference library as shipped: pins the doctest shim.
* GPU build = the same tests with cpi.cpp/tpa.cpp replaced by the drop-in
  integration/rwrank_dropin.cpp over libtpa_gpu.so (and the graph.cpp sweep
  overridden): every cpi_run / pagerank / exact_rwr / cpi_partition /
  preprocess / query / query_na / propagation_sweep call in those tests runs
  the sm_100a kernels.
"""
from __future__ import annotations

import os
import re
import subprocess

import pytest

from conftest import ROOT

CPU_BIN = os.path.join(ROOT, "oracle", "_ref", "rwrank_unit_tests_cpu")
GPU_BIN = os.path.join(ROOT, "oracle", "_ref", "rwrank_unit_tests_gpu")


def run_suite(path, tmp_path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C integration, needs /root/reference at build time)")
    r = subprocess.run([path], capture_output=True, text=True, cwd=tmp_path, timeout=900)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert m, r.stdout + r.stderr
    return int(m.group(1)), int(m.group(2)), int(m.group(3)), r


def test_reference_suite_cpu_pins_the_shim(tmp_path):
    total, passed, failed, r = run_suite(CPU_BIN, tmp_path)
    assert total == 76 and failed == 0, r.stderr[-4000:]


@pytest.mark.gpu
def test_reference_suite_on_gpu_dropin(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    total, passed, failed, r = run_suite(GPU_BIN, tmp_path)
    assert total == 76 and failed == 0, r.stderr[-4000:]
