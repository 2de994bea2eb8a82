"""Shared fixtures.  `-m gpu` tests need a B200 (they call the C-ABI);
everything else runs on the CPU build box."""
from __future__ import annotations

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# Parity bar (BASELINE.json north_star): per RWR vector, per-node max-abs and L1.
MAX_ABS = 1e-12
L1 = 1e-9


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size parity case (seconds of oracle CPU time)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref/librwrank_ref.so not built (needs /root/reference at build time)")
    return Reference()


def golden_files():
    return sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(path):
    return dict(np.load(path))


class CsrGraph:
    """A graph given by the reference's out-CSR arrays (golden fixtures)."""

    def __init__(self, rec):
        self.n = int(rec["n"])
        self.out_offsets = rec["out_offsets"]
        self.out_targets = rec["out_targets"]
        self.policy = int(rec["policy"])


def assert_close(got, want, max_abs=MAX_ABS, l1=L1, what=""):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    d = np.abs(got - want)
    if want.ndim == 1:
        assert d.max(initial=0.0) <= max_abs, f"{what}: max-abs {d.max():.3e}"
        assert d.sum() <= l1, f"{what}: L1 {d.sum():.3e}"
    else:
        for k in range(want.shape[0]):
            assert d[k].max(initial=0.0) <= max_abs, f"{what}[{k}]: max-abs {d[k].max():.3e}"
            assert d[k].sum() <= l1, f"{what}[{k}]: L1 {d[k].sum():.3e}"
