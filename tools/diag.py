"""Minimal device bring-up check: one tiny graph through the C-ABI."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
print("CUDA_VISIBLE_DEVICES", os.environ.get("CUDA_VISIBLE_DEVICES"))
import numpy as np  # noqa: E402

import paper_1708_02574_b200 as P  # noqa: E402

g = P.Graph(2, [(0, 1), (1, 0)], "selfloop")
try:
    g.device()
    print("graph ok")
    print(P.propagation_sweep(g, np.array([0.15, 0.0]), 0.15))
except Exception as e:  # noqa: BLE001
    print("ERR", e)
