"""Bring-up check with torch's CUDA runtime initialised first (as in pytest)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

print("torch cuda", torch.cuda.is_available(), torch.cuda.device_count())
import numpy as np  # noqa: E402

import paper_1708_02574_b200 as P  # noqa: E402

g = P.Graph(2, [(0, 1), (1, 0)], "selfloop")
try:
    g.device()
    print("graph ok", P.propagation_sweep(g, np.array([0.15, 0.0]), 0.15))
except Exception as e:  # noqa: BLE001
    print("ERR", e)
