"""Calibration only (not a product path): cuSPARSE CSR x dense SpMM on the C2
CSR(A^T) with a 32-wide fp64 row-major right-hand side, to bound what this
gather pattern achieves on the B200 (vs our fused sweep's gather phase)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402

g = bench.build_graph(sys.argv[1] if len(sys.argv) > 1 else "c2")
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
rp, col = g.device().transpose()
n = g.node_count()
crow = torch.as_tensor(rp, dtype=torch.int64).cuda()
coli = torch.as_tensor(col.astype("int64")).cuda()
vals = torch.ones(len(col), dtype=torch.float64, device="cuda")
A = torch.sparse_csr_tensor(crow, coli, vals, size=(n, n))
X = torch.rand(n, B, dtype=torch.float64, device="cuda")
for _ in range(3):
    Y = torch.sparse.mm(A, X)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    Y = torch.sparse.mm(A, X)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"cuSPARSE SpMM n={n} m={len(col)} B={B}: {ms:.3f} ms/launch "
      f"(gather stream {len(col) * B * 8 / ms / 1e6:.0f} GB/s of L2 traffic)")
# dense-RHS column-major variant
Xc = X.t().contiguous().t()
for _ in range(3):
    Y = torch.sparse.mm(A, Xc)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    Y = torch.sparse.mm(A, Xc)
e1.record()
torch.cuda.synchronize()
print(f"  column-major RHS: {e0.elapsed_time(e1) / 10:.3f} ms/launch")
