"""D2H bandwidth into pinned memory: one copy vs k concurrent copies on k streams."""
import os
import sys
import time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "local":
    import bench
    c = bench.gpu_local_cpus(0)
    print("local cpus", sorted(c) if c else None)
    if c:
        os.sched_setaffinity(0, c)
N = 268 << 20
src = torch.empty(N, dtype=torch.uint8, device="cuda")
dst = torch.empty(N, dtype=torch.uint8, pin_memory=True)
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = N // k
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for it in range(8):
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{k} streams: {8 * N / dt / 1e9:.1f} GB/s")
h2d_src = torch.empty(N, dtype=torch.uint8, pin_memory=True)
torch.cuda.synchronize(); t0 = time.perf_counter()
for it in range(8):
    src.copy_(h2d_src, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D: {8 * N / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
