"""CPU restatement of the row-partitioned CPI (csrc/tpa_part.cuh) for the
multi-process tests: each torch.distributed (gloo) rank owns the rows
[bounds[r], bounds[r+1]) of CSR(Ãᵀ), sweeps them in the reference's order
(ascending sources, graph.cpp:249-259 restated as a sequential sum), and the
ranks exchange exactly what the GPU partitions exchange:
  * an all-gather of the share slices in the padded global layout;
  * an all-reduce of the exact fixed-point |y| / dangling totals (limbs), so
    the residual is the same integer on every rank (and for every G).
Test infrastructure only (pure Python loops: small graphs)."""
from __future__ import annotations

import math

import numpy as np

KEEP_BITS = 120  # fixed point: value * 2^120 truncated (cpi_spmm.cuh fx_add)
MASK64 = (1 << 64) - 1


def fx(v: float) -> int:
    """floor(|v| * 2^120), the device's per-row fixed-point term (exact)."""
    t = min(math.ldexp(abs(v), 56), 2.0 ** 62)
    return int(math.ldexp(t, 64)) if t < 2.0 ** 62 else (1 << 126)


def fx_decode(total: int) -> float:
    hi, lo = total >> 64, total & MASK64
    return float(hi) * 2.0 ** -56 + float(lo) * 2.0 ** -120


def partition_rows(indeg, G):
    from paper_1708_02574_b200.partition import partition_rows as pr
    return pr(indeg, G)


def _allreduce_int(total: int, dist) -> int:
    import torch
    limbs = torch.tensor([(total >> (32 * k)) & 0xFFFFFFFF for k in range(4)], dtype=torch.int64)
    dist.all_reduce(limbs)
    return sum(int(limbs[k]) << (32 * k) for k in range(4))


def _allgather(local: np.ndarray, dist) -> np.ndarray:
    import torch
    t = torch.from_numpy(np.ascontiguousarray(local))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return np.concatenate([o.numpy() for o in out])


def run(off, tgt, n, policy, c, eps, start, terminal, seeds, G, rank, dist=None):
    """cpi_run over partition `rank` of G; returns (acc of all rows, iters, converged, residual).
    dist=None: G must be 1."""
    off = np.asarray(off, np.int64)
    tgt = np.asarray(tgt, np.int64)
    keep = 1.0 - c
    deg = off[1:] - off[:-1]
    indeg = np.bincount(tgt, minlength=n)
    b = partition_rows(indeg, G)
    S = max(1, int(max(b[k + 1] - b[k] for k in range(G))))
    lo, hi = int(b[rank]), int(b[rank + 1])
    owner = np.searchsorted(b, np.arange(n), side="right") - 1
    # a row's owner is the last partition starting at or before it (skips empty ones)
    owner = np.minimum(owner, G - 1)
    pad = owner * S + (np.arange(n) - b[owner])
    rows = [[] for _ in range(hi - lo)]
    for u in range(n):  # ascending sources, as the reference scatters
        for e in range(off[u], off[u + 1]):
            v = int(tgt[e])
            if lo <= v < hi:
                rows[v - lo].append(int(pad[u]))
    uniform = policy == 1

    x0 = np.zeros(hi - lo)
    if seeds is None:
        x0[:] = c / n
    else:
        for s in seeds:
            if lo <= s < hi:
                x0[s - lo] = c / len(seeds)
    acc = x0.copy() if start == 0 else np.zeros(hi - lo)
    share_loc = np.zeros(S)
    l1, dm = 0, 0
    for k in range(hi - lo):
        d = deg[lo + k]
        share_loc[k] = (keep * x0[k]) / d if d else 0.0
        l1 += fx(x0[k])
        if d == 0:
            dm += fx(x0[k])
    if dist is not None:
        l1, dm = _allreduce_int(l1, dist), _allreduce_int(dm, dist)
        share = _allgather(share_loc, dist)
    else:
        share = share_loc
    residual = fx_decode(l1)
    dmt = fx_decode(dm)
    has_spread = uniform and dmt != 0.0
    spread = (keep * dmt) / n if has_spread else 0.0
    active = terminal != 0
    converged = False
    it = 0
    i = 0
    while active:
        i += 1
        y = np.zeros(hi - lo)
        l1, dm = 0, 0
        for k, r in enumerate(rows):
            s = 0.0
            for p in r:
                s += share[p]
            if has_spread:
                s += spread
            y[k] = s
        inw = i >= start and (terminal < 0 or i <= terminal)
        if inw:
            acc += y
        share_loc = np.zeros(S)
        for k in range(hi - lo):
            d = deg[lo + k]
            share_loc[k] = (keep * y[k]) / d if d else 0.0
            l1 += fx(y[k])
            if uniform and d == 0:
                dm += fx(y[k])
        if dist is not None:
            l1, dm = _allreduce_int(l1, dist), _allreduce_int(dm, dist)
            share = _allgather(share_loc, dist)
        else:
            share = share_loc
        residual = fx_decode(l1)
        dmt = fx_decode(dm)
        it = i
        converged = residual < eps
        active = not converged and (terminal < 0 or i < terminal)
        has_spread = uniform and dmt != 0.0
        spread = (keep * dmt) / n if has_spread else 0.0
    full = acc
    if dist is not None:
        padded = np.zeros(S)
        padded[:hi - lo] = acc
        allp = _allgather(padded, dist)
        full = np.concatenate([allp[k * S:k * S + int(b[k + 1] - b[k])] for k in range(G)])
    return full, it, converged, residual
