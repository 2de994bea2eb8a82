"""The process-per-GPU row partition over CUDA IPC (the fused exchange,
csrc/tpa_part.cuh): 2 and 3 processes, each one partition, all sharing cuda:0
(NCCL refuses duplicate devices; IPC does not).  Every sweep's epilogue
stores its shares and exact residual limbs straight into the peers' buffers;
the ranks meet per sweep on interprocess events (stream waits -- no kernel
waits on another process's kernel).  Results must equal the whole-graph run
on one GPU bit for bit: PageRank / preprocess (116 sweeps), a windowed
multi-seed cpi_run with a terminal sweep (the limb all-reduce path), all
three dangling policies (cpi.cpp:55-101, tpa.cpp:19-37)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

C, EPS, T = 0.15, 1e-9, 10


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    import paper_1708_02574_b200 as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    res = {}
    for policy in ("selfloop", "uniform", "drop"):
        g = P.generate_rmat(13, 8, rng_seed=5, policy=policy)
        pg = P.PartitionedGraph.from_process_group(g, device=0, transport="ipc")
        res[f"{policy}_stranger"] = pg.preprocess(C, EPS, T)
        r = pg.cpi_run(P.SeedSet([3, 77, 1000, 5000]), P.CpiParams(C, EPS, 2, 6))
        res[f"{policy}_win"] = r.scores
        res[f"{policy}_win_meta"] = np.array([r.iterations_run, r.converged, r.residual_l1])
        pr = pg.pagerank(P.CpiParams(C, EPS))
        res[f"{policy}_pr"] = pr.scores
        res[f"{policy}_pr_meta"] = np.array([pr.iterations_run, pr.converged, pr.residual_l1])
        dist.barrier()
        pg.close()
        dist.barrier()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_partition_equals_one_gpu(world, tmp_path):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1708_02574_b200 as P
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    got = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    for policy in ("selfloop", "uniform", "drop"):
        g = P.generate_rmat(13, 8, rng_seed=5, policy=policy)
        want_st = P.preprocess(g, C, EPS, T).stranger_scores
        w = P.cpi_run(g, P.SeedSet([3, 77, 1000, 5000]), P.CpiParams(C, EPS, 2, 6))
        pr = P.pagerank(g, P.CpiParams(C, EPS))
        for r in range(world):
            assert np.array_equal(got[r][f"{policy}_stranger"], want_st), (policy, r)
            assert np.array_equal(got[r][f"{policy}_win"], w.scores), (policy, r)
            assert np.array_equal(got[r][f"{policy}_win_meta"], [w.iterations_run, w.converged, w.residual_l1])
            assert np.array_equal(got[r][f"{policy}_pr"], pr.scores), (policy, r)
            assert np.array_equal(got[r][f"{policy}_pr_meta"], [pr.iterations_run, pr.converged, pr.residual_l1])
