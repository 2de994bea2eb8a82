#!/usr/bin/env python3
"""Benchmark of the CPI hot path (TPA preprocessing + batched online RWR queries).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

The default workload is BASELINE.json configs[3] (C4: R-MAT scale 24, edge
factor 32, 529 M edges): the metric names no config, so the headline is the
largest config that runs on one GPU (C5 is stated row-sharded over 2/4/8).
One *step* is one pass of the hot path over one job of the chosen config:
PageRank preprocessing (the stranger vector, 116 sweeps at c=0.15, eps=1e-9)
followed by the config's online queries (1,024 seeds at C4) in SpMM batches
(32 at C4), S=5, T=10.  Inputs (graph CSR, seeds) are resident on the
device before the timed region; outputs stay in HBM.  Between timed steps the
L2 is flushed (a 512 MiB write, outside the events).

Metric (BASELINE.json): CPI edges/s (GTEPS) -- algorithmic edge traversals
m * (sweeps x active columns) per second -- with queries/s and the HBM
roofline fraction of the dominant sweep kernel reported beside it.

--impl reference times the reference's own CPU implementation
(oracle/_ref/librwrank_ref.so, built from /root/reference/proj/src) on the
host cores, same config and metric, importing nothing of the product: the
graph comes from the reference's own Graph constructor fed by the benchmark
generator restated in oracle/ref_capi.cpp (fingerprint printed in `config`,
equal to our arm's), each step one bounded sample (RefCpuSampler).

Multi-GPU (torchrun, one rank per GPU): the one job strong-scaled --
PageRank preprocessing row-partitioned across the ranks (the fused exchange:
each sweep's epilogue stores the iterate's shares + exact residual limbs
straight into every peer's buffer over NVLink, CUDA IPC; TPA_BENCH_TRANSPORT=nccl
for one NCCL all-gather per sweep instead) and the job's queries split over the
ranks' whole-graph replicas (no data-path collective);
TPA_BENCH_REPLICAS=1 runs N independent jobs instead (weak scaling).

Configs (--config): c1..c5 of BASELINE.json; c4/c5 graphs are generated and
built on the GPU (same graph as the host generator); c5 keeps each batch's
scores in HBM plus the device top-10 (a resident [16][n] output would not fit).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C, EPS, S, T = 0.15, 1e-9, 5, 10

CONFIGS = {
    # name: (kind, params, queries, batch, rng seed)
    "c1": ("rmat", dict(scale=16, edge_factor=16), 1, 1, 1),
    "c2": ("rmat", dict(scale=20, edge_factor=16), 1024, 32, 1),
    "c3": ("er", dict(n=4194304, m=67108864), 4096, 64, 1),
    "c4": ("rmat", dict(scale=24, edge_factor=32), 1024, 32, 1),
    "c5": ("rmat", dict(scale=28, edge_factor=16), 256, 16, 1),
}
# BASELINE.json's metric names no config, so the headline is the largest config
# that runs on one GPU as BASELINE states it: C4 (R-MAT 24, 529 M edges; C5 is
# stated as row-sharded across 2/4/8 GPUs)
DEFAULT_CONFIG = "c4"
THROTTLE_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def build_graph(cfg_name):
    import paper_1708_02574_b200 as P
    kind, p, *_ = CONFIGS[cfg_name]
    if kind == "rmat":
        # scale >= 22 (C4, C5): generated and constructed on the GPU -- the same
        # per-chunk mt19937_64 streams, so the same graph and fingerprint as the
        # host generator (tests/test_graph_build_gpu.py), in seconds not minutes
        dev = None
        if p["scale"] >= 22 and os.environ.get("TPA_HOST_GEN") != "1":
            import torch
            if torch.cuda.is_available():
                dev = int(os.environ.get("LOCAL_RANK", "0"))
        return P.generate_rmat(p["scale"], p["edge_factor"], 0.57, 0.19, 0.19, rng_seed=CONFIGS[cfg_name][4],
                               device=dev)
    return P.generate_random_graph(p["n"], p["m"], CONFIGS[cfg_name][4])


def workload_desc(cfg_name, n, m, n_dangling, fingerprint, nq, batch):
    kind, p, *_ = CONFIGS[cfg_name]
    gdesc = (f"R-MAT scale {p['scale']} ef {p['edge_factor']} (a,b,c)=(.57,.19,.19), mt19937_64 seed "
             f"{CONFIGS[cfg_name][4]}, no noise/permutation" if kind == "rmat"
             else f"ER G(n,m) n={p['n']} m={p['m']} (generate_random_graph seed {CONFIGS[cfg_name][4]})")
    return {
        "workload": f"{cfg_name.upper()}: TPA preprocess (PageRank CPI, window [T,inf)) + {nq} online queries "
                    f"in SpMM batches of {batch}",
        "graph": gdesc, "n": int(n), "m": int(m), "dangling": int(n_dangling), "fingerprint": f"{fingerprint:#018x}",
        "policy": "selfloop", "c": C, "eps": EPS, "S": S, "T": T, "queries": nq, "batch": batch,
        "seeds": "sample_seeds(mt19937_64 seed 1): uniform over non-dangling nodes (rwrank_main.cpp:65-83)",
        "l2": "flushed between timed steps (512 MiB write, untimed)",
    }


def a_step(n, m, B, acc):
    """SURVEY §8(d) algorithmic bytes of one CPI sweep over B columns."""
    return 4 * m + 8 * (n + 1) + 8 * n + 8 * B * n * (2 + 2 * acc)


def sweep_bytes(n, m, B, kind):
    """Compulsory bytes of one sweep as this engine runs it (every array touched
    once): CSR(A^T) indices 4m + row_ptr 8(n+1) + out-degree 4n + the share
    iterate read 8Bn, plus per kind
      'mid'     acc read+write and share_out write  (+24Bn)
      'last'    fused combine: acc read, stranger read, out write (+16Bn + 8n)
      'noacc'   share_out write only                (+8Bn)"""
    base = 4 * m + 8 * (n + 1) + 4 * n + 8 * B * n
    return base + {"mid": 24 * B * n, "last": 16 * B * n + 8 * n, "noacc": 8 * B * n}[kind]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the sampler is live before the timed region starts (short runs
            # would otherwise end before its first line)
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 5.0:
                time.sleep(0.01)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m_, r = float(parts[0]), float(parts[1]), int(parts[2], 16)
            except ValueError:
                continue
            mx = m_
            if r & ~0x1:  # ignore gpu_idle samples
                for bit, name in THROTTLE_BITS.items():
                    if r & bit and bit != 0x1:
                        reasons.add(name)
            if not (r == 0x1):
                sm.append(s)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(self.lines)}


def gpu_local_cpus(index):
    """The host cores on the GPU's own NUMA node (sysfs local_cpulist), or None."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(index)
        path = f"/sys/bus/pci/devices/{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0/local_cpulist"
        with open(path) as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            if "-" in part:
                a, b = part.split("-")
                cpus.update(range(int(a), int(b) + 1))
            elif part:
                cpus.add(int(part))
        return cpus & os.sched_getaffinity(0) or None
    except Exception:  # noqa: BLE001
        return None


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_per_launch(kernel, cfg_name=None):
    """DRAM bytes per launch of `kernel` from one ncu capture (profiles/traffic.json),
    keyed "<config>:<kernel>" where the config changes the working set."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        return t.get(f"{cfg_name}:{kernel}", t.get(kernel) if cfg_name in (None, "c2", "c1") else None)
    except Exception:  # noqa: BLE001
        return None


# ---------------------------------------------------------------------------
# CPU arm (the reference library built from its sources, oracle/_ref)
# ---------------------------------------------------------------------------
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def pagerank_sweeps(c=C, eps=EPS):
    """Sweeps of the reference PageRank under SelfLoop (mass-preserving):
    the first i with c(1-c)^i < eps (cpi.cpp:70-81; 116 at c=0.15, eps=1e-9)."""
    i, r = 0, c
    while not r < eps:
        i += 1
        r = c * (1 - c) ** i
    return i


def reference_graph(cfg_name):
    """The config's graph built by the reference's own Graph constructor from the
    benchmark generator's edges (oracle/ref_capi.cpp) -- no product code."""
    from oracle import Reference
    if not Reference.available():
        raise RuntimeError("oracle/_ref/librwrank_ref.so missing: run __graft_entry__.build() with "
                           "/root/reference present")
    ref = Reference()
    kind, p, _, _, seed = CONFIGS[cfg_name]
    if kind == "rmat":
        return ref.graph_rmat(p["scale"], p["edge_factor"], 0.57, 0.19, 0.19, seed=seed, threads=0)
    return ref.graph_random(p["n"], p["m"], seed)


class RefCpuSampler:
    """Times the reference CPU path (tpa.cpp preprocess / query through
    oracle/_ref, the CLI's timed calls rwrank_main.cpp:122-124, :153-156) on a
    bounded sample of one job and extrapolates the job time:

    * preprocess: the whole preprocess() when it fits the budget, else
      116 x one dense propagation_sweep (graph.cpp:230-270) -- at the faster of
      threads = 1 and threads = min(cores, 64) (picked once, untimed);
    * queries: a window of the job's seeds (one per core, at least 16) run as
      concurrent single-thread reference query() calls on every core
      (tpa_test.cpp:148-161: concurrent queries are the reference's contract),
      a different window each step.
    A C4 step is then ~12 s of CPU work (one 2.2 s sweep + 16 concurrent
    6-8 s queries), so a 20-step run stays within a few minutes."""

    def __init__(self, rg, seeds, budget_s=20.0, workers=None):
        self.rg, self.seeds = rg, np.ascontiguousarray(seeds, np.uint32)
        self.workers = workers or len(os.sched_getaffinity(0)) or 1
        self.n, self.m, self.nq = rg.n, rg.m, len(seeds)
        self.sweeps = pagerank_sweeps()
        t1 = rg.time_sweeps(1, C, 1)
        tmax = min(self.workers, 64)
        tt = rg.time_sweeps(1, C, tmax) if tmax > 1 else t1
        self.pre_threads = tmax if tt < t1 else 1
        self.t_sweep_cal = {"threads=1": t1, f"threads={tmax}": tt}
        t_sw = min(t1, tt)
        self.whole_pre = t_sw * (self.sweeps + 1) <= budget_s * 0.5
        self.stranger = np.zeros(self.n)
        if self.whole_pre:
            self.stranger = rg.preprocess(C, EPS, T, self.pre_threads)
        self.qs = int(min(self.nq, max(16, self.workers)))
        self.cursor = 0

    def step(self):
        rg = self.rg
        if self.whole_pre:
            _, t_pre = rg.time_preprocess(C, EPS, T, self.pre_threads)
            pre_note = f"preprocess() timed whole (threads={self.pre_threads})"
        else:
            t_pre = rg.time_sweeps(1, C, self.pre_threads) * self.sweeps
            pre_note = (f"preprocess extrapolated: {self.sweeps} x one dense propagation_sweep "
                        f"(threads={self.pre_threads})")
        idx = (self.cursor + np.arange(self.qs)) % self.nq
        self.cursor = int((self.cursor + self.qs) % self.nq)
        _, t_q = rg.query_many(self.stranger, C, EPS, T, self.seeds[idx], S, self.workers)
        t_job = t_pre + t_q * self.nq / self.qs
        return {"job_s": t_job, "preprocess_s": t_pre, "queries_per_s": self.qs / t_q,
                "sample": f"{pre_note} + {self.qs} of {self.nq} queries as concurrent reference query() "
                          f"calls on {self.workers} threads; job time extrapolated"}

    def baseline(self, recs):
        job = statistics.mean(r["job_s"] for r in recs)
        edges = self.m * (self.sweeps + (S - 1) * self.nq)
        return {"value": edges / job / 1e9, "unit": "GTEPS", "cores": int(self.workers), "kind": "reference",
                "cpu_model": cpu_model(), "sample": recs[-1]["sample"], "job_s": job,
                "preprocess_s": statistics.mean(r["preprocess_s"] for r in recs),
                "preprocess_threads": self.pre_threads, "sweep_calibration_s": self.t_sweep_cal,
                "queries_per_s": statistics.mean(r["queries_per_s"] for r in recs), "extrapolated": True}


def cpu_measure(rg, seeds, budget_s=20.0):
    """cpu_baseline of the GPU arm: one bounded reference sample."""
    smp = RefCpuSampler(rg, seeds, budget_s)
    return smp.baseline([smp.step()])


def run_reference_arm(args):
    """--impl reference: the reference's own CPU path (oracle/_ref, compiled from
    /root/reference/proj/src) on this box's host cores.  Imports nothing of the
    product package: graph, seeds and timing all come from the reference build."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg_name = args.config
    _, _, nq, batch, seed = CONFIGS[cfg_name]
    t0 = time.perf_counter()
    rg = reference_graph(cfg_name)
    t_build = time.perf_counter() - t0
    log(f"[reference] graph {cfg_name}: n={rg.n} m={rg.m} built in {t_build:.1f}s")
    seeds = rg.sample_seeds(nq, seed)
    smp = RefCpuSampler(rg, seeds, budget_s=args.cpu_budget)
    # warm-up steps: one dense sweep each (the CPU path has nothing to compile
    # or tune; this only warms caches and page tables)
    for _ in range(max(0, args.warmup)):
        rg.time_sweeps(1, C, smp.pre_threads)
    recs = [smp.step() for _ in range(max(1, args.steps))]
    cb = smp.baseline(recs)
    v = cb["value"]
    line = {"impl": "reference", "metric": "CPI edges/sec (GTEPS) and online RWR queries/sec; % of HBM roofline",
            "value": v, "unit": "GTEPS", "n_gpus": args.gpus, "steps": max(1, args.steps), "warmup": args.warmup,
            "ms_per_step": cb["job_s"] * 1e3, "higher_is_better": True,
            "scaling": "strong" if args.gpus > 1 else "weak",  # one job, as our arm's N > 1 line
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_desc(cfg_name, rg.n, rg.m, len(rg.dangling), rg.fingerprint, nq, batch),
            "queries_per_s": cb["queries_per_s"], "cpu_baseline": cb, "graph_build_s": t_build,
            "e2e": {"value": v, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1708_02574_b200 as P
    from paper_1708_02574_b200 import _native as N

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TPA_BENCH_SAME_DEVICE=1 (tests only): every rank on cuda:0 with a gloo
    # group -- walks the N > 1 code path (partition, IPC exchange, barriers, the
    # max-over-ranks reduce, the JSON line) on a one-GPU box; never a measurement
    same_device = world > 1 and os.environ.get("TPA_BENCH_SAME_DEVICE") == "1"
    if same_device:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if same_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t_ = torch.tensor([x], dtype=torch.float64, device="cpu" if same_device else dev)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        return float(t_.item())

    cfg_name = args.config
    _, _, nq, batch, seed = CONFIGS[cfg_name]
    t0 = time.perf_counter()
    g = build_graph(cfg_name)
    t_build = time.perf_counter() - t0
    n, m = g.node_count(), g.edge_count()
    # N > 1 (strong scaling of the one C2 job): PageRank preprocessing row-
    # partitioned across the ranks (one NCCL exchange per sweep, the north
    # star's layout) and the job's queries split across the ranks, each on a
    # whole-graph replica.  TPA_BENCH_REPLICAS=1: N independent jobs instead.
    replicas = world > 1 and os.environ.get("TPA_BENCH_REPLICAS") == "1"
    # TPA_BENCH_PART=1 at N = 1: the partitioned code path with one rank (NCCL
    # communicator of one), to exercise it on a single GPU
    partitioned = (world > 1 and not replicas) or os.environ.get("TPA_BENCH_PART") == "1"
    all_seeds = P.sample_seeds(g, nq * (world if replicas else 1), seed)
    if replicas:
        seeds = np.ascontiguousarray(all_seeds[rank * nq:(rank + 1) * nq])
    else:
        seeds = np.ascontiguousarray(np.array_split(all_seeds, world)[rank]) if world > 1 else all_seeds
    log(f"[rank {rank}] graph {cfg_name}: n={n} m={m} built in {t_build:.1f}s")

    t0 = time.perf_counter()
    dg = g.device(local)
    torch.cuda.synchronize()
    t_ingest = time.perf_counter() - t0
    # a dedicated (non-default) torch stream: the library enqueues on it, so the
    # torch events below bracket exactly the library's kernels
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    dg.set_stream(stream.cuda_stream)
    lib = N.lib
    h = dg.h
    import ctypes as C_

    # C5 (n = 2^28, B = 16): a resident [B][n] output would be 34 GB on top of
    # the 143 GB of graph + iterate buffers, so each batch's full score
    # vectors are written into the iterate buffer the last sweep leaves idle
    # (tpa_query_batch_topk) and only the top-10 per seed stays resident
    resident_topk = n * batch * 8 > (8 << 30) or os.environ.get("TPA_BENCH_TOPK") == "1"
    K_TOP = 10
    if resident_topk:
        out = None
        d_ids = torch.empty((batch, K_TOP), dtype=torch.int32, device=dev)
        d_vals = torch.empty((batch, K_TOP), dtype=torch.float64, device=dev)
    else:
        out = torch.empty((batch, n), dtype=torch.float64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    batches = [np.ascontiguousarray(seeds[i:i + batch]) for i in range(0, len(seeds), batch)]
    pg = None
    if partitioned:
        if world > 1:
            # the fused exchange (every sweep stores its shares into the peers'
            # buffers over NVLink, CUDA IPC); TPA_BENCH_TRANSPORT=nccl: one
            # NCCL all-gather per sweep instead
            pg = P.PartitionedGraph.from_process_group(
                g, device=local, transport=os.environ.get("TPA_BENCH_TRANSPORT", "ipc"))
        else:
            pg = P.PartitionedGraph(g, 1, 0, comm_id=P.partition.comm_unique_id(), device=local)
        N.check(lib.tpa_graph_set_stream(pg.h, stream.cuda_stream))
        d_str = torch.empty(n, dtype=torch.float64, device=dev)
        log(f"[rank {rank}] partition {pg.info()}")

    def device_step():
        art = C_.c_void_p()
        if pg is None:
            N.check(lib.tpa_preprocess(h, C, EPS, T, None, C_.byref(art), N.TPA_DEVICE_PTRS | N.TPA_ASYNC))
        else:
            # collective: every rank ends with the whole stranger vector on its GPU
            N.check(lib.tpa_preprocess(pg.h, C, EPS, T, d_str.data_ptr(), None, N.TPA_DEVICE_PTRS))
            N.check(lib.tpa_artifact_create(h, d_str.data_ptr(), g.fingerprint(), C, EPS, T, N.TPA_DEVICE_PTRS,
                                            C_.byref(art)))
        for b in batches:
            if resident_topk:
                N.check(lib.tpa_query_batch_topk(h, art, b.ctypes.data, len(b), S, K_TOP, d_ids.data_ptr(),
                                                 d_vals.data_ptr(), N.TPA_DEVICE_PTRS))
            else:
                N.check(lib.tpa_query_batch(h, art, b.ctypes.data, len(b), S, out.data_ptr(),
                                            N.TPA_DEVICE_PTRS | N.TPA_ASYNC))
        return art

    # warm-up
    for _ in range(args.warmup):
        a = device_step()
        lib.tpa_artifact_destroy(a)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    launches0 = dg.launches() + (N.lib.tpa_graph_launches(pg.h) if pg is not None else 0)
    times = []
    # The timed steps run without the library's per-kernel event pairs; the
    # per-sweep breakdown (roofline) comes from extra, separately profiled steps
    # after the timed region.  TPA_BENCH_PROFILE_TIMED=1: profile the timed steps.
    prof_timed = os.environ.get("TPA_BENCH_PROFILE_TIMED") == "1"

    def set_profile(on):
        dg.profile(on)
        if pg is not None:
            N.check(lib.tpa_graph_profile(pg.h, 1 if on else 0))

    if prof_timed:
        set_profile(True)
    prof_range = os.environ.get("TPA_PROFILE_RANGE") == "1"  # ncu --profile-from-start off
    if prof_range:
        torch.cuda.cudart().cudaProfilerStart()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            a = device_step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            lib.tpa_artifact_destroy(a)
    if prof_range:
        torch.cuda.cudart().cudaProfilerStop()
    launches = dg.launches() + (N.lib.tpa_graph_launches(pg.h) if pg is not None else 0) - launches0
    prof_total_ms = sum(times)
    if not prof_timed:
        # the profiled steps (same work, per-kernel CUDA events on the stream)
        set_profile(True)
        prof_total_ms = 0.0
        for _ in range(max(1, min(args.steps, 3))):
            flush.fill_(1)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            a = device_step()
            e1.record(stream)
            torch.cuda.synchronize()
            prof_total_ms += e0.elapsed_time(e1)
            lib.tpa_artifact_destroy(a)
    mv_cnt, mv_ms = dg.profile_read(1)
    if pg is not None:
        c_, ms_ = C_.c_uint64(), C_.c_double()
        N.check(lib.tpa_graph_profile_read(pg.h, 1, -1, C_.byref(c_), C_.byref(ms_)))
        mv_cnt, mv_ms = mv_cnt + c_.value, mv_ms + ms_.value
        N.check(lib.tpa_graph_profile(pg.h, 0))
    mm_cnt, mm_ms = dg.profile_read(batch if batch > 1 else 1)
    per_sweep = {}
    if batch > 1:
        for i in range(1, S):
            c_i, ms_i = dg.profile_read(batch, i)
            if c_i:
                kind = "last" if i == S - 1 else "mid"
                per_sweep[i] = {"launches": c_i, "avg_ms": ms_i / c_i,
                                "achieved_gbs_dense_bytes": sweep_bytes(n, m, batch, kind) / (ms_i / c_i / 1e3) / 1e9}
    dg.profile(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = sum(times)
    total_ms = max_over_ranks(total_ms)
    ms_per_step = total_ms / args.steps

    # sweeps actually run: 116 PageRank sweeps (the convergence break) + (S-1) per query
    pr = P.pagerank(g, P.CpiParams(C, EPS))
    pre_sweeps = pr.iterations_run
    jobs = 1 if partitioned else world  # independent C2 jobs per step
    edges_per_step = m * (pre_sweeps + (S - 1) * nq)
    value = edges_per_step * jobs * args.steps / (total_ms / 1e3) / 1e9
    qps = nq * jobs * args.steps / (total_ms / 1e3)

    # roofline of the dominant kernel (the SpMM sweep at batch width B)
    peak, peak_src = peak_hbm()
    Bk = batch if batch > 1 else 1
    if batch > 1 and mm_cnt:
        # dominant kernel: the SpMM sweep.  Roofline on its densest launch, the
        # last family sweep x^(S-1) (fused combine); the sparse early sweeps are
        # listed per index.
        kname = f"k_mm_fused<{Bk}>" if Bk >= 16 else f"k_step_spmm2<{Bk}>"
        last = per_sweep.get(S - 1)
        # SURVEY §8(d)'s per-sweep figure A_step(B, acc=1) (what the roofline is
        # defined on); the engine's own compulsory count is reported beside it
        bytes_launch = a_step(n, m, Bk, 1)
        avg_ms = last["avg_ms"] if last else mm_ms / mm_cnt
        share = mm_ms / prof_total_ms if prof_total_ms else None
    else:
        kname = "k_step_spmv2"
        bytes_launch = a_step(n, m, 1, 1)
        avg_ms = mv_ms / max(mv_cnt, 1)
        share = mv_ms / prof_total_ms if prof_total_ms else None
    achieved = bytes_launch / (avg_ms / 1e3) / 1e9
    # the access pattern's own ceiling (profiles/microbench.json): the sweeps are
    # gather-bound (L2 -> SM for the SpMM rows, L1 request rate for the SpMV)
    mb = {}
    try:
        with open(os.path.join(ROOT, "profiles", "microbench.json")) as f:
            mb = json.load(f)
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_source": peak_src,
                "traffic": traffic_per_launch(kname, cfg_name), "algorithmic_bytes_per_launch": bytes_launch,
                "avg_launch_ms": avg_ms, "launches_timed": mm_cnt if batch > 1 else mv_cnt,
                "share_of_step": share, "per_sweep": per_sweep,
                "bytes_definition": "SURVEY 8(d) A_step(B,1) = 4m + 8(n+1) + 8n + 32Bn per sweep",
                "engine_compulsory_bytes": sweep_bytes(n, m, Bk, "last") if batch > 1 else a_step(n, m, 1, 1),
                "spmv": {"launches": mv_cnt, "avg_ms": mv_ms / max(mv_cnt, 1),
                         "achieved_gbs": a_step(n, m, 1, 1) / (mv_ms / max(mv_cnt, 1) / 1e3) / 1e9
                         if mv_cnt else None}}
    # the measured ceiling of the access pattern at this working-set size: the
    # L2-resident one, or the one measured at C4's size once the iterate is far
    # beyond the 126 MB L2
    big = n * Bk * 8 > (1 << 30)
    key_mm = "gather_256B_rows_4GB" if big else "gather_256B_rows"
    if batch > 1 and mb.get(key_mm):
        g_gbs = m * Bk * 8 / (avg_ms / 1e3) / 1e9  # every nonzero gathers one B-wide share row
        pk = mb[key_mm]["best_gbs"] if Bk == 32 else None
        roofline["gather_bound"] = {"achieved_gbs": g_gbs, "peak_gbs": pk, "frac": g_gbs / pk if pk else None,
                                    "pattern": mb[key_mm]["pattern"],
                                    "source": "profiles/microbench.json (tools/gather_micro.cu)"}
    key_mv = "gather_8B_134MB" if n * 8 > (64 << 20) else "gather_8B"
    if mv_cnt and mb.get(key_mv):
        rate = m / (mv_ms / mv_cnt / 1e3)
        roofline["spmv"]["gather_bound"] = {"achieved_gathers_per_s": rate,
                                            "peak_gathers_per_s": mb[key_mv]["best_gathers_per_s"],
                                            "frac": rate / mb[key_mv]["best_gathers_per_s"],
                                            "pattern": mb[key_mv]["pattern"]}

    # end-to-end through the public API with host buffers
    # The e2e legs run with the process on the GPU's own NUMA node, so the
    # pinned result buffers are first-touched next to the GPU's PCIe root
    # (a remote node halves the D2H rate); the CPU baseline afterwards gets
    # every core back.
    all_cpus = os.sched_getaffinity(0)
    local_cpus = gpu_local_cpus(local) if os.environ.get("TPA_BENCH_NUMA", "1") == "1" else None
    if local_cpus:
        os.sched_setaffinity(0, local_cpus)
    e2e = None
    if not args.no_e2e and not resident_topk:
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        # two pinned result buffers, alternating: batch k+1 computes while batch k drains
        host_outs = [torch.empty((batch, n), dtype=torch.float64, pin_memory=True) for _ in range(2)]
        host_str = torch.empty(n, dtype=torch.float64, pin_memory=True)
        h2d = d2h = 0
        el = []
        for it in range(1 + e2e_steps):  # first one: untimed warm-up (stage buffers, copy stream, first drain)
            flush.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            art = C_.c_void_p()
            if pg is None:
                N.check(lib.tpa_preprocess(h, C, EPS, T, host_str.data_ptr(), C_.byref(art), 0))
            else:
                N.check(lib.tpa_preprocess(pg.h, C, EPS, T, host_str.data_ptr(), None, 0))
                N.check(lib.tpa_artifact_create(h, host_str.data_ptr(), g.fingerprint(), C, EPS, T, 0,
                                                C_.byref(art)))
            d2h_s = n * 8
            h2d_s = 0
            for i, b in enumerate(batches):
                N.check(lib.tpa_query_batch(h, art, b.ctypes.data, len(b), S, host_outs[i & 1].data_ptr(),
                                            N.TPA_ASYNC))
                h2d_s += len(b) * 4
                d2h_s += len(b) * n * 8
            N.check(lib.tpa_graph_sync(h))
            torch.cuda.synchronize()
            if it:
                el.append(time.perf_counter() - t0)
            else:
                e2e_warm_ms = (time.perf_counter() - t0) * 1e3
            lib.tpa_artifact_destroy(art)
            h2d, d2h = h2d_s, d2h_s
        e2e_s = max_over_ranks(sum(el))
        e2e = {"value": edges_per_step * jobs * e2e_steps / e2e_s / 1e9, "unit": "GTEPS",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "queries_per_s": nq * jobs * e2e_steps / e2e_s,
               "steps": e2e_steps, "ms_per_step": e2e_s / e2e_steps * 1e3,
               "step_ms": [round(x * 1e3, 1) for x in el], "warmup_step_ms": round(e2e_warm_ms, 1),
               "note": "C-ABI with host buffers: seeds from host, stranger + every full score vector "
                       "copied back to pinned host memory (the reference API returns ScoreVectors); "
                       "batch calls with TPA_ASYNC: batch k+1 computes while batch k drains over PCIe"}

    # the CLI's query output (rwrank_main.cpp:158-165, --top-k 10): device top-k,
    # only B*k ids + scores cross PCIe
    e2e_topk = None
    if not args.no_e2e:
        K = 10
        ids_h = torch.empty((batch, K), dtype=torch.int32, pin_memory=True)
        vals_h = torch.empty((batch, K), dtype=torch.float64, pin_memory=True)
        el = []
        for it in range(1 + max(1, min(args.steps, args.e2e_steps))):  # first one: untimed warm-up
            flush.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            art = C_.c_void_p()
            if pg is None:
                N.check(lib.tpa_preprocess(h, C, EPS, T, None, C_.byref(art), 0))
            else:
                N.check(lib.tpa_preprocess(pg.h, C, EPS, T, d_str.data_ptr(), None, N.TPA_DEVICE_PTRS))
                N.check(lib.tpa_artifact_create(h, d_str.data_ptr(), g.fingerprint(), C, EPS, T, N.TPA_DEVICE_PTRS,
                                                C_.byref(art)))
            for b in batches:
                N.check(lib.tpa_query_batch_topk(h, art, b.ctypes.data, len(b), S, K, ids_h.data_ptr(),
                                                 vals_h.data_ptr(), 0))
            torch.cuda.synchronize()
            if it:
                el.append(time.perf_counter() - t0)
            lib.tpa_artifact_destroy(art)
        e2e_s = max_over_ranks(sum(el))
        e2e_topk = {"value": edges_per_step * jobs * len(el) / e2e_s / 1e9, "unit": "GTEPS",
                    "k": K, "h2d_bytes_per_step": len(seeds) * 4, "d2h_bytes_per_step": len(seeds) * K * 12,
                    "queries_per_s": nq * jobs * len(el) / e2e_s,
                    "ms_per_step": e2e_s / len(el) * 1e3,
                    "note": "tpa_query_batch_topk: query batch + device top_k_nodes (metrics.cpp:25-36); "
                            "ids and scores of the top 10 per seed to pinned host memory"}

    if local_cpus:
        os.sched_setaffinity(0, all_cpus)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import Reference
    if rank == 0 and world == 1 and not args.no_cpu and Reference.available():
        t0 = time.perf_counter()
        off = g.out_offsets().astype(np.int64)
        rg = Reference().graph_from_edges(n, np.repeat(np.arange(n, dtype=np.uint32), np.diff(off)),
                                          g.out_targets(), "selfloop")
        del off
        assert rg.fingerprint == g.fingerprint(), "reference graph differs from the product's"
        log(f"[rank 0] reference graph for cpu_baseline in {time.perf_counter() - t0:.1f}s")
        cpu = cpu_measure(rg, seeds, budget_s=args.cpu_budget)
        del rg

    if rank == 0:
        clocks = clk.summary()
        gb = roofline.get("gather_bound")
        if gb and clocks.get("sm_mhz"):
            # a pull SpMM moves m x B x 8 bytes from L2 to the SMs whatever the hit
            # rate: the L2 slices' aggregate cap (B300_MICROARCH.md "LTS throughput
            # cap", ~6,300 B/clk, same L2 design) at the clock sustained in the run
            l2_peak = 6300.0 * clocks["sm_mhz"] * 1e6 / 1e9
            roofline["l2_bound"] = {"achieved_gbs": gb["achieved_gbs"], "peak_gbs": l2_peak,
                                    "frac": gb["achieved_gbs"] / l2_peak,
                                    "peak_source": "6,300 B/clk (microarchitecture notes, B300-measured) x "
                                                   "median SM clock of this run"}
        line = {
            "metric": "CPI edges/sec (GTEPS) and online RWR queries/sec; % of HBM roofline",
            "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if partitioned else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": workload_desc(cfg_name, n, m, len(g.dangling_nodes()), g.fingerprint(), nq, batch),
            "queries_per_s": qps, "preprocess_sweeps": pre_sweeps,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e if e2e is not None else e2e_topk,
            "e2e_topk": e2e_topk, "gpu_launches": launches,
            "clocks": clocks, "ingest_s": t_ingest, "graph_build_s": t_build,
            "e2e_host_cpus": sorted(local_cpus) if local_cpus else "all",
            "outputs": ("per batch: the B full score vectors written to HBM (the idle iterate buffer), then the "
                        "device top-10 per seed kept resident (tpa_query_batch_topk)" if resident_topk else
                        "the B full score vectors of every batch written to a resident [B][n] buffer"),
            "device_mem_gb": torch.cuda.max_memory_reserved(dev) / 1e9 + dg.device_bytes() / 1e9,
            "parallelism": (f"row-partitioned preprocess ({pg.transport} exchange per sweep: shares + exact residual "
                            f"limbs) + queries split over {world} whole-graph replicas" if partitioned else
                            f"independent replicas x{world}" if world > 1 else "single GPU"),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
