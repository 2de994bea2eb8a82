"""Parity checkers for the CPI hot path -- TEST INFRASTRUCTURE ONLY.

Two CPU implementations live here, both used strictly as checkers:

* ``Oracle`` -- ctypes binding of ``cpi_oracle.c``, the plain-C restatement of
  the reference's algorithm (graph.cpp sweep, cpi.cpp run_series / cpi_run /
  cpi_partition, tpa.cpp preprocess / query / query_na).
* ``Reference`` -- ctypes binding of ``_ref/librwrank_ref.so``: the unmodified
  reference library compiled from /root/reference/proj/src plus the
  ``ref_capi.cpp`` extern "C" shim.  Present wherever ``make -C oracle`` ran
  while /root/reference existed (it travels to the GPU box prebuilt).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_1708_02574_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libcpi_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "librwrank_ref.so")

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

POLICIES = {"selfloop": 0, "uniform": 1, "drop": 2}


def build() -> None:
    """Compile the C oracle (and the reference, when its sources are present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _policy(p) -> int:
    return POLICIES[p] if isinstance(p, str) else int(p)


class Oracle:
    """C restatement of the reference CPI path (cpi_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        lib.oracle_sweep.argtypes = [C.c_uint32, _u64p, _u32p, C.c_int, _f64p, _f64p, C.c_double]
        lib.oracle_sweep.restype = None
        lib.oracle_run_series.argtypes = [
            C.c_uint32, _u64p, _u32p, C.c_int, C.c_void_p, C.c_uint64, C.c_double, C.c_double,
            C.c_uint32, C.c_int64, C.c_void_p, C.c_size_t, _f64p,
            C.POINTER(C.c_uint32), C.POINTER(C.c_int), C.POINTER(C.c_double)]
        lib.oracle_run_series.restype = C.c_int
        lib.oracle_neighbor_scale_factor.argtypes = [C.c_double, C.c_uint32, C.c_uint32]
        lib.oracle_neighbor_scale_factor.restype = C.c_double
        lib.oracle_query.argtypes = [C.c_uint32, _u64p, _u32p, C.c_int, C.c_void_p, C.c_double,
                                     C.c_double, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, _f64p]
        lib.oracle_query.restype = C.c_int
        self.lib = lib

    @staticmethod
    def _csr(g):
        """(n, off, tgt, policy) from any graph exposing the reference accessors
        (node_count(), out_offsets(), out_targets(), dangling_policy()) or plain
        attributes (n, out_offsets, out_targets, policy)."""
        def get(*names):
            for nm in names:
                if hasattr(g, nm):
                    v = getattr(g, nm)
                    return v() if callable(v) else v
            raise AttributeError(names)
        return (int(get("node_count", "n")), np.ascontiguousarray(get("out_offsets"), np.uint64),
                np.ascontiguousarray(get("out_targets"), np.uint32),
                _policy(get("dangling_policy", "policy")))

    def sweep(self, g, x, c):
        n, off, tgt, pol = self._csr(g)
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(n, np.float64)
        self.lib.oracle_sweep(n, off, tgt, pol, x, y, c)
        return y

    def run_series(self, g, seeds, c, eps, start=0, terminal=None, bounds=None):
        """seeds=None -> all nodes (pagerank).  Returns (scores, iters, converged, residual);
        with bounds, scores is (len(bounds)+1, n)."""
        n, off, tgt, pol = self._csr(g)
        sd = None if seeds is None else np.ascontiguousarray(sorted(seeds), np.uint32)
        bd = None if bounds is None else np.ascontiguousarray(bounds, np.uint32)
        nout = n if bd is None else n * (len(bd) + 1)
        out = np.empty(max(nout, 1), np.float64)
        it, conv, res = C.c_uint32(), C.c_int(), C.c_double()
        self.lib.oracle_run_series(
            n, off, tgt, pol, None if sd is None else sd.ctypes.data, 0 if sd is None else len(sd),
            c, eps, start, -1 if terminal is None else int(terminal),
            None if bd is None else bd.ctypes.data, 0 if bd is None else len(bd), out,
            C.byref(it), C.byref(conv), C.byref(res))
        out = out[:nout]
        if bd is not None:
            out = out.reshape(len(bd) + 1, n)
        return out, it.value, bool(conv.value), res.value

    def cpi_run(self, g, seeds, c, eps, start=0, terminal=None):
        return self.run_series(g, seeds, c, eps, start, terminal)

    def pagerank(self, g, c, eps, start=0, terminal=None):
        return self.run_series(g, None, c, eps, start, terminal)

    def exact_rwr(self, g, seed, c=0.15, eps=1e-9):
        return self.run_series(g, [seed], c, eps)[0]

    def cpi_partition(self, g, seeds, c, eps, bounds):
        return self.run_series(g, seeds, c, eps, bounds=list(bounds))[0]

    def neighbor_scale_factor(self, c, S, T):
        return self.lib.oracle_neighbor_scale_factor(c, S, T)

    def preprocess(self, g, c, eps, T):
        return self.run_series(g, None, c, eps, start=T)[0]

    def query(self, g, stranger, c, eps, T, seed, S, na=False):
        n, off, tgt, pol = self._csr(g)
        out = np.empty(n, np.float64)
        st = None if stranger is None else np.ascontiguousarray(stranger, np.float64)
        self.lib.oracle_query(n, off, tgt, pol, None if st is None else st.ctypes.data, c, eps,
                              T, seed, S, 1 if na else 0, out)
        return out


class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Reference:
    """The unmodified reference library (oracle/_ref/librwrank_ref.so)."""

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def __init__(self, path: str = REF_SO):
        lib = C.CDLL(path)
        vp = C.c_void_p
        sig = {
            "ref_last_error": ([], C.c_char_p),
            "ref_graph_from_edges": ([C.c_uint32, _u32p, _u32p, C.c_uint64, C.c_int, C.POINTER(vp)], C.c_int),
            "ref_graph_random": ([C.c_uint32, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(vp)], C.c_int),
            "ref_graph_rmat": ([C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_int,
                                C.c_int, C.POINTER(vp)], C.c_int),
            "ref_sample_seeds": ([vp, C.c_uint64, C.c_uint64, _u32p], C.c_int),
            "ref_graph_max_indeg": ([vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)], None),
            "ref_graph_free": ([vp], None),
            "ref_graph_n": ([vp], C.c_uint32),
            "ref_graph_m": ([vp], C.c_uint64),
            "ref_graph_fingerprint": ([vp], C.c_uint64),
            "ref_graph_n_dangling": ([vp], C.c_uint64),
            "ref_graph_csr": ([vp, vp, vp, vp], None),
            "ref_sweep": ([vp, _f64p, _f64p, C.c_double, C.c_int], C.c_int),
            "ref_cpi_run": ([vp, vp, C.c_uint64, C.c_double, C.c_double, C.c_uint32, C.c_int64, C.c_int,
                             _f64p, C.POINTER(C.c_uint32), C.POINTER(C.c_int), C.POINTER(C.c_double)], C.c_int),
            "ref_exact_rwr": ([vp, C.c_uint32, C.c_double, C.c_double, C.c_int, _f64p], C.c_int),
            "ref_cpi_partition": ([vp, _u32p, C.c_uint64, C.c_double, C.c_double, _u32p, C.c_uint64, C.c_int,
                                   _f64p], C.c_int),
            "ref_neighbor_scale_factor": ([C.c_double, C.c_uint32, C.c_uint32], C.c_double),
            "ref_preprocess": ([vp, C.c_double, C.c_double, C.c_uint32, C.c_int, _f64p, C.POINTER(C.c_uint64)], C.c_int),
            "ref_query": ([vp, _f64p, C.c_uint64, C.c_double, C.c_double, C.c_uint32, C.c_uint32, C.c_uint32,
                           C.c_int, _f64p], C.c_int),
            "ref_query_na": ([vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_int, _f64p], C.c_int),
            "ref_query_many": ([vp, _f64p, C.c_uint64, C.c_double, C.c_double, C.c_uint32, _u32p, C.c_uint32,
                                C.c_uint32, C.c_int, vp, C.POINTER(C.c_double)], C.c_int),
            "ref_time_preprocess": ([vp, C.c_double, C.c_double, C.c_uint32, C.c_int, vp, C.POINTER(C.c_double)], C.c_int),
            "ref_time_sweeps": ([vp, C.c_uint32, C.c_double, C.c_int, C.POINTER(C.c_double)], C.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        self.lib = lib

    def _chk(self, rc):
        if rc != 0:
            raise RefError(rc, self.lib.ref_last_error().decode())

    # --- graphs -----------------------------------------------------------
    def graph_from_edges(self, n, src, dst, policy="selfloop"):
        h = C.c_void_p()
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        self._chk(self.lib.ref_graph_from_edges(n, src, dst, len(src), _policy(policy), C.byref(h)))
        return RefGraph(self, h)

    def graph_random(self, n, m, seed, policy="selfloop"):
        h = C.c_void_p()
        self._chk(self.lib.ref_graph_random(n, m, seed, _policy(policy), C.byref(h)))
        return RefGraph(self, h)

    def graph_rmat(self, scale, edge_factor, a=0.57, b=0.19, c=0.19, seed=1, policy="selfloop", threads=0):
        """The benchmark R-MAT graph built by the reference Graph constructor
        (ref_capi.cpp ref_graph_rmat; same edges as the product's generator)."""
        h = C.c_void_p()
        self._chk(self.lib.ref_graph_rmat(scale, edge_factor, a, b, c, seed, _policy(policy), threads, C.byref(h)))
        return RefGraph(self, h)


class RefGraph:
    """A reference rwrank::Graph living in the reference library."""

    def __init__(self, ref: Reference, h):
        self.ref, self.h = ref, h
        lib = ref.lib
        self.n = lib.ref_graph_n(h)
        self.m = lib.ref_graph_m(h)
        self.fingerprint = lib.ref_graph_fingerprint(h)
        nd = lib.ref_graph_n_dangling(h)
        self.out_offsets = np.empty(self.n + 1, np.uint64)
        self.out_targets = np.empty(self.m, np.uint32)
        self.dangling = np.empty(nd, np.uint32)
        lib.ref_graph_csr(h, self.out_offsets.ctypes.data, self.out_targets.ctypes.data,
                          self.dangling.ctypes.data)
        self._policy = None

    def __del__(self):
        try:
            self.ref.lib.ref_graph_free(self.h)
        except Exception:
            pass

    # the policy is not exported by the shim; callers set it
    @property
    def policy(self):
        return self._policy

    def sample_seeds(self, count, rng_seed):
        """rwrank_main.cpp:65-83 restated (ref_capi.cpp ref_sample_seeds)."""
        out = np.empty(count, np.uint32)
        self.ref._chk(self.ref.lib.ref_sample_seeds(self.h, count, rng_seed, out))
        return out

    def max_indeg(self):
        node, deg = C.c_uint32(), C.c_uint64()
        self.ref.lib.ref_graph_max_indeg(self.h, C.byref(node), C.byref(deg))
        return node.value, deg.value

    def sweep(self, x, c, threads=1):
        y = np.empty(self.n, np.float64)
        self.ref._chk(self.ref.lib.ref_sweep(self.h, np.ascontiguousarray(x, np.float64), y, c, threads))
        return y

    def cpi_run(self, seeds, c, eps, start=0, terminal=None, threads=1):
        out = np.empty(self.n, np.float64)
        it, conv, res = C.c_uint32(), C.c_int(), C.c_double()
        sd = None if seeds is None else np.ascontiguousarray(seeds, np.uint32)
        self.ref._chk(self.ref.lib.ref_cpi_run(
            self.h, None if sd is None else sd.ctypes.data, 0 if sd is None else len(sd), c, eps, start,
            -1 if terminal is None else terminal, threads, out, C.byref(it), C.byref(conv), C.byref(res)))
        return out, it.value, bool(conv.value), res.value

    def exact_rwr(self, seed, c=0.15, eps=1e-9, threads=1):
        out = np.empty(self.n, np.float64)
        self.ref._chk(self.ref.lib.ref_exact_rwr(self.h, seed, c, eps, threads, out))
        return out

    def cpi_partition(self, seeds, c, eps, bounds, threads=1):
        bd = np.ascontiguousarray(bounds, np.uint32)
        out = np.empty((len(bd) + 1) * self.n, np.float64)
        sd = np.ascontiguousarray(seeds, np.uint32)
        self.ref._chk(self.ref.lib.ref_cpi_partition(self.h, sd, len(sd), c, eps, bd, len(bd), threads, out))
        return out.reshape(len(bd) + 1, self.n)

    def preprocess(self, c, eps, T, threads=1):
        out = np.empty(self.n, np.float64)
        fp = C.c_uint64()
        self.ref._chk(self.ref.lib.ref_preprocess(self.h, c, eps, T, threads, out, C.byref(fp)))
        return out

    def query(self, stranger, c, eps, T, seed, S, fingerprint=None, threads=1):
        out = np.empty(self.n, np.float64)
        fp = self.fingerprint if fingerprint is None else fingerprint
        self.ref._chk(self.ref.lib.ref_query(self.h, np.ascontiguousarray(stranger, np.float64), fp, c, eps,
                                             T, seed, S, threads, out))
        return out

    def query_na(self, seed, S, T, c, eps, threads=1):
        out = np.empty(self.n, np.float64)
        self.ref._chk(self.ref.lib.ref_query_na(self.h, seed, S, T, c, eps, threads, out))
        return out

    def query_many(self, stranger, c, eps, T, seeds, S, workers, keep=False):
        sd = np.ascontiguousarray(seeds, np.uint32)
        out = np.empty((len(sd), self.n), np.float64) if keep else None
        sec = C.c_double()
        self.ref._chk(self.ref.lib.ref_query_many(
            self.h, np.ascontiguousarray(stranger, np.float64), self.fingerprint, c, eps, T, sd, len(sd), S,
            workers, None if out is None else out.ctypes.data, C.byref(sec)))
        return out, sec.value

    def time_preprocess(self, c, eps, T, threads=1, keep=False):
        out = np.empty(self.n, np.float64) if keep else None
        sec = C.c_double()
        self.ref._chk(self.ref.lib.ref_time_preprocess(self.h, c, eps, T, threads,
                                                       None if out is None else out.ctypes.data, C.byref(sec)))
        return out, sec.value

    def time_sweeps(self, sweeps, c, threads=1):
        sec = C.c_double()
        self.ref._chk(self.ref.lib.ref_time_sweeps(self.h, sweeps, c, threads, C.byref(sec)))
        return sec.value
