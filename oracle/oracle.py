"""TEST INFRASTRUCTURE ONLY — ctypes front end of the C restatement
(oracle/grem_oracle.c) of the reference GREM path.

It is the checker the CUDA path is compared against, and the timed CPU
baseline of bench.py (kind "port").  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs import it; the product package
never does.

Parity pin: tests/test_oracle.py checks it label-for-label against the Python
reference (streamcut, installed under baseline/_ref) on random multigraphs in
the distribution of the reference's own tests (tests/helpers.py:16) and against
the golden fixtures in tests/golden/ (made by tests/golden/make_golden.py from
streamcut itself).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from math import ceil

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libgrem_oracle.so")
_lib = None

SEED_CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_int8), ctypes.c_void_p)
CHUNK_CB = ctypes.CFUNCTYPE(None, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int8), ctypes.c_void_p)


class OracleStats(ctypes.Structure):
    _fields_ = [("chunks", ctypes.c_int64), ("visits", ctypes.c_int64),
                ("moves", ctypes.c_int64), ("ties", ctypes.c_int64)]


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.oracle_bisect.argtypes = [P, i64, i64, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, SEED_CB, P, CHUNK_CB, P, P, P, P]
        L.oracle_bisect.restype = ctypes.c_int
        L.oracle_partition.argtypes = [P, i64, i64, i64, ctypes.c_double, ctypes.c_double, i64,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       SEED_CB, P, P, P]
        L.oracle_partition.restype = ctypes.c_int
        L.oracle_count_cuts.argtypes = [P, i64, i64, P, P, P, i64, P]
        L.oracle_count_cuts.restype = ctypes.c_int
        L.oracle_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc: int):
    if rc:
        raise OracleError(rc, lib().oracle_last_error().decode())


def _random_seed_cb(rng_seed: int):
    def cb(nn, out, user):
        rng = np.random.default_rng(rng_seed)         # seed.py:48-52
        labels = np.ones(nn, dtype=np.int8)
        labels[rng.permutation(nn)[: ceil(nn / 2)]] = 0
        ctypes.memmove(out, labels.ctypes.data, nn)
        return 0
    return SEED_CB(cb)


def _edges_u32(edges) -> np.ndarray:
    e = np.ascontiguousarray(np.asarray(edges).reshape(-1, 2))
    if e.size and int(e.max()) >= 2**32:
        raise ValueError("oracle handles 32-bit ids only")
    return np.ascontiguousarray(e.astype(np.uint32))


def chunk_edges_for(num_edges: int, chunk_edges=None, chunk_frac=None) -> int:
    """ChunkPlan.plan (edgefile.py:338-349); default frac 0.1 (grem.py:72-75)."""
    if chunk_edges is None and chunk_frac is None:
        chunk_frac = 0.1
    if chunk_frac is not None:
        return max(1, ceil(chunk_frac * num_edges))
    return int(chunk_edges)


def bisect(edges, n: int, chunk_edges: int, cap: int, refine=True, passes=1, seed_algo="bfs_grow",
           seed_refinement_passes=2, rng_seed=0, on_chunk=None, stats=None):
    e = _edges_u32(edges)
    labels = np.empty(n, dtype=np.int8)
    sizes = np.zeros(2, dtype=np.int64)
    seed_cb = _random_seed_cb(rng_seed) if seed_algo == "random" else SEED_CB(0)
    if on_chunk is not None:
        def _cb(s, parts, u):
            try:
                on_chunk((s[0], s[1]), np.ctypeslib.as_array(parts, shape=(n,)).astype(np.int32))
            except TypeError:
                on_chunk((s[0], s[1]))
        chunk_cb = CHUNK_CB(_cb)
    else:
        chunk_cb = CHUNK_CB(0)
    st = stats if stats is not None else OracleStats()
    rc = lib().oracle_bisect(e.ctypes.data, e.shape[0], n, chunk_edges, cap, int(refine), passes,
                             1 if seed_algo == "random" else 0, seed_refinement_passes, seed_cb, None,
                             chunk_cb, None, labels.ctypes.data, sizes.ctypes.data, ctypes.byref(st))
    _check(rc)
    return labels.astype(np.int32)


def partition(edges, n: int, p: int, slack=0.0, chunk_frac=None, chunk_edges=None, refine=True, passes=1,
              seed_algo="bfs_grow", seed_refinement_passes=2, rng_seed=0, stats=None):
    e = _edges_u32(edges)
    labels = np.empty(n, dtype=np.int32)
    if chunk_edges is None and chunk_frac is None:
        chunk_frac = 0.1
    frac = -1.0 if chunk_frac is None else float(chunk_frac)
    seed_cb = _random_seed_cb(rng_seed) if seed_algo == "random" else SEED_CB(0)
    st = stats if stats is not None else OracleStats()
    rc = lib().oracle_partition(e.ctypes.data, e.shape[0], n, p, float(slack), frac, int(chunk_edges or 0),
                                int(refine), passes, 1 if seed_algo == "random" else 0,
                                seed_refinement_passes, seed_cb, None, labels.ctypes.data, ctypes.byref(st))
    _check(rc)
    return labels


def count_cuts(edges, n: int, labels):
    """Returns (cut_edges, partition_sizes tuple) like grem.count_cuts (grem.py:227-252)."""
    e = _edges_u32(edges)
    lab = np.ascontiguousarray(np.asarray(labels, dtype=np.int32))
    sizes = np.zeros(max(2, int(lab.max()) + 2 if lab.size else 2), dtype=np.int64)
    cut = ctypes.c_int64()
    nparts = ctypes.c_int64()
    rc = lib().oracle_count_cuts(e.ctypes.data, e.shape[0], n, lab.ctypes.data, ctypes.byref(cut),
                                 sizes.ctypes.data, sizes.shape[0], ctypes.byref(nparts))
    _check(rc)
    return int(cut.value), tuple(int(x) for x in sizes[: nparts.value])
