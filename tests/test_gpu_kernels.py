"""GPU unit test of the sizes-chain kernels (speculative clamp scan, tie
verification and trajectory-bundle repair) against a sequential evaluation
of the same node maps on random feasible trajectories."""
import ctypes

import numpy as np
import pytest

from paper_2502_17846_b200 import _abi, grem

pytestmark = pytest.mark.gpu


def _seq(meta, newb, x0, cap):
    nc = len(meta)
    x = np.empty(nc + 1, np.int64)
    cur = x0
    for i in range(nc):
        m = int(meta[i])
        x[i] = cur
        if not m & 4:
            continue
        old = (m & 3) - 1
        o = 1 if old == 0 else 0
        sl = int(newb[i]) - (1 if old != -1 else 0)
        pref = (m >> 4) & 3
        t = cap - 1 if pref == 0 else (sl - cap if pref == 1 else sl >> 1)
        xl = cur - o
        cur = xl + (1 if xl <= t else 0)
    x[nc] = cur
    return x


def _random_chain(rng, nc):
    cap = int(rng.integers(nc // 4 + 1, nc + 10))
    meta = np.zeros(nc, np.uint8)
    newb = np.zeros(nc, np.int32)
    x = int(rng.integers(0, cap // 2 + 1))
    s = x + int(rng.integers(0, cap // 2 + 1))
    x0 = x
    tie_bias = rng.random()
    for i in range(nc):
        active = rng.random() < 0.9
        old = int(rng.choice([-1, 0, 1])) if s > 0 else -1
        if old == 0 and x == 0:
            old = 1 if s - x > 0 else -1
        if old == 1 and s - x == 0:
            old = 0 if x > 0 else -1
        pref = 2 if rng.random() < tie_bias else int(rng.choice([0, 1]))
        meta[i] = (old + 1) | (4 if active else 0) | (8 if old == -1 else 0) | (pref << 4) | (int(rng.integers(0, 2)) << 6)
        newb[i] = s
        if not active:
            continue
        o = 1 if old == 0 else 0
        lift = 1 if old != -1 else 0
        sl = s - lift
        xl = x - o
        t = cap - 1 if pref == 0 else (sl - cap if pref == 1 else sl // 2)
        x = xl + (1 if xl <= t else 0)
        s = sl + 1
    return meta, newb, x0, cap


def test_chunk_scan_and_bundle_exact():
    L = _abi.lib()
    L.grem_debug_chunk_scan.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] * 3 + [ctypes.c_int] + \
        [ctypes.c_void_p] * 3
    rng = np.random.default_rng(0)
    for trial in range(30):
        nc = int(rng.choice([1, 5, 100, 4095, 4097, 20000, 150000]))
        meta, newb, x0, cap = _random_chain(rng, nc)
        ref = _seq(meta, newb, x0, cap)
        for mode in (2, 3, 1):   # 2/3: trajectory bundles with 3/2 windows (production), 1: sequential walk
            xo = np.empty(nc + 1, np.int32)
            bo = np.empty(nc, np.uint8)
            nb = np.zeros(2, np.int64)
            rc = L.grem_debug_chunk_scan(grem.context(), meta.ctypes.data, newb.ctypes.data, nc, x0, cap, mode,
                                         xo.ctypes.data, bo.ctypes.data, nb.ctypes.data)
            assert rc == 0, _abi.last_error()
            assert np.array_equal(xo.astype(np.int64), ref), (trial, nc, mode)
