"""Unit test of the chunk scan kernels vs a sequential evaluation of the same maps."""
import sys, ctypes
sys.path.insert(0, ".")
import numpy as np
from paper_2502_17846_b200 import _abi, grem

L = _abi.lib()
L.grem_debug_chunk_scan.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]

def seq(meta, newb, x0, cap, spec_exact=False):
    nc = len(meta); x = np.empty(nc + 1, np.int64); cur = x0; xs = np.empty(nc + 1, np.int64)
    for i in range(nc):
        m = int(meta[i]); x[i] = cur
        active = m & 4
        if not active: continue
        old = (m & 3) - 1; o = 1 if old == 0 else 0; lift = 1 if old != -1 else 0
        sl = int(newb[i]) - lift; pref = (m >> 4) & 3
        if pref == 0: t = cap - 1
        elif pref == 1: t = sl - cap
        else: t = sl >> 1
        b0 = (cur - o) <= t
        cur = cur - o + (1 if b0 else 0)
    x[nc] = cur
    return x

rng = np.random.default_rng(0)
bad = 0
for trial in range(40):
    nc = int(rng.choice([5, 100, 4095, 4097, 20000, 100000, 300000]))
    cap = int(rng.integers(nc // 4 + 1, nc + 10))
    # generate a feasible trajectory by simulating random maps sequentially
    meta = np.zeros(nc, np.uint8); newb = np.zeros(nc, np.int32)
    x = int(rng.integers(0, cap // 2 + 1)); s = x + int(rng.integers(0, cap // 2 + 1))
    x0 = x
    for i in range(nc):
        active = rng.random() < 0.9
        old = int(rng.choice([-1, 0, 1])) if s > 0 else -1
        if old == 0 and x == 0: old = 1 if s - x > 0 else -1
        if old == 1 and s - x == 0: old = 0 if x > 0 else -1
        pref = int(rng.choice([0, 1, 2]))
        spec = int(rng.integers(0, 2))
        m = (old + 1) | (4 if active else 0) | (8 if old == -1 else 0) | (pref << 4) | (spec << 6)
        meta[i] = m
        newb[i] = s + (1 if (active and old != -1) else 0) if False else s + 0
        # newb holds s before node i; s_l = newb - lift
        newb[i] = s
        if not active: continue
        o = 1 if old == 0 else 0; lift = 1 if old != -1 else 0
        sl = s - lift; xl = x - o
        if 2 * cap < sl + 1: break
        if pref == 0: b0 = xl <= cap - 1
        elif pref == 1: b0 = xl <= sl - cap
        else: b0 = xl <= sl // 2
        x = xl + (1 if b0 else 0); s = sl + 1
    xo = np.empty(nc + 1, np.int32); bo = np.empty(nc, np.uint8); nb = np.zeros(2, np.int64)
    rc = L.grem_debug_chunk_scan(grem.context(), meta.ctypes.data, newb.ctypes.data, nc, x0, cap, 1,
                                 xo.ctypes.data, bo.ctypes.data, nb.ctypes.data)
    assert rc == 0, _abi.last_error()
    ref = seq(meta, newb, x0, cap)
    ok = np.array_equal(xo.astype(np.int64), ref)
    if not ok:
        bad += 1
        first = int(np.flatnonzero(xo.astype(np.int64) != ref)[0])
        print(f"trial {trial} nc={nc}: MISMATCH first at {first} (tile {first // 4096}) gpu={xo[first]} ref={ref[first]} flagged={nb[0]} walk={nb[1]}")
    else:
        print(f"trial {trial} nc={nc}: ok flagged={nb[0]} walk={nb[1]}")
print("SCAN BAD", bad)
