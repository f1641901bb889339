"""Prototype of the trajectory-bundle repair: per segment of L nodes simulate
64 trajectories starting at two windows (centers c1, c2, +-16); chain segments
exactly; count window misses (segments whose exact input is in no window)."""
import sys, os
sys.path.insert(0, ".")
from math import ceil
import numpy as np
import tools.proto_rounds as pr

MISS = {"segs": 0, "miss": 0, "calls": 0}

def step(xv, i, pref, o, thr, sl, cap):
    p = pref[i]
    if p == 3:
        return xv
    xl = xv - o[i]
    return xl + (xl <= thr[i]).astype(np.int64)

def bundle_exact(x0, pref, o, thr, s_l, cap, c1, c2, L):
    """returns exact x (len nn+1) using the bundle method; c1/c2: candidate x at each node"""
    nn = len(pref)
    MISS["calls"] += 1
    W = int(os.environ.get("BW", "16")); off = np.arange(-W, W)
    ends = []
    for st in range(0, nn, L):
        starts = np.concatenate([c1[st] + off, c2[st] + off])
        xv = starts.copy()
        for i in range(st, min(st + L, nn)):
            xv = step(xv, i, pref, o, thr, s_l, cap)
        ends.append((starts, xv))
    x = np.empty(nn + 1, np.int64)
    cur = x0
    for si, st in enumerate(range(0, nn, L)):
        MISS["segs"] += 1
        starts, xv = ends[si]
        hit = np.flatnonzero(starts == cur)
        out = None
        if hit.size:
            out = xv[hit[0]]
        else:
            MISS["miss"] += 1
        xe = cur
        for i in range(st, min(st + L, nn)):
            x[i] = xe
            xe = int(step(np.array([xe]), i, pref, o, thr, s_l, cap)[0])
        if out is not None:
            assert out == xe
        cur = xe
    x[nn] = cur
    return x
