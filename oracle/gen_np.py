"""TEST INFRASTRUCTURE ONLY — numpy restatement of the benchmark generator
(paper_2502_17846_b200/csrc/grem_gen.h), so that bench.py's reference arm
builds its input graph without loading the product library
(libgrem_b200.so).  tests/test_oracle.py checks it byte-for-byte against the
library's host generator.

Same model and op sequence as grem_gen.h: a splitmix64 counter hash per
endpoint, u in [0, 1) from its top 53 bits, x = (1 + u * scale)^beta by the
fixed left-to-right binary exponentiation (every product a correctly-rounded
binary64 multiply — numpy never contracts to FMA), node = floor(x) - 1, then
the keyed xorshift-multiply bijection with cycle walking.
"""

from __future__ import annotations

import numpy as np

_U64 = np.uint64
_M1 = _U64(0xBF58476D1CE4E5B9)
_M2 = _U64(0x94D049BB133111EB)
_GOLD = _U64(0x9E3779B97F4A7C15)


def _mix64(z):
    z = z + _GOLD
    z = (z ^ (z >> _U64(30))) * _M1
    z = (z ^ (z >> _U64(27))) * _M2
    return z ^ (z >> _U64(31))


def _mix64_scalar(z: int) -> int:
    m = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def _ipow(v, beta: int):
    r = np.ones_like(v) if isinstance(v, np.ndarray) else 1.0
    for bit in range(31, -1, -1):
        r = r * r
        if (beta >> bit) & 1:
            r = r * v
    return r


def _root_scale(n: int, beta: int) -> float:
    a = float(n + 1)
    r = 1.0
    while _ipow(r * 2.0, beta) <= a:
        r = r * 2.0
    lo, hi = r, r * 2.0
    for _ in range(200):
        mid = (lo + hi) * 0.5
        if mid == lo or mid == hi:
            break
        if _ipow(mid, beta) <= a:
            lo = mid
        else:
            hi = mid
    return lo - 1.0


def _perm_step(x, key: int, bits: int, mask):
    sh = _U64(bits // 2 + 1)
    sh2 = _U64(bits // 2 if bits // 2 + 1 > 2 else 1)
    x = (x ^ _U64(key)) & mask
    x = (x * _U64(0xD6E8FEB86659FD93)) & mask
    x ^= x >> sh
    x = (x * _GOLD + _U64(key | 1)) & mask
    x ^= x >> sh
    x = (x * _M1) & mask
    x ^= x >> sh2
    return x & mask


def powerlaw_edges(num_nodes: int, num_edges: int, beta: int = 11, seed: int = 0, e0: int = 0) -> np.ndarray:
    """(num_edges, 2) uint32: edges [e0, e0 + num_edges) of the graph (num_nodes, beta, seed)."""
    n = int(num_nodes)
    bits = 1
    while (1 << bits) < n:
        bits += 1
    mask = _U64((1 << bits) - 1)
    scale = _root_scale(n, beta)
    hseed = _U64(_mix64_scalar(seed))
    k0 = _mix64_scalar(seed ^ 0x5DEECE66D)
    k1 = _mix64_scalar(k0)
    out = np.empty(2 * num_edges, dtype=np.uint32)
    step = 1 << 22
    with np.errstate(over="ignore"):
        for lo in range(0, 2 * num_edges, step):
            j = np.arange(2 * e0 + lo, 2 * e0 + min(2 * num_edges, lo + step), dtype=np.uint64)
            h = _mix64(hseed ^ j)
            u = (h >> _U64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
            x = _ipow(1.0 + u * scale, beta)
            raw = x.astype(np.uint64)
            raw = np.where(raw >= 1, raw - _U64(1), _U64(0))
            raw = np.minimum(raw, _U64(n - 1))
            pending = np.ones(raw.shape, dtype=bool)
            while pending.any():
                y = _perm_step(raw[pending], k0, bits, mask)
                y = _perm_step(y, k1, bits, mask)
                raw[pending] = y
                pending[pending] = y >= _U64(n)
            out[lo:lo + raw.size] = raw.astype(np.uint32)
    return out.reshape(-1, 2)
