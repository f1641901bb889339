"""Node statistics of the analytical cut model on the GPU — drop-in for
streamcut.theory.compute_node_stats (theory.py:97-122).

``compute_node_stats(efile, labels)`` is one pass over the edge list: per
node, ``k`` = neighbour endpoints excluding self-loops (duplicates count with
multiplicity) and ``k0`` = those on the node's majority side of the bisection
``labels``.  It runs behind the C ABI (``grem_node_stats_u32``: two label
gathers and two 64-bit REDs per edge, then k = c0 + c1, k0 = max) and returns
the reference's ``NodeStats`` when it is importable.

``expected_cuts(stats, x, multiplier)`` / ``theory_curve(stats, xs,
multiplier)`` (theory.py:125-146) run behind ``grem_theory_curve``: one
thread per node sums its hypergeometric tail (long tails: one CTA per node)
from a device log-gamma table, and the per-node expected cut endpoints are
reduced in a fixed order.  The domain errors are the reference's, raised in
the order its per-node loop would meet them.
"""

from __future__ import annotations

import os

import numpy as np

from . import _abi
from .edgefile import edges_u32, is_native_binary
from .errors import FormatError
from .grem import _raise, context

try:   # the reference's class, so callers' isinstance checks hold
    from streamcut.model import NodeStats  # type: ignore
except Exception:  # noqa: BLE001
    class NodeStats:
        """Per-node degree ``k`` and majority-side degree ``k0`` (model.py:135-160)."""

        __slots__ = ("k", "k0")

        def __init__(self, k, k0):
            k = np.asarray(k, dtype=np.int64)
            k0 = np.asarray(k0, dtype=np.int64)
            if k.shape != k0.shape:
                raise FormatError("k and k0 must have the same shape")
            if np.any(k0 < 0) or np.any(k0 > k) or np.any(2 * k0 < k):
                raise FormatError("need 0 <= k - k0 <= k0 <= k for every node")
            self.k = k
            self.k0 = k0

        def __len__(self) -> int:
            return len(self.k)

        @property
        def total_endpoints(self) -> int:
            return int(self.k.sum())


try:   # the reference's point type, so callers comparing results see the same class
    from streamcut.theory import TheoryCurvePoint  # type: ignore
except Exception:  # noqa: BLE001
    from dataclasses import dataclass

    @dataclass(frozen=True)
    class TheoryCurvePoint:
        """theory.py:29-32."""
        x: float
        expected_cuts: float
        expected_cut_fraction: float


def _curve(stats, xs, multiplier):
    """expected cut endpoints for every x (GPU), with the reference's errors"""
    xs = list(xs)
    if not xs:
        return [], 0
    k = np.ascontiguousarray(np.asarray(stats.k, dtype=np.int64))
    k0 = np.ascontiguousarray(np.asarray(stats.k0, dtype=np.int64))
    xa = np.ascontiguousarray(np.asarray([float(x) for x in xs], dtype=np.float64))
    out = np.zeros(len(xs), dtype=np.float64)
    info = np.full(3, -1, dtype=np.int64)
    rc = _abi.lib().grem_theory_curve(context(), k.ctypes.data, k0.ctypes.data, k.shape[0], 0, xa.ctypes.data,
                                      len(xs), float(multiplier), out.ctypes.data, info.ctypes.data)
    if rc == 1 and k.shape[0] > 0 and info[0] >= 0:   # a domain error: the reference's message and order
        first, bad = int(info[0]), int(info[1])

        def majority(i):
            return FormatError(f"k0 must be the majority side: got k={int(k[i])}, k0={int(k0[i])}")
        if bad == first:
            raise majority(first)
        if not 0 < xs[0] <= 1:
            raise FormatError(f"chunk fraction must be in (0, 1], got {xs[0]}")
        if multiplier < 1:
            raise FormatError(f"multiplier must be >= 1, got {multiplier}")
        if bad >= 0:
            raise majority(bad)
        for x in xs[1:]:
            if not 0 < x <= 1:
                raise FormatError(f"chunk fraction must be in (0, 1], got {x}")
    _raise(rc)
    return [float(v) for v in out], int(info[2])


def expected_cuts(stats, x: float, multiplier: float = 1.0):
    """theory.py:125-142: expected cut endpoints at chunk fraction x."""
    (total,), endpoints = _curve(stats, [x], multiplier)
    return TheoryCurvePoint(float(x), total, total / endpoints if endpoints else 0.0)


def theory_curve(stats, xs, multiplier: float = 1.0):
    """theory.py:145-146 (all points from one staging of the node stats)."""
    xs = [float(x) for x in xs]
    totals, endpoints = _curve(stats, xs, multiplier)
    return [TheoryCurvePoint(x, t, t / endpoints if endpoints else 0.0) for x, t in zip(xs, totals)]


def curve_csv(points, multiplier: float) -> str:
    """theory.py:149-153."""
    lines = ["x,expected_cuts,expected_cut_fraction,multiplier"]
    for pt in points:
        lines.append(f"{pt.x},{pt.expected_cuts},{pt.expected_cut_fraction},{multiplier}")
    return "\n".join(lines) + "\n"


def node_stats_edges(edges, num_nodes: int, labels, on_device_ptr: int | None = None,
                     num_edges: int | None = None):
    """Array-level entry: (m, 2) u32 edges on the host, or a device pointer."""
    lab = np.ascontiguousarray(np.asarray(labels).astype(np.int32))
    n = int(num_nodes)
    if lab.shape[0] != n:
        raise FormatError(f"labels cover {lab.shape[0]} nodes, file has {n}")
    k = np.empty(n, dtype=np.int64)
    k0 = np.empty(n, dtype=np.int64)
    if on_device_ptr is not None:
        ptr, m, dev = on_device_ptr, int(num_edges), 1
    else:
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        ptr, m, dev = e.ctypes.data, e.shape[0], 0
    rc = _abi.lib().grem_node_stats_u32(context(), ptr, m, n, dev, lab.ctypes.data, 0, k.ctypes.data,
                                        k0.ctypes.data)
    _raise(rc)
    return NodeStats(k, k0)


def compute_node_stats(efile, labels):
    """theory.py:97-122."""
    n = int(efile.meta.num_nodes)
    labels = np.asarray(labels)
    if labels.shape[0] != n:
        raise FormatError(f"labels cover {labels.shape[0]} nodes, file has {n}")
    if not is_native_binary(efile):
        return node_stats_edges(edges_u32(efile), n, labels)
    lab = np.ascontiguousarray(labels.astype(np.int32))
    k = np.empty(n, dtype=np.int64)
    k0 = np.empty(n, dtype=np.int64)
    rc = _abi.lib().grem_node_stats_file(context(), os.fsencode(efile.path), lab.ctypes.data, 0, k.ctypes.data,
                                         k0.ctypes.data)
    _raise(rc)
    return NodeStats(k, k0)
