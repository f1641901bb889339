"""Node statistics of the analytical cut model on the GPU — drop-in for
streamcut.theory.compute_node_stats (theory.py:97-122).

``compute_node_stats(efile, labels)`` is one pass over the edge list: per
node, ``k`` = neighbour endpoints excluding self-loops (duplicates count with
multiplicity) and ``k0`` = those on the node's majority side of the bisection
``labels``.  It runs behind the C ABI (``grem_node_stats_u32``: two label
gathers and two 64-bit REDs per edge, then k = c0 + c1, k0 = max) and returns
the reference's ``NodeStats`` when it is importable.  The curve math on top
(``expected_cuts``, ``theory_curve``: per-(k, k0) hypergeometric tails summed
in node order) is host arithmetic over the returned arrays and stays the
reference's.
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
