"""Test helpers (own code, modelled on the reference's tests/helpers.py)."""
import hashlib
import os
import struct

import numpy as np


def random_multigraph(rng, max_nodes=40, max_edges=400, self_loops=True):
    """Random directed multigraph with duplicates and self-loops — the
    distribution of the reference's helpers.random_multigraph (tests/helpers.py:16)."""
    num_nodes = int(rng.integers(2, max_nodes + 1))
    num_edges = int(rng.integers(1, max_edges + 1))
    edges = rng.integers(0, num_nodes, size=(num_edges, 2))
    if not self_loops:
        loops = edges[:, 0] == edges[:, 1]
        edges[loops, 1] = (edges[loops, 1] + 1) % num_nodes
    return edges.astype(np.int64), num_nodes


def write_grpe(path, edges, num_nodes, wide=False):
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    with open(path, "wb") as fh:
        fh.write(struct.pack("<4sIIQQ", b"GRPE", 1, 1 if wide else 0, int(num_nodes), int(edges.shape[0])))
        edges.astype("<u8" if wide else "<u4").tofile(fh)
    return str(path)


def labels_sha(labels):
    return hashlib.sha256(np.asarray(labels, dtype="<i4").tobytes()).hexdigest()


def brute_force_cut(edges, labels):
    e = np.asarray(edges).reshape(-1, 2)
    lab = np.asarray(labels)
    return int((lab[e[:, 0]] != lab[e[:, 1]]).sum())
