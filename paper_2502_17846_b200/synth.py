"""Synthetic power-law graphs of the benchmark shapes (BASELINE.json configs).

The reference has no power-law generator (streamcut/synth.py:101-115; SPEC.md:542
lists it as a non-goal), so this package defines one — Chung-Lu endpoint
sampling, see csrc/grem_gen.h — whose host and device implementations produce
identical bytes.  The CPU oracle, the reference Python CPU path and the GPU path
all partition the same edges.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from ._abi import lib

# gamma -> integer beta = 1/(1 - 1/(gamma-1)) (grem_gen.h)
BETA_GAMMA_2_1 = 11
BETA_GAMMA_2_33 = 4


@dataclass(frozen=True)
class GraphShape:
    name: str
    num_nodes: int
    num_edges: int
    k: int
    beta: int = BETA_GAMMA_2_1
    seed: int = 0


# BASELINE.json "configs" / BASELINE.md §3 shapes
SHAPES = {
    "tiny": GraphShape("tiny", 10_000, 100_000, 4),
    "arxiv": GraphShape("arxiv", 169_343, 1_166_243, 8),
    "products": GraphShape("products", 2_449_029, 61_859_140, 16),
    "papers100m": GraphShape("papers100m", 111_059_956, 1_615_685_872, 16),
    "friendster": GraphShape("friendster", 65_608_366, 1_806_067_135, 16, beta=BETA_GAMMA_2_33),
}


def powerlaw_edges(num_nodes: int, num_edges: int, beta: int = BETA_GAMMA_2_1, seed: int = 0,
                   e0: int = 0, threads: int = 0) -> np.ndarray:
    """(num_edges, 2) uint32 edges [e0, e0+num_edges) of the graph (num_nodes, beta, seed)."""
    out = np.empty((num_edges, 2), dtype=np.uint32)
    rc = lib().grem_gen_edges_host(num_nodes, beta, seed, e0, num_edges, out.ctypes.data, threads)
    if rc:
        raise ValueError(f"generator failed ({rc})")
    return out


def shape_edges(shape: GraphShape | str, threads: int = 0) -> np.ndarray:
    s = SHAPES[shape] if isinstance(shape, str) else shape
    return powerlaw_edges(s.num_nodes, s.num_edges, s.beta, s.seed, threads=threads)


def write_grpe(path: str, edges: np.ndarray, num_nodes: int) -> None:
    """GRPE u32 file (edgefile.py:1-14,68-95 layout: <4sIIQQ header + pairs)."""
    import struct
    edges = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1, 2)
    with open(path, "wb") as fh:
        fh.write(struct.pack("<4sIIQQ", b"GRPE", 1, 0, int(num_nodes), int(edges.shape[0])))
        edges.tofile(fh)


def ensure_grpe(path: str, shape: GraphShape | str, threads: int = 0) -> str:
    s = SHAPES[shape] if isinstance(shape, str) else shape
    expect = 32 + 8 * s.num_edges
    if not (os.path.exists(path) and os.path.getsize(path) == expect):
        write_grpe(path, shape_edges(s, threads), s.num_nodes)
    return path
