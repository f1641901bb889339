"""Edge-file front end of the drop-in (streamcut/edgefile.py formats).

GRPE binary u32 files go straight to the native ingest (pinned, double
buffered file -> HBM, grem_bisect_file).  Text files and 64-bit-id binary files
are parsed here into a u32 edge array (the GPU path supports < 2^31 nodes), with
the reference's validation and error messages (edgefile.py:107-219).
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass

import numpy as np

from .errors import FormatError

EDGE_MAGIC = b"GRPE"
FLAG_WIDE_IDS = 1
TEXT = "text"
BINARY = "binary"
_EDGE_HEADER = struct.Struct("<4sIIQQ")


@dataclass(frozen=True)
class GraphMeta:
    num_nodes: int
    num_edges: int
    node_id_width: int = 32


@dataclass(frozen=True)
class EdgeFile:
    path: str
    meta: GraphMeta
    format: str


def _read_binary_header(path: str) -> GraphMeta:
    size = os.path.getsize(path)
    if size < _EDGE_HEADER.size:
        raise FormatError(f"{path}: too short for a binary edge header")
    with open(path, "rb") as fh:
        magic, version, flags, num_nodes, num_edges = _EDGE_HEADER.unpack(fh.read(_EDGE_HEADER.size))
    if magic != EDGE_MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}")
    if version != 1:
        raise FormatError(f"{path}: unsupported version {version}")
    width = 64 if flags & FLAG_WIDE_IDS else 32
    expected = _EDGE_HEADER.size + num_edges * 2 * (width // 8)
    if size != expected:
        raise FormatError(f"{path}: payload length {size - _EDGE_HEADER.size} does not match "
                          f"header num_edges {num_edges}")
    return GraphMeta(num_nodes, num_edges, width)


def open_edge_file(path: str, num_nodes: int | None = None) -> EdgeFile:
    """Binary GRPE only here; text files are accepted through streamcut's own
    EdgeFile objects (their meta is trusted) or parsed by edges_u32()."""
    with open(path, "rb") as fh:
        head = fh.read(4)
    if head != EDGE_MAGIC:
        n_edges, max_id = 0, -1
        for u, v in _iter_text(path):
            n_edges += 1
            max_id = max(max_id, u, v)
        if num_nodes is None:
            num_nodes = max_id + 1 if max_id >= 0 else 1
        elif max_id >= num_nodes:
            raise FormatError(f"{path}: edge endpoint {max_id} >= num_nodes {num_nodes}")
        return EdgeFile(path, GraphMeta(max(num_nodes, 1), n_edges, 32), TEXT)
    meta = _read_binary_header(path)
    if num_nodes is not None and num_nodes != meta.num_nodes:
        raise FormatError(f"{path}: num_nodes {meta.num_nodes} in header != requested {num_nodes}")
    return EdgeFile(path, meta, BINARY)


def _iter_text(path: str):
    with open(path, "r", encoding="ascii") as fh:
        for lineno, line in enumerate(fh, 1):
            stripped = line.strip()
            if not stripped or stripped.startswith("#"):
                continue
            parts = stripped.split()
            if len(parts) != 2:
                raise FormatError(f"{path}:{lineno}: expected 'src dst', got {line.rstrip()!r}")
            try:
                u, v = int(parts[0]), int(parts[1])
            except ValueError:
                raise FormatError(f"{path}:{lineno}: non-integer node id in {line.rstrip()!r}") from None
            if u < 0 or v < 0:
                raise FormatError(f"{path}:{lineno}: negative node id")
            yield u, v


def is_native_binary(efile) -> bool:
    """True when the native ingest can read the file directly (GRPE, u32 ids)."""
    fmt = getattr(efile, "format", BINARY)
    return fmt == BINARY and getattr(efile.meta, "node_id_width", 32) == 32


def edges_u32(efile) -> np.ndarray:
    """All edges of the file, in order, as a contiguous (m, 2) uint32 array."""
    n = int(efile.meta.num_nodes)
    if n >= 2**31:
        raise FormatError("num_nodes >= 2^31 is not supported by the GPU path")
    if getattr(efile, "format", BINARY) == BINARY:
        meta = _read_binary_header(efile.path)
        dtype = np.dtype("<u4") if meta.node_id_width == 32 else np.dtype("<u8")
        raw = np.fromfile(efile.path, dtype=dtype, offset=_EDGE_HEADER.size, count=2 * meta.num_edges)
        if raw.size != 2 * meta.num_edges:
            raise FormatError(f"{efile.path}: truncated payload")
        if raw.size and int(raw.max()) >= meta.num_nodes:
            raise FormatError(f"{efile.path}: edge endpoint {int(raw.max())} >= num_nodes {meta.num_nodes}")
        return np.ascontiguousarray(raw.astype(np.uint32, copy=False).reshape(-1, 2))
    pairs = list(_iter_text(efile.path))
    arr = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if arr.size and int(arr.max()) >= n:
        raise FormatError(f"{efile.path}: edge endpoint {int(arr.max())} >= num_nodes {n}")
    return np.ascontiguousarray(arr.astype(np.uint32))
