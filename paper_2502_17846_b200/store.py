"""Partitioned storage layout on the GPU — drop-in for streamcut/store.py.

``write_buckets`` (store.py:55-104) scatters the edge list into p x p buckets
(bucket (i, j): source labeled i, destination labeled j; input order inside a
bucket) and ``reorder_features`` (store.py:201-235) groups fixed-width node
records by partition.  The scatter / grouping runs on the B200 behind the C
ABI (``grem_write_buckets_u32``, ``grem_reorder_records``: one label-gather
pass, one stable radix sort, extents by binary search); this module only does
the file I/O of the reference's byte layout:

  bucket file  ``<4sIIIQ`` header (GRPB, version 1, p, id-width flag,
               num_edges) + the concatenated buckets (u32 or u64 pairs, the
               input file's width), sidecar ``<store>.idx`` = p*p (offset u64,
               count u64), store.py:1-14
  layout       ``<out>.layout``: ``<4sIQI`` header (GRPF, record_width,
               num_nodes, num_parts) + u64 permutation + u64 (start, count)
               extents

``read_index`` / ``read_bucket`` are host file reads with the reference's
cross-checks.  The classes are the reference's when it is importable.
"""

from __future__ import annotations

import ctypes
import os
import struct
from dataclasses import dataclass

import numpy as np

from . import _abi
from .edgefile import FLAG_WIDE_IDS, edges_u32, is_native_binary
from .errors import FormatError
from .grem import _raise, context

BUCKET_MAGIC = b"GRPB"
FEATURE_MAGIC = b"GRPF"
_BUCKET_HEADER = struct.Struct("<4sIIIQ")
_FEATURE_HEADER = struct.Struct("<4sIQI")

try:   # the reference's result classes, so callers' isinstance checks hold
    from streamcut.store import BucketIndex, FeatureLayout  # type: ignore
except Exception:  # noqa: BLE001
    @dataclass(frozen=True)
    class BucketIndex:
        """Byte offsets and edge counts of the p x p buckets of one store file."""

        p: int
        offsets: np.ndarray
        counts: np.ndarray
        node_id_width: int

        @property
        def total_edges(self) -> int:
            return int(self.counts.sum())

        @property
        def pair_bytes(self) -> int:
            return 2 * (self.node_id_width // 8)

    @dataclass(frozen=True)
    class FeatureLayout:
        """Node -> record slot permutation grouping each partition contiguously."""

        record_width: int
        permutation: np.ndarray
        extents: tuple

        @property
        def num_nodes(self) -> int:
            return len(self.permutation)

        def slot_of(self, node: int) -> int:
            return int(self.permutation[node])

        def read_record(self, grouped_path: str, node: int) -> bytes:
            with open(grouped_path, "rb") as fh:
                fh.seek(self.slot_of(node) * self.record_width)
                return fh.read(self.record_width)

        def save(self, path: str) -> None:
            _save_layout(self, path)

        @staticmethod
        def load(path: str):
            return load_layout(path)


def _index_path(store_path: str) -> str:
    return store_path + ".idx"


def _offsets(counts: np.ndarray, pair: int) -> np.ndarray:
    starts = np.zeros(counts.size, dtype=np.int64)
    if counts.size > 1:
        np.cumsum(counts[:-1], out=starts[1:])
    return _BUCKET_HEADER.size + starts * pair


_BUCKET_PIECE_EDGES = 16 << 20   # 128 MB of u32 pairs per host piece


def write_buckets(efile, labels, out_path: str):
    """store.py:55-104 on the GPU (same file bytes as the reference)."""
    labels = np.asarray(labels)
    n = int(efile.meta.num_nodes)
    if labels.shape[0] != n:
        raise FormatError(f"labels cover {labels.shape[0]} nodes, file has {n}")
    lab = np.ascontiguousarray(labels.astype(np.int32))
    width = int(getattr(efile.meta, "node_id_width", 32))
    assigned = lab[lab >= 0]
    p_guess = int(assigned.max()) + 1 if assigned.size else 1
    counts = np.zeros(p_guess * p_guess, dtype=np.uint64)
    p_out = ctypes.c_int64()
    # the bucket-ordered edges stay on the device and are written in bounded
    # pieces (the reference streams blocks too, store.py:86-101)
    if is_native_binary(efile):   # GRPE u32: the overlapped native reader
        m = int(efile.meta.num_edges)
        rc = _abi.lib().grem_write_buckets_file(context(), os.fsencode(efile.path), lab.ctypes.data, 0,
                                                None, 0, counts.ctypes.data, counts.size, ctypes.byref(p_out))
    else:
        edges = edges_u32(efile)
        m = int(edges.shape[0])
        rc = _abi.lib().grem_write_buckets_u32(context(), edges.ctypes.data, m, n, 0, lab.ctypes.data, 0,
                                               None, 0, counts.ctypes.data, counts.size, ctypes.byref(p_out))
        del edges
    _raise(rc)
    p = int(p_out.value)
    pair = 2 * (width // 8)
    cnt = counts.astype(np.int64)
    offsets = _offsets(cnt, pair)
    piece = max(1, _BUCKET_PIECE_EDGES)
    buf = np.empty((min(piece, max(m, 1)), 2), dtype=np.uint32)
    with open(out_path, "wb") as fh:
        fh.write(_BUCKET_HEADER.pack(BUCKET_MAGIC, 1, p, FLAG_WIDE_IDS if width == 64 else 0, m))
        for lo in range(0, m, piece):
            k = min(piece, m - lo)
            _raise(_abi.lib().grem_bucket_edges(context(), buf.ctypes.data, lo, k))
            buf[:k].astype("<u8" if width == 64 else "<u4", copy=False).tofile(fh)
    side = np.empty((p * p, 2), dtype="<u8")
    side[:, 0] = offsets
    side[:, 1] = cnt
    side.tofile(_index_path(out_path))
    return BucketIndex(p, offsets.reshape(p, p), cnt.reshape(p, p), width)


def read_index(store_path: str):
    """Loads the sidecar and checks it against the store file (store.py:107-132)."""
    size = os.path.getsize(store_path)
    if size < _BUCKET_HEADER.size:
        raise FormatError(f"{store_path}: too short for a bucket header")
    with open(store_path, "rb") as fh:
        magic, version, p, flags, num_edges = _BUCKET_HEADER.unpack(fh.read(_BUCKET_HEADER.size))
    if magic != BUCKET_MAGIC:
        raise FormatError(f"{store_path}: bad magic {magic!r}")
    if version != 1:
        raise FormatError(f"{store_path}: unsupported version {version}")
    width = 64 if flags & FLAG_WIDE_IDS else 32
    pair = 2 * (width // 8)
    idx = _index_path(store_path)
    if os.path.getsize(idx) != p * p * 16:
        raise FormatError(f"{idx}: index size does not match p={p}")
    side = np.fromfile(idx, dtype="<u8").reshape(p * p, 2).astype(np.int64)
    offsets, counts = side[:, 0], side[:, 1]
    if (int(counts.sum()) != num_edges or not np.array_equal(offsets, _offsets(counts, pair))
            or size != _BUCKET_HEADER.size + num_edges * pair):
        raise FormatError(f"{store_path}: index/file mismatch")
    return BucketIndex(p, offsets.reshape(p, p), counts.reshape(p, p), width)


def read_bucket(store_path: str, i: int, j: int, index=None) -> np.ndarray:
    """Bucket (i, j) as an (m, 2) int64 array, one contiguous read (store.py:135-148)."""
    if index is None:
        index = read_index(store_path)
    if not (0 <= i < index.p and 0 <= j < index.p):
        raise FormatError(f"bucket ({i}, {j}) out of range for p={index.p}")
    count = int(index.counts[i, j])
    dtype = np.dtype("<u4") if index.node_id_width == 32 else np.dtype("<u8")
    with open(store_path, "rb") as fh:
        fh.seek(int(index.offsets[i, j]))
        raw = np.fromfile(fh, dtype=dtype, count=2 * count)
    if raw.size != 2 * count:
        raise FormatError(f"{store_path}: index/file mismatch reading bucket ({i}, {j})")
    return raw.astype(np.int64).reshape(-1, 2)


def _save_layout(layout, path: str) -> None:
    with open(path, "wb") as fh:
        fh.write(_FEATURE_HEADER.pack(FEATURE_MAGIC, layout.record_width, len(layout.permutation),
                                      len(layout.extents)))
        np.asarray(layout.permutation, dtype="<u8").tofile(fh)
        np.asarray(layout.extents, dtype="<u8").reshape(-1, 2).tofile(fh)


def load_layout(path: str):
    with open(path, "rb") as fh:
        head = fh.read(_FEATURE_HEADER.size)
        if len(head) < _FEATURE_HEADER.size:
            raise FormatError(f"{path}: too short for a layout header")
        magic, record_width, num_nodes, num_parts = _FEATURE_HEADER.unpack(head)
        if magic != FEATURE_MAGIC:
            raise FormatError(f"{path}: bad magic {magic!r}")
        perm = np.fromfile(fh, dtype="<u8", count=num_nodes).astype(np.int64)
        ext = np.fromfile(fh, dtype="<u8", count=2 * num_parts).astype(np.int64)
    if perm.size != num_nodes or ext.size != 2 * num_parts:
        raise FormatError(f"{path}: truncated layout")
    return FeatureLayout(record_width, perm, tuple((int(s), int(c)) for s, c in ext.reshape(num_parts, 2)))


_REORDER_DEVICE_MAX_BYTES = int(os.environ.get("GREM_REORDER_DEVICE_MAX", str(1 << 30)))
_REORDER_BLOCK_BYTES = 16 << 20   # store.py:226-231 streams 16 MB blocks


def reorder_features(features_path: str, labels, record_width: int, out_path: str):
    """store.py:201-235 on the GPU: records regrouped by partition (ascending
    node id inside one), layout saved as ``<out>.layout``."""
    labels = np.asarray(labels)
    n = int(labels.shape[0])
    if record_width < 1:
        raise FormatError("record_width must be >= 1")
    if n and int(labels.min()) < 0:
        raise FormatError("all nodes must be labeled")
    size = os.path.getsize(features_path)
    if size != n * record_width:
        raise FormatError(f"{features_path}: length {size} != num_nodes {n} x width {record_width}")
    lab = np.ascontiguousarray(labels.astype(np.int32))
    p_guess = int(lab.max()) + 1 if n else 1
    # small stores: records gathered on the device in one go; large ones
    # (e.g. papers100M x 128 fp32 = 57 GB): only the permutation on the
    # device, records streamed through bounded blocks of a memmap like the
    # reference (store.py:226-231), so neither host RAM nor HBM holds a copy
    streamed = size > _REORDER_DEVICE_MAX_BYTES
    records = None if streamed else np.fromfile(features_path, dtype=np.uint8)
    out = None if streamed else np.empty_like(records)
    perm = np.empty(max(n, 1), dtype=np.int64)
    counts = np.zeros(max(p_guess, 1), dtype=np.uint64)
    p_out = ctypes.c_int64()
    if n:
        rc = _abi.lib().grem_reorder_records(context(), lab.ctypes.data, n, 0,
                                             None if streamed else records.ctypes.data, record_width,
                                             None if streamed else out.ctypes.data, perm.ctypes.data,
                                             counts.ctypes.data, counts.size, ctypes.byref(p_out))
        _raise(rc)
        p = int(p_out.value)
    else:
        p = 1
    cnt = counts[:p].astype(np.int64)
    starts = np.zeros(p, dtype=np.int64)
    if p > 1:
        np.cumsum(cnt[:-1], out=starts[1:])
    extents = tuple((int(s), int(c)) for s, c in zip(starts, cnt))
    if streamed:
        order = np.empty(n, dtype=np.int64)          # slot -> node (perm: node -> slot)
        order[perm[:n]] = np.arange(n, dtype=np.int64)
        src = np.memmap(features_path, dtype=np.uint8, mode="r", shape=(n, record_width))
        per = max(1, _REORDER_BLOCK_BYTES // record_width)
        with open(out_path, "wb") as fh:
            for lo in range(0, n, per):
                fh.write(np.ascontiguousarray(src[order[lo:lo + per]]).tobytes())
        del src
    else:
        out.tofile(out_path)
    layout = FeatureLayout(record_width, perm[:n].copy(), extents)
    _save_layout(layout, out_path + ".layout")
    return layout


__all__ = ["BucketIndex", "FeatureLayout", "write_buckets", "read_index", "read_bucket", "reorder_features",
           "load_layout"]
