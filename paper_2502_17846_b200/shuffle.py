"""External shuffle on the GPU — drop-in for streamcut.edgefile.external_shuffle
(edgefile.py:248-327): a uniform random permutation of an edge file, the
"edges in random order" precondition of the streaming partitioner.

The reference draws from numpy's PCG64 Generator in a budgeted two-pass
scatter/gather; here the whole edge list is permuted in HBM behind the C ABI
(``grem_shuffle_file`` / ``grem_shuffle_u32``: a 64-bit counter-hash key per
edge position, one radix sort of (key, edge) pairs), so the output order is
not the reference's — parity is what the reference's own tests pin
(tests/test_edgefile.py:87-135): same multiset, byte-identical output for a
fixed seed, positions uniform over seeds, and the same budget errors.  The
host side holds at most one 128 MB pinned piece of the payload at a time.
"""

from __future__ import annotations

import ctypes
import os
import struct
from math import ceil

import numpy as np

from . import _abi
from .edgefile import FLAG_WIDE_IDS, edges_u32, is_native_binary, open_edge_file
from .errors import FormatError
from .grem import _raise, context

IO_BLOCK = 64 * 1024            # edgefile.py:41
_MAX_SCATTER_BUCKETS = 4096     # edgefile.py:42


def _check_budget(num_edges: int, memory_budget: int) -> None:
    """The reference's budget errors (edgefile.py:262-263, 271-275)."""
    if memory_budget < IO_BLOCK:
        raise FormatError(f"memory_budget must be at least one I/O block ({IO_BLOCK} bytes)")
    total = num_edges * 16
    if total > memory_budget:
        nbuckets = ceil(total / max(16, memory_budget // 2))
        if nbuckets > _MAX_SCATTER_BUCKETS:
            raise FormatError(f"memory budget too small: shuffle would need {nbuckets} scatter buckets")


def external_shuffle(efile, out_path: str, memory_budget: int, rng_seed: int):
    """edgefile.py:248-327 (signature and errors); returns the shuffled EdgeFile."""
    meta = efile.meta
    _check_budget(int(meta.num_edges), int(memory_budget))
    seed = int(rng_seed) & 0xFFFFFFFFFFFFFFFF
    L = _abi.lib()
    if is_native_binary(efile):
        _raise(L.grem_shuffle_file(context(), os.fsencode(efile.path), seed, os.fsencode(out_path)))
        return open_edge_file(out_path)
    e = edges_u32(efile)
    m = int(e.shape[0])
    out = np.empty((m, 2), dtype=np.uint32)
    _raise(L.grem_shuffle_u32(context(), e.ctypes.data, m, int(meta.num_nodes), 0, seed, out.ctypes.data, 0))
    width = int(getattr(meta, "node_id_width", 32))
    with open(out_path, "wb") as fh:
        fh.write(struct.pack("<4sIIQQ", b"GRPE", 1, FLAG_WIDE_IDS if width == 64 else 0, int(meta.num_nodes), m))
        out.astype("<u8" if width == 64 else "<u4", copy=False).tofile(fh)
    return open_edge_file(out_path)
