"""Multi-GPU partition: recursion subtrees sharded across ranks.

One process per GPU (torch.distributed, NCCL).  Every rank holds the level's
edges in its own HBM and calls ``grem_partition_shard_u32``: the owners of a
recursion node (all ranks at the root) are split between its two sides in
proportion to the sides' edge counts, so from level ⌈log2 W⌉ on the bisections
run on disjoint GPUs with no exchange at all.  Ancestors owned by several
ranks are computed redundantly — the path is deterministic, so the copies are
bit-identical.  Each rank ends with its own leaves' labels (-1 elsewhere) in
a device tensor; ONE all-reduce(MAX) over NCCL merges them and count_cuts
(grem.py:227-252) runs on the merged labels.

The reference runs partition() (grem.py:277-319) in one process; the merged
labels equal its labels bit for bit (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from .grem import _cfg_struct, _raise, _report, _report_struct, context


def owner_split(r0: int, r1: int, m0: int, m1: int) -> tuple[tuple[int, int], tuple[int, int]]:
    """Rank ranges of the two sides of a recursion node owned by [r0, r1).

    Mirrors recurse() in csrc/grem_runtime.cu: a single owner keeps both
    sides; otherwise side 0 gets round(W·(m0+1)/(m0+m1+2)) ranks, clamped to
    [1, W-1].  A last-level bisection (two leaves) is not split: each of its
    owners writes both leaves.
    """
    w = r1 - r0
    if w < 2:
        return (r0, r1), (r0, r1)
    w0 = int(np.floor(w * (m0 + 1.0) / (m0 + m1 + 2.0) + 0.5))
    w0 = min(max(w0, 1), w - 1)
    return (r0, r0 + w0), (r0 + w0, r1)


def owned_leaves(edges, labels, p: int, rank: int, world: int) -> set:
    """Leaves (final part ids) whose bisection chain includes ``rank``, given a
    finished partition: host-side mirror of the ownership rule, used to check
    the merge logic without a GPU.  A side's edge count is the number of edges
    with both endpoints inside the side's leaf range (the induced subgraph
    grem.py:255-274 extracts)."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    lab = np.asarray(labels, dtype=np.int64)
    lu, lv = lab[e[:, 0]], lab[e[:, 1]]
    out: set = set()

    def side_edges(lo, hi):
        return int(((lu >= lo) & (lu < hi) & (lv >= lo) & (lv < hi)).sum())

    def rec(base, pl, r0, r1):
        if not (r0 <= rank < r1):
            return
        if pl <= 2:                     # the last bisection writes both its leaves
            out.update(range(base, base + pl))
            return
        h = pl // 2
        (a0, a1), (b0, b1) = owner_split(r0, r1, side_edges(base, base + h), side_edges(base + h, base + pl))
        rec(base, h, a0, a1)
        rec(base + h, h, b0, b1)

    rec(0, int(p), 0, int(world))
    return out


def partition_shard(edges_ptr: int, num_edges: int, num_nodes: int, p: int, config, rank: int, world: int,
                    labels_out, edges_on_device: bool = True) -> None:
    """This rank's share of partition(): labels_out (int32 device tensor or
    numpy array, num_nodes entries) receives the leaves this rank owns and -1
    elsewhere.  ``edges_ptr`` is a device pointer on the context's GPU."""
    import torch

    cfg = _cfg_struct(config, None)
    if isinstance(labels_out, torch.Tensor):
        assert labels_out.dtype == torch.int32 and labels_out.numel() == num_nodes and labels_out.is_contiguous()
        out = labels_out.data_ptr()
    else:
        assert labels_out.dtype == np.int32 and labels_out.shape[0] == num_nodes
        out = labels_out.ctypes.data
    rc = _abi.lib().grem_partition_shard_u32(context(), int(edges_ptr), int(num_edges), int(num_nodes),
                                             1 if edges_on_device else 0, int(p),
                                             ctypes.byref(cfg), int(rank), int(world), out)
    _raise(rc)


def merge_labels(labels, group=None):
    """Element-wise max over ranks: every node is owned by exactly one leaf
    and hence one rank; the others hold -1."""
    import torch.distributed as dist

    dist.all_reduce(labels, op=dist.ReduceOp.MAX, group=group)
    return labels


def count_cuts_device(edges_ptr: int, num_edges: int, num_nodes: int, labels, p: int):
    """count_cuts (grem.py:227-252) on device-resident edges and labels."""
    rep, sizes = _report_struct(max(2, int(p)))
    rc = _abi.lib().grem_count_cuts_u32(context(), int(edges_ptr), int(num_edges), int(num_nodes), 1,
                                        labels.data_ptr(), 1, ctypes.byref(rep))
    _raise(rc)
    return _report(int(num_nodes), rep, sizes)


def upload_slice(m: int, rank: int, world: int) -> tuple[int, int, int]:
    """(slot size, lo, hi): the edges [lo, hi) rank uploads into its slot of an
    all-gather buffer of world * slot rows (equal slots; the last is padded)."""
    per = -(-int(m) // int(world))
    return per, min(rank * per, m), min((rank + 1) * per, m)


def partition_distributed(edges_ptr: int, num_edges: int, num_nodes: int, p: int, config, group=None,
                          edges_on_device: bool = True):
    """partition() over all ranks of ``group``: returns (labels device tensor,
    CutReport), identical on every rank.  With ``edges_on_device=False`` the
    pointer is a (page-locked) host edge list.  Up to 3 ranks, each uploads
    it with the overlapped ingest of its level-0 bisection (count_cuts reuses
    that copy); from 4 ranks on, W full uploads contend for the host, so each
    rank uploads only its 1/W slice and an in-place NCCL all-gather over
    NVLink assembles the list on every GPU (papers100M k=16 e2e at 4 GPUs
    831 -> 717 ms; at 2 GPUs the overlapped full upload is faster, 771 vs
    828 ms)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    from .grem import _current_device
    dev = _current_device()     # the native context's device (GREM_DEVICE / LOCAL_RANK), not torch's current one
    if not edges_on_device and world >= 4 and num_edges > 0:
        m = int(num_edges)
        per, lo, hi = upload_slice(m, rank, world)
        buf = torch.empty((per * world, 2), dtype=torch.int32, device=f"cuda:{dev}")
        if hi > lo:
            _raise(_abi.lib().grem_memcpy_h2d(context(), ctypes.c_void_p(buf[lo:hi].data_ptr()),
                                              ctypes.c_void_p(int(edges_ptr) + lo * 8), (hi - lo) * 8))
        with torch.cuda.device(buf.device):
            dist.all_gather_into_tensor(buf, buf[rank * per:(rank + 1) * per], group=group)
            torch.cuda.synchronize(buf.device)     # NCCL stream -> library stream
        labels, rep = partition_distributed(buf.data_ptr(), m, num_nodes, p, config, group, True)
        del buf
        return labels, rep
    labels = torch.empty(int(num_nodes), dtype=torch.int32, device=f"cuda:{dev}")
    partition_shard(edges_ptr, num_edges, num_nodes, p, config, rank, world, labels, edges_on_device)
    dev_ptr = int(edges_ptr)
    if not edges_on_device:
        staged, cnt = ctypes.c_void_p(), ctypes.c_int64()
        _raise(_abi.lib().grem_staged_edges(context(), ctypes.byref(staged), ctypes.byref(cnt)))
        dev_ptr = int(staged.value or 0)
    if world > 1:
        merge_labels(labels, group)
        torch.cuda.synchronize(labels.device)      # NCCL stream -> library stream
    return labels, count_cuts_device(dev_ptr, num_edges, num_nodes, labels, p)


__all__ = ["owner_split", "owned_leaves", "partition_shard", "merge_labels", "count_cuts_device",
           "upload_slice", "partition_distributed"]
