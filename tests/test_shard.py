"""Multi-GPU subtree sharding (paper_2502_17846_b200/shard.py).

CPU: the ownership rule and the label merge over a world_size-2 gloo group,
on labels the oracle computes.  GPU: every rank's share computed through the
C ABI (grem_partition_shard_u32) and merged equals partition() bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import random_multigraph
from oracle import oracle
from paper_2502_17846_b200 import GremConfig, grem, synth
from paper_2502_17846_b200.shard import owned_leaves, owner_split


def test_owner_split_rule():
    assert owner_split(0, 1, 10, 10) == ((0, 1), (0, 1))
    assert owner_split(0, 2, 10, 10) == ((0, 1), (1, 2))
    assert owner_split(0, 2, 1000, 0) == ((0, 1), (1, 2))      # never starve a side
    assert owner_split(0, 4, 98, 2) == ((0, 3), (3, 4))
    assert owner_split(2, 8, 1, 1) == ((2, 5), (5, 8))
    for w in range(2, 9):
        for m0, m1 in [(0, 0), (1, 5), (7, 3), (10**9, 1)]:
            (a0, a1), (b0, b1) = owner_split(0, w, m0, m1)
            assert a0 == 0 and a1 == b0 and b1 == w and a1 - a0 >= 1 and b1 - b0 >= 1


def _case():
    rng = np.random.default_rng(5)
    edges, n = random_multigraph(rng, max_nodes=300, max_edges=3000)
    lab = oracle.partition(edges, n, 8, chunk_frac=0.2)
    return edges, n, lab


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_owned_leaves_cover_every_leaf(world):
    edges, n, lab = _case()
    cover = [owned_leaves(edges, lab, 8, r, world) for r in range(world)]
    assert set().union(*cover) == set(range(8))
    if world >= 8:
        assert all(len(c) >= 1 for c in cover)


def _merge_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    edges, n, lab = _case()
    mine = owned_leaves(edges, lab, 8, rank, world)
    part = torch.from_numpy(np.where(np.isin(lab, sorted(mine)), lab, -1).astype(np.int32))
    dist.all_reduce(part, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put(bool(np.array_equal(part.numpy(), lab)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_merge_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_merge_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok


def _shards(e32, n, p, cfg, world):
    from paper_2502_17846_b200.shard import partition_shard
    dev = torch.from_numpy(e32).cuda()
    parts = []
    for r in range(world):
        out = np.empty(n, dtype=np.int32)
        partition_shard(dev.data_ptr(), e32.shape[0], n, p, cfg, r, world, out)
        parts.append(out)
    return parts


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_gpu_shards_merge_to_partition(world):
    rng = np.random.default_rng(11 + world)
    for trial in range(6):
        edges, n = random_multigraph(rng, max_nodes=2000, max_edges=20000)
        e32 = edges.astype(np.uint32)
        p = int(2 ** rng.integers(1, 5))
        cfg = GremConfig(chunk_frac=float(rng.choice([0.05, 0.1, 0.3])))
        full, _ = grem.partition_edges(e32, n, p, cfg)
        parts = _shards(e32, n, p, cfg, world)
        assert np.array_equal(np.maximum.reduce(parts), full)
        for r, part in enumerate(parts):
            mine = owned_leaves(e32, full, p, r, world)
            assert np.array_equal(part >= 0, np.isin(full, sorted(mine))), (trial, r)


@pytest.mark.gpu
def test_gpu_shards_arxiv_k8():
    s = synth.SHAPES["arxiv"]
    e32 = np.ascontiguousarray(synth.shape_edges(s).astype(np.uint32))
    cfg = GremConfig(chunk_frac=0.1)
    full, rep = grem.partition_edges(e32, s.num_nodes, 8, cfg)
    for world in (2, 4, 8):
        parts = _shards(e32, s.num_nodes, 8, cfg, world)
        assert np.array_equal(np.maximum.reduce(parts), full), world


def _gather_worker(rank, world, port, m, q):
    """the upload-slice + in-place all-gather of partition_distributed's host
    path, on CPU tensors over gloo"""
    import os
    import torch
    import torch.distributed as dist
    from paper_2502_17846_b200.shard import upload_slice
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    host = torch.arange(2 * m, dtype=torch.int32).reshape(m, 2)
    per, lo, hi = upload_slice(m, rank, world)
    buf = torch.full((per * world, 2), -7, dtype=torch.int32)
    buf[lo:hi] = host[lo:hi]
    dist.all_gather_into_tensor(buf, buf[rank * per:(rank + 1) * per].clone())
    q.put((rank, bool(torch.equal(buf[:m], host))))
    dist.destroy_process_group()


@pytest.mark.parametrize("m", [1, 7, 1000])
def test_gloo_upload_slices_reassemble_the_edge_list(m):
    import multiprocessing as mp
    world = 2 if m == 1 else 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29650 + m % 97
    ps = [ctx.Process(target=_gather_worker, args=(r, world, port, m, q)) for r in range(world)]
    for p_ in ps:
        p_.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p_ in ps:
        p_.join(timeout=60)
    assert all(ok for _, ok in res), res
