"""Partitioned storage: write_buckets / read_index /
read_bucket / reorder_features (streamcut/store.py) on the GPU, byte-for-byte
against fixtures made by the real reference (tests/golden/golden_store.json)
and against the numpy restatement (oracle/store_oracle.py) on seeded cases;
error behaviour follows store.py and the reference's tests/test_store.py."""
import hashlib
import json
import os
import struct

import numpy as np
import pytest

from helpers import random_multigraph, write_grpe
from oracle import store_oracle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_store.json")


def _sha(b):
    return hashlib.sha256(b).hexdigest()


def _inputs(case):
    from paper_2502_17846_b200 import synth
    rng = np.random.default_rng(case["seed"])
    if case["kind"] == "random":
        edges, n = random_multigraph(rng, max_nodes=60, max_edges=800)
    else:
        n, m = 3000, 40000
        edges = synth.powerlaw_edges(n, m, seed=case["seed"]).astype(np.int64)
    labels = rng.integers(0, case["p"], size=n)
    feats = np.random.default_rng(case["seed"] + 100).integers(0, 256, size=n * case["record_width"],
                                                                dtype=np.uint8)
    return edges, n, labels, feats


def _layout_bytes(rw, perm, extents):
    return (struct.pack("<4sIQI", b"GRPF", rw, len(perm), len(extents)) + np.asarray(perm, "<u8").tobytes()
            + np.asarray(extents, "<u8").reshape(-1, 2).tobytes())


CASES = json.load(open(GOLD))["cases"]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['kind']}-{c['seed']}-p{c['p']}{'-wide' if c['wide'] else ''}")
def test_oracle_matches_reference_golden(case):
    """The restatement reproduces the reference's files (pins the oracle)."""
    edges, n, labels, feats = _inputs(case)
    store, side = store_oracle.bucket_file_bytes(edges, labels, 64 if case["wide"] else 32)
    assert _sha(store) == case["store_sha256"]
    assert _sha(side) == case["idx_sha256"]
    order, perm, ext = store_oracle.grouping(labels)
    rw = case["record_width"]
    assert _sha(feats.reshape(n, rw)[order].tobytes()) == case["features_out_sha256"]
    assert _sha(_layout_bytes(rw, perm, ext)) == case["layout_sha256"]


# ------------------------------------------------------------------- GPU
def _ef(tmp_path, edges, n, wide=False):
    from paper_2502_17846_b200.edgefile import open_edge_file
    return open_edge_file(write_grpe(tmp_path / "g.grpe", edges, n, wide=wide))


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['kind']}-{c['seed']}-p{c['p']}{'-wide' if c['wide'] else ''}")
def test_gpu_store_equals_reference_golden(tmp_path, case):
    from paper_2502_17846_b200 import store
    edges, n, labels, feats = _inputs(case)
    path = str(tmp_path / "s.grpb")
    idx = store.write_buckets(_ef(tmp_path, edges, n, case["wide"]), labels, path)
    assert idx.p == case["index_p"] and idx.total_edges == case["num_edges"]
    assert _sha(open(path, "rb").read()) == case["store_sha256"]
    assert _sha(open(path + ".idx", "rb").read()) == case["idx_sha256"]
    fin, fout = tmp_path / "f.bin", str(tmp_path / "f.out")
    feats.tofile(fin)
    lay = store.reorder_features(str(fin), labels, case["record_width"], fout)
    assert _sha(open(fout, "rb").read()) == case["features_out_sha256"]
    assert _sha(open(fout + ".layout", "rb").read()) == case["layout_sha256"]
    assert lay.num_nodes == n
    # the streamed form (device permutation + bounded memmap blocks, used for
    # stores above GREM_REORDER_DEVICE_MAX) writes the same bytes
    import paper_2502_17846_b200.store as st
    old = st._REORDER_DEVICE_MAX_BYTES, st._REORDER_BLOCK_BYTES
    st._REORDER_DEVICE_MAX_BYTES, st._REORDER_BLOCK_BYTES = 0, 3 * case["record_width"]
    try:
        lay2 = store.reorder_features(str(fin), labels, case["record_width"], fout + "2")
    finally:
        st._REORDER_DEVICE_MAX_BYTES, st._REORDER_BLOCK_BYTES = old
    assert _sha(open(fout + "2", "rb").read()) == case["features_out_sha256"]
    assert _sha(open(fout + "2.layout", "rb").read()) == case["layout_sha256"]
    assert lay2.num_nodes == n


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 2, 5, 16, 64])
def test_gpu_buckets_vs_oracle_powerlaw(tmp_path, p):
    from paper_2502_17846_b200 import store, synth
    n, m = 200_000, 2_000_000
    edges = synth.powerlaw_edges(n, m, seed=p).astype(np.int64)
    labels = np.random.default_rng(p).integers(0, p, size=n)
    path = str(tmp_path / "s.grpb")
    idx = store.write_buckets(_ef(tmp_path, edges, n), labels, path)
    want, want_side = store_oracle.bucket_file_bytes(edges, labels)
    assert open(path, "rb").read() == want and open(path + ".idx", "rb").read() == want_side
    rel = store.read_index(path)
    assert np.array_equal(rel.counts, idx.counts) and rel.p == idx.p
    i, j = (p - 1, 0) if p > 1 else (0, 0)
    got = store.read_bucket(path, i, j, rel)
    assert (labels[got[:, 0]] == i).all() and (labels[got[:, 1]] == j).all()


@pytest.mark.gpu
def test_gpu_bucket_order_is_input_order_and_errors(tmp_path):
    from paper_2502_17846_b200 import store
    from paper_2502_17846_b200.errors import FormatError
    edges = [[1, 0], [0, 1], [1, 1]]
    path = str(tmp_path / "s.grpb")
    idx = store.write_buckets(_ef(tmp_path, edges, 2), np.array([1, 1]), path)
    assert store.read_bucket(path, 1, 1, idx).tolist() == edges and idx.p == 2
    with pytest.raises(FormatError):   # unlabeled endpoint (store.py:77-78)
        store.write_buckets(_ef(tmp_path, [[0, 1]], 2), np.array([0, -1]), path)
    with pytest.raises(FormatError):   # labels length
        store.write_buckets(_ef(tmp_path, [[0, 1]], 2), np.array([0, 1, 1]), path)
    # unlabeled nodes that are no endpoint are fine; p from assigned labels only
    idx = store.write_buckets(_ef(tmp_path, [[0, 1]], 3), np.array([0, 1, -1]), path)
    assert idx.p == 2 and idx.total_edges == 1
    # empty edge list
    idx = store.write_buckets(_ef(tmp_path, np.zeros((0, 2), np.int64), 4), np.array([0, 1, 2, 0]), path)
    assert idx.p == 3 and idx.total_edges == 0 and os.path.getsize(path) == 24
    # sidecar corruption is detected (tests/test_store.py:86-97 of the reference)
    store.write_buckets(_ef(tmp_path, [[0, 1], [1, 0]], 2), np.array([0, 1]), path)
    raw = np.fromfile(path + ".idx", dtype="<u8")
    raw[-1] += 1
    raw.tofile(path + ".idx")
    with pytest.raises(FormatError):
        store.read_index(path)
    # reorder: unlabeled node / length mismatch
    f = tmp_path / "f.bin"
    np.zeros(6, np.uint8).tofile(f)
    with pytest.raises(FormatError):
        store.reorder_features(str(f), np.array([0, -1, 1]), 2, str(tmp_path / "o"))
    with pytest.raises(FormatError):
        store.reorder_features(str(f), np.array([0, 1]), 2, str(tmp_path / "o"))
