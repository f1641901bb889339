"""Golden fixtures for the partitioned storage path, produced by the REAL
reference (streamcut.store.write_buckets / reorder_features, pure Python) in
the build container.  The GPU box only reads the committed JSON.

Cases: seeded random multigraphs (tests/helpers.random_multigraph, the
reference tests' distribution) and a power-law graph (synth.powerlaw_edges)
with seeded random labels for p in {1, 2, 3, 4, 8, 16}, 32- and 64-bit id
files; sha256 of the store file, the .idx sidecar, the regrouped feature
file and its .layout.

usage: python tests/golden/make_golden_store.py
"""
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(cand):
        sys.path.insert(0, cand)
        break

import streamcut  # noqa: E402
from streamcut import open_edge_file, reorder_features, write_buckets  # noqa: E402

from helpers import random_multigraph, write_grpe  # noqa: E402
from paper_2502_17846_b200 import synth  # noqa: E402


def sha(path):
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


def cases():
    out = []
    for seed, p, wide in [(1, 1, False), (2, 2, False), (3, 3, False), (4, 4, False), (5, 8, False),
                          (6, 16, False), (7, 4, True), (8, 8, True)]:
        out.append(("random", seed, p, wide))
    for seed, p in [(11, 4), (12, 16)]:
        out.append(("powerlaw", seed, p, False))
    return out


def inputs(kind, seed, p):
    rng = np.random.default_rng(seed)
    if kind == "random":
        edges, n = random_multigraph(rng, max_nodes=60, max_edges=800)
    else:
        n, m = 3000, 40000
        edges = synth.powerlaw_edges(n, m, seed=seed).astype(np.int64)
    labels = rng.integers(0, p, size=n)
    return edges, n, labels


def main():
    gold = []
    with tempfile.TemporaryDirectory() as td:
        for kind, seed, p, wide in cases():
            edges, n, labels = inputs(kind, seed, p)
            g = write_grpe(os.path.join(td, "g.grpe"), edges, n, wide=wide)
            ef = open_edge_file(g)
            store = os.path.join(td, "s.grpb")
            idx = write_buckets(ef, labels, store)
            rw = 5
            feats = os.path.join(td, "f.bin")
            np.random.default_rng(seed + 100).integers(0, 256, size=n * rw, dtype=np.uint8).tofile(feats)
            fout = os.path.join(td, "f.out")
            reorder_features(feats, labels, rw, fout)
            gold.append({"kind": kind, "seed": seed, "p": p, "wide": wide, "num_nodes": int(n),
                         "num_edges": int(len(edges)), "index_p": int(idx.p),
                         "store_sha256": sha(store), "idx_sha256": sha(store + ".idx"), "record_width": rw,
                         "features_out_sha256": sha(fout), "layout_sha256": sha(fout + ".layout")})
    json.dump({"generator": "streamcut " + getattr(streamcut, "__version__", "?") + " (store.py)", "cases": gold},
              open(os.path.join(HERE, "golden_store.json"), "w"), indent=1)
    print(f"{len(gold)} cases")


if __name__ == "__main__":
    main()
