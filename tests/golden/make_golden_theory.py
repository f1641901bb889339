"""Golden fixtures for the node-statistics path, produced by the REAL
reference (streamcut.compute_node_stats, theory.py:97-122) in the build
container.  The GPU box only reads the committed JSON.

Cases: seeded random multigraphs (the reference tests' distribution, with
self-loops and duplicates) and power-law graphs (synth.powerlaw_edges) with a
random bisection and with streamcut's own bisection; sha256 of k and k0
(int64 little-endian) and total_endpoints.

usage: python tests/golden/make_golden_theory.py
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
from streamcut import GremConfig, compute_node_stats, open_edge_file  # noqa: E402

from helpers import random_multigraph, write_grpe  # noqa: E402
from paper_2502_17846_b200 import synth  # noqa: E402


def sha(a):
    return hashlib.sha256(np.asarray(a, dtype="<i8").tobytes()).hexdigest()


def cases():
    return [("random", s, "random") for s in range(1, 7)] + [("powerlaw", 11, "random"), ("powerlaw", 12, "grem")]


def inputs(kind, seed, lab_kind, path):
    rng = np.random.default_rng(seed)
    if kind == "random":
        edges, n = random_multigraph(rng, max_nodes=60, max_edges=800)
    else:
        n, m = 3000, 40000
        edges = synth.powerlaw_edges(n, m, seed=seed).astype(np.int64)
    g = write_grpe(path, edges, n)
    if lab_kind == "random":
        labels = rng.integers(0, 2, size=n)
    else:
        labels, _ = streamcut.bisect(open_edge_file(g), GremConfig(chunk_frac=0.1))
    return edges, n, np.asarray(labels, dtype=np.int64), g


def main():
    gold = []
    with tempfile.TemporaryDirectory() as td:
        for kind, seed, lab_kind in cases():
            edges, n, labels, g = inputs(kind, seed, lab_kind, os.path.join(td, "g.grpe"))
            st = compute_node_stats(open_edge_file(g), labels)
            gold.append({"kind": kind, "seed": seed, "labels": lab_kind, "num_nodes": int(n),
                         "num_edges": int(len(edges)), "labels_sha256": sha(labels), "k_sha256": sha(st.k),
                         "k0_sha256": sha(st.k0), "total_endpoints": int(st.total_endpoints)})
    json.dump({"generator": "streamcut " + getattr(streamcut, "__version__", "?") + " (theory.py)", "cases": gold},
              open(os.path.join(HERE, "golden_theory.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
