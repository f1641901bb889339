"""Generate the golden fixtures from the REAL reference (streamcut, pure
Python) — run in the build container, where /root/reference (or its install
under baseline/_ref) exists.  The GPU box never runs this; it only reads the
committed outputs:

  golden_random.npz   40 random multigraphs in the distribution of the
                      reference's own tests (tests/helpers.py:16), with
                      streamcut.bisect / partition labels and reports
  golden_shapes.json  tiny (10K/100K, k=4) and arxiv-shaped (169K/1.17M, k=8)
                      streamcut.partition reports + labels sha256
  golden_tiny_k4.npy  full streamcut labels of the tiny shape

usage: python tests/golden/make_golden.py [--products]   (products k=16 takes ~20 min)
"""
import hashlib
import json
import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(cand):
        sys.path.insert(0, cand)
        break

import streamcut  # noqa: E402
from streamcut import BinaryEdgeWriter, GremConfig, SeedConfig, open_edge_file  # noqa: E402

from paper_2502_17846_b200 import synth  # noqa: E402


def make_file(path, edges, n):
    with BinaryEdgeWriter(path, n) as w:
        w.write(np.asarray(edges, dtype=np.int64).reshape(-1, 2))
    return open_edge_file(path)


def sha(labels):
    return hashlib.sha256(np.asarray(labels, dtype="<i4").tobytes()).hexdigest()


def random_cases(tmp):
    rng = np.random.default_rng(20261018)
    out = {}
    for t in range(40):
        n = int(rng.integers(2, 61))
        m = int(rng.integers(1, 1001))
        edges = rng.integers(0, n, size=(m, 2)).astype(np.int64)
        ef = make_file(os.path.join(tmp, f"r{t}.grpe"), edges, n)
        ce = int(rng.integers(1, m + 1))
        refine = bool(rng.integers(0, 2)) or t < 20
        passes = int(rng.integers(1, 3))
        slack = float(rng.choice([0.0, 0.1, 0.25]))
        algo = "random" if t % 10 == 9 else "bfs_grow"
        rp = int(rng.integers(0, 4))
        cfg = GremConfig(chunk_edges=ce, refine=refine, passes=passes, capacity_slack=slack,
                         seed=SeedConfig(algorithm=algo, refinement_passes=rp, rng_seed=t))
        lab, rep = streamcut.bisect(ef, cfg)
        p = int(rng.choice([2, 4, 8]))
        frac = float(rng.choice([0.05, 0.1, 0.3, 1.0]))
        cfg2 = GremConfig(chunk_frac=frac, refine=refine, passes=passes, capacity_slack=slack,
                          seed=SeedConfig(algorithm=algo, refinement_passes=rp, rng_seed=t))
        lab2, rep2 = streamcut.partition(ef, p, cfg2, os.path.join(tmp, "w"))
        out[f"c{t}_edges"] = edges.astype(np.uint32)
        out[f"c{t}_params"] = np.array([n, ce, int(refine), passes, p, rp, t, 1 if algo == "random" else 0],
                                       dtype=np.int64)
        out[f"c{t}_floats"] = np.array([slack, frac], dtype=np.float64)
        out[f"c{t}_bisect"] = lab.astype(np.int32)
        out[f"c{t}_partition"] = lab2.astype(np.int32)
        out[f"c{t}_rep"] = np.array([rep.cut_edges, rep2.cut_edges], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "golden_random.npz"), **out)


def shape_case(tmp, name, k, frac=0.1):
    s = synth.SHAPES[name]
    e = synth.shape_edges(s)
    ef = make_file(os.path.join(tmp, f"{name}.grpe"), e, s.num_nodes)
    t0 = time.time()
    lab, rep = streamcut.partition(ef, k, GremConfig(chunk_frac=frac), os.path.join(tmp, "w"))
    dt = time.time() - t0
    return lab, dict(shape=name, num_nodes=s.num_nodes, num_edges=s.num_edges, k=k, chunk_frac=frac,
                     reference_seconds=round(dt, 2), cut_edges=rep.cut_edges, cut_fraction=rep.cut_fraction,
                     partition_sizes=list(rep.partition_sizes), balance_ratio=rep.balance_ratio,
                     labels_sha256=sha(lab), edges_sha256=hashlib.sha256(e.tobytes()).hexdigest())


def main():
    tmp = tempfile.mkdtemp()
    path = os.path.join(HERE, "golden_shapes.json")
    shapes = json.load(open(path)) if os.path.exists(path) else {}
    if "--products" in sys.argv:
        _, shapes["products_k16"] = shape_case(tmp, "products", 16)
    else:
        random_cases(tmp)
        lab, shapes["tiny_k4"] = shape_case(tmp, "tiny", 4)
        np.save(os.path.join(HERE, "golden_tiny_k4.npy"), lab.astype(np.int32))
        _, shapes["arxiv_k8"] = shape_case(tmp, "arxiv", 8)
    merged = json.load(open(path)) if os.path.exists(path) else {}
    merged.update(shapes)
    json.dump(merged, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps(shapes, indent=1))


if __name__ == "__main__":
    main()
