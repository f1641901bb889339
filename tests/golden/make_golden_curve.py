"""Golden fixtures for expected_cuts / theory_curve (streamcut/theory.py:125-146),
produced by the REAL reference in the build container; the GPU box only reads
the committed npz.

Cases (node statistics -> expected cut endpoints for xs x multipliers):
* seeded random NodeStats (k up to 60, some zero-degree nodes);
* node statistics of power-law graphs (synth.powerlaw_edges) against a random
  bisection, from streamcut.compute_node_stats -- hubs with tails longer than
  the per-thread limit (1024 terms) exercise the per-CTA kernel;
* a few extreme (k, k0) pairs up to k = 200000.

usage: python tests/golden/make_golden_curve.py
"""
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

from streamcut import compute_node_stats, expected_cuts, open_edge_file  # noqa: E402
from streamcut.model import NodeStats  # noqa: E402

from helpers import write_grpe  # noqa: E402
from paper_2502_17846_b200 import synth  # noqa: E402

XS = [0.001, 0.01, 0.05, 0.1, 0.25, 0.5, 1.0]
MULTS = [1.0, 2.0, 3.5]


def random_stats(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 400))
    k = rng.integers(0, 61, size=n)
    k[rng.random(n) < 0.1] = 0
    k0 = (k + 1) // 2 + (rng.random(n) * (k - (k + 1) // 2 + 1)).astype(np.int64)
    return k.astype(np.int64), np.minimum(k0, k).astype(np.int64)


def powerlaw_stats(n, m, seed, tmp):
    edges = synth.powerlaw_edges(n, m, seed=seed).astype(np.int64)
    g = write_grpe(os.path.join(tmp, f"pl{seed}.grpe"), edges, n)
    labels = np.random.default_rng(seed).integers(0, 2, size=n)
    st = compute_node_stats(open_edge_file(g), labels)
    return st.k.astype(np.int64), st.k0.astype(np.int64)


def main():
    cases = {}
    for s in range(1, 5):
        cases[f"random{s}"] = random_stats(s)
    with tempfile.TemporaryDirectory() as tmp:
        cases["powerlaw_small"] = powerlaw_stats(3000, 40000, 11, tmp)
        cases["powerlaw_hubs"] = powerlaw_stats(50000, 600000, 12, tmp)
    ek = np.array([1, 2, 3, 7, 4096, 4097, 20000, 200000, 200000, 131071], dtype=np.int64)
    ek0 = np.array([1, 1, 2, 4, 2048, 2049, 10001, 100000, 150000, 100000], dtype=np.int64)
    cases["extreme"] = (ek, ek0)
    out = {}
    for name, (k, k0) in cases.items():
        st = NodeStats(k, k0)
        vals = np.array([[expected_cuts(st, x, mu).expected_cuts for x in XS] for mu in MULTS])
        out[f"{name}_k"] = k
        out[f"{name}_k0"] = k0
        out[f"{name}_cuts"] = vals
        print(name, len(k), int(k.max()), vals[0][:3], flush=True)
    out["xs"] = np.array(XS)
    out["mults"] = np.array(MULTS)
    out["names"] = np.array(list(cases))
    np.savez_compressed(os.path.join(HERE, "golden_curve.npz"), **out)


if __name__ == "__main__":
    main()
