"""Quick GPU-vs-oracle sweep used during development (prints mismatches)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from oracle import oracle
from paper_2502_17846_b200 import GremConfig, SeedConfig, grem, synth

def check(tag, a, b):
    ok = np.array_equal(a, b)
    print(f"{tag}: {'OK' if ok else 'MISMATCH %d' % int((a != b).sum())}", flush=True)
    return ok

rng = np.random.default_rng(2024)
bad = 0
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    n = int(rng.integers(2, 61)); m = int(rng.integers(1, 1001))
    edges = rng.integers(0, n, size=(m, 2)).astype(np.uint32)
    ce = int(rng.integers(1, m + 1)); refine = bool(rng.integers(0, 2)); passes = int(rng.integers(1, 3))
    slack = float(rng.choice([0.0, 0.1, 0.25]))
    cfg = GremConfig(chunk_edges=ce, refine=refine, passes=passes, capacity_slack=slack)
    cap = -(-int((1.0 + slack) * n * 1) // 1)
    from math import ceil
    cap = ceil((1.0 + slack) * n / 2)
    lab, rep = grem.bisect_edges(edges, n, cfg)
    ok = check(f"bisect t{trial} n={n} m={m} ce={ce} r={refine} p={passes}", lab, oracle.bisect(edges, n, ce, cap, refine, passes))
    p = int(rng.choice([2, 4, 8]))
    frac = float(rng.choice([0.05, 0.1, 0.3, 1.0]))
    cfg2 = GremConfig(chunk_frac=frac, refine=refine, passes=passes, capacity_slack=slack)
    lab2, rep2 = grem.partition_edges(edges, n, p, cfg2)
    ok &= check(f"partition t{trial} p={p}", lab2, oracle.partition(edges, n, p, slack=slack, chunk_frac=frac, refine=refine, passes=passes))
    bad += not ok
for name in ["tiny", "arxiv"]:
    s = synth.SHAPES[name]
    e = synth.shape_edges(s)
    t = time.time(); lab, rep = grem.partition_edges(e, s.num_nodes, s.k, GremConfig(chunk_frac=0.1)); t1 = time.time() - t
    st = grem.last_stats()
    t = time.time(); ref = oracle.partition(e, s.num_nodes, s.k, chunk_frac=0.1); t2 = time.time() - t
    bad += not check(f"{name} k={s.k} gpu {t1:.3f}s oracle {t2:.3f}s {rep} {st}", lab, ref)
print("TOTAL BAD", bad)
