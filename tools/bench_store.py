"""GPU write_buckets / reorder_features throughput on a
device-resident synthetic graph, with the numpy restatement of the reference
(store.py: stable argsort by bucket id) timed on the host beside it.

  python tools/bench_store.py [SHAPE] [P]      (default papers100m 16)

Roofline (HBM): write_buckets moves 24 algorithmic B/edge (8 B edge read,
2 x 4 B label gathers, 8 B bucketed edge write); reorder_features moves
2 x record_width B/node + 4 B label read + 8 B permutation write.
"""
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_17846_b200 import _abi, grem, synth  # noqa: E402
from oracle import store_oracle  # noqa: E402  (CPU baseline only)

name = sys.argv[1] if len(sys.argv) > 1 else "papers100m"
p = int(sys.argv[2]) if len(sys.argv) > 2 else 16
s = synth.SHAPES[name]
n, m = s.num_nodes, s.num_edges
L = _abi.lib()
ctx = grem.context()
c_vp = ctypes.c_void_p
dptr, lptr, optr = c_vp(), c_vp(), c_vp()
assert L.grem_device_alloc(ctx, m * 8, ctypes.byref(dptr)) == 0
assert L.grem_gen_edges_device(ctx, n, s.beta, s.seed, 0, m, dptr) == 0
labels = np.random.default_rng(0).integers(0, p, size=n).astype(np.int32)
assert L.grem_device_alloc(ctx, n * 4, ctypes.byref(lptr)) == 0
assert L.grem_memcpy_h2d(ctx, lptr, labels.ctypes.data, n * 4) == 0
assert L.grem_device_alloc(ctx, m * 8, ctypes.byref(optr)) == 0
counts = np.zeros(p * p, dtype=np.uint64)
pp = ctypes.c_int64()


def run():
    rc = L.grem_write_buckets_u32(ctx, dptr, m, n, 1, lptr, 1, optr, 1, counts.ctypes.data, counts.size,
                                  ctypes.byref(pp))
    assert rc == 0, _abi.last_error()


for _ in range(3):
    run()
reps = 5
t = time.perf_counter()
for _ in range(reps):
    run()   # each call ends with a stream synchronise (counts to the host)
ms = (time.perf_counter() - t) * 1e3 / reps
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6535.7
gbs = 24.0 * m / (ms / 1e3) / 1e9
assert int(counts.sum()) == m
# CPU: the numpy restatement of store.py on a bounded sample of the same graph
scale = max(1, m // 20_000_000)
ns, ms_ = max(1000, n // scale), max(10000, m // scale)
es = synth.powerlaw_edges(ns, ms_, beta=s.beta, seed=s.seed).astype(np.int64)
ls = np.random.default_rng(0).integers(0, p, size=ns)
t = time.perf_counter()
store_oracle.buckets(es, ls)
cpu = ms_ / (time.perf_counter() - t)
print(json.dumps({"metric": "write_buckets edges/s (bucketed edge list in HBM)", "workload": f"{name}-shaped p={p}",
                  "num_edges": m, "ms": ms, "value": m / (ms / 1e3), "unit": "edges/s",
                  "roofline": {"bound": "hbm", "algorithmic_bytes_per_edge": 24, "achieved": gbs, "peak": peak,
                               "unit": "GB/s", "frac": gbs / peak},
                  "cpu_baseline": {"value": cpu, "unit": "edges/s", "cores": 1, "kind": "port",
                                   "sample": f"1/{scale} scale ({ns} nodes, {ms_} edges), numpy stable argsort "
                                             f"(oracle/store_oracle.py, store.py:55-104 restated)"}}))
