"""external_shuffle on the GPU, papers100M-shaped device-resident edges:
python tools/bench_shuffle.py [SHAPE] -> one JSON line (per-call time)."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_17846_b200 import grem, synth, _abi
name = sys.argv[1] if len(sys.argv) > 1 else "papers100m"
s = synth.SHAPES[name]
L = _abi.lib(); ctx = grem.context(); ptr = ctypes.c_void_p(); out = ctypes.c_void_p()
assert L.grem_device_alloc(ctx, s.num_edges * 8, ctypes.byref(ptr)) == 0
assert L.grem_device_alloc(ctx, s.num_edges * 8, ctypes.byref(out)) == 0
assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, s.num_edges, ptr) == 0
ms = []
for i in range(4):
    t0 = time.perf_counter()
    assert L.grem_shuffle_u32(ctx, ptr, s.num_edges, s.num_nodes, 1, i, out, 1) == 0, L.grem_last_error()
    ms.append((time.perf_counter() - t0) * 1e3)
best = min(ms[1:])
print(json.dumps({"shape": name, "edges": s.num_edges, "ms": round(best, 2), "edges_per_s": s.num_edges / best * 1e3}))
