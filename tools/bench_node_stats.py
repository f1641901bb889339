"""compute_node_stats on the GPU (theory.py:97-122), papers100M-shaped,
device-resident edges and labels, k / k0 written to device buffers: one JSON
line with the per-call time and edges/s (CUDA events on the library stream
are inside grem_get_stats; here wall time around a synchronous call).

    python tools/bench_node_stats.py [SHAPE]
"""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2502_17846_b200 import grem, synth, _abi

name = sys.argv[1] if len(sys.argv) > 1 else "papers100m"
s = synth.SHAPES[name]
L = _abi.lib(); ctx = grem.context(); ptr = ctypes.c_void_p()
assert L.grem_device_alloc(ctx, s.num_edges * 8, ctypes.byref(ptr)) == 0
assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, s.num_edges, ptr) == 0
lab = torch.randint(0, 2, (s.num_nodes,), dtype=torch.int32, device="cuda")
k = torch.empty(s.num_nodes, dtype=torch.int64, device="cuda")
k0 = torch.empty_like(k)
torch.cuda.synchronize()
ms = []
for i in range(6):
    t0 = time.perf_counter()
    rc = L.grem_node_stats_u32(ctx, ptr, s.num_edges, s.num_nodes, 1, lab.data_ptr(), 1, k.data_ptr(), k0.data_ptr())
    assert rc == 0, L.grem_last_error()
    ms.append((time.perf_counter() - t0) * 1e3)
st = grem.last_stats()
best = min(ms[1:])
# algorithmic bytes: 8 B edge + 2 x 4 B label gathers + 2 x 8 B counter REDs per edge, 16 B (k, k0) per node
alg = s.num_edges * (8 + 8 + 16) + s.num_nodes * (16 + 16)
print(json.dumps({"shape": name, "edges": s.num_edges, "ms": round(best, 3), "edges_per_s": s.num_edges / best * 1e3,
                  "alg_GBps": alg / best / 1e6, "total_endpoints": int(k.sum().item()),
                  "lib_ms_total": st.get("ms_total")}))
