"""Timeline of one papers100M-shaped k=16 partition from page-locked host
edges (the bench's e2e path) vs device-resident edges:
GREM_DEBUG_LEVELS=1 python tools/gpu_levels_e2e.py [SHAPE] [K]"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2502_17846_b200 import GremConfig, grem, synth, _abi
name = sys.argv[1] if len(sys.argv) > 1 else "papers100m"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 16
s = synth.SHAPES[name]
L = _abi.lib(); ctx = grem.context(); ptr = ctypes.c_void_p()
assert L.grem_device_alloc(ctx, s.num_edges * 8, ctypes.byref(ptr)) == 0
assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, s.num_edges, ptr) == 0
host = torch.empty((s.num_edges, 2), dtype=torch.int32, pin_memory=True)
assert L.grem_memcpy_d2h(ctx, ctypes.c_void_p(host.data_ptr()), ptr, s.num_edges * 8) == 0
hv = host.numpy().view(np.uint32)
cfg = GremConfig(chunk_frac=0.1)
for r in range(2):
    print(f"==== device-resident run {r}", flush=True)
    t0 = time.perf_counter()
    grem.partition_edges(None, s.num_nodes, k, cfg, on_device_ptr=ptr.value, num_edges=s.num_edges)
    print("wall_ms", (time.perf_counter() - t0) * 1e3, "lib_ms", grem.last_stats()["ms_total"], flush=True)
for r in range(2):
    print(f"==== pinned-host run {r}", flush=True)
    t0 = time.perf_counter()
    grem.partition_edges(hv, s.num_nodes, k, cfg)
    print("wall_ms", (time.perf_counter() - t0) * 1e3, "lib_ms", grem.last_stats()["ms_total"], flush=True)
