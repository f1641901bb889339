"""e2e partition() from pinned host memory vs device-resident, same box:
python tools/e2e_time.py SHAPE K [REPS]   (GREM_LIB selects a library build)"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2502_17846_b200 import GremConfig, grem, synth, _abi
name = sys.argv[1]; k = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
s = synth.SHAPES[name]
L = _abi.lib(); ctx = grem.context(); ptr = ctypes.c_void_p()
E = s.num_edges
assert L.grem_device_alloc(ctx, E * 8, ctypes.byref(ptr)) == 0
assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, E, ptr) == 0
host = torch.empty((E, 2), dtype=torch.int32, pin_memory=True)
assert L.grem_memcpy_d2h(ctx, ctypes.c_void_p(host.data_ptr()), ptr, E * 8) == 0
hv = host.numpy().view(np.uint32)
cfg = GremConfig(chunk_frac=0.1)
dev, e2e = [], []
for r in range(reps):
    grem.partition_edges(None, s.num_nodes, k, cfg, on_device_ptr=ptr.value, num_edges=E)
    dev.append(grem.last_stats()["ms_total"])
    t0 = time.perf_counter()
    lab, _ = grem.partition_edges(hv, s.num_nodes, k, cfg)
    e2e.append((time.perf_counter() - t0) * 1e3)
tag = os.environ.get("GREM_LIB", "default").split("/")[-1]
print(f"[{tag}] {name} k={k} device ms {['%.1f' % v for v in dev]}  e2e ms {['%.1f' % v for v in e2e]}  "
      f"min {min(dev[1:] or dev):.1f} / {min(e2e[1:] or e2e):.1f}", flush=True)
