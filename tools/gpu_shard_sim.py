"""Per-rank time of the subtree-sharded partition, all ranks simulated one
after another on one GPU (max over ranks = the N-GPU step without the merge)."""
import sys, time, ctypes, hashlib
sys.path.insert(0, ".")
import numpy as np
from paper_2502_17846_b200 import GremConfig, grem, synth, _abi
from paper_2502_17846_b200.shard import partition_shard

name = sys.argv[1]; k = int(sys.argv[2])
s = synth.SHAPES[name]
L = _abi.lib(); ctx = grem.context()
ptr = ctypes.c_void_p()
assert L.grem_device_alloc(ctx, s.num_edges * 8, ctypes.byref(ptr)) == 0
assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, s.num_edges, ptr) == 0
cfg = GremConfig(chunk_frac=0.1)
for _ in range(2):
    full, rep = grem.partition_edges(None, s.num_nodes, k, cfg, on_device_ptr=ptr.value, num_edges=s.num_edges)
print("full", grem.last_stats()["ms_total"], flush=True)
for world in (2, 4, 8):
    parts, ms = [], []
    for r in range(world):
        out = np.empty(s.num_nodes, dtype=np.int32)
        partition_shard(ptr.value, s.num_edges, s.num_nodes, k, cfg, r, world, out)
        partition_shard(ptr.value, s.num_edges, s.num_nodes, k, cfg, r, world, out)
        ms.append(grem.last_stats()["ms_total"]); parts.append(out)
    ok = np.array_equal(np.maximum.reduce(parts), full)
    print(f"world {world}: per-rank ms {[round(x,1) for x in ms]} max {max(ms):.1f} merged==full {ok}", flush=True)
