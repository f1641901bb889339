"""Scale run: generate a benchmark shape on the device, partition it, report
time, stats and the labels sha256 (compared with oracle hashes offline)."""
import sys, time, ctypes, hashlib
sys.path.insert(0, ".")
import numpy as np
from paper_2502_17846_b200 import GremConfig, grem, synth, _abi

name = sys.argv[1]; k = int(sys.argv[2]) if len(sys.argv) > 2 else None
frac = float(sys.argv[3]) if len(sys.argv) > 3 else 0.1
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
s = synth.SHAPES[name]; k = k or s.k
L = _abi.lib(); ctx = grem.context()
ptr = ctypes.c_void_p()
assert L.grem_device_alloc(ctx, s.num_edges * 8, ctypes.byref(ptr)) == 0
t = time.time()
assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, s.num_edges, ptr) == 0
print(f"{name}: device gen {time.time() - t:.2f}s", flush=True)
for r in range(reps):
    t = time.time()
    lab, rep = grem.partition_edges(None, s.num_nodes, k, GremConfig(chunk_frac=frac), on_device_ptr=ptr.value,
                                    num_edges=s.num_edges)
    wall = time.time() - t
    st = grem.last_stats()
    print(f"rep {r}: wall {wall*1e3:.1f} ms dev {st['ms_total']:.1f} ms  edges/s {s.num_edges/(st['ms_total']/1e3)/1e9:.3f} G"
          f"  cut {rep.cut_edges} sizes {rep.partition_sizes[:4]}.. sha {hashlib.sha256(lab.astype('<i4').tobytes()).hexdigest()[:16]}"
          f"  stats {st}", flush=True)
