"""Time partition() on a device-generated synthetic shape: python tools/gpu_time.py SHAPE K [REPS]
Prints per-rep ms, rounds and the labels sha256 (compare with tests/golden)."""
import ctypes, hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_17846_b200 import GremConfig, grem, synth, _abi
name = sys.argv[1]; k = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
s = synth.SHAPES[name]
L = _abi.lib(); ctx = grem.context(); ptr = ctypes.c_void_p()
assert L.grem_device_alloc(ctx, s.num_edges * 8, ctypes.byref(ptr)) == 0
assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, s.num_edges, ptr) == 0
ts = []
for r in range(reps):
    lab, rep = grem.partition_edges(None, s.num_nodes, k, GremConfig(chunk_frac=0.1), on_device_ptr=ptr.value,
                                    num_edges=s.num_edges)
    st = grem.last_stats()
    ts.append(st["ms_total"])
sha = hashlib.sha256(lab.astype("<i4").tobytes()).hexdigest()
tag = " ".join(f"{k2}={v}" for k2, v in os.environ.items() if k2.startswith("GREM_"))
print(f"{name} k={k} [{tag}] ms={['%.1f' % t for t in ts]} min={min(ts[1:] or ts):.1f} rounds={st['rounds']} "
      f"kernels={st['kernels']} cut={rep.cut_edges} sha={sha[:16]}", flush=True)
