"""Per-phase device time of one partition (serial siblings, CUDA events per
launch group) for A/B of library builds: GREM_LIB=... python tools/phase_ab.py SHAPE K"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GREM_SERIAL_SIBLINGS", "1")
from paper_2502_17846_b200 import GremConfig, grem, synth, _abi
name = sys.argv[1]; k = int(sys.argv[2])
s = synth.SHAPES[name]
L = _abi.lib(); ctx = grem.context(); ptr = ctypes.c_void_p()
assert L.grem_device_alloc(ctx, s.num_edges * 8, ctypes.byref(ptr)) == 0
assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, s.num_edges, ptr) == 0
grem.set_profiling(2 if os.environ.get("PHASE_K") else True)
for r in range(3):
    lab, rep = grem.partition_edges(None, s.num_nodes, k, GremConfig(chunk_frac=0.1), on_device_ptr=ptr.value,
                                    num_edges=s.num_edges)
st = grem.last_stats(); ph = grem.phase_times()
print(f"[{os.environ.get('GREM_LIB', 'default').split('/')[-1]}] total {st['ms_total']:.1f} ms  " +
      " ".join(f"{kk}={v[0]:.1f}" for kk, v in sorted(ph.items()) if v[1] and (os.environ.get("PHASE_K") or not kk.startswith("k."))), flush=True)
