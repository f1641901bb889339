"""Per-bisection phase split (serial siblings): GREM_DEBUG_LEVELS=1 GREM_SERIAL_SIBLINGS=1 python tools/gpu_levels_phases.py SHAPE K"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_17846_b200 import GremConfig, grem, synth, _abi
name = sys.argv[1]; k = int(sys.argv[2]); s = synth.SHAPES[name]
L = _abi.lib(); ctx = grem.context(); ptr = ctypes.c_void_p()
assert L.grem_device_alloc(ctx, s.num_edges * 8, ctypes.byref(ptr)) == 0
assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, s.num_edges, ptr) == 0
for r in range(2):
    if r == 1:
        print("---- warm", file=sys.stderr, flush=True)
        grem.set_profiling(True)
    lab, rep = grem.partition_edges(None, s.num_nodes, k, GremConfig(chunk_frac=0.1), on_device_ptr=ptr.value,
                                    num_edges=s.num_edges)
print(grem.last_stats()["ms_total"])
