import sys, time, ctypes
sys.path.insert(0, ".")
from paper_2502_17846_b200 import GremConfig, grem, synth, _abi
name = sys.argv[1]; k = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
s = synth.SHAPES[name]
L = _abi.lib(); ctx = grem.context(); ptr = ctypes.c_void_p()
assert L.grem_device_alloc(ctx, s.num_edges * 8, ctypes.byref(ptr)) == 0
assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, s.num_edges, ptr) == 0
grem.set_profiling(True)
for r in range(reps):
    lab, rep = grem.partition_edges(None, s.num_nodes, k, GremConfig(chunk_frac=0.1), on_device_ptr=ptr.value, num_edges=s.num_edges)
    st = grem.last_stats()
    ph = grem.phase_times()
    tot = sum(v[0] for v in ph.values())
    print(f"rep {r}: total {st['ms_total']:.1f} ms, phases sum {tot:.1f} ms, rounds {st['rounds']} kernels {st['kernels']}")
    for kname, (ms, n) in sorted(ph.items(), key=lambda kv: -kv[1][0]):
        if n: print(f"   {kname:12s} {ms:9.2f} ms  {n:6d} groups")
