"""One sparse bisection like papers' level-3 sparse subtrees (n 13.9M,
m 5.4M power-law), serial, with per-phase device times and wall time."""
import sys, time, ctypes
sys.path.insert(0, ".")
from paper_2502_17846_b200 import GremConfig, grem, _abi
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 13882495
m = int(float(sys.argv[2])) if len(sys.argv) > 2 else 5408253
L = _abi.lib(); ctx = grem.context(); ptr = ctypes.c_void_p()
assert L.grem_device_alloc(ctx, m * 8, ctypes.byref(ptr)) == 0
assert L.grem_gen_edges_device(ctx, n, 11, 7, 0, m, ptr) == 0
grem.set_profiling(True)
for r in range(3):
    t = time.perf_counter()
    lab, rep = grem.partition_edges(None, n, 2, GremConfig(chunk_frac=0.1), on_device_ptr=ptr.value, num_edges=m)
    wall = (time.perf_counter() - t) * 1e3
    st = grem.last_stats(); ph = grem.phase_times()
    print(f"rep {r}: wall {wall:.1f} ms dev {st['ms_total']:.1f} ms rounds {st['rounds']} kernels {st['kernels']}")
    for k, (ms, c) in sorted(ph.items(), key=lambda kv: -kv[1][0]):
        if c: print(f"   {k:12s} {ms:8.2f} ms {c:5d}")
