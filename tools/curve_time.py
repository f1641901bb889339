"""Time theory_curve on papers100M-shaped node statistics (GPU) vs the
reference restatement on a sample: python tools/curve_time.py"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2502_17846_b200 import GremConfig, grem, synth, _abi, theory_curve
from paper_2502_17846_b200.theory import node_stats_edges
from oracle import theory_oracle as O
s = synth.SHAPES["papers100m"]
L = _abi.lib(); ctx = grem.context(); ptr = ctypes.c_void_p()
assert L.grem_device_alloc(ctx, s.num_edges * 8, ctypes.byref(ptr)) == 0
assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, s.num_edges, ptr) == 0
lab, _ = grem.bisect_edges(None, s.num_nodes, GremConfig(chunk_frac=0.1), on_device_ptr=ptr.value, num_edges=s.num_edges)
st = node_stats_edges(None, s.num_nodes, lab, on_device_ptr=ptr.value, num_edges=s.num_edges)
xs = [0.001, 0.01, 0.1, 0.5, 1.0]
for r in range(3):
    t0 = time.perf_counter(); pts = theory_curve(st, xs, 2.0); t1 = time.perf_counter()
    print(f"theory_curve papers100m n={s.num_nodes} {len(xs)} points: {1e3 * (t1 - t0):.1f} ms "
          f"(incl. {16 * s.num_nodes / 1e9:.2f} GB host->device)", flush=True)
print([round(p.expected_cut_fraction, 9) for p in pts])
# oracle on a 200k-node sample of the same statistics (memoised like the reference)
idx = np.random.default_rng(0).choice(s.num_nodes, 200000, replace=False)
t0 = time.perf_counter(); v = O.expected_cuts(st.k[idx], st.k0[idx], 0.1, 2.0); t1 = time.perf_counter()
from paper_2502_17846_b200.theory import NodeStats, expected_cuts
g = expected_cuts(NodeStats(st.k[idx], st.k0[idx]), 0.1, 2.0).expected_cuts
print(f"oracle (python, reference algorithm) 200k-node sample x=0.1: {1e3 * (t1 - t0):.0f} ms; gpu {g!r} oracle {v!r} rel {abs(g - v) / v:.2e}")
