"""The level-1 sparse side of papers100M (n ~ 55.5M, m ~ 27.5M) as a
standalone bisection, for profiling the sparse rounds:
python tools/sparse_side.py [REPS]   (phase times of the last rep; GREM_LIB selects a build)"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2502_17846_b200 import GremConfig, grem, synth, _abi
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = synth.SHAPES["papers100m"]
cache = "/tmp/papers_sparse_side.npy"
L = _abi.lib(); ctx = grem.context()
if os.path.exists(cache):
    sub = np.load(cache)
    nsub = int(open(cache + ".n").read())
else:
    ptr = ctypes.c_void_p()
    assert L.grem_device_alloc(ctx, s.num_edges * 8, ctypes.byref(ptr)) == 0
    assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, s.num_edges, ptr) == 0
    lab, _ = grem.bisect_edges(None, s.num_nodes, GremConfig(chunk_frac=0.1), on_device_ptr=ptr.value,
                               num_edges=s.num_edges)
    e = np.empty((s.num_edges, 2), dtype=np.uint32)
    assert L.grem_memcpy_d2h(ctx, ctypes.c_void_p(e.ctypes.data), ptr, s.num_edges * 8) == 0
    L.grem_device_free(ctx, ptr)
    lab = np.asarray(lab)
    # the side with fewer induced edges (grem.py:305-316 recursion: the sparse sibling)
    cnt = [int(np.count_nonzero((lab[e[:, 0]] == sd) & (lab[e[:, 1]] == sd))) for sd in (0, 1)]
    sd = int(np.argmin(cnt))
    keep = (lab[e[:, 0]] == sd) & (lab[e[:, 1]] == sd)
    rank = np.cumsum(lab == sd) - 1
    sub = rank[e[keep]].astype(np.uint32)
    nsub = int((lab == sd).sum())
    np.save(cache, sub)
    open(cache + ".n", "w").write(str(nsub))
print(f"sparse side: n={nsub} m={len(sub)}", flush=True)
cfg = GremConfig(chunk_frac=0.1)
dsub = ctypes.c_void_p()
assert L.grem_device_alloc(ctx, max(1, sub.nbytes), ctypes.byref(dsub)) == 0
assert L.grem_memcpy_h2d(ctx, dsub, ctypes.c_void_p(sub.ctypes.data), sub.nbytes) == 0
if os.environ.get("PHASES"):
    grem.set_profiling(2)
for r in range(reps):
    t0 = time.perf_counter()
    lab, rep = grem.bisect_edges(None, nsub, cfg, on_device_ptr=dsub.value, num_edges=len(sub))
    st = grem.last_stats()
    print(f"rep {r}: {st['ms_total']:.1f} ms (wall {1e3 * (time.perf_counter() - t0):.1f}) rounds={st['rounds']} "
          f"kernels={st['kernels']} cut={rep.cut_edges}", flush=True)
if os.environ.get("PHASES"):
    print(" ".join(f"{k}={v[0]:.2f}/{v[1]}" for k, v in sorted(grem.phase_times().items()) if v[1]))
