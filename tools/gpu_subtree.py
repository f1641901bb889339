"""Re-create a recursion node of papers100m k=16 (side path like '1' or '10')
as a standalone bisection on the GPU, then time it with per-phase profiling."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2502_17846_b200 import GremConfig, grem, synth, _abi

path = sys.argv[1] if len(sys.argv) > 1 else "1"
s = synth.SHAPES["papers100m"]
L = _abi.lib(); ctx = grem.context()
e = torch.empty((s.num_edges, 2), dtype=torch.int32, device="cuda")
assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, s.num_edges, e.data_ptr()) == 0
n = s.num_nodes
cfg = GremConfig(chunk_frac=0.1)
for side in path:
    m = e.shape[0]
    # partition() bisects each level with the level capacity of the ORIGINAL n
    lab, _ = grem.partition_edges(None, n, 2, cfg, on_device_ptr=e.data_ptr(), num_edges=m)
    lab = torch.from_numpy(lab).cuda()
    sel = lab == int(side)
    newid = torch.cumsum(sel.to(torch.int64), 0) - 1
    ei = e.long()
    keep = sel[ei[:, 0]] & sel[ei[:, 1]]
    e = newid[ei[keep]].to(torch.int32).contiguous()
    n = int(sel.sum())
    del ei, keep, newid, sel, lab
    print(f"side {side}: n {n} m {e.shape[0]}", flush=True)
import os
prof = os.environ.get('SUBTREE_PROFILE', '1') == '1'
grem.set_profiling(prof)
m = e.shape[0]
for r in range(3):
    t = time.perf_counter()
    lab, rep = grem.partition_edges(None, n, 2, cfg, on_device_ptr=e.data_ptr(), num_edges=m)
    wall = (time.perf_counter() - t) * 1e3
    st = grem.last_stats(); ph = grem.phase_times()
    print(f"rep {r}: wall {wall:.1f} ms dev {st['ms_total']:.1f} ms rounds {st['rounds']} kernels {st['kernels']} misses {st['walk_steps']}")
    for k, (ms, c) in sorted(ph.items(), key=lambda kv: -kv[1][0]):
        if c: print(f"   {k:12s} {ms:8.2f} ms {c:5d}")
