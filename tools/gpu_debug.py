"""Localize a GPU/oracle divergence: seed-only, then per-chunk sizes."""
import sys
sys.path.insert(0, ".")
from math import ceil
import numpy as np
from oracle import oracle
from paper_2502_17846_b200 import GremConfig, grem, synth

name = sys.argv[1] if len(sys.argv) > 1 else "arxiv"
s = synth.SHAPES[name]
e = synth.shape_edges(s)
n = s.num_nodes
cap = ceil(n / 2)
for frac in [1.0, 0.5, 0.2, 0.1]:
    ce = max(1, ceil(frac * len(e)))
    lab, _ = grem.bisect_edges(e, n, GremConfig(chunk_edges=ce))
    st = grem.last_stats()
    ref = oracle.bisect(e, n, ce, cap)
    print(f"frac={frac}: mismatches={int((lab != ref).sum())} stats={st}", flush=True)
# per-chunk sizes with hooks through the file API
import tempfile, os
d = tempfile.mkdtemp()
p = os.path.join(d, "g.grpe")
synth.write_grpe(p, e, n)
from paper_2502_17846_b200.edgefile import open_edge_file
ef = open_edge_file(p)
gs = []
grem.bisect(ef, GremConfig(chunk_frac=0.1), on_chunk=lambda st: gs.append((tuple(st.sizes), st.recount_sizes())))
os_ = []
oracle.bisect(e, n, ceil(0.1 * len(e)), cap, on_chunk=lambda sz: os_.append(tuple(sz)))
for i, (g, o) in enumerate(zip(gs, os_)):
    print(i, "gpu", g, "oracle", o, "OK" if g[0] == o and list(g[0]) == g[1] else "DIFF")
