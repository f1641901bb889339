"""First chunk where GPU labels diverge from the oracle (level-0 bisect)."""
import sys, os, tempfile
sys.path.insert(0, ".")
from math import ceil
import numpy as np
from oracle import oracle
from paper_2502_17846_b200 import GremConfig, grem, synth
from paper_2502_17846_b200.edgefile import open_edge_file

s = synth.SHAPES[sys.argv[1] if len(sys.argv) > 1 else "arxiv"]
e = synth.shape_edges(s); n = s.num_nodes; cap = ceil(n / 2)
d = tempfile.mkdtemp(); p = os.path.join(d, "g.grpe"); synth.write_grpe(p, e, n)
ef = open_edge_file(p)
gl = []
grem.bisect(ef, GremConfig(chunk_frac=0.1), on_chunk=lambda st: gl.append((tuple(st.sizes), st.labels_array())))
ol = []
oracle.bisect(e, n, ceil(0.1 * len(e)), cap, on_chunk=lambda sz, parts: ol.append((tuple(sz), parts.copy())))
ce = ceil(0.1 * len(e))
for i, ((gs, gp), (os_, op)) in enumerate(zip(gl, ol)):
    diff = np.flatnonzero(gp != op)
    print(i, gs, os_, "label diffs", diff.size, diff[:10], flush=True)
    if diff.size:
        chunk = e[i * ce:(i + 1) * ce]
        nodes = np.unique(chunk)
        for g in diff[:5]:
            j = np.searchsorted(nodes, g)
            print("  node", g, "local", j, "gpu", gp[g], "oracle", op[g], "prev gpu", gl[i-1][1][g], "prev oracle", ol[i-1][1][g])
        break
