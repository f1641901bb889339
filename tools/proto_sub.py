import sys, os, importlib
sys.path.insert(0, ".")
from math import ceil
import numpy as np
from oracle import oracle
from paper_2502_17846_b200 import synth
s = synth.SHAPES["arxiv"]; e = synth.shape_edges(s); N = s.num_nodes
lab0 = oracle.bisect(e, N, ceil(0.1 * len(e)), ceil(N / 2))
def sub(edges, lab, side):
    members = np.flatnonzero(lab == side)
    newid = np.full(lab.shape[0], -1, np.int64); newid[members] = np.arange(members.size)
    keep = (lab[edges[:, 0]] == side) & (lab[edges[:, 1]] == side)
    se = edges[keep]
    return np.column_stack([newid[se[:, 0]], newid[se[:, 1]]]).astype(np.uint32), members.size
for side in (1, 0):
    ed, n = sub(e, lab0, side)
    cap = ceil(N / 4)
    ref = oracle.bisect(ed, n, ceil(0.1 * len(ed)), cap)
    for J in [int(v) for v in os.environ.get("JS", "0,1,2,3").split(",")]:
        os.environ["JACOBI"] = str(J)
        import tools.proto_rounds as pr
        importlib.reload(pr)
        st = dict(rounds=0, max_rounds=0, visits=0, walk=0, flagged=0, jacobi=0)
        got = pr.bisect_proto(ed, n, ceil(0.1 * len(ed)), cap, stats=st)
        print(f"side {side} n={n} m={len(ed)} J={J}: equal={np.array_equal(got, ref)} {st}", flush=True)
