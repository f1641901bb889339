"""Localize partition divergences: recursion replayed level by level."""
import sys
sys.path.insert(0, ".")
from math import ceil
import numpy as np
from oracle import oracle
from paper_2502_17846_b200 import GremConfig, grem, synth

s = synth.SHAPES[sys.argv[1] if len(sys.argv) > 1 else "arxiv"]
e = synth.shape_edges(s)
N = s.num_nodes
for k in (2, 4, 8):
    lab, _ = grem.partition_edges(e, N, k, GremConfig(chunk_frac=0.1))
    ref = oracle.partition(e, N, k, chunk_frac=0.1)
    print(f"partition k={k}: mismatches {int((lab != ref).sum())}", flush=True)

def sub(edges, lab, side):
    members = np.flatnonzero(lab == side)
    newid = np.full(lab.shape[0], -1, np.int64); newid[members] = np.arange(members.size)
    keep = (lab[edges[:, 0]] == side) & (lab[edges[:, 1]] == side)
    se = edges[keep]
    return np.column_stack([newid[se[:, 0]], newid[se[:, 1]]]).astype(np.uint32), members.size

lvl = [(e, N)]
for level in range(3):
    cap = ceil(N / 2 ** (level + 1))
    nxt = []
    for (ed, n) in lvl:
        ce = max(1, ceil(0.1 * len(ed)))
        ref = oracle.bisect(ed, n, ce, cap)
        got, _ = grem.bisect_edges(ed, n, GremConfig(chunk_edges=ce), capacity=cap)
        st = grem.last_stats()
        print(f"level {level} n={n} m={len(ed)} cap={cap}: mismatches {int((got != ref).sum())} walk={st['walk_steps']} rounds={st['rounds']}", flush=True)
        for side in (0, 1):
            nxt.append(sub(ed, ref, side))
    lvl = nxt
