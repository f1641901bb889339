import sys
sys.path.insert(0, ".")
from math import ceil
import numpy as np
from oracle import oracle
from paper_2502_17846_b200 import GremConfig, grem, synth
s = synth.SHAPES["arxiv"]
e = synth.shape_edges(s); N = s.num_nodes
order = [int(x) for x in sys.argv[1:]] or [8, 8, 2, 4, 8]
refs = {}
for k in order:
    if k not in refs: refs[k] = oracle.partition(e, N, k, chunk_frac=0.1)
    lab, _ = grem.partition_edges(e, N, k, GremConfig(chunk_frac=0.1))
    st = grem.last_stats()
    print(f"k={k}: mismatches {int((lab != refs[k]).sum())} walk={st['walk_steps']} rounds={st['rounds']} ms={st['ms_total']:.1f}", flush=True)
ce = ceil(0.1 * len(e)); ref = oracle.bisect(e, N, ce, ceil(N / 2))
lab, _ = grem.bisect_edges(e, N, GremConfig(chunk_edges=ce))
print("bisect after:", int((lab != ref).sum()))
