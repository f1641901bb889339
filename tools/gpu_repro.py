import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import oracle
from paper_2502_17846_b200 import GremConfig, grem, synth
s = synth.SHAPES["arxiv"]
e = synth.shape_edges(s); N = s.num_nodes
ref = oracle.partition(e, N, 4, chunk_frac=0.1)
for rep in range(2):
    lab, _ = grem.partition_edges(e, N, 4, GremConfig(chunk_frac=0.1))
    print("rep", rep, "mismatches", int((lab != ref).sum()), flush=True)
