"""Determinism + where do final mismatches sit (filled nodes or streamed)."""
import sys, os, tempfile
sys.path.insert(0, ".")
from math import ceil
import numpy as np
from oracle import oracle
from paper_2502_17846_b200 import GremConfig, grem, synth
from paper_2502_17846_b200.edgefile import open_edge_file

s = synth.SHAPES["arxiv"]
e = synth.shape_edges(s); n = s.num_nodes; cap = ceil(n / 2); ce = ceil(0.1 * len(e))
ref = oracle.bisect(e, n, ce, cap)
seen = np.zeros(n, bool); seen[e.reshape(-1)] = True
for rep in range(3):
    lab, _ = grem.bisect_edges(e, n, GremConfig(chunk_edges=ce), capacity=cap)
    st = grem.last_stats()
    diff = np.flatnonzero(lab != ref)
    print("bisect_edges rep", rep, "diffs", diff.size, "in seen", int(seen[diff].sum()), "walk", st["walk_steps"], diff[:8], flush=True)
d = tempfile.mkdtemp(); p = os.path.join(d, "g.grpe"); synth.write_grpe(p, e, n)
ef = open_edge_file(p)
for rep in range(2):
    lab, _ = grem.bisect(ef, GremConfig(chunk_frac=0.1))
    print("bisect(file) rep", rep, "diffs", int((lab != ref).sum()), flush=True)
    lab, _ = grem.bisect(ef, GremConfig(chunk_frac=0.1), on_chunk=lambda st: None)
    print("bisect(file,hook) rep", rep, "diffs", int((lab != ref).sum()), flush=True)
