"""Run the C oracle on a large benchmark shape and store labels sha/report
(dev tool: the hashes become tests/golden/big_shapes.json)."""
import sys, time, json, hashlib
sys.path.insert(0, ".")
import numpy as np
from oracle import oracle
from paper_2502_17846_b200 import synth
name = sys.argv[1]; k = int(sys.argv[2]); frac = float(sys.argv[3]) if len(sys.argv) > 3 else 0.1
s = synth.SHAPES[name]
t = time.time(); e = synth.shape_edges(s, threads=8); tg = time.time() - t
print(name, "generated", e.shape, f"{tg:.1f}s", flush=True)
st = oracle.OracleStats()
t = time.time(); lab = oracle.partition(e, s.num_nodes, k, chunk_frac=frac, stats=st); dt = time.time() - t
cut, sizes = oracle.count_cuts(e, s.num_nodes, lab)
out = dict(shape=name, num_nodes=s.num_nodes, num_edges=s.num_edges, k=k, chunk_frac=frac, seconds=dt,
           cut_edges=cut, partition_sizes=list(sizes), visits=st.visits, chunks=st.chunks,
           labels_sha256=hashlib.sha256(lab.astype("<i4").tobytes()).hexdigest())
print(json.dumps(out), flush=True)
json.dump(out, open(f"/root/golden_big/{name}_k{k}_f{frac}.json", "w"))
