"""Golden fixtures for the BASELINE configs that the round-1 goldens left open:
the Friendster-shaped k = 4..256 sweep (BASELINE.json config 5) and the
frac = 0.01 secondary sweep at products / papers scale.

Run in the build container (never on the GPU box, which only reads the
committed JSON).  Two oracles:

* ``streamcut`` itself (baseline/_ref) where it finishes in minutes
  (arxiv k=64/256, products frac=0.01 k=16);
* the C restatement ``oracle/grem_oracle.c`` (pinned to streamcut by
  tests/test_oracle.py) at Friendster / papers scale, where streamcut is
  projected at many hours.

One k=256 partition yields the k = 2^j labels for every j <= 8: the level
capacity depends only on the level and the original node count
(grem.py:299) and the chunk plan only on the sub-file (edgefile.py:346), so
the first j levels of a k=256 run are the k=2^j run, and its leaf ids
``base = leaf_base + side * p_level/2`` (grem.py:306) make
``label_{2^j} = label_256 >> (8 - j)``.  ``check_shift`` verifies this with
streamcut on arxiv (k=64 run vs k=256 >> 2).

usage:
  python tests/golden/make_golden_big.py arxiv          # streamcut, k=64 and k=256 + shift check
  python tests/golden/make_golden_big.py products_f001  # streamcut, products frac=0.01 slack=0.1 k=16
  python tests/golden/make_golden_big.py friendster     # C oracle, k=256 -> k=4..256
  python tests/golden/make_golden_big.py papers_f001    # C oracle, papers frac=0.01 k=16
Each writes tests/golden/big/<name>.json; ``merge`` folds them into golden_shapes.json.
"""
import hashlib
import json
import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
OUT = os.path.join(HERE, "big")


def sha(labels):
    return hashlib.sha256(np.asarray(labels, dtype="<i4").tobytes()).hexdigest()


def report(name, s, k, frac, slack, lab, cut, sizes, seconds, pinned_by):
    n_parts = len(sizes)
    bal = max(sizes) / -(-s.num_nodes // n_parts)
    return dict(shape=name, num_nodes=s.num_nodes, num_edges=s.num_edges, k=k, chunk_frac=frac,
                capacity_slack=slack, cut_edges=int(cut), cut_fraction=int(cut) / s.num_edges,
                partition_sizes=[int(x) for x in sizes], balance_ratio=bal, labels_sha256=sha(lab),
                seconds=round(seconds, 1), pinned_by=pinned_by)


def _streamcut():
    for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(cand):
            sys.path.insert(0, cand)
            break
    import streamcut
    return streamcut


def streamcut_run(name, k, frac, slack, tmp):
    sc = _streamcut()
    from paper_2502_17846_b200 import synth
    s = synth.SHAPES[name]
    e = synth.shape_edges(s, threads=8)
    path = os.path.join(tmp, f"{name}.grpe")
    with sc.BinaryEdgeWriter(path, s.num_nodes) as w:
        w.write(e.astype(np.int64))
    ef = sc.open_edge_file(path)
    t0 = time.time()
    lab, rep = sc.partition(ef, k, sc.GremConfig(chunk_frac=frac, capacity_slack=slack), os.path.join(tmp, "w"))
    dt = time.time() - t0
    return s, e, lab, rep, dt


def cmd_arxiv():
    tmp = tempfile.mkdtemp()
    res = {}
    s, e, lab64, rep64, dt64 = streamcut_run("arxiv", 64, 0.1, 0.0, tmp)
    _, _, lab256, rep256, dt256 = streamcut_run("arxiv", 256, 0.1, 0.0, tmp)
    assert np.array_equal(lab256 >> 2, lab64), "k=256 >> 2 != k=64 (shift property)"
    pin = "streamcut (baseline/_ref) run in the build container"
    res["arxiv_k64"] = report("arxiv", s, 64, 0.1, 0.0, lab64, rep64.cut_edges, rep64.partition_sizes, dt64, pin)
    res["arxiv_k256"] = report("arxiv", s, 256, 0.1, 0.0, lab256, rep256.cut_edges, rep256.partition_sizes,
                               dt256, pin)
    res["arxiv_k256"]["shift_check"] = "streamcut k=256 labels >> 2 == streamcut k=64 labels"
    return res


def cmd_products_f001():
    tmp = tempfile.mkdtemp()
    s, e, lab, rep, dt = streamcut_run("products", 16, 0.01, 0.1, tmp)
    return {"products_k16_f0.01_s0.1": report("products", s, 16, 0.01, 0.1, lab, rep.cut_edges,
                                              rep.partition_sizes, dt,
                                              "streamcut (baseline/_ref) run in the build container")}


def oracle_run(name, k, frac, slack, ks):
    from oracle import oracle
    from paper_2502_17846_b200 import synth
    s = synth.SHAPES[name]
    e = synth.shape_edges(s, threads=8)
    t0 = time.time()
    lab = oracle.partition(e, s.num_nodes, k, slack=slack, chunk_frac=frac)
    dt = time.time() - t0
    print(f"{name} k={k} frac={frac}: {dt:.0f} s", flush=True)
    res = {}
    lk = int(np.log2(k))
    pin = ("C oracle (oracle/grem_oracle.c, pinned to streamcut by tests/test_oracle.py); "
           "streamcut itself is projected at many hours for this shape")
    for kk in ks:
        sub = lab >> (lk - int(np.log2(kk)))
        cut, sizes = oracle.count_cuts(e, s.num_nodes, sub)
        key = f"{name}_k{kk}" + ("" if frac == 0.1 else f"_f{frac}") + ("" if slack == 0 else f"_s{slack}")
        res[key] = report(name, s, kk, frac, slack, sub, cut, sizes, dt, pin)
        if kk != k:
            res[key]["derived_from"] = f"{name} k={k} labels >> {lk - int(np.log2(kk))} (see module docstring)"
        print(json.dumps(res[key]), flush=True)
    return res


def cmd_friendster():
    return oracle_run("friendster", 256, 0.1, 0.0, [4, 8, 16, 32, 64, 128, 256])


def cmd_papers_f001():
    return oracle_run("papers100m", 16, 0.01, 0.0, [16])


def cmd_merge():
    path = os.path.join(HERE, "golden_shapes.json")
    merged = json.load(open(path))
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".json"):
            merged.update(json.load(open(os.path.join(OUT, f))))
    json.dump(merged, open(path, "w"), indent=1, sort_keys=True)


def main():
    cmd = sys.argv[1]
    if cmd == "merge":
        return cmd_merge()
    res = globals()["cmd_" + cmd]()
    os.makedirs(OUT, exist_ok=True)
    json.dump(res, open(os.path.join(OUT, f"{cmd}.json"), "w"), indent=1, sort_keys=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
