"""CPU: pin the C oracle (oracle/grem_oracle.c) to the real reference.

(1) label-for-label against streamcut itself (imported from baseline/_ref) on
    random multigraphs in the distribution of the reference's own fidelity test
    (tests/test_acceptance.py:72-96, criterion c01), for bisect, partition and
    count_cuts, including the random seed algorithm and slack/passes/refine
    variants;
(2) against the committed golden fixtures produced by streamcut
    (tests/golden/make_golden.py), so the pin also holds where the reference
    cannot be imported.
"""
import json
import os
from math import ceil

import numpy as np
import pytest

from conftest import have_streamcut
from helpers import labels_sha, random_multigraph
from oracle import oracle
from paper_2502_17846_b200 import synth


def test_oracle_matches_golden_random(golden_dir):
    g = np.load(os.path.join(golden_dir, "golden_random.npz"))
    cases = sorted({k.split("_")[0] for k in g.files})
    assert len(cases) == 40
    for c in cases:
        e = g[f"{c}_edges"]
        n, ce, refine, passes, p, rp, t, rnd = (int(v) for v in g[f"{c}_params"])
        slack, frac = (float(v) for v in g[f"{c}_floats"])
        algo = "random" if rnd else "bfs_grow"
        cap = ceil((1.0 + slack) * n / 2)
        lab = oracle.bisect(e, n, ce, cap, bool(refine), passes, seed_algo=algo, seed_refinement_passes=rp,
                            rng_seed=t)
        assert np.array_equal(lab, g[f"{c}_bisect"]), c
        lab2 = oracle.partition(e, n, p, slack=slack, chunk_frac=frac, refine=bool(refine), passes=passes,
                                seed_algo=algo, seed_refinement_passes=rp, rng_seed=t)
        assert np.array_equal(lab2, g[f"{c}_partition"]), c
        cut, _ = oracle.count_cuts(e, n, lab2)
        assert cut == int(g[f"{c}_rep"][1])


def test_oracle_matches_golden_shapes(golden_dir):
    shapes = json.load(open(os.path.join(golden_dir, "golden_shapes.json")))
    tiny = np.load(os.path.join(golden_dir, "golden_tiny_k4.npy"))
    for key in ("tiny_k4", "arxiv_k8"):
        gs = shapes[key]
        s = synth.SHAPES[gs["shape"]]
        e = synth.shape_edges(s)
        import hashlib
        assert hashlib.sha256(e.tobytes()).hexdigest() == gs["edges_sha256"], "generator drifted"
        lab = oracle.partition(e, s.num_nodes, gs["k"], chunk_frac=gs["chunk_frac"])
        assert labels_sha(lab) == gs["labels_sha256"], key
        cut, sizes = oracle.count_cuts(e, s.num_nodes, lab)
        assert cut == gs["cut_edges"] and list(sizes) == gs["partition_sizes"]
        if key == "tiny_k4":
            assert np.array_equal(lab, tiny)


@pytest.mark.skipif(not have_streamcut(), reason="reference package not importable here")
def test_oracle_matches_streamcut_random(tmp_path):
    import streamcut
    from streamcut import BinaryEdgeWriter, GremConfig, SeedConfig, open_edge_file

    rng = np.random.default_rng(2024)
    for trial in range(60):
        edges, n = random_multigraph(rng, max_nodes=60, max_edges=1000)
        path = str(tmp_path / f"g{trial}.grpe")
        with BinaryEdgeWriter(path, n) as w:
            w.write(edges)
        ef = open_edge_file(path)
        ce = int(rng.integers(1, len(edges) + 1))
        refine = bool(rng.integers(0, 2)) or trial < 25
        passes = int(rng.integers(1, 3))
        slack = float(rng.choice([0.0, 0.1, 0.25]))
        cfg = GremConfig(chunk_edges=ce, refine=refine, passes=passes, capacity_slack=slack)
        ref, rep = streamcut.bisect(ef, cfg)
        got = oracle.bisect(edges, n, ce, ceil((1.0 + slack) * n / 2), refine, passes)
        assert np.array_equal(ref, got), trial
        cut, sizes = oracle.count_cuts(edges, n, got)
        assert cut == rep.cut_edges and sizes == rep.partition_sizes
        p = int(rng.choice([2, 4, 8]))
        frac = float(rng.choice([0.05, 0.1, 0.3, 1.0]))
        ref2, _ = streamcut.partition(ef, p, GremConfig(chunk_frac=frac, refine=refine, passes=passes,
                                                        capacity_slack=slack), str(tmp_path / "w"))
        got2 = oracle.partition(edges, n, p, slack=slack, chunk_frac=frac, refine=refine, passes=passes)
        assert np.array_equal(ref2, got2), trial
        if trial % 6 == 0:
            cfg3 = GremConfig(chunk_edges=ce, seed=SeedConfig(algorithm="random", rng_seed=trial))
            ref3, _ = streamcut.bisect(ef, cfg3)
            got3 = oracle.bisect(edges, n, ce, ceil(n / 2), True, 1, seed_algo="random", rng_seed=trial)
            assert np.array_equal(ref3, got3), trial


@pytest.mark.skipif(not have_streamcut(), reason="reference package not importable here")
def test_oracle_known_answers(tmp_path):
    """Known answers of the reference tests (tests/test_grem.py:224-237, 291-321)."""
    # isolated nodes are filled 5/5 (test_grem.py:224-230)
    lab = oracle.bisect(np.array([[0, 1], [2, 3]]), 10, 2, 5)
    assert np.bincount(lab, minlength=2).tolist() == [5, 5]
    # empty edge list -> sizes {2, 3} (test_grem.py:231-237)
    lab = oracle.bisect(np.empty((0, 2)), 5, 1, 3)
    assert sorted(np.bincount(lab, minlength=2).tolist()) == [2, 3]
    # K2,2 all cut (test_grem.py:300-303)
    cut, sizes = oracle.count_cuts(np.array([[0, 2], [0, 3], [1, 2], [1, 3]]), 4, np.array([0, 0, 1, 1]))
    assert cut == 4 and sizes == (2, 2)
    # self-loops are never cut (test_grem.py:305-308)
    cut, _ = oracle.count_cuts(np.array([[0, 0], [0, 1]]), 2, np.array([0, 1]))
    assert cut == 1
    with pytest.raises(oracle.OracleError):
        oracle.partition(np.array([[0, 1]]), 2, 3)


def test_numpy_generator_matches_library_generator():
    """oracle/gen_np.py (the reference arm's input, no product library) ==
    the library's host generator (csrc/grem_gen.h), byte for byte."""
    from oracle import gen_np
    from paper_2502_17846_b200 import synth
    for (n, m, beta, seed, e0) in [(10_000, 100_000, 11, 0, 0), (169_343, 50_000, 11, 0, 777),
                                   (65_608_366, 40_000, 4, 0, 0), (111_059_956, 40_000, 11, 3, 10**9), (7, 1000, 11, 5, 0)]:
        assert np.array_equal(gen_np.powerlaw_edges(n, m, beta, seed, e0), synth.powerlaw_edges(n, m, beta, seed, e0))
