"""Node statistics of the analytical cut model:
compute_node_stats (streamcut/theory.py:97-122) on the GPU, bit-exact against
fixtures made by the real reference (tests/golden/golden_theory.json) and the
numpy restatement (oracle/theory_oracle.py); the reference tests' examples
(tests/test_theory.py:87-116) and error behaviour."""
import hashlib
import json
import os
from math import ceil

import numpy as np
import pytest

from helpers import random_multigraph, write_grpe
from oracle import theory_oracle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_theory.json")


def _sha(a):
    return hashlib.sha256(np.asarray(a, dtype="<i8").tobytes()).hexdigest()


def _inputs(case, bisect_fn):
    from paper_2502_17846_b200 import synth
    rng = np.random.default_rng(case["seed"])
    if case["kind"] == "random":
        edges, n = random_multigraph(rng, max_nodes=60, max_edges=800)
    else:
        n, m = 3000, 40000
        edges = synth.powerlaw_edges(n, m, seed=case["seed"]).astype(np.int64)
    if case["labels"] == "random":
        labels = rng.integers(0, 2, size=n)
    else:
        labels = bisect_fn(edges, n)
    labels = np.asarray(labels, dtype=np.int64)
    assert _sha(labels) == case["labels_sha256"]
    return edges, n, labels


def _oracle_bisect(edges, n):
    from oracle import oracle
    return oracle.bisect(edges, n, ceil(0.1 * len(edges)), ceil(n / 2))


def test_oracle_matches_reference_fixtures():
    for case in json.load(open(GOLD))["cases"]:
        edges, n, labels = _inputs(case, _oracle_bisect)
        k, k0 = theory_oracle.node_stats(edges, n, labels)
        assert _sha(k) == case["k_sha256"] and _sha(k0) == case["k0_sha256"], case
        assert int(k.sum()) == case["total_endpoints"]


@pytest.mark.gpu
def test_gpu_matches_reference_fixtures(tmp_path):
    from paper_2502_17846_b200 import GremConfig, compute_node_stats, grem
    from paper_2502_17846_b200.edgefile import open_edge_file

    def gpu_bisect(edges, n):
        return grem.bisect_edges(np.asarray(edges, dtype=np.uint32), n, GremConfig(chunk_frac=0.1))[0]

    for case in json.load(open(GOLD))["cases"]:
        edges, n, labels = _inputs(case, gpu_bisect)
        st = compute_node_stats(open_edge_file(write_grpe(tmp_path / "g.grpe", edges, n)), labels)
        assert _sha(st.k) == case["k_sha256"] and _sha(st.k0) == case["k0_sha256"], case
        assert st.total_endpoints == case["total_endpoints"]


@pytest.mark.gpu
def test_gpu_reference_examples_and_errors(tmp_path):
    from paper_2502_17846_b200 import FormatError, compute_node_stats
    from paper_2502_17846_b200.edgefile import open_edge_file
    tri = open_edge_file(write_grpe(tmp_path / "t.grpe", [[0, 1], [1, 2], [0, 2]], 3))
    st = compute_node_stats(tri, np.array([0, 0, 1]))           # test_theory.py:87-91
    assert st.k.tolist() == [2, 2, 2] and st.k0.tolist() == [1, 1, 2]
    star = open_edge_file(write_grpe(tmp_path / "s.grpe", [[0, i] for i in range(1, 6)], 6))
    st = compute_node_stats(star, np.array([1, 0, 0, 0, 0, 0]))  # test_theory.py:94-100
    assert (st.k[0], st.k0[0]) == (5, 5) and st.k[1:].tolist() == [1] * 5
    for bad in (np.array([0, 0]), np.array([0, 2, 1]), np.array([0, -1, 1])):
        with pytest.raises(FormatError):
            compute_node_stats(tri, bad)
    # self-loops are skipped even on unlabeled nodes; an unlabeled isolated node is fine
    g = open_edge_file(write_grpe(tmp_path / "l.grpe", [[2, 2], [0, 1], [0, 1]], 4))
    st = compute_node_stats(g, np.array([0, 1, -1, -1]))
    assert st.k.tolist() == [2, 2, 0, 0] and st.k0.tolist() == [2, 2, 0, 0]
    empty = open_edge_file(write_grpe(tmp_path / "e.grpe", np.empty((0, 2)), 3))
    st = compute_node_stats(empty, np.array([0, 1, 0]))
    assert st.k.tolist() == [0, 0, 0]


@pytest.mark.gpu
def test_gpu_random_and_large_vs_oracle():
    from paper_2502_17846_b200 import node_stats_edges, synth
    rng = np.random.default_rng(9)
    for _ in range(30):
        edges, n = random_multigraph(rng, max_nodes=200, max_edges=3000)
        lab = rng.integers(0, 2, size=n)
        st = node_stats_edges(edges, n, lab)
        k, k0 = theory_oracle.node_stats(edges, n, lab)
        assert np.array_equal(st.k, k) and np.array_equal(st.k0, k0)
    n, m = 2_000_000, 20_000_000
    edges = synth.powerlaw_edges(n, m, seed=5)
    lab = np.random.default_rng(5).integers(0, 2, size=n)
    st = node_stats_edges(edges, n, lab)
    k, k0 = theory_oracle.node_stats(edges, n, lab)
    assert np.array_equal(st.k, k) and np.array_equal(st.k0, k0)


@pytest.mark.gpu
def test_gpu_unpacked_fallback_matches():
    """The two-counter form (used when num_edges >= 2^32) gives the same stats:
    forced with GREM_NODE_STATS_UNPACKED in a subprocess (the switch is read once)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path[:0] = [%r, %r]\n"
            "import numpy as np\n"
            "from helpers import random_multigraph\n"
            "from oracle import theory_oracle\n"
            "from paper_2502_17846_b200 import node_stats_edges\n"
            "rng = np.random.default_rng(21)\n"
            "for _ in range(10):\n"
            "    e, n = random_multigraph(rng, max_nodes=300, max_edges=4000)\n"
            "    lab = rng.integers(0, 2, size=n)\n"
            "    st = node_stats_edges(e, n, lab)\n"
            "    k, k0 = theory_oracle.node_stats(e, n, lab)\n"
            "    assert np.array_equal(st.k, k) and np.array_equal(st.k0, k0)\n"
            "print('ok')\n") % (root, os.path.join(root, "tests"))
    env = dict(os.environ, GREM_NODE_STATS_UNPACKED="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.gpu
def test_gpu_file_front_end(tmp_path, monkeypatch):
    """compute_node_stats on a GRPE u32 file goes through grem_node_stats_file
    (overlapped reader, small pieces forced): equal to the array entry point
    and the oracle on a hub-sized case; an out-of-range id raises FormatError."""
    from paper_2502_17846_b200 import FormatError, compute_node_stats, node_stats_edges, synth
    from paper_2502_17846_b200.edgefile import open_edge_file
    monkeypatch.setenv("GREM_INGEST_PIECE", "100003")
    n, m = 300_000, 3_000_000
    edges = synth.powerlaw_edges(n, m, seed=8)
    lab = np.random.default_rng(8).integers(0, 2, size=n)
    st = compute_node_stats(open_edge_file(write_grpe(tmp_path / "p.grpe", edges, n)), lab)
    st2 = node_stats_edges(edges, n, lab)
    k, k0 = theory_oracle.node_stats(edges, n, lab)
    assert np.array_equal(st.k, k) and np.array_equal(st.k0, k0)
    assert np.array_equal(st2.k, k) and np.array_equal(st2.k0, k0)
    bad = edges.astype(np.int64)
    bad[m - 3] = (1, n + 7)
    with pytest.raises(FormatError):
        compute_node_stats(open_edge_file(write_grpe(tmp_path / "b.grpe", bad, n)), lab)
