"""expected_cuts / theory_curve (streamcut/theory.py:125-146): the GPU path
against fixtures made by streamcut itself (tests/golden/make_golden_curve.py)
and against the restatement in oracle/theory_oracle.py.

Tolerance: relative 1e-9.  Both sides sum the same log-gamma tail terms in
binary64; they differ in the log-gamma implementation (CPython's vs CUDA's,
a few ulps of values up to ~2.3e6 for k = 2e5, i.e. ~1e-9 absolute in a log
term) and in the summation order of the node totals."""
import os

import numpy as np
import pytest

from oracle import theory_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "golden_curve.npz"))
RTOL = 1e-9


def _stats(name):
    from paper_2502_17846_b200.theory import NodeStats
    return NodeStats(GOLD[f"{name}_k"], GOLD[f"{name}_k0"])


@pytest.mark.parametrize("name", [str(n) for n in GOLD["names"]])
def test_oracle_matches_reference_fixtures(name):
    k, k0 = GOLD[f"{name}_k"], GOLD[f"{name}_k0"]
    for a, mu in enumerate(GOLD["mults"]):
        for b, x in enumerate(GOLD["xs"]):
            got = O.expected_cuts(k, k0, float(x), float(mu))
            assert got == pytest.approx(float(GOLD[f"{name}_cuts"][a, b]), rel=1e-13, abs=1e-9)


def test_theory_curve_without_points_touches_nothing():
    from paper_2502_17846_b200 import theory_curve
    from paper_2502_17846_b200.theory import NodeStats
    assert theory_curve(NodeStats(np.zeros(0, np.int64), np.zeros(0, np.int64)), []) == []   # theory.py:146


def test_curve_csv_format():
    from paper_2502_17846_b200.theory import TheoryCurvePoint, curve_csv
    pts = [TheoryCurvePoint(0.1, 12.5, 0.25), TheoryCurvePoint(1.0, 3.0, 0.0625)]
    assert curve_csv(pts, 2.0) == ("x,expected_cuts,expected_cut_fraction,multiplier\n"
                                   "0.1,12.5,0.25,2.0\n1.0,3.0,0.0625,2.0\n")


@pytest.mark.gpu
@pytest.mark.parametrize("name", [str(n) for n in GOLD["names"]])
def test_gpu_curve_matches_reference_fixtures(name):
    from paper_2502_17846_b200 import expected_cuts, theory_curve
    st = _stats(name)
    total = int(np.asarray(st.k).sum())
    for a, mu in enumerate(GOLD["mults"]):
        pts = theory_curve(st, GOLD["xs"], float(mu))
        for b, x in enumerate(GOLD["xs"]):
            want = float(GOLD[f"{name}_cuts"][a, b])
            assert pts[b].x == float(x)
            assert pts[b].expected_cuts == pytest.approx(want, rel=RTOL, abs=1e-9), (name, mu, x)
            assert pts[b].expected_cut_fraction == pytest.approx(want / total, rel=RTOL)
        one = expected_cuts(st, float(GOLD["xs"][2]), float(mu))
        assert one.expected_cuts == pts[2].expected_cuts   # same kernels, same order


@pytest.mark.gpu
def test_gpu_curve_random_against_oracle():
    from paper_2502_17846_b200 import expected_cuts
    from paper_2502_17846_b200.theory import NodeStats
    rng = np.random.default_rng(7)
    for _ in range(20):
        n = int(rng.integers(1, 3000))
        k = rng.integers(0, int(rng.choice([5, 50, 3000])), size=n).astype(np.int64)
        k0 = np.minimum(k, (k + 1) // 2 + rng.integers(0, 20, size=n)).astype(np.int64)
        x = float(rng.choice([1e-4, 0.03, 0.3, 0.77, 1.0]))
        mu = float(rng.choice([1.0, 1.5, 4.0]))
        got = expected_cuts(NodeStats(k, k0), x, mu).expected_cuts
        assert got == pytest.approx(O.expected_cuts(k, k0, x, mu), rel=RTOL, abs=1e-9)


@pytest.mark.gpu
def test_gpu_curve_errors_in_reference_order():
    from paper_2502_17846_b200 import FormatError, expected_cuts, theory_curve
    from paper_2502_17846_b200.theory import NodeStats
    st = NodeStats(np.array([0, 3, 4]), np.array([0, 2, 2]))
    with pytest.raises(FormatError, match="empty node stats"):
        expected_cuts(NodeStats(np.zeros(0, np.int64), np.zeros(0, np.int64)), 0.5)
    with pytest.raises(FormatError, match=r"chunk fraction must be in \(0, 1\], got 0.0"):
        expected_cuts(st, 0.0)
    with pytest.raises(FormatError, match=r"chunk fraction must be in \(0, 1\], got 1.5"):
        theory_curve(st, [0.5, 1.5])
    with pytest.raises(FormatError, match="multiplier must be >= 1, got 0.5"):
        theory_curve(st, [0.5, 1.5], multiplier=0.5)   # the first point fails on the multiplier first
    # no node with k >= 1: nothing is evaluated, so no domain check (theory.py:133-135)
    zero = expected_cuts(NodeStats(np.zeros(4, np.int64), np.zeros(4, np.int64)), 7.0)
    assert zero.expected_cuts == 0.0 and zero.expected_cut_fraction == 0.0


@pytest.mark.gpu
def test_gpu_curve_on_node_stats_of_a_partition():
    """compute_node_stats -> theory_curve end to end on the GPU, vs the oracle."""
    from paper_2502_17846_b200 import node_stats_edges, theory_curve
    from oracle.gen_np import powerlaw_edges
    n, m = 20000, 300000
    e = powerlaw_edges(n, m, beta=11, seed=5)
    lab = np.random.default_rng(5).integers(0, 2, size=n).astype(np.int32)
    st = node_stats_edges(e, n, lab)
    pts = theory_curve(st, [0.02, 0.2, 1.0], 2.0)
    for p in pts:
        assert p.expected_cuts == pytest.approx(O.expected_cuts(st.k, st.k0, p.x, 2.0), rel=RTOL)
