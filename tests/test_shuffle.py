"""External shuffle: external_shuffle
(streamcut/edgefile.py:248-327) on the GPU.  The reference's order comes from
numpy's PCG64 Generator and is not reproduced; parity is what the reference's
own tests pin (tests/test_edgefile.py:87-135): the output is a permutation of
the input, byte-identical for a fixed seed, uniform over seeds (chi-squared),
and the budget errors match."""
import numpy as np
import pytest

from helpers import write_grpe



def _read(ef):
    from paper_2502_17846_b200.edgefile import edges_u32
    return edges_u32(ef).astype(np.int64)


def _multiset(a):
    a = np.asarray(a, dtype=np.int64).reshape(-1, 2)
    return a[np.lexsort((a[:, 1], a[:, 0]))]


@pytest.mark.gpu
def test_permutation_and_deterministic(tmp_path):
    from paper_2502_17846_b200 import external_shuffle
    from paper_2502_17846_b200.edgefile import open_edge_file
    edges = np.array([[i, (i + 1) % 10] for i in range(10)], dtype=np.int64)
    ef = open_edge_file(write_grpe(tmp_path / "g.grpe", edges, 10))
    out1 = external_shuffle(ef, str(tmp_path / "s1.grpe"), 1 << 20, rng_seed=42)
    external_shuffle(ef, str(tmp_path / "s2.grpe"), 1 << 20, rng_seed=42)
    s1 = _read(out1)
    assert np.array_equal(_multiset(s1), _multiset(edges))
    assert (tmp_path / "s1.grpe").read_bytes() == (tmp_path / "s2.grpe").read_bytes()
    out3 = external_shuffle(ef, str(tmp_path / "s3.grpe"), 1 << 20, rng_seed=43)
    assert _read(out3).shape == s1.shape
    assert out1.meta.num_nodes == 10 and out1.meta.num_edges == 10


@pytest.mark.gpu
def test_budget_errors_and_scatter_sized_input(tmp_path):
    from paper_2502_17846_b200 import FormatError, external_shuffle
    from paper_2502_17846_b200.edgefile import open_edge_file
    ef = open_edge_file(write_grpe(tmp_path / "g.grpe", [[0, 1]], 2))
    with pytest.raises(FormatError):
        external_shuffle(ef, str(tmp_path / "s.grpe"), 1024, rng_seed=0)   # test_edgefile.py:114-117
    rng = np.random.default_rng(9)
    edges = rng.integers(0, 300, size=(20000, 2)).astype(np.int64)
    ef = open_edge_file(write_grpe(tmp_path / "h.grpe", edges, 300))
    out = external_shuffle(ef, str(tmp_path / "t.grpe"), 1 << 16, rng_seed=1)   # :101-111
    sh = _read(out)
    assert np.array_equal(_multiset(sh), _multiset(edges)) and not np.array_equal(sh, edges)


def test_budget_rules_host():
    """The reference's budget arithmetic (edgefile.py:262-263, 271-275): below one
    I/O block, or more than 4096 scatter buckets of budget/2 bytes, is a FormatError."""
    from paper_2502_17846_b200 import FormatError
    from paper_2502_17846_b200.shuffle import IO_BLOCK, _check_budget
    _check_budget(600_000, IO_BLOCK)                 # 9.6 MB / 32 KB = 293 buckets
    _check_budget(10, 1 << 20)                       # in-memory path
    with pytest.raises(FormatError):
        _check_budget(9_000_000, IO_BLOCK)           # 4395 buckets
    with pytest.raises(FormatError):
        _check_budget(1, IO_BLOCK - 1)


@pytest.mark.gpu
def test_uniform_positions_chi_squared(tmp_path):
    """test_edgefile.py:120-135: where the first edge of a 10-edge file lands over 1000 seeds."""
    import scipy.stats
    from paper_2502_17846_b200 import external_shuffle
    from paper_2502_17846_b200.edgefile import open_edge_file
    edges = np.array([[i, (i + 1) % 10] for i in range(10)], dtype=np.int64)
    ef = open_edge_file(write_grpe(tmp_path / "g.grpe", edges, 10))
    counts = np.zeros(10, dtype=np.int64)
    for seed in range(1000):
        rows = _read(external_shuffle(ef, str(tmp_path / "s.grpe"), 1 << 20, rng_seed=seed))
        counts[int(np.flatnonzero((rows == edges[0]).all(axis=1))[0])] += 1
    expected = counts.sum() / 10
    stat = float(((counts - expected) ** 2 / expected).sum())
    assert stat < scipy.stats.chi2.ppf(0.99, df=9), counts


@pytest.mark.gpu
def test_large_wide_and_multi_piece(tmp_path, monkeypatch):
    """A 3M-edge power-law file (reader and writer in many pieces), a 64-bit-id
    file and an in-memory array: multiset preserved, seeds give different orders."""
    from paper_2502_17846_b200 import external_shuffle, synth
    from paper_2502_17846_b200.edgefile import open_edge_file
    monkeypatch.setenv("GREM_INGEST_PIECE", "65537")
    edges = synth.powerlaw_edges(200_000, 3_000_000, seed=4).astype(np.int64)
    ef = open_edge_file(write_grpe(tmp_path / "p.grpe", edges, 200_000))
    a = _read(external_shuffle(ef, str(tmp_path / "a.grpe"), 1 << 30, rng_seed=5))
    b = _read(external_shuffle(ef, str(tmp_path / "b.grpe"), 1 << 30, rng_seed=6))
    ms = _multiset(edges)
    assert np.array_equal(_multiset(a), ms) and np.array_equal(_multiset(b), ms)
    assert not np.array_equal(a, b) and not np.array_equal(a, edges)
    # position of each original edge is spread over the output (no locality left)
    assert abs(np.corrcoef(np.arange(len(a)) % 1000, a[:, 0] % 1000)[0, 1]) < 0.01
    efw = open_edge_file(write_grpe(tmp_path / "w.grpe", edges[:5000], 200_000, wide=True))
    outw = external_shuffle(efw, str(tmp_path / "w2.grpe"), 1 << 20, rng_seed=7)
    assert outw.meta.node_id_width == 64
    assert np.array_equal(_multiset(_read(outw)), _multiset(edges[:5000]))
