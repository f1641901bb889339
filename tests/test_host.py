"""CPU: the C-ABI library loads and exports every symbol of include/grem_b200.h
(no compute calls), the deterministic generator, host-side config/report
mirrors, and the clamp algebra the sizes scan relies on."""
import ctypes
import hashlib
import os
import re
from math import ceil

import numpy as np
import pytest

from conftest import ROOT, have_streamcut
from paper_2502_17846_b200 import _abi, synth
from paper_2502_17846_b200.config import ChunkPlan, GremConfig, SeedConfig, default_capacity, make_report
from paper_2502_17846_b200.errors import CapacityError, FormatError


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_abi.LIB_PATH)
    header = open(os.path.join(ROOT, "include", "grem_b200.h")).read()
    declared = set(re.findall(r"\b(grem_[a-z0-9_]+)\s*\(", header))
    declared -= {"grem_seed_fn", "grem_chunk_fn", "grem_meter_fn"}
    assert declared, "no declarations parsed"
    for name in sorted(declared):
        getattr(lib, name)   # raises AttributeError if missing
    assert declared <= set(_abi.EXPORTS)


def test_product_path_has_no_oracle_dependency():
    """The product never imports, links or calls the checker (oracle/)."""
    pkg = os.path.join(ROOT, "paper_2502_17846_b200")
    bad = re.compile(r"^\s*(from\s+oracle|import\s+oracle)|\boracle\.|\boracle_[a-z]+\s*\(|grem_oracle", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h", "Makefile")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not bad.search(txt), f
    assert "oracle" not in open(os.path.join(pkg, "csrc", "Makefile")).read()


def test_generator_deterministic_and_in_range():
    a = synth.powerlaw_edges(10_000, 50_000, seed=3, threads=1)
    b = synth.powerlaw_edges(10_000, 50_000, seed=3, threads=4)
    assert np.array_equal(a, b)
    assert a.max() < 10_000
    # a window of the stream equals the same edges generated from an offset
    c = synth.powerlaw_edges(10_000, 1_000, seed=3, e0=20_000)
    assert np.array_equal(a[20_000:21_000], c)
    # heavy-tailed degrees, duplicates and self-loops present
    deg = np.bincount(a.reshape(-1), minlength=10_000)
    assert deg.max() > 50 * deg.mean()
    assert (a[:, 0] == a[:, 1]).any()


def test_generator_pinned_hash(golden_dir):
    import json
    shapes = json.load(open(os.path.join(golden_dir, "golden_shapes.json")))
    e = synth.shape_edges("tiny")
    assert hashlib.sha256(e.tobytes()).hexdigest() == shapes["tiny_k4"]["edges_sha256"]


def test_config_mirror_validation():
    with pytest.raises(FormatError):
        GremConfig(chunk_edges=5, chunk_frac=0.1)
    with pytest.raises(FormatError):
        GremConfig(capacity_slack=-0.1)
    with pytest.raises(FormatError):
        GremConfig(passes=0)
    with pytest.raises(FormatError):
        SeedConfig(algorithm="metis")
    with pytest.raises(FormatError):
        ChunkPlan.plan(10, chunk_frac=1.5)
    assert ChunkPlan.plan(1_166_243, chunk_frac=0.1) == ChunkPlan(116_625, 10)
    assert ChunkPlan.plan(0, chunk_edges=3) == ChunkPlan(3, 0)
    assert default_capacity(111_059_956 * 2, 0.1) == ceil((1.0 + 0.1) * 111_059_956 * 2 / 2)
    assert issubclass(CapacityError, Exception)


@pytest.mark.skipif(not have_streamcut(), reason="reference package not importable here")
def test_report_floats_match_reference(tmp_path):
    import streamcut
    from streamcut import BinaryEdgeWriter, open_edge_file
    rng = np.random.default_rng(5)
    for _ in range(20):
        n = int(rng.integers(2, 50))
        e = rng.integers(0, n, size=(int(rng.integers(1, 300)), 2))
        lab = rng.integers(0, int(rng.integers(1, 9)), size=n)
        p = str(tmp_path / "g.grpe")
        with BinaryEdgeWriter(p, n) as w:
            w.write(e)
        rep = streamcut.count_cuts(open_edge_file(p), lab)
        mine = make_report(n, len(e), rep.cut_edges, np.bincount(lab, minlength=int(lab.max()) + 1))
        assert mine == rep


# ------------------------------------------- clamp algebra of the sizes scan
INF = 1 << 60


def clampv(v, lo, hi):
    return lo if v < lo else (hi if v > hi else v)


def then(a, b):
    return (a[0] + b[0], clampv(a[1] + b[0], b[1], b[2]), clampv(a[2] + b[0], b[1], b[2]))


def apply(f, x):
    return clampv(x + f[0], f[1], f[2])


def test_clamp_composition_is_associative_and_exact():
    rng = np.random.default_rng(0)
    for _ in range(2000):
        fs = []
        for _ in range(3):
            d = int(rng.integers(-3, 4))
            lo = int(rng.integers(-20, 20)) if rng.random() < 0.7 else -INF
            hi = lo + int(rng.integers(0, 20)) if lo != -INF and rng.random() < 0.7 else INF
            fs.append((d, lo, hi))
        a, b, c = fs
        assert then(then(a, b), c) == then(a, then(b, c))
        for x in range(-30, 30):
            assert apply(then(a, b), x) == apply(b, apply(a, x))



def _assign(c0, c1, sizes, cap):   # grem.py:100-116
    if c0 < c1 and sizes[1] < cap:
        return 1
    if c1 < c0 and sizes[0] < cap:
        return 0
    if sizes[0] <= sizes[1]:
        assert sizes[0] < cap
        return 0
    assert sizes[1] < cap
    return 1


def test_node_maps_match_assign_exhaustive():
    for cap in range(1, 9):
        for x in range(0, cap + 1):
            for y in range(0, cap + 1):
                for old in (-1, 0, 1):
                    if old == 0 and x == 0 or old == 1 and y == 0:
                        continue
                    xl, yl = x - (old == 0), y - (old == 1)
                    if xl >= cap and yl >= cap:
                        continue
                    sl = xl + yl
                    o = 1 if old == 0 else 0
                    for pref, (c0, c1) in ((0, (2.0, 1.0)), (1, (1.0, 2.0)), (2, (1.0, 1.0))):
                        b = _assign(c0, c1, [xl, yl], cap)
                        t = cap - 1 if pref == 0 else (sl - cap if pref == 1 else sl // 2)
                        assert b == (0 if x - o <= t else 1)
                        xn = xl + (b == 0)
                        if pref == 0:
                            f = (1 - o, -INF, cap)
                        elif pref == 1:
                            f = (-o, sl - cap + 1, INF)
                        else:
                            # tie speculated as the clamp of the guessed side
                            # (grem_core.cuh node_map): exact on its region
                            for guess in (0, 1):
                                f = (1 - o, -INF, t + 1) if guess == 0 else (-o, t + 1, INF)
                                exact = (x - o <= t + 1) if guess == 0 else (x - o >= t)
                                if exact:
                                    assert apply(f, x) == xn
                            continue
                        assert apply(f, x) == xn


def test_bench_shapes_match_package_shapes():
    import bench
    from paper_2502_17846_b200 import synth
    for name, s in synth.SHAPES.items():
        assert bench.SHAPES[name] == (s.num_nodes, s.num_edges, s.k, s.beta, s.seed)


def test_reference_arm_loads_no_product_code():
    """bench.py --impl reference: streamcut on a bounded sample whose input
    comes from the numpy generator; the product package and its .so are never
    loaded (the arm's native_so_loaded listed libgrem_b200.so)."""
    import subprocess
    import sys
    code = r'''
import io, json, os, sys, contextlib
sys.argv = ["bench.py", "--impl", "reference", "--workload", "tiny", "--steps", "1", "--warmup", "0"]
import bench
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    bench.main()
line = json.loads(buf.getvalue().strip().splitlines()[-1])
maps = open("/proc/self/maps").read()
assert "libgrem_b200" not in maps, "product library loaded"
assert not any(m.startswith("paper_2502_17846_b200") for m in sys.modules), "product package imported"
assert line["impl"] == "reference" and line["value"] > 0 and line["config"]["k"] == 4
print("ok", line["cpu_baseline"]["kind"])
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
