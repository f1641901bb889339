"""The BASELINE configs the round-1 goldens left open:

* the Friendster-shaped k = 4..256 sweep (BASELINE.json config 5) — deep
  recursion (255 bisections at k=256), seed restarts and hundreds of tiny
  sparse bisections;
* the frac = 0.01 secondary sweep at products / papers scale;
* arxiv-shaped k = 64 / 256.

Goldens (tests/golden/big/*.json, made by tests/golden/make_golden_big.py):
streamcut itself where it runs in minutes (arxiv, products), the C oracle
(pinned to streamcut by tests/test_oracle.py) at Friendster / papers scale.
Edges are generated on the device (bit-identical to the host generator).
Each case also records the device-pool HBM high-water mark of the call.
"""
import ctypes
import glob
import json
import os

import pytest

from helpers import labels_sha
from paper_2502_17846_b200 import GremConfig, _abi, grem, synth

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _cases():
    out = {}
    for f in sorted(glob.glob(os.path.join(HERE, "golden", "big", "*.json"))):
        out.update(json.load(open(f)))
    return out


CASES = _cases()
_dev = {}


def _device_edges(shape):
    """Device-resident edge list of a benchmark shape (kept for the module)."""
    if shape not in _dev:
        for k in list(_dev):
            _abi.lib().grem_device_free(grem.context(), _dev.pop(k))
        assert _abi.lib().grem_trim(grem.context()) == 0   # the previous shape's workspaces
        s = synth.SHAPES[shape]
        ptr = ctypes.c_void_p()
        L = _abi.lib()
        assert L.grem_device_alloc(grem.context(), s.num_edges * 8, ctypes.byref(ptr)) == 0
        assert L.grem_gen_edges_device(grem.context(), s.num_nodes, s.beta, s.seed, 0, s.num_edges, ptr) == 0
        _dev[shape] = ptr
    return _dev[shape]


@pytest.fixture(scope="module", autouse=True)
def _free_edges():
    yield
    for k in list(_dev):
        _abi.lib().grem_device_free(grem.context(), _dev.pop(k))


@pytest.mark.parametrize("key", sorted(CASES, key=lambda k: (CASES[k]["shape"], CASES[k]["k"])))
def test_sweep_golden(key):
    g = CASES[key]
    s = synth.SHAPES[g["shape"]]
    ptr = _device_edges(g["shape"])
    L = _abi.lib()
    used, res = ctypes.c_int64(), ctypes.c_int64()
    L.grem_mem_high_water(grem.context(), None, None, 1)
    cfg = GremConfig(chunk_frac=g["chunk_frac"], capacity_slack=g.get("capacity_slack", 0.0))
    lab, rep = grem.partition_edges(None, s.num_nodes, g["k"], cfg, on_device_ptr=ptr.value,
                                    num_edges=s.num_edges)
    st = grem.last_stats()
    assert L.grem_mem_high_water(grem.context(), ctypes.byref(used), ctypes.byref(res), 0) == 0
    print(f"[sweep] {key}: {st['ms_total']:.1f} ms, {st['bisections']} bisections, {st['rounds']} rounds, "
          f"pool HBM high water {used.value / 2**30:.2f} GiB used / {res.value / 2**30:.2f} GiB reserved "
          f"(+ {s.num_edges * 8 / 2**30:.2f} GiB caller-owned edges)")
    assert labels_sha(lab) == g["labels_sha256"]
    assert rep.cut_edges == g["cut_edges"] and list(rep.partition_sizes) == g["partition_sizes"]
    assert rep.balance_ratio == g["balance_ratio"]
