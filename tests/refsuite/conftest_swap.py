"""conftest.py for the reference's own test suite run against the drop-in.

``__graft_entry__.build()`` copies the reference tests
(/root/reference/pkg/tests) next to the reference install under
baseline/_ref/streamcut_tests/ (git-ignored; it travels to the GPU box) and
installs this file there as conftest.py.  pytest imports it before it
collects the test modules, so their ``from streamcut import bisect, partition,
...`` (tests/test_grem.py:6-24, tests/test_acceptance.py:18-38) already bind
the B200 entry points.
"""
import os
import sys

ROOT = os.environ["GREM_REPO_ROOT"]
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

import streamcut  # noqa: E402

import paper_2502_17846_b200 as _b200  # noqa: E402

_b200.install_into_streamcut(support=os.environ.get("GREM_SWAP_SUPPORT", "1") == "1")
assert streamcut.bisect is _b200.bisect and streamcut.grem.partition is _b200.partition
_b200.grem.set_device(int(os.environ.get("GREM_DEVICE", "0")))


def pytest_report_header(config):
    return "streamcut GREM entry points swapped for paper_2502_17846_b200 (B200 CUDA path)"
