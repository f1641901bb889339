"""ctypes binding of libgrem_b200.so (include/grem_b200.h).

The library is built in-tree by __graft_entry__.build() (csrc/Makefile).  There
is no CPU fallback: if the shared object is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
# GREM_LIB: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("GREM_LIB") or os.path.join(_HERE, "libgrem_b200.so")
CSRC = os.path.join(_HERE, "csrc")
_lib = None

c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_u32 = ctypes.c_uint32
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p


class GremConfigC(ctypes.Structure):
    _fields_ = [("chunk_edges", c_i64), ("chunk_frac", c_dbl), ("capacity_slack", c_dbl),
                ("refine", ctypes.c_int32), ("passes", ctypes.c_int32), ("seed_algo", ctypes.c_int32),
                ("seed_refinement_passes", ctypes.c_int32)]


class GremReportC(ctypes.Structure):
    _fields_ = [("total_edges", c_i64), ("cut_edges", c_i64), ("num_parts", c_i64),
                ("partition_sizes", ctypes.POINTER(c_i64)), ("sizes_cap", c_i64)]


SEED_FN = ctypes.CFUNCTYPE(c_int, c_i64, ctypes.POINTER(ctypes.c_int8), c_vp)
CHUNK_FN = ctypes.CFUNCTYPE(c_int, ctypes.POINTER(c_i64), c_vp)
METER_FN = ctypes.CFUNCTYPE(None, c_i64, c_vp)


class GremHooksC(ctypes.Structure):
    _fields_ = [("seed", SEED_FN), ("on_chunk", CHUNK_FN), ("meter", METER_FN), ("user", c_vp)]


class GremStatsC(ctypes.Structure):
    _fields_ = [("chunks", c_i64), ("rounds", c_i64), ("max_rounds", c_i64), ("visits", c_i64),
                ("walk_steps", c_i64), ("seed_bfs_levels", c_i64), ("bisections", c_i64),
                ("kernels", c_i64), ("ms_total", c_dbl), ("count_bytes", c_i64), ("path_bytes", c_i64),
                ("delta_bytes", c_i64)]


# every exported symbol of include/grem_b200.h (tests check they all resolve)
EXPORTS = [
    "grem_create", "grem_destroy", "grem_last_error", "grem_get_stats", "grem_set_profiling",
    "grem_get_phase_times", "grem_get_phase_bytes", "grem_mem_high_water", "grem_trim", "grem_bucket_edges",
    "grem_bisect_u32", "grem_partition_u32", "grem_partition_shard_u32", "grem_staged_edges", "grem_count_cuts_u32",
    "grem_write_buckets_u32", "grem_write_buckets_file", "grem_reorder_records", "grem_node_stats_u32", "grem_shuffle_u32", "grem_shuffle_file", "grem_node_stats_file", "grem_theory_curve",
    "grem_bisect_file", "grem_partition_file", "grem_count_cuts_file", "grem_state_parts",
    "grem_device_alloc", "grem_device_free", "grem_memcpy_h2d", "grem_memcpy_d2h",
    "grem_gen_scale", "grem_gen_edges_host", "grem_gen_edges_device",
]


def build(force: bool = False) -> str:
    cmd = ["make", "-s", "-C", CSRC]
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    subprocess.run(cmd, check=True)
    return LIB_PATH


class _Missing:
    def __init__(self, name):
        self.name = name

    def __call__(self, *a, **k):
        raise RuntimeError(f"libgrem_b200.so does not export {self.name}")


def _declare(L):
    for name in EXPORTS:
        try:
            getattr(L, name)
        except AttributeError:
            setattr(L, name, _Missing(name))
    P = ctypes.POINTER
    L.grem_create.argtypes = [c_int]
    L.grem_create.restype = c_vp
    L.grem_destroy.argtypes = [c_vp]
    L.grem_destroy.restype = None
    L.grem_last_error.argtypes = []
    L.grem_last_error.restype = ctypes.c_char_p
    L.grem_get_stats.argtypes = [c_vp, P(GremStatsC)]
    L.grem_set_profiling.argtypes = [c_vp, c_int]
    L.grem_get_phase_times.argtypes = [c_vp, c_vp, c_vp, c_int, c_vp]
    L.grem_get_phase_bytes.argtypes = [c_vp, c_vp, c_int]
    L.grem_mem_high_water.argtypes = [c_vp, c_vp, c_vp, c_int]
    L.grem_trim.argtypes = [c_vp]
    L.grem_bucket_edges.argtypes = [c_vp, c_vp, c_i64, c_i64]
    L.grem_bisect_u32.argtypes = [c_vp, c_vp, c_i64, c_i64, c_int, P(GremConfigC), c_i64,
                                  P(GremHooksC), c_vp, P(GremReportC)]
    L.grem_partition_u32.argtypes = [c_vp, c_vp, c_i64, c_i64, c_int, c_i64, P(GremConfigC),
                                     P(GremHooksC), c_vp, P(GremReportC)]
    L.grem_count_cuts_u32.argtypes = [c_vp, c_vp, c_i64, c_i64, c_int, c_vp, c_int, P(GremReportC)]
    L.grem_partition_shard_u32.argtypes = [c_vp, c_vp, c_i64, c_i64, c_int, c_i64, P(GremConfigC), c_int, c_int,
                                           c_vp]
    L.grem_staged_edges.argtypes = [c_vp, P(c_vp), P(c_i64)]
    L.grem_write_buckets_u32.argtypes = [c_vp, c_vp, c_i64, c_i64, c_int, c_vp, c_int, c_vp, c_int, c_vp, c_i64,
                                         P(c_i64)]
    L.grem_node_stats_u32.argtypes = [c_vp, c_vp, c_i64, c_i64, c_int, c_vp, c_int, c_vp, c_vp]
    L.grem_node_stats_file.argtypes = [c_vp, ctypes.c_char_p, c_vp, c_int, c_vp, c_vp]
    L.grem_theory_curve.argtypes = [c_vp, c_vp, c_vp, c_i64, c_int, c_vp, c_i64, ctypes.c_double, c_vp, c_vp]
    L.grem_write_buckets_file.argtypes = [c_vp, ctypes.c_char_p, c_vp, c_int, c_vp, c_int, c_vp, c_i64, P(c_i64)]
    L.grem_shuffle_u32.argtypes = [c_vp, c_vp, c_i64, c_i64, c_int, ctypes.c_uint64, c_vp, c_int]
    L.grem_shuffle_file.argtypes = [c_vp, ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p]
    L.grem_reorder_records.argtypes = [c_vp, c_vp, c_i64, c_int, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, P(c_i64)]
    L.grem_count_cuts_file.argtypes = [c_vp, ctypes.c_char_p, c_vp, c_int, P(GremReportC)]
    L.grem_bisect_file.argtypes = [c_vp, ctypes.c_char_p, P(GremConfigC), c_i64, P(GremHooksC), c_vp,
                                   P(GremReportC)]
    L.grem_partition_file.argtypes = [c_vp, ctypes.c_char_p, c_i64, P(GremConfigC), P(GremHooksC), c_vp,
                                      P(GremReportC)]
    L.grem_state_parts.argtypes = [c_vp, c_vp, c_i64]
    L.grem_device_alloc.argtypes = [c_vp, c_u64, P(c_vp)]
    L.grem_device_free.argtypes = [c_vp, c_vp]
    L.grem_memcpy_h2d.argtypes = [c_vp, c_vp, c_vp, c_u64]
    L.grem_memcpy_d2h.argtypes = [c_vp, c_vp, c_vp, c_u64]
    L.grem_gen_scale.argtypes = [c_u64, c_u32]
    L.grem_gen_scale.restype = c_dbl
    L.grem_gen_edges_host.argtypes = [c_u64, c_u32, c_u64, c_u64, c_u64, c_vp, c_int]
    L.grem_gen_edges_device.argtypes = [c_vp, c_u64, c_u32, c_u64, c_u64, c_u64, c_vp]
    for name in EXPORTS:
        if name not in ("grem_create", "grem_destroy", "grem_last_error", "grem_gen_scale"):
            getattr(L, name).restype = c_int
    return L


def lib():
    """The loaded library; raises if it was not built (no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        _lib = _declare(ctypes.CDLL(LIB_PATH))
    return _lib


def last_error() -> str:
    return (lib().grem_last_error() or b"").decode()
