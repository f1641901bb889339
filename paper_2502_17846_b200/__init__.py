"""B200-native GREM partitioner — a drop-in for the reference streamcut
package's GREM path (streamcut.grem.partition / bisect / count_cuts).

    from paper_2502_17846_b200 import bisect, partition, count_cuts, GremConfig

The entry points keep the reference's signatures, inputs (EdgeFile + config)
and outputs (int32 labels + CutReport); the work runs in hand-written sm_100a
CUDA kernels behind the C ABI in include/grem_b200.h (libgrem_b200.so).
``install_into_streamcut()`` rebinds the reference module's entry points so
existing callers (CLI, tests) use the GPU path unchanged.
"""

from .config import ChunkPlan, CutReport, GremConfig, SeedConfig, default_capacity
from .errors import CapacityError, DeviceError, FormatError, StreamcutError
from .theory import compute_node_stats, curve_csv, expected_cuts, node_stats_edges, theory_curve
from .shuffle import external_shuffle
from .grem import bisect, bisect_edges, count_cuts, last_stats, partition, partition_edges, set_device

__version__ = "0.1.0"


def install_into_streamcut(support: bool = False):
    """Swap streamcut's GREM entry points for the B200 ones (before callers
    bind them by name).  partition() inside streamcut resolves bisect through
    the grem module globals (grem.py:300), so rebinding grem.* covers
    recursion as well.  ``support=True`` also swaps the label consumers this
    package provides (store.write_buckets / reorder_features,
    theory.compute_node_stats / expected_cuts / theory_curve, edgefile.external_shuffle), everywhere the
    reference binds them (package, module, CLI)."""
    import importlib

    import streamcut  # type: ignore

    from . import store as _store

    swaps = {"bisect": bisect, "partition": partition, "count_cuts": count_cuts}
    mods = ["streamcut", "streamcut.grem", "streamcut.cli"]
    if support:
        swaps.update(compute_node_stats=compute_node_stats, expected_cuts=expected_cuts, theory_curve=theory_curve,
                     write_buckets=_store.write_buckets,
                     reorder_features=_store.reorder_features, external_shuffle=external_shuffle)
        mods += ["streamcut.theory", "streamcut.store", "streamcut.edgefile"]
    for name in mods:
        try:
            mod = importlib.import_module(name)
        except Exception:  # noqa: BLE001
            continue
        for attr, fn in swaps.items():
            if hasattr(mod, attr):
                setattr(mod, attr, fn)
    return streamcut


__all__ = [
    "bisect", "partition", "count_cuts", "bisect_edges", "partition_edges", "set_device", "last_stats",
    "GremConfig", "SeedConfig", "ChunkPlan", "CutReport", "default_capacity",
    "StreamcutError", "FormatError", "CapacityError", "DeviceError", "install_into_streamcut",
    "compute_node_stats", "node_stats_edges", "expected_cuts", "theory_curve", "curve_csv", "external_shuffle",
]
