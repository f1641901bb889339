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
from .theory import compute_node_stats, node_stats_edges
from .shuffle import external_shuffle
from .grem import bisect, bisect_edges, count_cuts, last_stats, partition, partition_edges, set_device

__version__ = "0.1.0"


def install_into_streamcut():
    """Swap streamcut's GREM entry points for the B200 ones (before callers
    bind them by name).  partition() inside streamcut resolves bisect through
    the grem module globals (grem.py:300), so rebinding grem.* covers
    recursion as well."""
    import streamcut  # type: ignore
    import streamcut.grem as sg  # type: ignore

    for mod in (streamcut, sg):
        mod.bisect = bisect
        mod.partition = partition
        mod.count_cuts = count_cuts
    streamcut.compute_node_stats = compute_node_stats
    try:
        import streamcut.theory as st  # type: ignore

        st.compute_node_stats = compute_node_stats
    except Exception:  # noqa: BLE001
        pass
    try:
        import streamcut.cli as cli  # type: ignore

        cli.partition = partition
        cli.count_cuts = count_cuts
    except Exception:  # noqa: BLE001
        pass
    return streamcut


__all__ = [
    "bisect", "partition", "count_cuts", "bisect_edges", "partition_edges", "set_device", "last_stats",
    "GremConfig", "SeedConfig", "ChunkPlan", "CutReport", "default_capacity",
    "StreamcutError", "FormatError", "CapacityError", "DeviceError", "install_into_streamcut",
    "compute_node_stats", "node_stats_edges", "external_shuffle",
]
