"""Configuration and value types of the GREM path, mirroring the reference
names and validation so the drop-in accepts the same arguments:

  SeedConfig   streamcut/seed.py:23-33
  GremConfig   streamcut/grem.py:45-75  (plan_for -> ChunkPlan.plan, edgefile.py:330-349)
  CutReport    streamcut/model.py:115-132
  default_capacity  streamcut/grem.py:78-79

Objects of the reference's own classes are accepted too (duck typing on the
same attribute names).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from math import ceil

from .errors import FormatError

ALGORITHMS = ("bfs_grow", "random")


@dataclass(frozen=True)
class SeedConfig:
    algorithm: str = "bfs_grow"
    refinement_passes: int = 2  # bfs_grow only
    rng_seed: int = 0

    def __post_init__(self):
        if self.algorithm not in ALGORITHMS:
            raise FormatError(f"unknown seed algorithm {self.algorithm!r}")
        if self.refinement_passes < 0:
            raise FormatError("refinement_passes must be >= 0")


@dataclass(frozen=True)
class ChunkPlan:
    chunk_size: int
    num_chunks: int

    @staticmethod
    def plan(num_edges: int, chunk_edges: int | None = None, chunk_frac: float | None = None) -> "ChunkPlan":
        if (chunk_edges is None) == (chunk_frac is None):
            raise FormatError("specify exactly one of chunk_edges / chunk_frac")
        if chunk_frac is not None:
            if not 0 < chunk_frac <= 1:
                raise FormatError(f"chunk_frac must be in (0, 1], got {chunk_frac}")
            chunk_edges = max(1, ceil(chunk_frac * num_edges))
        if chunk_edges < 1:
            raise FormatError(f"chunk_size must be >= 1, got {chunk_edges}")
        return ChunkPlan(chunk_edges, ceil(num_edges / chunk_edges) if num_edges else 0)


@dataclass(frozen=True)
class GremConfig:
    chunk_edges: int | None = None
    chunk_frac: float | None = None
    capacity_slack: float = 0.0
    refine: bool = True
    seed: SeedConfig = field(default_factory=SeedConfig)
    passes: int = 1

    def __post_init__(self):
        if self.chunk_edges is not None and self.chunk_frac is not None:
            raise FormatError("set chunk_edges or chunk_frac, not both")
        if self.capacity_slack < 0:
            raise FormatError("capacity_slack must be >= 0")
        if self.passes < 1:
            raise FormatError("passes must be >= 1")

    def plan_for(self, num_edges: int) -> ChunkPlan:
        return plan_for(self, num_edges)


def plan_for(config, num_edges: int) -> ChunkPlan:
    if config.chunk_edges is None and config.chunk_frac is None:
        return ChunkPlan.plan(num_edges, chunk_frac=0.1)
    return ChunkPlan.plan(num_edges, config.chunk_edges, config.chunk_frac)


def default_capacity(num_nodes: int, slack: float = 0.0) -> int:
    return ceil((1.0 + slack) * num_nodes / 2)


try:  # reuse the reference's report type when present, so reports compare equal
    from streamcut.model import CutReport  # type: ignore
except Exception:  # noqa: BLE001
    @dataclass(frozen=True)
    class CutReport:
        total_edges: int
        cut_edges: int
        cut_fraction: float
        partition_sizes: tuple
        balance_ratio: float

        def to_dict(self) -> dict:
            return {
                "total_edges": self.total_edges,
                "cut_edges": self.cut_edges,
                "cut_fraction": self.cut_fraction,
                "partition_sizes": list(self.partition_sizes),
                "balance_ratio": self.balance_ratio,
            }


def make_report(num_nodes: int, total: int, cut: int, sizes) -> "CutReport":
    """The float fields exactly as count_cuts derives them (grem.py:241-252)."""
    sizes = tuple(int(s) for s in sizes)
    num_parts = len(sizes)
    ideal = ceil(num_nodes / num_parts)
    return CutReport(
        total_edges=int(total),
        cut_edges=int(cut),
        cut_fraction=cut / total if total else 0.0,
        partition_sizes=sizes,
        balance_ratio=float(max(sizes)) / ideal,
    )
