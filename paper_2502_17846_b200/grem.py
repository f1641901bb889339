"""Drop-in GREM entry points on B200 (streamcut/grem.py:192-319).

    bisect(efile, config, *, capacity=None, meter=None, on_chunk=None, prefetch=False)
        -> (np.int32[n] in {0,1}, CutReport)                     grem.py:192-224
    partition(efile, p, config, workdir, *, meter=None)
        -> (np.int32[n] in [0,p), CutReport)                     grem.py:277-319
    count_cuts(efile, labels) -> CutReport                       grem.py:227-252

Same names, argument meaning, results (bit-identical labels; exact integer
report fields, float fields from the same expressions) and error classes as the
reference.  The work runs in libgrem_b200.so on the GPU; there is no CPU
fallback — a missing library or GPU raises.
"""

from __future__ import annotations

import ctypes
import os
from math import ceil

import numpy as np

from . import _abi
from .config import ChunkPlan, default_capacity, make_report, plan_for
from .edgefile import edges_u32, is_native_binary
from .errors import CapacityError, DeviceError, FormatError, StreamcutError

_CODES = {1: FormatError, 2: CapacityError, 3: DeviceError, 4: DeviceError, 5: StreamcutError}

_ctx = {}
_device = None


def set_device(device: int) -> None:
    """Select the CUDA device used by subsequent calls (default: LOCAL_RANK or 0)."""
    global _device
    _device = int(device)


def _current_device() -> int:
    if _device is not None:
        return _device
    return int(os.environ.get("GREM_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def context():
    """Native context (stream, device workspaces) of the current device."""
    dev = _current_device()
    c = _ctx.get(dev)
    if c is None:
        c = _abi.lib().grem_create(dev)
        if not c:
            raise DeviceError(f"cannot create a GREM context on cuda:{dev}: {_abi.last_error()}")
        _ctx[dev] = c
    return c


def _host_labels(n: int) -> np.ndarray:
    """Label output buffer in page-locked memory (torch's caching host
    allocator, reused across calls) so the device->host copy of the labels
    runs at DMA speed; the array keeps its block alive."""
    if n >= (1 << 20):
        try:
            import torch
            if torch.cuda.is_available():
                return torch.empty(n, dtype=torch.int32, pin_memory=True).numpy()
        except Exception:  # noqa: BLE001
            pass
    return np.empty(n, dtype=np.int32)


def _raise(rc: int, pending=None):
    if pending:
        raise pending[0]
    if rc:
        raise _CODES.get(rc, StreamcutError)(_abi.last_error())


def _cfg_struct(config, chunk_edges_abs: int | None):
    seed = getattr(config, "seed", None)
    algo = getattr(seed, "algorithm", "bfs_grow")
    c = _abi.GremConfigC()
    if chunk_edges_abs is not None:
        c.chunk_edges = int(chunk_edges_abs)
        c.chunk_frac = 0.0
    elif config.chunk_edges is not None:
        c.chunk_edges = int(config.chunk_edges)
        c.chunk_frac = 0.0
    else:
        c.chunk_edges = 0
        c.chunk_frac = float(config.chunk_frac if config.chunk_frac is not None else 0.1)
    c.capacity_slack = float(config.capacity_slack)
    c.refine = 1 if config.refine else 0
    c.passes = int(config.passes)
    c.seed_algo = 1 if algo == "random" else 0
    c.seed_refinement_passes = int(getattr(seed, "refinement_passes", 2))
    return c


class _StateProxy:
    """What on_chunk(state) sees (PartitionState, model.py:79-112): live sizes
    always; parts / recount_sizes() copy the device labels on demand."""

    def __init__(self, ctx, num_nodes: int, capacity: int):
        self._ctx = ctx
        self._n = num_nodes
        self.capacity = int(capacity)
        self.sizes = [0, 0]

    @property
    def num_nodes(self) -> int:
        return self._n

    def labels_array(self) -> np.ndarray:
        out = np.empty(self._n, dtype=np.int32)
        rc = _abi.lib().grem_state_parts(self._ctx, out.ctypes.data, self._n)
        _raise(rc)
        return out

    @property
    def parts(self) -> list:
        return self.labels_array().tolist()

    def recount_sizes(self) -> list:
        lab = self.labels_array()
        return [int((lab == 0).sum()), int((lab == 1).sum())]


def _hooks(config, meter=None, on_chunk=None, state=None):
    pending = []
    seed = getattr(config, "seed", None)

    def seed_cb(nn, out, user):
        try:   # seed_bisect(..., "random"), seed.py:48-52
            rng = np.random.default_rng(getattr(seed, "rng_seed", 0))
            labels = np.ones(nn, dtype=np.int8)
            labels[rng.permutation(nn)[: ceil(nn / 2)]] = 0
            ctypes.memmove(out, labels.ctypes.data, nn)
            return 0
        except BaseException as exc:  # noqa: BLE001
            pending.append(exc)
            return 1

    def chunk_cb(sizes, user):
        try:
            state.sizes = [int(sizes[0]), int(sizes[1])]
            on_chunk(state)
            return 0
        except BaseException as exc:  # noqa: BLE001
            pending.append(exc)
            return 1

    def meter_cb(delta, user):
        try:
            if delta >= 0:
                meter.acquire(int(delta))
            else:
                meter.release(int(-delta))
        except BaseException as exc:  # noqa: BLE001
            pending.append(exc)

    h = _abi.GremHooksC()
    keep = []
    if getattr(seed, "algorithm", "bfs_grow") == "random":
        f = _abi.SEED_FN(seed_cb)
        keep.append(f)
        h.seed = f
    if on_chunk is not None:
        f = _abi.CHUNK_FN(chunk_cb)
        keep.append(f)
        h.on_chunk = f
    if meter is not None:
        f = _abi.METER_FN(meter_cb)
        keep.append(f)
        h.meter = f
    return h, keep, pending


def _report_struct(cap: int):
    sizes = (ctypes.c_int64 * cap)()
    r = _abi.GremReportC()
    r.partition_sizes = ctypes.cast(sizes, ctypes.POINTER(ctypes.c_int64))
    r.sizes_cap = cap
    return r, sizes


def _report(num_nodes: int, r, sizes) -> "CutReport":
    return make_report(num_nodes, r.total_edges, r.cut_edges, [sizes[k] for k in range(r.num_parts)])


def bisect(efile, config, *, capacity=None, meter=None, on_chunk=None, prefetch: bool = False):
    """grem.py:192-224.  ``prefetch`` is accepted for signature parity; the
    native ingest always double-buffers and results never depend on it."""
    meta = efile.meta
    n = int(meta.num_nodes)
    cap = capacity if capacity is not None else default_capacity(n, config.capacity_slack)
    if 2 * cap < n:
        raise CapacityError(f"capacity {cap} cannot hold {n} nodes across two parts")
    plan = plan_for(config, int(meta.num_edges))
    ctx = context()
    L = _abi.lib()
    state = _StateProxy(ctx, n, cap) if on_chunk is not None else None
    hooks, keep, pending = _hooks(config, meter, on_chunk, state)
    cfg = _cfg_struct(config, plan.chunk_size)
    labels = _host_labels(n)
    rep, sizes = _report_struct(2)
    if is_native_binary(efile):
        rc = L.grem_bisect_file(ctx, os.fsencode(efile.path), ctypes.byref(cfg), int(cap), ctypes.byref(hooks),
                                labels.ctypes.data, ctypes.byref(rep))
    else:
        e = edges_u32(efile)
        rc = L.grem_bisect_u32(ctx, e.ctypes.data, e.shape[0], n, 0, ctypes.byref(cfg), int(cap),
                               ctypes.byref(hooks), labels.ctypes.data, ctypes.byref(rep))
    del keep
    _raise(rc, pending)
    return labels, _report(n, rep, sizes)


def partition(efile, p: int, config, workdir: str, *, meter=None):
    """grem.py:277-319.  Induced subgraphs stay in HBM (no temp files are
    written); ``workdir`` is created for signature parity, as the reference does."""
    if p < 2 or (p & (p - 1)) != 0:
        raise FormatError(f"number of parts must be a power of two >= 2, got {p}")
    os.makedirs(workdir, exist_ok=True)
    n = int(efile.meta.num_nodes)
    plan_for(config, int(efile.meta.num_edges))   # same validation as the reference
    ctx = context()
    L = _abi.lib()
    hooks, keep, pending = _hooks(config, meter, None, None)
    cfg = _cfg_struct(config, None)
    labels = _host_labels(n)
    rep, sizes = _report_struct(max(2, int(p)))
    if is_native_binary(efile):
        rc = L.grem_partition_file(ctx, os.fsencode(efile.path), int(p), ctypes.byref(cfg), ctypes.byref(hooks),
                                   labels.ctypes.data, ctypes.byref(rep))
    else:
        e = edges_u32(efile)
        rc = L.grem_partition_u32(ctx, e.ctypes.data, e.shape[0], n, 0, int(p), ctypes.byref(cfg),
                                  ctypes.byref(hooks), labels.ctypes.data, ctypes.byref(rep))
    del keep
    _raise(rc, pending)
    return labels, _report(n, rep, sizes)


def count_cuts(efile, labels):
    """grem.py:227-252."""
    labels = np.asarray(labels)
    n = int(efile.meta.num_nodes)
    if labels.shape[0] != n:
        raise FormatError(f"labels cover {labels.shape[0]} nodes, file has {n}")
    lab = np.ascontiguousarray(labels.astype(np.int32))
    cap = max(2, int(lab.max()) + 1 if lab.size else 2)
    rep, sizes = _report_struct(cap)
    if is_native_binary(efile):
        rc = _abi.lib().grem_count_cuts_file(context(), os.fsencode(efile.path), lab.ctypes.data, 0,
                                             ctypes.byref(rep))
    else:
        e = edges_u32(efile)
        rc = _abi.lib().grem_count_cuts_u32(context(), e.ctypes.data, e.shape[0], n, 0, lab.ctypes.data, 0,
                                            ctypes.byref(rep))
    _raise(rc)
    return _report(n, rep, sizes)


# ------------------------------------------------- array-level entry points
# (edges already in memory: used by bench.py, the tests and the C-ABI users)

def bisect_edges(edges, num_nodes: int, config, capacity=None, on_device_ptr: int | None = None,
                 num_edges: int | None = None):
    n = int(num_nodes)
    m = int(num_edges if on_device_ptr is not None else np.asarray(edges).reshape(-1, 2).shape[0])
    cap = capacity if capacity is not None else default_capacity(n, config.capacity_slack)
    plan = plan_for(config, m)
    hooks, keep, pending = _hooks(config)
    cfg = _cfg_struct(config, plan.chunk_size)
    labels = _host_labels(n)
    rep, sizes = _report_struct(2)
    if on_device_ptr is None:
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        ptr, dev = e.ctypes.data, 0
    else:
        ptr, dev = on_device_ptr, 1
    rc = _abi.lib().grem_bisect_u32(context(), ptr, m, n, dev, ctypes.byref(cfg), int(cap), ctypes.byref(hooks),
                                    labels.ctypes.data, ctypes.byref(rep))
    del keep
    _raise(rc, pending)
    return labels, _report(n, rep, sizes)


def partition_edges(edges, num_nodes: int, p: int, config, on_device_ptr: int | None = None,
                    num_edges: int | None = None):
    n = int(num_nodes)
    if p < 2 or (p & (p - 1)) != 0:
        raise FormatError(f"number of parts must be a power of two >= 2, got {p}")
    hooks, keep, pending = _hooks(config)
    cfg = _cfg_struct(config, None)
    labels = _host_labels(n)
    rep, sizes = _report_struct(max(2, int(p)))
    if on_device_ptr is None:
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        ptr, m, dev = e.ctypes.data, e.shape[0], 0
    else:
        ptr, m, dev = on_device_ptr, int(num_edges), 1
    rc = _abi.lib().grem_partition_u32(context(), ptr, m, n, dev, int(p), ctypes.byref(cfg), ctypes.byref(hooks),
                                       labels.ctypes.data, ctypes.byref(rep))
    del keep
    _raise(rc, pending)
    return labels, _report(n, rep, sizes)


def set_profiling(on=True) -> None:
    """Per-phase CUDA-event timing of subsequent calls (see phase_times());
    ``on=2`` adds the kernel-level marks ("k.*") and their algorithmic bytes."""
    _abi.lib().grem_set_profiling(context(), 2 if on == 2 else (1 if on else 0))


def phase_times() -> dict:
    """{phase: (ms, launch groups)} of the last call (profiling on)."""
    L = _abi.lib()
    ms = (ctypes.c_double * 32)()
    cnt = (ctypes.c_int64 * 32)()
    names = (ctypes.c_char_p * 32)()
    n = L.grem_get_phase_times(context(), ms, cnt, 32, names)
    return {names[k].decode(): (ms[k], cnt[k]) for k in range(n)}


def phase_bytes() -> dict:
    """{kernel phase: algorithmic bytes} of the last call (profiling level 2)."""
    L = _abi.lib()
    by = (ctypes.c_double * 32)()
    names = (ctypes.c_char_p * 32)()
    n = L.grem_get_phase_times(context(), None, None, 32, names)
    L.grem_get_phase_bytes(context(), by, 32)
    return {names[k].decode(): by[k] for k in range(n) if by[k] > 0}


def count_cuts_edges(edges, num_nodes: int, labels):
    """count_cuts on an in-memory edge array (grem.py:227-252)."""
    n = int(num_nodes)
    lab = np.ascontiguousarray(np.asarray(labels).astype(np.int32))
    if lab.shape[0] != n:
        raise FormatError(f"labels cover {lab.shape[0]} nodes, file has {n}")
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
    cap = max(2, int(lab.max()) + 1 if lab.size else 2)
    rep, sizes = _report_struct(cap)
    rc = _abi.lib().grem_count_cuts_u32(context(), e.ctypes.data, e.shape[0], n, 0, lab.ctypes.data, 0,
                                        ctypes.byref(rep))
    _raise(rc)
    return _report(n, rep, sizes)


def last_stats() -> dict:
    st = _abi.GremStatsC()
    _abi.lib().grem_get_stats(context(), ctypes.byref(st))
    return {k: getattr(st, k) for k, _ in st._fields_}


__all__ = ["bisect", "partition", "count_cuts", "bisect_edges", "partition_edges", "set_device", "context",
           "last_stats", "ChunkPlan"]
