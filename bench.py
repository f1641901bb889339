"""bench.py — GREM edges/s on B200 (BASELINE.json metric).

Workload (BASELINE.json north_star target, fits one B200): papers100M-shaped
synthetic power-law graph, 111,059,956 nodes / 1,615,685,872 edges
(Chung-Lu gamma=2.1, paper_2502_17846_b200/synth.py), partitioned into k=16 by
recursive GREM bisection with the reference defaults (chunk_frac 0.1,
slack 0, refine, 1 pass, bfs_grow seed with 2 refinement passes).

A step = one full partition(k=16) of the whole graph.  `value` is whole-job
edges/s (original E / step time) with the edges resident in HBM; `e2e` is the
same metric through the public API from pinned host memory (H2D of the edge
list and D2H of the labels inside every timed step).  Device times are CUDA
events on the library's stream (grem_stats.ms_total); max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload papers100m|friendster|products|arxiv|tiny] [--k K]

N > 1: one process per GPU (torchrun), ONE partition of the same graph
sharded across the ranks ("scaling": "strong"): recursion subtrees are split
between GPUs in proportion to their edges (paper_2502_17846_b200/shard.py),
labels merged with one NCCL all-reduce, count_cuts on the merged labels.
`--replicas` instead has every rank partition its own copy ("weak").
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0


def measured_peak():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return HBM_FALLBACK_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        loaded = [v for v in sm if v > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)   # >= 3 for a valid bench line
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="papers100m")
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent replicas (weak scaling)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        return run_reference_arm(args)

    import numpy as np
    import torch

    from paper_2502_17846_b200 import GremConfig, _abi, grem, synth

    dist = None
    if world > 1:
        import torch.distributed as dist_
        dist = dist_
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    grem.set_device(local)
    shape = synth.SHAPES[args.workload]
    k = args.k or shape.k
    E, n = shape.num_edges, shape.num_nodes
    L = _abi.lib()
    ctx = grem.context()
    cfg = GremConfig(chunk_frac=0.1)

    # edges resident in HBM (device generator == host generator, bit for bit)
    dptr = ctypes.c_void_p()
    assert L.grem_device_alloc(ctx, E * 8, ctypes.byref(dptr)) == 0, _abi.last_error()
    assert L.grem_gen_edges_device(ctx, n, shape.beta, shape.seed, 0, E, dptr) == 0, _abi.last_error()

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    sharded = world > 1 and not args.replicas
    if sharded:
        from paper_2502_17846_b200 import shard
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step_device():
        if not sharded:
            lab, rep = grem.partition_edges(None, n, k, cfg, on_device_ptr=dptr.value, num_edges=E)
            return lab, rep, grem.last_stats()
        # events on torch's stream bracket the whole step: the library call
        # (its own stream, synchronised inside), the NCCL merge and count_cuts
        torch.cuda.synchronize()
        ev0.record()
        labels = torch.empty(n, dtype=torch.int32, device="cuda")
        shard.partition_shard(dptr.value, E, n, k, cfg, rank, world, labels)
        st = grem.last_stats()
        st["_phases"] = grem.phase_times()
        shard.merge_labels(labels)
        torch.cuda.synchronize()
        rep = shard.count_cuts_device(dptr.value, E, n, labels, k)
        ev1.record()
        torch.cuda.synchronize()
        st["ms_total"] = ev0.elapsed_time(ev1)
        st["kernels"] += 2    # the count_cuts launches (hist + cut)
        return labels, rep, st

    for _ in range(args.warmup):
        lab, rep, st = step_device()
    ref_sha = None

    # timed steps run without the phase profiler (its per-phase CUDA events
    # cost real time on launch-bound shapes); one extra profiled step after
    # the timed region gives the phase split
    barrier()
    dev_ms, kernels, phases = [], 0, {}
    sampler = ClockSampler(local)
    t0 = time.perf_counter()
    with sampler:
        for _ in range(args.steps):
            lab, rep, st = step_device()
            dev_ms.append(st["ms_total"])
            kernels += st["kernels"]
    barrier()
    wall_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    grem.set_profiling(2)
    _, _, st_p = step_device()
    for name, (ms, cnt) in (st_p.pop("_phases", None) or grem.phase_times()).items():
        phases[name] = [ms * args.steps, cnt * args.steps]   # per-step figures below divide by steps
    grem.set_profiling(False)
    ms_step = sum(dev_ms) / len(dev_ms)
    if dist:
        t = torch.tensor([ms_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    units = E if sharded else world * E
    value = units / (ms_step / 1e3)

    import hashlib
    if sharded:
        lab = lab.cpu().numpy()
    labels_sha = hashlib.sha256(np.asarray(lab, dtype="<i4").tobytes()).hexdigest()

    # e2e: public API from pinned host memory, labels read back every step
    e2e = None
    if not args.no_e2e:
        host = torch.empty((E, 2), dtype=torch.int32, pin_memory=True)
        assert L.grem_memcpy_d2h(ctx, ctypes.c_void_p(host.data_ptr()), dptr, E * 8) == 0
        hv = host.numpy().view(np.uint32)

        def e2e_step():
            if not sharded:
                lab2, _ = grem.partition_edges(hv, n, k, cfg)
                return lab2, grem.last_stats()["ms_total"]
            # every rank uploads the edge list from pinned host memory into its
            # own HBM (overlapped with its level-0 bisection), then the sharded
            # partition; labels read back to the host
            t_0 = time.perf_counter()
            labels, _ = shard.partition_distributed(host.data_ptr(), E, n, k, cfg, edges_on_device=False)
            lab2 = labels.cpu().numpy()
            return lab2, (time.perf_counter() - t_0) * 1e3

        for _ in range(2):   # warm the host path (first call sizes the staging buffers)
            e2e_step()
        barrier()
        e_ms = []
        te = time.perf_counter()
        lab2 = None
        for _ in range(max(1, min(args.steps, 3))):
            lab2 = None   # the caller is done with the previous labels (their pinned block is reused)
            lab2, ms_ = e2e_step()
            e_ms.append(ms_)
        barrier()
        e_wall = (time.perf_counter() - te) * 1e3 / len(e_ms)
        print(f"[bench] e2e steps ms {['%.1f' % v for v in e_ms]} wall/step {e_wall:.1f}", file=sys.stderr)
        assert np.array_equal(lab2, lab), "e2e labels differ from the device-resident run"
        e_step = max(sum(e_ms) / len(e_ms), 0.0)
        e_step = max(e_step, e_wall)   # include host-side staging the event window may not see
        if dist:
            t = torch.tensor([e_step], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_step = float(t.item())
        e2e = {"value": units / (e_step / 1e3), "unit": "edges/s", "ms_per_step": e_step,
               "h2d_bytes_per_step": E * 8, "d2h_bytes_per_step": n * 4}
        del host

    # Roofline.  Lead: the whole path, SURVEY.md 8(d) algorithmic bytes of the
    # step (grem_stats.path_bytes) / step time.  Rows: the top kernels by
    # share of the step, each timed with CUDA events on the library stream
    # around its launches (kernel marks, profiling level 2) in a level-0
    # bisection (k=2: one stream, no concurrent sibling subtrees), achieved =
    # the kernel's algorithmic bytes per launch / its average
    # launch time; traffic = ncu DRAM bytes per launch of this build
    # (profiles/r02_traffic.json) when captured.
    peak, peak_kind = measured_peak()
    traffic = {}
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "r02_traffic.json")))
    except Exception:  # noqa: BLE001
        pass
    grem.set_profiling(2)
    grem.partition_edges(None, n, 2, cfg, on_device_ptr=dptr.value, num_edges=E)
    ph_l0, by_l0 = grem.phase_times(), grem.phase_bytes()
    grem.set_profiling(False)
    step_ms_sum = sum(v[0] for kk, v in phases.items() if "." not in kk) or 1e-9
    rows = []
    for kk, (ms_l0, cnt_l0) in ph_l0.items():
        if not kk.startswith("k.") or cnt_l0 <= 0 or ms_l0 <= 0 or by_l0.get(kk, 0) <= 0:
            continue
        base = kk[:-5] if kk.endswith("_full") else kk   # round kernels: bytes from full rounds,
        kname = "k_" + base[2:]                            # share from all their launches
        ach = by_l0[kk] / (ms_l0 / 1e3) / 1e9
        tr = traffic.get(kname, {})
        share = (phases.get(base, (0.0, 0))[0] + (phases.get(kk, (0.0, 0))[0] if kk != base else 0.0)) / step_ms_sum
        rows.append({"kernel": kname, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "algorithmic_bytes_per_launch": by_l0[kk] / cnt_l0, "avg_launch_ms": ms_l0 / cnt_l0,
                     "launches_timed": cnt_l0, "timed_launches": "full rounds" if kk != base else "all",
                     "traffic": tr.get("dram_bytes_per_launch"), "traffic_source": tr.get("source"),
                     "share_of_step": share})
    rows.sort(key=lambda r: -r["share_of_step"])
    path_bytes = st.get("path_bytes")
    roof = None
    if path_bytes:
        ach = path_bytes / (ms_step / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": "whole path (partition to k)", "achieved": ach, "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": ach / peak,
                "traffic": (traffic.get("step", {}) or {}).get("dram_bytes"),
                "traffic_source": (traffic.get("step", {}) or {}).get("source"),
                "algorithmic_bytes_per_step": path_bytes, "formula": "SURVEY.md 8(d): per level 8E+2E+34V, "
                "+10E_l+8E_(l+1) per extraction, +10E final cut",
                "kernels": rows[:3], "kernels_other": rows[3:],   # the remaining marked kernels (round-1 binning)
                "kernels_timed_in": f"{args.workload} level-0 bisection (k=2), CUDA events",
                "kernel_share_from": "kernel marks in the profiled k-way step (sum of kernel times across streams)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_port(args.workload, k)

    if rank == 0:
        out = {
            "metric": "GREM edges/s (partition to k, bit-equal labels/edge-cut)", "value": value,
            "unit": "edges/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "wall_ms_per_step": wall_ms, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "u32/f64",
            "data": "synthetic",
            "config": bench_config(args.workload, k, world, sharded),
            "report": {"cut_edges": rep.cut_edges, "cut_fraction": rep.cut_fraction,
                       "balance_ratio": rep.balance_ratio, "labels_sha256": labels_sha},
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu,
            "gpu_launches": kernels, "clocks": sampler.summary(),
            "phases_ms_per_step": {kk: round(v[0] / args.steps, 3) for kk, v in sorted(phases.items())},
            "phases_note": "one extra step with the phase profiler on (CUDA events per launch group; sums of concurrent subtrees exceed the step)",
            "stats": {kk: st[kk] for kk in ("rounds", "visits", "bisections", "chunks")},
        }
        _emit(json.dumps(out))
    if dist:
        dist.destroy_process_group()
    return 0


# Shapes of paper_2502_17846_b200/synth.SHAPES (tests/test_host.py checks the
# two tables agree), repeated here so the reference arm never imports the
# product package: (num_nodes, num_edges, default k, generator beta, seed)
SHAPES = {
    "tiny": (10_000, 100_000, 4, 11, 0),
    "arxiv": (169_343, 1_166_243, 8, 11, 0),
    "products": (2_449_029, 61_859_140, 16, 11, 0),
    "papers100m": (111_059_956, 1_615_685_872, 16, 11, 0),
    "friendster": (65_608_366, 1_806_067_135, 16, 4, 0),
}


def bench_config(workload, k, world, sharded):
    """The workload; identical for both arms (the reference arm's bounded
    sample is described in its cpu_baseline.sample)."""
    n, E = SHAPES[workload][:2]
    return {"workload": f"{workload}-shaped power-law k={k}", "num_nodes": n, "num_edges": E,
            "k": k, "chunk_frac": 0.1, "capacity_slack": 0.0, "refine": True, "passes": 1,
            "seed": "bfs_grow/2", "parallelism": (f"subtree-sharded x{world}" if sharded else
                                                  f"replicas x{world}" if world > 1 else "single"),
            "l2": "inputs larger than L2 (edge list %.1f GB)" % (E * 8 / 1e9)}


def _golden_full_run(workload, k):
    """The committed same-config single-thread run of the C restatement
    (tests/golden/golden_shapes.json, measured in the build container)."""
    try:
        gs = json.load(open(os.path.join(ROOT, "tests", "golden", "golden_shapes.json")))
        g = gs.get(f"{workload}_k{k}") or {}
        sec = g.get("oracle_seconds") or g.get("reference_seconds") or (None if g.get("derived_from") else
                                                                           g.get("seconds"))
        if not sec or g.get("chunk_frac", 0.1) != 0.1:
            return None
        who = ("streamcut itself (pure Python)" if "reference_seconds" in g else
               "C restatement oracle/grem_oracle.c (bit-exact with streamcut)")
        return {"value": g["num_edges"] / sec, "unit": "edges/s", "cores": 1, "seconds": sec,
                "source": f"tests/golden/golden_shapes.json[{workload}_k{k}]: {who}, full graph, 1 core, "
                          "build container (Intel Xeon), not this host"}
    except Exception:  # noqa: BLE001
        return None


def cpu_baseline_port(workload, k):
    """The C restatement (oracle/, single thread) on a bounded sample of the
    same workload on this host: a 1/scale graph of the same shape family (same
    generator, same average degree), partitioned to the same k; plus the
    committed full-size run of the same config."""
    from oracle import gen_np, oracle
    n0, m0, _, beta, seed = SHAPES[workload]
    # ~0.5-4 M edges/s single-thread: size the sample for ~10-30 s of CPU work
    scale = max(1, m0 // 30_000_000)
    n = max(1000, n0 // scale)
    m = max(10000, m0 // scale)
    e = gen_np.powerlaw_edges(n, m, beta=beta, seed=seed)
    t = time.perf_counter()
    oracle.partition(e, n, k, chunk_frac=0.1)
    dt = time.perf_counter() - t
    return {"value": m / dt, "unit": "edges/s", "cores": 1, "kind": "port",
            "sample": f"{workload}-shaped 1/{scale} scale ({n} nodes, {m} edges, same generator), k={k}, "
                      f"C restatement of streamcut (oracle/grem_oracle.c, bit-exact), {dt:.1f} s on this host",
            "same_config": _golden_full_run(workload, k)}


def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation (streamcut,
    pure Python, single-threaded by construction, from baseline/_ref) on a
    bounded sample of the workload on this host.  The input comes from the
    numpy restatement of the generator (oracle/gen_np.py): nothing of the
    product package or its library is loaded in this arm."""
    import tempfile

    import numpy as np

    from oracle import gen_np
    workload = args.workload
    n0, m0, k0, beta, seed = SHAPES[workload]
    k = args.k or k0
    scale = 1000 if m0 > 100_000_000 else 10
    n = max(1000, n0 // scale)
    m = max(10000, m0 // scale)
    e = gen_np.powerlaw_edges(n, m, beta=beta, seed=seed)
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref_dir):
        sys.path.insert(0, ref_dir)
    try:
        import streamcut
        from streamcut import BinaryEdgeWriter, GremConfig, open_edge_file
        kind = "reference"
    except Exception:  # noqa: BLE001
        streamcut = None
        kind = "port"
    tmp = tempfile.mkdtemp()
    path = os.path.join(tmp, "g.grpe")
    if streamcut is not None:
        with BinaryEdgeWriter(path, n) as w:
            w.write(e.astype(np.int64))
    times = []
    for i in range(args.warmup + args.steps):
        t = time.perf_counter()
        if streamcut is not None:
            streamcut.partition(open_edge_file(path), k, GremConfig(chunk_frac=0.1), os.path.join(tmp, "w"))
        else:
            from oracle import oracle
            oracle.partition(e, n, k, chunk_frac=0.1)
        if i >= args.warmup:
            times.append(time.perf_counter() - t)
    dt = sum(times) / len(times)
    value = m / dt
    sample = (f"{workload}-shaped 1/{scale} scale ({n} nodes, {m} edges, same generator via oracle/gen_np.py), "
              f"k={k}, {'streamcut (pure Python, single thread)' if kind == 'reference' else 'C restatement'}; "
              f"{dt:.2f} s per partition")
    out = {"impl": "reference", "metric": "GREM edges/s (partition to k, bit-equal labels/edge-cut)",
           "value": value, "unit": "edges/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak",
           "vs_baseline": None, "dtype": "u32/f64", "data": "synthetic",
           "config": bench_config(workload, k, args.gpus, args.gpus > 1 and not args.replicas),
           "cpu_baseline": {"value": value, "unit": "edges/s", "cores": 1, "kind": kind, "sample": sample},
           "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    _emit(json.dumps(out))
    return 0


# The JSON line is the only thing on stdout: native chatter written straight to
# file descriptor 1 (e.g. NCCL's "NCCL version" banner at communicator init
# under torchrun) is sent to stderr instead.
_JSON_OUT = None


def _emit(line: str) -> None:
    (_JSON_OUT or sys.stdout).write(line + "\n")
    (_JSON_OUT or sys.stdout).flush()


if __name__ == "__main__":
    try:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)
    except OSError:
        _JSON_OUT = None
    sys.exit(main())
