"""File front end: partition(EdgeFile) from a page-cached
GRPE u32 file vs the device-resident path, same labels.  One JSON line.

    python tools/bench_file_ingest.py [SHAPE] [K] [DIR]

The file is written once (to DIR, default /dev/shm when it has room, else
/tmp), read once to warm the page cache, then partitioned `reps` times through
the reference-shaped `partition(efile, p, config, workdir)`; each step's wall
time includes the file read, the H2D copies, the path and the label readback.
"""
import ctypes, json, os, shutil, struct, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2502_17846_b200 import GremConfig, grem, synth, _abi, partition
from paper_2502_17846_b200.edgefile import open_edge_file

name = sys.argv[1] if len(sys.argv) > 1 else "papers100m"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 16
s = synth.SHAPES[name]
need = s.num_edges * 8 + (1 << 30)
d = sys.argv[3] if len(sys.argv) > 3 else None
if d is None:
    d = "/dev/shm" if shutil.disk_usage("/dev/shm").free > need else "/tmp"
if shutil.disk_usage(d).free < need:
    print(json.dumps({"skipped": f"{d}: {shutil.disk_usage(d).free} B free < {need}"}))
    sys.exit(0)
L = _abi.lib(); ctx = grem.context(); ptr = ctypes.c_void_p()
assert L.grem_device_alloc(ctx, s.num_edges * 8, ctypes.byref(ptr)) == 0
assert L.grem_gen_edges_device(ctx, s.num_nodes, s.beta, s.seed, 0, s.num_edges, ptr) == 0
cfg = GremConfig(chunk_frac=0.1)
lab, rep = grem.partition_edges(None, s.num_nodes, k, cfg, on_device_ptr=ptr.value, num_edges=s.num_edges)
dev_ms = []
for _ in range(3):
    t0 = time.perf_counter()
    grem.partition_edges(None, s.num_nodes, k, cfg, on_device_ptr=ptr.value, num_edges=s.num_edges)
    dev_ms.append((time.perf_counter() - t0) * 1e3)
host = np.empty((s.num_edges, 2), dtype=np.uint32)
assert L.grem_memcpy_d2h(ctx, ctypes.c_void_p(host.ctypes.data), ptr, s.num_edges * 8) == 0
path = os.path.join(d, f"grem_{name}.grpe")
t0 = time.perf_counter()
with open(path, "wb") as fh:
    fh.write(struct.pack("<4sIIQQ", b"GRPE", 1, 0, s.num_nodes, s.num_edges))
    host.tofile(fh)
write_s = time.perf_counter() - t0
del host
with open(path, "rb") as fh:   # warm the page cache
    while fh.read(1 << 28):
        pass
ef = open_edge_file(path)
out = {"shape": name, "k": k, "edges": s.num_edges, "file_dir": d, "file_bytes": os.path.getsize(path),
       "threads": os.environ.get("GREM_INGEST_THREADS", "default"), "write_s": round(write_s, 2),
       "device_resident_ms": round(min(dev_ms), 1)}
ms = []
for i in range(3):
    t0 = time.perf_counter()
    lab_f, rep_f = partition(ef, k, cfg, "/tmp/grem_work")
    ms.append((time.perf_counter() - t0) * 1e3)
    assert np.array_equal(lab_f, lab) and rep_f == rep, "file path labels differ"
out.update({"file_ms": [round(x, 1) for x in ms], "file_edges_per_s": s.num_edges / (min(ms) / 1e3),
            "file_GBps": s.num_edges * 8 / (min(ms) / 1e3) / 1e9, "labels_equal": True})
os.unlink(path)
print(json.dumps(out))
