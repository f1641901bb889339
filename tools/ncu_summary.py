"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum
[,dram__bytes_read.sum,dram__bytes_write.sum]): time and DRAM bytes per
kernel name.  With --traffic OUT.json also writes the per-launch DRAM bytes of
every kernel and the whole capture's total (bench.py's roofline.traffic).

  python tools/ncu_summary.py launches.csv[.gz] [--traffic OUT.json --source NAME]
"""
import collections
import csv
import gzip
import json
import sys

path = sys.argv[1]
opener = gzip.open if path.endswith(".gz") else open
rows = list(csv.reader(opener(path, "rt")))
hdr = None
per = collections.defaultdict(dict)   # launch id -> {metric: value}
names = {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    lid = d.get("ID")
    names[lid] = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    if d["Metric Name"] == "gpu__time_duration.sum":
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
    else:
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    per[lid][d["Metric Name"]] = v
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for lid, m in per.items():
    a = agg[names[lid]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(v[1] for v in agg.values())
totb = sum(v[2] for v in agg.values())
print(f"total kernel time {tot/1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches; "
      f"DRAM {totb/1e9:.2f} GB")
for name, (n, us, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{us/1e3:9.3f} ms {100*us/tot:5.1f}% {n:6d}x  {b/1e9:8.2f} GB  {b/max(us,1e-9)/1e3:7.0f} GB/s  {name}")
if "--traffic" in sys.argv:
    out = sys.argv[sys.argv.index("--traffic") + 1]
    src = sys.argv[sys.argv.index("--source") + 1] if "--source" in sys.argv else path
    step = {k: v for k, v in agg.items() if "k_gen" not in k}   # input generation is not part of the step
    js = {"step": {"dram_bytes": sum(v[2] for v in step.values()), "kernel_ms": sum(v[1] for v in step.values()) / 1e3,
                   "launches": sum(v[0] for v in step.values()), "source": src,
                   "note": "ncu launch list of one partition (GREM_NO_GRAPH=1 so every launch is listed), "
                           "cold caches, serialised; k_gen (input generation) excluded"}}
    for name, (n, us, b) in agg.items():
        js[name.split("::")[-1]] = {"dram_bytes_per_launch": b / n, "launches": n, "avg_launch_us_cold": us / n,
                                    "source": src}
    json.dump(js, open(out, "w"), indent=1, sort_keys=True)
