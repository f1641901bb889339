"""Summarise an ncu source-page export (per-SASS-instruction counters):
python tools/sass_hot.py sass_k.csv[.gz] [N]
Prints the stall-reason mix, the N hottest instructions by warp-stall samples
and the N largest shared-memory wavefront counts with their conflict excess."""
import csv
import gzip
import io
import sys

path = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 15
raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr, data = rows[hi], [r for r in rows[hi + 1:] if len(r) > 3]
ix = {h: i for i, h in enumerate(hdr)}


def f(r, k):
    try:
        return float(r[ix[k]])
    except (KeyError, ValueError):
        return 0.0


S = "Warp Stall Sampling (All Samples)"
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {k: sum(f(r, k) for r in data) for k in reasons}
T = sum(tot.values()) or 1.0
print(rows[0][1][:100] if len(rows[0]) > 1 else "")
print("stalls: " + ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
ST = sum(f(r, S) for r in data) or 1.0
WF = sum(f(r, "L1 Wavefronts Shared") for r in data) or 1.0
WI = sum(f(r, "L1 Wavefronts Shared Ideal") for r in data)
print(f"samples {ST:.0f}; shared wavefronts {WF:.3g} (ideal {WI:.3g})")
print("-- hottest instructions")
for r in sorted(data, key=lambda r: -f(r, S))[:N]:
    print(f"{100 * f(r, S) / ST:5.1f}%  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()[:70]}")
print("-- shared wavefronts")
for r in sorted(data, key=lambda r: -f(r, "L1 Wavefronts Shared"))[:N]:
    w, wi = f(r, "L1 Wavefronts Shared"), f(r, "L1 Wavefronts Shared Ideal")
    print(f"{100 * w / WF:5.1f}%  x{w / wi if wi else 0:4.1f}  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()[:70]}")
