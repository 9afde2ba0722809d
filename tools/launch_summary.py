"""Per-kernel time shares from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        hdr = r; start = i + 1; break
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = {}
for r in rows[start:]:
    agg.setdefault(r[ki][:60], []).append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
for n, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{n:60s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:9.3f}us share={sum(v) / tot * 100:5.1f}%")
