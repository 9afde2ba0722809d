"""Top SASS instructions by warp-stall samples from an ncu report (--page source)."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
for i, r in enumerate(rows):
    if "Source" in r and "Warp Stall Sampling (All Samples)" in r:
        hdr = r; start = i + 1; break
si, ssi = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
ai = hdr.index("Address")
data = []
for r in rows[start:]:
    if len(r) < len(hdr):
        continue
    try:
        data.append((int(r[ssi] or 0), r[ai], r[si].strip()))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
byop = {}
for c, a, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    byop[op] = byop.get(op, 0) + c
print("total samples", tot)
for op, c in sorted(byop.items(), key=lambda x: -x[1])[:15]:
    print(f"{op:28s} {c:8d} {100*c/tot:5.1f}%")
print("--- hottest instructions")
for c, a, src in sorted(data, key=lambda x: -x[0])[:n]:
    print(f"{c:7d} {a} {src[:90]}")
