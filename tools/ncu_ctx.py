"""SASS context (+-N instructions) around the hottest stall addresses of an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 4; ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 6
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
for i, r in enumerate(rows):
    if "Source" in r and "Warp Stall Sampling (All Samples)" in r:
        hdr = r; start = i + 1; break
si, ssi = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = [(int(r[ssi] or 0), r[si].strip()) for r in rows[start:] if len(r) >= len(hdr)]
order = sorted(range(len(data)), key=lambda j: -data[j][0])[:top]
for j in order:
    print(f"---- around #{j} ({data[j][0]} samples)")
    for k in range(max(0, j - ctx), min(len(data), j + ctx + 1)):
        print(f"{'>>' if k == j else '  '} {data[k][0]:6d} {data[k][1][:100]}")
