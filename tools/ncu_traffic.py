"""Write profiles/<name>.json: per-kernel DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
from one `ncu --set full` capture per kernel, for bench.py's roofline "traffic" field.

    python tools/ncu_traffic.py profiles/r02_traffic.json [--config N] gpurun_out/ncu_bwd4.ncu-rep [...]
(with --config N the entries go under "configN", the layout bench.py reads)
"""
import csv, json, subprocess, sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def kernel_bytes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u, v = r[0], r[1], r[2]
    name = v[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("qem::", "").split("<")[0]
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(k)
        tot += float(v[i].replace(",", "")) * UNIT[u[i]]
    dur = float(v[h.index("gpu__time_duration.sum")].replace(",", ""))
    return name, {"dram_bytes": tot, "ncu_duration": dur, "ncu_duration_unit": u[h.index("gpu__time_duration.sum")],
                  "report": rep.split("/")[-1]}


if __name__ == "__main__":
    dst = sys.argv[1]
    args = sys.argv[2:]
    cfg = None
    if args and args[0] == "--config":
        cfg, args = "config" + args[1], args[2:]
    try:
        data = json.load(open(dst))
    except Exception:
        data = {}
    for rep in args:
        n, d = kernel_bytes(rep)
        (data.setdefault(cfg, {}) if cfg else data)[n] = d
        print(cfg, n, d)
    json.dump(data, open(dst, "w"), indent=1)
