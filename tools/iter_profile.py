"""Per-iteration kernel times over a whole QEM run (diagnostic, not the bench).

    python tools/iter_profile.py --config 4 [--iters 50]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_08264_b200 import synth  # noqa: E402
from paper_2503_08264_b200.qem import QEM  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--n", type=int, default=0)
    a = ap.parse_args()
    m = synth.config(a.config, n=a.n or None)
    T = a.iters or m.T
    g = QEM(m)
    g.set_data(synth.make_data(m))
    st = torch.cuda.current_stream()
    rows = []
    for t in range(1, T + 1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(st)
        g.sample_q(seed=100 + a.config, iter=t)
        ev[1].record(st)
        g.estep_forward()
        ev[2].record(st)
        g.estep_backward()
        ev[3].record(st)
        g.mstep(t)
        ev[4].record(st)
        torch.cuda.synchronize()
        lp = g.log_pe.item()
        w = g.levels[0]["w"]
        ess = (1.0 / (w.double() ** 2).sum()).item()
        hist = g.mode_hist() if m.family == 2 else []
        rows.append(dict(t=t, sample=ev[0].elapsed_time(ev[1]), fwd=ev[1].elapsed_time(ev[2]),
                         bwd=ev[2].elapsed_time(ev[3]), mstep=ev[3].elapsed_time(ev[4]), log_pe=lp, root_ess=ess))
        r = rows[-1]
        print(f"t={t:3d} sample {r['sample']:.3f} fwd {r['fwd']:.3f} bwd {r['bwd']:.3f} mstep {r['mstep']:.3f} ms"
              f"  logPe {lp:.6e}  root ESS {ess:.2f}  modes {hist}", flush=True)
    print(json.dumps(dict(config=a.config, rows=rows)))


if __name__ == "__main__":
    main()
