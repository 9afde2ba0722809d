"""Diagnostic (not a test): per-iteration root-weight and plate-message errors of config 4's shape on the
current pair path (FFMA tiles; QEM_TC1=1 for the compact tensor-core path), teacher-forced from the oracle's trajectory.
    python tools/diag_c4tc.py [n] [T]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle import oracle as orc  # noqa: E402
from paper_2503_08264_b200 import synth  # noqa: E402
from paper_2503_08264_b200.qem import QEM  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
T = int(sys.argv[2]) if len(sys.argv) > 2 else 12
m = synth.config(4, n=n)
data = synth.make_data(m)
seed = 104
ref_run = orc.run_qem(m, data, T, seed)
g = QEM(m)
g.set_data(data)
print("pair path", g.pair_path())
state = orc.initial_state(m)
q = [orc.mstep(a, b)[:2] for a, b in state]
for t in range(1, T + 1):
    eps = orc.eps_for_iteration(m, t, seed)
    g.set_state([(a, b - a * a) for a, b in state])
    g.set_q(q)
    g.sample_q(eps=eps)
    g.estep()
    out = g.result()
    dg, c = [x.cpu().numpy() for x in g.messages()]
    hist = g.mode_hist()
    ref = ref_run[t - 1]["est"]
    z = ref_run[t - 1]["z"]
    wr = ref["w"][0].reshape(-1)
    zr = np.asarray(z[0], np.float64).reshape(m.R, m.K)
    d2 = ((zr - np.asarray(q[0][0], np.float64)[:, None]) ** 2 / np.asarray(q[0][1], np.float64)[:, None]).sum(0)
    kref = int(np.argmin(d2))
    ps = g.plate_sum.cpu().numpy()
    G_gpu = ps[:m.K] + ps[m.K]  # sum_i g_i(k) from the fp64 plate sum (no fp32 message storage)
    G_ref = ref["g"].sum(0)
    full = c[:, None] + dg.astype(np.float64)
    gerr = full - ref["g"]
    rows = wr > 1e-3
    G_err = G_gpu - G_ref
    print(f"t={t:2d} ess={1/np.sum(wr**2):7.2f} modes={hist} w_root err={np.abs(out['w'][0].reshape(-1)-wr).max():.2e} "
          f"G err (weighted rows, fp64 plate sum) mean={G_err[rows].mean():+.2e} spread={np.abs(G_err[rows]-G_err[rows].mean()).max():.2e} "
          f"msg err mean={gerr[:, rows].mean():.2e} max={np.abs(gerr[:, rows]).max():.2e} "
          f"logpe rel={abs(out['log_pe']-ref['log_pe'])/abs(ref['log_pe']):.1e}", flush=True)
    if t in (7, 9):
        idx = np.argsort(-wr)[:8]
        zr0 = zr[0]
        print("   k    w_ref     G_err      mu_k     s_k   (kref=%d)" % kref)
        for k in idx:
            print(f"  {k:3d} {wr[k]:.3e} {G_err[k]:+.3e} {zr0[k]:+.4f} {zr[1][k]:+.4f}")
    state, q = ref_run[t - 1]["state"], ref_run[t - 1]["q_next"]
g.close()
