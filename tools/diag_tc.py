"""Diagnostic: message / weight errors of one E-step vs the oracle for a config-5-shaped case."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from helpers import make_case, posterior_like_q
from oracle import oracle as orc
from paper_2503_08264_b200 import synth
from paper_2503_08264_b200.qem import QEM

n, K, shrink = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
m = synth.config(5, n=n, K=K)
data = synth.make_data(m)
q = posterior_like_q(m, data, seed=7, shrink=shrink)
_, _, eps, _ = make_case(m, q=q)
z = [orc.sample(qm, qv, e) for (qm, qv), e in zip(q, eps)]
ref = orc.estep(m, z, q, data)
g = QEM(m)
g.set_data(data); g.set_q(q); g.sample_q(eps=eps); g.estep()
out = g.result(); hist = g.mode_hist(); dg, c = g.messages()
print("pair path", g.pair_path(), "modes", list(hist))
w0 = ref["w"][0].reshape(-1); ks = int(w0.argmax())
full = c.cpu().numpy()[:, None] + dg.cpu().numpy().astype(np.float64)
e = full - ref["g"]
print("log Pe", out["log_pe"], ref["log_pe"], "diff", out["log_pe"] - ref["log_pe"])
print("row k* message err: max %.3g mean %.3g | c_i err max %.3g" % (np.abs(e[:, ks]).max(), e[:, ks].mean(),
      0.0))
print("weights err level0 %.3g level1 %.3g" % (np.abs(out["w"][0].reshape(-1) - w0).max(),
      np.abs(out["w"][1].reshape(ref["w"][1].shape) - ref["w"][1]).max()))
