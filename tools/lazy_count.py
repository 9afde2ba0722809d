"""Experiment: how often the forward's lazy-max chunks (QEM_FWD_LAZY) fall back to the exact path
(counted per epilogue warp in mode-hist slot 7 by a QEM_FWD_REDO_COUNT=1 build; the figures in DESIGN.md R41 were taken per chunk), per QEM iteration of config 5."""
import sys
import torch
from paper_2503_08264_b200 import synth
from paper_2503_08264_b200.qem import QEM

m = synth.config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
data = synth.make_data(m)
g = QEM(m)
g.set_data(data)
g.set_q(synth.initial_q(m))
K = m.K
lazy_chunks = m.n * (K // 128) * (K // 256 - 1) * 16  # (group, row block, column block > 0, epilogue warp)
for t in range(1, 9):
    g.sample_q(seed=1, iter=t)
    g.estep()
    g.mstep(t)
    torch.cuda.synchronize()
    h = g.mode_hist()
    print(t, "redo warps", h[7], "of", lazy_chunks, f"({h[7] / lazy_chunks:.3%})", "online groups", h[5], flush=True)
