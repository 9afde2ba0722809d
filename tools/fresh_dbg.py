import sys, os
sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo")
import numpy as np
from oracle import oracle as orc
from paper_2503_08264_b200 import synth
from paper_2503_08264_b200.qem import QEM
m = synth.config(2, n=40)
data = synth.make_data(m)
g = QEM(m, fresh_denominator=True)
g.set_data(data)
state = orc.initial_state(m)
q = [orc.mstep(a, b)[:2] for a, b in state]
g.set_state([(a, b - a * a) for a, b in state]); g.set_q(q)
import torch
for name, fn in [("sample_new", lambda: g.sample_q(eps=orc.eps_for_iteration(m, 1, 7))), ("evidence", g.estep_evidence),
                 ("sample", lambda: g.sample_q(eps=orc.eps_for_iteration(m, 1, 8))), ("estep", g.estep), ("mstep", lambda: g.mstep(1))]:
    fn(); torch.cuda.synchronize(); print(name, "ok", flush=True)
