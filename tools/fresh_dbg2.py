import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2503_08264_b200 import synth
from paper_2503_08264_b200.qem import QEM
m = synth.config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
data = synth.make_data(m)
g = QEM(m, fresh_denominator=True)
g.set_data(data)
for t in range(1, 8):
    for name, fn in [("sample_new", lambda: g.sample_q(seed=105, iter=t | (1 << 23))), ("evidence", g.estep_evidence),
                     ("sample", lambda: g.sample_q(seed=105, iter=t)), ("fwd", g.estep_forward), ("bwd", g.estep_backward),
                     ("mstep", lambda: g.mstep(t))]:
        fn(); torch.cuda.synchronize()
    print(t, "ok log_pe", g.log_pe.item(), "fresh", g.log_pe_fresh.item(), "flags", g.read_flags(), flush=True)
