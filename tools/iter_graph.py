import sys, torch
sys.path.insert(0, '.')
from paper_2503_08264_b200 import synth
from paper_2503_08264_b200.qem import QEM
for cid in (1, 2, 3, 4, 5):
    m = synth.config(cid); data = synth.make_data(m)
    g = QEM(m, trace_len=200); g.set_data(data); g.set_q(synth.initial_q(m))
    g.iterate(1, 5, seed=100 + cid, use_graph=True)
    torch.cuda.synchronize()
    T = 200 if cid <= 3 else 20
    for use_graph in (True, False):
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record(); g.iterate(6, T, seed=100 + cid, use_graph=use_graph); en.record(); torch.cuda.synchronize()
        ms = st.elapsed_time(en) / T
        print(f"config {cid} {'graph' if use_graph else 'eager'}: {ms*1000:.1f} us/iteration, {1000/ms:.0f} iterations/s")
    g.close()
