"""Diagnostic (not the bench): where config 4's end-to-end overhead comes from.  Times 10 QEM
iterations on the device alone and with host copies in several arrangements.
    python tools/e2e_diag.py [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_08264_b200 import synth  # noqa: E402
from paper_2503_08264_b200.qem import QEM  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
m = synth.config(cid)
g = QEM(m)
g.set_data(synth.make_data(m))
seed, steps = 100 + cid, 10
stream = torch.cuda.current_stream()
cs = torch.cuda.Stream()
x_host = g.x.cpu().pin_memory()
y_host = g.y.cpu().pin_memory() if g.y is not None else None
outs = [torch.empty_like(lv["q_mean"], device="cpu").pin_memory() for lv in g.levels]
outv = [torch.empty_like(lv["q_var"], device="cpu").pin_memory() for lv in g.levels]
stage = [(torch.empty_like(lv["q_mean"]), torch.empty_like(lv["q_var"])) for lv in g.levels]
prep_done = torch.cuda.Event()


def step(t, mode):
    if mode == "serial_up":
        g.x.copy_(x_host, non_blocking=True)
    g.sample_q(seed=seed, iter=t)
    g.estep_forward()
    if mode in ("async_up", "async_both", "snap_down_up"):
        cs.wait_event(prep_done)
        with torch.cuda.stream(cs):
            g.x.copy_(x_host, non_blocking=True)
        e = torch.cuda.Event()
        e.record(cs)
        stream.wait_event(e)
    g.estep_backward()
    g.mstep(t)
    if mode in ("serial_down", "serial_up"):
        for o, lv in zip(outs, g.levels):
            o.copy_(lv["q_mean"], non_blocking=True)
    if mode == "async_both":
        e = torch.cuda.Event()
        e.record(stream)
        cs.wait_event(e)
        with torch.cuda.stream(cs):
            for o, lv in zip(outs, g.levels):
                o.copy_(lv["q_mean"], non_blocking=True)
    if mode in ("snap_down", "snap_down_up"):  # the bench's download: D2D snapshot, then D2H on cs
        for (sm, sv), lv in zip(stage, g.levels):
            sm.copy_(lv["q_mean"])
            sv.copy_(lv["q_var"])
        e = torch.cuda.Event()
        e.record(stream)
        cs.wait_event(e)
        with torch.cuda.stream(cs):
            for o, ov, (sm, sv) in zip(outs, outv, stage):
                o.copy_(sm, non_blocking=True)
                ov.copy_(sv, non_blocking=True)


t = 1
for mode in ("device", "async_up", "snap_down", "snap_down_up", "async_both", "serial_down", "device"):
    g.set_kernel_events([prep_done])
    for _ in range(3):
        step(t, mode)
        t += 1
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(steps):
        step(t, mode)
        t += 1
    en.record()
    torch.cuda.synchronize()
    print(f"config {cid} {mode:12s} {st.elapsed_time(en) / steps:.3f} ms/step", flush=True)
