"""Per-rank step time of an N-way group sharding, measured on ONE GPU (a proxy for the strong-scaling
curve no 1-GPU run can measure): a context over rank 0's shard [0, n/N) runs the iteration's phases
(sampler + forward, backward, M-step) without the all-reduce (the plate sums stay local, so the
numbers are timings only).  Efficiency proxy = T_1 / (N T_N); the real N-rank step adds one (K+1)
fp64 NCCL all-reduce.  Usage: python tools/shard_proxy.py [config ...] [--world=N]"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_08264_b200 import synth  # noqa: E402
from paper_2503_08264_b200.qem import QEM, shard_range  # noqa: E402


def per_rank_ms(m, data, world, steps=10, warmup=3):
    gb, ge = shard_range(m.n, 0, world)
    g = QEM(m, group_begin=gb, group_end=ge)
    g.set_data(data)
    seed = 100 + m.config_id
    t = 1

    def step(t):
        g.sample_estep_forward(seed, t)
        g.estep_backward()
        g.mstep(t)

    for _ in range(warmup):
        step(t)
        t += 1
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step(t)
        t += 1
    b.record()
    torch.cuda.synchronize()
    g.close()
    return a.elapsed_time(b) / steps, ge - gb


args = [a for a in sys.argv[1:] if not a.startswith("--world=")]
worlds = [int(a.split("=")[1]) for a in sys.argv[1:] if a.startswith("--world=")] or [1, 2, 4, 8]
out = {}
for cid in [int(c) for c in args] or [5, 4]:
    m = synth.config(cid)
    data = synth.make_data(m)
    rows = {}
    for world in worlds:
        ms, n = per_rank_ms(m, data, world)
        rows[world] = {"groups": n, "ms_per_step": ms}
    if 1 in rows:
        t1 = rows[1]["ms_per_step"]
        for w, r in rows.items():
            r["efficiency_proxy"] = t1 / (w * r["ms_per_step"])
    out[f"config{cid}"] = rows
print(json.dumps(out))
