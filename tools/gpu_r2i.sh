#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_gpu_tc.py -q -rf -x 2>&1 | tail -3
for v in "" variant_sum2 variant_sum6 variant_sum8; do
  if [ -n "$v" ]; then export QEM_LIB_OVERRIDE=$PWD/paper_2503_08264_b200/$v.so; fi
  timeout 300 python bench.py --config 5 --no-cpu --no-variants --no-e2e > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_i.json').read().strip().splitlines()[-1]); print('${v:-default}', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), d['roofline']['kernels_ms'])"
done
unset QEM_LIB_OVERRIDE
python - <<'P'
import sys, torch
sys.path.insert(0, '.')
from paper_2503_08264_b200 import synth
from paper_2503_08264_b200.qem import QEM
m = synth.config(5); g = QEM(m); g.set_data(synth.make_data(m)); g.set_q(synth.initial_q(m))
for t in range(1, 14):
    g.sample_q(seed=105, iter=t); g.estep(); g.mstep(t)
    print(t, g.mode_hist())
P
