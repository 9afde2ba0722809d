#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest_gpu_h.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu_h.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_h.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_h.log
timeout 900 python bench.py > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_h.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['roofline']['frac'], d['roofline']['kernels_ms'], d['e2e']['ms_per_step']); v=d['variants']; print('c4', v['config4']['ms_per_step'], v['config4']['roofline']['frac'], v['config4']['roofline']['kernels_ms'])"
