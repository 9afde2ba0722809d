#!/bin/bash
# quick check: parity subset + config 5 / 4 bench lines (no variants)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_tc.py tests/test_gpu_qem.py} -q -rf 2>&1 | grep -E "Error|FAILED|passed|failed" | head
for c in 5 4; do
  timeout 300 python bench.py --config $c --no-cpu --no-variants --no-e2e > gpurun_out/bench_q$c.json 2> gpurun_out/bench_q$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_q$c.json').read().strip().splitlines()[-1]); print($c, round(d['ms_per_step'],3), d['roofline']['kernel'], round(d['roofline']['frac'],4), d['roofline']['kernels_ms'])"
done
