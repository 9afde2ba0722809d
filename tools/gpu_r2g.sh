#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in "" variant_lpepi; do
  if [ -n "$v" ]; then export QEM_LIB_OVERRIDE=$PWD/paper_2503_08264_b200/$v.so; fi
  echo "== ${v:-default}"
  timeout 600 python tools/diag_c4tc.py 1000 12 2>&1 | grep "^t=" | tail -4
  for c in 4 5; do timeout 300 python bench.py --config $c --no-cpu --no-variants --no-e2e > gpurun_out/bench_g$c.json 2> gpurun_out/bench_g$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_g$c.json').read().strip().splitlines()[-1]); print($c, round(d['ms_per_step'],3), d['roofline']['kernel'], round(d['roofline']['frac'],4), d['roofline']['kernels_ms'])"; done
done
