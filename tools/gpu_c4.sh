#!/bin/bash
# parity subset + the config-4 bench line (with its forward mode histogram)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_fullsize.py::test_config4_full_size} -q -x 2>&1 | tail -3
for c in ${CFGS:-4}; do
for rep in 1 2; do
timeout 300 python bench.py --config $c --no-cpu --no-variants --no-e2e > gpurun_out/c4.json 2> gpurun_out/c4.err
python -c "
import json; d=json.loads(open('gpurun_out/c4.json').read().strip().splitlines()[-1]); r=d['roofline']; print($c, round(d['ms_per_step'],3), {k: round(v,3) for k,v in r['kernels_ms'].items()}, round(r['frac'],4), r.get('forward_mode_hist'))"
done
done
