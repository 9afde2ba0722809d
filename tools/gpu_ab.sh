#!/bin/bash
# interleaved A/B of library variants on the config-5 bench (the power-capped part drifts over a call):
#   VARIANTS="variant_x variant_y" bash tools/gpu_ab.sh
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for rep in 1 2; do
  for v in default $VARIANTS; do
    if [ "$v" = default ]; then unset QEM_LIB_OVERRIDE; else export QEM_LIB_OVERRIDE=$PWD/paper_2503_08264_b200/$v.so; fi
    timeout 300 python bench.py --config ${CFG:-5} --no-cpu --no-variants --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels_ms']; print('$v', round(d['ms_per_step'],3), round(k['forward'],3), round(k['backward'],3), round(d['roofline']['frac'],4))"
  done
done
