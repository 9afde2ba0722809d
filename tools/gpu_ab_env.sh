#!/bin/bash
# interleaved A/B over "lib:ENV=val" specs on one config:  SPECS="default:X=1 vA:QEM_RP=1" bash tools/gpu_ab_env.sh
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for rep in 1 2; do
  for sp in $SPECS; do
    lib=${sp%%:*}; env=${sp#*:}
    if [ "$lib" = default ]; then unset QEM_LIB_OVERRIDE; else export QEM_LIB_OVERRIDE=$PWD/paper_2503_08264_b200/$lib.so; fi
    env $env timeout 300 python bench.py --config ${CFG:-4} --no-cpu --no-variants --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels_ms']; print('$sp', round(d['ms_per_step'],3), round(k['forward'],3), round(k['backward'],3), round(d['roofline']['frac'],4))"
  done
done
