#!/bin/bash
# round-2 late A/B: parity of the candidate variants on the tensor-core tests, then an interleaved
# config-5 A/B of the library variants (column-prep occupancy, forward lazy max, software-exp share)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in ${PARITY:-vlazy}; do
  QEM_LIB_OVERRIDE=$PWD/paper_2503_08264_b200/$v.so timeout 900 python -m pytest -q -x tests/test_gpu_tc.py tests/test_gpu_parity.py > gpurun_out/ab_par_$v.log 2>&1
  echo "$v parity rc=$? $(tail -1 gpurun_out/ab_par_$v.log)"
done
VARIANTS="${VARIANTS:-vprep3 vfwd4 vlazy vlazy4}" CFG=5 bash tools/gpu_ab.sh
