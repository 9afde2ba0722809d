#!/bin/bash
# parity subset on the default library, then the interleaved A/B of tools/gpu_ab.sh, then the
# parity subset again on each variant named in CHECK
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity.py} -q -x 2>&1 | tail -3
CFG=${CFG:-4} bash tools/gpu_ab.sh
for v in $CHECK; do
  echo "check $v"
  QEM_LIB_OVERRIDE=$PWD/paper_2503_08264_b200/$v.so timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity.py} -q -x 2>&1 | tail -3
done
