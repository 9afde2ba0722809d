#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in "" variant_sum2 variant_sum6; do
  if [ -n "$v" ]; then export QEM_LIB_OVERRIDE=$PWD/paper_2503_08264_b200/$v.so; fi
  echo "== ${v:-default}"
  timeout 300 python tools/iter_profile.py --config 5 --iters 14 2>&1 | grep "^t=" | sed -E 's/ *ms  logPe.*modes/ modes/'
done
