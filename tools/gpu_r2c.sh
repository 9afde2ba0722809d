#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 python tools/diag_c4tc.py 1000 14 > gpurun_out/diag_tc.log 2>&1
QEM_NO_TC1=1 timeout 600 python tools/diag_c4tc.py 1000 14 > gpurun_out/diag_ffma.log 2>&1
cat gpurun_out/diag_tc.log gpurun_out/diag_ffma.log
