#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 python tools/diag_c4tc.py 1000 14 > gpurun_out/diag_tc.log 2>&1; cat gpurun_out/diag_tc.log
timeout 1200 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_qem.py tests/test_gpu_sharded.py -q -rf > gpurun_out/t_d.log 2>&1
tail -8 gpurun_out/t_d.log
