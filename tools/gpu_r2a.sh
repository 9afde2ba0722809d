#!/bin/bash
# round-2 GPU check: new sharded / iterate parity tests, full-size parity, the bench line
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
nproc > gpurun_out/nproc.txt
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_qem.py -q -rf 2>&1 | tail -40 > gpurun_out/t_sharded_qem.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -rf --durations=10 2>&1 | tail -40 > gpurun_out/t_fullsize.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
echo done
