#!/bin/bash
# round-2 check b: compact (d = 1) tensor-core path, eps-bank qem_iterate parity, sharded details
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "n40_K256_post1 and compact" > gpurun_out/guard_b.log 2>&1 || { echo guard failed; tail -40 gpurun_out/guard_b.log; }
timeout 600 python -m pytest tests/test_gpu_sharded.py -q -x -k "virtual_ranks and tc_d16" > gpurun_out/t_sharded_tc.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_qem.py tests/test_gpu_sharded.py -q -rf > gpurun_out/t_b.log 2>&1
tail -30 gpurun_out/t_b.log
timeout 300 python bench.py --config 4 --no-cpu --no-variants --no-e2e > gpurun_out/bench_b4.json 2> gpurun_out/bench_b4.err
timeout 300 python bench.py --config 5 --no-cpu --no-variants --no-e2e > gpurun_out/bench_b5.json 2> gpurun_out/bench_b5.err
python - <<'P'
import json
for f in ("gpurun_out/bench_b4.json", "gpurun_out/bench_b5.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["frac"], d["roofline"]["kernels_ms"])
        for k, v in d["variants"].items():
            print("  ", k, v.get("ms_per_step"), v["roofline"]["kernel"], v["roofline"]["frac"], v["roofline"]["kernels_ms"])
    except Exception as e:
        print(f, "ERR", e)
P
