#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
QEM_NO_TC1=1 timeout 600 python tools/diag_c4tc.py 1000 12 2>&1 | grep "^t=" | tail -4
timeout 1500 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_qem.py tests/test_gpu_sharded.py tests/test_gpu_flags.py tests/test_gpu_fresh.py tests/test_gpu_invariance.py "tests/test_gpu_fullsize.py::test_config4_full_size" -q -rf > gpurun_out/t_f.log 2>&1
tail -12 gpurun_out/t_f.log
timeout 300 python bench.py --config 4 --no-cpu --no-variants --no-e2e > gpurun_out/bench_f4.json 2> gpurun_out/bench_f4.err
timeout 300 python bench.py --config 5 --no-cpu --no-variants --no-e2e > gpurun_out/bench_f5.json 2> gpurun_out/bench_f5.err
python - <<'P'
import json
for f in ("gpurun_out/bench_f4.json", "gpurun_out/bench_f5.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["ms_per_step"], 3), d["roofline"]["kernel"], round(d["roofline"]["frac"], 4), d["roofline"]["kernels_ms"])
    except Exception as e:
        print(f, "ERR", e, open(f.replace("json", "err")).read()[-2000:])
P
