#!/bin/bash
# Round-end evidence on the committed build: the driver's own pytest line, smoke, the three bench arms
# (config 5 default, config 4, reference), the 1-rank torchrun launch, the sharding proxy.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
( time timeout 1500 python -m pytest tests/ -x -q -m gpu --durations=8 ) > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?"; tail -14 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_final.log
timeout 600 python bench.py > gpurun_out/r02_bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench5 rc=$?"
timeout 600 python bench.py --config 4 > gpurun_out/r02_bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench4 rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r02_bench_reference_c5.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu --no-variants > gpurun_out/r02_bench_c5_torchrun1.json 2> gpurun_out/bench_tr.err; echo "torchrun1 rc=$?"
timeout 600 python tools/shard_proxy.py 5 4 > gpurun_out/r02_shard_proxy.json 2> gpurun_out/shard.err; echo "shard proxy rc=$?"
cat gpurun_out/r02_shard_proxy.json
python - <<'P'
import json
for f in ("r02_bench_c5", "r02_bench_c4", "r02_bench_reference_c5", "r02_bench_c5_torchrun1"):
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        r = d.get("roofline", {})
        print(f, round(d["ms_per_step"], 3), d["value"], r.get("frac"), r.get("traffic"), r.get("kernels_ms"), d.get("e2e", {}).get("ms_per_step"), d.get("clocks"))
    except Exception as e:
        print(f, "unreadable", e)
P
