set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench5 rc=$?"
timeout 300 python bench.py --config 4 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench4 rc=$?"
cat gpurun_out/bench_c5.json gpurun_out/bench_c4.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --config 5 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_c5.log 2>&1; echo "ncu rc=$?"
