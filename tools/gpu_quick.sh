set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest --timeout=240 tests/test_gpu_tc.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_q.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/pytest_q.log
timeout 300 python tools/iter_profile.py --config 5 --iters 5 2>&1 | head -5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c5.csv python bench.py --config 5 --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_c5.csv
