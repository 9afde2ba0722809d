python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
# hang guard: one small tensor-core E-step first
timeout 120 python -m pytest --timeout=100 -x -q tests/test_gpu_tc.py -k "n40_K256" > gpurun_out/guard.log 2>&1; rc=$?; echo "guard rc=$rc"; if [ $rc -ne 0 ]; then tail -20 gpurun_out/guard.log; exit 1; fi
timeout 600 python -m pytest --timeout=240 tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_qem.py tests/test_gpu_fullsize.py -q -x -k "c5 or tc or config5 or d8 or sampler" > gpurun_out/pytest_q.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/pytest_q.log
timeout 300 python bench.py --config 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernels_ms'], d['roofline']['frac'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c5.csv python bench.py --config 5 --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_c5.csv
