# TC path: build, parity (tc sweep + c5 cases), then bench config 5
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest --timeout=240 tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "tc rc=$?"; tail -30 gpurun_out/pytest_tc.log
timeout 900 python -m pytest --timeout=240 tests -x -q -m gpu -k "c5 or tc or config5" > gpurun_out/pytest_c5.log 2>&1; echo "c5 rc=$?"; tail -5 gpurun_out/pytest_c5.log
timeout 300 python tools/iter_profile.py --config 5 --iters 6 > gpurun_out/iter_c5.log 2>&1; head -6 gpurun_out/iter_c5.log
timeout 300 python bench.py --config 5 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench rc=$?"; cat gpurun_out/bench_c5.json; tail -5 gpurun_out/bench_c5.err
