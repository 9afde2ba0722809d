set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest --timeout=240 tests/test_gpu_tc.py -q -x > gpurun_out/pytest_tc.log 2>&1; echo "tc rc=$?"; tail -15 gpurun_out/pytest_tc.log
timeout 1500 python -m pytest --timeout=240 tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "gpu rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for c in 161:256:10 161:256:3; do a=(${c//:/ }); QEM_NO_TC=1 timeout 120 python tools/diag_tc.py ${a[0]} ${a[1]} ${a[2]}; done
timeout 300 python bench.py --config 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench rc=$?"; cat gpurun_out/bench_c5.json
timeout 300 python bench.py --config 4 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; cat gpurun_out/bench_c4.json
