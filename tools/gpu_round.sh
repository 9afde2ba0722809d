# Full evidence pass: gpu tests, bench (config 5 default + config 4), launch lists, ncu --set full of the
# dominant kernels, traffic json.  Outputs land in gpurun_out/ (copied to profiles/ by hand).
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest --timeout=240 tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench5 rc=$?"
timeout 400 python bench.py --config 4 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench4 rc=$?"
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
cat gpurun_out/bench_c5.json gpurun_out/bench_c4.json gpurun_out/bench_ref.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config 4 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
for k in k_backward_tc k_forward_tc k_colprep_tc k_sample; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o gpurun_out/ncu_c5_$k $B --config 5 > /dev/null 2>&1
done
for k in k_forward k_backward; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"^$k\$" -s 4 -c 1 -o gpurun_out/ncu_c4_$k $B --config 4 > /dev/null 2>&1
done
ls gpurun_out
