# Full evidence pass: gpu tests, smoke, bench (config 5 default + config 4 + reference arm), launch lists,
# ncu --set full of the dominant kernels -> text summaries + traffic json (reports deleted on the box
# except the two pair kernels: gpurun copies back at most 64 MiB).
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 120 python -m pytest --timeout=100 -x -q tests/test_gpu_tc.py -k "n40_K256" > gpurun_out/guard.log 2>&1 || { echo guard failed; tail -20 gpurun_out/guard.log; exit 1; }
timeout 1500 python -m pytest --timeout=240 tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench5 rc=$?"
timeout 400 python bench.py --config 4 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench4 rc=$?"
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
cat gpurun_out/bench_c5.json gpurun_out/bench_c4.json gpurun_out/bench_ref.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-variants > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config 4 --steps 2 --warmup 3 --no-cpu --no-e2e --no-variants > /dev/null 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-variants"
for k in k_backward_tc k_forward_tc k_colprep_tc k_sample; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o gpurun_out/ncu_c5_$k $B --config 5 > /dev/null 2>&1
done
for k in k_forward k_backward; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"^$k\$" -s 4 -c 1 -o gpurun_out/ncu_c4_$k $B --config 4 > /dev/null 2>&1
done
rm -f gpurun_out/traffic.json
python tools/ncu_traffic.py gpurun_out/traffic.json gpurun_out/ncu_c5_*.ncu-rep gpurun_out/ncu_c4_*.ncu-rep > /dev/null 2>&1
for r in gpurun_out/ncu_c5_*.ncu-rep gpurun_out/ncu_c4_*.ncu-rep; do
  n=$(basename $r .ncu-rep); python tools/ncu_summary.py $r > gpurun_out/$n.summary.txt 2>&1; python tools/ncu_hot.py $r 25 >> gpurun_out/$n.summary.txt 2>&1
done
rm -f gpurun_out/ncu_c5_k_colprep_tc.ncu-rep gpurun_out/ncu_c5_k_sample.ncu-rep gpurun_out/ncu_c4_*.ncu-rep
du -sh gpurun_out; ls gpurun_out
