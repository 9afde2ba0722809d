# ncu --set full captures of the hot kernels (one kernel per capture, steady-state launch)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/iter_profile.py --config 5 --iters 13 > gpurun_out/iter_c5.log 2>&1
timeout 300 python tools/iter_profile.py --config 4 --iters 13 > gpurun_out/iter_c4.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
for k in k_forward_tc k_backward_tc k_colprep k_sample; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o gpurun_out/ncu_c5_$k $B --config 5 > gpurun_out/ncu_c5_$k.log 2>&1
done
for k in k_forward k_backward; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${k}<" -s 4 -c 1 -o gpurun_out/ncu_c4_$k $B --config 4 > gpurun_out/ncu_c4_$k.log 2>&1
done
ls -la gpurun_out
