python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for case in "161 256 10" "161 256 3" "40 256 1"; do
  echo "== $case TC"; timeout 120 python tools/diag_tc.py $case
  echo "== $case FFMA"; QEM_NO_TC=1 timeout 120 python tools/diag_tc.py $case
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_backward_tc -s 4 -c 1 -o gpurun_out/ncu_bwd_aux python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bwd_aux.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_forward_tc -s 4 -c 1 -o gpurun_out/ncu_fwd3 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_fwd3.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_colprep_tc -s 4 -c 1 -o gpurun_out/ncu_colprep3 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_colprep3.log 2>&1
ls gpurun_out
