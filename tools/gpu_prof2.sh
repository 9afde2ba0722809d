python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_backward_tc -s 4 -c 1 -o gpurun_out/ncu_bwd4 $B --config 5 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_colprep_tc -s 4 -c 1 -o gpurun_out/ncu_colprep4 $B --config 5 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_forward_tc -s 4 -c 1 -o gpurun_out/ncu_fwd4 $B --config 5 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"^k_forward$" -s 4 -c 1 -o gpurun_out/ncu_c4fwd4 $B --config 4 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_sample -s 4 -c 1 -o gpurun_out/ncu_sample4 $B --config 5 > /dev/null 2>&1
timeout 300 python bench.py --config 5 --no-cpu --no-e2e
ls gpurun_out
