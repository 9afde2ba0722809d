python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --config 5"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_backward_tc -s 4 -c 1 -o gpurun_out/ncu_bwd6 $B > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_forward_tc -s 4 -c 1 -o gpurun_out/ncu_fwd6 $B > /dev/null 2>&1
ls gpurun_out | grep 6
