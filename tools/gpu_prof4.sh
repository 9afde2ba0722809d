python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 120 python -m pytest --timeout=100 -x -q tests/test_gpu_tc.py -k "n40_K256" > gpurun_out/guard.log 2>&1 || { echo guard failed; exit 1; }
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --config 5"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_forward_tc -s 4 -c 1 -o gpurun_out/ncu_fwd7 $B > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_backward_tc -s 4 -c 1 -o gpurun_out/ncu_bwd7 $B > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_root -s 8 -c 2 -o gpurun_out/ncu_root7 $B > /dev/null 2>&1
bash tools/gpu_variants.sh QEM_POLY_EXP_BWD=2 QEM_POLY_EXP_BWD=6
