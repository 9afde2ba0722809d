# ncu --set full of one named kernel (KREG regex, default k_colprep_tc), summarised on the box
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 120 python -m pytest --timeout=100 -x -q tests/test_gpu_tc.py -k "n40_K256" > gpurun_out/guard.log 2>&1 || { echo guard failed; exit 1; }
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e ${VARIANTS:---no-variants} --config ${CFG:-5}"
K=${KREG:-k_colprep_tc}
rm -f /tmp/ncu_k.ncu-rep
timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-4} -c 1 -o /tmp/ncu_k $B > gpurun_out/ncu_k.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_k.log
python tools/ncu_summary.py /tmp/ncu_k.ncu-rep > gpurun_out/ncu_k_summary.txt 2>&1
python tools/ncu_hot.py /tmp/ncu_k.ncu-rep >> gpurun_out/ncu_k_summary.txt 2>&1
cp /tmp/ncu_k.ncu-rep gpurun_out/ 2>/dev/null
cat gpurun_out/ncu_k_summary.txt | head -60
