python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rp in 1 2; do echo "== QEM_RP=$rp"; QEM_RP=$rp timeout 300 python bench.py --config 4 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernels_ms'], d['roofline']['frac'])"; done
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --config 4"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"^k_forward$" -s 4 -c 1 -o gpurun_out/ncu_c4f8 $B > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu_c4f8.ncu-rep; python tools/ncu_hot.py gpurun_out/ncu_c4f8.ncu-rep 30
