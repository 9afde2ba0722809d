#!/bin/bash
# one ncu --set full capture of kernel $K on config $CFG (after the same bench exits 0 without ncu)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-variants --config ${CFG:-4}"
timeout 300 $B > gpurun_out/prof_b.json 2>&1 || { echo "bench failed"; tail -5 gpurun_out/prof_b.json; exit 1; }
for k in ${K:-k_forward}; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"^$k\$" -s 4 -c 1 -o gpurun_out/ncu_${TAG:-x}_$k $B > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/ncu_${TAG:-x}_$k.ncu-rep; python tools/ncu_hot.py gpurun_out/ncu_${TAG:-x}_$k.ncu-rep 10
done
