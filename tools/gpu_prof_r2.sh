#!/bin/bash
# Profiles of the current build (round 2): launch lists (c5, c4), ncu --set full of the main kernels,
# per-config DRAM traffic json, text summaries.  Each ncu command only after the same bench exits 0.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=${TAG:-r02}
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-variants"
for c in 5 4; do
  timeout 300 $B --config $c > gpurun_out/prof_b$c.json 2>&1 || { echo "bench c$c failed"; tail -5 gpurun_out/prof_b$c.json; exit 1; }
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_c$c.csv $B --config $c > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/${TAG}_launches_c$c.csv > gpurun_out/${TAG}_launches_c${c}_summary.txt 2>&1
done
K5=${K5:-"k_forward_tc k_backward_tc k_colprep_tc k_sample"}
for k in $K5; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"^$k\$" -s 4 -c 1 -o gpurun_out/ncu_c5_$k $B --config 5 > /dev/null 2>&1
done
K4=${K4:-"k_forward k_backward"}
for k in $K4; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"^$k\$" -s 4 -c 1 -o gpurun_out/ncu_c4_$k $B --config 4 > /dev/null 2>&1
done
rm -f gpurun_out/${TAG}_traffic.json
python tools/ncu_traffic.py gpurun_out/${TAG}_traffic.json --config 5 gpurun_out/ncu_c5_*.ncu-rep > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/${TAG}_traffic.json --config 4 gpurun_out/ncu_c4_*.ncu-rep > /dev/null 2>&1
for r in gpurun_out/ncu_c5_*.ncu-rep gpurun_out/ncu_c4_*.ncu-rep; do
  n=$(basename $r .ncu-rep); python tools/ncu_summary.py $r > gpurun_out/${TAG}_$n.summary.txt 2>&1; python tools/ncu_hot.py $r 25 >> gpurun_out/${TAG}_$n.summary.txt 2>&1
done
rm -f gpurun_out/ncu_c5_k_colprep_tc.ncu-rep gpurun_out/ncu_c5_k_sample.ncu-rep gpurun_out/ncu_c4_*.ncu-rep
cat gpurun_out/${TAG}_launches_c5_summary.txt gpurun_out/${TAG}_launches_c4_summary.txt
for f in gpurun_out/${TAG}_ncu_*.summary.txt; do echo "== $f"; head -30 $f; done
