cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo

for c in 4 5; do timeout 300 python bench.py --config $c --no-cpu --no-variants > gpurun_out/bench_e$c.json 2> gpurun_out/bench_e$c.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_e$c.json').read().strip().splitlines()[-1]); print($c, round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), round(d['e2e']['ms_per_step_same_loop_without_copies'],3))"; done
exit 0
timeout 300 python -c "
import sys, json, torch; sys.path.insert(0, '.')
import bench
print(json.dumps(bench.run_crossed_variant(torch.device('cuda', 0))))"
