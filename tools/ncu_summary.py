import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]; v = r[2]
def g(k):
    return v[h.index(k)] if k in h else None
keys = ['gpu__time_duration.sum','sm__throughput.avg.pct_of_peak_sustained_elapsed','sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active','sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','dram__bytes_read.sum','dram__bytes_write.sum','launch__grid_size','launch__block_size','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem','smsp__inst_executed.sum','sm__sass_thread_inst_executed_op_ffma_pred_on.sum','sm__sass_thread_inst_executed_op_fadd_pred_on.sum','sm__sass_thread_inst_executed_op_fmul_pred_on.sum']
for k in keys:
    print(k, g(k))
items=[(k,v[i]) for i,k in enumerate(h) if 'smsp__average_warp' in k and 'issue_stalled' in k and 'ratio' in k]
items=sorted(items,key=lambda x:-float(x[1] or 0))[:8]
for k,x in items: print(k.replace('smsp__average_warps_issue_stalled_','stall_').replace('_per_issue_active.ratio',''),x)
