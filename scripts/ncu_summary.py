"""Print the key metrics of an ncu report (raw page) for the sampler kernel."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
want = ['gpu__time_duration.sum', 'sm__inst_executed.sum', 'sm__inst_executed_pipe_fp64.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__pipe_fp64_cycles_active.avg.pct',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'sm__maximum_warps_per_active_cycle_pct', 'l1tex__t_sector_hit_rate.pct',
        'smsp__inst_executed_op_global_st.sum', 'smsp__inst_executed_op_global_ld.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_st.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'sm__inst_executed_pipe_lsu', 'sm__inst_executed_pipe_alu',
        'sm__inst_executed_pipe_fma', 'sm__inst_executed_pipe_xu', 'l1tex__throughput', 'lts__throughput',
        'sm__sass_thread_inst_executed.sum', 'smsp__sass_inst_executed.sum']
for i, n in enumerate(h):
    if any(n.startswith(w) for w in want) or ('issue_stalled' in n and n.endswith('per_issue_active.ratio')):
        if v[i] not in ('0', '0.000000', ''):
            print(f"{n:80s} {u[i]:>10s} {v[i]}")
