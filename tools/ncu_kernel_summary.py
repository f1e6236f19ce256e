"""Launch configuration and pipe utilisation of every kernel in ncu reports:
python tools/ncu_kernel_summary.py A.ncu-rep [B.ncu-rep ...].  Development aid."""
import csv,subprocess,sys
want=['Kernel Name','gpu__time_duration.sum','launch__grid_size','launch__block_size','launch__cluster_dim_x','launch__registers_per_thread','launch__shared_mem_per_block_dynamic','launch__occupancy_limit_registers','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active','sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__cycles_elapsed.avg.per_second','smsp__inst_executed.sum','dram__bytes_read.sum','dram__bytes_write.sum','sm__throughput.avg.pct_of_peak_sustained_elapsed','smsp__average_warp_latency_issue_stalled_barrier','smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct','smsp__inst_executed_pipe_xu.sum','smsp__sass_thread_inst_executed_op_fp32_pred_on.sum','smsp__inst_executed_op_mufu_ex2.sum']
for f in sys.argv[1:]:
    out=subprocess.run(['ncu','-i',f,'--page','raw','--csv'],capture_output=True,text=True).stdout
    rows=list(csv.reader([l for l in out.splitlines() if l.startswith('"')]))
    h,u=rows[0],rows[1]
    for v in rows[2:]:
        print('==',f)
        for w in want:
            if w in h:
                i=h.index(w); print(f'  {w:70s} {v[i][:90]} {u[i]}')
