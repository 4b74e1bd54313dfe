# key counters of one ncu report: bash tools/ncu_keys.sh REP
ncu -i "$1" --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
keys=['gpu__time_duration.sum','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','smsp__inst_executed.sum','smsp__sass_inst_executed_op_shared_ld.sum','smsp__sass_inst_executed_op_shared_st.sum','dram__bytes_read.sum','dram__bytes_write.sum','launch__registers_per_thread','sm__sass_thread_inst_executed_op_dfma_pred_on.sum','sm__sass_thread_inst_executed_op_dmul_pred_on.sum','sm__sass_thread_inst_executed_op_dadd_pred_on.sum']
d=dict(zip(h,v))
for k in keys: print(k, d.get(k))
st={n[33:]:float(v[i]) for i,n in enumerate(h) if n.startswith('smsp__pcsamp_warps_issue_stalled') and 'not_issued' not in n and v[i] not in ('','0')}
t=sum(st.values()); print('stalls:', ', '.join(f'{k} {100*x/t:.1f}%' for k,x in sorted(st.items(), key=lambda x:-x[1])[:9]))
"
