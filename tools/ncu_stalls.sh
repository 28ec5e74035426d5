#!/bin/bash
# usage: tools/ncu_stalls.sh <report.ncu-rep>  — stall-sample breakdown + key SOL metrics
ncu -i "$1" --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]; v=rows[2] if len(rows)>2 else rows[1]
d=dict(zip(h,v))
tot=0; st={}
for k in d:
    if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued'):
        try: st[k[33:]]=float(d[k]); tot+=float(d[k])
        except: pass
for k,x in sorted(st.items(), key=lambda kv:-kv[1])[:10]: print('%-28s %6.1f%%' % (k, 100*x/tot))
for k in ['gpu__time_duration.sum','sm__inst_executed.avg.per_cycle_active','smsp__issue_active.avg.pct_of_peak_sustained_active','smsp__warps_active.avg.per_cycle_active','smsp__warps_eligible.avg.per_cycle_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum','smsp__inst_executed.sum','launch__registers_per_thread']:
    print(k, d.get(k))
"
