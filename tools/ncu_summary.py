import csv, subprocess, sys
KEYS=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','launch__registers_per_thread','launch__occupancy_limit_registers','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__inst_executed.sum','smsp__inst_executed.sum','sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed','smsp__thread_inst_executed_per_inst_executed.ratio','launch__grid_size','launch__block_size','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active']
def summ(path):
    out=subprocess.run(['ncu','-i',path,'--page','raw','--csv'],capture_output=True,text=True).stdout
    rows=list(csv.reader(out.splitlines()))
    hdr=rows[0]; units=rows[1]
    res=[]
    for vals in rows[2:]:
        d={h:(v,u) for h,u,v in zip(hdr,units,vals)}
        r={'kernel':d.get('Kernel Name',('?',''))[0][:70]}
        for k in KEYS:
            if k in d: r[k]=d[k][0]+' '+d[k][1]
        st={}
        for h in hdr:
            if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued'):
                try: st[h.replace('smsp__pcsamp_warps_issue_stalled_','')]=float(d[h][0])
                except: pass
        tot=sum(st.values()) or 1
        r['stalls_pct']={k:round(100*v/tot,1) for k,v in sorted(st.items(),key=lambda x:-x[1])[:8]}
        res.append(r)
    return res
for p in sys.argv[1:]:
    for r in summ(p):
        print('==',p)
        for k,v in r.items(): print('  ',k,':',v)
