"""Summarise an ncu --page raw --csv export: stall breakdown + key throughput metrics."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
st = [(h, float(v.replace(',', ''))) for h, (v, u) in d.items()
      if 'warps_issue_stalled' in h and 'pcsamp' in h and 'not_issued' not in h]
st = [x for x in st if x[1] > 0]
st.sort(key=lambda x: -x[1])
tot = sum(v for _, v in st) or 1
for h, v in st[:8]:
    print(f"{100*v/tot:5.1f}% {h.replace('smsp__pcsamp_warps_issue_stalled_','stall_')}")
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'smsp__inst_executed.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active']
for k in keys:
    if k in d:
        print(f"{k} = {d[k][0]} {d[k][1]}")
