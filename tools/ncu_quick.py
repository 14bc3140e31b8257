"""Quick per-kernel summary of an ncu report: time, DRAM bytes, issue/fp64 activity, top stalls."""
import csv
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active']
st = [h for h in hdr if re.match(r'smsp__average_warps_issue_stalled_.*_per_issue_active.ratio', h)]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(d['Kernel Name'][:80])
    print('   ', {k.split('__')[1][:24]: d[k] for k in keys})
    s = {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''): float(d[k]) for k in st}
    print('   ', {k: round(v, 2) for k, v in sorted(s.items(), key=lambda x: -x[1]) if v > 0.1})
