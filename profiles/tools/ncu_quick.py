"""Print key counters per launch of an ncu report (scratch analysis)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
names = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
         'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum',
         'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
         'smsp__issue_active.avg.pct_of_peak_sustained_active', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
         'sm__warps_active.avg.pct_of_peak_sustained_active', 'lts__t_sectors_op_read.sum']
ki = hdr.index('Kernel Name')
print('kernels:', [r[ki].split('(')[0][-40:] for r in rows[2:]])
for n in names + sys.argv[2:]:
    idx = [i for i, h in enumerate(hdr) if h == n]
    if not idx:
        print('missing', n); continue
    i = idx[0]
    print(f"{n:70s} {rows[1][i]:8s}", [r[i] for r in rows[2:]])
