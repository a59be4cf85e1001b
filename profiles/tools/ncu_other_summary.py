"""Table of an ncu --set full capture of the non-histogram kernels (profiles/r02/ncu_other_summary.md).
usage: ncu_other_summary.py REPORT > out.md"""
import csv, io, json, subprocess, sys
rep = sys.argv[1]
PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw))); hdr, units = rows[0], rows[1]
def col(r, name):
    for i, h in enumerate(hdr):
        if h == name:
            return r[i], units[i]
    raise KeyError(name)
def num(r, name, scale=None):
    v, u = col(r, name)
    v = float(v.replace(',', ''))
    if scale:
        v *= scale.get(u.strip(), 1.0)
    return v
T = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
B = {'byte': 1e-6, 'Kbyte': 1e-3, 'Mbyte': 1.0, 'Gbyte': 1e3}
print("| kernel | time us | DRAM read MB | DRAM write MB | DRAM % | warp instr | issue active % | warps active % | L1/TEX % | grid |")
print("|---|---|---|---|---|---|---|---|---|---|")
for r in rows[2:]:
    k = r[hdr.index('Kernel Name')].split('(')[0].replace('void ', '').replace('gbm::', '')
    t = num(r, 'gpu__time_duration.sum', T)
    rd = num(r, 'dram__bytes_read.sum', B); wr = num(r, 'dram__bytes_write.sum', B)
    pct = (rd + wr) * 1e6 / (t * 1e-6) / (PEAK * 1e9) * 100
    print(f"| {k} | {t:.1f} | {rd:.1f} | {wr:.1f} | {pct:.1f} | {num(r, 'smsp__inst_executed.sum') / 1e6:.2f}M | "
          f"{num(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f} | "
          f"{num(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} | "
          f"{num(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active'):.0f} | {num(r, 'launch__grid_size'):.0f} |")
