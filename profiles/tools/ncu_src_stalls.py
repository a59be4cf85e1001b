"""Source lines ranked by warp-stall samples (all files) for one launch of an ncu report (scratch).
usage: ncu_src_stalls.py REPORT KERNEL_REGEX LAUNCH_SKIP [N]"""
import csv, io, subprocess, sys
rep, regex, skip = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
raw = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass', '-k', f'regex:{regex}',
                      '--launch-skip', skip, '--launch-count', '1'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
L, fname, h = [], "?", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Name":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        h = r
    elif h and r[0].isdigit():
        try:
            sm = int(r[h.index('Warp Stall Sampling (All Samples)')] or 0)
            ie = int(r[h.index('Instructions Executed')] or 0)
        except (ValueError, IndexError):
            continue
        L.append((sm, ie, fname, r[0], r[1][:110]))
ts = sum(x[0] for x in L) or 1
ti = sum(x[1] for x in L) or 1
print("samples", ts, "inst", ti)
for x in sorted(L, reverse=True)[:n]:
    print(f"smp {100*x[0]/ts:5.1f}%  inst {100*x[1]/ti:5.1f}%  {x[2]}:{x[3]:>5} {x[4]}")
