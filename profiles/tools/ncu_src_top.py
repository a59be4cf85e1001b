"""Top source lines by executed instructions for one launch of an ncu report (scratch)."""
import csv, io, subprocess, sys
rep, regex, skip = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass', '-k', f'regex:{regex}',
                      '--launch-skip', skip, '--launch-count', '1'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[hi]
ie = hdr.index("Instructions Executed"); sm = hdr.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows[hi + 1:]:
    try:
        if r[0].isdigit():
            lines.append((int(r[ie] or 0), int(r[sm] or 0), r[0], r[1][:110]))
    except Exception:
        pass
tot = sum(l[0] for l in lines); ts = sum(l[1] for l in lines)
print("total inst", tot, "samples", ts)
for l in sorted(lines, reverse=True)[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{l[0]:>10} {100*l[0]/tot:5.1f}% smp {100*l[1]/max(ts,1):5.1f}%  L{l[2]:>5} {l[3]}")
