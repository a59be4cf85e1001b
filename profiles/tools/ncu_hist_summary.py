"""Summarise an ncu --set full capture of the histogram kernels into profiles/ (md + json)."""
import csv, subprocess, io, json, sys
rep, tag = sys.argv[1], sys.argv[2]
raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(io.StringIO(raw))); hdr=rows[0]; units=rows[1]
def find(name):
    for h in hdr:
        if h==name or h.endswith('.'+name): return hdr.index(h)
    raise KeyError(name)
keys={'time':'gpu__time_duration.sum','rd':'dram__bytes_read.sum','wr':'dram__bytes_write.sum','dpct':'dram__throughput.avg.pct_of_peak_sustained_elapsed',
'l1':'l1tex__throughput.avg.pct_of_peak_sustained_active','aw':'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum','ac':'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum',
'inst':'inst_executed','regs':'launch__registers_per_thread','smem':'launch__shared_mem_per_block_dynamic'}
out=[]
for r in rows[2:]:
    d={'kernel': r[hdr.index('Kernel Name')].split('(')[0].replace('void ','').replace('gbm::','')}
    for k,m in keys.items():
        i=find(m); d[k]=(r[i]+' '+units[i]).strip()
    out.append(d)
def tob(s):
    v,u=s.split(' ',1); v=float(v.replace(',',''))
    return v*{'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}[u.strip()]
tr=[tob(d['rd'])+tob(d['wr']) for d in out]
def tof(x):
    try: return float(x.split(' ')[0].replace(',',''))
    except Exception: return None
l1=[tof(d['l1']) for d in out]
summary={"source":f"ncu --set full (profiles/{tag}_ncu_hist_summary.md): bench.py --steps 3 --warmup 3, Higgs 11M x 28, one round = root + 5 level launches",
         "dram_bytes_per_launch": sum(tr)/len(tr),
         "l1tex_pct_of_peak_active_mean": sum(v for v in l1 if v is not None)/max(1,len([v for v in l1 if v is not None])),
         "launches": [ {"kernel":d['kernel'], "dram_bytes": t, "l1tex_pct_active": l, "smem_atom_wavefronts": tof(d['aw']),
                        "smem_atom_bank_conflicts": tof(d['ac'])} for d,t,l in zip(out,tr,l1)]}
json.dump(summary, open('profiles/ncu_hist_higgs.json','w'), indent=1)
lines=[f"# {tag} ncu --set full: histogram kernels, one boosting round (Higgs-shaped 11M x 28, depth 6)","",
"Capture: `ncu --set full --clock-control none --import-source on -k regex:\"hist_cs_range|hist_range|part_hist\" -s 6 -c 6`",
"on `python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline` (round 2: root + levels 1..5).  The .ncu-rep",
"stays in gpurun_out/ (scratch); this table is the committed summary.","",
"| launch | kernel | time | DRAM read | DRAM write | DRAM % of peak | L1/TEX % (active) | smem atom wavefronts | of which bank conflicts | warp instr | regs | dyn smem |",
"|---|---|---|---|---|---|---|---|---|---|---|---|"]
for i,d in enumerate(out):
    lines.append('| '+' | '.join([str(i)]+[d[k] for k in ['kernel','time','rd','wr','dpct','l1','aw','ac','inst','regs','smem']])+' |')
lines+=["",f"Average DRAM traffic per histogram launch: {sum(tr)/len(tr)/1e6:.1f} MB (bench.py `roofline.traffic`)."]
open(f'profiles/{tag}_ncu_hist_summary.md','w').write("\n".join(lines)+"\n")
print("\n".join(lines))
