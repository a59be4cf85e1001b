"""Summarise an ncu --set full capture of the histogram kernels into profiles/ (md + json).
usage: ncu_hist_summary.py REPORT TAG [capture description]"""
import csv, subprocess, io, json, sys
rep, tag = sys.argv[1], sys.argv[2]
capture = sys.argv[3] if len(sys.argv) > 3 else "bench.py --steps 3 --warmup 3, Higgs 11M x 28, one round = root + 5 level launches"
PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6546.6
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
def tous(x):
    v,u=x.split(' ',1); v=float(v.replace(',',''))
    return v*{'nsecond':1e-3,'usecond':1.0,'msecond':1e3,'ns':1e-3,'us':1.0,'ms':1e3}[u.strip()]
times=[tous(d['time']) for d in out]
for d,t,us in zip(out,tr,times):
    d['dpct']=f"{100*t/(us*1e-6)/1e9/PEAK:.1f} %"
summary={"source":f"ncu --set full (profiles/{tag}_ncu_hist_summary.md): {capture}",
         "dram_bytes_per_launch": sum(tr)/len(tr),
         "l1tex_pct_of_peak_active_mean": sum(v for v in l1 if v is not None)/max(1,len([v for v in l1 if v is not None])),
         "launches": [ {"kernel":d['kernel'], "dram_bytes": t, "time_us": us, "l1tex_pct_active": l, "smem_atom_wavefronts": tof(d['aw']),
                        "smem_atom_bank_conflicts": tof(d['ac'])} for d,t,l,us in zip(out,tr,l1,times)]}
json.dump(summary, open('profiles/ncu_hist_higgs.json','w'), indent=1)
lines=[f"# {tag} ncu --set full: histogram kernels, one boosting round (Higgs-shaped 11M x 28, depth 6)","",
f"Capture: {capture}.  DRAM % of peak = (read + write) / duration / {PEAK} GB/s (MEASURED_PEAKS.json).  The .ncu-rep",
"stays in gpurun_out/ (scratch); this table is the committed summary.","",
"| launch | kernel | time | DRAM read | DRAM write | DRAM % of peak | L1/TEX % (active) | smem atom wavefronts | of which bank conflicts | warp instr | regs | dyn smem |",
"|---|---|---|---|---|---|---|---|---|---|---|---|"]
for i,d in enumerate(out):
    lines.append('| '+' | '.join([str(i)]+[d[k] for k in ['kernel','time','rd','wr','dpct','l1','aw','ac','inst','regs','smem']])+' |')
lines+=["",f"Average DRAM traffic per histogram launch: {sum(tr)/len(tr)/1e6:.1f} MB (bench.py `roofline.traffic`)."]
open(f'profiles/{tag}_ncu_hist_summary.md','w').write("\n".join(lines)+"\n")
print("\n".join(lines))
