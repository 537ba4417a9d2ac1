"""Compact summary of one ncu --set full capture (profiles/ write-ups).

    python tools/ncu_summary.py gpurun_out/prof_v7.ncu-rep [top_lines]
Prints duration, DRAM bytes, instructions/IPC, the warp-stall mix and the
source lines with the most stall samples.
"""
import csv,sys,subprocess
rep=sys.argv[1]
IDX=int(sys.argv[3]) if len(sys.argv)>3 else 0  # which captured launch
sel=['--launch-skip',str(IDX),'--launch-count','1']
raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
r=list(csv.reader(raw.splitlines())); h=r[0]; v=r[2+IDX]
def g(k):
    return v[h.index(k)] if k in h else None
print('dur', g('gpu__time_duration.sum'), 'inst', g('smsp__inst_executed.sum'), 'ipc', g('sm__inst_executed.avg.per_cycle_active'))
U=r[1]
def gu(k):
    return (v[h.index(k)] + " " + U[h.index(k)]) if k in h else None
print("dram read", gu("dram__bytes_read.sum"), "write", gu("dram__bytes_write.sum"))
tot=0; out=[]
for i,k in enumerate(h):
  if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('_not_issued'):
    try: x=float(v[i].replace(',','')); out.append((x,k[33:])); tot+=x
    except: pass
print(' '.join(f'{k}:{100*x/tot:.1f}%' for x,k in sorted(out,reverse=True)[:9]))
src=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source=cuda,sass']+sel,capture_output=True,text=True).stdout
rows=list(csv.reader(src.splitlines()))
f=None; agg=[]
for x in rows:
    if x and x[0]=='File Path': f=x[1].split('/')[-1]; continue
    if len(x)>=10 and x[0] and x[0]!='Line No' and x[2]=='-':
        try: agg.append((int(x[4]), int(x[7]), f, x[0], x[1][:90]))
        except: pass
ts=sum(a[0] for a in agg); ti=sum(a[1] for a in agg)
N=int(sys.argv[2]) if len(sys.argv)>2 else 25
for a in sorted(agg, key=lambda x:-x[0])[:N]:
    print(f"{a[0]*100/ts:5.1f}%st {a[1]*100/ti:5.1f}%in {a[2]}:{a[3]} {a[4]}")
