"""Per-source-line instruction counts of one captured launch: python tools/ncu_lines.py rep [top] [records]"""
import csv,subprocess,sys
rep=sys.argv[1]; N=int(sys.argv[2]) if len(sys.argv)>2 else 50; recs=float(sys.argv[3]) if len(sys.argv)>3 else 100e6
src=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source=cuda,sass','--launch-skip','0','--launch-count','1'],capture_output=True,text=True).stdout
rows=list(csv.reader(src.splitlines()))
f=None; agg=[]
for x in rows:
    if x and x[0]=='File Path': f=x[1].split('/')[-1]; continue
    if len(x)>=10 and x[0] and x[0]!='Line No' and x[2]=='-':
        try: agg.append((int(x[4]), int(x[7]), f, x[0], x[1][:100]))
        except: pass
ti=sum(a[1] for a in agg)
print('warp instr', ti, 'thread-instr/record', ti*32/recs)
for a in sorted(agg, key=lambda x:-x[1])[:N]:
    print(f"{a[1]*100/ti:5.1f}%in {a[1]/recs*32:6.1f}/rec {a[2]}:{a[3]} {a[4]}")
