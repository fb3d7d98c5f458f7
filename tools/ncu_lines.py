import csv,sys,collections
rows=list(csv.reader(open(sys.argv[1])))
fn="";res=collections.Counter();src={}
hdr=None
for r in rows:
    if len(r)>=2 and r[0] in("File Path","File Name"): fn=r[1].split('/')[-1]; continue
    if r and r[0]=='Line No': hdr=r; I={k:i for i,k in enumerate(r)}; continue
    if hdr is None or len(r)<len(hdr) or not r[0]: continue
    try: ln=int(r[0])
    except: continue
    v=int(r[I['Instructions Executed']] or 0)
    res[(fn,ln)]+=v; src[(fn,ln)]=r[1][:80]
tot=sum(res.values()); print("total",tot)
for k,v in sorted(res.items()):
    if v>tot*0.004: print(f"{k[0][:12]}:{k[1]:4d} {v/1e6:7.2f}M {src[k]}")
