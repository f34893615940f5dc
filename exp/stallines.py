import csv,gzip,collections,sys
name=sys.argv[1]; cols=sys.argv[2].split(",")
fh=gzip.open(f"gpurun_out/ncu_{name}_src.csv.gz","rt")
hdr=None;cur=None;agg=collections.defaultdict(collections.Counter);src={}
for r in csv.reader(fh):
    if not r: continue
    if r[0]=="File Path": cur=r[1].split("/")[-1]; continue
    if r[0]=="Line No": hdr={h:i for i,h in enumerate(r)}; continue
    if hdr is None or not r[0].isdigit(): continue
    k=(cur,int(r[0])); src[k]=r[1][:70]
    for c in cols:
        try: agg[k][c]+=int(float(r[hdr[c]]))
        except: pass
for c in cols:
    tot=sum(v[c] for v in agg.values()) or 1
    print("==",c,tot)
    for k,v in sorted(agg.items(),key=lambda kv:-kv[1][c])[:10]:
        print(f"  {100*v[c]/tot:5.1f}% {k[0]}:{k[1]} {src[k]}")
