import csv, sys, collections
rows=list(csv.reader(open(sys.argv[1])))
h=None
for i,r in enumerate(rows):
    if r and r[0]=='Line No': h=r; start=i; break
iS=h.index('Warp Stall Sampling (All Samples)')
iI=h.index('Instructions Executed')
stall_cols=[(j,c) for j,c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
agg=collections.OrderedDict(); cur=None; src={}
for r in rows[start+1:]:
    if not r: continue
    if r[0] and r[0].isdigit() and (len(r)<3 or not r[2]):
        cur=int(r[0]); src[cur]=r[1][:100]; continue
    if r[0] and r[0].isdigit():
        cur=int(r[0]); src[cur]=r[1][:100]
    try: v=float(r[iS]); n=float(r[iI] or 0)
    except: continue
    a=agg.setdefault(cur,[0,0,collections.Counter()])
    a[0]+=v; a[1]+=n
    for j,c in stall_cols:
        try: a[2][c]+=float(r[j] or 0)
        except: pass
tot=sum(a[0] for a in agg.values()); toti=sum(a[1] for a in agg.values())
print('samples',tot,'inst',toti)
for l,a in sorted(agg.items(), key=lambda kv:-kv[1][0])[:int(sys.argv[2]) if len(sys.argv)>2 else 40]:
    top=', '.join(f"{k[6:]}:{int(v)}" for k,v in a[2].most_common(3))
    print(f"{100*a[0]/tot:5.1f}% smp {100*a[1]/toti:5.1f}% ins L{l}: {src.get(l,'')[:70]} | {top}")
