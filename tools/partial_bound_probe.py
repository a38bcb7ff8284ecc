"""How many walked rows could stop after a prefix of their dimensions?  For
100 queries at 10M rows (lifted, C=8, D=350, k=10, CPU oracle), the fraction of
window entries whose partial squared distance over the first m dims already
exceeds the running top-10 threshold (a valid lower bound: every term is >= 0).
Measured: m = 16 / 32 / 48 / 64 / 96 -> 0.38 / 0.39 / 0.43 / 0.56 / 0.85.  The
two-stage kernel built on it (first 64 bytes, then the second 64 only for rows
still below the threshold) was slower on the B200 -- 7.57 vs 5.12 ms per
launch -- and read MORE DRAM bytes (40.2 vs 31.2 GB; any L2 fetch-granularity
hint: same), see DESIGN.md §4."""
import numpy as np, sys, time
sys.path.insert(0,'/root/repo')
from oracle import pyoracle as P
n=10_000_000
t=time.time()
rows=P.gen_rows(0,n)
qs=P.gen_queries(0,100,n)
oi=P.Oracle(P.view_floats(rows,1),8,16)
print('built', time.time()-t, flush=True)
r,b,e=oi.windows(P.view_floats(qs,1),350)
sorted_ids=[oi.sorted(c)[1] for c in range(8)]
tot=0; rej={16:0,32:0,48:0,64:0,96:0}
for q in range(100):
    walk=[]
    for c in range(8):
        walk+=list(sorted_ids[c][b[q,c]:e[q,c]])
    walk=np.array(walk,dtype=np.int64)
    R=rows[walk].astype(np.int32); Q=qs[q].astype(np.int32)
    d=(R-Q)**2
    full=d.sum(1)
    parts={m:d[:,:m].sum(1) for m in rej}
    seen=set(); top=[]; thr=np.inf
    for i,(row,f) in enumerate(zip(walk,full)):
        tot+=1
        for m in rej:
            if parts[m][i]>thr: rej[m]+=1
        if row in seen: continue
        seen.add(row)
        top.append(f); top.sort(); top=top[:10]
        if len(top)==10: thr=top[-1]
print({m: round(v/tot,3) for m,v in rej.items()})
