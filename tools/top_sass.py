#!/usr/bin/env python3
"""Top stall sites of an `ncu --page source --csv` export: tools/top_sass.py file.csv [n] [context]"""
import csv, sys
f=sys.argv[1]; n=int(sys.argv[2]) if len(sys.argv)>2 else 25; ctx=int(sys.argv[3]) if len(sys.argv)>3 else 0
rows=list(csv.reader(open(f)))
hdr=rows[1]; body=rows[2:]
ix={h:i for i,h in enumerate(hdr)}
S=ix['# Samples']
stalls=[h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot=sum(int(r[S] or 0) for r in body)
print('total samples',tot,'instructions',len(body))
agg={s:sum(int(r[ix[s]] or 0) for r in body) for s in stalls}
print({k:round(100*v/tot,1) for k,v in sorted(agg.items(), key=lambda kv:-kv[1])[:8]})
order=sorted(range(len(body)), key=lambda i:-int(body[i][S] or 0))[:n]
for i in sorted(order):
    r=body[i]
    top=sorted(((int(r[ix[s]] or 0),s[6:]) for s in stalls), reverse=True)[:2]
    for j in range(max(0,i-ctx), i):
        print('      ', j, body[j][ix['Source']].strip()[:90])
    print('%5.1f%% %5d %-70s %s wf=%s/%s'%(100*int(r[S])/tot, i, r[ix['Source']].strip()[:70], top, r[ix['L1 Wavefronts Shared']], r[ix['L1 Wavefronts Shared Ideal']]))
