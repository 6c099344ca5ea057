"""Summarise a CHFSI_K1_LOG trace (stderr of a bench/solve run): K1 time vs the DMMA-peak ideal by width and variant.
Usage: python tools/k1_log_summary.py <stderr file> [n]  (n defaults to 13000, the c2 size)"""
import collections, sys
rows=[l.split() for l in open(sys.argv[1]) if l.startswith('k1 ')]
# k1 rank R n N nloc N ka K variant V ms T
n=int(sys.argv[2]) if len(sys.argv)>2 else 13000
tot=0; ideal=0; byw=collections.defaultdict(lambda:[0,0,0]); byv=collections.defaultdict(lambda:[0,0,0])
for r in rows:
    d=dict(zip(r[1::2], r[2::2]))
    ka=int(d['ka']); v=int(d['variant']); ms=float(d['ms'])
    idl=6*n*n*ka/37.07e12*1e3 if v>=200 else 8*n*n*ka/37.07e12*1e3
    tot+=ms; ideal+=idl
    b=(ka//48)*48
    for D,key in ((byw,b),(byv,v)):
        D[key][0]+=ms; D[key][1]+=idl; D[key][2]+=1
print('launches',len(rows),'total ms %.1f ideal %.1f frac %.4f'%(tot,ideal,ideal/tot))
for name,D in (('width',byw),('variant',byv)):
    loss=sorted(((v[0]-v[1],k,v) for k,v in D.items()),reverse=True)
    for l,k,v in loss[:12]: print(name,k, 'n=%d'%v[2], 'ms=%.1f'%v[0], 'eff=%.3f'%(v[1]/v[0]), 'loss ms=%.1f'%l)
