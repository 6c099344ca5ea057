"""Summarise tools/ab_lib.sh output: best-of-reps time per width for the base and the new build."""
import collections, json, sys
for path in sys.argv[1:]:
    d = collections.defaultdict(list)
    for l in open(path):
        if l.startswith('{'):
            r = json.loads(l); d[(r['k'], r['lib'])].append(r['ms'])
    tb = tn = 0
    for k in sorted({k for k, _ in d}, reverse=True):
        b = min(d[(k, 'base')]); nw = min(d[(k, 'new')]); tb += b; tn += nw
        print(path.split('/')[-1], k, 'base %.3f new %.3f ratio %.4f' % (b, nw, nw / b))
    print('total ratio %.4f' % (tn / tb))
