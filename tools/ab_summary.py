import sys, json, collections
d = collections.defaultdict(list)
for ln in sys.stdin:
    if not (ln.startswith('base ') or ln.startswith('cur ')):
        continue
    lib, js = ln.split(' ', 1)
    j = json.loads(js)
    d[(j['kind'], j['L'], lib)].append(j['ms'])
for k, L in sorted(set((k, L) for k, L, _ in d)):
    b = min(d[(k, L, 'base')]); c = min(d[(k, L, 'cur')])
    print(f'{k:12s} L={L:2d} base {b:.4f} cur {c:.4f}  ratio {c / b:.3f}')
