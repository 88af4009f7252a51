import sys, json, collections, re
d = collections.defaultdict(list)
for ln in sys.stdin:
    m = re.match(r'^\[([^\]]*=[^\]]*)\] (\{.*\})\s*$', ln)
    if not m:
        continue
    cfg, j = m.group(1), json.loads(m.group(2))
    if 'ms' not in j:
        continue
    d[(j['kind'], j['L'], j.get('C', 0), cfg)].append(j['ms'])
cfgs = sorted(set(c for *_, c in d))
for k, L, C in sorted(set(x[:3] for x in d)):
    print(f'{k:12s} L={L:2d}' + (f' C={C}' if C else '') + '  ' + '  '.join(f'{c}: {min(d[(k, L, C, c)]):.4f}' for c in cfgs if d[(k, L, C, c)]))
