"""Stall-reason breakdown per source-line range of an ncu source page CSV (--print-source cuda,sass).
usage: ncu_stalls.py page.csv "name:file:lo-hi,..." """
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; cur = None
acc = collections.defaultdict(lambda: collections.Counter())
specs = []
for spec in sys.argv[2].split(','):
    n, f, rng = spec.split(':'); lo, hi = map(int, rng.split('-')); specs.append((n, f, lo, hi))
for r in rows:
    if r and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': hdr = r; continue
    if hdr is None or not r or not r[0].isdigit(): continue
    ln = int(r[0]); d = dict(zip(hdr[2:], r[2:]))
    for n, f, lo, hi in specs:
        if cur.startswith(f) and lo <= ln <= hi:
            for k, v in d.items():
                if k.startswith('stall_') and '(Not' not in k or k == 'Instructions Executed':
                    try: acc[n][k] += float(v.replace(',', '') or 0)
                    except ValueError: pass
for n, c in acc.items():
    tot = sum(v for k, v in c.items() if k.startswith('stall_'))
    top = sorted(((v, k) for k, v in c.items() if k.startswith('stall_')), reverse=True)[:7]
    print(f"{n:10s} inst {c['Instructions Executed']:.3e} samples {tot:.0f}: " +
          ", ".join(f"{k[6:]} {100*v/max(tot,1):.0f}%" for v, k in top))
