"""Per-region stall breakdown from an ncu source page (--print-source cuda,sass --csv):
python tools/ncu_regions.py page.csv name:file:lo-hi ..."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
cur, hdr = None, None
acc = collections.defaultdict(collections.Counter)
specs = []
for a in sys.argv[2:]:
    n, f, r = a.split(':'); lo, hi = map(int, r.split('-')); specs.append((n, f, lo, hi))
R = ['stall_long_sb', 'stall_wait', 'stall_short_sb', 'stall_no_inst', 'stall_mio', 'stall_lg', 'stall_math',
     'stall_branch_resolving', 'stall_selected', 'stall_not_selected', 'stall_dispatch']
tot = collections.Counter()
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None or not r[0] or not r[0].isdigit(): continue
    d = dict(zip(hdr[4:], r[4:]))
    ln = int(r[0])
    name = 'other'
    for n, f, lo, hi in specs:
        if cur.startswith(f) and lo <= ln <= hi: name = n; break
    for k in R + ['Warp Stall Sampling (All Samples)', 'Instructions Executed']:
        try: v = float(d.get(k, '0').replace(',', ''))
        except ValueError: v = 0
        acc[name][k] += v; tot[k] += v
S = tot['Warp Stall Sampling (All Samples)']
print(f"{'region':12s} {'samp%':>6s} {'inst%':>6s} " + ' '.join(f'{k[6:12]:>6s}' for k in R))
for n, c in sorted(acc.items(), key=lambda x: -x[1]['Warp Stall Sampling (All Samples)']):
    print(f"{n:12s} {100*c['Warp Stall Sampling (All Samples)']/S:6.1f} {100*c['Instructions Executed']/tot['Instructions Executed']:6.1f} " +
          ' '.join(f'{100*c[k]/S:6.1f}' for k in R))
