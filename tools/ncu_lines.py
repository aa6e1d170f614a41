"""Summarise an ncu source page (--print-source cuda,sass --csv): per CUDA line, instructions
executed and warp-stall samples, top N by samples."""
import csv, sys, collections
path = sys.argv[1]
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
cur_file = None
hdr = None
lines = []
for r in rows:
    if r and r[0] == 'File Path':
        cur_file = r[1].split('/')[-1]
        continue
    if r and r[0] == 'Line No':
        hdr = r
        continue
    if hdr is None or not r or r[0] == '' or r[0] == 'Function Name':
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    def f(k):
        v = d.get(k, '0')
        try: return float(v.replace(',', ''))
        except: return 0.0
    lines.append((cur_file, ln, r[1][:80], f('Instructions Executed'), f('Warp Stall Sampling (All Samples)'),
                  f('stall_barrier'), f('stall_no_inst')))
ti = sum(l[3] for l in lines) or 1; ts = sum(l[4] for l in lines) or 1
print(f'total warp-inst {ti:.3e}  samples {ts:.0f}')
for l in sorted(lines, key=lambda l: -l[4])[:topn]:
    print(f'{l[0][:12]:12s}:{l[1]:4d} inst {100*l[3]/ti:5.1f}% samp {100*l[4]/ts:5.1f}% bar {l[5]:6.0f} noi {l[6]:5.0f} | {l[2]}')

if len(sys.argv) > 3:
    # region aggregation: "name:file:lo-hi,..."
    for spec in sys.argv[3].split(','):
        name, f, rng = spec.split(':')
        lo, hi = map(int, rng.split('-'))
        si = sum(l[3] for l in lines if l[0].startswith(f) and lo <= l[1] <= hi)
        ss = sum(l[4] for l in lines if l[0].startswith(f) and lo <= l[1] <= hi)
        print(f'{name:20s} inst {100*si/ti:5.1f}%  samples {100*ss/ts:5.1f}%  ({si:.3e} warp-inst)')
