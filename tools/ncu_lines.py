"""Summarise an ncu source page exported with `--page source --csv --print-source cuda,sass`: per CUDA
source line, instructions executed and warp-stall samples (top N by samples); optional region sums
"name:file:lo-hi,...".  Optional --sass: the top SASS instructions by samples."""
import csv, sys

path = sys.argv[1]
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
cur_file, hdr = None, None
lines, sass = [], []
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        cur_file = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = r
        continue
    if hdr is None or r[0] in ('Function Name',):
        continue
    d = dict(zip(hdr[4:], r[4:]))

    def f(k):
        try:
            return float(d.get(k, '0').replace(',', ''))
        except ValueError:
            return 0.0
    ent = (cur_file, r[0], (r[1] if r[0] else r[3])[:90], f('Instructions Executed'),
           f('Warp Stall Sampling (All Samples)'))
    (lines if r[0] else sass).append(ent)
ti = sum(l[3] for l in lines) or 1
ts = sum(l[4] for l in lines) or 1
print(f'total warp-inst {ti:.3e}  samples {ts:.0f}')
for l in sorted(lines, key=lambda l: -l[4])[:topn]:
    print(f'{l[0][:12]:12s}:{l[1]:>4s} inst {100*l[3]/ti:5.1f}% samp {100*l[4]/ts:5.1f}% | {l[2]}')
if '--sass' in sys.argv:
    for l in sorted(sass, key=lambda l: -l[4])[:topn]:
        print(f'samp {100*l[4]/ts:5.1f}% inst {l[3]:9.0f} | {l[2]}')
for a in sys.argv[3:]:
    if a.startswith('--'):
        continue
    for spec in a.split(','):
        name, fn, rng = spec.split(':')
        lo, hi = map(int, rng.split('-'))
        sel = [l for l in lines if l[0].startswith(fn) and lo <= int(l[1]) <= hi]
        print(f'{name:20s} inst {100*sum(l[3] for l in sel)/ti:5.1f}%  samples {100*sum(l[4] for l in sel)/ts:5.1f}%')
