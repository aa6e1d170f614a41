"""Top source lines by instructions executed (and stall samples) from an ncu source CSV.
usage: ncu_top.py page.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None; cur = None; out = []
def num(v):
    try: return float(v.replace(',', ''))
    except ValueError: return 0.0
for r in rows:
    if r and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': hdr = r; continue
    if hdr is None or not r or not r[0].isdigit(): continue
    d = dict(zip(hdr[2:], r[2:]))
    out.append((num(d.get('Instructions Executed', '0')), num(d.get('Warp Stall Sampling (All Samples)', '0')), cur,
                int(r[0]), r[1][:100]))
tot = sum(o[0] for o in out) or 1; ts = sum(o[1] for o in out) or 1
print(f"total inst {tot:.4g}")
for o in sorted(out, reverse=True)[:n]:
    print(f"{100*o[0]/tot:5.2f}% s{100*o[1]/ts:5.2f}% {o[2][:12]}:{o[3]:5d} {o[4]}")
