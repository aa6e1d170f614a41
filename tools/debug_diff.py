"""Debug helper: diff GPU extract vs oracle extract on a woven field, print the differing faces."""
import sys, collections
import numpy as np, torch
sys.path.insert(0, '.')
import ftk_inputs as fi, oracle, paper_2011_08697_b200 as ftk

nt, ny, nx = [int(v) for v in sys.argv[1:4]]
sigma = float(sys.argv[4]) if len(sys.argv) > 4 else 0.02
w = fi.Woven(nx, ny, nt, sigma=sigma)
f = w.generate()
g = ftk.to_numpy(ftk.extract(f.cuda(), 26))
r, _ = oracle.extract(f.numpy(), 26)
gs, rs = set(g['face_id'].tolist()), set(r['face_id'].tolist())
print('gpu', len(gs), 'oracle', len(rs), 'missing', len(rs - gs), 'extra', len(gs - rs))
def dec(fid):
    I, ty = divmod(fid, 12); x = I % nx; y = (I // nx) % ny; t = I // (nx * ny); return x, y, t, ty
for name, s in (('missing', rs - gs), ('extra', gs - rs)):
    c = collections.Counter()
    for fid in sorted(s)[:2000]:
        x, y, t, ty = dec(fid); c[(x % 128, y % 32, ty)] += 1
    print(name, c.most_common(12))
    for fid in sorted(s)[:10]: print('  ', dec(fid))
