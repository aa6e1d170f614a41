"""compute-sanitizer cases (SURVEY.md 5 "Race detection / sanitizers"): tiny inputs that drive every
kernel of the library once -- run each case under racecheck / synccheck / memcheck / initcheck, e.g.

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize.py c1

Cases: c1 (2D woven C1 track: TMA scan with its mbarrier ring, exact stage, pass 2), ragged2d (ragged
woven, generic loader + x/y boundary tiles, heavy-noise survivors), woven3d (ragged 3D woven: the 3D
scan's TMA ring and per-pair z exchange, k_exact3d), slabs (3 virtual time slabs through the device
seam path: export, pack, resolve, relabel), stream (push_field_data windows), vector (2D/3D vector
fields), post (adjacency / slice / filter / simplification / smoothing), iso (isovolume edges + cell unions).
Prints one line per case; no oracle (the parity suite checks results)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import ftk_inputs as fi  # noqa: E402
import paper_2011_08697_b200 as ftk  # noqa: E402


def c1():
    f = fi.CONFIGS["C1"].make().generate().cuda()
    return len(ftk.track(f, 26))


def ragged2d():
    n = 0
    for shape, sigma in (((9, 70, 131), 0.02), ((7, 37, 42), 0.08)):
        nt, ny, nx = shape
        n += len(ftk.track(fi.Woven(nx, ny, nt, sigma=sigma).generate().cuda(), 26))
    return n


def woven3d():
    f = fi.Woven(37, 21, 6, L=15.0, sigma=0.02, nz=19).generate().cuda()
    return len(ftk.track(f, 26))


def slabs():
    f = fi.Woven(96, 80, 13, sigma=0.02).generate()
    nt, G, cap = f.shape[0], 3, 4096
    b = ftk.slab_bounds(nt, G)
    stride = ftk.seam_block_size(cap)
    blocks = torch.full((G * stride,), -7, dtype=torch.int64, device="cuda")
    recs = []
    for r in range(G):
        ghost = r < G - 1
        sub = f[b[r]: b[r + 1] + (1 if ghost else 0)].contiguous().cuda()
        rec, buf = ftk.track(sub, 26, t0=b[r], nt_global=nt, ghost=ghost, return_buffers=True)
        ftk.seam_pack(sub, 26, b[r], nt, ghost, buf, blocks[r * stride:(r + 1) * stride], cap)
        recs.append(rec)
    for rec in recs:
        ftk.seam_resolve(blocks, G, cap, rec)
    return sum(len(r) for r in recs)


def stream():
    f = fi.Woven(64, 48, 9, sigma=0.02).generate()
    tr = ftk.Tracker((48, 64), torch.float32, 26, capacity=1 << 14, window=3)
    for k in range(f.shape[0]):
        tr.push(f[k].cuda())
    return len(tr.finish())


def vector():
    a = len(ftk.track(fi.DoubleGyre(70, 37, 7).generate().cuda(), 26, vector=True))
    b = len(ftk.track(fi.ABCFlow(20, 18, 17, 5).generate().cuda(), 26, vector=True))
    return a + b


def post():
    f = fi.Woven(64, 48, 12, sigma=0.02).generate().cuda()
    rec, buf = ftk.track(f, 26, return_buffers=True)
    tj = ftk.Trajectories(rec, buf, f.shape, f.dtype, 26)
    n = len(tj.slice(5.5)) + len(tj.filter(3.0, drop_loops=True))
    tj.simplify_types(2.0)
    tj.smooth_types(2)
    return n


def iso():
    f = fi.Woven(40, 33, 6, L=15.0).generate().cuda()
    g = fi.Woven(17, 15, 5, L=15.0, nz=13).generate().cuda()
    return len(ftk.iso_track(f, 26, 0.25)) + len(ftk.iso_track(g, 26, 0.5))


CASES = dict(c1=c1, ragged2d=ragged2d, woven3d=woven3d, slabs=slabs, stream=stream, vector=vector, post=post,
             iso=iso)

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for name in names:
        n = CASES[name]()
        torch.cuda.synchronize()
        print(f"sanitize case {name}: ok ({n} records)", flush=True)
