"""Full-size parity at the BASELINE.json configurations the oracle cannot finish whole (C4 2D
4096^2 x 512, C5 3D 256^3 x 64) and the 3D vector config V5, in the launch configuration bench.py
times: the GPU tracks the whole field; the oracle extracts a cropped block (a time window, and a
spatial box) of the same bytes, and the faces anchored far enough inside the box that neither the
crop's one-sided boundary differences nor its Hessian/Jacobian stencils reach them must agree with the
GPU's records of the same region: identical face set, types and flags, locations within 1e-6 (the
box offset is added after the oracle's fixed-order sums, so the last bits may differ)."""
import numpy as np
import pytest
import torch

import ftk_inputs as fi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ftk():
    import paper_2011_08697_b200 as m
    from paper_2011_08697_b200 import build as b
    b.build()
    m.lib()
    assert torch.cuda.is_available()
    return m


def decode(fid, ext, T):
    """face ids -> (anchor coords per axis x, y, [z,] t, type)"""
    I, ty = np.divmod(fid, T)
    out = []
    for n in ext[:-1]:
        I, c = np.divmod(I, n)
        out.append(c)
    out.append(I)
    return out, ty


def crop_parity(ftk, oracle_lib, field_dev, s, box, ta, tb, vector=False, margin=2):
    """box: per spatial axis (lo, size) in x, y[, z] order; lo = None centres the box on the median
    GPU record of the time window (deterministic: the record set is)"""
    nsp = len(box)
    shape = tuple(field_dev.shape)
    ext = tuple(reversed(shape[1:1 + nsp])) + (shape[0],)  # (nx, ny[, nz], nt)
    T = 12 if nsp == 2 else 60
    rec = ftk.to_numpy(ftk.track(field_dev, s, vector=vector))
    # the GPU's records anchored inside the inner box and the time window
    (gc, gty) = decode(rec["face_id"], ext, T)
    if ta is None:  # a two-step window at the median record's time
        ta = int(np.sort(gc[-1])[len(rec) // 2])
        ta, tb = min(ta, shape[0] - 3), min(ta, shape[0] - 3) + 2
    if any(lo is None for lo, _ in box):
        w = np.flatnonzero((gc[-1] >= ta) & (gc[-1] < tb))
        assert len(w) > 0
        c = w[len(w) // 2]
        box = [(int(min(max(gc[a][c] - size // 2, 0), ext[a] - size)) if lo is None else lo, size)
               for a, (lo, size) in enumerate(box)]
    keep = (gc[-1] >= ta) & (gc[-1] < tb)
    for a, (lo, size) in enumerate(box):
        keep &= (gc[a] >= lo + margin) & (gc[a] < lo + size - margin - 2)
    g = rec[keep]
    # the oracle on the crop (planes ta .. tb, the box) as a window of the global time axis
    sl = [slice(ta, tb + 1)] + [slice(lo, lo + size) for lo, size in reversed(box)]
    sub = field_dev[tuple(sl)].cpu().numpy()
    ref, _ = oracle_lib.extract(sub, s, t0=ta, nt_global=shape[0], ta=ta, tb=tb, vector=vector)
    sub_ext = tuple(size for _, size in box) + (shape[0],)
    (rc, rty) = decode(ref["face_id"], sub_ext, T)
    rk = np.ones(len(ref), bool)
    for a, (lo, size) in enumerate(box):
        rk &= (rc[a] >= margin) & (rc[a] < size - margin - 2)
    r = ref[rk]
    # map the oracle's face ids and locations into the global grid
    rc = [c[rk] for c in rc]
    gid = rc[-1]
    for a in reversed(range(nsp)):
        gid = gid * ext[a] + rc[a] + box[a][0]
    rid = gid * T + rty[rk]
    order = np.argsort(rid)
    g = g[np.argsort(g["face_id"])]
    assert np.array_equal(g["face_id"], rid[order]), (len(g), len(rid))
    r = r[order]
    assert np.array_equal(g["type"], r["type"])
    assert np.array_equal(g["flags"], r["flags"])
    names = ("x", "y", "z")[:nsp]
    for a, k in enumerate(names):
        assert np.max(np.abs(g[k] - (r[k] + box[a][0]))) <= 1e-6, k
    assert np.max(np.abs(g["t"] - r["t"])) <= 1e-6
    return len(g)


def test_c4_full_size_crop(ftk, oracle_lib):
    cfg = fi.CONFIGS["C4"]
    f = cfg.make().generate(device="cuda")
    n = crop_parity(ftk, oracle_lib, f, cfg.scale_log2, [(1500, 384), (2900, 320)], 300, 303)
    assert n > 100


def test_c5_full_size_crop(ftk, oracle_lib):
    cfg = fi.CONFIGS["C5"]
    f = cfg.make().generate(device="cuda")
    n = crop_parity(ftk, oracle_lib, f, cfg.scale_log2, [(None, 40), (None, 40), (None, 40)], 30, 32)
    assert n > 0


def test_v5_full_size_crop(ftk, oracle_lib):
    cfg = fi.CONFIGS["V5"]
    f = cfg.make().generate(device="cuda")
    n = crop_parity(ftk, oracle_lib, f, cfg.scale_log2, [(None, 48), (None, 48), (None, 48)], None, None, vector=True)
    assert n > 0
