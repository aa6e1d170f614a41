"""FTK_SORTED (include/ftk_cp.h; SURVEY.md 8(b) descriptor flag, 7 "Determinism"): with the flag the
records come back in face-id order -- a hand-written device radix sort (csrc/sort.cu) after pass 2 --
and they are byte for byte the unsorted call's records in that order (the record SET is
deterministic; only the append order of the exact kernel varies)."""
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


def check_sorted(ftk, fn, *args, **kw):
    a = ftk.to_numpy(fn(*args, **kw))
    b = ftk.to_numpy(fn(*args, sorted_output=True, **kw))
    assert len(a) == len(b)
    assert np.all(np.diff(b["face_id"]) > 0)
    assert a[np.argsort(a["face_id"])].tobytes() == b.tobytes()
    return len(b)


def test_sorted_c1_track_and_extract(ftk):
    f = fi.CONFIGS["C1"].make().generate().cuda()
    assert check_sorted(ftk, ftk.track, f, 26) == 1116
    assert check_sorted(ftk, ftk.extract, f, 26) == 1116


@pytest.mark.parametrize("shape,sigma", [((40, 300, 260), 0.02), ((9, 70, 131), 0.08)])
def test_sorted_woven_many_tiles(ftk, shape, sigma):
    nt, ny, nx = shape
    n = check_sorted(ftk, ftk.track, fi.Woven(nx, ny, nt, sigma=sigma).generate().cuda(), 26)
    assert n > 4096  # several sort tiles


def test_sorted_3d_and_vector(ftk):
    check_sorted(ftk, ftk.track, fi.Woven(37, 21, 7, L=15.0, sigma=0.02, nz=19).generate().cuda(), 26)
    check_sorted(ftk, ftk.track, fi.ABCFlow(24, 20, 18, 6).generate().cuda(), 26, vector=True)
    check_sorted(ftk, ftk.track, fi.DoubleGyre(150, 75, 23).generate().cuda(), 26, vector=True)


def test_sorted_slab_with_ghost(ftk):
    f = fi.Woven(96, 80, 30, sigma=0.02).generate()
    sub = f[11:20].contiguous().cuda()
    check_sorted(ftk, ftk.track, sub, 26, t0=11, nt_global=30, ghost=True)


def test_sorted_c2_full_size(ftk):
    cfg = fi.CONFIGS["C2"]
    f = cfg.make().generate(device="cuda")
    assert check_sorted(ftk, ftk.track, f, cfg.scale_log2) > 2_500_000
