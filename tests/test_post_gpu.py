"""GPU trajectory post-processing (include/ftk_cp.h ftk_post_*) against the
plain-Python reference oracle/post.py on the oracle's records: adjacency (as a set of linked face-id
pairs), slices at integer and fractional t0, duration / loop filtering, simplification in time and type
smoothing -- bit-exact
(same records, same fixed-order FP64)."""
import numpy as np
import pytest
import torch

import ftk_inputs as fi
from oracle import post

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ftk():
    import paper_2011_08697_b200 as m
    from paper_2011_08697_b200 import build as b
    b.build()
    m.lib()
    assert torch.cuda.is_available()
    return m


def _key(a):
    return a[np.lexsort((a["z"], a["y"], a["x"], a["face_id"]))]


def setup_case(ftk, oracle_lib, field, s, dims):
    rec, buf = ftk.track(field.cuda(), s, return_buffers=True)
    tj = ftk.Trajectories(rec, buf, tuple(field.shape), field.dtype, s)
    g = ftk.to_numpy(rec)
    ref, _, _ = oracle_lib.track(field.numpy(), s)
    # same record set (ordering differs): map the GPU adjacency to face ids
    assert np.array_equal(np.sort(g["face_id"]), ref["face_id"])
    nbr_ref = post.adjacency(ref, dims)
    fid = g["face_id"]
    nb = tj.nbr.cpu().numpy()
    got = {(int(fid[i]), int(fid[j])) for i in range(len(g)) for j in nb[i] if j >= 0}
    want = {(int(ref["face_id"][i]), int(ref["face_id"][j])) for i, js in nbr_ref.items() for j in js}
    assert got == want
    return tj, ref, nbr_ref


CASES = [
    ("C1", lambda: fi.CONFIGS["C1"].make().generate(), 26, (32, 32, 8)),
    ("woven-noise", lambda: fi.Woven(48, 40, 12, L=15.0, sigma=0.02).generate(), 26, (48, 40, 12)),
    ("moving-min", lambda: fi.MovingExtremum((16, 15), 9, c0=(5.0, 6.0), v=(0.5, 0.25)).generate(), 8, (16, 15, 9)),
]


@pytest.mark.parametrize("name,make,s,dims", CASES)
def test_slice(ftk, oracle_lib, name, make, s, dims):
    tj, ref, nbr = setup_case(ftk, oracle_lib, make(), s, dims)
    for t0 in (0.0, 2.5, 3.25, 4.0, 6.875):
        g = _key(ftk.to_numpy(tj.slice(t0)))
        r = _key(post.slice_at(ref, nbr, t0))
        assert g.tobytes() == r.tobytes(), (name, t0, len(g), len(r))


@pytest.mark.parametrize("name,make,s,dims", CASES[:2])
def test_filter(ftk, oracle_lib, name, make, s, dims):
    tj, ref, nbr = setup_case(ftk, oracle_lib, make(), s, dims)
    for dmin, loops in ((0.0, True), (2.0, False), (5.0, True), (100.0, False)):
        g = _key(ftk.to_numpy(tj.filter(dmin, loops)))
        r = _key(post.filter_trajectories(ref, nbr, dmin, loops))
        assert g.tobytes() == r.tobytes(), (dmin, loops, len(g), len(r))


@pytest.mark.parametrize("w", [1, 2, 3])
def test_smooth(ftk, oracle_lib, w):
    field = fi.Woven(48, 40, 12, L=15.0, sigma=0.08).generate()
    tj, ref, nbr = setup_case(ftk, oracle_lib, field, 26, (48, 40, 12))
    g = _key(ftk.to_numpy(tj.smooth_types(w)))
    r = _key(post.smooth_types(ref, nbr, w))
    assert np.array_equal(g["type"], r["type"])
    assert (r["type"] != _key(ref)["type"]).any()  # the case exercises the rule


@pytest.mark.parametrize("tau", [0.5, 1.0, 3.0])
def test_simplify(ftk, oracle_lib, tau):
    field = fi.Woven(48, 40, 12, L=15.0, sigma=0.08).generate()
    tj, ref, nbr = setup_case(ftk, oracle_lib, field, 26, (48, 40, 12))
    g = _key(ftk.to_numpy(tj.simplify_types(tau)))
    r = _key(post.simplify_types(ref, nbr, tau))
    assert np.array_equal(g["type"], r["type"])
    if tau == 3.0:
        assert (r["type"] != _key(ref)["type"]).any()  # the case exercises the rule


def test_3d_adjacency_and_slice(ftk, oracle_lib):
    field = fi.Woven(14, 12, 5, L=15.0, sigma=0.02, nz=11).generate()
    tj, ref, nbr = setup_case(ftk, oracle_lib, field, 26, (14, 12, 11, 5))
    for t0 in (1.0, 2.5):
        g = _key(ftk.to_numpy(tj.slice(t0)))
        r = _key(post.slice_at(ref, nbr, t0))
        assert g.tobytes() == r.tobytes()
