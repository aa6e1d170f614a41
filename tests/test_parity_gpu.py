"""GPU parity: the CUDA path (through the C-ABI) against the independent CPU oracle, element by
element on the same seeded input bytes.

Bar (BASELINE.json north_star): bit-exact punctured-face set, trajectory labels, CP types and
flags; locations within 1e-6 grid units (the kernel and the oracle evaluate the same fixed-order
FP64 expressions without FMA, so they are in fact expected to agree to the last bit -- the test
reports the max difference)."""
import os

import numpy as np
import pytest
import torch

import ftk_inputs as fi

pytestmark = pytest.mark.gpu

LOC_TOL = 1e-6


@pytest.fixture(scope="module")
def ftk():
    import paper_2011_08697_b200 as m
    from paper_2011_08697_b200 import build as b
    b.build()
    m.lib()
    assert torch.cuda.is_available()
    return m


def _sorted(a):
    return a[np.argsort(a["face_id"], kind="stable")]


def compare(gpu, ref, labels=True):
    g, r = _sorted(gpu), _sorted(ref)
    assert len(g) == len(r), (len(g), len(r))
    assert np.array_equal(g["face_id"], r["face_id"])
    assert np.array_equal(g["type"], r["type"])
    assert np.array_equal(g["flags"].astype(np.int64), r["flags"].astype(np.int64))
    if labels:
        assert np.array_equal(g["label"], r["label"])
    dmax = 0.0
    for k in ("x", "y", "z", "t"):
        if len(g):
            dmax = max(dmax, float(np.max(np.abs(g[k] - r[k]))))
    assert dmax <= LOC_TOL, dmax
    return dmax


def run_pair(ftk, oracle_lib, field_cpu: torch.Tensor, s: int, labels=True):
    dev = field_cpu.cuda()
    if labels:
        rec = ftk.to_numpy(ftk.track(dev, s))
        ref, nf, info = oracle_lib.track(field_cpu.numpy(), s)
    else:
        rec = ftk.to_numpy(ftk.extract(dev, s))
        ref, nf = oracle_lib.extract(field_cpu.numpy(), s)
    return compare(rec, ref, labels), len(ref)


def test_c1_track_bit_exact(ftk, oracle_lib):
    w = fi.CONFIGS["C1"].make()
    d, n = run_pair(ftk, oracle_lib, w.generate(), 26)
    assert n == 1116 and d == 0.0


@pytest.mark.parametrize("shape,L,sigma", [
    ((40, 70, 100), None, 0.02),      # ragged nx (not a multiple of 4: generic loader), 2 time chunks
    ((70, 140, 260), None, 0.02),     # several tiles in x and y, ragged edges, TMA path
    ((33, 64, 128), 15.0, 0.0),       # exact tile multiples, chunk boundary at t = 32
    ((35, 97, 131), None, 0.08),      # heavy noise: half of the cubes survive the prefilter
])
def test_woven_track_parity(ftk, oracle_lib, shape, L, sigma):
    nt, ny, nx = shape
    w = fi.Woven(nx, ny, nt, L=L, sigma=sigma)
    run_pair(ftk, oracle_lib, w.generate(), 26)


@pytest.mark.parametrize("shape,values", [
    ((5, 6, 7), (-1.0, 0.0, 1.0)),
    ((40, 33, 3), (-1.0, 0.0, 1.0)),
    ((6, 37, 150), (-2.0, -1.0, 0.0, 1.0, 2.0)),
])
def test_degenerate_fields_parity(ftk, oracle_lib, shape, values):
    for seed in range(3):
        f = fi.random_degenerate(shape, values=values, seed=seed)
        run_pair(ftk, oracle_lib, f, 0)


@pytest.mark.parametrize("signs", [(1, 1), (1, -1), (-1, -1)])
def test_moving_extremum_2d_parity(ftk, oracle_lib, signs):
    me = fi.MovingExtremum((150, 140), 40, c0=(20.0, 100.0), v=(2.5, -1.25), signs=signs)
    d, n = run_pair(ftk, oracle_lib, me.generate(), me.scale_log2)
    assert n >= 40


def test_fp64_input(ftk, oracle_lib):
    w = fi.Woven(66, 50, 12, sigma=0.02)
    run_pair(ftk, oracle_lib, w.generate(dtype=torch.float64), 26)


def test_generic_loader_matches_tma(ftk, oracle_lib):
    w = fi.Woven(132, 72, 20, sigma=0.02)
    f = w.generate().cuda()
    a = ftk.to_numpy(ftk.track(f, 26))
    ftk.set_debug(ftk.DEBUG_FORCE_GENERIC)
    try:
        b = ftk.to_numpy(ftk.track(f, 26))
    finally:
        ftk.set_debug(0)
    assert _sorted(a).tobytes() == _sorted(b).tobytes()


def test_closed_form_link_verification(ftk, oracle_lib):
    """K1 pairs faces per cell; the independent closed-form side_of verifier (FTK_DEBUG_VERIFY_LINK)
    re-derives every punctured face's parent cells and finds exactly one partner in each."""
    ftk.set_debug(ftk.DEBUG_VERIFY_LINK)
    try:
        for f in (fi.Woven(150, 140, 40, sigma=0.08).generate(), fi.random_degenerate((6, 37, 150), seed=4)):
            s = 26 if f.abs().max() < 2 and f.dtype == torch.float32 and (f != f.round()).any() else 0
            run_pair(ftk, oracle_lib, f, s)
    finally:
        ftk.set_debug(0)


def test_extract_window_with_ghost(ftk, oracle_lib):
    w = fi.Woven(96, 80, 30, sigma=0.02)
    f = w.generate()
    ta, tb = 11, 19
    sub = f[ta: tb + 1]  # owned planes [ta, tb) + ghost plane tb
    g = ftk.to_numpy(ftk.extract(sub.cuda(), 26, t0=ta, nt_global=30, ghost=True))
    r, _ = oracle_lib.extract(sub.numpy(), 26, t0=ta, nt_global=30, ta=ta, tb=tb)
    compare(g, r, labels=False)


def test_small_and_single_plane(ftk, oracle_lib):
    w = fi.Woven(3, 3, 1, L=15.0)
    run_pair(ftk, oracle_lib, w.generate(), 26, labels=False)
    w = fi.Woven(5, 4, 2, L=15.0)
    run_pair(ftk, oracle_lib, w.generate(), 26)


def test_determinism_and_capacity_retry(ftk):
    w = fi.Woven(200, 150, 20, sigma=0.08)
    f = w.generate().cuda()
    a = ftk.to_numpy(ftk.track(f, 26, capacity=1000))  # forces ERR_CAPACITY + retry
    b = ftk.to_numpy(ftk.track(f, 26))
    assert len(a) > 1000
    assert _sorted(a).tobytes() == _sorted(b).tobytes()


def test_range_error(ftk):
    f = torch.zeros(3, 8, 8)
    f[1, 3, 3] = 2.0**40
    with pytest.raises(ftk.FtkError) as e:
        ftk.track(f.cuda(), 20)
    assert e.value.status == ftk.ERR_RANGE
    f[1, 3, 3] = float("nan")
    with pytest.raises(ftk.FtkError) as e:
        ftk.track(f.cuda(), 0)
    assert e.value.status == ftk.ERR_RANGE


def test_c2_full_size_sampled_parity(ftk, oracle_lib):
    """C2 (1024^2 x 256) in the bench's launch configuration: the oracle checks a window of anchor
    timesteps record by record; labels are checked by properties that hold at any size."""
    cfg = fi.CONFIGS["C2"]
    w = cfg.make()
    f = w.generate(device="cuda")
    rec = ftk.to_numpy(ftk.track(f, cfg.scale_log2))
    nx, ny, nt = 1024, 1024, 256
    T = 12
    t_of = rec["face_id"] // T // (nx * ny)
    for ta in (0, 137, 254):
        tb = ta + 2
        sub = f[ta: tb + 1].cpu()
        ref, _ = oracle_lib.extract(sub.numpy(), cfg.scale_log2, t0=ta, nt_global=nt, ta=ta, tb=tb)
        g = rec[(t_of >= ta) & (t_of < tb)]
        compare(g, ref, labels=False)
    # properties of the labels: label = min face_id of its component; open trajectories have two
    # boundary ends, loops none; no loops at sigma = 0
    order = np.argsort(rec["label"], kind="stable")
    lab = rec["label"][order]
    fid = rec["face_id"][order]
    bnd = (rec["flags"][order] & ftk.CP_BOUNDARY) != 0
    starts = np.flatnonzero(np.r_[True, lab[1:] != lab[:-1]])
    mins = np.minimum.reduceat(fid, starts)
    assert np.array_equal(mins, lab[starts])
    nb = np.add.reduceat(bnd.astype(np.int64), starts)
    assert set(np.unique(nb).tolist()) <= {2}
    assert 2.5e6 < len(rec) < 3.2e6


# ----------------------------------------------------------------------------------- 3D + t
@pytest.mark.parametrize("signs", [(1, 1, 1), (1, -1, 1), (-1, -1, 1), (-1, -1, -1)])
def test_moving_extremum_3d_parity(ftk, oracle_lib, signs):
    me = fi.MovingExtremum((20, 19, 18), 6, c0=(6.0, 7.0, 9.0), v=(1.5, 1.25, -0.75), signs=signs)
    d, n = run_pair(ftk, oracle_lib, me.generate(), me.scale_log2)
    assert n >= 6


@pytest.mark.parametrize("shape,L,sigma", [
    ((5, 18, 20, 24), 15.0, 0.0),     # ragged tiles in x, y, z
    ((4, 13, 11, 37), None, 0.08),    # heavy noise, ragged
])
def test_woven3d_parity(ftk, oracle_lib, shape, L, sigma):
    nt, nz, ny, nx = shape
    w = fi.Woven(nx, ny, nt, L=L, sigma=sigma, nz=nz)
    run_pair(ftk, oracle_lib, w.generate(), 26)


@pytest.mark.parametrize("s", [14, 25, 27, 36])
def test_woven3d_scale_paths(ftk, oracle_lib, s):
    """K1b (3D) decides determinant signs with an FP64 filter when every gradient component of the
    hypercube is below 2^26 and with exact int128 otherwise: s = 14 / 25 keep every hypercube on the
    filter, 27 mixes both, 36 (|q| < 2^38, the 3D range limit) forces the exact path everywhere."""
    w = fi.Woven(21, 19, 5, L=15.0, sigma=0.02, nz=17)
    run_pair(ftk, oracle_lib, w.generate(), s)


def test_degenerate_3d_parity(ftk, oracle_lib):
    for seed in range(2):
        f = fi.random_degenerate((3, 5, 6, 7), seed=seed)
        run_pair(ftk, oracle_lib, f, 0)


def test_c3_closed_form_full_size(ftk, oracle_lib):
    """C3 (128^3 x 32, moving minimum): exactly one punctured ordinal face per
    timestep, located at c(t), type MIN, one trajectory; plus a sampled oracle window."""
    cfg = fi.CONFIGS["C3"]
    me = cfg.make()
    f = me.generate(device="cuda")
    rec = ftk.to_numpy(ftk.track(f, cfg.scale_log2))
    ordn = rec[(rec["flags"] & ftk.CP_ORDINAL) != 0]
    assert len(ordn) == 32
    for r in ordn:
        c = me.center(r["t"])
        assert abs(r["x"] - c[0]) < 1e-9 and abs(r["y"] - c[1]) < 1e-9 and abs(r["z"] - c[2]) < 1e-9
    assert set(rec["type"].tolist()) == {ftk.MIN}
    assert len(set(rec["label"].tolist())) == 1
    nt = 32
    t_of = rec["face_id"] // 60 // (128 ** 3)
    ta, tb = 15, 17
    sub = f[ta: tb + 1].cpu()
    ref, _ = oracle_lib.extract(sub.numpy(), cfg.scale_log2, t0=ta, nt_global=nt, ta=ta, tb=tb)
    compare(rec[(t_of >= ta) & (t_of < tb)], ref, labels=False)


@pytest.mark.parametrize("where", [(0, 0, 0), (1, 0, 7), (2, 5, 0), (1, 39, 66), (0, 17, 66)])
def test_range_error_anywhere_2d(ftk, where):
    """the range check covers every vertex, grid boundary rows and columns included"""
    f = fi.Woven(67, 40, 3, sigma=0.0).generate()
    f[where] = float("nan")
    with pytest.raises(ftk.FtkError) as e:
        ftk.track(f.cuda(), 26)
    assert e.value.status == ftk.ERR_RANGE


@pytest.mark.parametrize("where", [(0, 0, 0, 0), (1, 12, 0, 7), (2, 0, 9, 0), (1, 12, 9, 66), (0, 5, 0, 66)])
def test_range_error_anywhere_3d(ftk, where):
    f = fi.Woven(67, 10, 3, L=15.0, sigma=0.0, nz=13).generate()
    f[where] = float("nan")
    with pytest.raises(ftk.FtkError) as e:
        ftk.track(f.cuda(), 26)
    assert e.value.status == ftk.ERR_RANGE


@pytest.mark.parametrize("nx", [124, 125, 127, 128, 129, 248, 252, 253, 256])
def test_x_tile_boundaries_2d(ftk, oracle_lib, nx):
    """widths around the 124-column tiles and the full-width last tile"""
    w = fi.Woven(nx, 70, 6, sigma=0.02)
    run_pair(ftk, oracle_lib, w.generate(), 26)


@pytest.mark.parametrize("nx", [124, 128, 129, 133])
def test_x_tile_boundaries_3d(ftk, oracle_lib, nx):
    w = fi.Woven(nx, 9, 3, L=15.0, sigma=0.02, nz=10)
    run_pair(ftk, oracle_lib, w.generate(), 26)


@pytest.mark.parametrize("shape,sigma", [
    ((5, 19, 14, 300), 0.0),    # x tile 128..255 is interior (MODE 0): the dz region test rejects most
    ((4, 19, 14, 300), 0.02),   # warps; the slice through z = 0 (dz = 0 exactly) is never rejected
    ((4, 21, 13, 261), 0.05),   # x-boundary tiles (MODE 1) with out-of-grid positions and column x0 + 128
])
def test_woven3d_region_test_parity(ftk, oracle_lib, shape, sigma):
    """k_scan3d rejects whole warp regions when dz keeps one strict sign on both planes of a pair; the
    survivor set must stay that of the per-vertex codes (checked through the oracle's result)."""
    nt, nz, ny, nx = shape
    w = fi.Woven(nx, ny, nt, sigma=sigma, nz=nz)
    _, n = run_pair(ftk, oracle_lib, w.generate(), 26)
    assert n > 0


def test_moving_extremum_3d_region_test(ftk, oracle_lib):
    """a paraboloid: dz changes sign only near the centre's slice, dx / dy keep one sign far from it"""
    me = fi.MovingExtremum((300, 12, 20), 5, c0=(200.0, 6.0, 10.0), v=(0.5, 0.25, 0.75))
    d, n = run_pair(ftk, oracle_lib, me.generate(), me.scale_log2)
    assert n >= 4


@pytest.mark.parametrize("where", [(0, 9, 5, 200), (1, 10, 7, 299), (2, 0, 0, 150), (1, 18, 13, 128), (0, 4, 6, 255)])
def test_range_error_region_path_3d(ftk, where):
    """the range statistics of the region-test path (interior tiles) cover every vertex"""
    f = fi.Woven(300, 14, 3, sigma=0.0, nz=19).generate()
    f[where] = float("inf") if where[0] == 2 else float("nan")
    with pytest.raises(ftk.FtkError) as e:
        ftk.track(f.cuda(), 26)
    assert e.value.status == ftk.ERR_RANGE
