"""Pins of the oracle's whole tracking result against closed forms and invariants:

* moving minimum / saddle: the PL gradient is exactly affine,
  so each timestep has exactly one punctured ordinal face, located at c(t), with the analytic
  type, and all punctured faces form ONE trajectory -- including timesteps where c(t) is a grid
  vertex (the SoS path);
* woven census at t = 0: the punctured ordinal faces equal the analytic CPs
  of cos x sin y in number, type and (within 0.01 cell) location;
* invariants: every cell has 0 or 2 punctured faces; trajectories end on the
  domain boundary or are loops; noise-free woven trajectories keep one type;
  power-of-two rescaling of the field with the matching scale changes nothing.
"""
import collections
import math

import numpy as np
import pytest
import torch

import ftk_inputs as fi


def _components(rec):
    comp = collections.defaultdict(list)
    for r in rec:
        comp[int(r["label"])].append(r)
    return comp


def _check_common(oracle, rec, info):
    assert info["bad_cells"] == 0
    # labels are the minimum face id of their component
    for lab, rs in _components(rec).items():
        assert lab == min(int(r["face_id"]) for r in rs)
        nb = sum(1 for r in rs if r["flags"] & oracle.FL_BOUNDARY)
        assert nb in (0, 2)  # open trajectory: two boundary ends; loop: none


@pytest.mark.parametrize("signs,expect", [((1, 1), "MIN"), ((1, -1), "SADDLE"), ((-1, -1), "MAX")])
def test_moving_extremum_2d(oracle_lib, signs, expect):
    me = fi.MovingExtremum((16, 16), 9, c0=(5.0, 6.0), v=(0.5, 0.25), signs=signs)
    f = me.generate().numpy()
    rec, nf, info = oracle_lib.track(f, me.scale_log2)
    _check_common(oracle_lib, rec, info)
    ordn = rec[(rec["flags"] & oracle_lib.FL_ORDINAL) != 0]
    for t in range(9):
        at = ordn[np.abs(ordn["t"] - t) < 1e-9]
        assert len(at) == 1, t  # exactly once, also at vertex hits t = 0, 4, 8
        cx, cy = me.center(t)
        assert abs(at["x"][0] - cx) < 1e-12 and abs(at["y"][0] - cy) < 1e-12
    assert len(ordn) == 9
    assert set(rec["type"].tolist()) == {getattr(oracle_lib, expect)}
    for r in rec:  # every punctured face lies on the line x = c(t)
        cx, cy = me.center(r["t"])
        assert abs(r["x"] - cx) < 1e-9 and abs(r["y"] - cy) < 1e-9
    assert info["components"] == 1


@pytest.mark.parametrize("signs,expect", [((1, 1, 1), "MIN"), ((1, -1, 1), "SADDLE1"),
                                          ((1, -1, -1), "SADDLE2"), ((-1, -1, -1), "MAX")])
def test_moving_extremum_3d(oracle_lib, signs, expect):
    me = fi.MovingExtremum((8, 8, 8), 5, c0=(3.0, 3.0, 4.0), v=(0.5, 0.25, 0.125), signs=signs)
    f = me.generate().numpy()
    rec, nf, info = oracle_lib.track(f, me.scale_log2)
    _check_common(oracle_lib, rec, info)
    ordn = rec[(rec["flags"] & oracle_lib.FL_ORDINAL) != 0]
    assert len(ordn) == 5
    for r in ordn:
        c = me.center(r["t"])
        assert abs(r["x"] - c[0]) < 1e-12 and abs(r["y"] - c[1]) < 1e-12 and abs(r["z"] - c[2]) < 1e-12
    assert set(rec["type"].tolist()) == {getattr(oracle_lib, expect)}
    assert info["components"] == 1


def test_moving_minimum_paper_suite(oracle_lib):
    """x0 = (10,10,10) on a 21^3 grid, rational directions that hit grid points;
    with SoS the trajectory is one line, one detection per timestep (5 steps here)."""
    rng = np.random.default_rng(11)
    for _ in range(3):
        d = tuple(float(rng.integers(-4, 5)) / 4.0 for _ in range(3))
        me = fi.MovingExtremum((21, 21, 21), 5, c0=(10.0, 10.0, 10.0), v=d)
        rec, nf, info = oracle_lib.track(me.generate().numpy(), me.scale_log2)
        assert info["bad_cells"] == 0 and info["components"] == 1
        ordn = rec[(rec["flags"] & oracle_lib.FL_ORDINAL) != 0]
        assert sorted(np.round(ordn["t"]).tolist()) == [0, 1, 2, 3, 4]


def test_woven_c1_census_t0(oracle_lib):
    cfg = fi.CONFIGS["C1"]
    w = cfg.make()
    f = w.generate().numpy()
    rec, nf, info = oracle_lib.track(f, cfg.scale_log2)
    assert nf == 83514 and len(rec) == 1116  # SURVEY.md 8(d) C1 counts
    _check_common(oracle_lib, rec, info)
    t0 = rec[((rec["flags"] & oracle_lib.FL_ORDINAL) != 0) & (rec["t"] == 0)]
    cps = w.analytic_cps_t0()
    assert len(t0) == len(cps) == 40
    kinds = {"max": oracle_lib.MAX, "min": oracle_lib.MIN, "saddle": oracle_lib.SADDLE}
    assert collections.Counter(t0["type"].tolist()) == collections.Counter(kinds[k] for *_, k in cps)
    for gx, gy, k in cps:
        dist = np.hypot(t0["x"] - gx, t0["y"] - gy)
        i = int(np.argmin(dist))
        assert dist[i] < 0.01 and t0["type"][i] == kinds[k]
    # noise-free woven: no loops, each trajectory keeps one type
    comps = _components(rec)
    assert info["pairs"] == len(rec) - len(comps)  # forest of paths: no loop closes
    for rs in comps.values():
        assert len({int(r["type"]) for r in rs}) == 1


def test_woven_paper_density_census_t0(oracle_lib):
    """128^2 grid over [-7.5, 7.5]^2 (the paper's woven): 40 CPs at t=0."""
    w = fi.Woven(128, 128, 1)
    rec, nf = oracle_lib.extract(w.generate().numpy(), 26)
    cps = w.analytic_cps_t0()
    assert len(rec) == len(cps) == 40
    for gx, gy, k in cps:
        assert np.min(np.hypot(rec["x"] - gx, rec["y"] - gy)) < 0.01


def test_woven_noise_loops_and_invariants(oracle_lib):
    """sigma = 0.02 produces small loops; the 0/2 invariant still holds."""
    w = fi.Woven(64, 64, 10, sigma=0.02)  # paper density h = 15/127
    rec, nf, info = oracle_lib.track(w.generate().numpy(), 26)
    _check_common(oracle_lib, rec, info)
    comps = _components(rec)
    loops = sum(1 for rs in comps.values() if not any(r["flags"] & oracle_lib.FL_BOUNDARY for r in rs))
    assert loops > 0


@pytest.mark.parametrize("shape", [(4, 5, 6), (5, 4, 4), (3, 4, 4, 3), (3, 3, 4, 4)])
@pytest.mark.parametrize("values", [(-1.0, 0.0, 1.0), (-3.0, -2.0, -1.0, 0.0, 1.0, 2.0, 3.0)])
def test_zero_or_two_on_degenerate_fields(oracle_lib, shape, values):
    for seed in range(4):
        f = fi.random_degenerate(shape, values=values, seed=seed).numpy()
        rec, nf, info = oracle_lib.track(f, 0)
        _check_common(oracle_lib, rec, info)


def test_scale_invariance(oracle_lib):
    w = fi.Woven(24, 20, 6, L=15.0, sigma=0.02)
    f = w.generate(dtype=torch.float64).numpy()
    a, _, _ = oracle_lib.track(f, 26)
    b, _, _ = oracle_lib.track(f * 2.0, 25)
    c, _, _ = oracle_lib.track(f * 0.25, 28)
    assert a.tobytes() == b.tobytes() == c.tobytes()


def test_extract_window_matches_track(oracle_lib):
    w = fi.Woven(20, 18, 9, L=15.0)
    f = w.generate().numpy()
    full, _, _ = oracle_lib.track(f, 26)
    part, _ = oracle_lib.extract(f[3:7], 26, t0=3, nt_global=9, ta=3, tb=6)
    sel = full[(full["face_id"] >= part["face_id"].min()) & (full["face_id"] <= part["face_id"].max())]
    ids_full = set(full["face_id"].tolist())
    assert set(part["face_id"].tolist()) <= ids_full
    keys = ["x", "y", "z", "t", "type", "flags"]
    fm = {int(r["face_id"]): r for r in full}
    for r in part:
        for k in keys:
            assert r[k] == fm[int(r["face_id"])][k]
    assert len(sel) == len(part)


def test_range_error(oracle_lib):
    f = np.zeros((2, 4, 4), np.float32)
    f[0, 1, 1] = 2.0**40
    with pytest.raises(oracle_lib.OracleError) as e:
        oracle_lib.track(f, 20)
    assert e.value.status == oracle_lib.RANGE


def test_woven3d_census_t0(oracle_lib):
    """3D woven (our field): cos X sin Y + cos z at t = 0 has CPs at the 2D woven
    CPs x planes z = m pi; 40^3 with L = 15 -> 30 MAX + 80 SADDLE2 + 70 SADDLE1 + 20 MIN."""
    w = fi.Woven(40, 40, 1, L=15.0, nz=40)
    rec, nf = oracle_lib.extract(w.generate().numpy(), 26)
    cnt = collections.Counter(rec["type"].tolist())
    assert cnt == {oracle_lib.MAX: 30, oracle_lib.SADDLE2: 80, oracle_lib.SADDLE1: 70, oracle_lib.MIN: 20}
    # analytic: z = (k/(nz-1) - 1/2) L with cos z = +-1 at z = m pi
    L = 15.0
    for r in rec:
        z = (r["z"] / 39 - 0.5) * L
        assert abs(z / math.pi - round(z / math.pi)) * math.pi < 0.01 * L / 39 * 3
