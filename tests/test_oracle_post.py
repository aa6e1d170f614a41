"""Pins of the post-processing reference (oracle/post.py):

* slicing: the moving minimum's trajectory is the straight line c(t) (its PL gradient is exactly
  affine), so the slice at any t0 -- integer or not -- is exactly one point, at c(t0);
* adjacency: every face has at most two partners; open trajectories have exactly two ends, loops none
  (P:447); the partition it induces equals the labels of the track;
* filtering: on the noisy woven field dropping loops leaves exactly the open
  trajectories, and a duration threshold keeps exactly the trajectories at least that long;
* smoothing: a single-record type spike inside a uniform trajectory is corrected, ends and
  genuine type changes are kept;
* simplification in time (R23), on hand-built trajectories whose folds, segment extents
  and outer types are worked out by hand: the Fig. 9(b) pattern (a sink, a short backward saddle segment
  between a death and a birth fold, a sink again) becomes one sink below tau and not at tau; a segment
  between different types, the end segments and tau <= 0 change nothing; a fold between two qualifying
  segments of different types keeps its own; a loop is cut at all four of its folds."""
import collections

import numpy as np
import pytest

import ftk_inputs as fi
from oracle import post


@pytest.mark.parametrize("t0", [0.0, 2.5, 3.25, 7.75])
def test_slice_moving_minimum(oracle_lib, t0):
    me = fi.MovingExtremum((16, 15), 9, c0=(5.0, 6.0), v=(0.5, 0.25))
    rec, _, _ = oracle_lib.track(me.generate().numpy(), me.scale_log2)
    nbr = post.adjacency(rec, (16, 15, 9))
    pts = post.slice_at(rec, nbr, t0)
    # one distinct point (several faces share it at a vertex hit, t0 = 0, 4, 8: the SoS path)
    distinct = {(int(p["label"]), float(p["x"]), float(p["y"])) for p in pts}
    assert len(distinct) == 1
    cx, cy = me.center(t0)
    assert abs(pts[0]["x"] - cx) < 1e-9 and abs(pts[0]["y"] - cy) < 1e-9 and pts[0]["t"] == t0


def _components(rec, nbr):
    seen, comps = set(), []
    for i in range(len(rec)):
        if i in seen:
            continue
        stack, comp = [i], []
        seen.add(i)
        while stack:
            k = stack.pop()
            comp.append(k)
            for j in nbr[k]:
                if j not in seen:
                    seen.add(j)
                    stack.append(j)
        comps.append(comp)
    return comps


def test_adjacency_partition_and_ends(oracle_lib):
    w = fi.Woven(48, 40, 12, L=15.0, sigma=0.02)
    rec, _, _ = oracle_lib.track(w.generate().numpy(), 26)
    nbr = post.adjacency(rec, (48, 40, 12))
    assert all(len(v) <= 2 for v in nbr.values())
    for comp in _components(rec, nbr):
        labels = {int(rec[k]["label"]) for k in comp}
        assert labels == {min(int(rec[k]["face_id"]) for k in comp)}
        ends = sum(1 for k in comp if len(nbr[k]) < 2)
        assert ends in (0, 2)
        nb = sum(1 for k in comp if rec[k]["flags"] & oracle_lib.FL_BOUNDARY)
        assert ends == nb  # an end is exactly a domain-boundary face


def test_filter_loops_and_duration(oracle_lib):
    w = fi.Woven(64, 64, 16, L=15.0, sigma=0.02)
    rec, _, _ = oracle_lib.track(w.generate().numpy(), 26)
    nbr = post.adjacency(rec, (64, 64, 16))
    comps = _components(rec, nbr)
    loops = [c for c in comps if all(len(nbr[k]) == 2 for k in c)]
    assert len(loops) > 0
    kept = post.filter_trajectories(rec, nbr, 0.0, drop_loops=True)
    assert len(kept) == len(rec) - sum(len(c) for c in loops)
    dur = {int(rec[c[0]]["label"]): float(np.ptp(rec["t"][c])) for c in comps}
    for d in (1.0, 4.0, 10.0):
        k = post.filter_trajectories(rec, nbr, d)
        assert set(k["label"].tolist()) == {lab for lab, v in dur.items() if v >= d}


def test_smoothing_on_a_path():
    import oracle
    n = 9
    rec = np.zeros(n, oracle.CP_DTYPE)
    rec["t"] = np.arange(n)
    rec["face_id"] = np.arange(n)
    types = [1, 1, 1, 2, 1, 1, 5, 5, 5]  # a spike at 3; a genuine change at 6
    rec["type"] = types
    nbr = {i: [j for j in (i - 1, i + 1) if 0 <= j < n] for i in range(n)}
    out = post.smooth_types(rec, nbr, 2)
    assert out["type"].tolist() == [1, 1, 1, 1, 1, 1, 5, 5, 5]
    out1 = post.smooth_types(rec, nbr, 1)
    assert out1["type"].tolist() == [1, 1, 1, 1, 1, 1, 5, 5, 5]


def _path(t, types, loop=False):
    import oracle
    n = len(t)
    rec = np.zeros(n, oracle.CP_DTYPE)
    rec["t"] = t
    rec["face_id"] = np.arange(n)
    rec["type"] = types
    if loop:
        nbr = {i: [(i - 1) % n, (i + 1) % n] for i in range(n)}
    else:
        nbr = {i: [j for j in (i - 1, i + 1) if 0 <= j < n] for i in range(n)}
    return rec, nbr


def test_simplification_fig9b():
    # sink forward to the death fold at t = 3 (index 3), saddle back to the birth fold at t = 2.25
    # (index 5), sink forward: the saddle segment [3, 5] spans 3 - 2.25 = 0.75 in time (exact in binary),
    # outer records 2, 6
    t = [0, 1, 2, 3, 2.5, 2.25, 2.75, 4, 5]
    rec, nbr = _path(t, [1, 1, 1, 2, 2, 2, 1, 1, 1])
    assert post.simplify_types(rec, nbr, 0.76)["type"].tolist() == [1] * 9
    assert post.simplify_types(rec, nbr, 0.75)["type"].tolist() == [1, 1, 1, 2, 2, 2, 1, 1, 1]
    assert post.simplify_types(rec, nbr, 0.0)["type"].tolist() == [1, 1, 1, 2, 2, 2, 1, 1, 1]
    assert post.simplify_types(rec, nbr, -1.0)["type"].tolist() == [1, 1, 1, 2, 2, 2, 1, 1, 1]
    # a genuine change: the outer records differ
    rec2, _ = _path(t, [1, 1, 1, 2, 2, 2, 3, 3, 3])
    assert post.simplify_types(rec2, nbr, 10.0)["type"].tolist() == [1, 1, 1, 2, 2, 2, 3, 3, 3]


def test_simplification_ends_and_clash():
    # folds at 1 (t 1: both partners earlier) and 2 (t 0.5: both later); end segments are never cut
    rec, nbr = _path([0, 1, 0.5, 3], [1, 2, 2, 1])
    assert post.simplify_types(rec, nbr, 1.0)["type"].tolist() == [1, 1, 1, 1]
    rec, nbr = _path([0, 1, 0.5, 3], [2, 1, 1, 1])
    assert post.simplify_types(rec, nbr, 1.0)["type"].tolist() == [2, 1, 1, 1]
    # folds at 1, 2, 3, 4; segments [1,2] (extent 0.5, outer 0 / 3: types 1 / 1), [2,3] (0.25, outer 1 / 4:
    # 7 / 7), [3,4] (0.125, outer 2 / 5: 4 / 3); record 2 is in two qualifying segments with T = 1 and 7
    rec, nbr = _path([0, 2, 1.5, 1.75, 1.625, 3], [1, 7, 4, 1, 7, 3])
    assert post.simplify_types(rec, nbr, 1.0)["type"].tolist() == [1, 1, 4, 7, 7, 3]


def test_simplification_loop():
    # every record of this 4-loop is a fold; segments [0,1] 1.0, [1,2] 0.625, [2,3] 0.875, [3,0] 1.25
    rec, nbr = _path([0, 1, 0.375, 1.25], [5, 2, 2, 5], loop=True)
    assert post.simplify_types(rec, nbr, 0.7)["type"].tolist() == [5, 5, 5, 5]
    assert post.simplify_types(rec, nbr, 0.5)["type"].tolist() == [5, 2, 2, 5]
    # [2,3] also qualifies at 0.9 (outer 1 / 0: types 2 / 5 differ) -- nothing more changes
    assert post.simplify_types(rec, nbr, 0.9)["type"].tolist() == [5, 5, 5, 5]
