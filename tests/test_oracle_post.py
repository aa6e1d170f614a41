"""Pins of the post-processing reference (oracle/post.py):

* slicing: the moving minimum's trajectory is the straight line c(t) (its PL gradient is exactly
  affine), so the slice at any t0 -- integer or not -- is exactly one point, at c(t0);
* adjacency: every face has at most two partners; open trajectories have exactly two ends, loops none
  (P:447); the partition it induces equals the labels of the track;
* filtering: on the noisy woven field dropping loops leaves exactly the open
  trajectories, and a duration threshold keeps exactly the trajectories at least that long;
* smoothing: a single-record type spike inside a uniform trajectory is corrected, ends and
  genuine type changes are kept."""
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
