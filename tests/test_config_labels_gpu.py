"""Trajectory-label parity at the BASELINE.json configurations (north_star: "bit-exact trajectories
against the oracle on all configs").

Labels depend on the whole domain (Alg. 1 pass 2: a trajectory is the connected
component of punctured faces over every cell of the mesh), so a time window of records cannot check
them.  Here the oracle tracks a whole domain and every record is compared, labels included:

* C2 (2D woven 1024^2 x 256): the full configuration, in the launch configuration bench.py times --
  the oracle runs on all host cores (~3.2e9 faces, a few minutes on the GPU box);
* C4 (2D woven 4096^2 x 512) and C5 (3D woven 256^3 x 64): a spatial crop over the FULL time extent,
  cut from the config's own bytes and tracked as its own domain by both sides (its edges are the
  crop's domain boundary for both);
* C3 (3D moving extremum 128^3 x 32): a 48^3 crop around the trajectory over the full time extent
  (the full C3 oracle run would take ~10 min), plus its closed form: one trajectory, MIN everywhere.

Bar: identical face ids, labels, types and flags; locations within 1e-6 grid units.
"""
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


def compare_all(gpu, ref):
    g, r = _sorted(gpu), _sorted(ref)
    assert len(g) == len(r), (len(g), len(r))
    assert np.array_equal(g["face_id"], r["face_id"])
    assert np.array_equal(g["label"], r["label"])
    assert np.array_equal(g["type"], r["type"])
    assert np.array_equal(g["flags"].astype(np.int64), r["flags"].astype(np.int64))
    dmax = 0.0
    for k in ("x", "y", "z", "t"):
        if len(g):
            dmax = max(dmax, float(np.max(np.abs(g[k] - r[k]))))
    assert dmax <= LOC_TOL, dmax
    return len(np.unique(g["label"]))


def test_c2_full_config_labels(ftk, oracle_lib):
    cfg = fi.CONFIGS["C2"]
    f = cfg.make().generate(device="cuda")
    rec = ftk.to_numpy(ftk.track(f, cfg.scale_log2))
    ref, n_faces, info = oracle_lib.track(f.cpu().numpy(), cfg.scale_log2)
    assert n_faces == 3205515258
    ntraj = compare_all(rec, ref)
    assert info["bad_cells"] == 0
    assert ntraj == info["components"] > 100


def _crop_track(ftk, oracle_lib, f_dev, s, box):
    """box: per spatial axis (lo, size) in x, y[, z] order; the full time extent"""
    sl = [slice(None)] + [slice(lo, lo + size) for lo, size in reversed(box)]
    sub = f_dev[tuple(sl)].contiguous()
    rec = ftk.to_numpy(ftk.track(sub, s))
    ref, _, info = oracle_lib.track(sub.cpu().numpy(), s)
    assert info["bad_cells"] == 0
    return compare_all(rec, ref), len(ref)


def test_c4_full_time_crop_labels(ftk, oracle_lib):
    cfg = fi.CONFIGS["C4"]
    f = cfg.make().generate(device="cuda")
    ntraj, n = _crop_track(ftk, oracle_lib, f, cfg.scale_log2, [(1536, 512), (2560, 448)])
    del f
    torch.cuda.empty_cache()
    assert n > 100000 and ntraj > 50


def test_c5_full_time_crop_labels(ftk, oracle_lib):
    cfg = fi.CONFIGS["C5"]
    f = cfg.make().generate(device="cuda")
    ntraj, n = _crop_track(ftk, oracle_lib, f, cfg.scale_log2, [(96, 64), (80, 64), (104, 64)])
    assert n > 1000 and ntraj > 5


def test_c3_trajectory_crop_labels(ftk, oracle_lib):
    cfg = fi.CONFIGS["C3"]
    f = cfg.make().generate(device="cuda")
    # c(t) = (60, 62, 64) + (1/4, 1/8, -1/16) t, t < 32: inside [40, 88)^3 with a margin of 12
    ntraj, n = _crop_track(ftk, oracle_lib, f, cfg.scale_log2, [(40, 48), (40, 48), (40, 48)])
    full = ftk.to_numpy(ftk.track(f, cfg.scale_log2))
    # closed form: one trajectory, one ordinal face per timestep, MIN everywhere
    assert len(np.unique(full["label"])) == 1
    assert set(full["type"].tolist()) == {ftk.MIN}
    assert int(np.sum((full["flags"] & ftk.CP_ORDINAL) != 0)) == 32
    assert ntraj >= 1
