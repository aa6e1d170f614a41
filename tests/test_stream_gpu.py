"""Streaming ingestion (PAPER.md:709 push_field_data; include/ftk_cp.h ftk_tracker_*): pushing the
timesteps one at a time must give exactly the records of one track() over the whole field -- same
punctured faces, labels (trajectory = min face id across all windows), types, flags and locations --
whatever the window, for device and host planes; and the CPU oracle agrees."""
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


def _sorted(a):
    return a[np.argsort(a["face_id"], kind="stable")]


def stream(ftk, field, s, window, capacity=None, host=False, pinned=False):
    cap = capacity or max(1 << 14, field.numel() // 16)
    tr = ftk.Tracker(tuple(field.shape[1:]), field.dtype, s, cap, window=window)
    src = field.cpu() if host else field.cuda()
    for t in range(field.shape[0]):
        p = src[t]
        if pinned:
            p = p.pin_memory()
        tr.push(p)
    return ftk.to_numpy(tr.finish())


def same(a, b):
    a, b = _sorted(a), _sorted(b)
    assert len(a) == len(b)
    assert a.tobytes() == b.tobytes()  # every field, bit for bit


@pytest.mark.parametrize("window", [1, 2, 3, 7, 8, 64])
def test_c1_stream_equals_oracle_and_batch(ftk, oracle_lib, window):
    f = fi.CONFIGS["C1"].make().generate()
    rec = stream(ftk, f, 26, window)
    ref, _, _ = oracle_lib.track(f.numpy(), 26)
    g, r = _sorted(rec), _sorted(ref)
    assert len(g) == len(r) == 1116
    for k in ("face_id", "label", "type", "flags"):
        assert np.array_equal(g[k], r[k]), k
    for k in ("x", "y", "t"):
        assert np.max(np.abs(g[k] - r[k])) <= 1e-6
    same(rec, ftk.to_numpy(ftk.track(f.cuda(), 26)))


@pytest.mark.parametrize("host,pinned", [(True, False), (True, True)])
def test_host_planes(ftk, host, pinned):
    f = fi.Woven(150, 70, 21, sigma=0.02).generate()
    same(stream(ftk, f, 26, 5, host=host, pinned=pinned), ftk.to_numpy(ftk.track(f.cuda(), 26)))


def test_noisy_ragged_windows(ftk, oracle_lib):
    f = fi.Woven(131, 97, 35, sigma=0.08).generate()
    rec = stream(ftk, f, 26, 6, capacity=f.numel())
    ref, _, _ = oracle_lib.track(f.numpy(), 26)
    g, r = _sorted(rec), _sorted(ref)
    assert np.array_equal(g["face_id"], r["face_id"]) and np.array_equal(g["label"], r["label"])
    same(rec, ftk.to_numpy(ftk.track(f.cuda(), 26)))


@pytest.mark.parametrize("window", [2, 5])
def test_3d_stream(ftk, oracle_lib, window):
    f = fi.Woven(24, 20, 9, L=15.0, sigma=0.02, nz=18).generate()
    rec = stream(ftk, f, 26, window)
    ref, _, _ = oracle_lib.track(f.numpy(), 26)
    g, r = _sorted(rec), _sorted(ref)
    assert np.array_equal(g["face_id"], r["face_id"]) and np.array_equal(g["label"], r["label"])
    same(rec, ftk.to_numpy(ftk.track(f.cuda(), 26)))


def test_c2_full_size_stream(ftk):
    """C2 (1024^2 x 256) pushed plane by plane from the device in windows of 64: bit-identical to the
    batch track (2.7 M records, labels over trajectories that cross every window boundary)."""
    cfg = fi.CONFIGS["C2"]
    f = cfg.make().generate(device="cuda")
    batch = ftk.to_numpy(ftk.track(f, cfg.scale_log2))
    rec = stream(ftk, f, cfg.scale_log2, 64, capacity=4 << 20)
    same(rec, batch)


def test_errors(ftk):
    f = fi.CONFIGS["C1"].make().generate()
    tr = ftk.Tracker((32, 32), torch.float32, 26, 4096, window=4)
    tr.push(f[0].cuda())
    with pytest.raises(ftk.FtkError) as e:  # tracking needs two timesteps
        tr.finish()
    assert e.value.status == ftk.ERR_INVALID_ARG
    tr = ftk.Tracker((32, 32), torch.float32, 26, 100, window=3)
    for t in range(8):
        tr.push(f[t].cuda())
    with pytest.raises(ftk.FtkError) as e:  # 1116 records do not fit
        tr.finish()
    assert e.value.status == ftk.ERR_CAPACITY
    with pytest.raises(ftk.FtkError):
        tr.push(f[0].cuda())
