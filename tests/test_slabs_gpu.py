"""Time slabs on one GPU (virtual ranks): every slab runs the real track kernels with its ghost
plane, exports its stitch lists, the lists are concatenated (standing in for the NCCL allgather),
resolved, and applied with the device relabel kernel.  The union over slabs must equal the
single-domain result and the oracle bit for bit, labels included."""
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
    return m


def run_slabs(ftk, field_cpu, s, G, vector=False):
    nt = field_cpu.shape[0]
    b = ftk.slab_bounds(nt, G)
    parts = []
    for r in range(G):
        ghost = r < G - 1
        sub = field_cpu[b[r]: b[r + 1] + (1 if ghost else 0)].contiguous().cuda()
        rec, buf = ftk.track(sub, s, t0=b[r], nt_global=nt, ghost=ghost, return_buffers=True, vector=vector)
        A, B = ftk.stitch_export(sub, s, b[r], nt, ghost, buf, vector=vector)
        parts.append((sub, rec, buf, A, B))
    GA = np.concatenate([p[3] for p in parts])
    GB = np.concatenate([p[4] for p in parts])
    out = []
    for sub, rec, buf, A, B in parts:
        mine = np.concatenate([A[:, 1], B[:, 1]])
        old, new = ftk.stitch_resolve(GA, GB, mine)
        ftk.relabel(rec, old, new, buf)
        out.append(ftk.to_numpy(rec))
    return np.concatenate(out)


def _sorted(a):
    return a[np.argsort(a["face_id"], kind="stable")]


@pytest.mark.parametrize("G", [2, 3, 4, 7])
def test_virtual_slabs_match_single_domain(ftk, oracle_lib, G):
    w = fi.Woven(96, 80, 29, sigma=0.02)
    f = w.generate()
    got = _sorted(run_slabs(ftk, f, 26, G))
    single = _sorted(ftk.to_numpy(ftk.track(f.cuda(), 26)))
    ref, _, _ = oracle_lib.track(f.numpy(), 26)
    ref = _sorted(ref)
    assert got.tobytes() == single.tobytes()
    assert np.array_equal(got["face_id"], ref["face_id"]) and np.array_equal(got["label"], ref["label"])


def test_virtual_slabs_3d(ftk, oracle_lib):
    w = fi.Woven(23, 21, 9, L=15.0, sigma=0.02, nz=19)
    f = w.generate()
    got = _sorted(run_slabs(ftk, f, 26, 3))
    ref, _, _ = oracle_lib.track(f.numpy(), 26)
    ref = _sorted(ref)
    assert np.array_equal(got["face_id"], ref["face_id"]) and np.array_equal(got["label"], ref["label"])


@pytest.mark.parametrize("G", [2, 3])
def test_virtual_slabs_vector(ftk, oracle_lib, G):
    """time slabs of 2D and 3D vector fields (FTK_VECTOR_FIELD): same records and labels as one domain"""
    for f, s in ((fi.DoubleGyre(150, 75, 23).generate(), 26), (fi.ABCFlow(24, 20, 18, 9).generate(), 26)):
        got = _sorted(run_slabs(ftk, f, s, G, vector=True))
        single = _sorted(ftk.to_numpy(ftk.track(f.cuda(), s, vector=True)))
        ref, _, _ = oracle_lib.track(f.numpy(), s, vector=True)
        ref = _sorted(ref)
        assert got.tobytes() == single.tobytes()
        assert np.array_equal(got["face_id"], ref["face_id"]) and np.array_equal(got["label"], ref["label"])


def test_nccl_communicator_single_rank(ftk):
    """the NCCL communicator initialises (world 1: track runs without a stitch)"""
    import ctypes
    import os
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29571")
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = ftk.Comm(0, 1)
        w = fi.Woven(64, 48, 10, sigma=0.02)
        f = w.generate().cuda()
        a = ftk.to_numpy(ftk.track(f, 26, comm=comm.ptr))
        b = ftk.to_numpy(ftk.track(f, 26))
        assert _sorted(a).tobytes() == _sorted(b).tobytes()
        comm.close()
    finally:
        dist.destroy_process_group()


def run_slabs_device(ftk, field_cpu, s, G, cap=4096):
    """the device seam path: packed blocks concatenated (standing in for the NCCL allgather), resolved
    and relabelled on the GPU by every slab"""
    nt = field_cpu.shape[0]
    b = ftk.slab_bounds(nt, G)
    stride = ftk.seam_block_size(cap)
    blocks = torch.full((G * stride,), -7, dtype=torch.int64, device="cuda")
    parts = []
    for r in range(G):
        ghost = r < G - 1
        sub = field_cpu[b[r]: b[r + 1] + (1 if ghost else 0)].contiguous().cuda()
        rec, buf = ftk.track(sub, s, t0=b[r], nt_global=nt, ghost=ghost, return_buffers=True)
        ftk.seam_pack(sub, s, b[r], nt, ghost, buf, blocks[r * stride:(r + 1) * stride], cap)
        parts.append(rec)
    out = []
    for rec in parts:
        ftk.seam_resolve(blocks, G, cap, rec)
        out.append(ftk.to_numpy(rec))
    return np.concatenate(out)


@pytest.mark.parametrize("G", [2, 3, 5])
def test_device_seam_resolve_matches_single_domain(ftk, oracle_lib, G):
    w = fi.Woven(96, 80, 29, sigma=0.02)
    f = w.generate()
    got = _sorted(run_slabs_device(ftk, f, 26, G))
    ref, _, _ = oracle_lib.track(f.numpy(), 26)
    ref = _sorted(ref)
    assert np.array_equal(got["face_id"], ref["face_id"]) and np.array_equal(got["label"], ref["label"])


def test_device_seam_resolve_3d_and_overflow(ftk, oracle_lib):
    w = fi.Woven(23, 21, 9, L=15.0, sigma=0.02, nz=19)
    f = w.generate()
    got = _sorted(run_slabs_device(ftk, f, 26, 3))
    ref, _, _ = oracle_lib.track(f.numpy(), 26)
    ref = _sorted(ref)
    assert np.array_equal(got["face_id"], ref["face_id"]) and np.array_equal(got["label"], ref["label"])
    # a block too small for a slab's list: FTK_ERR_CAPACITY and nothing relabelled
    with pytest.raises(ftk.FtkError) as e:
        run_slabs_device(ftk, fi.Woven(96, 80, 29, sigma=0.02).generate(), 26, 2, cap=2)
    assert e.value.status == ftk.ERR_CAPACITY
