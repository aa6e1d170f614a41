"""GPU isovolume tracking (ftk_iso_track) against the oracle's iso_track on the same
bytes: bit-exact crossed-edge set, component labels, types and flags; locations within 1e-6 (equal)."""
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


def run_pair(ftk, oracle_lib, f: torch.Tensor, s: int, c: float):
    g = ftk.to_numpy(ftk.iso_track(f.cuda(), s, c))
    r, _, info = oracle_lib.iso_track(f.numpy(), s, c)
    assert info["bad_cells"] == 0
    g = g[np.argsort(g["face_id"], kind="stable")]
    assert len(g) == len(r), (len(g), len(r))
    for k in ("face_id", "label", "type", "flags"):
        assert np.array_equal(g[k], r[k]), k
    for k in ("x", "y", "z", "t"):
        if len(g):
            assert np.max(np.abs(g[k] - r[k])) <= 1e-6, k
    return g, info


def plane(alpha, shape):
    nt, nx = shape[0], shape[-1]
    t = torch.arange(nt, dtype=torch.float64).reshape((nt,) + (1,) * (len(shape) - 1))
    x = torch.arange(nx, dtype=torch.float64).reshape((1,) * (len(shape) - 1) + (nx,))
    return (x - alpha * t).expand(shape).to(torch.float32).contiguous()


def test_paper_moving_plane(ftk, oracle_lib):
    """f = x - 0.9 t on 21^3 x 12 at f = 0 -- one component on x = 0.9 t"""
    g, info = run_pair(ftk, oracle_lib, plane(0.9, (12, 21, 21, 21)), 20, 0.0)
    assert info["components"] == 1 and len(set(g["label"].tolist())) == 1
    assert np.max(np.abs(g["x"] - 0.9 * g["t"])) < 1e-6


def test_moving_line_2d(ftk, oracle_lib):
    run_pair(ftk, oracle_lib, plane(0.875, (9, 13, 140)), 20, 0.0)


@pytest.mark.parametrize("shape,c", [((6, 40, 150), 0.3), ((5, 33, 47), -0.2), ((4, 12, 11, 140), 0.25),
                                     ((3, 9, 10, 11), 0.0)])
def test_woven_levels(ftk, oracle_lib, shape, c):
    if len(shape) == 3:
        nt, ny, nx = shape
        f = fi.Woven(nx, ny, nt, L=15.0, sigma=0.02).generate()
    else:
        nt, nz, ny, nx = shape
        f = fi.Woven(nx, ny, nt, L=15.0, sigma=0.02, nz=nz).generate()
    g, info = run_pair(ftk, oracle_lib, f, 26, c)
    assert len(g) > 0


@pytest.mark.parametrize("shape,seed", [((4, 5, 6, 7), 0), ((5, 9, 131), 1), ((3, 4, 4, 5), 2)])
def test_degenerate(ftk, oracle_lib, shape, seed):
    gen = torch.Generator().manual_seed(seed)
    v = torch.tensor([-1.0, 0.0, 1.0])[torch.randint(0, 3, shape, generator=gen)].to(torch.float32)
    run_pair(ftk, oracle_lib, v, 0, 0.0)


def test_fp64(ftk, oracle_lib):
    f = fi.Woven(50, 40, 5, L=15.0).generate(dtype=torch.float64)
    run_pair(ftk, oracle_lib, f, 26, 0.1)


# ----------------------------------------------------------------------- isovolume mesh
def mesh_pair(ftk, oracle_lib, f: torch.Tensor, s: int, c: float):
    """the GPU's simplices (ftk_iso_track_mesh) against the oracle's iso_mesh: the same set of simplices,
    each with the same edge ids in the same (staircase path) order"""
    rec, el = ftk.iso_track(f.cuda(), s, c, mesh=True)
    g = el.cpu().numpy()
    r = oracle_lib.iso_mesh(f.numpy(), s, c)
    assert g.shape == r.shape, (g.shape, r.shape)
    gs = set(map(tuple, g.tolist()))
    assert len(gs) == len(g)
    assert gs == set(map(tuple, r.tolist()))
    # every simplex vertex is one of the call's crossed-edge records
    assert set(np.unique(g).tolist()) <= set(ftk.to_numpy(rec)["face_id"].tolist())
    return len(g)


def test_mesh_paper_plane(ftk, oracle_lib):
    assert mesh_pair(ftk, oracle_lib, plane(0.9, (12, 21, 21, 21)), 20, 0.0) > 1000
    assert mesh_pair(ftk, oracle_lib, plane(0.875, (9, 13, 140)), 20, 0.0) > 100


@pytest.mark.parametrize("shape,c", [((6, 40, 150), 0.3), ((4, 12, 11, 140), 0.25), ((3, 9, 10, 11), 0.0)])
def test_mesh_woven(ftk, oracle_lib, shape, c):
    if len(shape) == 3:
        nt, ny, nx = shape
        f = fi.Woven(nx, ny, nt, L=15.0, sigma=0.02).generate()
    else:
        nt, nz, ny, nx = shape
        f = fi.Woven(nx, ny, nt, L=15.0, sigma=0.02, nz=nz).generate()
    assert mesh_pair(ftk, oracle_lib, f, 26, c) > 0


@pytest.mark.parametrize("shape,seed", [((4, 5, 6, 7), 0), ((5, 9, 131), 1)])
def test_mesh_degenerate(ftk, oracle_lib, shape, seed):
    gen = torch.Generator().manual_seed(seed)
    v = torch.tensor([-1.0, 0.0, 1.0])[torch.randint(0, 3, shape, generator=gen)].to(torch.float32)
    mesh_pair(ftk, oracle_lib, v, 0, 0.0)


def test_mesh_capacity_retry(ftk, oracle_lib):
    """a too-small element buffer reports FTK_ERR_CAPACITY with the count; the binding retries"""
    import ctypes
    f = fi.Woven(40, 30, 5, L=15.0).generate().cuda()
    rec, el = ftk.iso_track(f, 26, 0.2, mesh=True, capacity=1 << 16)
    desc = ftk.make_desc(tuple(f.shape), f.dtype, 26)
    buf = ftk.Buffers.allocate(desc, 1 << 16, f.device)
    small = torch.empty((4, 3), dtype=torch.int64, device="cuda")
    n_out, n_el = ctypes.c_int64(0), ctypes.c_int64(0)
    st = ftk.lib().ftk_iso_track_mesh(ctypes.byref(desc), ctypes.c_double(0.2), ctypes.c_void_p(f.data_ptr()),
                                      ctypes.c_void_p(buf.records.data_ptr()), buf.capacity, ctypes.byref(n_out),
                                      ctypes.c_void_p(small.data_ptr()), 4, ctypes.byref(n_el),
                                      ctypes.c_void_p(buf.workspace.data_ptr()), buf.workspace.numel(), None)
    assert st == ftk.ERR_CAPACITY and n_el.value == el.shape[0] > 4


def test_iso_dense_blocked_hash(ftk, oracle_lib):
    """an isovolume far denser than the critical points the pass-2 table blocks were sized for: every
    coarse cell must spread over a group of blocks (a single 4096-slot block per cell made the probe
    chains quadratic -- the C2 isovolume never finished)"""
    f = fi.Woven(512, 384, 20, sigma=0.0).generate()
    g, info = run_pair(ftk, oracle_lib, f, 26, 0.5)
    assert len(g) > 500_000
