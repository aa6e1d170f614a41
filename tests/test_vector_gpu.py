"""GPU parity of the vector-field paths (FTK_VECTOR_FIELD; §8(f) NEXT row 2): 2D
(k_scanvec2d, k_expand2d, k_exactvec2d) and 3D (k_scanvec3d, k_exact3d<T, true>), plus pass 2, against
the CPU oracle, element by element -- bit-exact punctured faces, labels, types and flags, locations
within 1e-6 (in fact equal)."""
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


def compare(g, r, labels=True):
    g, r = _sorted(g), _sorted(r)
    assert len(g) == len(r), (len(g), len(r))
    assert np.array_equal(g["face_id"], r["face_id"])
    assert np.array_equal(g["type"], r["type"])
    assert np.array_equal(g["flags"].astype(np.int64), r["flags"].astype(np.int64))
    if labels:
        assert np.array_equal(g["label"], r["label"])
    for k in ("x", "y", "z", "t"):
        if len(g):
            assert np.max(np.abs(g[k] - r[k])) <= 1e-6, k
    return len(g)


def run_pair(ftk, oracle_lib, v: torch.Tensor, s: int):
    rec = ftk.to_numpy(ftk.track(v.cuda(), s, vector=True))
    ref, _, info = oracle_lib.track(v.numpy(), s, vector=True)
    assert info["bad_cells"] == 0
    return compare(rec, ref), rec


@pytest.mark.parametrize("A", [((2, 1), (0, 3)), ((-2, -1), (0, -3)), ((1, 0), (0, -2)), ((1, -3), (3, 1)),
                               ((0, -1), (1, 0))])
def test_moving_linear(ftk, oracle_lib, A):
    m = fi.MovingLinear((150, 37), 9, A=A, c0=(70.0, 16.0), w=(0.5, 0.25))
    n, rec = run_pair(ftk, oracle_lib, m.generate(), m.scale_log2)
    assert n >= 9 and len(set(rec["label"].tolist())) == 1


@pytest.mark.parametrize("nx,ny,nt", [(129, 65, 12), (257, 130, 9), (131, 67, 40), (300, 150, 5)])
def test_double_gyre(ftk, oracle_lib, nx, ny, nt):
    dg = fi.DoubleGyre(nx, ny, nt)
    n, _ = run_pair(ftk, oracle_lib, dg.generate(), dg.scale_log2)
    assert n > 0


@pytest.mark.parametrize("seed,shape", [(0, (4, 6, 7, 2)), (1, (5, 9, 131, 2)), (2, (3, 17, 140, 2))])
def test_degenerate(ftk, oracle_lib, seed, shape):
    g = torch.Generator().manual_seed(seed)
    v = torch.tensor([-1.0, 0.0, 1.0], dtype=torch.float64)[torch.randint(0, 3, shape, generator=g)]
    run_pair(ftk, oracle_lib, v.to(torch.float32), 0)


def test_fp64_input(ftk, oracle_lib):
    dg = fi.DoubleGyre(133, 70, 7)
    run_pair(ftk, oracle_lib, dg.generate(dtype=torch.float64), dg.scale_log2)


def test_gradient_equivalence_gpu(ftk):
    """v = (integer gradient of f) / 2^s: the vector path reproduces the scalar path's faces, labels and
    locations bit for bit on the GPU (C1)"""
    s = 26
    f = fi.CONFIGS["C1"].make().generate()
    q = torch.round(f.double() * 2.0 ** s)  # round-half-even, exact
    g = torch.zeros(q.shape + (2,), dtype=torch.float64)
    for comp, ax in ((0, 2), (1, 1)):
        n = q.shape[ax]
        d = torch.zeros_like(q)
        d.narrow(ax, 1, n - 2).copy_(q.narrow(ax, 2, n - 2) - q.narrow(ax, 0, n - 2))
        d.narrow(ax, 0, 1).copy_(2 * (q.narrow(ax, 1, 1) - q.narrow(ax, 0, 1)))
        d.narrow(ax, n - 1, 1).copy_(2 * (q.narrow(ax, n - 1, 1) - q.narrow(ax, n - 2, 1)))
        g[..., comp] = d
    v = g * 2.0 ** -s
    vec = _sorted(ftk.to_numpy(ftk.track(v.cuda(), s, vector=True)))
    sca = _sorted(ftk.to_numpy(ftk.track(f.cuda(), s)))
    assert len(vec) == len(sca) == 1116
    for k in ("face_id", "label", "x", "y", "t", "flags"):
        assert np.array_equal(vec[k], sca[k]), k


@pytest.mark.parametrize("window", [1, 4, 64])
def test_vector_stream(ftk, window):
    dg = fi.DoubleGyre(200, 100, 15)
    v = dg.generate()
    tr = ftk.Tracker((100, 200, 2), torch.float32, dg.scale_log2, 1 << 16, window=window, vector=True)
    for t in range(v.shape[0]):
        tr.push(v[t].cuda())
    a = _sorted(ftk.to_numpy(tr.finish()))
    b = _sorted(ftk.to_numpy(ftk.track(v.cuda(), dg.scale_log2, vector=True)))
    assert a.tobytes() == b.tobytes()


def test_v2_full_size_sampled(ftk, oracle_lib):
    """V2 (double gyre 2048 x 1024 x 256, the vector bench config) at full size: a window of
    timesteps against the oracle's extract on the same bytes."""
    cfg = fi.CONFIGS["V2"]
    dg = cfg.make()
    v = dg.generate(device="cuda")
    rec = ftk.to_numpy(ftk.track(v, cfg.scale_log2, vector=True))
    nt = v.shape[0]
    t_of = rec["face_id"] // 12 // (v.shape[1] * v.shape[2])
    ta, tb = 100, 102
    sub = v[ta: tb + 1].cpu().numpy()
    ref, _ = oracle_lib.extract(sub, cfg.scale_log2, t0=ta, nt_global=nt, ta=ta, tb=tb, vector=True)
    compare(rec[(t_of >= ta) & (t_of < tb)], ref, labels=False)


# ------------------------------------------------------------------------------------ 3D vector fields
@pytest.mark.parametrize("A", [((1, 0, 0), (0, 2, 0), (0, 0, 3)), ((1, 0, 0), (0, 2, 0), (0, 0, -3)),
                               ((-1, -2, 0), (2, -1, 0), (0, 0, -1)), ((0, -1, 0), (1, 0, 0), (0, 0, -1))])
def test_moving_linear_3d(ftk, oracle_lib, A):
    m = fi.MovingLinear3((140, 9, 10), 5, A=A, c0=(70.0, 3.0, 4.0), w=(0.5, 0.25, 0.125))
    n, rec = run_pair(ftk, oracle_lib, m.generate(), m.scale_log2)
    assert n >= 5 and len(set(rec["label"].tolist())) == 1


@pytest.mark.parametrize("shape,s", [((24, 20, 18, 6), 26), ((131, 9, 7, 4), 26), ((16, 16, 16, 5), 36)])
def test_abc_flow_3d(ftk, oracle_lib, shape, s):
    nx, ny, nz, nt = shape
    v = fi.ABCFlow(nx, ny, nz, nt, scale_log2=s).generate()
    run_pair(ftk, oracle_lib, v, s)


def test_degenerate_3d_vector(ftk, oracle_lib):
    g = torch.Generator().manual_seed(7)
    v = torch.tensor([-1.0, 0.0, 1.0], dtype=torch.float64)[torch.randint(0, 3, (3, 5, 6, 7, 3), generator=g)]
    run_pair(ftk, oracle_lib, v.to(torch.float32), 0)


def test_gradient_equivalence_3d_gpu(ftk):
    s = 26
    f = fi.Woven(20, 18, 6, L=15.0, nz=16).generate()
    q = torch.round(f.double() * 2.0 ** s)
    g = torch.zeros(q.shape + (3,), dtype=torch.float64)
    for comp, ax in ((0, 3), (1, 2), (2, 1)):
        n = q.shape[ax]
        d = torch.zeros_like(q)
        d.narrow(ax, 1, n - 2).copy_(q.narrow(ax, 2, n - 2) - q.narrow(ax, 0, n - 2))
        d.narrow(ax, 0, 1).copy_(2 * (q.narrow(ax, 1, 1) - q.narrow(ax, 0, 1)))
        d.narrow(ax, n - 1, 1).copy_(2 * (q.narrow(ax, n - 1, 1) - q.narrow(ax, n - 2, 1)))
        g[..., comp] = d
    v = g * 2.0 ** -s
    vec = _sorted(ftk.to_numpy(ftk.track(v.cuda(), s, vector=True)))
    sca = _sorted(ftk.to_numpy(ftk.track(f.cuda(), s)))
    assert len(vec) == len(sca) > 0
    for k in ("face_id", "label", "x", "y", "z", "t", "flags"):
        assert np.array_equal(vec[k], sca[k]), k


def test_3d_vector_stream(ftk):
    v = fi.ABCFlow(24, 20, 18, 9).generate()
    tr = ftk.Tracker((18, 20, 24, 3), torch.float32, 26, 1 << 14, window=3, vector=True)
    for t in range(v.shape[0]):
        tr.push(v[t].cuda())
    a = _sorted(ftk.to_numpy(tr.finish()))
    b = _sorted(ftk.to_numpy(ftk.track(v.cuda(), 26, vector=True)))
    assert a.tobytes() == b.tobytes()
