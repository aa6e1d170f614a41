"""Pins of the oracle's vector-field path (critical points of a 2D time-varying
vector field, typed as sources, sinks and saddles from the Jacobian's eigensystem; R17):

* gradient equivalence: the vector field v = g / 2^s, with g the integer gradient of a scalar field
  computed HERE (numpy, reading R7), quantizes back to exactly g, so the vector path must reproduce
  the scalar path's punctured faces, trajectory labels and locations bit for bit; the Jacobian of a
  gradient field is the symmetric wide-stencil Hessian, so minima come out as sources, maxima as
  sinks and saddles as saddles (checked on the generic bulk);
* closed form: v = A (x - c(t)) is exactly linear, so every timestep has one punctured ordinal face at
  c(t), all of them one trajectory, typed by A (source, sink, saddle, spiral source, centre);
* double gyre census at t = 0: exactly the two interior vortex centres
  (0.5, 0.5) and (1.5, 0.5), not saddles;
* the 0/2 invariant on degenerate vector fields (values in {-1, 0, 1})."""
import numpy as np
import pytest
import torch

import ftk_inputs as fi


def int_gradient(f: np.ndarray, s: int) -> np.ndarray:
    """[t][y][x] -> [t][y][x][2] integer gradient (2x derivative, one-sided doubled at the boundary)"""
    q = np.rint(np.ldexp(f.astype(np.float64), s)).astype(np.int64)
    g = np.zeros(q.shape + (2,), np.int64)
    for a, ax in ((0, 2), (1, 1)):  # component 0 = x (array axis 2), 1 = y (axis 1)
        n = q.shape[ax]
        sl = lambda i: tuple(slice(None) if k != ax else i for k in range(3))
        g[sl(slice(1, n - 1)) + (a,)] = q[sl(slice(2, n))] - q[sl(slice(0, n - 2))]
        g[sl(0) + (a,)] = 2 * (q[sl(1)] - q[sl(0)])
        g[sl(n - 1) + (a,)] = 2 * (q[sl(n - 1)] - q[sl(n - 2)])
    return g


def test_gradient_equivalence(oracle_lib):
    s = 26
    f = fi.CONFIGS["C1"].make().generate().numpy()
    g = int_gradient(f, s)
    v = np.ldexp(g.astype(np.float64), -s)  # exact: |g| < 2^53
    vec, _, vinfo = oracle_lib.track(v, s, vector=True)
    sca, _, sinfo = oracle_lib.track(f, s)
    assert vinfo["bad_cells"] == 0 and len(vec) == len(sca) == 1116
    for k in ("face_id", "label", "x", "y", "t", "flags"):
        assert np.array_equal(vec[k], sca[k]), k
    o = oracle_lib
    mapped = {o.MIN: o.SOURCE, o.MAX: o.SINK, o.SADDLE: o.SADDLE}
    agree = np.mean([mapped.get(int(a), -1) == int(b) for a, b in zip(sca["type"], vec["type"])])
    assert agree > 0.9, agree


@pytest.mark.parametrize("A,expect", [
    (((2, 1), (0, 3)), "SOURCE"),
    (((-2, -1), (0, -3)), "SINK"),
    (((1, 0), (0, -2)), "SADDLE"),
    (((1, -3), (3, 1)), "SOURCE"),   # spiral source: complex eigenvalues, positive real part
    (((0, -1), (1, 0)), "CENTER"),   # trace exactly 0
])
def test_moving_linear_closed_form(oracle_lib, A, expect):
    m = fi.MovingLinear((16, 15), 9, A=A, c0=(5.0, 6.0), w=(0.5, 0.25))  # vertex hits at t = 0, 4, 8
    rec, _, info = oracle_lib.track(m.generate().numpy(), m.scale_log2, vector=True)
    assert info["bad_cells"] == 0
    ordn = rec[(rec["flags"] & oracle_lib.FL_ORDINAL) != 0]
    assert len(ordn) == 9
    for r in ordn:
        cx, cy = m.center(r["t"])
        assert abs(r["x"] - cx) < 1e-12 and abs(r["y"] - cy) < 1e-12
    assert set(rec["type"].tolist()) == {getattr(oracle_lib, expect)}
    assert len(set(rec["label"].tolist())) == 1


def test_double_gyre_census_t0(oracle_lib):
    dg = fi.DoubleGyre(129, 65, 3)
    rec, _, info = oracle_lib.track(dg.generate().numpy(), dg.scale_log2, vector=True)
    assert info["bad_cells"] == 0
    h = 2.0 / 128
    t0 = rec[((rec["flags"] & oracle_lib.FL_ORDINAL) != 0) & (rec["t"] == 0.0)]
    inner = t0[(t0["x"] * h > 0.1) & (t0["x"] * h < 1.9) & (t0["y"] * h > 0.1) & (t0["y"] * h < 0.9)]
    assert len(inner) == 2
    got = sorted((float(r["x"]) * h, float(r["y"]) * h) for r in inner)
    for (x, y), (ex, ey) in zip(got, [(0.5, 0.5), (1.5, 0.5)]):
        assert abs(x - ex) < 0.01 and abs(y - ey) < 0.01
    assert all(int(r["type"]) in (oracle_lib.SOURCE, oracle_lib.SINK, oracle_lib.CENTER) for r in inner)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_zero_or_two_vector_degenerate(oracle_lib, seed):
    g = torch.Generator().manual_seed(seed)
    v = torch.tensor([-1.0, 0.0, 1.0], dtype=torch.float64)[torch.randint(0, 3, (4, 6, 7, 2), generator=g)]
    rec, _, info = oracle_lib.track(v.numpy().astype(np.float32), 0, vector=True)
    assert info["bad_cells"] == 0 and len(rec) > 0


# ------------------------------------------------------------------------------------ 3D vector fields
def int_gradient3(f: np.ndarray, s: int) -> np.ndarray:
    """[t][z][y][x] -> [t][z][y][x][3] integer gradient (R7), components x, y, z"""
    q = np.rint(np.ldexp(f.astype(np.float64), s)).astype(np.int64)
    g = np.zeros(q.shape + (3,), np.int64)
    for a, ax in ((0, 3), (1, 2), (2, 1)):
        n = q.shape[ax]
        sl = lambda i: tuple(slice(None) if k != ax else i for k in range(4))
        g[sl(slice(1, n - 1)) + (a,)] = q[sl(slice(2, n))] - q[sl(slice(0, n - 2))]
        g[sl(0) + (a,)] = 2 * (q[sl(1)] - q[sl(0)])
        g[sl(n - 1) + (a,)] = 2 * (q[sl(n - 1)] - q[sl(n - 2)])
    return g


def test_gradient_equivalence_3d(oracle_lib):
    s = 26
    f = fi.Woven(12, 11, 5, L=15.0, nz=10).generate().numpy()
    v = np.ldexp(int_gradient3(f, s).astype(np.float64), -s)
    vec, _, vinfo = oracle_lib.track(v, s, vector=True)
    sca, _, _ = oracle_lib.track(f, s)
    assert vinfo["bad_cells"] == 0 and len(vec) == len(sca) > 0
    for k in ("face_id", "label", "x", "y", "z", "t", "flags"):
        assert np.array_equal(vec[k], sca[k]), k


@pytest.mark.parametrize("A,expect", [
    (((1, 0, 0), (0, 2, 0), (0, 0, 3)), "SOURCE"),
    (((-1, 0, 0), (0, -2, 0), (0, 0, -3)), "SINK"),
    (((1, 0, 0), (0, 2, 0), (0, 0, -3)), "SADDLE"),     # trace 0: Routh's epsilon rule
    (((1, 1, 0), (0, 1, 0), (0, 0, -1)), "SADDLE"),     # eigenvalues 1, 1, -1: a1 a2 == a3, a2 < 0
    (((-1, -2, 0), (2, -1, 0), (0, 0, -1)), "SINK"),    # spiral sink
    (((0, -1, 0), (1, 0, 0), (0, 0, -1)), "CENTER"),    # +-i and -1: a1 a2 == a3, a2 > 0
])
def test_moving_linear_3d(oracle_lib, A, expect):
    m = fi.MovingLinear3((9, 8, 10), 5, A=A, c0=(3.0, 3.0, 4.0), w=(0.5, 0.25, 0.125))
    rec, _, info = oracle_lib.track(m.generate().numpy(), m.scale_log2, vector=True)
    assert info["bad_cells"] == 0
    ordn = rec[(rec["flags"] & oracle_lib.FL_ORDINAL) != 0]
    assert len(ordn) == 5
    for r in ordn:
        c = m.center(r["t"])
        assert max(abs(r["x"] - c[0]), abs(r["y"] - c[1]), abs(r["z"] - c[2])) < 1e-12
    assert set(rec["type"].tolist()) == {getattr(oracle_lib, expect)}
    assert len(set(rec["label"].tolist())) == 1
