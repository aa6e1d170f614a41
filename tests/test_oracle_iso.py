"""Pins of the oracle's isovolume tracking (Alg. 1 right):

* the paper's synthetic case: f = x - alpha t on a 21^3 grid x 12 timesteps, isovalue 0 -- every
  crossing point lies on the hyperplane x = alpha t (exactly for the dyadic alpha = 7/8, within the
  2^-20 quantization of 0.9 otherwise) and the isovolume is ONE component;
* the 2D+t analogue: f = x - alpha t on a 2D grid gives the line x = alpha t in every timestep;
* exactly-once / case I-II invariant: every cell has 0, d or 2(d-1) crossed edges,
  also on massively degenerate fields (values in {-1, 0, 1} at isovalue 0: the SoS rule counts a vertex
  on the level set as above it);
* brute force: the crossed-edge set equals a numpy enumeration of all Kuhn edges with differing signs."""
import itertools

import numpy as np
import pytest
import torch


def plane(alpha, shape):
    nt = shape[0]
    nx = shape[-1]
    t = torch.arange(nt, dtype=torch.float64).reshape((nt,) + (1,) * (len(shape) - 1))
    x = torch.arange(nx, dtype=torch.float64).reshape((1,) * (len(shape) - 1) + (nx,))
    return (x - alpha * t).expand(shape).to(torch.float32).numpy().copy()


@pytest.mark.parametrize("alpha,tol", [(0.9, 1e-6), (0.875, 1e-12)])
def test_moving_plane_3d(oracle_lib, alpha, tol):
    rec, ne, info = oracle_lib.iso_track(plane(alpha, (12, 21, 21, 21)), 20, 0.0)
    assert info["bad_cells"] == 0 and info["components"] == 1 and len(rec) > 0
    assert np.max(np.abs(rec["x"] - alpha * rec["t"])) < tol
    assert ne == sum(int(np.prod([n - ((m >> a) & 1) for a, n in enumerate((21, 21, 21, 12))])) for m in range(1, 16))


def test_moving_plane_2d(oracle_lib):
    rec, ne, info = oracle_lib.iso_track(plane(0.875, (9, 13, 17)), 20, 0.0)
    assert info["bad_cells"] == 0 and info["components"] == 1
    assert np.max(np.abs(rec["x"] - 0.875 * rec["t"])) < 1e-12


@pytest.mark.parametrize("shape,seed", [((4, 5, 6, 7), 0), ((5, 9, 11), 1), ((3, 4, 4, 5), 2)])
def test_invariant_degenerate(oracle_lib, shape, seed):
    g = torch.Generator().manual_seed(seed)
    v = torch.tensor([-1.0, 0.0, 1.0])[torch.randint(0, 3, shape, generator=g)].numpy().astype(np.float32)
    rec, ne, info = oracle_lib.iso_track(v, 0, 0.0)
    assert info["bad_cells"] == 0 and len(rec) > 0


def test_crossed_edges_brute_force(oracle_lib):
    g = torch.Generator().manual_seed(3)
    f = torch.randn((4, 5, 6), generator=g).numpy().astype(np.float32)
    rec, _, _ = oracle_lib.iso_track(f, 10, 0.1)
    q = np.rint(np.ldexp(f.astype(np.float64), 10)).astype(np.int64) - int(np.rint(0.1 * 2 ** 10))
    nt, ny, nx = f.shape
    want = set()
    for t, y, x in itertools.product(range(nt), range(ny), range(nx)):
        for m in range(1, 8):
            b = (x + (m & 1), y + ((m >> 1) & 1), t + ((m >> 2) & 1))
            if b[0] < nx and b[1] < ny and b[2] < nt and (q[t, y, x] >= 0) != (q[b[2], b[1], b[0]] >= 0):
                want.add((x + nx * (y + ny * t)) * 7 + m - 1)
    assert set(rec["face_id"].tolist()) == want
