"""Pins of the oracle's isovolume mesh (oracle.iso_mesh) against what the
paper and geometry fix:

* the paper's synthetic case f = x - alpha t, level 0: the zero set is the hyperplane x = alpha t,
  so the simplices (vertices at the records' Eq. 2 locations) must tile its piece inside the domain --
  their total (n)-volume equals the analytic one, sqrt(1 + alpha^2) * (ny - 1) [(nz - 1)] * T;
* the simplices form a combinatorial manifold: every facet is shared by at most two simplices, and a
  facet of only one lies on the domain boundary;
* brute force on tiny degenerate fields: an independent enumeration of every cell (itertools over
  cube corners and axis permutations), the SoS signs (g >= 0 positive), and the staircase of
  simplex(P) x simplex(M) (C(|P| + |M| - 2, |P| - 1) simplices, 1 in case I, 3 for ++--- in 3D+t)
  gives the same simplex set; every simplex vertex is a crossed edge of ftko_iso_track."""
import itertools
import math

import numpy as np
import pytest

import ftk_inputs as fi


def plane_field(shape, alpha):
    """f = x - alpha t on integer grid coordinates, [t][(z)][y][x] float32 (exact for dyadic alpha)"""
    nt = shape[0]
    nx = shape[-1]
    t = np.arange(nt, dtype=np.float64).reshape((nt,) + (1,) * (len(shape) - 1))
    x = np.arange(nx, dtype=np.float64)
    return (x - alpha * t + np.zeros(shape)).astype(np.float32)


def positions(rec, d):
    cols = ["x", "y"] + (["z"] if d == 4 else []) + ["t"]
    return {int(r["face_id"]): np.array([r[c] for c in cols]) for r in rec}


def simplex_volume(P):
    E = (P[1:] - P[0]).T  # d x k
    g = E.T @ E
    det = max(float(np.linalg.det(g)), 0.0)
    return math.sqrt(det) / math.factorial(P.shape[0] - 1)


@pytest.mark.parametrize("shape", [(12, 9, 21), (12, 6, 7, 21)])
def test_plane_isovolume_tiles_the_hyperplane(oracle_lib, shape):
    alpha = 0.875
    f = plane_field(shape, alpha)
    rec, _, info = oracle_lib.iso_track(f, 10, 0.0)
    el = oracle_lib.iso_mesh(f, 10, 0.0)
    d = len(shape)
    assert el.shape[1] == d
    pos = positions(rec, d)
    vol = sum(simplex_volume(np.array([pos[int(e)] for e in row])) for row in el)
    nt, nx = shape[0], shape[-1]
    T = min(nt - 1, (nx - 1) / alpha)
    cross = np.prod([n - 1 for n in shape[1:-1]])
    assert abs(vol - math.sqrt(1 + alpha * alpha) * cross * T) < 1e-9 * vol
    # every simplex vertex is a crossed edge
    assert set(np.unique(el).tolist()) <= set(pos)


@pytest.mark.parametrize("shape", [(6, 7, 8), (4, 5, 6, 7)])
def test_mesh_is_a_manifold_with_boundary(oracle_lib, shape):
    f = fi.Woven(shape[-1], shape[-2], shape[0], L=9.0, nz=shape[1] if len(shape) == 4 else 1).generate().numpy()
    rec, _, _ = oracle_lib.iso_track(f, 26, 0.3)
    el = oracle_lib.iso_mesh(f, 26, 0.3)
    d = len(shape)
    pos = positions(rec, d)
    ext = [shape[-1], shape[-2]] + ([shape[1]] if d == 4 else []) + [shape[0]]
    count = {}
    for row in el:
        for k in range(d):
            fac = tuple(sorted(int(e) for j, e in enumerate(row) if j != k))
            count[fac] = count.get(fac, 0) + 1
    assert max(count.values()) <= 2
    for fac, c in count.items():
        if c == 1:  # a boundary facet: all its points on one face of the domain box
            P = np.array([pos[e] for e in fac])
            on = [(np.all(np.abs(P[:, a]) < 1e-12) or np.all(np.abs(P[:, a] - (ext[a] - 1)) < 1e-12)) for a in range(d)]
            assert any(on), fac


def brute_mesh(f, s, c):
    """independent enumeration: every cube, every axis permutation (cell), SoS signs, staircase paths"""
    q = np.rint(f.astype(np.float64) * 2.0 ** s).astype(np.int64) - int(np.rint(c * 2.0 ** s))
    shape = f.shape
    d = len(shape)
    ext = list(reversed(shape[1:])) + [shape[0]]  # x, y, [z,] t
    E = (1 << d) - 1

    def val(v):  # v in (x, y, [z,] t)
        return q[(v[-1],) + tuple(reversed(v[:-1]))]

    def vid(v):
        i, stride = 0, 1
        for a in range(d):
            i += v[a] * stride
            stride *= ext[a]
        return i

    out = set()
    for anchor in itertools.product(*[range(n - 1) for n in ext]):
        for perm in itertools.permutations(range(d)):
            w = [list(anchor)]
            for a in perm:
                nxt = list(w[-1])
                nxt[a] += 1
                w.append(nxt)
            Pv = [k for k in range(d + 1) if val(w[k]) >= 0]
            Mv = [k for k in range(d + 1) if val(w[k]) < 0]
            if not Pv or not Mv:
                continue
            steps = len(Pv) + len(Mv) - 2
            paths = list(itertools.combinations(range(steps), len(Pv) - 1))
            assert len(paths) == math.comb(steps, len(Pv) - 1)
            for pstep in paths:
                ip = im = 0
                verts = []
                for st in range(-1, steps):
                    if st >= 0:
                        if st in pstep:
                            ip += 1
                        else:
                            im += 1
                    a, b = sorted((Pv[ip], Mv[im]))
                    m = sum((w[b][x] - w[a][x]) << x for x in range(d))
                    verts.append(vid(w[a]) * E + m - 1)
                out.add(tuple(sorted(verts)))
    return out


@pytest.mark.parametrize("shape,values,seed", [((3, 4, 5), (-1.0, 0.0, 1.0), 1), ((3, 3, 4, 3), (-1.0, 0.0, 1.0), 2),
                                                ((4, 5, 4), (-2.0, -1.0, 0.0, 1.0, 3.0), 3)])
def test_mesh_matches_brute_force(oracle_lib, shape, values, seed):
    f = fi.random_degenerate(shape, values=values, seed=seed).numpy()
    el = oracle_lib.iso_mesh(f, 0, 0.0)
    got = [tuple(sorted(int(e) for e in row)) for row in el]
    assert len(got) == len(set(got))
    assert set(got) == brute_mesh(f, 0, 0.0)
    rec, _, _ = oracle_lib.iso_track(f, 0, 0.0)
    assert set(np.unique(el).tolist()) <= set(rec["face_id"].tolist())
