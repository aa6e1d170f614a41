"""Brute-force pin of the oracle's whole tracking result on tiny grids (SURVEY.md 8(c) "Tiny brute
force").  An independent pure-Python checker -- exact rationals, no code shared with `oracle/` -- that
follows the definitions rather than the oracle's algorithm:

* simplices of the Kuhn mesh are found by brute force as vertex chains
  v0 < v1 < ... with nested, strictly growing offset masks (v_k - v0 in {0,1}^d), not from a table;
  face types are numbered by sorting their mask tuples (R2);
* the SoS sign (R4) is the sign of det(M + E) evaluated EXACTLY with a
  concrete, tiny epsilon, E[r][j] = eps^(2^(n r + j)) -- not by the oracle's enumeration of
  epsilon-monomials;
* a face is punctured iff the n + 1 signs (-1)^(k+n) sos(rows != k) agree (R5);
* cells are the full-span chains; each must hold 0 or 2 punctured faces, pairs are
  joined, labels are the minimum face id of a component (R13);
* locations are Eq. 2 in exact rationals; 2D types come from the exact sign of the
  determinant of the mu-interpolated Hessian (R8/R9), compared where it is not a near tie;
  3D types count the negative eigenvalues of the exact rational Hessian by Jacobi's rule on its
  leading principal minors (Sylvester's law of inertia), not by the oracle's Descartes count.
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import ftk_inputs as fi


def quantize(f, s):
    # round-half-even of f * 2^s, exact (Python's round on an exact Fraction)
    return round(Fraction(float(f)) * Fraction(2) ** s)


def grad_field(q, dims):
    """g_a = q[+a] - q[-a] inside, 2 (q[1] - q[0]) / 2 (q[N-1] - q[N-2]) on the boundary (spatial axes
    only); q is a dict keyed by (x, y[, z], t)."""
    nsp = len(dims) - 1
    g = {}
    for v in q:
        comp = []
        for a in range(nsp):
            n = dims[a]
            def at(k):
                w = list(v)
                w[a] = k
                return q[tuple(w)]
            if v[a] == 0:
                comp.append(2 * (at(1) - at(0)))
            elif v[a] == n - 1:
                comp.append(2 * (at(n - 1) - at(n - 2)))
            else:
                comp.append(at(v[a] + 1) - at(v[a] - 1))
        g[v] = comp
    return g


def det(M):
    n = len(M)
    if n == 1:
        return M[0][0]
    return sum((-1) ** c * M[0][c] * det([row[:c] + row[c + 1:] for row in M[1:]]) for c in range(n))


EPS = Fraction(1, 2 ** 160)


def sos_sign(rows):
    n = len(rows)
    d0 = det([list(r) for r in rows])
    if d0 != 0:
        # integer rows: |det(M)| >= 1, while every epsilon term of det(M + E) is below 2^-60 here
        # (entries < 2^40, epsilon <= 2^-160), so the unperturbed sign is the SoS sign
        assert max(abs(x) for r in rows for x in r) < 2 ** 40
        return 1 if d0 > 0 else -1
    M = [[Fraction(rows[r][j]) + EPS ** (2 ** (n * r + j)) for j in range(n)] for r in range(n)]
    d = det(M)
    assert d != 0
    return 1 if d > 0 else -1


def vid(v, dims):
    i = 0
    for a in reversed(range(len(dims))):
        i = i * dims[a] + v[a]
    return i


def nested_sequences(d, k):
    """strictly nested mask sequences m1 < m2 < ... < mk (subset and not equal), masks in 1..2^d-1"""
    return [seq for seq in itertools.product(range(1, 1 << d), repeat=k)
            if all(seq[i] != seq[i + 1] and (seq[i] & ~seq[i + 1]) == 0 for i in range(k - 1))]


def mesh(dims, k):
    """All k-simplices as vertex chains (brute force over anchors and nested mask sequences)."""
    d = len(dims)
    seqs = nested_sequences(d, k)
    out = []
    for anchor in itertools.product(*[range(n) for n in dims]):
        for seq in seqs:
            verts = [anchor] + [tuple(anchor[a] + ((m >> a) & 1) for a in range(d)) for m in seq]
            if all(all(0 <= w[a] < dims[a] for a in range(d)) for w in verts):
                out.append((anchor, seq, verts))
    return out


def brute_track(field, s):
    """field: numpy [t][(z)][y][x]; returns {face_id: (label, loc, type_or_None, degenerate)}"""
    arr = np.asarray(field)
    dims = tuple(reversed(arr.shape))  # (nx, ny[, nz], nt)
    d = len(dims)
    n = d - 1  # spatial dimension = face dimension
    q = {}
    for idx in itertools.product(*[range(m) for m in arr.shape]):
        q[tuple(reversed(idx))] = quantize(arr[idx], s)
    g = grad_field(q, dims)
    # face types: sort the mask tuples of all nested sequences (R2)
    types = sorted(nested_sequences(d, n))
    assert len(types) == (12 if d == 3 else 60)
    tid = {seq: i for i, seq in enumerate(types)}
    T = len(types)
    punct = {}
    for anchor, seq, verts in mesh(dims, n):
        rows = [g[v] for v in verts]  # chain order = global vertex order
        sig = [(-1) ** (k + n) * sos_sign(rows[:k] + rows[k + 1:]) for k in range(n + 1)]
        if len(set(sig)) == 1:
            punct[vid(anchor, dims) * T + tid[seq]] = (verts, rows)
    # cells: full-span chains; 0 or 2 punctured sides
    parent = {f: f for f in punct}

    def find(a):
        while parent[a] != a:
            a = parent[a]
        return a

    bad = 0
    for anchor, seq, verts in mesh(dims, d):
        if seq[-1] != (1 << d) - 1:
            continue
        sides = []
        for k in range(d + 1):
            fv = verts[:k] + verts[k + 1:]
            a0 = fv[0]
            fseq = tuple(sum(((w[a] - a0[a]) & 1) << a for a in range(d)) for w in fv[1:])
            fid = vid(a0, dims) * T + tid[fseq]
            if fid in punct:
                sides.append(fid)
        if len(sides) not in (0, 2):
            bad += 1
        elif len(sides) == 2:
            ra, rb = find(sides[0]), find(sides[1])
            if ra != rb:
                parent[max(ra, rb)] = min(ra, rb)
    out = {}
    for fid, (verts, rows) in punct.items():
        D = [(-1) ** (k + n) * det([list(map(Fraction, r)) for r in rows[:k] + rows[k + 1:]]) for k in range(n + 1)]
        S = sum(D)
        mu = [Fraction(1, n + 1)] * (n + 1) if S == 0 else [Dk / S for Dk in D]
        loc = [sum(mu[k] * verts[k][a] for k in range(n + 1)) for a in range(d)]
        typ = None
        if n == 2:
            H = []
            for v in verts:  # integer Hessian, centre clamped into [1, N-2] per differentiated axis
                x, y, t = v
                cx, cy = min(max(x, 1), dims[0] - 2), min(max(y, 1), dims[1] - 2)
                hxx = 4 * (q[(cx + 1, y, t)] - 2 * q[(cx, y, t)] + q[(cx - 1, y, t)])
                hyy = 4 * (q[(x, cy + 1, t)] - 2 * q[(x, cy, t)] + q[(x, cy - 1, t)])
                hxy = q[(cx + 1, cy + 1, t)] - q[(cx + 1, cy - 1, t)] - q[(cx - 1, cy + 1, t)] + q[(cx - 1, cy - 1, t)]
                H.append((hxx, hxy, hyy))
            a = sum(mu[k] * H[k][0] for k in range(3))
            b = sum(mu[k] * H[k][1] for k in range(3))
            dd = sum(mu[k] * H[k][2] for k in range(3))
            dt = a * dd - b * b
            scale = a * a + b * b + dd * dd
            if dt != 0 and abs(dt) > Fraction(1, 10 ** 9) * scale:
                typ = 2 if dt < 0 else (1 if a > 0 else 5)
        else:
            typ = type3d(q, dims, verts, mu)
        out[fid] = (find(fid), loc, typ, S == 0)
    return out, bad


def hessian3d(q, dims, v):
    """integer Hessian at v (R8): 4 x the compact second difference on the diagonal, the
    4-point cross difference off it, stencil centre clamped into [1, N-2] per differentiated axis"""
    H = [[0] * 3 for _ in range(3)]
    for a in range(3):
        for b in range(a, 3):
            c = list(v)
            c[a] = min(max(c[a], 1), dims[a] - 2)
            c[b] = min(max(c[b], 1), dims[b] - 2)

            def at(da, db):
                w = list(c)
                w[a] += da
                w[b] += db
                return q[tuple(w)]
            if a == b:
                w = list(c); w[a] += 1; p = q[tuple(w)]
                w[a] -= 2; m = q[tuple(w)]
                H[a][a] = 4 * (p - 2 * q[tuple(c)] + m)
            else:
                H[a][b] = H[b][a] = at(1, 1) - at(1, -1) - at(-1, 1) + at(-1, -1)
    return H


def type3d(q, dims, verts, mu):
    """3D type from the inertia of H_bar = sum mu_k H_k (R9): by Sylvester's law of
    inertia the number of negative eigenvalues is the number of sign changes in (1, D1, D2, D3) of
    the leading principal minors, under any symmetric axis permutation with D1, D2 != 0.  None for a
    near-singular H_bar (the oracle decides those in FP64) or when no permutation has nonzero minors."""
    Hs = [hessian3d(q, dims, v) for v in verts]
    Hb = [[sum(mu[k] * Hs[k][i][j] for k in range(4)) for j in range(3)] for i in range(3)]
    D3 = det(Hb)
    scale = max(abs(x) for r in Hb for x in r)
    if D3 == 0 or abs(D3) <= Fraction(1, 10 ** 9) * scale ** 3:
        return None
    for perm in itertools.permutations(range(3)):
        P = [[Hb[perm[i]][perm[j]] for j in range(3)] for i in range(3)]
        D1, D2 = P[0][0], P[0][0] * P[1][1] - P[0][1] * P[1][0]
        if D1 != 0 and D2 != 0:
            seq = [1, D1, D2, D3]
            neg = sum((seq[i] > 0) != (seq[i + 1] > 0) for i in range(3))
            return {0: 1, 1: 3, 2: 4, 3: 5}[neg]  # MIN, SADDLE1, SADDLE2, MAX (oracle enum)
    return None


def check(oracle_lib, field, s):
    ref, _, info = oracle_lib.track(np.ascontiguousarray(field), s)
    bf, bad = brute_track(field, s)
    assert bad == 0 and info["bad_cells"] == 0
    got = {int(r["face_id"]): r for r in ref}
    assert set(got) == set(bf), (len(got), len(bf))
    names = ("x", "y", "t") if field.ndim == 3 else ("x", "y", "z", "t")
    nt = 0
    for fid, (lab, loc, typ, degen) in bf.items():
        r = got[fid]
        assert int(r["label"]) == lab
        for a, k in enumerate(names):
            assert abs(float(r[k]) - float(loc[a])) <= 1e-12 * max(1.0, abs(float(loc[a])))
        assert bool(r["flags"] & oracle_lib.FL_DEGEN_LOC) == degen
        if typ is not None:
            assert int(r["type"]) == typ
            nt += 1
    return len(bf), nt


@pytest.mark.parametrize("shape,values,seed", [
    ((3, 4, 5), (-1.0, 0.0, 1.0), 0),
    ((3, 4, 5), (-1.0, 0.0, 1.0), 1),
    ((3, 5, 4), (-3.0, -1.0, 0.0, 2.0, 3.0), 2),
    ((4, 3, 3), (-1.0, 1.0), 3),
])
def test_bruteforce_2d_degenerate(oracle_lib, shape, values, seed):
    f = fi.random_degenerate(shape, values=values, seed=seed).numpy()
    n, _ = check(oracle_lib, f, 0)
    assert n > 0


def test_bruteforce_2d_woven(oracle_lib):
    """a C1-like woven window at the C1 scale (s = 26): types compared as well"""
    f = fi.Woven(9, 8, 3, L=15.0).generate().numpy()
    n, nt = check(oracle_lib, f, 26)
    assert n > 0 and nt == n


def test_bruteforce_3d_degenerate(oracle_lib):
    f = fi.random_degenerate((2, 3, 3, 3), seed=5).numpy()
    n, _ = check(oracle_lib, f, 0)
    assert n > 0


@pytest.mark.parametrize("nz,L,sigma", [(4, 4.0, 0.0), (5, 5.0, 0.05)])
def test_bruteforce_3d_woven(oracle_lib, nz, L, sigma):
    """3D woven windows (generic values, s = 26): labels, locations and the 3D Hessian types
    (22 / 26 punctured faces, SADDLE1, SADDLE2 and MAX all present, every type decided)"""
    f = fi.Woven(6, 6, 2, nz=nz, L=L, sigma=sigma).generate().numpy()
    n, nt = check(oracle_lib, f, 26)
    assert n > 0 and nt == n
