"""Pins of the oracle's exact predicates (PAPER.md:465-467 SoS point-in-simplex; Eq. 2 at
PAPER.md:431-436) against computations that do not share its formula:

* SoS sign == sign of det(M + E) evaluated in exact rationals with a concrete small epsilon,
  E[r][j] = eps^(2^(n r + j)) (reading R4), on random small-integer (highly degenerate)
  matrices;
* the face test on generic inputs == "all barycentric coordinates of Eq. 2 lie in (0, 1)", solved
  exactly with Fractions by Gaussian elimination;
* SPEC.md examples for point_in_simplex_sos;
* correctly-rounded int128 -> double (Python's int -> float is correctly rounded).
"""
from fractions import Fraction

import numpy as np
import pytest


def _det(M):
    """exact determinant by fraction-free Bareiss elimination on a copy (rationals)"""
    A = [[Fraction(x) for x in row] for row in M]
    n = len(A)
    sign = 1
    for i in range(n):
        piv = next((k for k in range(i, n) if A[k][i] != 0), None)
        if piv is None:
            return Fraction(0)
        if piv != i:
            A[i], A[piv] = A[piv], A[i]
            sign = -sign
        for k in range(i + 1, n):
            f = A[k][i] / A[i][i]
            A[k] = [x - f * y for x, y in zip(A[k], A[i])]
    p = Fraction(sign)
    for i in range(n):
        p *= A[i][i]
    return p


def _sos_concrete(M, eps_log2=24):
    n = len(M)
    eps = Fraction(1, 1 << eps_log2)
    P = [[Fraction(M[r][j]) + eps ** (1 << (n * r + j)) for j in range(n)] for r in range(n)]
    d = _det(P)
    assert d != 0
    return 1 if d > 0 else -1


@pytest.mark.parametrize("n,trials,lo,hi", [(2, 3000, -2, 2), (2, 500, -50, 50), (3, 300, -2, 2), (3, 100, -9, 9)])
def test_sos_sign_vs_concrete_epsilon(oracle_lib, n, trials, lo, hi):
    rng = np.random.default_rng(n * 1000 + hi)
    for _ in range(trials):
        M = rng.integers(lo, hi + 1, size=(n, n))
        if rng.random() < 0.3:  # force duplicated / zero rows (degenerate cases)
            M[rng.integers(n)] = M[rng.integers(n)] if rng.random() < 0.5 else 0
        assert oracle_lib.sos_sign(M) == _sos_concrete(M.tolist()), M


def test_sos_order_2x2_matches_appendix_c(oracle_lib):
    """SURVEY.md Appendix C 2x2 chain (rows a<b, columns u, v): det, +v_b, -u_b, -v_a, -1.
    The oracle's epsilon-order starts with exactly these monomials."""
    order = oracle_lib.sos_order(2).tolist()
    # monomials as (col of row 0, col of row 1); -1 = row unperturbed
    assert order[:5] == [[-1, -1], [0, -1], [1, -1], [-1, 0], [1, 0]]


def _bary(G):
    """Eq. 2: solve [g_0..g_n; 1..1] mu = [0..0, 1] exactly; None if singular"""
    n = len(G) - 1
    M = [[Fraction(G[j][a]) for j in range(n + 1)] for a in range(n)] + [[Fraction(1)] * (n + 1)]
    if _det(M) == 0:
        return None
    rhs = [Fraction(0)] * n + [Fraction(1)]
    A = [row[:] + [r] for row, r in zip(M, rhs)]
    m = n + 1
    for i in range(m):
        piv = next(k for k in range(i, m) if A[k][i] != 0)
        A[i], A[piv] = A[piv], A[i]
        for k in range(m):
            if k != i and A[k][i] != 0:
                f = A[k][i] / A[i][i]
                A[k] = [x - f * y for x, y in zip(A[k], A[i])]
    return [A[i][m] / A[i][i] for i in range(m)]


@pytest.mark.parametrize("n", [2, 3])
def test_face_test_generic_vs_barycentric(oracle_lib, n):
    rng = np.random.default_rng(7 + n)
    hits = 0
    for _ in range(1500 if n == 2 else 800):
        G = rng.integers(-10**6, 10**6, size=(n + 1, n))
        mu = _bary(G.tolist())
        if mu is None or any(m == 0 for m in mu):
            continue  # not generic: covered by the SoS tests
        expect = all(0 < m < 1 for m in mu)
        hits += expect
        assert oracle_lib.punctured(G) == expect
    assert hits > 50


def test_spec_examples(oracle_lib):
    assert oracle_lib.punctured([[2, 0], [0, 2], [-2, -2]]) is True
    assert oracle_lib.punctured([[1, 1], [2, 1], [1, 2]]) is False


def test_exactly_once_around_degenerate_vertex(oracle_lib):
    """A zero exactly at a shared vertex / edge is claimed by exactly one triangle of a fan
    (PAPER.md:124-125, 467).  Planar affine fields g(x) = A (x - c) on the 2D Kuhn triangulation
    of a 4x4 patch, with c on vertices and edge midpoints."""
    # triangles of the 2D Kuhn triangulation (two per square), vertices sorted by row-major id
    tris = []
    for y in range(3):
        for x in range(3):
            v00, v10, v01, v11 = (x, y), (x + 1, y), (x, y + 1), (x + 1, y + 1)
            tris.append((v00, v10, v11))
            tris.append((v00, v01, v11))
    rng = np.random.default_rng(3)
    for c in [(1, 1), (2, 1), (1, 2), (Fraction(3, 2), 1), (1, Fraction(3, 2)), (Fraction(3, 2), Fraction(3, 2))]:
        for _ in range(20):
            A = rng.integers(-5, 6, size=(2, 2))
            if round(np.linalg.det(A)) == 0:
                continue
            def g(v):
                dx, dy = Fraction(v[0]) - c[0], Fraction(v[1]) - c[1]
                return [int(2 * (A[0, 0] * dx + A[0, 1] * dy)), int(2 * (A[1, 0] * dx + A[1, 1] * dy))]
            count = 0
            for tri in tris:
                tri = sorted(tri, key=lambda v: (v[1], v[0]))
                count += oracle_lib.punctured([g(v) for v in tri])
            assert count == 1, (c, A)


def test_cvt_correctly_rounded(oracle_lib):
    rng = np.random.default_rng(5)
    vals = [0, 1, -1, 2**53 + 1, -(2**53 + 1), 2**64 - 1, -(2**64) + 1, 2**100 + 2**47, -(2**100 + 2**47),
            2**126 - 1, -(2**126)]
    for _ in range(2000):
        bits = int(rng.integers(1, 127))
        v = int(rng.integers(0, 2**62)) << max(0, bits - 62) | int(rng.integers(0, 2**20))
        v = v % (1 << 126)
        vals.append(v if rng.random() < 0.5 else -v)
    for v in vals:
        assert oracle_lib.cvt(v) == float(v), v
