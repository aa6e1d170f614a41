"""Pins of the oracle's Kuhn spacetime mesh against the paper's printed
listings (tests/golden/kuhn_listings.txt), the staircase construction of Table 1,
geometry (volumes, point location) and brute-force enumeration on tiny grids."""
import itertools
import math
import os
from fractions import Fraction

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "kuhn_listings.txt")


def _golden():
    blocks, cur = {}, None
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line.startswith("["):
            cur = line[1:line.index("]")]
            blocks[cur] = []
        else:
            blocks[cur].append(line.split())
    return blocks


def _cells_as_vertex_lists(oracle, d):
    """The oracle's cells of the unit d-cube: chains 0 -> e_p0 -> e_p0+e_p1 -> ... (coordinates)."""
    out = []
    for perm in oracle.cell_perms(d):
        v = [0] * d
        chain = [tuple(v)]
        for a in perm:
            v[a] += 1
            chain.append(tuple(v))
        out.append(chain)
    return out


def _digits_to_coords(s, mapping):
    return tuple(int(s[mapping[a]]) for a in range(len(s)))


def test_cube_listings_match_paper(oracle_lib):
    g = _golden()
    for name, d in (("cube2", 2), ("cube3_partial", 3), ("cube4_partial", 4)):
        cells = {frozenset(c) for c in _cells_as_vertex_lists(oracle_lib, d)}
        assert len(cells) == math.factorial(d)  # PAPER.md:303 n! simplices
        ok_any = False
        for mapping in itertools.permutations(range(d)):
            listed = {frozenset(_digits_to_coords(s, mapping) for s in row) for row in g[name]}
            if listed <= cells:
                ok_any = True
                break
        assert ok_any, f"{name}: printed simplices not in the oracle's subdivision"
        if name == "cube2":  # complete listing: equality
            assert any({frozenset(_digits_to_coords(s, m) for s in row) for row in g[name]} == cells
                       for m in itertools.permutations(range(d)))


def test_counts_listing(oracle_lib):
    g = _golden()
    for key, *vals in g["counts"]:
        if key == "cube_simplices":
            d, n = map(int, vals)
            assert len(oracle_lib.cell_perms(d)) == n
        elif key == "edge_types_2d":
            # unique edge types owned by a 2-cube: sub-chains of length 2 of the 2 triangles,
            # translated to their anchor (componentwise minimum)
            types = set()
            for c in _cells_as_vertex_lists(oracle_lib, 2):
                for a, b in itertools.combinations(c, 2):
                    types.add(tuple(y - x for x, y in zip(a, b)))
            assert len(types) == int(vals[0])


def test_staircase_extrusion_table1(oracle_lib):
    """Recursive extrusion: every triangle c0<c1<c2 of the 2-cube, extruded along
    the top axis, splits into Table 1's staircases a0a1a2b2, a0a1b1b2, a0b0b1b2; these are exactly
    the oracle's 3-cube cells, and likewise 3-cube tets -> 4-cube pentachora (Table 1, 4D)."""
    for d in (3, 4):
        lower = _cells_as_vertex_lists(oracle_lib, d - 1)
        got = {frozenset(c) for c in _cells_as_vertex_lists(oracle_lib, d)}
        built = set()
        for c in lower:
            a = [v + (0,) for v in c]
            b = [v + (1,) for v in c]
            for k in range(d):  # staircase k: a0..ak bk..b_{d-1}
                built.add(frozenset(a[: k + 1] + b[k:]))
        assert built == got
    g = _golden()
    assert g["table1"][0] == ["a0a1a2b2", "a0a1b1b2", "a0b0b1b2"]


def test_unit_volume_and_disjointness(oracle_lib):
    rng = np.random.default_rng(1)
    for d in (2, 3, 4):
        cells = _cells_as_vertex_lists(oracle_lib, d)
        for c in cells:  # each simplex has volume 1/d! (unimodular edge matrix)
            E = np.array([np.subtract(c[i + 1], c[0]) for i in range(d)], dtype=float)
            assert abs(abs(np.linalg.det(E)) - 1.0) < 1e-12
        # random interior points lie in exactly one simplex
        for _ in range(200):
            p = [Fraction(int(x), 10007) for x in rng.integers(1, 10006, size=d)]
            inside = 0
            for c in cells:
                # barycentric coordinates by exact solve
                M = [[Fraction(c[j][a]) for j in range(d + 1)] for a in range(d)] + [[Fraction(1)] * (d + 1)]
                rhs = p + [Fraction(1)]
                lam = _solve(M, rhs)
                inside += all(x > 0 for x in lam)
            assert inside == 1


def _solve(M, rhs):
    n = len(M)
    A = [row[:] + [r] for row, r in zip(M, rhs)]
    for i in range(n):
        piv = next(k for k in range(i, n) if A[k][i] != 0)
        A[i], A[piv] = A[piv], A[i]
        for k in range(n):
            if k != i and A[k][i] != 0:
                f = A[k][i] / A[i][i]
                A[k] = [x - f * y for x, y in zip(A[k], A[i])]
    return [A[i][n] / A[i][i] for i in range(n)]


def _types_from_cells(oracle_lib, d, k):
    """unique k-simplex types owned by a cube: k+1-vertex sub-chains of the cells, translated so
    that the anchor (componentwise min = first vertex) is the origin, as cumulative masks"""
    types = set()
    for c in _cells_as_vertex_lists(oracle_lib, d):
        for sub in itertools.combinations(c, k + 1):
            base = sub[0]
            types.add(tuple(sum((v[a] - base[a]) << a for a in range(d)) for v in sub[1:]))
    return types


def test_face_types_are_the_cells_sides(oracle_lib):
    for d, T, n_ord in ((3, 12, 2), (4, 60, 6)):
        ft = oracle_lib.face_types(d)
        assert ft.shape == (T, d - 1)
        assert {tuple(int(x) for x in r) for r in ft} == _types_from_cells(oracle_lib, d, d - 1)
        rows = [tuple(int(x) for x in r) for r in ft]
        assert rows == sorted(rows)  # canonical numbering = lexicographic (R2)
        top = 1 << (d - 1)
        ordinal = [i for i, r in enumerate(rows) if not (r[-1] & top)]
        assert len(ordinal) == n_ord
    # SURVEY.md Appendix B anchors: 2D+t ordinal types {0, 3}; 3D+t type 0 and type 59
    assert [i for i, r in enumerate(oracle_lib.face_types(3)) if not (r[-1] & 4)] == [0, 3]
    ft4 = oracle_lib.face_types(4)
    assert tuple(ft4[0]) == (1, 3, 7) and tuple(ft4[59]) == (12, 14, 15)
    assert [i for i, r in enumerate(ft4) if not (r[-1] & 8)] == [0, 3, 12, 15, 26, 29]


def test_euler_characteristic_per_cube(oracle_lib):
    """sum_k (-1)^k N_k = 0 for the k-simplex types owned by one cube of an infinite lattice."""
    for d, expect in ((3, [1, 7, 12, 6]), (4, [1, 15, 50, 60, 24])):
        counts = [1] + [len(_types_from_cells(oracle_lib, d, k)) for k in range(1, d + 1)]
        assert counts == expect
        assert sum((-1) ** k * c for k, c in enumerate(counts)) == 0


def _brute_face_count(ext):
    """all sides of all cells of the grid, as vertex sets (every face of the grid is a side of at
    least one cell when all extents >= 2)"""
    d = len(ext)
    faces = set()
    for anchor in itertools.product(*[range(e - 1) for e in ext]):
        for perm in itertools.permutations(range(d)):
            v = list(anchor)
            chain = [tuple(v)]
            for a in perm:
                v[a] += 1
                chain.append(tuple(v))
            for j in range(d + 1):
                faces.add(tuple(chain[:j] + chain[j + 1:]))
    return len(faces)


@pytest.mark.parametrize("ext", [(3, 4, 3), (4, 3, 3), (5, 3, 2), (3, 3, 3, 3), (4, 3, 3, 2)])
def test_face_count_brute_force(oracle_lib, ext):
    import torch
    shape = tuple(reversed(ext))  # [t][(z)][y][x]
    field = np.random.default_rng(0).standard_normal(shape).astype(np.float32)
    _, nf = oracle_lib.extract(field, 10)
    assert nf == _brute_face_count(ext)
