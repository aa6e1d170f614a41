"""ctypes wrapper of the CPU oracle (oracle/ftk_oracle.c).

TEST INFRASTRUCTURE: only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
(``paper_2011_08697_b200``) never imports it, and this package never imports the product.

See ftk_oracle.c's header for the step-by-step algorithm and its PAPER.md citations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ftk_oracle.c")
_LIB = os.path.join(_HERE, "libftk_oracle.so")

OK, INVALID_ARG, RANGE, CAPACITY, INVARIANT, NOMEM = 0, 1, 2, 3, 6, 7
DEGENERATE, MIN, SADDLE, SADDLE1, SADDLE2, MAX, SOURCE, SINK, CENTER = 0, 1, 2, 3, 4, 5, 6, 7, 8
FL_ORDINAL, FL_BOUNDARY, FL_DEGEN_LOC = 1, 2, 4

CP_DTYPE = np.dtype(
    [("face_id", "<i8"), ("label", "<i8"), ("x", "<f8"), ("y", "<f8"), ("z", "<f8"),
     ("t", "<f8"), ("type", "<i4"), ("flags", "<i4")]
)
assert CP_DTYPE.itemsize == 56


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"oracle {what} failed with status {status}")
        self.status = status


class _Desc(ctypes.Structure):
    _fields_ = [
        ("ndim", ctypes.c_int32), ("dtype", ctypes.c_int32), ("n", ctypes.c_int64 * 3),
        ("nt", ctypes.c_int64), ("t0", ctypes.c_int64), ("nt_global", ctypes.c_int64),
        ("scale_log2", ctypes.c_int32), ("nthreads", ctypes.c_int32),
        ("kind", ctypes.c_int32), ("pad_", ctypes.c_int32),
    ]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C11, OpenMP, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-std=gnu11", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
             "-fno-fast-math", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        P = ctypes.c_void_p
        L.ftko_face_types.argtypes = [ctypes.c_int, P]
        L.ftko_cell_perms.argtypes = [ctypes.c_int, P]
        L.ftko_sos_sign.argtypes = [ctypes.c_int, P]
        L.ftko_sos_order.argtypes = [ctypes.c_int, P]
        L.ftko_punctured.argtypes = [ctypes.c_int, P]
        L.ftko_cvt.argtypes = [ctypes.c_int64, ctypes.c_uint64]
        L.ftko_cvt.restype = ctypes.c_double
        L.ftko_extract.argtypes = [ctypes.POINTER(_Desc), P, ctypes.c_int64, ctypes.c_int64, P,
                                   ctypes.c_int64, P, P]
        L.ftko_track.argtypes = [ctypes.POINTER(_Desc), P, P, ctypes.c_int64, P, P, P]
        L.ftko_iso_track.argtypes = [ctypes.POINTER(_Desc), P, ctypes.c_double, P, ctypes.c_int64, P, P, P]
        L.ftko_iso_mesh.argtypes = [ctypes.POINTER(_Desc), P, ctypes.c_double, P, ctypes.c_int64, P]
    return _lib


def face_types(d: int) -> np.ndarray:
    """Canonical face types of the d-dimensional Kuhn cube: array [T, d-1] of cumulative masks."""
    T = lib().ftko_face_types(d, None)
    out = np.zeros((T, d - 1), np.int32)
    lib().ftko_face_types(d, out.ctypes.data)
    return out


def cell_perms(d: int) -> np.ndarray:
    P = lib().ftko_cell_perms(d, None)
    out = np.zeros((P, d), np.int32)
    lib().ftko_cell_perms(d, out.ctypes.data)
    return out


def sos_sign(M) -> int:
    M = np.ascontiguousarray(np.asarray(M, dtype=np.int64))
    n = M.shape[0]
    return lib().ftko_sos_sign(n, M.ctypes.data)


def sos_order(n: int) -> np.ndarray:
    out = np.zeros((64, n), np.int32)
    k = lib().ftko_sos_order(n, out.ctypes.data)
    return out[:k]


def punctured(G) -> bool:
    G = np.ascontiguousarray(np.asarray(G, dtype=np.int64))
    n = G.shape[1]
    return bool(lib().ftko_punctured(n, G.ctypes.data))


def cvt(v: int) -> float:
    lo = v & ((1 << 64) - 1)
    hi = (v - lo) >> 64
    return lib().ftko_cvt(hi, lo)


def _desc(field: np.ndarray, scale_log2: int, t0: int, nt_global: int | None, nthreads: int,
          vector: bool = False):
    """vector=True: a vector field [t][y][x][2] (2D) or [t][z][y][x][3] (3D), components interleaved,
    tracked as given."""
    if field.dtype not in (np.float32, np.float64):
        raise TypeError("field must be float32 or float64")
    field = np.ascontiguousarray(field)
    if vector:
        if field.ndim == 4 and field.shape[3] == 2:
            nt, ny, nx, _ = field.shape
            nz, ndim = 1, 2
        elif field.ndim == 5 and field.shape[4] == 3:
            nt, nz, ny, nx, _ = field.shape
            ndim = 3
        else:
            raise ValueError("vector field must be [t][y][x][2] or [t][z][y][x][3]")
    elif field.ndim == 3:
        nt, ny, nx = field.shape
        nz, ndim = 1, 2
    elif field.ndim == 4:
        nt, nz, ny, nx = field.shape
        ndim = 3
    else:
        raise ValueError("field must be [t][y][x] or [t][z][y][x]")
    d = _Desc()
    d.ndim = ndim
    d.dtype = 0 if field.dtype == np.float32 else 1
    d.n[0], d.n[1], d.n[2] = nx, ny, nz
    d.nt = nt
    d.t0 = t0
    d.nt_global = nt_global if nt_global is not None else t0 + nt
    d.scale_log2 = scale_log2
    d.nthreads = nthreads
    d.kind = 1 if vector else 0
    return d, field


def extract(field: np.ndarray, scale_log2: int, t0: int = 0, nt_global: int | None = None,
            ta: int | None = None, tb: int | None = None, nthreads: int = 0, vector: bool = False):
    """Pass 1 over anchors with global t in [ta, tb). Returns (records sorted by face_id, n_faces)."""
    d, field = _desc(field, scale_log2, t0, nt_global, nthreads, vector)
    ta = t0 if ta is None else ta
    tb = min(t0 + d.nt, d.nt_global) if tb is None else tb
    n_out = ctypes.c_int64(0)
    n_faces = ctypes.c_int64(0)
    st = lib().ftko_extract(ctypes.byref(d), field.ctypes.data, ta, tb, None, 0,
                            ctypes.byref(n_out), ctypes.byref(n_faces))
    if st not in (OK, CAPACITY):
        raise OracleError(st, "extract")
    out = np.zeros(max(n_out.value, 1), CP_DTYPE)
    st = lib().ftko_extract(ctypes.byref(d), field.ctypes.data, ta, tb, out.ctypes.data,
                            n_out.value, ctypes.byref(n_out), ctypes.byref(n_faces))
    if st != OK:
        raise OracleError(st, "extract")
    return out[: n_out.value], n_faces.value


def track(field: np.ndarray, scale_log2: int, nthreads: int = 0, check: bool = True, vector: bool = False):
    """Full two-pass tracking. Returns (records sorted by face_id with labels, n_faces, stats)."""
    d, field = _desc(field, scale_log2, 0, None, nthreads, vector)
    n_out = ctypes.c_int64(0)
    n_faces = ctypes.c_int64(0)
    stats = np.zeros(4, np.int64)
    cap = 1 << 16
    while True:
        out = np.zeros(cap, CP_DTYPE)
        st = lib().ftko_track(ctypes.byref(d), field.ctypes.data, out.ctypes.data, cap,
                              ctypes.byref(n_out), ctypes.byref(n_faces), stats.ctypes.data)
        if n_out.value > cap:
            cap = n_out.value
            continue
        break
    if st != OK and (check or st != INVARIANT):
        raise OracleError(st, "track")
    info = dict(cells=int(stats[0]), bad_cells=int(stats[1]), components=int(stats[2]),
                pairs=int(stats[3]), status=st)
    return out[: n_out.value], n_faces.value, info


def iso_track(field: np.ndarray, scale_log2: int, isovalue: float, nthreads: int = 0, check: bool = True):
    """Isovolume tracking: crossed spacetime edges of f = isovalue with Eq. 2
    locations and component labels (min edge id).  Returns (records sorted by edge id, n_edges, stats)."""
    d, field = _desc(field, scale_log2, 0, None, nthreads)
    n_out = ctypes.c_int64(0)
    n_edges = ctypes.c_int64(0)
    stats = np.zeros(4, np.int64)
    cap = 1 << 16
    while True:
        out = np.zeros(cap, CP_DTYPE)
        st = lib().ftko_iso_track(ctypes.byref(d), field.ctypes.data, ctypes.c_double(isovalue), out.ctypes.data, cap,
                                  ctypes.byref(n_out), ctypes.byref(n_edges), stats.ctypes.data)
        if st == CAPACITY:
            cap = n_out.value
            continue
        break
    if st != OK and (check or st != INVARIANT):
        raise OracleError(st, "iso_track")
    info = dict(cells=int(stats[0]), bad_cells=int(stats[1]), components=int(stats[2]), status=st)
    return out[: n_out.value], n_edges.value, info


def iso_mesh(field: np.ndarray, scale_log2: int, isovalue: float, nthreads: int = 0) -> np.ndarray:
    """The isovolume's simplices: int64 [n_elems, n + 1] edge ids (triangles in
    2D+t, tetrahedra in 3D+t), one per staircase path of every cell the level set crosses."""
    d, field = _desc(field, scale_log2, 0, None, nthreads)
    dim = d.ndim + 1
    n_out = ctypes.c_int64(0)
    st = lib().ftko_iso_mesh(ctypes.byref(d), field.ctypes.data, ctypes.c_double(isovalue), None, 0,
                             ctypes.byref(n_out))
    if st not in (OK, CAPACITY):
        raise OracleError(st, "iso_mesh")
    out = np.zeros((max(n_out.value, 1), dim), np.int64)
    st = lib().ftko_iso_mesh(ctypes.byref(d), field.ctypes.data, ctypes.c_double(isovalue), out.ctypes.data,
                             n_out.value, ctypes.byref(n_out))
    if st != OK:
        raise OracleError(st, "iso_mesh")
    return out[: n_out.value]
