"""B200-native FTK critical-point tracking: thin Python binding of the C-ABI (include/ftk_cp.h).

Argument marshalling only -- every step of the path runs in the CUDA kernels of libftk_cp.so.
PyTorch provides device memory and the current stream.  There is no CPU fallback: if the library
is missing or no GPU is present, calls raise.

    import paper_2011_08697_b200 as ftk
    rec = ftk.track(field_cuda, scale_log2=26)      # torch.int64 [n, 7] on the device
    arr = ftk.to_numpy(rec)                         # structured numpy view (face_id, label, x..t, type, flags)
"""
from __future__ import annotations

import collections
import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FTK_LIB") or os.path.join(_HERE, "libftk_cp.so")

OK, ERR_INVALID_ARG, ERR_RANGE, ERR_CAPACITY, ERR_CUDA, ERR_NCCL, ERR_INVARIANT, ERR_NOMEM = range(8)
F32, F64 = 0, 1
DEGENERATE, MIN, SADDLE, SADDLE1, SADDLE2, MAX, SOURCE, SINK, CENTER = range(9)
GHOST_PLANE, SORTED, VECTOR_FIELD = 1, 2, 4
DEBUG_FORCE_GENERIC, DEBUG_VERIFY_LINK, DEBUG_STITCH_HOST, DEBUG_NO_GRAPH, DEBUG_UF_BY_ID = 1, 2, 4, 8, 16
CP_ORDINAL, CP_BOUNDARY, CP_DEGENERATE_LOC = 1, 2, 4

RECORD_DTYPE = np.dtype(
    [("face_id", "<i8"), ("label", "<i8"), ("x", "<f8"), ("y", "<f8"), ("z", "<f8"), ("t", "<f8"),
     ("type", "<i4"), ("flags", "<u4")]
)
RECORD_BYTES = 56
assert RECORD_DTYPE.itemsize == RECORD_BYTES

EXPORTS = [
    "ftk_abi_version", "ftk_strerror", "ftk_last_error", "ftk_num_faces", "ftk_workspace_size",
    "ftk_cp_extract", "ftk_cp_track", "ftk_cp_track_host", "ftk_set_profiling", "ftk_last_timings",
    "ftk_last_kernel_timings",
    "ftk_comm_get_unique_id", "ftk_comm_init", "ftk_comm_reserve", "ftk_comm_destroy", "ftk_stitch_export",
    "ftk_stitch_resolve", "ftk_set_debug",
    "ftk_relabel", "ftk_seam_pack", "ftk_seam_resolve",
    "ftk_tracker_workspace_size", "ftk_tracker_begin", "ftk_tracker_push", "ftk_tracker_finish", "ftk_tracker_abort",
    "ftk_post_adjacency", "ftk_post_slice", "ftk_post_filter", "ftk_post_smooth_types", "ftk_post_simplify_types", "ftk_iso_track",
    "ftk_iso_track_mesh",
]


class FtkError(RuntimeError):
    def __init__(self, status: int, what: str, detail: str = ""):
        msg = f"{what}: status {status}"
        if _lib is not None:
            msg += f" ({_lib.ftk_strerror(status).decode()})"
        if detail:
            msg += f": {detail}"
        super().__init__(msg)
        self.status = status


class Desc(ctypes.Structure):
    _fields_ = [
        ("ndim", ctypes.c_int32), ("dtype", ctypes.c_int32), ("n", ctypes.c_int64 * 3),
        ("nt", ctypes.c_int64), ("t0", ctypes.c_int64), ("nt_global", ctypes.c_int64),
        ("scale_log2", ctypes.c_int32), ("flags", ctypes.c_uint32),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libftk_cp.so (built by __graft_entry__.build() / paper_2011_08697_b200/build.py)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FtkError(-1, f"{LIB_PATH} is missing; run python paper_2011_08697_b200/build.py")
        L = ctypes.CDLL(LIB_PATH)
        P, I64, PD = ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(Desc)
        L.ftk_strerror.restype = ctypes.c_char_p
        L.ftk_strerror.argtypes = [ctypes.c_int]
        L.ftk_last_error.restype = ctypes.c_char_p
        L.ftk_num_faces.argtypes = [PD, P]
        L.ftk_workspace_size.argtypes = [PD, I64, P]
        L.ftk_cp_extract.argtypes = [PD, P, P, I64, P, P, ctypes.c_size_t, P]
        L.ftk_cp_track.argtypes = [PD, P, P, I64, P, P, ctypes.c_size_t, P, P]
        L.ftk_cp_track_host.argtypes = [PD, P, P, P, P, I64, P, P, ctypes.c_size_t, P]
        L.ftk_set_profiling.argtypes = [ctypes.c_int]
        L.ftk_last_timings.argtypes = [P, P]
        L.ftk_last_kernel_timings.argtypes = [P, ctypes.c_int]
        L.ftk_seam_pack.argtypes = [P, P, ctypes.c_size_t, ctypes.c_int64, P, ctypes.c_int64, P]
        L.ftk_seam_resolve.argtypes = [P, ctypes.c_int, ctypes.c_int64, P, ctypes.c_int64, P]
        L.ftk_comm_get_unique_id.argtypes = [P]
        L.ftk_comm_init.argtypes = [P, ctypes.c_int, ctypes.c_int, P]
        L.ftk_comm_reserve.argtypes = [P, I64]
        L.ftk_set_debug.argtypes = [ctypes.c_uint32]
        L.ftk_comm_destroy.argtypes = [P]
        L.ftk_stitch_export.argtypes = [PD, P, ctypes.c_size_t, I64, P, I64, P, P, I64, P, P]
        L.ftk_stitch_resolve.argtypes = [P, I64, P, I64, P, I64, P, P, P]
        L.ftk_relabel.argtypes = [P, I64, P, P, I64, P, ctypes.c_size_t, I64, P]
        L.ftk_tracker_workspace_size.argtypes = [PD, I64, ctypes.c_int32, P]
        L.ftk_tracker_begin.argtypes = [P, PD, ctypes.c_int32, P, I64, P, ctypes.c_size_t, P]
        L.ftk_tracker_push.argtypes = [P, P]
        L.ftk_tracker_finish.argtypes = [P, P]
        L.ftk_tracker_abort.argtypes = [P]
        SZ = ctypes.c_size_t
        L.ftk_post_adjacency.argtypes = [PD, P, I64, P, P, SZ, I64, P]
        L.ftk_post_slice.argtypes = [PD, P, P, I64, ctypes.c_double, P, I64, P, P, SZ, I64, P]
        L.ftk_post_filter.argtypes = [PD, P, P, I64, ctypes.c_double, ctypes.c_int32, P, I64, P, P, SZ, I64, P]
        L.ftk_post_smooth_types.argtypes = [PD, P, P, I64, ctypes.c_int32, P, SZ, I64, P]
        L.ftk_post_simplify_types.argtypes = [PD, P, P, I64, ctypes.c_double, P, SZ, I64, P]
        L.ftk_iso_track.argtypes = [PD, ctypes.c_double, P, P, I64, P, P, SZ, P]
        L.ftk_iso_track_mesh.argtypes = [PD, ctypes.c_double, P, P, I64, P, P, I64, P, P, SZ, P]
        _lib = L
    return _lib


def make_desc(shape, dtype, scale_log2: int, t0: int = 0, nt_global: int | None = None,
              ghost: bool = False, sorted_output: bool = False, vector: bool = False) -> Desc:
    """shape: [t][y][x] (2D scalar), [t][z][y][x] (3D scalar) or, with vector=True, [t][y][x][2] /
    [t][z][y][x][3] (2D / 3D vector field, components interleaved; FTK_VECTOR_FIELD)."""
    d = Desc()
    if vector:
        if len(shape) == 4 and shape[3] == 2:
            nt, ny, nx, _ = shape
            nz, d.ndim = 1, 2
        elif len(shape) == 5 and shape[4] == 3:
            nt, nz, ny, nx, _ = shape
            d.ndim = 3
        else:
            raise ValueError("vector field must be [t][y][x][2] or [t][z][y][x][3]")
    elif len(shape) == 3:
        nt, ny, nx = shape
        nz, d.ndim = 1, 2
    elif len(shape) == 4:
        nt, nz, ny, nx = shape
        d.ndim = 3
    else:
        raise ValueError("field must be [t][y][x] or [t][z][y][x]")
    if dtype in (torch.float32, np.float32):
        d.dtype = F32
    elif dtype in (torch.float64, np.float64):
        d.dtype = F64
    else:
        raise TypeError(f"unsupported field dtype {dtype}")
    d.n[0], d.n[1], d.n[2] = nx, ny, nz
    d.nt, d.t0 = nt, t0
    d.nt_global = t0 + nt if nt_global is None else nt_global
    d.scale_log2 = scale_log2
    d.flags = (GHOST_PLANE if ghost else 0) | (SORTED if sorted_output else 0) | (VECTOR_FIELD if vector else 0)
    return d


def num_faces(desc: Desc) -> int:
    n = ctypes.c_int64(0)
    _check(lib().ftk_num_faces(ctypes.byref(desc), ctypes.byref(n)), "ftk_num_faces")
    return n.value


def workspace_size(desc: Desc, capacity: int) -> int:
    b = ctypes.c_size_t(0)
    _check(lib().ftk_workspace_size(ctypes.byref(desc), capacity, ctypes.byref(b)), "ftk_workspace_size")
    return b.value


def _check(status: int, what: str):
    if status != OK:
        raise FtkError(status, what, lib().ftk_last_error().decode())


MAX_CAPACITY = (1 << 31) - 2  # int32 record slots (include/ftk_cp.h)


def default_capacity(field: torch.Tensor) -> int:
    return min(MAX_CAPACITY, max(1 << 16, field.numel() // 64))


@dataclass
class Buffers:
    """Caller-owned device buffers (records + workspace), reusable across calls."""
    records: torch.Tensor     # uint8 [capacity * 56]
    workspace: torch.Tensor   # uint8
    capacity: int

    @staticmethod
    def allocate(desc: Desc, capacity: int, device) -> "Buffers":
        ws = workspace_size(desc, capacity)
        return Buffers(torch.empty(max(capacity, 1) * RECORD_BYTES, dtype=torch.uint8, device=device),
                       torch.empty(ws, dtype=torch.uint8, device=device), capacity)


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _run(fn_name: str, field: torch.Tensor, scale_log2: int, t0: int, nt_global, capacity, ghost,
         buffers: Buffers | None, comm=None, sorted_output=False, vector=False):
    if not field.is_cuda:
        raise FtkError(ERR_INVALID_ARG, f"{fn_name}: field must be a CUDA tensor (no CPU fallback)")
    if not field.is_contiguous():
        field = field.contiguous()
    desc = make_desc(tuple(field.shape), field.dtype, scale_log2, t0, nt_global, ghost, sorted_output, vector)
    cap = capacity if capacity is not None else (buffers.capacity if buffers else default_capacity(field))
    while True:
        if buffers is None or buffers.capacity < cap:
            buffers = Buffers.allocate(desc, cap, field.device)
        n_out = ctypes.c_int64(0)
        args = [ctypes.byref(desc), ctypes.c_void_p(field.data_ptr()), ctypes.c_void_p(buffers.records.data_ptr()),
                buffers.capacity, ctypes.byref(n_out), ctypes.c_void_p(buffers.workspace.data_ptr()),
                buffers.workspace.numel(), ctypes.c_void_p(_stream_ptr(field.device))]
        if fn_name == "ftk_cp_track":
            args.append(comm)
        st = getattr(lib(), fn_name)(*args)
        if st == ERR_CAPACITY:
            if cap >= MAX_CAPACITY:
                _check(st, fn_name)
            cap = min(MAX_CAPACITY, int(n_out.value * 1.25) + 1024)
            buffers = None
            continue
        _check(st, fn_name)
        rec = buffers.records[: n_out.value * RECORD_BYTES].view(torch.int64).view(-1, 7)
        return rec, buffers


def iso_track(field: torch.Tensor, scale_log2: int, isovalue: float, capacity: int | None = None,
              buffers: Buffers | None = None, return_buffers: bool = False, mesh: bool = False):
    """Isovolume tracking: the crossed spacetime edges of f = isovalue as 56-byte
    records (face_id = edge id, Eq. 2 location, type 1 = upward crossing, label = min edge id of the
    connected isovolume piece).  field: [t][y][x] or [t][z][y][x] on the device, the whole domain.
    mesh=True also returns the isovolume's simplices (ftk_iso_track_mesh: triangles in 2D+t, tetrahedra in
    3D+t) as an int64 [n, ndim + 1] device tensor of edge ids: (rec, elems[, buffers])."""
    if not field.is_cuda:
        raise FtkError(ERR_INVALID_ARG, "iso_track: field must be a CUDA tensor (no CPU fallback)")
    field = field.contiguous()
    desc = make_desc(tuple(field.shape), field.dtype, scale_log2)
    cap = capacity if capacity is not None else (buffers.capacity if buffers else default_capacity(field))
    ecap = 4 * cap
    elems = None
    while True:
        if buffers is None or buffers.capacity < cap:
            buffers = Buffers.allocate(desc, cap, field.device)
        n_out = ctypes.c_int64(0)
        n_el = ctypes.c_int64(0)
        common = (ctypes.byref(desc), ctypes.c_double(isovalue), ctypes.c_void_p(field.data_ptr()),
                  ctypes.c_void_p(buffers.records.data_ptr()), buffers.capacity, ctypes.byref(n_out))
        tail = (ctypes.c_void_p(buffers.workspace.data_ptr()), buffers.workspace.numel(),
                ctypes.c_void_p(_stream_ptr(field.device)))
        if mesh:
            if elems is None or elems.shape[0] < ecap:
                elems = torch.empty((max(ecap, 1), desc.ndim + 1), dtype=torch.int64, device=field.device)
            st = lib().ftk_iso_track_mesh(*common, ctypes.c_void_p(elems.data_ptr()), elems.shape[0],
                                          ctypes.byref(n_el), *tail)
        else:
            st = lib().ftk_iso_track(*common, *tail)
        if st == ERR_CAPACITY and cap < MAX_CAPACITY:
            if n_out.value > buffers.capacity:
                cap = min(MAX_CAPACITY, int(n_out.value * 1.25) + 1024)
                buffers = None
            if mesh and n_el.value > elems.shape[0]:
                ecap = n_el.value
            continue
        _check(st, "ftk_iso_track")
        rec = buffers.records[: n_out.value * RECORD_BYTES].view(torch.int64).view(-1, 7)
        out = (rec, elems[: n_el.value]) if mesh else (rec,)
        out = out + (buffers,) if return_buffers else out
        return out if len(out) > 1 else out[0]


def extract(field: torch.Tensor, scale_log2: int, t0: int = 0, nt_global: int | None = None,
            capacity: int | None = None, ghost: bool = False, buffers: Buffers | None = None,
            return_buffers: bool = False, vector: bool = False, sorted_output: bool = False):
    """Pass 1: punctured faces of the buffer's owned timesteps (label = -1).
    Returns an int64 [n, 7] device tensor of 56-byte records (see RECORD_DTYPE); in face-id order with
    sorted_output=True (FTK_SORTED), else in an unspecified order."""
    rec, buf = _run("ftk_cp_extract", field, scale_log2, t0, nt_global, capacity, ghost, buffers, vector=vector,
                    sorted_output=sorted_output)
    return (rec, buf) if return_buffers else rec


def track(field: torch.Tensor, scale_log2: int, t0: int = 0, nt_global: int | None = None,
          capacity: int | None = None, ghost: bool = False, buffers: Buffers | None = None,
          comm=None, return_buffers: bool = False, vector: bool = False, sorted_output: bool = False):
    """Pass 1 + pass 2: punctured faces labelled with their trajectory (min face_id).  vector=True:
    field is a vector field [t][y][x][2] / [t][z][y][x][3] whose own zeros are tracked.
    sorted_output=True: records in face-id order (FTK_SORTED)."""
    rec, buf = _run("ftk_cp_track", field, scale_log2, t0, nt_global, capacity, ghost, buffers, comm, vector=vector,
                    sorted_output=sorted_output)
    return (rec, buf) if return_buffers else rec


def track_host(field_host: torch.Tensor, scale_log2: int, stage: torch.Tensor, buffers: Buffers,
               out_host: torch.Tensor, vector: bool = False):
    """End-to-end from host memory (pinned for speed): H2D inside the call, records copied back to
    out_host (uint8 [capacity * 56], pinned).  Returns the record count."""
    desc = make_desc(tuple(field_host.shape), field_host.dtype, scale_log2, vector=vector)
    n_out = ctypes.c_int64(0)
    st = lib().ftk_cp_track_host(
        ctypes.byref(desc), ctypes.c_void_p(field_host.data_ptr()), ctypes.c_void_p(stage.data_ptr()),
        ctypes.c_void_p(buffers.records.data_ptr()), ctypes.c_void_p(out_host.data_ptr()), buffers.capacity,
        ctypes.byref(n_out), ctypes.c_void_p(buffers.workspace.data_ptr()), buffers.workspace.numel(),
        ctypes.c_void_p(_stream_ptr(stage.device)))
    _check(st, "ftk_cp_track_host")
    return n_out.value


class Tracker:
    """Streaming ingestion (PAPER.md:709 push_field_data; include/ftk_cp.h ftk_tracker_*): push the
    timesteps one at a time (host or device tensors of shape [y][x] or [z][y][x]), then finish() runs
    the rest of pass 1 and pass 2 and returns the labelled records -- identical to track() over the
    whole field, with only window + 1 planes resident on the device.  `capacity` bounds the records
    of the whole stream (FtkError with FTK_ERR_CAPACITY otherwise)."""

    def __init__(self, spatial_shape, dtype, scale_log2: int, capacity: int, window: int = 64, device="cuda",
                 records: torch.Tensor | None = None, workspace: torch.Tensor | None = None, vector: bool = False):
        self.device = torch.device(device)
        self.desc = make_desc((2, *spatial_shape), dtype, scale_log2, vector=vector)
        self.capacity = int(capacity)
        need = self.workspace_bytes(spatial_shape, dtype, scale_log2, capacity, window, vector)
        # caller-owned buffers may be passed in (reused across streams), else allocated here
        if records is None or records.numel() < max(self.capacity, 1) * RECORD_BYTES:
            records = torch.empty(max(self.capacity, 1) * RECORD_BYTES, dtype=torch.uint8, device=self.device)
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, dtype=torch.uint8, device=self.device)
        self.records, self.workspace = records, workspace
        self.dtype = torch.float32 if self.desc.dtype == F32 else torch.float64
        self.spatial_shape = tuple(spatial_shape)
        self._h = ctypes.c_void_p(0)
        self._keep = collections.deque()  # (host plane, event after its copy): copies may be in flight
        self._window = window
        # every copy and kernel of the stream runs on the stream current at construction
        self.stream = torch.cuda.current_stream(self.device)
        _check(lib().ftk_tracker_begin(ctypes.byref(self._h), ctypes.byref(self.desc), window,
                                       ctypes.c_void_p(self.records.data_ptr()), self.capacity,
                                       ctypes.c_void_p(self.workspace.data_ptr()), self.workspace.numel(),
                                       ctypes.c_void_p(self.stream.cuda_stream)), "ftk_tracker_begin")

    @staticmethod
    def workspace_bytes(spatial_shape, dtype, scale_log2: int, capacity: int, window: int,
                        vector: bool = False) -> int:
        desc = make_desc((2, *spatial_shape), dtype, scale_log2, vector=vector)
        b = ctypes.c_size_t(0)
        _check(lib().ftk_tracker_workspace_size(ctypes.byref(desc), int(capacity), window, ctypes.byref(b)),
               "ftk_tracker_workspace_size")
        return b.value

    def push(self, plane: torch.Tensor):
        if self._h is None:
            raise FtkError(ERR_INVALID_ARG, "Tracker.push after finish")
        if tuple(plane.shape) != self.spatial_shape or plane.dtype != self.dtype:
            raise FtkError(ERR_INVALID_ARG, f"Tracker.push: plane must be {self.spatial_shape} {self.dtype}")
        plane = plane.contiguous()
        # the plane may have been produced on another stream: order the tracker's copy after it, and
        # keep the caching allocator from reusing a device plane before the copy has run
        cur = torch.cuda.current_stream(self.device)
        if cur != self.stream:
            self.stream.wait_stream(cur)
        if plane.is_cuda:
            plane.record_stream(self.stream)
        _check(lib().ftk_tracker_push(self._h, ctypes.c_void_p(plane.data_ptr())), "ftk_tracker_push")
        if not plane.is_cuda:  # keep the host buffer alive until its asynchronous copy has run
            ev = torch.cuda.Event()
            ev.record(self.stream)
            self._keep.append((plane, ev))
            while len(self._keep) > 2 * self._window + 2:
                self._keep.popleft()[1].synchronize()

    def finish(self) -> torch.Tensor:
        n_out = ctypes.c_int64(0)
        h, self._h = self._h, None
        st = lib().ftk_tracker_finish(h, ctypes.byref(n_out))
        self._keep.clear()
        _check(st, "ftk_tracker_finish")
        return self.records[: n_out.value * RECORD_BYTES].view(torch.int64).view(-1, 7)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ftk_tracker_abort(self._h)
            self._h = None


class Trajectories:
    """Post-processing of the labelled records of one track() call (
    include/ftk_cp.h ftk_post_*): adjacency along the trajectories, slicing at a time t0, filtering by
    duration / loops, simplification in time, type smoothing.  `buffers` are the ones the track call used (return_buffers=True);
    `shape` is the tracked field's shape."""

    def __init__(self, rec: torch.Tensor, buffers: Buffers, shape, dtype, scale_log2: int, vector: bool = False):
        self.rec = rec
        self.buffers = buffers
        self.desc = make_desc(tuple(shape), dtype, scale_log2, vector=vector)
        self.n = rec.shape[0]
        self.nbr = torch.empty((max(self.n, 1), 2), dtype=torch.int64, device=rec.device)
        _check(lib().ftk_post_adjacency(ctypes.byref(self.desc), ctypes.c_void_p(rec.data_ptr()), self.n,
                                        ctypes.c_void_p(self.nbr.data_ptr()), *self._ws()), "ftk_post_adjacency")

    def _ws(self):
        b = self.buffers
        return (ctypes.c_void_p(b.workspace.data_ptr()), b.workspace.numel(), b.capacity,
                ctypes.c_void_p(_stream_ptr(self.rec.device)))

    def _out(self, fn, *args):
        cap = max(self.n, 16)
        while True:
            out = torch.empty(cap * RECORD_BYTES, dtype=torch.uint8, device=self.rec.device)
            n_out = ctypes.c_int64(0)
            st = fn(ctypes.byref(self.desc), ctypes.c_void_p(self.rec.data_ptr()), ctypes.c_void_p(self.nbr.data_ptr()),
                    self.n, *args, ctypes.c_void_p(out.data_ptr()), cap, ctypes.byref(n_out), *self._ws())
            if st == ERR_CAPACITY:
                cap = n_out.value
                continue
            _check(st, fn.__name__)
            return out[: n_out.value * RECORD_BYTES].view(torch.int64).view(-1, 7)

    def slice(self, t0: float) -> torch.Tensor:
        return self._out(lib().ftk_post_slice, ctypes.c_double(t0))

    def filter(self, min_duration: float, drop_loops: bool = False) -> torch.Tensor:
        return self._out(lib().ftk_post_filter, ctypes.c_double(min_duration), 1 if drop_loops else 0)

    def smooth_types(self, half_window: int = 2) -> torch.Tensor:
        """in place on the records (half-window of two in the paper's experiments)"""
        _check(lib().ftk_post_smooth_types(ctypes.byref(self.desc), ctypes.c_void_p(self.rec.data_ptr()),
                                           ctypes.c_void_p(self.nbr.data_ptr()), self.n, half_window, *self._ws()),
               "ftk_post_smooth_types")
        return self.rec

    def simplify_types(self, tau: float) -> torch.Tensor:
        """in place on the records: short-lived fold-to-fold segments (time extent < tau) take the type
        of the trajectory around them (simplification by persistence in time)"""
        _check(lib().ftk_post_simplify_types(ctypes.byref(self.desc), ctypes.c_void_p(self.rec.data_ptr()),
                                             ctypes.c_void_p(self.nbr.data_ptr()), self.n, ctypes.c_double(tau),
                                             *self._ws()), "ftk_post_simplify_types")
        return self.rec


def to_numpy(rec: torch.Tensor) -> np.ndarray:
    """Copy device records to a structured numpy array (RECORD_DTYPE)."""
    a = rec.detach().cpu().contiguous().numpy()
    return a.view(np.uint8).view(RECORD_DTYPE).reshape(-1)


def set_profiling(enable: bool):
    lib().ftk_set_profiling(1 if enable else 0)


def set_debug(flags: int):
    """Testing switches of the calling thread (DEBUG_FORCE_GENERIC | DEBUG_VERIFY_LINK |
    DEBUG_STITCH_HOST, DEBUG_NO_GRAPH, DEBUG_UF_BY_ID; include/ftk_cp.h ftk_set_debug): they change the path taken, never the
    result."""
    _check(lib().ftk_set_debug(int(flags)), "ftk_set_debug")


def last_kernel_timings():
    """[K1a scan, K1b exact, pass 2, stitch] device ms of the last profiled call (2D; 3D: K1 in [0])"""
    ms = (ctypes.c_float * 4)()
    _check(lib().ftk_last_kernel_timings(ms, 4), "ftk_last_kernel_timings")
    return list(ms)


def last_timings():
    """(ms[4]: pass1, pass2, stitch, call; stats[3]: faces, prefilter survivors, punctured)"""
    ms = (ctypes.c_float * 4)()
    st = (ctypes.c_int64 * 3)()
    lib().ftk_last_timings(ms, st)
    return list(ms), list(st)


# ----------------------------------------------------------------------------- time slabs
def _np_ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else None


def stitch_export(field: torch.Tensor, scale_log2: int, t0: int, nt_global: int, ghost: bool, buffers: Buffers,
                  vector: bool = False):
    """After track() on a slab with these buffers: the slab's (A, B) pair lists as int64 [n, 2]."""
    desc = make_desc(tuple(field.shape), field.dtype, scale_log2, t0, nt_global, ghost, vector=vector)
    nA, nB = ctypes.c_int64(0), ctypes.c_int64(0)
    args = lambda a, b, ca, cb: [ctypes.byref(desc), ctypes.c_void_p(buffers.workspace.data_ptr()),
                                 buffers.workspace.numel(), buffers.capacity, _np_ptr(a), ca, ctypes.byref(nA),
                                 _np_ptr(b), cb, ctypes.byref(nB), ctypes.c_void_p(_stream_ptr(field.device))]
    st = lib().ftk_stitch_export(*args(None, None, 0, 0))
    if st not in (OK, ERR_CAPACITY):
        _check(st, "ftk_stitch_export")
    A = np.zeros((nA.value, 2), np.int64)
    B = np.zeros((nB.value, 2), np.int64)
    _check(lib().ftk_stitch_export(*args(A, B, nA.value, nB.value)), "ftk_stitch_export")
    return A, B


def stitch_resolve(A: np.ndarray, B: np.ndarray, mine: np.ndarray):
    """Host-side union over all slabs' gathered pairs; returns (old labels, new labels) for `mine`."""
    A = np.ascontiguousarray(A, np.int64).reshape(-1, 2)
    B = np.ascontiguousarray(B, np.int64).reshape(-1, 2)
    mine = np.ascontiguousarray(mine, np.int64).reshape(-1)
    old = np.zeros(max(len(mine), 1), np.int64)
    new = np.zeros(max(len(mine), 1), np.int64)
    n = ctypes.c_int64(0)
    _check(lib().ftk_stitch_resolve(_np_ptr(A), len(A), _np_ptr(B), len(B), _np_ptr(mine), len(mine), _np_ptr(old),
                                    _np_ptr(new), ctypes.byref(n)), "ftk_stitch_resolve")
    return old[: n.value], new[: n.value]


def relabel(rec: torch.Tensor, old: np.ndarray, new: np.ndarray, buffers: Buffers):
    """Apply a label map to device records (rec: int64 [n, 7] view into buffers.records)."""
    old = np.ascontiguousarray(old, np.int64)
    new = np.ascontiguousarray(new, np.int64)
    _check(lib().ftk_relabel(ctypes.c_void_p(rec.data_ptr()), rec.shape[0], _np_ptr(old), _np_ptr(new), len(old),
                             ctypes.c_void_p(buffers.workspace.data_ptr()), buffers.workspace.numel(),
                             buffers.capacity, ctypes.c_void_p(_stream_ptr(rec.device))), "ftk_relabel")


def seam_block_size(cap: int) -> int:
    """int64 elements of one packed seam block (include/ftk_cp.h)"""
    return 2 + 4 * cap


def seam_pack(field: torch.Tensor, scale_log2: int, t0: int, nt_global: int, ghost: bool, buffers: Buffers,
              block: torch.Tensor, cap: int):
    """After track() on a slab with these buffers: write its packed seam block into `block` (device int64)."""
    desc = make_desc(tuple(field.shape), field.dtype, scale_log2, t0, nt_global, ghost)
    _check(lib().ftk_seam_pack(ctypes.byref(desc), ctypes.c_void_p(buffers.workspace.data_ptr()),
                               buffers.workspace.numel(), buffers.capacity, ctypes.c_void_p(block.data_ptr()), cap,
                               ctypes.c_void_p(_stream_ptr(block.device))), "ftk_seam_pack")


def seam_resolve(all_blocks: torch.Tensor, world: int, cap: int, rec: torch.Tensor):
    """Device resolve of the concatenated blocks of all slabs; relabels rec (int64 [n, 7] device view)."""
    _check(lib().ftk_seam_resolve(ctypes.c_void_p(all_blocks.data_ptr()), world, cap, ctypes.c_void_p(rec.data_ptr()),
                                  rec.shape[0], ctypes.c_void_p(_stream_ptr(rec.device))), "ftk_seam_resolve")


class Comm:
    """NCCL communicator of the library (one process per GPU).  The 128-byte unique id is created by
    rank 0 and broadcast with torch.distributed (the process group's own backend)."""

    def __init__(self, rank: int, world: int, group=None, device=None):
        import torch.distributed as dist
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _check(lib().ftk_comm_get_unique_id(uid), "ftk_comm_get_unique_id")
        backend = dist.get_backend(group)
        dev = device if backend == "nccl" else "cpu"
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=dev)
        dist.broadcast(t, 0, group=group)
        uid = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
        self.ptr = ctypes.c_void_p()
        _check(lib().ftk_comm_init(ctypes.byref(self.ptr), rank, world, uid), "ftk_comm_init")
        self.rank, self.world = rank, world

    def reserve(self, seam_pairs: int):
        """grow the pre-sized seam blocks (same value on every rank; outside the hot path)"""
        _check(lib().ftk_comm_reserve(self.ptr, int(seam_pairs)), "ftk_comm_reserve")

    def close(self):
        if self.ptr:
            lib().ftk_comm_destroy(self.ptr)
            self.ptr = ctypes.c_void_p()


def slab_bounds(nt_global: int, world: int):
    """Contiguous time slabs: rank r owns timesteps [b[r], b[r+1]) and reads one ghost plane."""
    return [nt_global * r // world for r in range(world + 1)]
