/*
 * ftk_cp.h -- C-ABI of the B200-native FTK critical-point tracking hot path.
 *
 * Method: Guo et al., "FTK: A Simplicial Spacetime Meshing Framework for Robust and Scalable
 * Feature Tracking", arXiv 2011.08697 (PAPER.md = /root/reference/PAPER.md, cited "P:<line>").
 *
 * Problem: a time-varying scalar field f on a regular nx x ny [x nz] grid, nt
 * timesteps.  Its gradient g (central differences) is piecewise linear on the Kuhn
 * (Freudenthal) subdivision of the (n+1)-D spacetime grid.  A spacetime critical point
 * is a zero of g; the zeros form trajectories.  Two-pass algorithm (Alg. 1 left,
 * P:350-369): pass 1 tests every n-simplex ("face") for a zero with an exact Simulation-of-
 * Simplicity point-in-simplex predicate on int64 fixed-point values, and gives each
 * punctured face its barycentric location (Eq. 2) and Hessian type; pass 2
 * joins the punctured faces of every (n+1)-simplex ("cell") by union-find.
 *
 * Every entry point returns an ftk_status (0 = FTK_OK).  No entry point allocates device memory
 * on the hot path; the caller owns every buffer it passes and nothing is retained after return.
 * All device work is enqueued on `stream`; the calls return after the result count is known
 * (one device->host read at the end), i.e. they are synchronous with respect to `stream`.
 * Results are deterministic: the SET of records and every field of each record depend only on the
 * input bytes and the descriptor (not on scheduling, tiling, or the number of GPUs); the ORDER of
 * records is unspecified unless FTK_SORTED is set.
 */
#ifndef FTK_CP_H
#define FTK_CP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FTK_ABI_VERSION 1

#if defined(__GNUC__)
#define FTK_API __attribute__((visibility("default")))
#else
#define FTK_API
#endif

typedef enum {
  FTK_OK = 0,
  FTK_ERR_INVALID_ARG = 1, /* bad descriptor / null pointer / workspace too small */
  FTK_ERR_RANGE = 2,       /* some |q| = |rint(f * 2^s)| >= 2^59 (2D) or 2^38 (3D), or a non-
                              finite input: the exact integer predicates could overflow */
  FTK_ERR_CAPACITY = 3,    /* more records than `capacity` (or more prefilter-surviving cubes
                              than the workspace's survivor list of max(1024, capacity) entries):
                              *n_out = the capacity to retry with, contents unspecified; the call
                              is idempotent, retry with larger buffers */
  FTK_ERR_CUDA = 4,        /* a CUDA runtime error (message via ftk_last_error()) */
  FTK_ERR_NCCL = 5,        /* an NCCL error in the multi-GPU stitch */
  FTK_ERR_INVARIANT = 6,   /* a cell with a punctured-face count not in {0, 2}; impossible under
                              SoS, so this signals a bug */
  FTK_ERR_NOMEM = 7
} ftk_status;

typedef enum { FTK_F32 = 0, FTK_F64 = 1 } ftk_dtype;

/* Critical point types (for a gradient field, maxima, minima and saddles). */
typedef enum {
  FTK_CP_DEGENERATE = 0, /* singular interpolated Hessian (exact zero determinant) */
  FTK_CP_MIN = 1,
  FTK_CP_SADDLE = 2,  /* 2D saddle */
  FTK_CP_SADDLE1 = 3, /* 3D, Morse index 1 (one negative eigenvalue) */
  FTK_CP_SADDLE2 = 4, /* 3D, Morse index 2 */
  FTK_CP_MAX = 5,
  /* vector fields (FTK_VECTOR_FIELD; "sources, sinks, and saddles"), from the mu-interpolated
   * Jacobian J: 2D: det J < 0 saddle (FTK_CP_SADDLE); det J > 0: trace > 0 source, < 0 sink, == 0
   * centre.  3D: eigenvalues with positive real part by Routh-Hurwitz: none sink, all source, else
   * saddle; an imaginary pair (a1 a2 == a3, a2 > 0) centre; det J == 0 degenerate (R17) */
  FTK_CP_SOURCE = 6,
  FTK_CP_SINK = 7,
  FTK_CP_CENTER = 8
} ftk_cp_type;

/* ftk_desc.flags */
#define FTK_GHOST_PLANE 1u      /* the buffer's last plane is a read-only ghost (time slab):
                                   faces anchored on it are tested for linking but not returned */
#define FTK_SORTED 2u           /* return records sorted by face_id (a device radix sort after pass 2
                                   and the stitch; without it the order of records is unspecified) */
#define FTK_VECTOR_FIELD 4u     /* the field is a VECTOR field: ndim components per vertex,
                                   interleaved, layout [t][y][x][2] (2D) or [t][z][y][x][3] (3D); its
                                   own zeros are tracked (no gradient step) and typed from its Jacobian */

/* ftk_cp.flags */
#define FTK_CP_ORDINAL 1u       /* all vertices in one timestep */
#define FTK_CP_BOUNDARY 2u      /* face shared by fewer than two cells (domain boundary) */
#define FTK_CP_DEGENERATE_LOC 4u /* sum of barycentric numerators == 0: location = centroid */

typedef struct {
  int32_t ndim;        /* spatial dimension n: 2 or 3 */
  int32_t dtype;       /* ftk_dtype of the field; layout dense row-major [t][z][y][x], x fastest */
  int64_t n[3];        /* nx, ny, nz; nz = 1 when ndim == 2; every spatial extent >= 3 */
  int64_t nt;          /* planes in the buffer (incl. the ghost plane when FTK_GHOST_PLANE) >= 1 */
  int64_t t0;          /* global timestep of the buffer's first plane (0 on a single GPU) */
  int64_t nt_global;   /* global number of timesteps; t0 + nt <= nt_global */
  int32_t scale_log2;  /* fixed point: q = rint(f * 2^scale_log2), round-half-even; [-64, 64] */
  uint32_t flags;      /* FTK_GHOST_PLANE | FTK_SORTED | FTK_VECTOR_FIELD */
} ftk_desc;

/* One punctured face (56 bytes). */
typedef struct {
  int64_t face_id;     /* I(anchor) * T + type; I = x + nx*(y + ny*(z + nz*t)) with global t;
                          T = 12 (2D+t) or 60 (3D+t) face types of the Kuhn cube */
  int64_t label;       /* trajectory id = the minimum face_id of its component; -1 from extract */
  double x, y, z, t;   /* spacetime location in grid units, t in global timesteps (z = 0 in 2D) */
  int32_t type;        /* ftk_cp_type */
  uint32_t flags;      /* FTK_CP_ORDINAL | FTK_CP_BOUNDARY | FTK_CP_DEGENERATE_LOC */
} ftk_cp;

typedef struct CUstream_st* ftk_stream; /* == cudaStream_t; NULL = legacy default stream */
typedef struct ftk_comm ftk_comm;       /* opaque multi-GPU communicator (NCCL) */

FTK_API int ftk_abi_version(void);
FTK_API const char* ftk_strerror(int status);
/* last CUDA/NCCL error text of the calling thread (empty if none) */
FTK_API const char* ftk_last_error(void);

/* Number of faces this buffer OWNS (anchors t in [t0, t0 + nt - ghost)): the faces every call
 * classifies; used for the faces/s metric.  Host-only arithmetic. */
FTK_API int ftk_num_faces(const ftk_desc* desc, int64_t* n_faces);

/* Device workspace needed by extract/track for up to `capacity` records (0 <= capacity < 2^31 - 1,
 * else FTK_ERR_INVALID_ARG).  It includes a list of max(1024, capacity) prefilter-surviving cubes,
 * handed from the scan kernel to the exact kernel. */
FTK_API int ftk_workspace_size(const ftk_desc* desc, int64_t capacity, size_t* bytes);

/* Pass 1: test every owned face, write the punctured ones to d_out[0 .. *n_out)
 * (label = -1; in face-id order with FTK_SORTED).  d_field: device pointer to the buffer; d_out: device array of `capacity`
 * records; d_ws: device workspace of ws_bytes >= ftk_workspace_size(). */
FTK_API int ftk_cp_extract(const ftk_desc* desc, const void* d_field, ftk_cp* d_out, int64_t capacity,
                   int64_t* n_out, void* d_ws, size_t ws_bytes, ftk_stream stream);

/* Pass 1 + pass 2: as extract, then join the punctured faces of every cell with a
 * lock-free union-find and label each record with its trajectory's minimum face_id.  With a
 * communicator (time slabs, one process per GPU): every rank passes its slab with one ghost plane
 * (FTK_GHOST_PLANE on all but the last rank), returns only the records it owns, and the labels
 * are global (identical to a single-GPU run).  comm = NULL: single GPU. */
FTK_API int ftk_cp_track(const ftk_desc* desc, const void* d_field, ftk_cp* d_out, int64_t capacity,
                 int64_t* n_out, void* d_ws, size_t ws_bytes, ftk_stream stream, ftk_comm* comm);
/* With a communicator every rank must call ftk_cp_track the same number of times: each call ends in
 * one exchange of seam blocks (NCCL allgather over NVLink) that every rank enters even when its own
 * slab failed, carrying the failure code, so that ALL ranks return the same status (any error other
 * than FTK_ERR_CAPACITY outranks a capacity shortfall; with FTK_ERR_CAPACITY every rank retries with
 * its *n_out).  The exchange uses only the communicator's pre-sized blocks (no allocation); a seam list
 * longer than the blocks takes a host path once, which re-sizes them. */

/* End-to-end variant from HOST memory: h_field is a host buffer (pinned for full PCIe speed) of the
 * whole input; the library copies it to d_stage (device buffer of the field's size) on `stream`,
 * runs track, and copies the records to h_out (host array of `capacity` records).  The streaming
 * tracker below is the variant that never holds the whole field on the device. */
FTK_API int ftk_cp_track_host(const ftk_desc* desc, const void* h_field, void* d_stage, ftk_cp* d_out,
                      ftk_cp* h_out, int64_t capacity, int64_t* n_out, void* d_ws, size_t ws_bytes,
                      ftk_stream stream);

/* Per-phase device times (ms) of the last extract/track call on this thread, measured with CUDA
 * events on `stream` when profiling is enabled: [0] pass 1 (K1 extraction kernel), [1] pass 2
 * (hash + link + union-find + labels), [2] slab stitch, [3] whole call.  Also the survivor
 * statistics of the last call: stats[0] = faces tested (owned), stats[1] = cubes surviving the
 * sign prefilter, stats[2] = punctured faces. */
FTK_API int ftk_set_profiling(int enable);
FTK_API int ftk_last_timings(float* ms4, int64_t* stats3);
/* Per-kernel device times (ms) of this thread's last profiled call: [0] scan kernel K1a (2D; the
 * whole pass 1 in 3D), [1] exact kernel K1b (2D, else 0), [2] pass 2, [3] stitch.  Fills
 * min(n, 4) entries; FTK_ERR_INVALID_ARG for a null pointer. */
FTK_API int ftk_last_kernel_timings(float* ms, int n);

/* Slab stitch, exposed step by step (ftk_cp_track with a communicator runs all of it internally).
 * After a track call on a time slab (FTK_GHOST_PLANE and/or t0 > 0) the workspace holds two lists of
 * (face id, local label) pairs: A = faces on the ghost plane that close a cell of this slab, with the
 * label of their partner; B = this slab's punctured ordinal faces on its first plane.
 * ftk_stitch_export copies them to host arrays (pairs, row-major [n][2]).  Gathered over all slabs
 * (any transport), ftk_stitch_resolve (host only) unions the labels -- every A pair joins its label
 * with the owner slab's label of the same face id (B) -- and returns, for the labels in `mine`, the
 * sorted map old label -> global label (entries that change only); global labels are the minimum
 * face id of the global trajectory, identical to a single-domain run.  ftk_relabel applies a map to
 * device records (capacity = the one the workspace was sized for).  FTK_ERR_INVARIANT: an A face
 * without an owner record. */
FTK_API int ftk_stitch_export(const ftk_desc* desc, void* d_ws, size_t ws_bytes, int64_t capacity, int64_t* h_A,
                              int64_t capA, int64_t* nA, int64_t* h_B, int64_t capB, int64_t* nB,
                              ftk_stream stream);
FTK_API int ftk_stitch_resolve(const int64_t* A, int64_t nA, const int64_t* B, int64_t nB, const int64_t* mine,
                               int64_t nmine, int64_t* map_old, int64_t* map_new, int64_t* nmap);
FTK_API int ftk_relabel(ftk_cp* d_out, int64_t n, const int64_t* h_map_old, const int64_t* h_map_new, int64_t nmap,
                        void* d_ws, size_t ws_bytes, int64_t capacity, ftk_stream stream);

/* Device seam path (used by ftk_cp_track with a communicator; exposed for tests and custom
 * transports).  A packed seam block holds one slab's lists:
 *   [0] nA, [1] nB, [2, 2 + 2 cap) A pairs, [2 + 2 cap, 2 + 4 cap) B pairs   (int64, 2 + 4 cap total);
 * a slab whose track failed publishes [0] = -code instead (no pairs).
 * ftk_seam_pack writes this slab's block (from the workspace of its last track call) to d_block
 * (device).  ftk_seam_resolve takes the world blocks concatenated in slab order (device, e.g. an
 * allgather), unions every A pair's label with the B label of the same face on the device and
 * relabels d_out[0, n) with the component minima -- labels not on any seam are unchanged.  Returns
 * FTK_ERR_CAPACITY (nothing relabelled) when a count exceeds cap, FTK_ERR_INVARIANT when an A face
 * has no B entry in any block.  Synchronises `stream` once (flag check). */
FTK_API int ftk_seam_pack(const ftk_desc* desc, void* d_ws, size_t ws_bytes, int64_t capacity, int64_t* d_block,
                          int64_t cap, ftk_stream stream);
FTK_API int ftk_seam_resolve(const int64_t* d_all, int world, int64_t cap, ftk_cp* d_out, int64_t n,
                             ftk_stream stream);

/* Streaming ingestion (P:709 push_field_data; the mesh is traversed one timestep after another,
 * P:282-286).  Timesteps are pushed one at a time; the tracker stages them in a window of
 * `window` + 1 planes inside d_ws and runs pass 1 on each full window (anchors [t0, t0 + window),
 * plane t0 + window as the ghost plane -- the time-slab rule), keeping the last plane for the next
 * window.  Records, trajectory edges and in-cube unions accumulate in d_out / d_ws across windows;
 * ftk_tracker_finish runs pass 1 on the remaining planes (the last one is the final timestep),
 * then pass 2 once over all records, and returns *n_out.  The result -- records, labels, flags --
 * is identical to one ftk_cp_track over the whole field, but only window + 1 planes are ever
 * resident on the device.
 *   desc: ndim, dtype, n[], scale_log2 as for track (nt, t0, nt_global, flags are ignored);
 *   window >= 1 timesteps per pass-1 launch (larger windows fill the GPU better: DESIGN.md 10);
 *   d_out: device array of `capacity` records for the WHOLE stream; d_ws: device workspace of
 *   ws_bytes >= ftk_tracker_workspace_size() bytes.  The tracker (a small host object) keeps
 *   these pointers until finish/abort -- the one exception to "nothing is retained".
 *   push: `plane` is one timestep (nx*ny*nz values of dtype), host or device memory (copied
 *   asynchronously on `stream`; a host buffer must stay valid until the stream reaches the copy --
 *   pinned memory for overlap).  Errors of a push are sticky and reported again by finish.
 *   finish: frees the tracker (also on error).  FTK_ERR_INVALID_ARG with fewer than 2 timesteps;
 *   FTK_ERR_CAPACITY (*n_out = required count) when records or survivors overflowed -- the stream
 *   must then be pushed again with a larger capacity.  abort: frees the tracker, no result. */
typedef struct ftk_tracker ftk_tracker;
FTK_API int ftk_tracker_workspace_size(const ftk_desc* desc, int64_t capacity, int32_t window, size_t* bytes);
FTK_API int ftk_tracker_begin(ftk_tracker** tracker, const ftk_desc* desc, int32_t window, ftk_cp* d_out,
                              int64_t capacity, void* d_ws, size_t ws_bytes, ftk_stream stream);
FTK_API int ftk_tracker_push(ftk_tracker* tracker, const void* plane);
FTK_API int ftk_tracker_finish(ftk_tracker* tracker, int64_t* n_out);
FTK_API int ftk_tracker_abort(ftk_tracker* tracker);

/* Trajectory post-processing (P:419 slicing; P:470-479 filtering, simplification and type smoothing) over the labelled
 * records d_rec[0, n) of ONE ftk_cp_track call on the whole domain described by desc, with the
 * workspace of that call (d_ws, ws_bytes, capacity; n <= capacity; its hash table, face-id and scratch
 * regions are reused, so the workspace must not be in use by another call).  All arrays are device
 * memory; every call is synchronous with respect to stream (one device->host read).
 *   adjacency: d_nbr[2 i], d_nbr[2 i + 1] = record index of the partner of record i in each of its (at
 *     most two) parent cells (closed-form side_of), -1 where the parent cell lies outside the domain.
 *     A trajectory is thereby a path (two ends with one -1) or a loop.  FTK_ERR_INVARIANT if a parent
 *     cell does not hold exactly one partner.  Must precede filter on the same workspace.
 *   slice: the trajectories at time t0: every record with t == t0 (copied), and for every adjacent pair
 *     whose t values strictly straddle t0 the point on their straight segment (the zero set inside the
 *     cell) at t0 -- x = x_lo + s (x_hi - x_lo), s = (t0 - t_lo) / (t_hi - t_lo), FP64, no FMA --
 *     carrying the face id, label and type of the end nearer in t (the earlier one on a tie), flags 0.
 *     Where several faces share one location (a trajectory through a grid vertex, the SoS case) the
 *     point is reported once per such face.
 *   filter: copies the records of the trajectories whose time extent (max t - min t over its records)
 *     is >= min_duration and, with drop_loops, that are not loops.
 *   smooth_types: for every record, up to half_window records are visited along the trajectory on each
 *     side; if both sides are non-empty and all visited records share one type T different from the
 *     record's own, its type becomes T (decided on the unmodified types, then applied; in place).
 *   simplify_types (simplification by persistence in time; R23): a FOLD is a record
 *     with two partners that both lie strictly later, or both strictly earlier, in t (a critical-point
 *     pair is born or annihilates there).  Folds cut a trajectory into segments running from one fold
 *     to the next (both included).  A segment with a fold at each end whose time extent (max t - min t
 *     over its records) is < tau, and whose two outer records (the partners of its end folds outside
 *     it) share one type T, is a short-lived excursion: its records take type T.  A fold belongs to
 *     two segments and takes T when the qualifying ones agree.  A loop with fewer than two folds is not
 *     cut.  Decided on the unmodified types, then applied (in place).  tau must not be NaN
 *     (FTK_ERR_INVALID_ARG); tau <= 0 changes nothing.
 *   slice / filter write up to cap records to d_out and set *n_out to the full count (FTK_ERR_CAPACITY
 *   when it exceeds cap); the output order is unspecified. */
FTK_API int ftk_post_adjacency(const ftk_desc* desc, const ftk_cp* d_rec, int64_t n, int64_t* d_nbr, void* d_ws,
                               size_t ws_bytes, int64_t capacity, ftk_stream stream);
FTK_API int ftk_post_slice(const ftk_desc* desc, const ftk_cp* d_rec, const int64_t* d_nbr, int64_t n, double t0,
                           ftk_cp* d_out, int64_t cap, int64_t* n_out, void* d_ws, size_t ws_bytes,
                           int64_t capacity, ftk_stream stream);
FTK_API int ftk_post_filter(const ftk_desc* desc, const ftk_cp* d_rec, const int64_t* d_nbr, int64_t n,
                            double min_duration, int32_t drop_loops, ftk_cp* d_out, int64_t cap, int64_t* n_out,
                            void* d_ws, size_t ws_bytes, int64_t capacity, ftk_stream stream);
FTK_API int ftk_post_smooth_types(const ftk_desc* desc, ftk_cp* d_rec, const int64_t* d_nbr, int64_t n,
                                  int32_t half_window, void* d_ws, size_t ws_bytes, int64_t capacity,
                                  ftk_stream stream);
FTK_API int ftk_post_simplify_types(const ftk_desc* desc, ftk_cp* d_rec, const int64_t* d_nbr, int64_t n,
                                    double tau, void* d_ws, size_t ws_bytes, int64_t capacity, ftk_stream stream);

/* Isovolume tracking (Alg. 1 right): the level set f = isovalue of a 2D+t / 3D+t SCALAR
 * field (desc as for track, the whole domain: t0 = 0, nt = nt_global >= 2, no ghost plane) on the same
 * Kuhn spacetime mesh.  Edge pass: every spacetime edge v -> v + m (m a nonzero axis mask) is crossed
 * iff g = rint(f 2^s) - rint(isovalue 2^s) has different SoS signs at its two ends, 0 counting as
 * positive (the 1D case of P:640: a level set through a vertex is owned by exactly one of its edges).
 * Each crossed edge is one record: face_id = edge id = I(v) (2^(n+1) - 1) + m - 1 (I as for faces),
 * location by Eq. 2 with n = 1 (FP64, no FMA), type 1 when g increases along the edge else 0, flags
 * FTK_CP_ORDINAL when m has no t bit.  Cell pass: the crossed edges of every cell (0, n+1 or 2n of them,
 * P:629-633 cases I / II; else FTK_ERR_INVARIANT) are joined; label = minimum edge id of the connected
 * isovolume piece (its "trajectory").  d_out / d_ws / capacity as for track (workspace of
 * ftk_workspace_size(desc, capacity)); FTK_ERR_CAPACITY sets *n_out to the capacity needed for the
 * records AND the cell links (several per crossed edge). */
FTK_API int ftk_iso_track(const ftk_desc* desc, double isovalue, const void* d_field, ftk_cp* d_out, int64_t capacity,
                          int64_t* n_out, void* d_ws, size_t ws_bytes, ftk_stream stream);
/* As ftk_iso_track, plus the isovolume itself as a simplicial mesh ("the output isovolumes
 * ... can be represented as a tetrahedral grid"): for every cell the level set crosses, with P / M its
 * positive / negative vertices in chain order (|P| + |M| = n + 2), the staircase triangulation of the
 * product simplex(P) x simplex(M) -- one simplex per monotone lattice path from (P_0, M_0) to
 * (P_last, M_last), its n + 1 vertices the crossed edges (P_i, M_j) along the path, given by their edge
 * ids (= the records' face_id; the intersection points are the records' locations).  That is 1 simplex
 * in case I and C(|P| + |M| - 2, |P| - 1) in case II: 3 tetrahedra for ++--- in 3D+t, 2
 * triangles for ++-- in 2D+t.  d_elems: device int64 [elem_cap][n + 1] (n = desc->ndim), order
 * unspecified across cells; *n_elems = the simplex count, FTK_ERR_CAPACITY when it exceeds elem_cap
 * (retry with *n_elems).  FTK_ERR_INVALID_ARG for a null n_elems or elem_cap > 0 with a null d_elems. */
FTK_API int ftk_iso_track_mesh(const ftk_desc* desc, double isovalue, const void* d_field, ftk_cp* d_out,
                               int64_t capacity, int64_t* n_out, int64_t* d_elems, int64_t elem_cap, int64_t* n_elems,
                               void* d_ws, size_t ws_bytes, ftk_stream stream);

/* Multi-GPU communicator over NCCL (one process per GPU).  Rank 0 creates the unique id, the
 * caller broadcasts the 128 bytes (e.g. with torch.distributed), every rank calls init. */
FTK_API int ftk_comm_get_unique_id(uint8_t id[128]);
FTK_API int ftk_comm_init(ftk_comm** comm, int rank, int world, const uint8_t id[128]);
/* init allocates the seam blocks and resolve tables for 2^17 pairs per list and slab (every rank:
 * world blocks of 2 + 4 * 2^17 int64 plus hash tables); reserve grows them for larger seams, outside
 * the hot path (the same value on every rank).  Call both on the device the rank's track calls use. */
FTK_API int ftk_comm_reserve(ftk_comm* comm, int64_t seam_pairs);
FTK_API int ftk_comm_destroy(ftk_comm* comm);

/* Testing switches of the calling thread (off by default; they never change results, only the
 * path taken): FTK_DEBUG_FORCE_GENERIC stages the 2D planes with the generic loader instead of TMA,
 * FTK_DEBUG_VERIFY_LINK re-derives every punctured face's parent cells in closed form after pass 2
 * (side_of; a cell without exactly one partner counts as FTK_ERR_INVARIANT), FTK_DEBUG_STITCH_HOST
 * resolves time-slab seams through the host path, FTK_DEBUG_NO_GRAPH launches every kernel of a track
 * call directly instead of replaying the call's cached CUDA graph (ftk_cp_track captures the launch
 * sequence of a call on first use and replays it when the same call -- descriptor, pointers, capacity,
 * workspace, switches -- repeats on the same host thread and device; a caller capturing its own stream
 * gets plain launches), FTK_DEBUG_UF_BY_ID as below.  FTK_ERR_INVALID_ARG for unknown bits. */
#define FTK_DEBUG_FORCE_GENERIC 1u
#define FTK_DEBUG_VERIFY_LINK 2u
#define FTK_DEBUG_STITCH_HOST 4u
#define FTK_DEBUG_NO_GRAPH 8u
#define FTK_DEBUG_UF_BY_ID 16u  /* pass 2 links union-find roots by face id at any record count (by default
                                   by an index priority up to 2^24 records, with the labels gathered at the
                                   roots: the same labels, other paths) */
FTK_API int ftk_set_debug(uint32_t flags);

#ifdef __cplusplus
}
#endif
#endif /* FTK_CP_H */
