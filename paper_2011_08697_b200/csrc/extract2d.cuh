// extract2d.cuh -- launch interface of the pass-1 extraction kernels (K1).
#pragma once

#include "common.cuh"

namespace ftk {

struct ExtractParams {
  const void* field;   // device buffer [nt_buf][nz][ny][nx]
  int dtype;           // FTK_F32 / FTK_F64
  i64 nx, ny, nz;
  i64 nt_buf;          // planes in the buffer
  i64 t0;              // global timestep of plane 0
  i64 nt_global;
  i64 ta, tb;          // anchor timesteps (global) to test and emit: [ta, tb)
  i64 tchunk;          // anchor timesteps per CTA
  double scale;        // 2^s
  double thr;          // 2^(1-s): prefilter threshold on raw field differences
  ftk_cp* out;
  i64 capacity;
  unsigned long long* counters;  // Counter enum
  long long* edges;    // [capacity][2] trajectory-graph edges: (record, record or -1 - face_id)
  long long* fid;      // [capacity] face id of every record (compact copy for pass 2)
  // 2D: K1b also writes the union-find parents of its in-cube unions
  int* parent;         // [capacity]
  // K1a -> K1b survivor list.  3D: one entry per surviving hypercube, anchors wx, wy, wz and
  // wt = t | (t+1 in the buffer) << 31 (-1: no cube).  2D: group entries (first anchor wx, wy of a scan
  // lane's 4 x 8 anchors, wt as above, survivor mask in wz (bit 8i + r: position i, anchor row r;
  // 0: none)), expanded by k_expand2d into the cube list cx, cy, ct.  [wcap] each
  int *wx, *wy, *wt;
  int* wz;
  int *cx, *cy, *ct;
  i64 wcap;
  bool mesh;           // isovolume mesh requested: count the simplices, write up to elem_cap of them
  long long* elems;    // [elem_cap][ndim + 1] crossed-edge ids per simplex
  i64 elem_cap;
  bool force_generic;  // testing: disable TMA
  void* ev_mid;        // profiling: cudaEvent_t recorded between K1a and K1b (2D), or null
};

int launch_extract2d(const ExtractParams& P, cudaStream_t stream);
int launch_extract_vec2d(const ExtractParams& P, cudaStream_t stream);  // 2D vector fields
int launch_extract_vec3d(const ExtractParams& P, cudaStream_t stream);  // 3D vector fields
int launch_expand2d(const ExtractParams& P, cudaStream_t stream, int sms);  // group entries -> cube list
int launch_iso(const ExtractParams& P, long long cq, int ndim, cudaStream_t stream);  // isovolume edge + cell pass
int launch_extract3d(const ExtractParams& P, cudaStream_t stream);

}  // namespace ftk
