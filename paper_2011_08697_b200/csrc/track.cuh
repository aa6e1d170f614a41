// track.cuh -- launch interface of pass 2 (hash, link, union-find, labels).
#pragma once

#include "common.cuh"

namespace ftk {

struct TrackParams {
  ftk_cp* rec;                   // records from pass 1
  i64 capacity;
  unsigned long long* counters;  // CNT_NOUT holds the record count
  i64* keys;                     // hash table keys [hmask + 1] (face ids, -1 = empty)
  int* vals;                     // hash table values (record index)
  u64 hmask;
  i64* fid;                      // [capacity] face ids (compact copy, union-find keys)
  int* parent;                   // [capacity] union-find parents
};

// ext = {nx, ny, nz, nt_global}
int launch_track(const TrackParams& P, int ndim, const i64* ext, cudaStream_t stream);

}  // namespace ftk
