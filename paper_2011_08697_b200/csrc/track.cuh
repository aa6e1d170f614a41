// track.cuh -- launch interface of pass 2 (hash, link, union-find, labels).
#pragma once

#include "common.cuh"

namespace ftk {

struct HashSlot {
  long long key;  // face id, -1 = empty
  long long val;  // record index
};

struct TrackParams {
  ftk_cp* rec;                   // records from pass 1
  i64 capacity;
  unsigned long long* counters;  // CNT_NOUT holds the record count, CNT_EDGES the edge count
  HashSlot* table;               // face id -> record index; [table_cap] slots
  u64 table_cap;                 // power of two >= 1.5 * capacity; the kernels use
                                 // nextpow2(1.5 * n) <= table_cap slots, n = records found
  i64* fid;                      // [capacity] face ids (compact copy, union-find keys)
  int* parent;                   // [capacity] union-find parents
  const long long* edges;        // [capacity][2] edges from K1
  bool verify;                   // also re-derive every face's parent cells in closed form
};

// ext = {nx, ny, nz, nt_global}
int launch_track(const TrackParams& P, int ndim, const i64* ext, cudaStream_t stream);

}  // namespace ftk
