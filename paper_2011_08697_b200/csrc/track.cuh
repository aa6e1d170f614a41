// track.cuh -- launch interface of pass 2 (hash, link, union-find, labels).
#pragma once

#include "common.cuh"

namespace ftk {

struct TrackParams {
  ftk_cp* rec;                   // records from pass 1
  i64 capacity;
  unsigned long long* counters;  // CNT_NOUT holds the record count, CNT_EDGES the edge count
  int* table;                    // face id -> record index: open addressing over record indices
                                 // (-1 = empty), the key of slot r is fid[r]; [table_cap] slots
  u64 table_cap;                 // power of two >= 1.5 * capacity; the kernels use
                                 // nextpow2(1.5 * n) <= table_cap slots, n = records found
  i64* fid;                      // [capacity] face ids of the records, written by K1 (hash keys,
                                 // union-find keys, labels)
  int* parent;                   // [capacity] union-find parents
  long long* lab;                // [capacity] component minimum face id, kept at each root (priority linking)
  int* root;                     // [capacity] root of each record (priority linking)
  bool uf_by_id;                 // link by face id whatever the record count (FTK_DEBUG_UF_BY_ID)
  const long long* edges;        // [capacity][2] edges from K1
  bool verify;                   // also re-derive every face's parent cells in closed form
  unsigned long long lookup_types;  // face types (bit per type) inserted into the table: the types
                                 // an edge or the verifier can look up
  bool prelinked;                // K1 initialised parent[] with its in-cube unions and emitted only
                                 // the edges to faces of neighbour cubes (2D)
  // geometry of the face ids (the spatially blocked hash decodes them)
  int ndim;
  i64 ext[4];                    // nx, ny, nz, nt (global)
  double inv[4];                 // 1 / T, 1 / nx, 1 / ny, 1 / nz (first guess of the id divisions)
  // time slabs (multi-GPU stitch)
  int T;                         // face types per cube (12 / 60; isovolumes: edge types 7 / 15)
  i64 plane;                     // vertices per timestep (nx * ny * nz)
  i64 ghost_t;                   // global t of the ghost plane, -1 without one
  i64 first_t;                   // global t of the first owned plane if t0 > 0, else -1
  long long* cross;              // [capacity][2] (record, face id on the ghost plane)
  long long* exportA;            // [capacity][2] (face id on the ghost plane, local label)
  long long* exportB;            // [capacity][2] (own ordinal face id on the first plane, local label)
};

// map: sorted old labels (old[i] < old[i+1]) -> new labels
int launch_relabel(ftk_cp* rec, i64 n, const long long* old_labels, const long long* new_labels, i64 nmap,
                   cudaStream_t stream);
int launch_export(const TrackParams& P, cudaStream_t stream);

// ext = {nx, ny, nz, nt_global}
int launch_track(const TrackParams& P, int ndim, const i64* ext, cudaStream_t stream);
// post-processing
struct PostCall {
  const ftk_cp* rec;
  ftk_cp* rec_mut;            // smoothing writes the types here (== rec)
  const long long* nbr;       // [n][2]
  long long n;
  ftk_cp* out;
  long long cap;
  unsigned long long* count;  // device output counter
  long long* scratch;         // [3 n] int64 + [n] int32
  double t0, dmin;
  int drop_loops, half_window;
  double tau;                 // simplification: persistence-in-time threshold
};
int launch_post_adjacency(const TrackParams& P, int ndim, const i64* ext, long long n, long long* nbr,
                          cudaStream_t stream);
int launch_post(const TrackParams& P, int op, const PostCall& c, cudaStream_t stream);  // 0 slice, 1 filter, 2 smooth, 3 simplify

}  // namespace ftk

namespace ftk {

// Device-side seam resolve for time slabs (no host round trip).  A packed seam block per slab:
//   [0] nA (or -code when the slab's track failed), [1] nB, [2 .. 2 + 2 cap) A pairs (ghost-plane face id, local label),
//   [2 + 2 cap .. 2 + 4 cap) B pairs (first-plane ordinal face id, local label);
// the blocks of all slabs are concatenated (NCCL allgather), every rank resolves all of them the
// same way and relabels its own records.
__host__ __device__ inline long long seam_stride(long long cap) { return 2 + 4 * cap; }

struct SeamScratch {            // library-owned, sized for world * cap pairs per list
  long long* hb_key;            // face id -> B label table (open addressing, -1 empty)
  long long* hb_val;
  unsigned long long hb_mask;
  long long* hl_key;            // label -> node table; the node is the slot, parent per slot
  int* hl_parent;
  unsigned long long hl_mask;
  unsigned long long* flags;    // [0] overflow (a slab's list exceeded cap), [1] unmatched A pairs,
                                // [2] max status code of the slabs whose track failed (0: none)
};

// pack this slab's lists (from the workspace after k_export) into its seam block
int launch_seam_pack(const TrackParams& P, long long* block, long long cap, cudaStream_t stream);
// resolve all blocks and relabel d_out[0, n) (labels not on any seam are unchanged)
int launch_seam_resolve(const long long* all, int world, long long cap, const SeamScratch& S, ftk_cp* d_out,
                        long long n, cudaStream_t stream);

}  // namespace ftk
