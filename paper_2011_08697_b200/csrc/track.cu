// track.cu -- pass 2 of Alg. 1: join the punctured faces of every cell.
//
// K1 already evaluated every cell (each cell lies inside one cube) and emitted the trajectory-graph
// edges (record i, record j) or (record i, -1 - face id of a face owned by a neighbour cube).  Here:
//
//   K3  a GPU hash table face id -> record index, sized from the device-side record count
//       (nextpow2(1.5 n) 4-byte slots holding record indices -- the key of a slot is fid[record],
//       written by K1 -- linear probing; ~17 MB for 2.7 M records, resident in L2),
//   K4  edge resolution + lock-free union-find (north_star (4)): the root with the larger face id is
//       hooked under the smaller one with atomicCAS, path halving on finds,
//   K6  labels: every record gets the face id of its root = the minimum face id of its trajectory,
//       independent of scheduling.
//
// Optional verification (FTK_VERIFY_LINK): every punctured face re-derives its (at most two) parent
// cells in closed form (side_of) and checks that each holds exactly one
// other punctured face -- an independent check of K1's cell evaluation.
#include <utility>

#include "common.cuh"
#include "kuhn.cuh"
#include "track.cuh"

namespace ftk {

static int num_sms() {  // cached per host thread and device
  thread_local int cached_dev = -1, cached = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && dev != cached_dev) {
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    cached_dev = dev;
  }
  return cached;
}

namespace trk {

constexpr int EMPTY = -1;

__constant__ KuhnTables<3> cK3 = kKuhn3;
__constant__ KuhnTables<4> cK4 = kKuhn4;

__device__ __forceinline__ u64 mix(u64 k) { return hash_mix(k); }

// exact n / d for 0 <= n < 2^52 from a floating-point first guess (off by at most one)
__device__ __forceinline__ i64 divq(i64 n, i64 d, double inv) {
  i64 q = (i64)((double)n * inv);
  if (q * d > n) --q;
  else if ((q + 1) * d <= n) ++q;
  return q;
}

// Slot of a face id in the pass-2 table: spatially blocked open addressing.  The table is cut into
// blocks of HBLK slots; a face's block is picked by its coarse position -- the 128-column x tile, 64
// rows (3D: 8 rows x 8 slices) and 32 (3D: 16) timesteps, the grain of K1a's work items, whose records
// are emitted together -- and the slot inside it by a hash of the face id.  The inserts and lookups of
// one work item's records and edges (processed in emission order) thus stay within a few blocks that
// are resident in L2, instead of touching the whole table.  When the table has more blocks than there
// are coarse cells (dense records: noisy fields, isovolumes), every coarse cell owns a group of 2^gs
// consecutive blocks and the face-id hash picks the block within it, so a cell's records spread over
// as many slots as the table has per cell (gs = 0: one block per cell).  Probing (TProbe) is linear
// within a block for at most HRUN slots, then jumps to another block of the table, chosen by the key
// (home + j s, s odd: every block in turn), so a cell with more records than its blocks hold -- records
// concentrated in a few cells, or the spatially clustered first records of a call whose capacity is
// too small -- spills into the whole table at its load factor instead of growing one linear cluster.
constexpr int HBLK_LOG2 = 12;
#ifndef FTK_HRUN
#define FTK_HRUN 32
#endif
constexpr int HRUN = FTK_HRUN;  // slots probed per block before the jump
#ifndef FTK_UF_PRIO_MAX
#define FTK_UF_PRIO_MAX (1ll << 24)  // record counts up to which roots are linked by index priority
#endif
__device__ __forceinline__ u64 coarse_cells(const TrackParams& P) {
  if (P.ndim == 2)
    return (u64)((P.ext[0] + 127) >> 7) * (u64)((P.ext[1] + 63) >> 6) * (u64)((P.ext[3] + 31) >> 5);
  return (u64)((P.ext[0] + 127) >> 7) * (u64)((P.ext[1] + 7) >> 3) * (u64)((P.ext[2] + 7) >> 3) *
         (u64)((P.ext[3] + 15) >> 4);
}
__device__ __forceinline__ u64 slot_of(const TrackParams& P, u64 hm, long long key) {
  const u64 h = mix((u64)key);
  if (hm < (1ull << HBLK_LOG2)) return h & hm;
  const i64 I = divq(key, P.T, P.inv[0]);
  const i64 r1 = divq(I, P.ext[0], P.inv[1]);
  const i64 x = I - r1 * P.ext[0];
  const i64 r2 = divq(r1, P.ext[1], P.inv[2]);
  const i64 y = r1 - r2 * P.ext[1];
  u64 coarse;
  if (P.ndim == 2) {  // r2 = t
    coarse = ((u64)(r2 >> 5) * (u64)((P.ext[1] + 63) >> 6) + (u64)(y >> 6)) * (u64)((P.ext[0] + 127) >> 7) + (u64)(x >> 7);
  } else {
    const i64 t = divq(r2, P.ext[2], P.inv[3]);
    const i64 z = r2 - t * P.ext[2];
    coarse = (((u64)(t >> 4) * (u64)((P.ext[2] + 7) >> 3) + (u64)(z >> 3)) * (u64)((P.ext[1] + 7) >> 3) + (u64)(y >> 3)) *
                 (u64)((P.ext[0] + 127) >> 7) + (u64)(x >> 7);
  }
  // consecutive coarse cells take consecutive block groups (modulo the block count): no two cells share
  // a block while there are at least as many blocks as cells; a hashed group choice would collide cells
  // and grow long probe chains
  const int gs = (int)P.counters[CNT_HGROUP];
  const u64 blk = ((coarse << gs) | ((h >> HBLK_LOG2) & ((1ull << gs) - 1))) & (hm >> HBLK_LOG2);
  return (blk << HBLK_LOG2) | (h & ((1ull << HBLK_LOG2) - 1));
}

// the probe sequence of a key: slot_of, then HRUN-slot runs in the blocks home + j s
struct TProbe {
  u64 hm, h, blk0, stride;
  long long key;
  int run;
  long long j;
  __device__ TProbe(const TrackParams& P, u64 hm_, long long key_) : hm(hm_), key(key_), run(0), j(0) {
    h = slot_of(P, hm, key);
    blk0 = h >> HBLK_LOG2;
    stride = 0;  // computed at the first jump
  }
  __device__ __forceinline__ u64 slot() const { return h; }
  __device__ __forceinline__ void next() {
    if (hm < (1ull << HBLK_LOG2) || run < 0) {  // small table (or every block visited): linear probing
      h = (h + 1) & hm;
      return;
    }
    if (++run < HRUN) {
      h = (h & ~((1ull << HBLK_LOG2) - 1)) | ((h + 1) & ((1ull << HBLK_LOG2) - 1));
      return;
    }
    run = 0;
    ++j;
    const u64 nblk = (hm >> HBLK_LOG2) + 1;
    if ((u64)j >= nblk) {  // every block visited (cannot happen below full load): linear over the table
      h = (h + 1) & hm;
      run = -1;
      return;
    }
    if (j == 1) stride = (mix((u64)key ^ 0x5bd1e995ull) >> 20) | 1ull;
    const u64 blk = (blk0 + (u64)j * stride) & (nblk - 1);
    h = (blk << HBLK_LOG2) | (h & ((1ull << HBLK_LOG2) - 1));
  }
};

__device__ __forceinline__ i64 n_records(const TrackParams& P) {
  const i64 n = (i64)P.counters[CNT_NOUT];
  return n < P.capacity ? n : P.capacity;
}

// Union-find linking rule of this call (device-side, from the record count): by a pseudo-random
// priority of the record index, the label then gathered at the roots (k_root), while the records fit
// the L2-resident regime (C2: k_edges 106 -> 64 us, pass 2 0.211 -> 0.183 ms; C5 0.150 -> 0.096 ms);
// by face id beyond it, where the gather pass's extra DRAM traffic costs more than the shorter paths
// save (C4, 87 M records: pass 2 5.10 ms by face id, 5.70 by priority).  Labels are the same either way.
__device__ __forceinline__ bool uf_by_prio(const TrackParams& P) {
  return !P.uf_by_id && n_records(P) <= FTK_UF_PRIO_MAX;
}

// the slot mask chosen by k_clear for this call
__device__ __forceinline__ u64 table_mask(const TrackParams& P) { return P.counters[CNT_HMASK]; }

__global__ void k_clear(const __grid_constant__ TrackParams P) {
  const u64 hm = hash_slots(n_records(P), P.table_cap) - 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    P.counters[CNT_HMASK] = hm;
    // blocks per coarse cell: 2^gs, the largest power of two with 2^gs x (cells rounded up to a power of
    // two) <= blocks
    const u64 nblk = (hm + 1) >> HBLK_LOG2, nc = coarse_cells(P);
    int gs = 0;
    while ((1ull << (gs + 1)) * nc <= nblk) ++gs;
    P.counters[CNT_HGROUP] = (unsigned long long)gs;
  }
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= hm; i += (u64)gridDim.x * blockDim.x)
    P.table[i] = EMPTY;
}

__global__ void k_hash_insert(const __grid_constant__ TrackParams P) {
  const i64 n = n_records(P);
  const bool prio = uf_by_prio(P);
  const u64 hm = table_mask(P);
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const long long key = P.fid[i];
    if (!P.prelinked) P.parent[i] = (int)i;
    // a record K1 already hooked under its cube's root (a face of the same cube with a smaller face
    // id, 2D) is never a component minimum and never a root: -1 tells k_root to skip its atomic
    if (prio) P.lab[i] = (P.prelinked && P.parent[i] != (int)i) ? -1 : key;
    // only faces that some cell of a neighbour cube looks up (the "upper" types) need a slot
    if (!((P.lookup_types >> (int)(key % P.T)) & 1ull)) continue;
    TProbe pr(P, hm, key);
    // face ids are unique among the records: claim the first empty slot of the probe sequence
    [[maybe_unused]] u64 probes = 0;
    while (atomicCAS(&P.table[pr.slot()], EMPTY, (int)i) != EMPTY) {
      pr.next();
      FTK_ASSERT(++probes <= 2 * hm + 2);  // the table always has an empty slot (1.5 slots per record)
    }
  }
}

__device__ __forceinline__ long long lookup(const TrackParams& P, u64 hm, long long key) {
  TProbe pr(P, hm, key);
#if FTK_CHECKS
  u64 probes = 0;
#endif
  while (true) {
#if FTK_CHECKS
    FTK_ASSERT(++probes <= 2 * hm + 2);
#endif
    const int r = P.table[pr.slot()];
    if (r == EMPTY) return -1;
    if (P.fid[r] == key) return r;
    pr.next();
  }
}

__device__ __forceinline__ int uf_find(int* parent, int i) {
#if FTK_CHECKS
  long long steps = 0;
#endif
  while (true) {
    const int p = parent[i];
#if FTK_CHECKS
    FTK_ASSERT(p >= 0 && ++steps < (1ll << 31));  // a parent cycle would never reach a root
#endif
    if (p == i) return i;
    const int gp = parent[p];
    if (gp != p) parent[i] = gp;  // path halving; benign race (pointers only move to smaller keys)
    i = p;
  }
}

// Priority linking (uf_by_prio): roots are linked by a pseudo-random priority of their record index (the lower under
// the higher; a parent always outranks its child, so a path is an increasing run of hashes: O(log n)
// expected depth even when the edges of a trajectory are united concurrently) instead of by face id,
// whose order along a trajectory (time-major) chains its records into one long path when its edges are
// processed at once; the component minimum face id -- the label -- is then gathered at the roots
// (k_root) instead of being the root itself
__device__ __forceinline__ u64 uf_prio(int r) {
  unsigned x = (unsigned)r * 0x9E3779B1u;
  x ^= x >> 16;
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  x *= 0xC2B2AE35u;
  x ^= x >> 16;
  return ((u64)x << 32) | (unsigned)r;  // ties broken by the index: a strict order
}
// both finds of a union advanced together: the two parent chains' loads overlap instead of running
// one after the other (the same path splitting as uf_find on each)
__device__ __forceinline__ void uf_find2(int* parent, int& a, int& b) {
#if FTK_CHECKS
  long long steps = 0;
#endif
  while (true) {
    const int pa = parent[a], pb = parent[b];
    const bool ra = pa == a, rb = pb == b;
    if (ra && rb) return;
#if FTK_CHECKS
    FTK_ASSERT(pa >= 0 && pb >= 0 && ++steps < (1ll << 31));
#endif
    const int ga = ra ? pa : parent[pa];
    const int gb = rb ? pb : parent[pb];
    if (!ra) {
      if (ga != pa) parent[a] = ga;
      a = pa;
    }
    if (!rb) {
      if (gb != pb) parent[b] = gb;
      b = pb;
    }
  }
}

__device__ __forceinline__ void uf_unite(int* parent, const i64* key, int a, int b, bool prio) {
  while (true) {
    uf_find2(parent, a, b);
    if (a == b) return;
    if (prio ? uf_prio(a) > uf_prio(b) : key[a] < key[b]) {
      const int t = a;
      a = b;
      b = t;
    }
    // a has the larger key: hook it under b
    const int old = atomicCAS(&parent[a], a, b);
    if (old == a) return;
  }
}

__global__ void k_edges(const __grid_constant__ TrackParams P) {
  const i64 nrec = n_records(P);
  const i64 ne0 = (i64)P.counters[CNT_EDGES];
  const i64 ne = ne0 < P.capacity ? ne0 : P.capacity;
  const u64 hm = table_mask(P);
  const bool prio = uf_by_prio(P);
  // Edges are visited in emission order (K1b batch order follows the scan: time-major runs of one
  // region), coalesced across the threads.  Measured alternatives -- a scattered permutation, or
  // one contiguous run per thread -- are within 15% on C2 but 3x slower on C4, where the union-find
  // working set is far beyond L2 and the shallow trees of the in-order unions matter.
  for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (i64)gridDim.x * blockDim.x) {
    long long a = P.edges[2 * e];
    long long b = P.edges[2 * e + 1];
    if (a < 0) a = lookup(P, hm, -1 - a);  // isovolume links may name both ends by id
    if (b < 0) {
      const long long f = -1 - b;
      b = lookup(P, hm, f);  // face owned by the neighbour cube
      if (b < 0 && P.ghost_t >= 0 && f / P.T / P.plane == P.ghost_t && a >= 0 && a < nrec) {
        // partner owned by the next time slab: stitched after the local labels are known
        const unsigned long long c = atomicAdd(&P.counters[CNT_CROSS], 1ull);
        if (c < (unsigned long long)P.capacity) {
          P.cross[2 * c] = a;
          P.cross[2 * c + 1] = f;
        }
        continue;
      }
    }
    if (a < 0 || b < 0 || a >= nrec || b >= nrec) {
      atomicAdd(&P.counters[CNT_INVARIANT], 1ull);  // a cell's partner face was never emitted
      continue;
    }
    uf_unite(P.parent, P.fid, (int)a, (int)b, prio);
  }
}

#ifndef FTK_LABEL_JUMP
#define FTK_LABEL_JUMP 0  // pointer-jumping passes over all records before K6; measured (r1f, tools/gpu_check3.sh):
                          // 2 passes C2 pass 2 0.20 -> 0.20 ms, C4 5.63 -> 6.32, C5 0.131 -> 0.116; kept at 0
#endif
__global__ void k_jump(const __grid_constant__ TrackParams P) {
  const i64 n = n_records(P);
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const int p = P.parent[i];
    if (p == (int)i) continue;
    const int gp = P.parent[p];
    if (gp != p) P.parent[i] = gp;  // benign race, as in path halving
  }
}

__global__ void k_label(const __grid_constant__ TrackParams P) {
  const i64 n = n_records(P);
  const bool prio = uf_by_prio(P);
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    if (prio) {
      P.rec[i].label = P.lab[P.root[i]];
    } else {
      const int r = uf_find(P.parent, (int)i);
      P.rec[i].label = P.fid[r];
    }
  }
}

// priority linking: every record's root, and the minimum face id of each component at its root
__global__ void k_root(const __grid_constant__ TrackParams P) {
  if (!uf_by_prio(P)) return;
  const i64 n = n_records(P);
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const long long f = P.lab[i];  // loaded before the find: its latency hides behind the parent chain
    const int r = uf_find(P.parent, (int)i);
    P.root[i] = r;
    if (r != (int)i && f >= 0) atomicMin(&P.lab[r], f);
  }
}

// ------------------------------------------------------------------------- slab stitch (K7, K9)
// K7: export (ghost-plane face id, local label of its partner) for every cross edge (A list) and
// (face id, local label) for every own ordinal face on the first owned plane (B list).
__global__ void k_export(const __grid_constant__ TrackParams P) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const i64 i0 = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  const i64 nc0 = (i64)P.counters[CNT_CROSS];
  const i64 nc = nc0 < P.capacity ? nc0 : P.capacity;
  for (i64 c = i0; c < nc; c += stride) {
    P.exportA[2 * c] = P.cross[2 * c + 1];
    P.exportA[2 * c + 1] = P.rec[P.cross[2 * c]].label;
  }
  if (P.first_t < 0) return;
  const i64 n = n_records(P);
  for (i64 i = i0; i < n; i += stride) {
    const long long f = P.fid[i];
    if (f / P.T / P.plane == P.first_t && (P.rec[i].flags & FTK_CP_ORDINAL)) {
      const unsigned long long k = atomicAdd(&P.counters[CNT_EXPORT_B], 1ull);
      if (k < (unsigned long long)P.capacity) {
        P.exportB[2 * k] = f;
        P.exportB[2 * k + 1] = P.rec[i].label;
      }
    }
  }
}

// K9: replace every label found in the sorted map
__global__ void k_relabel(ftk_cp* rec, i64 n, const long long* old_l, const long long* new_l, i64 nmap) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const long long l = rec[i].label;
    i64 lo = 0, hi = nmap;
    while (lo < hi) {
      const i64 mid = (lo + hi) >> 1;
      if (old_l[mid] < l) lo = mid + 1; else hi = mid;
    }
    if (lo < nmap && old_l[lo] == l) rec[i].label = new_l[lo];
  }
}

// ------------------------------------------------------------------------- device seam resolve
__global__ void k_seam_pack(const __grid_constant__ TrackParams P, long long* block, long long cap) {
  const i64 nA = (i64)P.counters[CNT_CROSS], nB = (i64)P.counters[CNT_EXPORT_B];
  const i64 stride = (i64)gridDim.x * blockDim.x, i0 = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i0 == 0) {
    block[0] = nA;
    block[1] = nB;
  }
  const i64 mA = min(nA, (i64)cap), mB = min(nB, (i64)cap);
  for (i64 i = i0; i < mA; i += stride) {
    block[2 + 2 * i] = P.exportA[2 * i];
    block[3 + 2 * i] = P.exportA[2 * i + 1];
  }
  for (i64 i = i0; i < mB; i += stride) {
    block[2 + 2 * cap + 2 * i] = P.exportB[2 * i];
    block[3 + 2 * cap + 2 * i] = P.exportB[2 * i + 1];
  }
}

struct SeamArgs {
  const long long* all;
  int world;
  long long cap;
  SeamScratch S;
  ftk_cp* rec;
  long long n;
};

__global__ void k_seam_clear(const __grid_constant__ SeamArgs A) {
  const u64 stride = (u64)gridDim.x * blockDim.x, i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  for (u64 i = i0; i <= A.S.hb_mask; i += stride) A.S.hb_key[i] = -1;
  for (u64 i = i0; i <= A.S.hl_mask; i += stride) {
    A.S.hl_key[i] = -1;
    A.S.hl_parent[i] = (int)i;
  }
  if (i0 < 3) A.S.flags[i0] = 0;
}

__device__ __forceinline__ int hl_insert(const SeamScratch& S, long long label) {
  u64 h = hash_mix((u64)label) & S.hl_mask;
  while (true) {
    const long long prev = (long long)atomicCAS(reinterpret_cast<unsigned long long*>(&S.hl_key[h]), ~0ull,
                                                (unsigned long long)label);
    if (prev == -1 || prev == label) return (int)h;
    h = (h + 1) & S.hl_mask;
  }
}
__device__ __forceinline__ int hl_find(const SeamScratch& S, long long label) {
  u64 h = hash_mix((u64)label) & S.hl_mask;
  while (true) {
    const long long k = S.hl_key[h];
    if (k == label) return (int)h;
    if (k == -1) return -1;
    h = (h + 1) & S.hl_mask;
  }
}

// B faces into the face table, every label of A and B into the label table
__global__ void k_seam_insert(const __grid_constant__ SeamArgs A) {
  const i64 stride = (i64)gridDim.x * blockDim.x, i0 = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  const long long bs = seam_stride(A.cap);
  for (int r = 0; r < A.world; ++r) {
    const long long* blk = A.all + r * bs;
    const i64 nA = blk[0], nB = blk[1];
    if (nA < 0) {  // the slab's track failed: -nA is its status code (see seam_fail)
      if (i0 == 0) atomicMax(&A.S.flags[2], (unsigned long long)(-nA));
      continue;
    }
    if ((nA > A.cap || nB > A.cap) && i0 == 0) A.S.flags[0] = 1;
    const i64 mA = min(nA, (i64)A.cap), mB = min(nB, (i64)A.cap);
    for (i64 i = i0; i < mB; i += stride) {
      const long long f = blk[2 + 2 * A.cap + 2 * i], l = blk[3 + 2 * A.cap + 2 * i];
      u64 h = hash_mix((u64)f) & A.S.hb_mask;
      while (atomicCAS(reinterpret_cast<unsigned long long*>(&A.S.hb_key[h]), ~0ull, (unsigned long long)f) != ~0ull)
        h = (h + 1) & A.S.hb_mask;  // face ids are unique among the B lists
      A.S.hb_val[h] = l;
      hl_insert(A.S, l);
    }
    for (i64 i = i0; i < mA; i += stride) hl_insert(A.S, blk[3 + 2 * i]);
  }
}

__device__ __forceinline__ int seam_find(int* parent, int i) {
  while (true) {
    const int p = parent[i];
    if (p == i) return i;
    const int gp = parent[p];
    if (gp != p) parent[i] = gp;
    i = p;
  }
}

// every A pair joins its label with the B label of the same face (hook the larger label's root
// under the smaller: roots end up as component minima)
__global__ void k_seam_union(const __grid_constant__ SeamArgs A) {
  const i64 stride = (i64)gridDim.x * blockDim.x, i0 = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  const long long bs = seam_stride(A.cap);
  for (int r = 0; r < A.world; ++r) {
    const long long* blk = A.all + r * bs;
    const i64 mA = min(blk[0], (i64)A.cap);
    for (i64 i = i0; i < mA; i += stride) {
      const long long f = blk[2 + 2 * i], la = blk[3 + 2 * i];
      u64 h = hash_mix((u64)f) & A.S.hb_mask;
      long long lb = -1;
      while (true) {
        const long long k = A.S.hb_key[h];
        if (k == f) {
          lb = A.S.hb_val[h];
          break;
        }
        if (k == -1) break;
        h = (h + 1) & A.S.hb_mask;
      }
      if (lb < 0) {
        atomicAdd(&A.S.flags[1], 1ull);
        continue;
      }
      int a = hl_find(A.S, la), b = hl_find(A.S, lb);
      while (true) {
        a = seam_find(A.S.hl_parent, a);
        b = seam_find(A.S.hl_parent, b);
        if (a == b) break;
        if (A.S.hl_key[a] < A.S.hl_key[b]) {
          const int t = a;
          a = b;
          b = t;
        }
        if (atomicCAS(&A.S.hl_parent[a], a, b) == a) break;
      }
    }
  }
}

// records whose label is on a seam take the label of its component root
__global__ void k_seam_relabel(const __grid_constant__ SeamArgs A) {
  if (A.S.flags[0] || A.S.flags[2]) return;  // a list overflowed its block (the caller takes the host
                                              // path) or a slab failed (every rank reports it)
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (i64)gridDim.x * blockDim.x) {
    const long long l = A.rec[i].label;
    const int node = hl_find(A.S, l);
    if (node >= 0) A.rec[i].label = A.S.hl_key[seam_find(A.S.hl_parent, node)];
  }
}

// ------------------------------------------------------------------------- closed-form verifier
template <int D>
struct Geo {
  i64 ext[4];   // extents in axis order x, y, [z,] t (t global)
  i64 stride[4];
};

template <int D>
__device__ __forceinline__ void decode(const Geo<D>& G, i64 fid, i64* v, int& type) {
  constexpr int T = KuhnTables<D>::NT;
  i64 I = fid / T;
  type = (int)(fid - I * T);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (a < D - 1) {
      v[a] = I % G.ext[a];
      I /= G.ext[a];
    } else {
      v[a] = I;
    }
  }
}

template <int D>
__device__ __forceinline__ i64 encode(const Geo<D>& G, const i64* v, int m_idx) {
  constexpr int T = KuhnTables<D>::NT;
  i64 I = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) I += v[a] * G.stride[a];
  const int ty = D == 3 ? cK3.type_of[m_idx] : cK4.type_of[m_idx];
  return I * T + ty;
}

// number of OTHER punctured faces of the cell given as a chain of D+1 cumulative masks w[0..D]
template <int D>
__device__ __forceinline__ int visit_cell(const TrackParams& P, u64 hm, const Geo<D>& G, const i64* A, const int* w,
                                          i64 self, long long* partner = nullptr) {
  int hits = 0;
#pragma unroll
  for (int j = 0; j <= D; ++j) {
    i64 anc[4];
    int idx = 0, sh = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) anc[a] = A[a];
    if (j == 0) {
#pragma unroll
      for (int a = 0; a < D; ++a) anc[a] += (w[1] >> a) & 1;
#pragma unroll
      for (int k = 2; k <= D; ++k) {
        idx |= (w[k] ^ w[1]) << sh;
        sh += 4;
      }
    } else {
#pragma unroll
      for (int k = 1; k <= D; ++k) {
        if (k == j) continue;
        idx |= w[k] << sh;
        sh += 4;
      }
    }
    const i64 f = encode<D>(G, anc, idx);
    if (f == self) continue;
    const long long r = lookup(P, hm, f);
    if (r >= 0) {
      ++hits;
      if (partner) *partner = r;
    }
  }
  return hits;
}

// Parent cells of every record in closed form (side_of): ADJ = false checks that each
// holds exactly one other punctured face (FTK_VERIFY_LINK); ADJ = true writes that partner's record
// index to nbr[2 i + k] (k-th existing parent cell; -1: no parent cell, i.e. the domain boundary).
template <int D, bool ADJ = false>
__global__ void k_verify(const __grid_constant__ TrackParams P, const Geo<D> G, long long* nbr = nullptr) {
  const i64 n = n_records(P);
  const u64 hm = table_mask(P);
  constexpr int FULL = (1 << D) - 1;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i64 self = P.fid[i];
    int ns = 0;
    auto cell = [&](const i64* anc, const int* w) {
      long long partner = -1;
      const int h = visit_cell<D>(P, hm, G, anc, w, self, &partner);
      if (ADJ) nbr[2 * i + ns++] = h == 1 ? partner : -1;
      return h != 1;
    };
    if (ADJ) nbr[2 * i] = nbr[2 * i + 1] = -1;
    i64 v[4];
    int type;
    decode<D>(G, self, v, type);
    int m[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 1; k < D; ++k) m[k] = D == 3 ? cK3.masks[type][k - 1] : cK4.masks[type][k - 1];
    const int U = m[D - 1];
    int bad = 0;
    if (U != FULL) {
      const int cbit = FULL & ~U;
      const int c = __ffs(cbit) - 1;
      if (v[c] + 1 <= G.ext[c] - 1) {  // parent 1: append v_last + e_c (same anchor)
        int w[5];
        w[0] = 0;
#pragma unroll
        for (int k = 1; k < D; ++k) w[k] = m[k];
        w[D] = FULL;
        bad |= cell(v, w);
      }
      if (v[c] >= 1) {  // parent 2: prepend v0 - e_c (anchor moves down)
        i64 A[4];
#pragma unroll
        for (int a = 0; a < D; ++a) A[a] = v[a] - (a == c ? 1 : 0);
        int w[5];
        w[0] = 0;
#pragma unroll
        for (int k = 1; k <= D; ++k) w[k] = cbit | m[k - 1];
        bad |= cell(A, w);
      }
    } else {
      // the face spans all axes: one step has two axes {a, b}; the parents split it both ways
      int step = 0, pair = 0;
#pragma unroll
      for (int k = 1; k < D; ++k) {
        const int s = m[k] ^ m[k - 1];
        if (__popc(s) == 2) {
          step = k;
          pair = s;
        }
      }
      const int a = pair & -pair, b = pair & ~a;
#pragma unroll
      for (int which = 0; which < 2; ++which) {
        int w[5];
        int o = 0;
        for (int k = 0; k < D; ++k) {
          if (k == step) w[o++] = m[k - 1] | (which ? b : a);
          w[o++] = m[k];
        }
        bad |= cell(v, w);
      }
    }
    if (bad) atomicAdd(&P.counters[CNT_INVARIANT], 1ull);
  }
}


// ------------------------------------------------------------------------- post-processing
// Over the labelled records of a track call and their adjacency nbr[n][2] (partners in the parent
// cells; a trajectory is a path or a loop of faces).  Times are non-negative, so the IEEE bits of a
// double order like the values.
__global__ void k_post_prep(const __grid_constant__ TrackParams P, long long n) {
  if (blockIdx.x == 0 && threadIdx.x == 0) P.counters[CNT_NOUT] = (unsigned long long)n;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    P.fid[i] = P.rec[i].face_id;
}

struct PostArgs {
  const ftk_cp* rec;
  const long long* nbr;
  long long n;
  ftk_cp* out;
  long long cap;
  unsigned long long* count;  // output counter
  long long* tmin;            // [n] per trajectory root record: min / max t (double bits), open ends
  long long* tmax;
  long long* nends;
  int* newtype;               // [n]
  double t0, dmin;
  int drop_loops, half_window;
  double tau;
};

__device__ __forceinline__ void post_emit(const PostArgs& A, const ftk_cp& r) {
  const unsigned long long k = atomicAdd(A.count, 1ull);
  if (k < (unsigned long long)A.cap) A.out[k] = r;
}

// slice at t = t0: records with t == t0, and the point of every trajectory segment (the
// straight segment between the two punctured faces of a cell) that strictly straddles t0
__global__ void k_post_slice(const __grid_constant__ PostArgs A) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (i64)gridDim.x * blockDim.x) {
    const ftk_cp a = A.rec[i];
    if (a.t == A.t0) post_emit(A, a);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const long long j = A.nbr[2 * i + k];
      if (j <= i) continue;  // each segment once
      ftk_cp lo = a, hi = A.rec[j];
      if (lo.t > hi.t) {
        const ftk_cp tmp = lo;
        lo = hi;
        hi = tmp;
      }
      if (!(lo.t < A.t0 && A.t0 < hi.t)) continue;
      const double s = __ddiv_rn(__dsub_rn(A.t0, lo.t), __dsub_rn(hi.t, lo.t));
      ftk_cp r = __dsub_rn(A.t0, lo.t) <= __dsub_rn(hi.t, A.t0) ? lo : hi;  // type / id of the nearer end
      r.x = __dadd_rn(lo.x, __dmul_rn(s, __dsub_rn(hi.x, lo.x)));
      r.y = __dadd_rn(lo.y, __dmul_rn(s, __dsub_rn(hi.y, lo.y)));
      r.z = __dadd_rn(lo.z, __dmul_rn(s, __dsub_rn(hi.z, lo.z)));
      r.t = A.t0;
      r.flags = 0;
      post_emit(A, r);
    }
  }
}

// per-trajectory attributes: time extent and open ends, keyed by the root record (the one whose
// face id is the label)
__global__ void k_post_stats(const __grid_constant__ TrackParams P, const __grid_constant__ PostArgs A) {
  const u64 hm = table_mask(P);
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (i64)gridDim.x * blockDim.x) {
    const long long root = lookup(P, hm, A.rec[i].label);
    if (root < 0) {
      atomicAdd(&P.counters[CNT_INVARIANT], 1ull);
      continue;
    }
    const long long tb = __double_as_longlong(A.rec[i].t);
    atomicMin(reinterpret_cast<unsigned long long*>(&A.tmin[root]), (unsigned long long)tb);
    atomicMax(reinterpret_cast<unsigned long long*>(&A.tmax[root]), (unsigned long long)tb);
    if (A.nbr[2 * i] < 0 || A.nbr[2 * i + 1] < 0) atomicAdd(reinterpret_cast<unsigned long long*>(&A.nends[root]), 1ull);
  }
}

__global__ void k_post_stats_init(const __grid_constant__ PostArgs A) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (i64)gridDim.x * blockDim.x) {
    A.tmin[i] = 0x7fffffffffffffffll;
    A.tmax[i] = 0;
    A.nends[i] = 0;
  }
}

// filtering: keep the records of trajectories lasting >= dmin (and, with drop_loops, not
// loops -- a loop has no open end)
__global__ void k_post_filter(const __grid_constant__ TrackParams P, const __grid_constant__ PostArgs A) {
  const u64 hm = table_mask(P);
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (i64)gridDim.x * blockDim.x) {
    const long long root = lookup(P, hm, A.rec[i].label);
    if (root < 0) continue;
    const double dur = __dsub_rn(__longlong_as_double(A.tmax[root]), __longlong_as_double(A.tmin[root]));
    const bool loop = A.nends[root] == 0;
    if (dur >= A.dmin && !(A.drop_loops && loop)) post_emit(A, A.rec[i]);
  }
}

// type smoothing: walk half_window records along the trajectory on each side; when both
// sides are non-empty and every record seen has one type T != own, the record takes T.  The marks are
// computed from the unmodified types (newtype), then applied.
__global__ void k_post_smooth(const __grid_constant__ PostArgs A) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (i64)gridDim.x * blockDim.x) {
    const int own = A.rec[i].type;
    int T = -1, seen[2] = {0, 0};
    bool uniform = true;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      long long prev = i, cur = A.nbr[2 * i + side];
      for (int step = 0; step < A.half_window && cur >= 0 && cur != i; ++step) {
        const int ty = A.rec[cur].type;
        if (T < 0) T = ty;
        uniform = uniform && ty == T;
        ++seen[side];
        const long long a = A.nbr[2 * cur], b = A.nbr[2 * cur + 1];
        const long long nx = a == prev ? b : a;
        prev = cur;
        cur = nx;
      }
    }
    A.newtype[i] = (seen[0] > 0 && seen[1] > 0 && uniform && T != own) ? T : own;
  }
}

// simplification in time (R23).  A fold is a record whose two partners both lie
// strictly later or both strictly earlier in t (a pair is born or annihilates there); folds cut a
// trajectory into segments (fold to fold, both included).  A segment with folds on both ends, time
// extent (max t - min t) below tau and outer records (the partners of its folds outside it) of one
// type T is a short-lived excursion: its records take T; a fold, in two segments, takes T when the
// qualifying ones agree.  Each record walks its segment(s) along the trajectory, stopping as soon as the
// extent reaches tau (the extent only grows), so a walk visits the records within tau of it in time.
__device__ __forceinline__ bool post_is_fold(const PostArgs& A, long long i) {
  const long long a = A.nbr[2 * i], b = A.nbr[2 * i + 1];
  if (a < 0 || b < 0) return false;
  const double ti = A.rec[i].t, da = A.rec[a].t - ti, db = A.rec[b].t - ti;
  return (da > 0 && db > 0) || (da < 0 && db < 0);
}
// walk from record `from` (already in the segment, extent [lo, hi]) through `cur` to the next fold;
// returns the fold's outer record (-1: no fold before a trajectory end, back at `start`, or extent >= tau)
__device__ __forceinline__ long long post_to_fold(const PostArgs& A, long long start, long long from, long long cur,
                                                  double& lo, double& hi, long long& fold) {
  long long prev = from;
  while (true) {
    if (cur < 0 || cur == start) return -1;
    const double tc = A.rec[cur].t;
    lo = fmin(lo, tc);
    hi = fmax(hi, tc);
    if (!(hi - lo < A.tau)) return -1;
    const long long a = A.nbr[2 * cur], b = A.nbr[2 * cur + 1];
    const long long nx = a == prev ? b : a;
    if (post_is_fold(A, cur)) {
      fold = cur;
      return nx;
    }
    prev = cur;
    cur = nx;
  }
}
__global__ void k_post_simplify(const __grid_constant__ PostArgs A) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (i64)gridDim.x * blockDim.x) {
    const int own = A.rec[i].type;
    const double ti = A.rec[i].t;
    const long long n0 = A.nbr[2 * i], n1 = A.nbr[2 * i + 1];
    int T = -1;
    bool clash = false;
    if (post_is_fold(A, i)) {
      // two segments: one on each side, the other partner of i being the outer record at this end
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        double lo = ti, hi = ti;
        long long f;
        const long long o = post_to_fold(A, i, i, side ? n1 : n0, lo, hi, f);
        if (o < 0) continue;
        const int ta = A.rec[side ? n0 : n1].type, tb = A.rec[o].type;
        if (ta != tb) continue;
        if (T >= 0 && T != ta) clash = true;
        T = ta;
      }
    } else if (n0 >= 0 && n1 >= 0) {
      double lo = ti, hi = ti;
      long long f0 = -1, f1 = -1;
      const long long o0 = post_to_fold(A, i, i, n0, lo, hi, f0);
      const long long o1 = o0 < 0 ? -1 : post_to_fold(A, i, i, n1, lo, hi, f1);
      // (f0 == f1: a loop with a single fold, not cut into segments)
      if (o1 >= 0 && f0 != f1 && A.rec[o0].type == A.rec[o1].type) T = A.rec[o0].type;
    }
    A.newtype[i] = (T >= 0 && !clash) ? T : own;
  }
}

__global__ void k_post_apply_types(const __grid_constant__ PostArgs A, ftk_cp* rec) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (i64)gridDim.x * blockDim.x)
    rec[i].type = A.newtype[i];
}

}  // namespace trk

// ------------------------------------------------------------------------- post-processing launchers
int launch_post_adjacency(const TrackParams& P0, int ndim, const i64* ext, long long n, long long* nbr,
                          cudaStream_t stream) {
  using namespace trk;
  const int sms = num_sms(), threads = 256, blocks = sms * 8;
  TrackParams P = P0;
  P.prelinked = true;  // keep parent[]
  P.lookup_types = ~0ull;
  k_post_prep<<<blocks, threads, 0, stream>>>(P, n);
  FTK_CUDA_TRY(cudaGetLastError());
  k_clear<<<blocks, threads, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  k_hash_insert<<<blocks, threads, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  if (ndim == 2) {
    Geo<3> G;
    G.ext[0] = ext[0]; G.ext[1] = ext[1]; G.ext[2] = ext[3];
    G.stride[0] = 1; G.stride[1] = ext[0]; G.stride[2] = ext[0] * ext[1];
    k_verify<3, true><<<blocks, threads, 0, stream>>>(P, G, nbr);
  } else {
    Geo<4> G;
    G.ext[0] = ext[0]; G.ext[1] = ext[1]; G.ext[2] = ext[2]; G.ext[3] = ext[3];
    G.stride[0] = 1; G.stride[1] = ext[0]; G.stride[2] = ext[0] * ext[1]; G.stride[3] = ext[0] * ext[1] * ext[2];
    k_verify<4, true><<<blocks, threads, 0, stream>>>(P, G, nbr);
  }
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

int launch_post(const TrackParams& P, int op, const PostCall& c, cudaStream_t stream) {
  using namespace trk;
  const int sms = num_sms(), threads = 256, blocks = sms * 8;
  PostArgs A;
  A.rec = c.rec;
  A.nbr = c.nbr;
  A.n = c.n;
  A.out = c.out;
  A.cap = c.cap;
  A.count = c.count;
  A.tmin = c.scratch;
  A.tmax = c.scratch + c.n;
  A.nends = c.scratch + 2 * c.n;
  A.newtype = reinterpret_cast<int*>(c.scratch + 3 * c.n);
  A.t0 = c.t0;
  A.dmin = c.dmin;
  A.drop_loops = c.drop_loops;
  A.half_window = c.half_window;
  A.tau = c.tau;
  if (op == 0) {
    k_post_slice<<<blocks, threads, 0, stream>>>(A);
  } else if (op == 1) {
    k_post_stats_init<<<blocks, threads, 0, stream>>>(A);
    FTK_CUDA_TRY(cudaGetLastError());
    k_post_stats<<<blocks, threads, 0, stream>>>(P, A);
    FTK_CUDA_TRY(cudaGetLastError());
    k_post_filter<<<blocks, threads, 0, stream>>>(P, A);
  } else if (op == 3) {
    k_post_simplify<<<blocks, threads, 0, stream>>>(A);
    FTK_CUDA_TRY(cudaGetLastError());
    k_post_apply_types<<<blocks, threads, 0, stream>>>(A, c.rec_mut);
  } else {
    k_post_smooth<<<blocks, threads, 0, stream>>>(A);
    FTK_CUDA_TRY(cudaGetLastError());
    k_post_apply_types<<<blocks, threads, 0, stream>>>(A, c.rec_mut);
  }
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

int launch_export(const TrackParams& P, cudaStream_t stream) {
  using namespace trk;
  const int sms = num_sms();
  k_export<<<sms * 4, 256, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

int launch_relabel(ftk_cp* rec, i64 n, const long long* old_labels, const long long* new_labels, i64 nmap,
                   cudaStream_t stream) {
  using namespace trk;
  if (n <= 0 || nmap <= 0) return FTK_OK;
  const int sms = num_sms();
  k_relabel<<<sms * 4, 256, 0, stream>>>(rec, n, old_labels, new_labels, nmap);
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

int launch_track(const TrackParams& P, int ndim, const i64* ext, cudaStream_t stream) {
  using namespace trk;
  const int sms = num_sms();
  const int threads = 256, blocks = sms * 8;
  k_clear<<<blocks, threads, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  k_hash_insert<<<blocks, threads, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  k_edges<<<blocks, threads, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  for (int j = 0; j < FTK_LABEL_JUMP; ++j) k_jump<<<blocks, threads, 0, stream>>>(P);
  k_root<<<blocks, threads, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  k_label<<<blocks, threads, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  if (P.verify) {
    if (ndim == 2) {
      Geo<3> G;
      G.ext[0] = ext[0]; G.ext[1] = ext[1]; G.ext[2] = ext[3];
      G.stride[0] = 1; G.stride[1] = ext[0]; G.stride[2] = ext[0] * ext[1];
      k_verify<3><<<blocks, threads, 0, stream>>>(P, G);
    } else {
      Geo<4> G;
      G.ext[0] = ext[0]; G.ext[1] = ext[1]; G.ext[2] = ext[2]; G.ext[3] = ext[3];
      G.stride[0] = 1; G.stride[1] = ext[0]; G.stride[2] = ext[0] * ext[1]; G.stride[3] = ext[0] * ext[1] * ext[2];
      k_verify<4><<<blocks, threads, 0, stream>>>(P, G);
    }
    FTK_CUDA_TRY(cudaGetLastError());
  }
  return FTK_OK;
}

int launch_seam_pack(const TrackParams& P, long long* block, long long cap, cudaStream_t stream) {
  using namespace trk;
  k_seam_pack<<<num_sms() * 2, 256, 0, stream>>>(P, block, cap);
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

int launch_seam_resolve(const long long* all, int world, long long cap, const SeamScratch& S, ftk_cp* d_out,
                        long long n, cudaStream_t stream) {
  using namespace trk;
  SeamArgs A{all, world, cap, S, d_out, n};
  const int blocks = num_sms() * 2;
  k_seam_clear<<<blocks, 256, 0, stream>>>(A);
  FTK_CUDA_TRY(cudaGetLastError());
  k_seam_insert<<<blocks, 256, 0, stream>>>(A);
  FTK_CUDA_TRY(cudaGetLastError());
  k_seam_union<<<blocks, 256, 0, stream>>>(A);
  FTK_CUDA_TRY(cudaGetLastError());
  k_seam_relabel<<<num_sms() * 4, 256, 0, stream>>>(A);
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

}  // namespace ftk
