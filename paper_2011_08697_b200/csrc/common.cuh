// common.cuh -- device/host helpers shared by the FTK B200 kernels (product path only).
//
// Nothing here is shared with oracle/ (the CPU oracle is independent test infrastructure).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ftk_cp.h"

// Debug builds (-DFTK_CHECKS=1, paper_2011_08697_b200/build.py variant "checks"): device-side bounds
// and protocol assertions -- the stand-in for compute-sanitizer, which this pool does not run.  A failed
// check prints its location and traps (the call returns FTK_ERR_CUDA).  Compiled out otherwise.
#ifndef FTK_CHECKS
#define FTK_CHECKS 0
#endif
#if FTK_CHECKS
#include <cstdio>
#define FTK_ASSERT(cond)                                                                              \
  do {                                                                                                \
    if (!(cond)) {                                                                                    \
      printf("FTK_ASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, blockIdx.x, \
             threadIdx.x);                                                                            \
      __trap();                                                                                       \
    }                                                                                                 \
  } while (0)
#else
#define FTK_ASSERT(cond) \
  do {                   \
  } while (0)
#endif

namespace ftk {

using i64 = long long;
using u64 = unsigned long long;
using i128 = __int128;
using u128 = unsigned __int128;

// Workspace counters (u64 each), zeroed at the start of every call.
enum Counter : int {
  CNT_NOUT = 0,       // punctured faces found (may exceed capacity)
  CNT_SURVIVORS = 1,  // cubes surviving the sign prefilter
  CNT_MAXBITS = 2,    // max over |f| as IEEE bits (float bits for f32, double bits for f64)
  CNT_INVARIANT = 3,  // link: faces whose parent cell does not hold exactly one other punctured face
  CNT_EXPORT = 4,     // slab stitch: exported cross pairs (A list)
  CNT_WORK = 5,       // K1 persistent scheduler: next work item
  CNT_EDGES = 6,      // trajectory-graph edges emitted by K1 (one per cell holding two punctured faces)
  CNT_CROSS = 7,      // slab stitch: edges whose partner face lies on the ghost plane
  CNT_EXPORT_B = 8,   // slab stitch: own ordinal faces on the first owned plane
  CNT_WIN = 9,        // K1a: survivor-list entries reserved (2D: group entries; chunks of FTK_K1_CHUNK; may exceed wcap)
  CNT_HMASK = 10,     // pass 2: hash-table slot mask in use (set before the first insert)
  CNT_CUBES = 11,     // 2D: surviving cubes expanded from K1a's group entries (may exceed wcap)
  CNT_WIN_MAX = 12,   // streaming: max of CNT_WIN / CNT_CUBES over the chunks already processed
  CNT_POST = 13,      // post-processing: output records (slice / filter)
  CNT_HGROUP = 14,    // pass 2: log2 of the hash-table blocks per coarse cell (set with CNT_HMASK)
  CNT_ELEMS = 15,     // isovolume mesh: simplices emitted (may exceed the element capacity)
  CNT_PROF = 16,      // 16..25 : optional K1 cycle accounting (FTK_K1_PROF builds)
  CNT_XBATCH = 26,    // 2D K1b: next cube batch to claim (dynamic batch assignment)
  CNT_N = 32
};

// Correctly rounded (round-half-even) int128 -> double; the oracle's reading of step 5
// (R11) -- implemented independently with 64-bit conversions plus a sticky bit.
__device__ __forceinline__ double i128_to_double_rn(i128 v) {
  if (v == (i128)(i64)v) return __ll2double_rn((i64)v);
  const bool neg = v < 0;
  u128 m = neg ? (u128)0 - (u128)v : (u128)v;
  const u64 hi = (u64)(m >> 64);
  double d;
  if (hi == 0) {
    d = __ull2double_rn((u64)m);
  } else {
    const int k = 64 - __clzll((i64)hi);         // shift so the leading bit lands at bit 63
    const u64 w = (u64)(m >> k);
    const u64 sticky = ((m & (((u128)1 << k) - 1)) != 0) ? 1ull : 0ull;
    d = __ull2double_rn(w | sticky);              // bit 0 is below the round bit (bit 10)
    d = ldexp(d, k);                              // exact power-of-two scaling
  }
  return neg ? -d : d;
}

__device__ __forceinline__ int sgn128(i128 v) { return (v > 0) - (v < 0); }
__device__ __forceinline__ int sgn64(i64 v) { return (v > 0) - (v < 0); }

// Hash of a face id for the pass-2 table (face id -> record index; open addressing, linear probing).
__host__ __device__ __forceinline__ u64 hash_mix(u64 k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}
// slots for up to n keys: nextpow2(1.5 n), at least 1024, at most cap (a power of two)
__host__ __device__ __forceinline__ u64 hash_slots(long long n, u64 cap) {
  u64 h = 1024;
  while (h < (u64)(n + n / 2) && h < cap) h <<= 1;
  return h;
}

// Exact 2x2 determinant | ua va ; ub vb | in int128.
__device__ __forceinline__ i128 det2(i64 ua, i64 va, i64 ub, i64 vb) {
  return (i128)ua * vb - (i128)va * ub;
}

}  // namespace ftk

#define FTK_CUDA_TRY(expr)                                   \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return ::ftk::set_cuda_error(_e, #expr); \
  } while (0)

namespace ftk {
int set_cuda_error(cudaError_t e, const char* what);  // runtime.cu
}
