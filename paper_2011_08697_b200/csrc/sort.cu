// sort.cu -- FTK_SORTED (include/ftk_cp.h): the records of a call reordered by face_id, on the device.
//
// The record SET is deterministic but K1b appends records in scheduling order; a caller that asks for
// FTK_SORTED gets them in face-id order (SURVEY.md 8(b) "Determinism").  Face ids are unique, so the
// order is a total one.  Hand-written LSD radix sort of (face id, record index) pairs by 8-bit digits
// over the key's significant bits (the largest face id of the descriptor fixes them: 32 bits for C2,
// 37 for C4), then one gather of the 56-byte records:
//
//   k_rs_hist     per tile of TILE pairs, the 256-bin histogram of the digit  -> hist[digit][tile]
//   k_rs_scan     per digit, exclusive scan over the tiles; digit totals     -> tile offsets
//   k_rs_scatter  stable ranks inside the tile (warp match + per-warp counts in shared memory, in
//                 index order), pairs written to offset[digit][tile] + rank
//   k_rs_gather   records[i] = old_records[index[i]] (through a scratch copy)
//
// Every pass is stable, so after the last digit the pairs are in face-id order.  Scratch comes from
// the call's workspace regions that are dead once labels are final (edges, stitch lists, relabel map).
#include <algorithm>
#include <utility>

#include "common.cuh"
#include "sort.cuh"

namespace ftk {
namespace rsort {

constexpr int THREADS = 256;
constexpr int ITEMS = 8;
constexpr int TILE = THREADS * ITEMS;
constexpr int WARPS = THREADS / 32;

__device__ __forceinline__ int digit_of(unsigned long long k, int shift) { return (int)((k >> shift) & 255u); }

__global__ void __launch_bounds__(THREADS) k_rs_hist(const unsigned long long* keys, long long n, int shift,
                                                      int ntiles, unsigned int* hist) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * TILE;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const long long j = base + i * THREADS + threadIdx.x;
    if (j < n) atomicAdd(&h[digit_of(keys[j], shift)], 1u);
  }
  __syncthreads();
  hist[(long long)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// per digit (one block each): exclusive scan of the digit's tile counts in place, digit total -> dtot
__global__ void __launch_bounds__(1024) k_rs_scan(unsigned int* hist, int ntiles, unsigned int* dtot) {
  __shared__ unsigned int wsum[32];
  __shared__ unsigned int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  unsigned int* h = hist + (long long)blockIdx.x * ntiles;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c0 = 0; c0 < ntiles; c0 += 1024) {
    const int j = c0 + threadIdx.x;
    const unsigned int v = j < ntiles ? h[j] : 0u;
    unsigned int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      unsigned int s = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      wsum[lane] = s;  // inclusive prefix of the warp sums
    }
    __syncthreads();
    if (j < ntiles) h[j] = carry + (w ? wsum[w - 1] : 0u) + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) dtot[blockIdx.x] = carry;
}

__global__ void __launch_bounds__(THREADS) k_rs_scatter(const unsigned long long* kin, const int* vin,
                                                         unsigned long long* kout, int* vout, long long n,
                                                         int shift, int ntiles, const unsigned int* offs,
                                                         const unsigned int* dtot) {
  __shared__ unsigned int base[256];        // running position per digit for this tile's items
  __shared__ unsigned int wcnt[WARPS][256];  // this round's count per warp and digit
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  {  // digit base = exclusive prefix of the digit totals (256 values, one per thread)
    const unsigned int v = dtot[threadIdx.x];
    unsigned int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wcnt[0][w] = x;
    __syncthreads();
    unsigned int pre = 0;
    for (int q = 0; q < w; ++q) pre += wcnt[0][q];
    base[threadIdx.x] = pre + x - v + offs[(long long)threadIdx.x * ntiles + blockIdx.x];
    __syncthreads();
  }
  const long long t0 = (long long)blockIdx.x * TILE;
  const unsigned int lt = (1u << lane) - 1u;
  for (int i = 0; i < ITEMS; ++i) {
    // round i covers tile items [i * THREADS, (i + 1) * THREADS) in index order: warp-major, lane-minor
    const long long j = t0 + i * THREADS + threadIdx.x;
    const bool ok = j < n;
    const unsigned long long k = ok ? kin[j] : 0ull;
    const int v = ok ? vin[j] : 0;
    const int d = ok ? digit_of(k, shift) : 256 + lane;  // out-of-range items match nobody
#pragma unroll
    for (int q = 0; q < WARPS; ++q) wcnt[q][threadIdx.x] = 0;
    __syncthreads();
    const unsigned int peers = __match_any_sync(0xffffffffu, d);
    const unsigned int before_in_warp = __popc(peers & lt);
    if (ok && before_in_warp == 0) wcnt[w][d] = __popc(peers);
    __syncthreads();
    // per digit: the ranks of this round's warps follow the earlier rounds' items
    {
      unsigned int run = base[threadIdx.x];
#pragma unroll
      for (int q = 0; q < WARPS; ++q) {
        const unsigned int c = wcnt[q][threadIdx.x];
        wcnt[q][threadIdx.x] = run;
        run += c;
      }
      base[threadIdx.x] = run;
    }
    __syncthreads();
    if (ok) {
      const unsigned int pos = wcnt[w][d] + before_in_warp;
      FTK_ASSERT(pos < (unsigned long long)n);
      kout[pos] = k;
      vout[pos] = v;
    }
    __syncthreads();
  }
}

__global__ void k_rs_init(const long long* fid, unsigned long long* keys, int* vals, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    keys[i] = (unsigned long long)fid[i];
    vals[i] = (int)i;
  }
}

__global__ void k_rs_copy(const ftk_cp* __restrict__ src, ftk_cp* __restrict__ dst, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_rs_gather(const ftk_cp* __restrict__ src, const int* __restrict__ idx, ftk_cp* __restrict__ dst,
                            long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

}  // namespace rsort

int launch_sort_records(ftk_cp* rec, const long long* fid, long long n, int key_bits, const SortScratch& S,
                        cudaStream_t stream) {
  using namespace rsort;
  if (n <= 1) return FTK_OK;
  const int ntiles = (int)((n + TILE - 1) / TILE);
  const int grid = (int)std::min<long long>((n + 255) / 256, 148 * 16);
  unsigned long long *ka = S.keys0, *kb = S.keys1;
  int *va = S.vals0, *vb = S.vals1;
  k_rs_init<<<grid, 256, 0, stream>>>(fid, ka, va, n);
  FTK_CUDA_TRY(cudaGetLastError());
  for (int shift = 0; shift < key_bits; shift += 8) {
    k_rs_hist<<<ntiles, THREADS, 0, stream>>>(ka, n, shift, ntiles, S.hist);
    FTK_CUDA_TRY(cudaGetLastError());
    k_rs_scan<<<256, 1024, 0, stream>>>(S.hist, ntiles, S.dtot);
    FTK_CUDA_TRY(cudaGetLastError());
    k_rs_scatter<<<ntiles, THREADS, 0, stream>>>(ka, va, kb, vb, n, shift, ntiles, S.hist, S.dtot);
    FTK_CUDA_TRY(cudaGetLastError());
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  k_rs_copy<<<grid, 256, 0, stream>>>(rec, S.rec_tmp, n);
  FTK_CUDA_TRY(cudaGetLastError());
  k_rs_gather<<<grid, 256, 0, stream>>>(S.rec_tmp, va, rec, n);
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

}  // namespace ftk

namespace ftk {

static size_t al256(size_t v) { return (v + 255) / 256 * 256; }

size_t sort_scratch_bytes(long long n) {
  const long long ntiles = (n + rsort::TILE - 1) / rsort::TILE;
  return 2 * al256(8 * (size_t)n) + 2 * al256(4 * (size_t)n) + al256(4 * 256 * (size_t)ntiles) + al256(1024) +
         al256(sizeof(ftk_cp) * (size_t)n);
}

SortScratch sort_scratch(void* base, long long n) {
  const long long ntiles = (n + rsort::TILE - 1) / rsort::TILE;
  char* p = static_cast<char*>(base);
  SortScratch S;
  S.keys0 = reinterpret_cast<unsigned long long*>(p);
  p += al256(8 * (size_t)n);
  S.keys1 = reinterpret_cast<unsigned long long*>(p);
  p += al256(8 * (size_t)n);
  S.vals0 = reinterpret_cast<int*>(p);
  p += al256(4 * (size_t)n);
  S.vals1 = reinterpret_cast<int*>(p);
  p += al256(4 * (size_t)n);
  S.hist = reinterpret_cast<unsigned int*>(p);
  p += al256(4 * 256 * (size_t)ntiles);
  S.dtot = reinterpret_cast<unsigned int*>(p);
  p += al256(1024);
  S.rec_tmp = reinterpret_cast<ftk_cp*>(p);
  return S;
}

}  // namespace ftk
