// track.cu -- pass 2 of Alg. 1: join the punctured faces of every cell.
//
// Instead of visiting all cells, every punctured face visits its (at most two) parent cells in
// closed form (side_of) and looks up the cell's other d faces in a
// GPU hash table of punctured face ids.  Under SoS each cell holds 0 or 2 punctured faces
// (PAPER.md:437, 467), so a face finds exactly one partner per existing parent cell; anything
// else is counted as an invariant violation.
//
// Union-find (K5/K6, north_star (4)): lock-free hooking with atomicCAS, the root with the larger
// face_id is hooked under the smaller one, then path compression; every component's final root
// is its minimum face_id, which becomes the trajectory label -- independent of scheduling.
#include <utility>

#include "common.cuh"
#include "kuhn.cuh"
#include "track.cuh"

namespace ftk {
namespace trk {

constexpr i64 EMPTY = -1;

__constant__ KuhnTables<3> cK3 = kKuhn3;
__constant__ KuhnTables<4> cK4 = kKuhn4;

__device__ __forceinline__ u64 mix(u64 k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

__device__ __forceinline__ i64 n_records(const TrackParams& P) {
  const i64 n = (i64)P.counters[CNT_NOUT];
  return n < P.capacity ? n : P.capacity;
}

__global__ void k_hash_insert(const __grid_constant__ TrackParams P) {
  const i64 n = n_records(P);
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i64 key = P.rec[i].face_id;
    P.fid[i] = key;
    P.parent[i] = (int)i;
    u64 h = mix((u64)key) & P.hmask;
    while (true) {
      const i64 prev = (i64)atomicCAS(reinterpret_cast<u64*>(&P.keys[h]), (u64)EMPTY, (u64)key);
      if (prev == EMPTY || prev == key) {
        P.vals[h] = (int)i;
        break;
      }
      h = (h + 1) & P.hmask;
    }
  }
}

__device__ __forceinline__ int lookup(const TrackParams& P, i64 key) {
  u64 h = mix((u64)key) & P.hmask;
  while (true) {
    const i64 k = P.keys[h];
    if (k == key) return P.vals[h];
    if (k == EMPTY) return -1;
    h = (h + 1) & P.hmask;
  }
}

__device__ __forceinline__ int uf_find(int* parent, int i) {
  while (true) {
    const int p = parent[i];
    if (p == i) return i;
    const int gp = parent[p];
    if (gp != p) parent[i] = gp;  // path halving; benign race (pointers only move to smaller keys)
    i = p;
  }
}

__device__ __forceinline__ void uf_unite(int* parent, const i64* key, int a, int b) {
  while (true) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    if (key[a] < key[b]) {
      const int t = a;
      a = b;
      b = t;
    }
    // a has the larger key: hook it under b
    const int old = atomicCAS(&parent[a], a, b);
    if (old == a) return;
  }
}

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

// Visit one parent cell given as a chain of D+1 cumulative masks w[0..D] relative to anchor A;
// return the number of OTHER punctured faces found and the last one's index.
template <int D>
__device__ __forceinline__ int visit_cell(const TrackParams& P, const Geo<D>& G, const i64* A, const int* w,
                                          i64 self, int& partner) {
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
    const int r = lookup(P, f);
    if (r >= 0) {
      ++hits;
      partner = r;
    }
  }
  return hits;
}

template <int D>
__global__ void k_link(const __grid_constant__ TrackParams P, const Geo<D> G) {
  const i64 n = n_records(P);
  constexpr int FULL = (1 << D) - 1;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i64 self = P.fid[i];
    i64 v[4];
    int type;
    decode<D>(G, self, v, type);
    int m[4] = {0, 0, 0, 0};  // m[1..D-1]
#pragma unroll
    for (int k = 1; k < D; ++k) m[k] = D == 3 ? cK3.masks[type][k - 1] : cK4.masks[type][k - 1];
    const int U = m[D - 1];
    int bad = 0;
    if (U != FULL) {
      const int cbit = FULL & ~U;
      const int c = __ffs(cbit) - 1;
      // parent 1: append v_last + e_c (same anchor), exists iff v0[c] <= N_c - 2
      if (v[c] + 1 <= G.ext[c] - 1) {
        int w[5];
        w[0] = 0;
#pragma unroll
        for (int k = 1; k < D; ++k) w[k] = m[k];
        w[D] = FULL;
        int partner = -1;
        const int h = visit_cell<D>(P, G, v, w, self, partner);
        if (h != 1) bad = 1;
        else if (P.fid[partner] > self) uf_unite(P.parent, P.fid, (int)i, partner);
      }
      // parent 2: prepend v0 - e_c (anchor moves down), exists iff v0[c] >= 1
      if (v[c] >= 1) {
        i64 A[4];
#pragma unroll
        for (int a = 0; a < D; ++a) A[a] = v[a] - (a == c ? 1 : 0);
        int w[5];
        w[0] = 0;
#pragma unroll
        for (int k = 1; k <= D; ++k) w[k] = cbit | m[k - 1];
        int partner = -1;
        const int h = visit_cell<D>(P, G, A, w, self, partner);
        if (h != 1) bad = 1;
        else if (P.fid[partner] > self) uf_unite(P.parent, P.fid, (int)i, partner);
      }
    } else {
      // the face spans all axes: exactly one step has two axes {a, b}; the two parent cells
      // split it as a-then-b and b-then-a, same anchor, both always exist
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
        w[D] = m[D - 1];
        // rebuild: chain = m0, ..., m_{step-1}, m_{step-1}|x, m_step, ..., m_{D-1}
        int partner = -1;
        const int h = visit_cell<D>(P, G, v, w, self, partner);
        if (h != 1) bad = 1;
        else if (P.fid[partner] > self) uf_unite(P.parent, P.fid, (int)i, partner);
      }
    }
    if (bad) atomicAdd(&P.counters[CNT_INVARIANT], 1ull);
  }
}

__global__ void k_label(const __grid_constant__ TrackParams P) {
  const i64 n = n_records(P);
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const int r = uf_find(P.parent, (int)i);
    P.rec[i].label = P.fid[r];
  }
}

}  // namespace trk

int launch_track(const TrackParams& P, int ndim, const i64* ext, cudaStream_t stream) {
  using namespace trk;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 256, blocks = sms * 8;
  FTK_CUDA_TRY(cudaMemsetAsync(P.keys, 0xff, (size_t)(P.hmask + 1) * sizeof(i64), stream));
  k_hash_insert<<<blocks, threads, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  if (ndim == 2) {
    Geo<3> G;
    G.ext[0] = ext[0]; G.ext[1] = ext[1]; G.ext[2] = ext[3];
    G.stride[0] = 1; G.stride[1] = ext[0]; G.stride[2] = ext[0] * ext[1];
    k_link<3><<<blocks, threads, 0, stream>>>(P, G);
  } else {
    Geo<4> G;
    G.ext[0] = ext[0]; G.ext[1] = ext[1]; G.ext[2] = ext[2]; G.ext[3] = ext[3];
    G.stride[0] = 1; G.stride[1] = ext[0]; G.stride[2] = ext[0] * ext[1]; G.stride[3] = ext[0] * ext[1] * ext[2];
    k_link<4><<<blocks, threads, 0, stream>>>(P, G);
  }
  FTK_CUDA_TRY(cudaGetLastError());
  k_label<<<blocks, threads, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

}  // namespace ftk
