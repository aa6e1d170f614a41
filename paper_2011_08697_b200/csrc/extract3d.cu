// extract3d.cu -- K1 for 3D+t (4D spacetime, faces = tetrahedra, cells = pentachora).
//
// Pass 1 of Alg. 1 (generalised at P:439) plus the per-hypercube cell evaluation of
// pass 2.  A CTA owns a 32 x 4 x 2 block of anchors (x, y, z) and marches t over a chunk; each plane
// tile with its halo (x-1..x+33, y-1..y+5, z-1..z+3) is staged in shared memory (double buffered), so
// every vertex is read from HBM once per CTA and its neighbours come from shared memory.
//
//   prefilter: per vertex a 6-bit code, bit = 1 when a strict sign condition does NOT hold:
//     (dx >= thr), (dx <= -thr), (dy >= thr), (dy <= -thr), (dz >= thr), (dz <= -thr) on raw values,
//     thr = 2^(1-s), which implies the exact integer gradient component is strictly positive/negative
//     (DESIGN.md "prefilter").  ORed over the 16 corners of the spacetime hypercube; a code with all
//     six bits set survives (no gradient component is one-signed on every corner).
//   exact stage (survivors, one per thread): int64 gradients, the 60 face types with exact 3x3
//     determinants (int128) and the SoS epsilon-expansion of det(M + E) evaluated term by term in
//     decreasing magnitude (R4/R5), Eq. 2 location and the Descartes-rule
//     Hessian type in fixed-order FP64, and the 24 cells (pentachora) of the hypercube: 0 or 2
//     punctured sides each, emitted as trajectory edges.
#include <cstdio>
#include <cstring>
#include <utility>

#include "common.cuh"
#include "extract2d.cuh"
#include "kuhn.cuh"

namespace ftk {
namespace k3d {

constexpr int TX = 32, TY = 4, TZ = 2;          // anchors per CTA
constexpr int NT = TX * TY * TZ;                // threads (one anchor each)
constexpr int SX = TX + 3, SY = TY + 3, SZ = TZ + 3;  // tile with halo: x-1 .. x+TX+1
constexpr int SV = SX * SY * SZ;
constexpr int CX = TX + 1, CY = TY + 1, CZ = TZ + 1;  // vertex codes: x .. x+TX
constexpr int TCH = 16;                         // anchor timesteps per work item
constexpr int CHUNK3 = 32;                      // survivor-list entries a warp reserves at a time

__constant__ KuhnTables<4> cK4 = kKuhn4;

// ------------------------------------------------------------------------------ SoS, 3x3
// Partial permutations of a 3x3 matrix: the epsilon-monomials prod_{r in R} eps_{r, sigma(r)} of
// det(M + E), eps_{r,j} = eps^(2^(3r + j)); sorted by exponent = decreasing magnitude.  The empty
// sigma (the determinant itself) comes first; a full permutation has coefficient +-1.
struct PP3 {
  int n;
  int8_t col[34][3];
};
constexpr PP3 make_pp3() {
  PP3 t{};
  int keys[34] = {};
  int n = 0;
  for (int code = 0; code < 64; ++code) {
    int c[3] = {code % 4 - 1, (code / 4) % 4 - 1, (code / 16) % 4 - 1};
    bool ok = true;
    int key = 0;
    for (int r = 0; r < 3 && ok; ++r)
      if (c[r] >= 0) {
        for (int q = 0; q < r; ++q)
          if (c[q] == c[r]) ok = false;
        key |= 1 << (3 * r + c[r]);
      }
    if (!ok) continue;
    int pos = n;  // insertion sort by key
    while (pos > 0 && keys[pos - 1] > key) {
      keys[pos] = keys[pos - 1];
      for (int r = 0; r < 3; ++r) t.col[pos][r] = t.col[pos - 1][r];
      --pos;
    }
    keys[pos] = key;
    for (int r = 0; r < 3; ++r) t.col[pos][r] = (int8_t)c[r];
    ++n;
  }
  t.n = n;
  return t;
}
__constant__ PP3 cPP3 = make_pp3();
static_assert(make_pp3().n == 34, "34 monomials for 3x3");

__device__ __forceinline__ i128 det3(const i64* a, const i64* b, const i64* c) {
  return (i128)a[0] * ((i128)b[1] * c[2] - (i128)b[2] * c[1]) - (i128)a[1] * ((i128)b[0] * c[2] - (i128)b[2] * c[0]) +
         (i128)a[2] * ((i128)b[0] * c[1] - (i128)b[1] * c[0]);
}

// SoS sign of det of the row-sorted matrix rows[0..2] given the sign of the exact determinant
__device__ __noinline__ int sos3_chain(const i64* r0, const i64* r1, const i64* r2) {
  const i64* R[3] = {r0, r1, r2};
  constexpr int PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  constexpr int PSGN[6] = {1, -1, -1, 1, 1, -1};
  for (int i = 1; i < cPP3.n; ++i) {  // i = 0 is the exact determinant (already zero)
    i128 sum = 0;
    for (int p = 0; p < 6; ++p) {
      bool ok = true;
      i128 prod = PSGN[p];
      for (int r = 0; r < 3; ++r) {
        const int c = cPP3.col[i][r];
        if (c >= 0) {
          if (PERM[p][r] != c) ok = false;
        } else {
          prod *= (i128)R[r][PERM[p][r]];
        }
      }
      if (ok) sum += prod;
    }
    if (sum != 0) return sum > 0 ? 1 : -1;
  }
  return 1;  // unreachable
}

__device__ __forceinline__ int sos3(const i64* r0, const i64* r1, const i64* r2) {
  const i128 d = det3(r0, r1, r2);
  if (d != 0) return d > 0 ? 1 : -1;
  return sos3_chain(r0, r1, r2);
}

// ------------------------------------------------------------------------------ geometry
struct Geo3 {
  i64 nx, ny, nz, ntg;
  i64 x0, y0, z0;
  float scale_f;
  double scale;
};

template <typename T>
struct Tile {  // staged plane tile, value at global (x, y, z)
  const T* S;
  __device__ __forceinline__ T at(const Geo3& G, i64 x, i64 y, i64 z) const {
    return S[((int)(z - G.z0 + 1) * SY + (int)(y - G.y0 + 1)) * SX + (int)(x - G.x0 + 1)];
  }
};

template <typename T>
struct GTile {  // a plane of the field in global memory, value at global (x, y, z) (in the grid)
  const T* S;
  __device__ __forceinline__ T at(const Geo3& G, i64 x, i64 y, i64 z) const { return __ldg(S + (z * G.ny + y) * G.nx + x); }
};

template <typename T>
__device__ __forceinline__ i64 quant3(T f, const Geo3& G) {
  if constexpr (sizeof(T) == 4) return __float2ll_rn(__fmul_rn(f, G.scale_f));
  else return __double2ll_rn(__dmul_rn(f, G.scale));
}

// exact gradient (2x derivative, one-sided doubled at the boundary) at vertex (x, y, z) of a tile
template <typename T, typename Acc>
__device__ void grad3(const Acc& P, const Geo3& G, i64 x, i64 y, i64 z, i64* g) {
  const i64 N[3] = {G.nx, G.ny, G.nz};
  const i64 c[3] = {x, y, z};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    i64 lo[3] = {x, y, z}, hi[3] = {x, y, z};
    i64 f = 1;
    if (c[a] == 0) { hi[a] = 1; lo[a] = 0; f = 2; }
    else if (c[a] == N[a] - 1) { hi[a] = N[a] - 1; lo[a] = N[a] - 2; f = 2; }
    else { hi[a] = c[a] + 1; lo[a] = c[a] - 1; }
    g[a] = f * (quant3(P.at(G, hi[0], hi[1], hi[2]), G) - quant3(P.at(G, lo[0], lo[1], lo[2]), G));
  }
}

// integer Hessian (4x scale, centre clamped into [1, N-2]) from global memory; order xx xy xz yy yz zz
template <typename T>
__device__ void hess3(const ExtractParams& P, const Geo3& G, i64 x, i64 y, i64 z, i64 t, i64* H) {
  const T* base = reinterpret_cast<const T*>(P.field) + (t - P.t0) * G.nx * G.ny * G.nz;
  auto q = [&](i64 xx, i64 yy, i64 zz) { return quant3(base[(zz * G.ny + yy) * G.nx + xx], G); };
  const i64 N[3] = {G.nx, G.ny, G.nz};
  const i64 c[3] = {x, y, z};
  int k = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b) {
      i64 cc[3] = {c[0], c[1], c[2]};
      cc[a] = cc[a] < 1 ? 1 : (cc[a] > N[a] - 2 ? N[a] - 2 : cc[a]);
      cc[b] = cc[b] < 1 ? 1 : (cc[b] > N[b] - 2 ? N[b] - 2 : cc[b]);
      if (a == b) {
        i64 p[3] = {cc[0], cc[1], cc[2]}, m[3] = {cc[0], cc[1], cc[2]};
        p[a] += 1;
        m[a] -= 1;
        H[k++] = 4 * (q(p[0], p[1], p[2]) - 2 * q(cc[0], cc[1], cc[2]) + q(m[0], m[1], m[2]));
      } else {
        i64 pp[3] = {cc[0], cc[1], cc[2]}, pm[3] = {cc[0], cc[1], cc[2]}, mp[3] = {cc[0], cc[1], cc[2]},
            mm[3] = {cc[0], cc[1], cc[2]};
        pp[a] += 1; pp[b] += 1;
        pm[a] += 1; pm[b] -= 1;
        mp[a] -= 1; mp[b] += 1;
        mm[a] -= 1; mm[b] -= 1;
        H[k++] = q(pp[0], pp[1], pp[2]) - q(pm[0], pm[1], pm[2]) - q(mp[0], mp[1], mp[2]) + q(mm[0], mm[1], mm[2]);
      }
    }
}

__device__ __forceinline__ double dot4_nofma(const double* mu, const double* v) {
  return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(mu[0], v[0]), __dmul_rn(mu[1], v[1])), __dmul_rn(mu[2], v[2])),
                   __dmul_rn(mu[3], v[3]));
}

// punctured test of a face with vertex gradients g[0..3] (rows in global vertex order):
// s_k = (-1)^(k+3) sos(rows != k), all equal
__device__ __forceinline__ bool punctured4(const i64 (&g)[4][3]) {
  const int s0 = -sos3(g[1], g[2], g[3]);
  const int s1 = sos3(g[0], g[2], g[3]);
  if (s0 != s1) return false;
  const int s2 = -sos3(g[0], g[1], g[3]);
  if (s0 != s2) return false;
  const int s3 = sos3(g[0], g[1], g[2]);
  return s0 == s3;
}

// type from the interpolated Hessian (R9): Descartes' rule of signs on the characteristic
// polynomial det(lambda I - H) = lambda^3 - c2 lambda^2 + c1 lambda - c0
__device__ __forceinline__ int classify3(const double* h) {
  const double a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5];
  const double c2 = __dadd_rn(__dadd_rn(a, d), f);
  const double c1 = __dadd_rn(__dadd_rn(__dsub_rn(__dmul_rn(a, d), __dmul_rn(b, b)), __dsub_rn(__dmul_rn(a, f), __dmul_rn(c, c))),
                              __dsub_rn(__dmul_rn(d, f), __dmul_rn(e, e)));
  const double c0 = __dadd_rn(__dsub_rn(__dmul_rn(a, __dsub_rn(__dmul_rn(d, f), __dmul_rn(e, e))),
                                        __dmul_rn(b, __dsub_rn(__dmul_rn(b, f), __dmul_rn(c, e)))),
                              __dmul_rn(c, __dsub_rn(__dmul_rn(b, e), __dmul_rn(c, d))));
  if (c0 == 0) return FTK_CP_DEGENERATE;
  const double seq[4] = {1.0, -c2, c1, -c0};
  int changes = 0, last = 1;
#pragma unroll
  for (int i = 1; i < 4; ++i) {
    if (seq[i] == 0) continue;
    const int sg = seq[i] > 0 ? 1 : -1;
    if (sg != last) ++changes;
    last = sg;
  }
  return changes == 3 ? FTK_CP_MIN : changes == 2 ? FTK_CP_SADDLE1 : changes == 1 ? FTK_CP_SADDLE2 : FTK_CP_MAX;
}

// The 24 cells (pentachora) of a hypercube: axis permutations (p1..p4) of {x=1, y=2, z=4, t=8};
// chain w0 = 0, w_k = w_{k-1} | p_k.  Dropping w1..w4 leaves own faces; dropping w0 leaves the upper
// face (w1, w2, w3, 15) owned by the neighbour hypercube anchored at v + p1.
struct Cell4 {
  int8_t own[4];   // face types of the faces dropping w4, w3, w2, w1
  int8_t w[5];     // chain masks
  int8_t up_type;  // type of the upper face relative to v + p1
};
struct Cells4 {
  Cell4 c[24];
};
constexpr int type4(int a, int b, int c) { return kKuhn4.type_of[a | b << 4 | c << 8]; }
constexpr Cells4 make_cells4() {
  Cells4 t{};
  int n = 0;
  const int ax[4] = {1, 2, 4, 8};
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      for (int k = 0; k < 4; ++k)
        for (int l = 0; l < 4; ++l) {
          if (i == j || i == k || i == l || j == k || j == l || k == l) continue;
          const int w1 = ax[i], w2 = w1 | ax[j], w3 = w2 | ax[k], w4 = 15;
          Cell4& c = t.c[n++];
          c.w[0] = 0; c.w[1] = (int8_t)w1; c.w[2] = (int8_t)w2; c.w[3] = (int8_t)w3; c.w[4] = (int8_t)w4;
          c.own[0] = (int8_t)type4(w1, w2, w3);   // drop w4
          c.own[1] = (int8_t)type4(w1, w2, w4);   // drop w3
          c.own[2] = (int8_t)type4(w1, w3, w4);   // drop w2
          c.own[3] = (int8_t)type4(w2, w3, w4);   // drop w1
          c.up_type = (int8_t)type4(w2 ^ w1, w3 ^ w1, w4 ^ w1);
        }
  return t;
}
__constant__ Cells4 cCells4 = make_cells4();

// ------------------------------------------------------------------------------ exact stage
template <typename T, typename Acc>
__device__ void process_hypercube(const Acc& A, const Acc& B, bool hasB, const Geo3& G,
                                  const ExtractParams& P, i64 x, i64 y, i64 z, i64 t) {
  i64 g[16][3];
  uint32_t exists = 0;
#pragma unroll 1
  for (int c = 0; c < 16; ++c) {
    const i64 cx = x + (c & 1), cy = y + ((c >> 1) & 1), cz = z + ((c >> 2) & 1);
    const bool ex = cx < G.nx && cy < G.ny && cz < G.nz && ((c & 8) == 0 || hasB);
    if (ex) {
      grad3<T>((c & 8) ? B : A, G, cx, cy, cz, g[c]);
      exists |= 1u << c;
    } else {
      g[c][0] = g[c][1] = g[c][2] = 0;
    }
  }
  // own faces (60 types)
  unsigned long long pmask = 0;
#pragma unroll 1
  for (int ty = 0; ty < 60; ++ty) {
    const int m1 = cK4.masks[ty][0], m2 = cK4.masks[ty][1], m3 = cK4.masks[ty][2];
    if (!((exists >> m3) & 1)) continue;
    const i64 gv[4][3] = {{g[0][0], g[0][1], g[0][2]}, {g[m1][0], g[m1][1], g[m1][2]},
                          {g[m2][0], g[m2][1], g[m2][2]}, {g[m3][0], g[m3][1], g[m3][2]}};
    bool rej = false;  // exact sign reject: one component of one strict sign on all vertices
#pragma unroll
    for (int j = 0; j < 3; ++j)
      rej |= (gv[0][j] > 0 && gv[1][j] > 0 && gv[2][j] > 0 && gv[3][j] > 0) ||
             (gv[0][j] < 0 && gv[1][j] < 0 && gv[2][j] < 0 && gv[3][j] < 0);
    if (!rej && punctured4(gv)) pmask |= 1ull << ty;
  }
  // cells: only full hypercubes have cells anchored here
  const bool full = x + 1 < G.nx && y + 1 < G.ny && z + 1 < G.nz && hasB;
  const int npunct = __popcll(pmask);
  unsigned long long rbase = 0;
  if (npunct) rbase = atomicAdd(&P.counters[CNT_NOUT], (unsigned long long)npunct);
  if (full) {
#pragma unroll 1
    for (int ci = 0; ci < 24; ++ci) {
      const Cell4& cd = cCells4.c[ci];
      int k = 0;
      long long ends[2] = {-1, -1};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((pmask >> cd.own[q]) & 1ull) {
          if (k < 2) ends[k] = (long long)(rbase + __popcll(pmask & ((1ull << cd.own[q]) - 1ull)));
          ++k;
        }
      // upper face (w1, w2, w3, 15): vertices are hypercube corners
      const i64 gu[4][3] = {{g[cd.w[1]][0], g[cd.w[1]][1], g[cd.w[1]][2]}, {g[cd.w[2]][0], g[cd.w[2]][1], g[cd.w[2]][2]},
                            {g[cd.w[3]][0], g[cd.w[3]][1], g[cd.w[3]][2]}, {g[15][0], g[15][1], g[15][2]}};
      if (punctured4(gu)) {
        if (k < 2) {
          const int a1 = cd.w[1];
          const i64 fx = x + (a1 & 1), fy = y + ((a1 >> 1) & 1), fz = z + ((a1 >> 2) & 1), ft = t + ((a1 >> 3) & 1);
          ends[k] = -1 - ((((ft * G.nz + fz) * G.ny + fy) * G.nx + fx) * 60 + cd.up_type);
        }
        ++k;
      }
      if (k == 2) {
        const unsigned long long e = atomicAdd(&P.counters[CNT_EDGES], 1ull);
        if (e < (unsigned long long)P.capacity) {
          P.edges[2 * e] = ends[0] >= 0 ? ends[0] : ends[1];
          P.edges[2 * e + 1] = ends[0] >= 0 ? ends[1] : ends[0];
        }
      } else if (k != 0) {
        atomicAdd(&P.counters[CNT_INVARIANT], 1ull);
      }
    }
  }
  // records
  unsigned long long pm = pmask;
  while (pm) {
    const int ty = __ffsll((long long)pm) - 1;
    pm &= pm - 1;
    const unsigned long long slot = rbase + __popcll(pmask & ((1ull << ty) - 1ull));
    const int m[4] = {0, cK4.masks[ty][0], cK4.masks[ty][1], cK4.masks[ty][2]};
    i64 gv[4][3];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int j = 0; j < 3; ++j) gv[k][j] = g[m[k]][j];
    // D_k = (-1)^(k+3) det(rows != k)  (Eq. 2)
    const i128 D0 = -det3(gv[1], gv[2], gv[3]);
    const i128 D1 = det3(gv[0], gv[2], gv[3]);
    const i128 D2 = -det3(gv[0], gv[1], gv[3]);
    const i128 D3 = det3(gv[0], gv[1], gv[2]);
    const i128 S = D0 + D1 + D2 + D3;
    double mu[4];
    uint32_t flags = 0;
    if (S == 0) {
      mu[0] = mu[1] = mu[2] = mu[3] = 0.25;
      flags |= FTK_CP_DEGENERATE_LOC;
    } else {
      const double s = i128_to_double_rn(S);
      mu[0] = __ddiv_rn(i128_to_double_rn(D0), s);
      mu[1] = __ddiv_rn(i128_to_double_rn(D1), s);
      mu[2] = __ddiv_rn(i128_to_double_rn(D2), s);
      mu[3] = __ddiv_rn(i128_to_double_rn(D3), s);
    }
    double pv[4][4];  // x, y, z, t of each vertex
    double Hd[6][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const i64 vx = x + (m[k] & 1), vy = y + ((m[k] >> 1) & 1), vz = z + ((m[k] >> 2) & 1), vt = t + ((m[k] >> 3) & 1);
      pv[0][k] = (double)vx;
      pv[1][k] = (double)vy;
      pv[2][k] = (double)vz;
      pv[3][k] = (double)vt;
      i64 H[6];
      hess3<T>(P, G, vx, vy, vz, vt, H);
#pragma unroll
      for (int e = 0; e < 6; ++e) Hd[e][k] = __ll2double_rn(H[e]);
    }
    double Hb[6];
#pragma unroll
    for (int e = 0; e < 6; ++e) Hb[e] = dot4_nofma(mu, Hd[e]);
    const int type = classify3(Hb);
    const int span = m[3];
    if (!(span & 8)) flags |= FTK_CP_ORDINAL;
    if (span != 15) {
      const int c = 15 & ~span;
      const i64 vc = c == 1 ? x : c == 2 ? y : c == 4 ? z : t;
      const i64 Nc = c == 1 ? G.nx : c == 2 ? G.ny : c == 4 ? G.nz : G.ntg;
      if (vc == 0 || vc == Nc - 1) flags |= FTK_CP_BOUNDARY;
    }
    if (slot < (unsigned long long)P.capacity) {
      ftk_cp* r = P.out + slot;
      r->face_id = (((t * G.nz + z) * G.ny + y) * G.nx + x) * 60 + ty;
      P.fid[slot] = r->face_id;
      r->label = -1;
      r->x = dot4_nofma(mu, pv[0]);
      r->y = dot4_nofma(mu, pv[1]);
      r->z = dot4_nofma(mu, pv[2]);
      r->t = dot4_nofma(mu, pv[3]);
      r->type = type;
      r->flags = flags;
    }
  }
}

// ------------------------------------------------------------------------------ the kernel
template <typename T>
__device__ __forceinline__ uint32_t sbit(T v) {
  if constexpr (sizeof(T) == 4) return __float_as_uint(v) >> 31;
  else return (uint32_t)((unsigned long long)__double_as_longlong(v) >> 63);
}

template <typename T>
__global__ void __launch_bounds__(NT, 2) k_extract3d(const __grid_constant__ ExtractParams P) {
  __shared__ T tile[2][SV];
  __shared__ uint8_t code[CZ * CY * CX];
  __shared__ unsigned long long s_surv;
  __shared__ unsigned int s_max32;
  __shared__ unsigned long long s_max64;
  const int tid = threadIdx.x;
  Geo3 G;
  G.nx = P.nx;
  G.ny = P.ny;
  G.nz = P.nz;
  G.ntg = P.nt_global;
  G.scale = P.scale;
  G.scale_f = (float)P.scale;
  const T thr = (T)P.thr;
  const T* field = reinterpret_cast<const T*>(P.field);
  const i64 ntx = (G.nx + TX - 1) / TX, nty = (G.ny + TY - 1) / TY, ntz = (G.nz + TZ - 1) / TZ;
  const i64 nchunk = (P.tb - P.ta + TCH - 1) / TCH;
  const i64 nitems = ntx * nty * ntz * nchunk;
  if (tid == 0) {
    s_surv = 0;
    s_max32 = 0;
    s_max64 = 0;
  }
  unsigned long long my_surv = 0;
  uint32_t my_max32 = 0;
  double my_maxd = 0.0;
  const int lx = tid % TX, ly = (tid / TX) % TY, lz = tid / (TX * TY);
  const int lane = tid & 31;
  // survivor list (K1b input): per-warp chunks of CHUNK3 entries, one global atomic per chunk
  long long cur = 0, end = 0;
  auto enqueue = [&](bool surv, i64 x, i64 y, i64 z, int tflag) {
    const uint32_t ball = __ballot_sync(0xffffffffu, surv);
    if (!ball) return;
    const int n = __popc(ball);
    int rank = __popc(ball & ((1u << lane) - 1u));
    int done = 0;
    while (done < n) {
      if (cur == end) {
        long long c = 0;
        if (lane == 0) c = (long long)atomicAdd(&P.counters[CNT_WIN], (unsigned long long)CHUNK3);
        cur = __shfl_sync(0xffffffffu, c, 0);
        end = cur + CHUNK3;
      }
      const int k = (int)min((long long)(n - done), end - cur);
      if (surv && rank >= done && rank < done + k) {
        const long long e = cur + (rank - done);
        if (e < P.wcap) {
          P.wx[e] = (int)x;
          P.wy[e] = (int)y;
          P.wz[e] = (int)z;
          P.wt[e] = tflag;
        }
      }
      cur += k;
      done += k;
    }
    my_surv += surv ? 1 : 0;
  };

  for (i64 item = blockIdx.x; item < nitems; item += gridDim.x) {
    i64 r = item;
    const i64 tx = r % ntx; r /= ntx;
    const i64 ty = r % nty; r /= nty;
    const i64 tz = r % ntz; r /= ntz;
    const i64 ta = P.ta + r * TCH;
    const i64 tb = min(ta + TCH, P.tb);
    const i64 plast = min(tb, G.ntg - 1);
    G.x0 = tx * TX;
    G.y0 = ty * TY;
    G.z0 = tz * TZ;
    const i64 ax = G.x0 + lx, ay = G.y0 + ly, az = G.z0 + lz;
    uint32_t prev = 0x3Fu;
    for (i64 p = ta; p <= plast; ++p) {
      const int cur = (int)((p - ta) & 1);
      T* S = tile[cur];
      const T* src = field + (p - P.t0) * G.nx * G.ny * G.nz;
      __syncthreads();  // previous users of this buffer / of `code` are done
      for (int i = tid; i < SV; i += NT) {
        const int xx = i % SX, yy = (i / SX) % SY, zz = i / (SX * SY);
        const i64 gx = G.x0 - 1 + xx, gy = G.y0 - 1 + yy, gz = G.z0 - 1 + zz;
        T v = (T)0;
        if (gx >= 0 && gx < G.nx && gy >= 0 && gy < G.ny && gz >= 0 && gz < G.nz) {
          v = src[(gz * G.ny + gy) * G.nx + gx];
          // each vertex is owned by exactly one tile position for the range statistic
          if (xx >= 1 && xx <= TX && yy >= 1 && yy <= TY && zz >= 1 && zz <= TZ) {
            if constexpr (sizeof(T) == 4) {
              const uint32_t b = __float_as_uint(v) & 0x7fffffffu;
              my_max32 = max(my_max32, b);
            } else {
              const double a = fabs(v);
              my_maxd = (a != a || my_maxd != my_maxd) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(my_maxd, a);
            }
          }
        }
        S[i] = v;
      }
      __syncthreads();
      // vertex codes for x0..x0+TX, y0..y0+TY, z0..z0+TZ (0 = neutral outside the grid)
      const Tile<T> Pt{S};
      for (int i = tid; i < CX * CY * CZ; i += NT) {
        const int xx = i % CX, yy = (i / CX) % CY, zz = i / (CX * CY);
        const i64 vx = G.x0 + xx, vy = G.y0 + yy, vz = G.z0 + zz;
        uint32_t cval = 0x3Fu;
        if (vx < G.nx && vy < G.ny && vz < G.nz) {
          cval = 0;
          const i64 c[3] = {vx, vy, vz};
          const i64 N[3] = {G.nx, G.ny, G.nz};
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            i64 lo[3] = {vx, vy, vz}, hi[3] = {vx, vy, vz};
            if (c[a] > 0) lo[a] -= 1;
            if (c[a] < N[a] - 1) hi[a] += 1;
            const T d = Pt.at(G, hi[0], hi[1], hi[2]) - Pt.at(G, lo[0], lo[1], lo[2]);
            cval |= (sbit<T>(thr - d) << (2 * a)) | (sbit<T>(d + thr) << (2 * a + 1));
          }
        }
        code[i] = (uint8_t)cval;
      }
      __syncthreads();
      uint32_t cube = 0x3Fu;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        cube &= code[((lz + ((c >> 2) & 1)) * CY + ly + ((c >> 1) & 1)) * CX + lx + (c & 1)];
      const bool inside = ax < G.nx && ay < G.ny && az < G.nz;
      // anchors at p - 1 (hypercube over planes p - 1 and p), then anchors on the last timestep (no
      // t+1 corners)
      const bool s0 = p > ta && inside && ((prev & cube) & 0x3Fu) == 0;
      const bool s1 = p == G.ntg - 1 && p < tb && inside && (cube & 0x3Fu) == 0;
      enqueue(s0, ax, ay, az, (int)((uint32_t)(p - 1) | 0x80000000u));
      enqueue(s1, ax, ay, az, (int)p);
      prev = cube;
    }
  }
  // the unused rest of the warp's chunk holds no cube
  for (long long e = cur + lane; e < end; e += 32)
    if (e < P.wcap) P.wt[e] = -1;
  atomicAdd(&s_surv, my_surv);
  atomicMax(&s_max32, my_max32);
  atomicMax(&s_max64, (unsigned long long)__double_as_longlong(my_maxd));
  __syncthreads();
  if (tid == 0) {
    atomicAdd(&P.counters[CNT_SURVIVORS], s_surv);
    atomicMax(&P.counters[CNT_MAXBITS], sizeof(T) == 4 ? (unsigned long long)s_max32 : s_max64);
  }
}

// K1b (3D): one thread per surviving hypercube of the list; gradients and Hessians straight from the
// field (L2/HBM).
template <typename T>
__global__ void __launch_bounds__(128) k_exact3d(const __grid_constant__ ExtractParams P) {
  Geo3 G;
  G.nx = P.nx;
  G.ny = P.ny;
  G.nz = P.nz;
  G.ntg = P.nt_global;
  G.scale = P.scale;
  G.scale_f = (float)P.scale;
  G.x0 = G.y0 = G.z0 = 0;
  const long long nwin = min((long long)*(volatile unsigned long long*)&P.counters[CNT_WIN], (long long)P.wcap);
  const T* field = reinterpret_cast<const T*>(P.field);
  const i64 plane = G.nx * G.ny * G.nz;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nwin;
       e += (long long)gridDim.x * blockDim.x) {
    const int et = P.wt[e];
    if (et == -1) continue;
    const bool hasB = et < 0;
    const i64 t = et & 0x3fffffff;
    const GTile<T> A{field + (t - P.t0) * plane};
    const GTile<T> B{hasB ? A.S + plane : A.S};
    process_hypercube<T>(A, B, hasB, G, P, P.wx[e], P.wy[e], P.wz[e], t);
  }
}

}  // namespace k3d

template <typename T>
static int launch3_t(const ExtractParams& P, cudaStream_t stream) {
  using namespace k3d;
  int dev = 0, sms = 148, per_sm = 0;
  FTK_CUDA_TRY(cudaGetDevice(&dev));
  FTK_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  FTK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_extract3d<T>, NT, 0));
  const long long items = ((P.nx + TX - 1) / TX) * ((P.ny + TY - 1) / TY) * ((P.nz + TZ - 1) / TZ) *
                          ((P.tb - P.ta + TCH - 1) / TCH);
  if (items <= 0) return FTK_OK;
  const long long grid = std::min<long long>(items, (long long)sms * std::max(per_sm, 1) * 4);
  k_extract3d<T><<<(unsigned)grid, NT, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  if (P.ev_mid) FTK_CUDA_TRY(cudaEventRecord(reinterpret_cast<cudaEvent_t>(P.ev_mid), stream));
  int xper = 0;
  FTK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&xper, k_exact3d<T>, 128, 0));
  k_exact3d<T><<<(unsigned)(sms * std::max(xper, 1)), 128, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

int launch_extract3d(const ExtractParams& P, cudaStream_t stream) {
  if (P.dtype == FTK_F32) return launch3_t<float>(P, stream);
  return launch3_t<double>(P, stream);
}

}  // namespace ftk
