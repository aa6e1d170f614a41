// extract3d.cu -- K1 for 3D+t (4D spacetime, faces = tetrahedra, cells = pentachora).
//
// Pass 1 of Alg. 1 (generalised at P:439) plus the per-hypercube cell evaluation of
// pass 2, split like the 2D path:
//
//   K1a k_scan3d (namespace s3): TMA 4D halo boxes of 128 x 8 x 8 anchor tiles per timestep, one warp
//     per z-slice; per vertex a 6-bit "strict sign holds" code (dx > thr, dx < -thr, dy.., dz..) on raw
//     values, thr = 2^(1-s), which implies the exact integer gradient component is strictly
//     positive/negative; ANDed over the 16 corners of the spacetime hypercube
//     (y/x pairs in registers, z pairs through shared memory, t pairs across planes); a zero code is a
//     survivor and its anchor goes to the survivor list.
//   K1b k_exact3d: one warp per surviving hypercube, straight from the field: int64 gradients of the 16
//     corners, the 60 face types two per lane with 3x3 determinant signs from an FP64 filter (exact
//     int128 and the SoS epsilon-expansion of det(M + E) when it cannot decide; PAPER.md:465-467;
//     DESIGN.md R4/R5), Eq. 2 location and the Descartes-rule Hessian type in fixed-order FP64, and
//     the 24 cells (pentachora) of the hypercube: 0 or 2 punctured sides each, emitted
//     as trajectory edges.
//   Vector fields (FTK_VECTOR_FIELD): k_scanvec3d (namespace v3) and k_exact3d<T, true> (quantized
//     corner vectors, Routh-Hurwitz Jacobian type).
#include <cstdio>
#include <cstring>
#include <utility>

#include "common.cuh"
#include "extract2d.cuh"
#include "kuhn.cuh"
#include "sm100.cuh"

namespace ftk {
namespace k3d {
using namespace sm100;

constexpr int TCH = 16;                         // anchor timesteps per work item

__constant__ KuhnTables<4> cK4 = kKuhn4;

// ------------------------------------------------------------------------------ SoS, 3x3
// The epsilon-monomials of det(M + E), eps_{r,j} = eps^(2^(3r + j)) (R4), in decreasing
// magnitude (increasing exponent): per term, for each row r the perturbed column or -1.  A literal
// table, derived by tools/derive_sos3.py from the Leibniz expansion of det(M + E) (every permutation x
// every choice of perturbed rows, monomials collected by exponent); tests/test_sos3_table.py checks it
// against that derivation and the oracle's own order.  Term 0 is the determinant itself; a term's
// coefficient is the signed complementary minor.
struct PP3 {
  int n;
  int8_t col[34][3];
};
__constant__ PP3 cPP3 = {34, {{-1, -1, -1}, {0, -1, -1}, {1, -1, -1}, {2, -1, -1}, {-1, 0, -1}, {1, 0, -1}, {2, 0, -1}, {-1, 1, -1}, {0, 1, -1}, {2, 1, -1}, {-1, 2, -1}, {0, 2, -1}, {1, 2, -1}, {-1, -1, 0}, {1, -1, 0}, {2, -1, 0}, {-1, 1, 0}, {2, 1, 0}, {-1, 2, 0}, {1, 2, 0}, {-1, -1, 1}, {0, -1, 1}, {2, -1, 1}, {-1, 0, 1}, {2, 0, 1}, {-1, 2, 1}, {0, 2, 1}, {-1, -1, 2}, {0, -1, 2}, {1, -1, 2}, {-1, 0, 2}, {1, 0, 2}, {-1, 1, 2}, {0, 1, 2}}};

// the same determinant when every entry is below 2^31 in magnitude: the 2x2 minors are exact in int64
// (|.| < 2^63) and only the three outer products need 64 x 64 -> 128-bit multiplies
__device__ __forceinline__ i128 det3_mid(const i64* a, const i64* b, const i64* c) {
  const long long m0 = b[1] * c[2] - b[2] * c[1];
  const long long m1 = b[0] * c[2] - b[2] * c[0];
  const long long m2 = b[0] * c[1] - b[1] * c[0];
  return (i128)a[0] * m0 - (i128)a[1] * m1 + (i128)a[2] * m2;
}

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

// Sign of det[a; b; c] by a floating-point filter, for entries |.| < 2^26: the 2x2 minors are exact
// in FP64 (products < 2^52, differences < 2^53); the three products a_i m_i are rounded, and the
// rounded sum d differs from the exact determinant by at most 3.01 u (|p0| + |p1| + |p2|), u = 2^-53,
// which the computed bound 2^-50 (|p0| + |p1| + |p2|) exceeds -- so |d| > bound fixes the exact sign.
// Returns 0 when the filter cannot decide (the exact int128 path then runs).
__device__ __forceinline__ int det3_sign_fp(const i64* a, const i64* b, const i64* c) {
  const double b0 = (double)b[0], b1 = (double)b[1], b2 = (double)b[2];
  const double c0 = (double)c[0], c1 = (double)c[1], c2 = (double)c[2];
  const double m0 = __dsub_rn(__dmul_rn(b1, c2), __dmul_rn(b2, c1));
  const double m1 = __dsub_rn(__dmul_rn(b0, c2), __dmul_rn(b2, c0));
  const double m2 = __dsub_rn(__dmul_rn(b0, c1), __dmul_rn(b1, c0));
  const double p0 = __dmul_rn((double)a[0], m0), p1 = __dmul_rn((double)a[1], m1), p2 = __dmul_rn((double)a[2], m2);
  const double d = __dadd_rn(__dsub_rn(p0, p1), p2);
  const double bound = __dmul_rn(__dadd_rn(__dadd_rn(fabs(p0), fabs(p1)), fabs(p2)), 0x1p-50);
  return d > bound ? 1 : (d < -bound ? -1 : 0);
}

// small: every entry < 2^26 (the FP64 filter applies); mid: every entry < 2^31 (det3_mid applies)
__device__ __forceinline__ int sos3(const i64* r0, const i64* r1, const i64* r2, bool small, bool mid) {
  if (small) {
    const int f = det3_sign_fp(r0, r1, r2);
    if (f) return f;
  }
  const i128 d = mid ? det3_mid(r0, r1, r2) : det3(r0, r1, r2);
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
// small: every entry |.| < 2^26 (the floating-point filter of det3_sign_fp applies)
__device__ __forceinline__ bool punctured4(const i64 (&g)[4][3], bool small, bool mid) {
  const int s0 = -sos3(g[1], g[2], g[3], small, mid);
  const int s1 = sos3(g[0], g[2], g[3], small, mid);
  if (s0 != s1) return false;
  const int s2 = -sos3(g[0], g[1], g[3], small, mid);
  if (s0 != s2) return false;
  const int s3 = sos3(g[0], g[1], g[2], small, mid);
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

// Vector-field type (FTK_VECTOR_FIELD, R17) from the interpolated 3x3 Jacobian
// h = [u_x u_y u_z v_x v_y v_z w_x w_y w_z]: Routh-Hurwitz count of the eigenvalues with positive real
// part on det(lambda I - J) = lambda^3 + a1 lambda^2 + a2 lambda + a3 -- 0 sink, 3 source, else
// saddle; det == 0 degenerate; a1 == 0 saddle; a1 a2 == a3 centre if a2 > 0 (an imaginary pair) else
// saddle.  Fixed-order FP64, no FMA, as the oracle.
__device__ __forceinline__ int classify_vec3(const double* h) {
  const double a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7], k = h[8];
  const double tr = __dadd_rn(__dadd_rn(a, e), k);
  const double m2 = __dadd_rn(__dadd_rn(__dsub_rn(__dmul_rn(a, e), __dmul_rn(b, d)), __dsub_rn(__dmul_rn(a, k), __dmul_rn(c, g))),
                              __dsub_rn(__dmul_rn(e, k), __dmul_rn(f, hh)));
  const double det = __dadd_rn(__dsub_rn(__dmul_rn(a, __dsub_rn(__dmul_rn(e, k), __dmul_rn(f, hh))),
                                         __dmul_rn(b, __dsub_rn(__dmul_rn(d, k), __dmul_rn(f, g)))),
                               __dmul_rn(c, __dsub_rn(__dmul_rn(d, hh), __dmul_rn(e, g))));
  if (det == 0) return FTK_CP_DEGENERATE;
  const double a1 = -tr, a2 = m2, a3 = -det;
  const double r3 = __dsub_rn(__dmul_rn(a1, a2), a3);
  if (a1 == 0) return FTK_CP_SADDLE;
  if (r3 == 0) return a2 > 0 ? FTK_CP_CENTER : FTK_CP_SADDLE;
  const int s1 = a1 > 0 ? 1 : -1, s2 = (r3 > 0) == (a1 > 0) ? 1 : -1, s3 = a3 > 0 ? 1 : -1;
  const int changes = (s1 != 1) + (s2 != s1) + (s3 != s2);
  return changes == 0 ? FTK_CP_SINK : (changes == 3 ? FTK_CP_SOURCE : FTK_CP_SADDLE);
}

// Jacobian of a 3D vector field at (x, y, z, t): the gradient rule of R7 on each component;
// J[3 j + a] = d(component j) / d(axis a), 2x scale, one-sided doubled at the boundary
template <typename T>
__device__ void jac3(const ExtractParams& P, const Geo3& G, i64 x, i64 y, i64 z, i64 t, i64* J) {
  const T* base = reinterpret_cast<const T*>(P.field) + (t - P.t0) * G.nx * G.ny * G.nz * 3;
  auto q = [&](i64 xx, i64 yy, i64 zz, int j) { return quant3(base[((zz * G.ny + yy) * G.nx + xx) * 3 + j], G); };
  const i64 N[3] = {G.nx, G.ny, G.nz};
  const i64 c[3] = {x, y, z};
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      i64 lo[3] = {x, y, z}, hi[3] = {x, y, z};
      i64 f = 1;
      if (c[a] == 0) { hi[a] = 1; lo[a] = 0; f = 2; }
      else if (c[a] == N[a] - 1) { hi[a] = N[a] - 1; lo[a] = N[a] - 2; f = 2; }
      else { hi[a] = c[a] + 1; lo[a] = c[a] - 1; }
      J[3 * j + a] = f * (q(hi[0], hi[1], hi[2], j) - q(lo[0], lo[1], lo[2], j));
    }
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

// ------------------------------------------------------------------------------ K1a (3D): the scan
// Persistent, two CTAs per SM.  A work item is a 128 x RW x 8 tile of anchors (x, y, z) times a chunk
// of TCH anchor timesteps.  Per timestep the producer warp stages the 136 x (RW + 3) x 11 halo box
// (x0-4.., y0-1.., z0-1..) with one 4D TMA load into an NSTAGE-deep ring.  Scan warp w owns the
// hypercubes anchored at slice z0 + w (RW rows x 128 columns; lane = 4 consecutive x).
//
// Region test first (r2): a hypercube can hold a punctured face only if no gradient component keeps
// one strict sign on its 16 corners; so if dz > thr (or dz < -thr) on EVERY vertex of the warp's
// region -- slices z and z + 1, rows y0 .. y0 + RW, columns x0 .. x0 + 128 -- on both planes of a
// plane pair, every hypercube of the warp is rejected for that pair.  The test is a min / max of dz
// over the region (FMNMX3), per plane; the per-vertex codes below are computed only for the pairs it
// does not reject (smooth fields: most of them are).  It rejects nothing the per-vertex codes would
// keep and keeps nothing they would reject (the same fp32 dz and the same strict comparison), so the
// survivor set is unchanged.  A plane's stage is held until the next plane of the item has been
// tested, so its codes can still be computed when the following pair needs them.
//
// Per-vertex codes (the pairs the region test keeps): per vertex a 6-bit "strict sign holds" code
// (dx > thr, dx < -thr, dy.., dz..) in the top of a byte, ANDed over the y-pair and x-pair in
// registers (slice_squares), over the z-pair by computing slice z + 1's squares in the same warp, over
// the t-pair with the previous plane's cube codes; a zero byte is a survivor (the exact zero-byte test
// holds: the two low bits of every byte repeat bit 2, so no byte is 1..3).
namespace s3 {
#ifndef FTK_S3_RW
#define FTK_S3_RW 8
#endif
#ifndef FTK_S3_NSTAGE
#define FTK_S3_NSTAGE 3
#endif
#ifndef FTK_S3_MINB
#define FTK_S3_MINB 1
#endif
#ifndef FTK_S3_COUNT
#define FTK_S3_COUNT 0   // experiment builds: region-test statistics in counters[CNT_PROF..]
#endif
#ifndef FTK_S3_NOCODES
#define FTK_S3_NOCODES 0  // experiment builds: skip the per-vertex codes (timing floor; results invalid)
#endif
#ifndef FTK_S3_REGION
#define FTK_S3_REGION 1  // region-first dz test (0: per-vertex codes for every plane pair)
#endif
#ifndef FTK_S3_SPLIT
#define FTK_S3_SPLIT 1   // scan warps per z-slice (each owns RW / SPLIT anchor rows); 2 measured slower
#endif
#ifndef FTK_S3_TP
#define FTK_S3_TP 2      // squares tasks per slice (each RW / TP code rows): finer load balance
#endif
constexpr int LX = 128, TX = LX, RW = FTK_S3_RW, XOFF = 4, PITCH = LX + 8;  // tiles own all 128 columns
constexpr int ROWS = RW + 3;  // y0-1 .. y0+RW+1
constexpr int SPLIT = FTK_S3_SPLIT, NR = RW / SPLIT;  // NR: anchor rows of one scan warp
constexpr int TP = FTK_S3_TP, NRT = RW / TP;           // NRT: code rows of one squares task
static_assert(RW % SPLIT == 0 && RW % TP == 0 && NR % NRT == 0, "SPLIT, TP divide RW; tasks within a warp's rows");
static_assert(TP * 9 <= 64, "task masks are 64-bit");
template <typename T>
constexpr int nzw() { return sizeof(T) == 4 ? 8 : 4; }  // z-slice warps (owned slices per tile)
template <typename T>
constexpr int slices() { return nzw<T>() + 3; }         // z0-1 .. z0+NZW+1
template <typename T>
constexpr int nstage() { return sizeof(T) == 4 ? FTK_S3_NSTAGE : 2; }
template <typename T>
constexpr int nthreads() { return (nzw<T>() * SPLIT + 1) * 32; }  // NZW x SPLIT scan warps + producer
template <typename T>
constexpr int stage_elems() { return (PITCH * ROWS * slices<T>() * (int)sizeof(T) + 127) / 128 * 128 / (int)sizeof(T); }
constexpr uint32_t NEUTRAL = 0xFCFCFCFCu;
constexpr int CHUNK = 32;

struct Meta {
  int x0, y0, z0, p, k, nplanes, tb, done;
};

template <typename T>
struct alignas(128) Smem {
  static constexpr int NSTAGE = nstage<T>(), NZW = nzw<T>();
  T plane[NSTAGE][stage_elems<T>()];
  uint32_t sq[2][NZW + 1][RW][32];  // per plane parity: the squares of every slice computed this plane
  unsigned long long need[3][2];     // per plane (gk mod 3): squares tasks of this plane / the previous
                                     // plane that are needed (bit TP j + h: slice z0 + j, rows of part h)
  unsigned long long have[2];        // per plane parity: squares tasks whose results are in sq
  Meta meta[NSTAGE];
  uint64_t full[NSTAGE];
  uint64_t empty[NSTAGE];
  unsigned long long surv;
  unsigned int maxbits32;
  unsigned long long maxbits64;
};

#ifndef FTK_GATHER_SR
#define FTK_GATHER_SR 1
#endif
__device__ __forceinline__ uint32_t prmt_sr(uint32_t a, uint32_t b) {
  // result bytes [sign(a) x 8, sign(b) x 8, sign(a) x 8, sign(b) x 8]: PRMT selector nibbles with the
  // msb set replicate the sign bit of the selected byte (byte 3 of a = index 3, of b = index 7)
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, 0xFBFB;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t bitsel(uint32_t a, uint32_t b, uint32_t m) { return (a & ~m) | (b & m); }

// 6 conditions x 4 positions -> byte i bits 7..2 = [dx>thr, dx<-thr, dy>thr, dy<-thr, dz>thr, dz<-thr]
// (FTK_GATHER_SR: bits 1, 0 repeat bit 2, so a byte is zero iff its six condition bits are, and no byte
// is 0x01 -- the per-byte zero test stays exact)
__device__ __forceinline__ uint32_t gather6(const f2 (&c)[12]) {
  if constexpr (FTK_GATHER_SR) {
    // per condition: two sign-replicating PRMTs (positions 0, 1 and 2, 3) and two bit-selects
    uint32_t acc = bitsel(prmt_sr(lo32(c[0]), hi32(c[0])), prmt_sr(lo32(c[1]), hi32(c[1])), 0xFFFF0000u);
#pragma unroll
    for (int j = 1; j < 6; ++j) {
      const uint32_t m = j < 5 ? (0x80808080u >> j) : 0x07070707u;
      acc = bitsel(acc, prmt_sr(lo32(c[2 * j]), hi32(c[2 * j])), m & 0x0000FFFFu);
      acc = bitsel(acc, prmt_sr(lo32(c[2 * j + 1]), hi32(c[2 * j + 1])), m & 0xFFFF0000u);
    }
    return acc;
  } else {
    uint32_t w[6];  // FTK_GATHER_SR = 0: byte picks
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      const uint32_t p01 = __byte_perm(lo32(c[2 * j]), hi32(c[2 * j]), 0x0073);
      const uint32_t p23 = __byte_perm(lo32(c[2 * j + 1]), hi32(c[2 * j + 1]), 0x0073);
      w[j] = __byte_perm(p01, p23, 0x5410);
    }
    return (w[0] & 0x80808080u) | ((w[1] >> 1) & 0x40404040u) | ((w[2] >> 2) & 0x20202020u) |
           ((w[3] >> 3) & 0x10101010u) | ((w[4] >> 4) & 0x08080808u) | ((w[5] >> 5) & 0x04040404u);
  }
}

__device__ __forceinline__ uint32_t code6_f32(const float4 u, const float4 v, const float4 d, const float4 zm,
                                              const float4 zp, float l, float r, f2 thr2, f2 nthr2) {
  const f2 dx01 = pack2(__fsub_rn(v.y, l), __fsub_rn(v.z, v.x));
  const f2 dx23 = pack2(__fsub_rn(v.w, v.y), __fsub_rn(r, v.z));
  const f2 dy01 = sub2(pack2(d.x, d.y), pack2(u.x, u.y));
  const f2 dy23 = sub2(pack2(d.z, d.w), pack2(u.z, u.w));
  const f2 dz01 = sub2(pack2(zp.x, zp.y), pack2(zm.x, zm.y));
  const f2 dz23 = sub2(pack2(zp.z, zp.w), pack2(zm.z, zm.w));
  f2 c[12];
  c[0] = sub2(thr2, dx01);  c[1] = sub2(thr2, dx23);
  c[2] = sub2(dx01, nthr2); c[3] = sub2(dx23, nthr2);
  c[4] = sub2(thr2, dy01);  c[5] = sub2(thr2, dy23);
  c[6] = sub2(dy01, nthr2); c[7] = sub2(dy23, nthr2);
  c[8] = sub2(thr2, dz01);  c[9] = sub2(thr2, dz23);
  c[10] = sub2(dz01, nthr2); c[11] = sub2(dz23, nthr2);
  return gather6(c);
}

__device__ __forceinline__ uint32_t sgn64(double v) { return (uint32_t)((unsigned long long)__double_as_longlong(v) >> 63); }

struct Ctx {
  int lane;
  int rpos;        // position (0..3) of x = nx - 1 in this lane, else -1
  bool lpat;       // x = 0 is this lane's position 0
  uint32_t oob;    // NEUTRAL bits of this lane's out-of-grid positions
  bool xe_out;     // column x0 + 128 is outside the grid
  bool xe_last;    // column x0 + 128 is x = nx - 1
  long long gy0, ny;
  long long gz, nz;
};

// squares (AND over y-pair and x-pair) of the slice whose centre rows start at S (row 0 = y0-1),
// with the z -+ 1 slices at S -/+ slice_stride.  MODE 0: interior; 1: x boundary only (one-sided
// x differences, out-of-grid columns); 2: any boundary (fp64 input treats 1 as 2).
template <typename T, int MODE, int NR>
__device__ __forceinline__ void slice_squares(const T* S, int zstride, const Ctx& c, f2 thr2, f2 nthr2, T thr,
                                              uint32_t (&Sq)[NR], uint32_t& maxb, double& maxd, bool count) {
  constexpr bool XE = MODE >= 1, EDGE = sizeof(T) == 4 ? MODE >= 2 : MODE >= 1;
  const bool lane0 = c.lane == 0, lane31 = c.lane == 31;
  const int hcol = lane0 ? XOFF - 1 : XOFF + LX;
  const bool zlo = EDGE && c.gz == 0, zhi = EDGE && c.gz == c.nz - 1, zout = EDGE && c.gz >= c.nz;
  const T* Zm = zlo ? S : S - zstride;
  const T* Zp = zhi ? S : S + zstride;
  if constexpr (sizeof(T) == 4) {
    auto load = [&](int i, float4& v, float& l, float& r) {
      v = *reinterpret_cast<const float4*>(S + i * PITCH + XOFF + 4 * c.lane);
      const float h = S[i * PITCH + hcol];
      const float up = __shfl_up_sync(0xffffffffu, v.w, 1);
      const float dn = __shfl_down_sync(0xffffffffu, v.x, 1);
      l = lane0 ? h : up;
      r = lane31 ? h : dn;
      if (XE) {
        if (c.lpat) l = v.x;
        if (c.rpos == 0) v.y = v.x;
        if (c.rpos == 1) v.z = v.y;
        if (c.rpos == 2) v.w = v.z;
        if (c.rpos == 3) r = v.w;
      }
    };
    // codes of column x0 + 128 (the next tile's first column; they complete lane 31's cubes): lane k
    // computes code row k (centre row k + 1), Ye = the y-pair of code rows k, k + 1
    uint32_t Ye;
    {
      const int k = min(c.lane, NR);
      const int o = (k + 1) * PITCH + XOFF + LX;
      const float ctr = S[o], l = S[o - 1];
      float r = S[o + 1], u = S[o - PITCH], d = S[o + PITCH], zm = Zm[o], zp = Zp[o];
      bool out = false;
      if (XE) {
        if (c.xe_last) r = ctr;
        out = c.xe_out;
      }
      if (EDGE) {
        const long long gy = c.gy0 + k;
        if (gy == 0) u = ctr;
        if (gy == c.ny - 1) d = ctr;
        out = out || gy >= c.ny || zout;
      }
      const float th = __uint_as_float(lo32(thr2));
      const float dx = __fsub_rn(r, l), dy = __fsub_rn(d, u), dz = __fsub_rn(zp, zm);
      const uint32_t ce = out ? 0xFCu
                              : ((__float_as_uint(__fsub_rn(th, dx)) >> 31) << 7) |
                                    ((__float_as_uint(__fadd_rn(dx, th)) >> 31) << 6) |
                                    ((__float_as_uint(__fsub_rn(th, dy)) >> 31) << 5) |
                                    ((__float_as_uint(__fadd_rn(dy, th)) >> 31) << 4) |
                                    ((__float_as_uint(__fsub_rn(th, dz)) >> 31) << 3) |
                                    ((__float_as_uint(__fadd_rn(dz, th)) >> 31) << 2);
      Ye = ce & __shfl_down_sync(0xffffffffu, ce, 1);
    }
    float4 v0, v1, v2;
    float l0, r0, l1, r1, l2, r2;
    load(0, v0, l0, r0);
    load(1, v1, l1, r1);
    uint32_t Cprev = 0;
#pragma unroll
    for (int k = 0; k <= NR; ++k) {
      load(k + 2, v2, l2, r2);
      if (count && k < NR) maxb = max_abs_bits(maxb, v1.x, v1.y, v1.z, v1.w);
      const float4 zm = *reinterpret_cast<const float4*>(Zm + (k + 1) * PITCH + XOFF + 4 * c.lane);
      const float4 zp = *reinterpret_cast<const float4*>(Zp + (k + 1) * PITCH + XOFF + 4 * c.lane);
      uint32_t C;
      if (EDGE) {
        const long long gy = c.gy0 + k;
        const float4 u = gy == 0 ? v1 : v0;
        const float4 d = gy == c.ny - 1 ? v1 : v2;
        C = (gy >= c.ny || zout) ? NEUTRAL : (code6_f32(u, v1, d, zm, zp, l1, r1, thr2, nthr2) | c.oob);
      } else if (XE) {
        C = code6_f32(v0, v1, v2, zm, zp, l1, r1, thr2, nthr2) | c.oob;
      } else {
        C = code6_f32(v0, v1, v2, zm, zp, l1, r1, thr2, nthr2);
      }
      if (k >= 1) {
        const uint32_t Y = Cprev & C;
        uint32_t nb = __shfl_down_sync(0xffffffffu, Y, 1);  // next lane's position 0
        const uint32_t ne = __shfl_sync(0xffffffffu, Ye, k - 1);  // column x0 + 128
        if (c.lane == 31) nb = ne;
        Sq[k - 1] = Y & ((Y >> 8) | (nb << 24));
      }
      Cprev = C;
      v0 = v1; l0 = l1; r0 = r1;
      v1 = v2; l1 = l2; r1 = r2;
    }
  } else {
    // fp64: scalar arithmetic, same layout
    auto load = [&](int i, double (&f)[6]) {
      const double* p = S + i * PITCH;
      const double2 a = *reinterpret_cast<const double2*>(p + XOFF + 4 * c.lane);
      const double2 b = *reinterpret_cast<const double2*>(p + XOFF + 4 * c.lane + 2);
      const double h = p[hcol];
      f[1] = a.x; f[2] = a.y; f[3] = b.x; f[4] = b.y;
      const double up = __shfl_up_sync(0xffffffffu, b.y, 1);
      const double dn = __shfl_down_sync(0xffffffffu, a.x, 1);
      f[0] = lane0 ? h : up;
      f[5] = lane31 ? h : dn;
      if (EDGE) {
        if (c.lpat) f[0] = f[1];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (c.rpos == q) f[q + 2] = f[q + 1];
      }
    };
    uint32_t Ye;  // codes of column x0 + 128 (as for fp32)
    {
      const int k = min(c.lane, NR);
      const int o = (k + 1) * PITCH + XOFF + LX;
      const double ctr = S[o], l = S[o - 1];
      double r = S[o + 1], u = S[o - PITCH], d = S[o + PITCH], zm = Zm[o], zp = Zp[o];
      bool out = false;
      if (EDGE) {
        const long long gy = c.gy0 + k;
        if (c.xe_last) r = ctr;
        if (gy == 0) u = ctr;
        if (gy == c.ny - 1) d = ctr;
        out = c.xe_out || gy >= c.ny || zout;
      }
      const double th = (double)thr, dx = r - l, dy = d - u, dz = zp - zm;
      const uint32_t ce = out ? 0xFCu
                              : (sgn64(th - dx) << 7) | (sgn64(dx + th) << 6) | (sgn64(th - dy) << 5) |
                                    (sgn64(dy + th) << 4) | (sgn64(th - dz) << 3) | (sgn64(dz + th) << 2);
      Ye = ce & __shfl_down_sync(0xffffffffu, ce, 1);
    }
    double f0[6], f1[6], f2_[6];
    load(0, f0);
    load(1, f1);
    uint32_t Cprev = 0;
#pragma unroll
    for (int k = 0; k <= NR; ++k) {
      load(k + 2, f2_);
      if (count && k < NR)
#pragma unroll
        for (int q = 1; q <= 4; ++q) {
          const double a = fabs(f1[q]);
          maxd = (a != a || maxd != maxd) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(maxd, a);
        }
      const long long gy = c.gy0 + k;
      const double* fu = (EDGE && gy == 0) ? f1 : f0;
      const double* fd = (EDGE && gy == c.ny - 1) ? f1 : f2_;
      uint32_t W = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double zmv = Zm[(k + 1) * PITCH + XOFF + 4 * c.lane + q], zpv = Zp[(k + 1) * PITCH + XOFF + 4 * c.lane + q];
        const double dx = f1[q + 2] - f1[q], dy = fd[q + 1] - fu[q + 1], dz = zpv - zmv;
        const uint32_t b6 = (sgn64(thr - dx) << 5) | (sgn64(dx + thr) << 4) | (sgn64(thr - dy) << 3) |
                            (sgn64(dy + thr) << 2) | (sgn64(thr - dz) << 1) | sgn64(dz + thr);
        W |= b6 << (8 * q + 2);
      }
      const uint32_t C = (EDGE && (gy >= c.ny || zout)) ? NEUTRAL : (EDGE ? (W | c.oob) : W);
      if (k >= 1) {
        const uint32_t Y = Cprev & C;
        uint32_t nb = __shfl_down_sync(0xffffffffu, Y, 1);  // next lane's position 0
        const uint32_t ne = __shfl_sync(0xffffffffu, Ye, k - 1);  // column x0 + 128
        if (c.lane == 31) nb = ne;
        Sq[k - 1] = Y & ((Y >> 8) | (nb << 24));
      }
      Cprev = C;
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        f0[q] = f1[q];
        f1[q] = f2_[q];
      }
    }
  }
}

// Warp-region dz test of one plane (fp32; MODE 0 / 1: y and z interior, so every dz of the region is
// the central difference): returns bit 1 when dz > thr on every vertex of the warp's region -- slices
// z and z + 1, code rows 0 .. RW, columns x0 .. x0 + 128, out-of-grid columns excluded -- and bit 0 when
// dz < -thr on every one (the same fp32 dz and strict comparisons as the per-vertex codes).  Also tracks
// max |f| over the warp's owned vertices.  S: slice z - 1, row y0 of the stage.
template <int MODE>
__device__ __forceinline__ uint32_t region_dz(const float* S, const Ctx& c, float thr, f2 nan01, f2 nan23,
                                              uint32_t& maxb) {
  constexpr int ZS = PITCH * ROWS;
  float mn = __int_as_float(0x7f800000), mx = __int_as_float(0xff800000);  // +inf, -inf
#pragma unroll
  for (int k = 0; k <= NR; ++k) {
    const float* p = S + k * PITCH + XOFF + 4 * c.lane;
    const float4 a0 = *reinterpret_cast<const float4*>(p);
    const float4 a1 = *reinterpret_cast<const float4*>(p + ZS);
    const float4 a2 = *reinterpret_cast<const float4*>(p + 2 * ZS);
    const float4 a3 = *reinterpret_cast<const float4*>(p + 3 * ZS);
    if (k < NR) maxb = max_abs_bits(maxb, a1.x, a1.y, a1.z, a1.w);
    f2 d0 = sub2(pack2(a2.x, a2.y), pack2(a0.x, a0.y));  // dz at slice z, positions 0, 1
    f2 d1 = sub2(pack2(a2.z, a2.w), pack2(a0.z, a0.w));  //                 positions 2, 3
    f2 e0 = sub2(pack2(a3.x, a3.y), pack2(a1.x, a1.y));  // dz at slice z + 1
    f2 e1 = sub2(pack2(a3.z, a3.w), pack2(a1.z, a1.w));
    if (MODE == 1) {  // out-of-grid positions become NaN: neutral for fminf / fmaxf
      d0 = add2(d0, nan01);
      d1 = add2(d1, nan23);
      e0 = add2(e0, nan01);
      e1 = add2(e1, nan23);
    }
    mn = fminf(fminf(mn, __uint_as_float(lo32(d0))), __uint_as_float(hi32(d0)));
    mx = fmaxf(fmaxf(mx, __uint_as_float(lo32(d0))), __uint_as_float(hi32(d0)));
    mn = fminf(fminf(mn, __uint_as_float(lo32(d1))), __uint_as_float(hi32(d1)));
    mx = fmaxf(fmaxf(mx, __uint_as_float(lo32(d1))), __uint_as_float(hi32(d1)));
    mn = fminf(fminf(mn, __uint_as_float(lo32(e0))), __uint_as_float(hi32(e0)));
    mx = fmaxf(fmaxf(mx, __uint_as_float(lo32(e0))), __uint_as_float(hi32(e0)));
    mn = fminf(fminf(mn, __uint_as_float(lo32(e1))), __uint_as_float(hi32(e1)));
    mx = fmaxf(fmaxf(mx, __uint_as_float(lo32(e1))), __uint_as_float(hi32(e1)));
  }
  // column x0 + 128 (the next tile's first column: the x + 1 corners of lane 31's hypercubes), rows
  // 0 .. RW of slices z - 1 .. z + 2: lane 4 k + j holds row k of slice z - 1 + j, dz from lane + 2
  {
    const int k = c.lane >> 2, j = c.lane & 3;
    const float v = c.lane < 4 * (NR + 1) ? S[j * ZS + k * PITCH + XOFF + LX] : 0.f;
    const float w = __shfl_down_sync(0xffffffffu, v, 2);
    const bool ok = c.lane < 4 * (NR + 1) && j < 2 && !c.xe_out;
    const float d = ok ? __fsub_rn(w, v) : __int_as_float(0x7fc00000);
    mn = fminf(mn, d);
    mx = fmaxf(mx, d);
  }
  return (__all_sync(0xffffffffu, mn > thr) ? 2u : 0u) | (__all_sync(0xffffffffu, mx < -thr) ? 1u : 0u);
}

// max |f| over the warp's owned vertices of a plane (slice z, rows y0 .. y0 + RW - 1; positions outside
// the grid are zero-filled by the loaders); S: slice z, row y0 of the stage
template <typename T>
__device__ __forceinline__ void owned_max(const T* S, int lane, uint32_t& maxb, double& maxd) {
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    const T* p = S + k * PITCH + XOFF + 4 * lane;
    if constexpr (sizeof(T) == 4) {
      const float4 v = *reinterpret_cast<const float4*>(p);
      maxb = max_abs_bits(maxb, v.x, v.y, v.z, v.w);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double a = fabs(p[q]);
        maxd = (a != a || maxd != maxd) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(maxd, a);
      }
    }
  }
}

template <typename T, bool TMA>
__global__ void __launch_bounds__(nthreads<T>(), FTK_S3_MINB)
    k_scan3d(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ ExtractParams P) {
  constexpr int NZW = nzw<T>(), SL = slices<T>(), NSTAGE = nstage<T>();
  constexpr int PRODUCER = NZW * SPLIT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t mis = smem_u32(smem_raw) & 127u;
  Smem<T>& sm = *reinterpret_cast<Smem<T>*>(smem_raw + (mis ? 128 - mis : 0));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const i64 nx = P.nx, ny = P.ny, nz = P.nz;
  constexpr uint32_t STAGE_BYTES = PITCH * ROWS * SL * sizeof(T);
  const int ntx = (int)((nx + TX - 1) / TX), nty = (int)((ny + RW - 1) / RW), ntz = (int)((nz + NZW - 1) / NZW);
  const int tch = (int)P.tchunk;  // anchor timesteps per work item (set by the launcher)
  const int ntc = (int)((P.tb - P.ta + tch - 1) / tch);
  const long long nitems = (long long)ntx * nty * ntz * ntc;
  if (tid == 0) {
    sm.surv = 0;
    sm.maxbits32 = 0;
    sm.maxbits64 = 0;
    for (int i = 0; i < 3; ++i) sm.need[i][0] = sm.need[i][1] = 0ull;
    sm.have[0] = sm.have[1] = 0ull;
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], NZW * SPLIT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == PRODUCER) {
    const T* field = reinterpret_cast<const T*>(P.field);
    int gk = 0;
    while (true) {
      long long item = 0;
      if (lane == 0) item = (long long)atomicAdd(&P.counters[CNT_WORK], 1ull);
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item >= nitems) break;
      long long r = item;
      const int tx = (int)(r % ntx); r /= ntx;
      const int ty_ = (int)(r % nty); r /= nty;
      const int tz = (int)(r % ntz); r /= ntz;
      const i64 x0 = (i64)tx * TX, y0 = (i64)ty_ * RW, z0 = (i64)tz * NZW;
      const i64 ta = P.ta + r * tch;
      const i64 tb = min(ta + tch, P.tb);
      const i64 plast = min(tb, P.nt_global - 1);
      const int np = (int)(plast - ta + 1);
      for (int k = 0; k < np; ++k, ++gk) {
        const int s = gk % NSTAGE;
        if (gk >= NSTAGE) mbar_wait_sleep(&sm.empty[s], (uint32_t)((gk / NSTAGE - 1) & 1), 1, gk);
        if (lane == 0) {
          Meta& m = sm.meta[s];
          m.x0 = (int)x0; m.y0 = (int)y0; m.z0 = (int)z0;
          m.p = (int)(ta + k); m.k = k; m.nplanes = np; m.tb = (int)tb; m.done = 0;
        }
        if (TMA) {
          if (lane == 0) {
            mbar_expect_tx(&sm.full[s], STAGE_BYTES);
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
                    smem_u32(sm.plane[s])),
                "l"(&tmap), "r"(smem_u32(&sm.full[s])), "r"((int)(x0 - XOFF)), "r"((int)(y0 - 1)), "r"((int)(z0 - 1)),
                "r"((int)(ta + k - P.t0))
                : "memory");
          }
        } else {
          const T* src = field + (ta + k - P.t0) * nx * ny * nz;
          T* dst = sm.plane[s];
          for (int idx = lane; idx < PITCH * ROWS * SL; idx += 32) {
            const int xx = idx % PITCH, yy = (idx / PITCH) % ROWS, zz = idx / (PITCH * ROWS);
            const i64 gx = x0 - XOFF + xx, gy = y0 - 1 + yy, gz = z0 - 1 + zz;
            dst[idx] = (gx >= 0 && gx < nx && gy >= 0 && gy < ny && gz >= 0 && gz < nz) ? src[(gz * ny + gy) * nx + gx] : (T)0;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.full[s]);
        }
      }
    }
    const int s = gk % NSTAGE;
    if (gk >= NSTAGE) mbar_wait_sleep(&sm.empty[s], (uint32_t)((gk / NSTAGE - 1) & 1), 1, gk);
    if (lane == 0) {
      sm.meta[s].done = 1;
      mbar_arrive(&sm.full[s]);
    }
  } else {
    // scan warps: warp w owns the hypercubes anchored at slice z0 + w / SPLIT, rows y0 + r0 .. y0 + r0 +
    // NR - 1 (r0 = NR (w % SPLIT))
    const int slice = warp / SPLIT, part = warp % SPLIT, r0 = part * NR;
    const T thr = (T)P.thr;
    const f2 thr2 = pack2((float)P.thr, (float)P.thr);
    const f2 nthr2 = pack2(-(float)P.thr, -(float)P.thr);
    uint32_t maxb32 = 0;
    double maxd = 0.0;
    unsigned long long mysurv = 0;
    long long cur = 0, end = 0;
    const uint32_t lt_mask = (1u << lane) - 1u;
    auto enqueue = [&](uint32_t mask, int tflag, int x0, int y0, int z) {
      const uint32_t bal = __ballot_sync(0xffffffffu, mask != 0);
      if (bal == 0u) return;
      if (__all_sync(0xffffffffu, (mask & (mask - 1u)) == 0u)) {
        // common case: at most one survivor per lane -- ranks from the ballot, no warp scan
        const int n = __popc(bal), rank = __popc(bal & lt_mask);
        const int avail = (int)(end - cur);
        long long e = cur + rank;
        if (n > avail) {  // the chunk runs out: the rest goes to a fresh chunk (n <= 32 = CHUNK)
          long long cc = 0;
          if (lane == 0) cc = (long long)atomicAdd(&P.counters[CNT_WIN], (unsigned long long)CHUNK);
          cc = __shfl_sync(0xffffffffu, cc, 0);
          if (rank >= avail) {
            // entries [cur, end) of the old chunk are filled by the lanes of rank < avail
            e = cc + (rank - avail);
          }
          cur = cc + (n - avail);
          end = cc + CHUNK;
        } else {
          cur += n;
        }
        if (mask != 0u && e < P.wcap) {
          const int bb = __ffs(mask) - 1;
          P.wx[e] = x0 + 4 * lane + (bb >> 3);
          P.wy[e] = y0 + (bb & 7);
          P.wz[e] = z;
          P.wt[e] = tflag;
        }
        mysurv += n;
        return;
      }
      while (__any_sync(0xffffffffu, mask != 0)) {
        if (cur == end) {
          long long cc = 0;
          if (lane == 0) cc = (long long)atomicAdd(&P.counters[CNT_WIN], (unsigned long long)CHUNK);
          cur = __shfl_sync(0xffffffffu, cc, 0);
          end = cur + CHUNK;
        }
        const int cnt = __popc(mask);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        const int n = (int)min((long long)total, end - cur);
        int r = incl - cnt;
        while (mask && r < n) {
          const int bb = __ffs(mask) - 1;
          mask &= mask - 1;
          const long long e = cur + r++;
          if (e < P.wcap) {
            P.wx[e] = x0 + 4 * lane + (bb >> 3);
            P.wy[e] = y0 + (bb & 7);
            P.wz[e] = z;
            P.wt[e] = tflag;
          }
        }
        cur += n;
        mysurv += n;
      }
    };
    Ctx c;  // slice z0 + slice (the warp's own; region test and enqueue)
    c.lane = lane;
    c.ny = ny;
    c.nz = nz;
    int gk = 0, x0 = 0, y0 = 0, z0 = 0;
    int mode = 0;
    bool xedge = false, yedge = false;
    int chk_k = -1, chk_p = -1;  // FTK_CHECKS: the previous plane of the item
    c.xe_out = false;
    c.xe_last = false;
    f2 nan01 = pack2(0.f, 0.f), nan23 = nan01;  // NaN on the lane's out-of-grid positions (region test)
    int prev_s = -1;     // stage of the previous plane of the item (held until this plane is done)
    uint32_t prevR = 0;  // region code of the previous plane
    auto survivors_of = [&](const uint32_t* Q) {
      uint32_t mask = 0;
#pragma unroll
      for (int r = 0; r < NR; ++r) mask |= (((Q[r] - 0x01010101u) & ~Q[r] & 0x80808080u) >> (7 - r));
      return mask;
    };
    // squares of task part h (rows NRT h ..) of slice z0 + j of the plane in stage st into sq[par][j]
    auto squares_task = [&](int st, int j, int h, int par) {
      Ctx cj = c;
      cj.gz = z0 + j;
      cj.gy0 = y0 + h * NRT;
      const bool zedge = cj.gz < 1 || cj.gz + 1 >= nz;
      const int md = (yedge || zedge) ? 2 : (xedge ? 1 : 0);
      const T* S = sm.plane[st] + (j + 1) * (PITCH * ROWS) + h * NRT * PITCH;  // slice z0 + j, row y0 + NRT h - 1
      uint32_t Sq[NRT];
      if (md == 2) slice_squares<T, 2, NRT>(S, PITCH * ROWS, cj, thr2, nthr2, thr, Sq, maxb32, maxd, false);
      else if (md == 1) slice_squares<T, 1, NRT>(S, PITCH * ROWS, cj, thr2, nthr2, thr, Sq, maxb32, maxd, false);
      else slice_squares<T, 0, NRT>(S, PITCH * ROWS, cj, thr2, nthr2, thr, Sq, maxb32, maxd, false);
#pragma unroll
      for (int r = 0; r < NRT; ++r) sm.sq[par][j][h * NRT + r][lane] = Sq[r];
    };
    while (true) {
      const int s = gk % NSTAGE;
      mbar_wait(&sm.full[s], (uint32_t)((gk / NSTAGE) & 1), 3, gk, FTK_K1_MBSLEEP);
      const Meta m = sm.meta[s];
      if (m.done) break;
      // protocol: within a work item the planes arrive in order (a stage refilled too early shows here)
      FTK_ASSERT(m.k == 0 || (m.k == chk_k + 1 && m.p == chk_p + 1));
      chk_k = m.k;
      chk_p = m.p;
      if (m.k == 0) {
        x0 = m.x0;
        y0 = m.y0;
        z0 = m.z0;
        const i64 gx = (i64)x0 + 4 * lane;
        c.gy0 = y0 + r0;
        c.gz = z0 + slice;
        c.lpat = gx == 0;
        c.rpos = (nx - 1 >= gx && nx - 1 <= gx + 3) ? (int)(nx - 1 - gx) : -1;
        c.oob = 0;
        float nanv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool out = gx + i >= nx;
          if (out) c.oob |= 0xFCu << (8 * i);
          nanv[i] = out ? __int_as_float(0x7fc00000) : 0.f;
        }
        nan01 = pack2(nanv[0], nanv[1]);
        nan23 = pack2(nanv[2], nanv[3]);
        xedge = x0 < 1 || x0 + LX + 2 > nx;
        yedge = y0 < 1 || y0 + RW + 2 > ny;
        // region test: both slices of the warp's hypercubes (z, z + 1) z-interior (central dz)
        const bool zedge = c.gz < 1 || c.gz + 2 >= nz;
        mode = (yedge || zedge) ? 2 : (xedge ? 1 : 0);
        c.xe_out = x0 + LX >= nx;
        c.xe_last = x0 + LX == nx - 1;
        prevR = 0;
      }
      const int par = gk & 1;
      // 1. region test (and the range statistics of the owned vertices)
      uint32_t R = 0;
      if (sizeof(T) == 4 && FTK_S3_REGION && mode <= 1) {
        const float* S = reinterpret_cast<const float*>(sm.plane[s]) + slice * (PITCH * ROWS) + (r0 + 1) * PITCH;  // slice z - 1, row y0 + r0
        R = mode == 1 ? region_dz<1>(S, c, (float)P.thr, nan01, nan23, maxb32)
                      : region_dz<0>(S, c, (float)P.thr, nan01, nan23, maxb32);
      } else {
        owned_max<T>(sm.plane[s] + (slice + 1) * (PITCH * ROWS) + (r0 + 1) * PITCH, lane, maxb32, maxd);
      }
      const bool inz = z0 + slice < nz;
      const bool lastg = m.p == P.nt_global - 1 && m.p < m.tb;
      const bool pair = inz && m.k > 0 && (prevR & R) == 0 && !FTK_S3_NOCODES;  // anchors at p - 1
      const bool single = inz && lastg && R == 0 && !FTK_S3_NOCODES;           // anchors at p (no t + 1)
      if (FTK_S3_COUNT && lane == 0 && inz && m.k > 0) {
        atomicAdd(&P.counters[CNT_PROF + 0], 1ull);                    // plane pairs
        if (prevR & R) atomicAdd(&P.counters[CNT_PROF + 1], 1ull);    // rejected by the region test
        if (mode == 2) atomicAdd(&P.counters[CNT_PROF + 3], 1ull);
      }
      // 2. the CTA's squares tasks for this plane: slices z, z + 1 of every warp with a pair or single
      //    (this plane), and of every pair (the previous plane, unless computed there)
      const int slot = gk % 3;
      // the task parts covering the warp's rows, of slices z and z + 1
      const unsigned long long parts = ((1ull << (NR / NRT)) - 1ull) << (r0 / NRT);
      const unsigned long long mybits = (parts << (TP * slice)) | (parts << (TP * (slice + 1)));
      if (lane == 0 && (pair || single)) {
        atomicOr(&sm.need[slot][0], mybits);
        if (pair) atomicOr(&sm.need[slot][1], mybits);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(NZW * SPLIT * 32) : "memory");
      const unsigned long long needc = sm.need[slot][0];
      const unsigned long long needp = m.k > 0 ? sm.need[slot][1] & ~sm.have[par ^ 1] : 0ull;
      // the slot of plane gk + 2 was last read at plane gk - 1, which every warp has left
      if (warp == 0 && lane == 0) sm.need[(gk + 2) % 3][0] = sm.need[(gk + 2) % 3][1] = 0ull;
      const int nc = __popcll(needc), ntask = nc + __popcll(needp);
      if (ntask) {
        for (int i = warp; i < ntask; i += NZW * SPLIT) {
          const bool cur_plane = i < nc;
          unsigned long long mm = cur_plane ? needc : needp;
          for (int r = cur_plane ? i : i - nc; r > 0; --r) mm &= mm - 1;
          const int b = __ffsll((long long)mm) - 1;
          squares_task(cur_plane ? s : prev_s, b / TP, b % TP, cur_plane ? par : par ^ 1);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NZW * SPLIT * 32) : "memory");
        // 3. the owner ANDs the z-pair (and the t-pair) and hands the survivors on
        if (pair) {
          uint32_t Q[NR];
#pragma unroll
          for (int r = 0; r < NR; ++r)
            Q[r] = sm.sq[par ^ 1][slice][r0 + r][lane] & sm.sq[par ^ 1][slice + 1][r0 + r][lane] &
                   sm.sq[par][slice][r0 + r][lane] & sm.sq[par][slice + 1][r0 + r][lane];
          enqueue(survivors_of(Q), (int)((uint32_t)(m.p - 1) | 0x80000000u), x0, y0 + r0, z0 + slice);
        }
        if (single) {
          uint32_t Q[NR];
#pragma unroll
          for (int r = 0; r < NR; ++r) Q[r] = sm.sq[par][slice][r0 + r][lane] & sm.sq[par][slice + 1][r0 + r][lane];
          enqueue(survivors_of(Q), m.p, x0, y0 + r0, z0 + slice);
        }
        // (sq[par ^ 1] is rewritten only after the next plane's first barrier, when every warp is
        // past these reads)
      }
      if (warp == 0 && lane == 0) sm.have[par] = needc;  // squares of this plane, for the next plane's pairs
      __syncwarp();
      if (lane == 0) {
        if (m.k > 0) mbar_arrive(&sm.empty[prev_s]);         // the previous plane is done with
        if (m.k == m.nplanes - 1) mbar_arrive(&sm.empty[s]);  // the item's last plane: nothing follows
      }
      prev_s = s;
      prevR = R;
      ++gk;
    }
    for (long long e = cur + lane; e < end; e += 32)
      if (e < P.wcap) P.wt[e] = -1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      maxb32 = max(maxb32, __shfl_xor_sync(0xffffffffu, maxb32, o));
      const double od = __shfl_xor_sync(0xffffffffu, maxd, o);
      maxd = (od != od || maxd != maxd) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(maxd, od);
    }
    if (lane == 0) {
      atomicAdd(&sm.surv, mysurv);
      atomicMax(&sm.maxbits32, maxb32);
      atomicMax(&sm.maxbits64, (unsigned long long)__double_as_longlong(maxd));
    }
  }
  __syncthreads();
  if (tid == 0) {
    atomicAdd(&P.counters[CNT_SURVIVORS], sm.surv);
    atomicMax(&P.counters[CNT_MAXBITS], sizeof(T) == 4 ? (unsigned long long)sm.maxbits32 : sm.maxbits64);
  }
}
}  // namespace s3

// ------------------------------------------------------------------------------ K1a (3D vector field)
// FTK_VECTOR_FIELD, [t][z][y][x][3]: no stencil, so a plain warp-persistent scan (as k_scanvec2d): a
// work item is a 128 x 8 x 1 anchor tile (x, y, z0) x a chunk of timesteps; per plane the warp codes
// the slices z0 and z0 + 1 (9 rows each, plus their column x0 + 128), 6-bit "strict sign holds" codes
// (u, v, w against +-2^-s; bits 7..2, 0xFC neutral), ANDs y- and x-pairs in registers, the z-pair of
// the two slices and the t-pair with the previous plane; a zero byte is a surviving hypercube, handed
// to k_exact3d<T, true> one entry per hypercube.
namespace v3 {
constexpr int LX = 128, RW = 8, CHUNK = 32;
constexpr uint32_t NEUTRAL = 0xFCFCFCFCu;

template <typename T>
__device__ __forceinline__ uint32_t vcode3(T u, T v, T w, T thr) {
  auto sb = [](T a) -> uint32_t {
    if constexpr (sizeof(T) == 4) return __float_as_uint(a) >> 31;
    else return (uint32_t)((unsigned long long)__double_as_longlong(a) >> 63);
  };
  return (sb(thr - u) << 7) | (sb(u + thr) << 6) | (sb(thr - v) << 5) | (sb(v + thr) << 4) | (sb(thr - w) << 3) |
         (sb(w + thr) << 2);
}

template <typename T>
__device__ __forceinline__ void track_max(T a, uint32_t& maxb, double& maxd) {
  if constexpr (sizeof(T) == 4) {
    maxb = max(maxb, __float_as_uint(a) & 0x7fffffffu);
  } else {
    const double x = fabs(a);
    maxd = (x != x || maxd != maxd) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(maxd, x);
  }
}

template <typename T>
__device__ __forceinline__ uint32_t row_code(const T* plane, i64 nx, i64 ny, i64 nz, i64 y, i64 z, i64 xl, T thr,
                                             bool aligned, uint32_t& maxb, double& maxd) {
  if (y >= ny || z >= nz) return NEUTRAL;
  const T* r = plane + 3 * ((z * ny + y) * nx + xl);
  T q[12];
  if (xl + 3 < nx && aligned) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(r));
    const float4 b = __ldg(reinterpret_cast<const float4*>(r + 4));
    const float4 c = __ldg(reinterpret_cast<const float4*>(r + 8));
    q[0] = a.x; q[1] = a.y; q[2] = a.z; q[3] = a.w; q[4] = b.x; q[5] = b.y;
    q[6] = b.z; q[7] = b.w; q[8] = c.x; q[9] = c.y; q[10] = c.z; q[11] = c.w;
  } else {
#pragma unroll
    for (int k = 0; k < 12; ++k) q[k] = xl + k / 3 < nx ? __ldg(r + k) : (T)0;
  }
  uint32_t code = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool in = xl + i < nx;
    code |= (in ? vcode3<T>(q[3 * i], q[3 * i + 1], q[3 * i + 2], thr) : 0xFCu) << (8 * i);
    if (in) {
      track_max<T>(q[3 * i], maxb, maxd);
      track_max<T>(q[3 * i + 1], maxb, maxd);
      track_max<T>(q[3 * i + 2], maxb, maxd);
    }
  }
  return code;
}

// a work item is 128 x 8 x NZ anchors: the warp rolls through the NZ + 1 slices of each plane (each
// slice coded once), keeping the previous plane's NZ x 8 cube codes in shared memory for the t-pair
constexpr int NZ = 8;
#ifndef FTK_V3_MINB
#define FTK_V3_MINB 3  // 3 blocks of 8 warps per SM (measured on V5: 4.69 -> 3.87 ms)
#endif
template <typename T>
__global__ void __launch_bounds__(256, FTK_V3_MINB) k_scanvec3d(const __grid_constant__ ExtractParams P) {
  extern __shared__ uint32_t prevK_all[];  // [warp][NZ][RW][32]
  const int lane = threadIdx.x & 31;
  uint32_t* prevK = prevK_all + (threadIdx.x >> 5) * (NZ * RW * 32);
  const i64 nx = P.nx, ny = P.ny, nz = P.nz;
  const int ntx = (int)((nx + LX - 1) / LX), nty = (int)((ny + RW - 1) / RW);
  const int tch = (int)P.tchunk;
  const int ntc = (int)((P.tb - P.ta + tch - 1) / tch);
  const int ntz = (int)((nz + NZ - 1) / NZ);
  const long long nitems = (long long)ntx * nty * ntz * ntc;
  const T thr = (T)P.thr;
  const T* F = reinterpret_cast<const T*>(P.field);
  const bool aligned = sizeof(T) == 4 && (nx % 4 == 0) && ((reinterpret_cast<uintptr_t>(F) & 15) == 0);
  const uint32_t lt_mask = (1u << lane) - 1u;
  long long cur = 0, end = 0;
  unsigned long long mysurv = 0;
  uint32_t maxb = 0;
  double maxd = 0.0;
  // one list entry per surviving hypercube (survivors are rare in 3D): ranks from a ballot when every
  // lane has at most one, else one lane-serial round per survivor bit
  auto enqueue = [&](uint32_t mask, int tflag, int xl, int y0, int z) {
    while (__any_sync(0xffffffffu, mask != 0)) {
      const uint32_t bit = mask & (0u - mask);
      const uint32_t bal = __ballot_sync(0xffffffffu, bit != 0);
      const int n = __popc(bal), rank = __popc(bal & lt_mask);
      const int avail = (int)(end - cur);
      long long e = cur + rank;
      if (n > avail) {
        long long c = 0;
        if (lane == 0) c = (long long)atomicAdd(&P.counters[CNT_WIN], (unsigned long long)CHUNK);
        c = __shfl_sync(0xffffffffu, c, 0);
        if (rank >= avail) e = c + (rank - avail);
        cur = c + (n - avail);
        end = c + CHUNK;
      } else {
        cur += n;
      }
      if (bit && e < P.wcap) {
        const int bb = __ffs(bit) - 1;
        P.wx[e] = xl + (bb >> 3);
        P.wy[e] = y0 + (bb & 7);
        P.wz[e] = z;
        P.wt[e] = tflag;
      }
      mysurv += n;
      mask &= mask - 1;
    }
  };
  while (true) {
    long long item = 0;
    if (lane == 0) item = (long long)atomicAdd(&P.counters[CNT_WORK], 1ull);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= nitems) break;
    long long r = item;
    const int tx = (int)(r % ntx); r /= ntx;
    const int ty = (int)(r % nty); r /= nty;
    const i64 z0 = (r % ntz) * NZ; r /= ntz;
    const i64 x0 = (i64)tx * LX, y0 = (i64)ty * RW;
    const i64 ta = P.ta + r * tch, tb = min(ta + tch, P.tb);
    const i64 plast = min(tb, P.nt_global - 1);
    const i64 xl = x0 + 4 * lane;
    for (i64 p = ta; p <= plast; ++p) {
      const T* plane = F + (p - P.t0) * nx * ny * nz * 3;
      // squares (y- and x-pairs) of slice z
      auto slice_sq = [&](i64 z, uint32_t (&Sq)[RW]) {
        uint32_t C[RW + 1];
#pragma unroll
        for (int rr = 0; rr <= RW; ++rr) C[rr] = row_code<T>(plane, nx, ny, nz, y0 + rr, z, xl, thr, aligned, maxb, maxd);
        uint32_t Ye;
        {
          const int k = min(lane, RW);
          const i64 y = y0 + k, x = x0 + LX;
          uint32_t ce = 0xFCu;
          if (x < nx && y < ny && z < nz) {
            const T* q = plane + 3 * ((z * ny + y) * nx + x);
            ce = vcode3<T>(__ldg(q), __ldg(q + 1), __ldg(q + 2), thr);
          }
          Ye = ce & __shfl_down_sync(0xffffffffu, ce, 1);
        }
#pragma unroll
        for (int rr = 0; rr < RW; ++rr) {
          const uint32_t Y = C[rr] & C[rr + 1];
          uint32_t nb = __shfl_down_sync(0xffffffffu, Y, 1);
          const uint32_t ne = __shfl_sync(0xffffffffu, Ye, rr);
          if (lane == 31) nb = ne;
          Sq[rr] = Y & ((Y >> 8) | (nb << 24));
        }
      };
      auto survivors_of = [&](const uint32_t* Q) {
        uint32_t mask = 0;
#pragma unroll
        for (int rr = 0; rr < RW; ++rr) mask |= (((Q[rr] - 0x01010101u) & ~Q[rr] & 0x80808080u) >> (7 - rr));
        return mask;
      };
      uint32_t Sa[RW], Sb[RW];
      slice_sq(z0, Sa);
#pragma unroll 1
      for (int dz = 0; dz < NZ; ++dz) {
        const i64 z = z0 + dz;
        if (z >= nz) break;
        slice_sq(z + 1, Sb);
        uint32_t K[RW];
#pragma unroll
        for (int rr = 0; rr < RW; ++rr) K[rr] = Sa[rr] & Sb[rr];  // z-pair
        uint32_t* pk = prevK + dz * (RW * 32) + lane;
        if (p > ta) {
          uint32_t Q[RW];
#pragma unroll
          for (int rr = 0; rr < RW; ++rr) Q[rr] = pk[rr * 32] & K[rr];
          enqueue(survivors_of(Q), (int)((uint32_t)(p - 1) | 0x80000000u), (int)xl, (int)y0, (int)z);
        }
        if (p == P.nt_global - 1 && p < tb) enqueue(survivors_of(K), (int)p, (int)xl, (int)y0, (int)z);
#pragma unroll
        for (int rr = 0; rr < RW; ++rr) {
          pk[rr * 32] = K[rr];
          Sa[rr] = Sb[rr];
        }
      }
    }
  }
  for (long long e = cur + lane; e < end; e += 32)
    if (e < P.wcap) P.wt[e] = -1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    maxb = max(maxb, __shfl_xor_sync(0xffffffffu, maxb, o));
    const double od = __shfl_xor_sync(0xffffffffu, maxd, o);
    maxd = (od != od || maxd != maxd) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(maxd, od);
  }
  if (lane == 0) {
    atomicAdd(&P.counters[CNT_SURVIVORS], mysurv);
    atomicMax(&P.counters[CNT_MAXBITS],
              sizeof(T) == 4 ? (unsigned long long)maxb : (unsigned long long)__double_as_longlong(maxd));
  }
}
}  // namespace v3

// ------------------------------------------------------------------------------ K1b (3D)
// One warp per surviving hypercube of the list: lanes 0..15 take the 16 corner gradients (exact
// int64, straight from the field), the 60 face types are spread over the lanes (two each) for the
// SoS point-in-simplex test, lanes 0..23 take the 24 cells (pentachora) -- 0 or 2
// punctured sides each, pairs become trajectory edges -- and the punctured faces are
// spread over the lanes for the Eq. 2 location and the Descartes-rule Hessian type in fixed-order
// FP64.  A hypercube's 60 faces with their SoS chains are far too much serial work for one thread.
constexpr int XW3 = 4;  // warps per block

// VEC: a 3D vector field [t][z][y][x][3] (FTK_VECTOR_FIELD): the corner values are the quantized
// vectors themselves and the type comes from the Jacobian (R17)
#ifndef FTK_X3_MINB
#define FTK_X3_MINB 8  // 8 blocks of 4 warps per SM (64 registers, ~240 B spilled to L1; C5 K1b 1.01 -> 0.79 ms, C3 0.107 -> 0.121 ms)
#endif
template <typename T, bool VEC = false>
__global__ void __launch_bounds__(XW3 * 32, FTK_X3_MINB) k_exact3d(const __grid_constant__ ExtractParams P) {
  constexpr int NH = VEC ? 9 : 6;
  __shared__ i64 sg[XW3][16][3];
  __shared__ i64 sH[XW3][16][NH];  // corner Hessians / Jacobians (hypercubes with punctured faces)
  __shared__ i64 sW[XW3][128];     // interior hypercubes: the quantized 4x4x4 x 2-plane window
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
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
  const i64 plane = G.nx * G.ny * G.nz * (VEC ? 3 : 1);
  i64(&g)[16][3] = sg[w];
  // hypercubes are claimed dynamically (one atomic per hypercube and warp): their cost varies with the
  // punctured faces they hold, and a static stride leaves the slowest warps as a tail
  auto claim = [&]() -> long long {
    long long c = 0;
    if (lane == 0) c = (long long)atomicAdd(&P.counters[CNT_XBATCH], 1ull);
    return __shfl_sync(0xffffffffu, c, 0);
  };
  for (long long e = claim(); e < nwin; e = claim()) {
    const int et = P.wt[e];
    if (et == -1) continue;
    const bool hasB = et < 0;
    const i64 t = et & 0x3fffffff;
    const i64 x = P.wx[e], y = P.wy[e], z = P.wz[e];
    const GTile<T> A{field + (t - P.t0) * plane};
    const GTile<T> B{hasB ? A.S + plane : A.S};
    // interior hypercube (scalar field): the window x-1..x+2, y-1..y+2, z-1..z+2 of planes t, t+1,
    // quantized once into shared memory (4 values per lane); every corner is an interior vertex, so
    // its central differences and compact Hessian stencil read the window only
    const bool inner = !VEC && hasB && x >= 1 && x + 2 < G.nx && y >= 1 && y + 2 < G.ny && z >= 1 && z + 2 < G.nz;
    i64* W = sW[w];
    auto wat = [&](int pl, int zz, int yy, int xx) -> i64 { return W[pl * 64 + zz * 16 + yy * 4 + xx]; };
    if (inner) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = lane * 4 + j;
        const int xx = k & 3, yy = (k >> 2) & 3, zz = (k >> 4) & 3, pl = k >> 6;
        W[k] = quant3((pl ? B : A).at(G, x - 1 + xx, y - 1 + yy, z - 1 + zz), G);
      }
      __syncwarp();
    }
    // corner gradients
    uint32_t ex = 0;
    {
      const int c = lane & 15;
      const i64 cx = x + (c & 1), cy = y + ((c >> 1) & 1), cz = z + ((c >> 2) & 1);
      const bool e1 = cx < G.nx && cy < G.ny && cz < G.nz && ((c & 8) == 0 || hasB);
      if (lane < 16) {
        i64 gc[3] = {0, 0, 0};
        if (inner) {
          const int lx = 1 + (c & 1), ly = 1 + ((c >> 1) & 1), lz = 1 + ((c >> 2) & 1), pl = c >> 3;
          gc[0] = wat(pl, lz, ly, lx + 1) - wat(pl, lz, ly, lx - 1);
          gc[1] = wat(pl, lz, ly + 1, lx) - wat(pl, lz, ly - 1, lx);
          gc[2] = wat(pl, lz + 1, ly, lx) - wat(pl, lz - 1, ly, lx);
        } else if (e1) {
          if constexpr (VEC) {
            const T* q = ((c & 8) ? B : A).S + ((cz * G.ny + cy) * G.nx + cx) * 3;
#pragma unroll
            for (int j = 0; j < 3; ++j) gc[j] = quant3(__ldg(q + j), G);
          } else {
            grad3<T>((c & 8) ? B : A, G, cx, cy, cz, gc);
          }
        }
        g[c][0] = gc[0];
        g[c][1] = gc[1];
        g[c][2] = gc[2];
      }
      ex = __ballot_sync(0xffffffffu, lane < 16 && e1);
    }
    __syncwarp();
    // all 48 gradient components below 2^26 in magnitude: the FP64 determinant filter applies
    bool small, mid;
    {
      const int c = lane & 15;
      const i64 lim = 1ll << 26, lim31 = 1ll << 31;
      small = __all_sync(0xffffffffu, g[c][0] > -lim && g[c][0] < lim && g[c][1] > -lim && g[c][1] < lim &&
                                          g[c][2] > -lim && g[c][2] < lim);
      mid = __all_sync(0xffffffffu, g[c][0] > -lim31 && g[c][0] < lim31 && g[c][1] > -lim31 && g[c][1] < lim31 &&
                                        g[c][2] > -lim31 && g[c][2] < lim31);
    }
    // the 60 face types, two per lane
    unsigned long long pmask = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ty = lane + 32 * h;
      bool pu = false;
      if (ty < 60) {
        const int m1 = cK4.masks[ty][0], m2 = cK4.masks[ty][1], m3 = cK4.masks[ty][2];
        if ((ex >> m3) & 1) {
          const i64 gv[4][3] = {{g[0][0], g[0][1], g[0][2]}, {g[m1][0], g[m1][1], g[m1][2]},
                                {g[m2][0], g[m2][1], g[m2][2]}, {g[m3][0], g[m3][1], g[m3][2]}};
          bool rej = false;  // exact sign reject: one component of one strict sign on all vertices
#pragma unroll
          for (int j = 0; j < 3; ++j)
            rej |= (gv[0][j] > 0 && gv[1][j] > 0 && gv[2][j] > 0 && gv[3][j] > 0) ||
                   (gv[0][j] < 0 && gv[1][j] < 0 && gv[2][j] < 0 && gv[3][j] < 0);
          pu = !rej && punctured4(gv, small, mid);
        }
      }
      pmask |= (unsigned long long)__ballot_sync(0xffffffffu, pu) << (32 * h);
    }
    const int npunct = __popcll(pmask);
    if (npunct) {  // integer Hessians of the 16 corners, one per lane, for the records below
      const int c = lane & 15;
      if (lane < 16 && ((ex >> c) & 1))
      {
        if constexpr (VEC) {
          jac3<T>(P, G, x + (c & 1), y + ((c >> 1) & 1), z + ((c >> 2) & 1), t + ((c >> 3) & 1), sH[w][c]);
        } else if (inner) {  // compact stencil inside the window (order xx xy xz yy yz zz, as hess3)
          const int l[3] = {1 + (c & 1), 1 + ((c >> 1) & 1), 1 + ((c >> 2) & 1)};
          const int pl = c >> 3;
          auto q = [&](int dx, int dy, int dz) { return wat(pl, l[2] + dz, l[1] + dy, l[0] + dx); };
          i64* H = sH[w][c];
          H[0] = 4 * (q(1, 0, 0) - 2 * q(0, 0, 0) + q(-1, 0, 0));
          H[1] = q(1, 1, 0) - q(1, -1, 0) - q(-1, 1, 0) + q(-1, -1, 0);
          H[2] = q(1, 0, 1) - q(1, 0, -1) - q(-1, 0, 1) + q(-1, 0, -1);
          H[3] = 4 * (q(0, 1, 0) - 2 * q(0, 0, 0) + q(0, -1, 0));
          H[4] = q(0, 1, 1) - q(0, 1, -1) - q(0, -1, 1) + q(0, -1, -1);
          H[5] = 4 * (q(0, 0, 1) - 2 * q(0, 0, 0) + q(0, 0, -1));
        } else {
          hess3<T>(P, G, x + (c & 1), y + ((c >> 1) & 1), z + ((c >> 2) & 1), t + ((c >> 3) & 1), sH[w][c]);
        }
      }
      __syncwarp();
    }
    unsigned long long rbase = 0;
    if (lane == 0 && npunct) rbase = atomicAdd(&P.counters[CNT_NOUT], (unsigned long long)npunct);
    rbase = __shfl_sync(0xffffffffu, rbase, 0);
    // cells: only full hypercubes have cells anchored here
    const bool full = x + 1 < G.nx && y + 1 < G.ny && z + 1 < G.nz && hasB;
    if (full) {
      int k = 0;
      long long ends[2] = {-1, -1};
      if (lane < 24) {
        const Cell4& cd = cCells4.c[lane];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if ((pmask >> cd.own[q]) & 1ull) {
            if (k < 2) ends[k] = (long long)(rbase + __popcll(pmask & ((1ull << cd.own[q]) - 1ull)));
            ++k;
          }
        // upper face (w1, w2, w3, 15), owned by the neighbour hypercube: a cell holds 0 or 2 punctured
        // faces (SoS), so with k own faces punctured the upper one is punctured iff
        // k == 1 -- no test needed.  (Were the invariant ever broken, the edge would name a face no
        // record has and pass 2 reports FTK_ERR_INVARIANT; k > 2 is caught right here.)
        if (k == 1) {
          if (k < 2) {
            const int a1 = cd.w[1];
            const i64 fx = x + (a1 & 1), fy = y + ((a1 >> 1) & 1), fz = z + ((a1 >> 2) & 1), ft = t + ((a1 >> 3) & 1);
            ends[k] = -1 - ((((ft * G.nz + fz) * G.ny + fy) * G.nx + fx) * 60 + cd.up_type);
          }
          ++k;
        }
      }
      const uint32_t pairs = __ballot_sync(0xffffffffu, k == 2);
      const uint32_t bad = __ballot_sync(0xffffffffu, k != 0 && k != 2);
      if (lane == 0 && bad) atomicAdd(&P.counters[CNT_INVARIANT], (unsigned long long)__popc(bad));
      if (pairs) {
        unsigned long long eb = 0;
        if (lane == 0) eb = atomicAdd(&P.counters[CNT_EDGES], (unsigned long long)__popc(pairs));
        eb = __shfl_sync(0xffffffffu, eb, 0);
        if (k == 2) {
          const unsigned long long es = eb + __popc(pairs & ((1u << lane) - 1u));
          if (es < (unsigned long long)P.capacity) {
            P.edges[2 * es] = ends[0] >= 0 ? ends[0] : ends[1];
            P.edges[2 * es + 1] = ends[0] >= 0 ? ends[1] : ends[0];
          }
        }
      }
    }
    // records: the punctured faces spread over the lanes
    for (int i = lane; i < npunct; i += 32) {
      unsigned long long pm = pmask;
      for (int j = 0; j < i; ++j) pm &= pm - 1;
      const int ty = __ffsll((long long)pm) - 1;
      const unsigned long long slot = rbase + i;
      const int m[4] = {0, cK4.masks[ty][0], cK4.masks[ty][1], cK4.masks[ty][2]};
      i64 gv[4][3];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int j = 0; j < 3; ++j) gv[kk][j] = g[m[kk]][j];
      // D_k = (-1)^(k+3) det(rows != k)  (Eq. 2)
      const i128 D0 = -(mid ? det3_mid(gv[1], gv[2], gv[3]) : det3(gv[1], gv[2], gv[3]));
      const i128 D1 = mid ? det3_mid(gv[0], gv[2], gv[3]) : det3(gv[0], gv[2], gv[3]);
      const i128 D2 = -(mid ? det3_mid(gv[0], gv[1], gv[3]) : det3(gv[0], gv[1], gv[3]));
      const i128 D3 = mid ? det3_mid(gv[0], gv[1], gv[2]) : det3(gv[0], gv[1], gv[2]);
      const i128 S = D0 + D1 + D2 + D3;
      double mu[4];
      uint32_t flags = 0;
      if (S == 0) {
        mu[0] = mu[1] = mu[2] = mu[3] = 0.25;
        flags |= FTK_CP_DEGENERATE_LOC;
      } else {
        const double sd = i128_to_double_rn(S);
        mu[0] = __ddiv_rn(i128_to_double_rn(D0), sd);
        mu[1] = __ddiv_rn(i128_to_double_rn(D1), sd);
        mu[2] = __ddiv_rn(i128_to_double_rn(D2), sd);
        mu[3] = __ddiv_rn(i128_to_double_rn(D3), sd);
      }
      double pv[4][4];  // x, y, z, t of each vertex
      double Hd[NH][4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const i64 vx = x + (m[kk] & 1), vy = y + ((m[kk] >> 1) & 1), vz = z + ((m[kk] >> 2) & 1),
                  vt = t + ((m[kk] >> 3) & 1);
        pv[0][kk] = (double)vx;
        pv[1][kk] = (double)vy;
        pv[2][kk] = (double)vz;
        pv[3][kk] = (double)vt;
#pragma unroll
        for (int q = 0; q < NH; ++q) Hd[q][kk] = __ll2double_rn(sH[w][m[kk]][q]);
      }
      double Hb[NH];
#pragma unroll
      for (int q = 0; q < NH; ++q) Hb[q] = dot4_nofma(mu, Hd[q]);
      const int type = VEC ? classify_vec3(Hb) : classify3(Hb);
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
    __syncwarp();
  }
}

}  // namespace k3d

template <typename T, bool TMA>
static int launch3_t(const ExtractParams& P, cudaStream_t stream) {
  using namespace k3d;
  using namespace k3d::s3;
  CUtensorMap map;
  memset(&map, 0, sizeof map);
  if (TMA) {
    auto enc = sm100::get_encode();
    const cuuint64_t dims[4] = {(cuuint64_t)P.nx, (cuuint64_t)P.ny, (cuuint64_t)P.nz, (cuuint64_t)P.nt_buf};
    const cuuint64_t strides[3] = {(cuuint64_t)P.nx * sizeof(T), (cuuint64_t)P.nx * P.ny * sizeof(T),
                                   (cuuint64_t)P.nx * P.ny * P.nz * sizeof(T)};
    const cuuint32_t box[4] = {PITCH, ROWS, (cuuint32_t)slices<T>(), 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(&map, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                     const_cast<void*>(P.field), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return launch3_t<T, false>(P, stream);
  }
  const size_t smem = sizeof(Smem<T>) + 128;
  auto kern = k_scan3d<T, TMA>;
  const sm100::LaunchGeom lg = sm100::launch_geom(kern, nthreads<T>(), smem);
  if (lg.err != cudaSuccess) return set_cuda_error(lg.err, "k_scan3d launch geometry");
  const int sms = lg.sms, per_sm = lg.per_sm;
  const long long tiles = ((P.nx + TX - 1) / TX) * ((P.ny + RW - 1) / RW) * ((P.nz + nzw<T>() - 1) / nzw<T>());
  const long long slots = (long long)sms * std::max(per_sm, 1);
  ExtractParams Q = P;
  Q.tchunk = TCH;  // halved (down to 4) while there would be fewer than 8 work items per CTA: tail balance
  while (Q.tchunk > 4 && tiles * ((P.tb - P.ta + Q.tchunk - 1) / Q.tchunk) < 8 * slots) Q.tchunk /= 2;
  const long long items = tiles * ((P.tb - P.ta + Q.tchunk - 1) / Q.tchunk);
  if (items <= 0) return FTK_OK;
  const long long grid = std::min<long long>(items, slots);
  kern<<<(unsigned)grid, nthreads<T>(), smem, stream>>>(map, Q);
  FTK_CUDA_TRY(cudaGetLastError());
  if (P.ev_mid) FTK_CUDA_TRY(cudaEventRecord(reinterpret_cast<cudaEvent_t>(P.ev_mid), stream));
  const sm100::LaunchGeom xg = sm100::launch_geom(k_exact3d<T>, XW3 * 32, 0);
  if (xg.err != cudaSuccess) return set_cuda_error(xg.err, "k_exact3d launch geometry");
  const int xper = xg.per_sm;
  k_exact3d<T><<<(unsigned)(sms * std::max(xper, 1)), XW3 * 32, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

template <typename T>
static int launch_vec3_t(const ExtractParams& P, cudaStream_t stream) {
  using namespace k3d;
  auto scan = v3::k_scanvec3d<T>;
  const size_t smem = 8 * v3::NZ * v3::RW * 32 * sizeof(uint32_t);  // previous-plane cube codes per warp
  const sm100::LaunchGeom lg = sm100::launch_geom(scan, 256, smem);
  if (lg.err != cudaSuccess) return set_cuda_error(lg.err, "k_scanvec3d launch geometry");
  const long long tiles = ((P.nx + v3::LX - 1) / v3::LX) * ((P.ny + v3::RW - 1) / v3::RW) * ((P.nz + v3::NZ - 1) / v3::NZ);
  const long long warps = (long long)lg.sms * lg.per_sm * 8;
  ExtractParams Q = P;
  Q.tchunk = 16;
  while (Q.tchunk > 2 && tiles * ((P.tb - P.ta + Q.tchunk - 1) / Q.tchunk) < 4 * warps) Q.tchunk /= 2;
  const long long items = tiles * ((P.tb - P.ta + Q.tchunk - 1) / Q.tchunk);
  if (items <= 0) return FTK_OK;
  const long long blocks = std::min<long long>((items + 7) / 8, (long long)lg.sms * lg.per_sm);
  scan<<<(unsigned)blocks, 256, smem, stream>>>(Q);
  FTK_CUDA_TRY(cudaGetLastError());
  if (P.ev_mid) FTK_CUDA_TRY(cudaEventRecord(reinterpret_cast<cudaEvent_t>(P.ev_mid), stream));
  const sm100::LaunchGeom xg = sm100::launch_geom(k_exact3d<T, true>, XW3 * 32, 0);
  if (xg.err != cudaSuccess) return set_cuda_error(xg.err, "k_exact3d launch geometry");
  k_exact3d<T, true><<<(unsigned)(lg.sms * std::max(xg.per_sm, 1)), XW3 * 32, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

int launch_extract_vec3d(const ExtractParams& P, cudaStream_t stream) {
  if (P.nx >= (1ll << 31) - 256 || P.ny >= (1ll << 31) - 64 || P.nz >= (1ll << 31) - 64 || P.nt_global >= (1ll << 30))
    return FTK_ERR_INVALID_ARG;
  return P.dtype == FTK_F32 ? launch_vec3_t<float>(P, stream) : launch_vec3_t<double>(P, stream);
}

int launch_extract3d(const ExtractParams& P, cudaStream_t stream) {
  const size_t esz = P.dtype == FTK_F32 ? 4 : 8;
  const bool aligned = (reinterpret_cast<uintptr_t>(P.field) % 16 == 0) && ((P.nx * esz) % 16 == 0);
  const bool tma = aligned && sm100::get_encode() != nullptr && !P.force_generic;
  if (P.nx >= (1ll << 31) - 256 || P.ny >= (1ll << 31) - 64 || P.nz >= (1ll << 31) - 64 || P.nt_global >= (1ll << 30))
    return FTK_ERR_INVALID_ARG;
  if (P.dtype == FTK_F32) return tma ? launch3_t<float, true>(P, stream) : launch3_t<float, false>(P, stream);
  return tma ? launch3_t<double, true>(P, stream) : launch3_t<double, false>(P, stream);
}

}  // namespace ftk
