// extract2d.cu -- K1: pass 1 of Alg. 1 for 2D+t on sm_100a, split into three
// kernels:
//
//   K1a k_scan2d -- persistent, 2 CTAs per SM.  A work item is a 128 x 64 tile of anchors (x, y) times
//     a chunk of anchor timesteps; CTAs pull items from a global counter and march t through them.
//     Warp-specialised:
//     producer warp -- stages each plane of the tile with its halo (x0-4 .. x0+131, y0-1 .. y0+65)
//       into an NSTAGE-deep shared-memory ring with TMA (cp.async.bulk.tensor) under full/empty
//       mbarriers, so every vertex is read from HBM once and reused by all 12 faces of the 8 cubes it
//       belongs to (north_star (2));
//     8 scan warps (8 anchor rows x 128 columns each; lane = 4 consecutive x) -- a CONSERVATIVE sign
//       prefilter on raw field values: for g_a = q[+a] - q[-a] (q = rint(f 2^s)) the float test
//       d = f[+a] - f[-a] > 2^(1-s) implies g_a > 0 exactly, d < -2^(1-s) implies g_a < 0.  The sign
//       bits of 2^(1-s) - d and d + 2^(1-s) (paired FADD2) are gathered into a 4-bit "strict sign
//       holds" code per vertex and ANDed over the 8 corners of each spacetime cube (y-pair in
//       registers, x-pair by one shuffle plus the codes of column x0 + 128, t-pair with the previous
//       plane); a zero byte means no component has one strict sign on every corner, so the cube may
//       hold a punctured face -- a survivor.  A cube with a one-signed component cannot, even under
//       SoS (the perturbation is infinitesimal).  Grid boundaries: neighbour values patched in
//       registers (one-sided differences), out-of-grid positions AND-neutral.  Survivors leave as
//       group entries (one per lane: first anchor, plane flag, 32-bit survivor mask).
//   k_expand2d -- group entries -> dense cube list (one atomic per block).
//   K1b k_exact2d -- one warp per batch of 32 cubes (one per lane): the cube's 4x4x2 window from the
//     field, exact int32 quantization and gradients, the 19 distinct 2x2 determinants of the 12 faces,
//     SoS point-in-simplex (an exact int64/int128 path covers boundary cubes, zero
//     determinants and large values), the 6 cells (in-cube pairs joined, pairs with a neighbour cube's
//     face emitted as edges), then the punctured faces spread over the lanes for the Eq. 2 location
//     and Hessian type in fixed-order FP64 (no FMA).
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "common.cuh"
#include "extract2d.cuh"
#include "kuhn.cuh"
#include "sm100.cuh"

namespace ftk {
namespace k2d {

using namespace sm100;

// ---------------------------------------------------------------------------------------------
// Geometry and roles
// ---------------------------------------------------------------------------------------------
constexpr int LX = 128;             // x positions scanned per warp row (32 lanes x 4)
constexpr int TX = LX;              // anchors owned per tile in x: all 128 columns; lane 31's cubes take
                                    // their x + 1 corners from the codes of column x0 + 128, computed once
                                    // per plane (one row per lane)
#ifndef FTK_K1_RW
#define FTK_K1_RW 8
#endif
constexpr int RW = FTK_K1_RW;       // anchor rows per scan warp (4 or 8)
constexpr int NSW = 8;              // scan warps
constexpr int PRODUCER = NSW;       // warp id of the TMA producer
constexpr int NTHREADS = (NSW + 1) * 32;
constexpr int TY = RW * NSW;        // 32 anchor rows per tile
constexpr int XOFF = 4;             // smem column of x0
constexpr int YOFF = 1;             // smem row of y0
constexpr int PITCH = LX + 8;       // x0-4 .. x0+131
constexpr int ROWS = TY + 3;        // y0-1 .. y0+33
#ifndef FTK_K1_NSTAGE
#define FTK_K1_NSTAGE (RW == 8 ? 3 : 5)
#endif
#ifndef FTK_K1_MINB
#define FTK_K1_MINB 2
#endif
#ifndef FTK_K1_CHUNK
#define FTK_K1_CHUNK 32
#endif
constexpr int CHUNK = FTK_K1_CHUNK; // window-buffer entries a scan warp reserves at a time
#ifndef FTK_K1_TCHUNK
#define FTK_K1_TCHUNK 32
#endif
constexpr int TCHUNK = FTK_K1_TCHUNK;  // anchor timesteps per work item (halved by the launcher when
                                       // there would be fewer than 16 items per CTA: tail balance)
template <typename T>
constexpr int nstage() { return sizeof(T) == 4 ? FTK_K1_NSTAGE : 3; }

template <typename T>
constexpr int stage_elems() {       // plane tile padded to a multiple of 128 bytes (TMA alignment)
  return (ROWS * PITCH * (int)sizeof(T) + 127) / 128 * 128 / (int)sizeof(T);
}

struct StageMeta {                  // written by the producer before the plane lands
  int x0, y0;                       // tile origin
  int p;                            // global timestep of the plane
  int k;                            // index of the plane within its work item
  int nplanes;                      // planes in the work item
  int tb;                           // end of the item's anchor range
  int done;                         // no more work
};

template <typename T>
struct alignas(128) ScanSmem {
  static constexpr int NSTAGE = nstage<T>();
  T plane[NSTAGE][stage_elems<T>()];
  StageMeta meta[NSTAGE];
  uint64_t full[NSTAGE];
  uint64_t empty[NSTAGE];
  unsigned long long surv;
  unsigned int maxbits32;
  unsigned long long maxbits64;
};

// K1b: a batch of 32 cubes per warp.  Entry (32-bit words): [0, 32) the cube's 4x4x2 window
// W[pl*16 + r*4 + c] at (x - 1 + c, y - 1 + r, t + pl) -- as exact int32 q values for fast entries
// (fp32 input, interior cube, |q| < 2^29), else as raw values; [32, 48) the 8 corner gradients
// (fast entries).
template <typename T>
constexpr int ws_words() { return sizeof(T) == 4 ? 49 : 66; }  // odd stride for fp32: no bank conflicts
constexpr int MAXITEMS = 32 * 12;   // punctured faces per batch (upper bound)
constexpr int EXW = 8;              // warps per K1b block
#ifndef FTK_X_MINB
#define FTK_X_MINB 2                // 128 registers: the prefetched window stays in registers
#endif

struct BatchBuf {                   // one warp's batch in shared memory
  uint32_t* ring;                   // [32][ws_words]
  int* qx;
  int* qy;
  int* qt;                          // t | (t+1 exists) << 31 | fast << 30, -1: no cube
  uint16_t* items;                  // punctured faces of the batch: entry | type << 5
  unsigned long long* lp;           // [32] in-cube union-find of each entry (12 x 4-bit parents)
  uint32_t* pm;                     // [32] punctured own faces of each entry
  int* rs;                          // [32] first record of each entry, relative to the batch
};

template <typename T>
struct ExSmem {
  uint32_t ring[EXW * 32 * ws_words<T>()];
  int qx[EXW * 32], qy[EXW * 32], qt[EXW * 32];
  unsigned long long lp[EXW * 32];
  uint32_t pm[EXW * 32];
  int rs[EXW * 32];
  uint16_t items[EXW][MAXITEMS];
};

// ---------------------------------------------------------------------------------------------
// Exact stage
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ i64 quant(float f, float scale_f, double) {
  // f * 2^s is exact in fp32 (power-of-two scale); F2I.S64 rounds half-even
  return __float2ll_rn(__fmul_rn(f, scale_f));
}
__device__ __forceinline__ i64 quant(double f, float, double scale) { return __double2ll_rn(__dmul_rn(f, scale)); }

struct Geo {
  i64 nx, ny, ntg;   // grid extents (t = global)
  float scale_f;
  double scale;
  double qmax;       // |f| below this quantizes to |q| < 2^29 (int32 fast path)
};

template <typename T>
struct Win {  // window value (pl, c, r) = q at (x - 1 + c, y - 1 + r, t + pl)
  const uint32_t* W;
  bool isq;   // fast entry: exact int32 q values and precomputed gradients
  float sf;
  double sd;
  __device__ __forceinline__ i64 q(int pl, int c, int r) const {
    const int k = pl * 16 + r * 4 + c;
    if (isq) return (i64)(int)W[k];
    return quant(reinterpret_cast<const T*>(W)[k], sf, sd);
  }
};

// exact gradient (2x the derivative, one-sided doubled at the spatial boundary; R7) at
// cube corner c (bit0 x, bit1 y, bit2 t)
template <typename T>
__device__ __forceinline__ void corner_grad(const Win<T>& w, const Geo& G, i64 x, i64 y, int c, i64& gx, i64& gy) {
  if (w.isq) {  // fast entries are interior cubes: central differences precomputed by the scan warp
    gx = (int)w.W[32 + 2 * c];
    gy = (int)w.W[33 + 2 * c];
    return;
  }
  const int cx = c & 1, cy = (c >> 1) & 1, pl = c >> 2;
  const i64 xc = x + cx, yc = y + cy;
  if (xc == 0) gx = 2 * (w.q(pl, cx + 2, cy + 1) - w.q(pl, cx + 1, cy + 1));
  else if (xc == G.nx - 1) gx = 2 * (w.q(pl, cx + 1, cy + 1) - w.q(pl, cx, cy + 1));
  else gx = w.q(pl, cx + 2, cy + 1) - w.q(pl, cx, cy + 1);
  if (yc == 0) gy = 2 * (w.q(pl, cx + 1, cy + 2) - w.q(pl, cx + 1, cy + 1));
  else if (yc == G.ny - 1) gy = 2 * (w.q(pl, cx + 1, cy + 1) - w.q(pl, cx + 1, cy));
  else gy = w.q(pl, cx + 1, cy + 2) - w.q(pl, cx + 1, cy);
}

// SoS sign of | ua va ; ub vb | (rows a < b in global vertex order) given the sign of its exact
// value; perturbation eps_{r,j} = eps^(2^(2r+j)) (R4): the leading terms of det(M + E)
// in decreasing magnitude are det, +v_b, -u_b, -v_a, then the constant -1.
__device__ __forceinline__ int sos_sign(int ds, i64 ua, i64 va, i64 ub, i64 vb) {
  if (ds) return ds;
  if (vb) return vb > 0 ? 1 : -1;
  if (ub) return ub > 0 ? -1 : 1;
  if (va) return va > 0 ? -1 : 1;
  return -1;
}

template <int K>
struct Face3 {
  static constexpr int m1 = kKuhn3.masks[K][0];
  static constexpr int m2 = kKuhn3.masks[K][1];
};
// the masks of face type ty as 3-bit fields of two packed constants (two shifts, no branches)
template <int... K>
constexpr unsigned long long pack_masks(int which, std::integer_sequence<int, K...>) {
  return ((((unsigned long long)(which == 1 ? Face3<K>::m1 : Face3<K>::m2)) << (3 * K)) | ...);
}
constexpr unsigned long long kM1 = pack_masks(1, std::make_integer_sequence<int, 12>{});
constexpr unsigned long long kM2 = pack_masks(2, std::make_integer_sequence<int, 12>{});
template <int... K>
__device__ __forceinline__ void masks_of(int ty, int& m1, int& m2, std::integer_sequence<int, K...>) {
  m1 = (int)((kM1 >> (3 * ty)) & 7);
  m2 = (int)((kM2 >> (3 * ty)) & 7);
}

// The 6 cells (3-simplices) anchored at a cube: axis permutations (p1, p2, p3) of {x=1, y=2, t=4},
// chain w0 = 0, w1 = p1, w2 = p1|p2, w3 = 7.  Dropping w3, w2, w1 leaves the cube's own faces
// ta = (w1, w2), tb = (w1, 7), tc = (w2, 7); dropping w0 leaves the "upper" face (w1, w2, 7), which
// is owned by the neighbour cube anchored at v + p1 with type tf = (p2, p2|p3) (side_of in closed
// form).  Its three 2x2 determinants are the pair determinants of ta, tb and tc.
struct CellDef {
  int ta, tb, tc, axis, tf, w1, w2;
};
constexpr int type3(int m1, int m2) { return kKuhn3.type_of[m1 | m2 << 4]; }
constexpr CellDef make_cell(int p1, int p2, int p3) {
  return CellDef{type3(p1, p1 | p2), type3(p1, 7), type3(p1 | p2, 7), p1, type3(p2, p2 | p3), p1, p1 | p2};
}
template <int C>
struct Cell3 {
  static constexpr int P1[6] = {1, 1, 2, 2, 4, 4};
  static constexpr int P2[6] = {2, 4, 1, 4, 1, 2};
  static constexpr int P3[6] = {4, 2, 4, 1, 2, 1};
  static constexpr CellDef d = make_cell(P1[C], P2[C], P3[C]);
};

template <int... C>
constexpr int cell_code(int c, std::integer_sequence<int, C...>) {
  int r = 0;
  ((c == C ? (r = Cell3<C>::d.ta | Cell3<C>::d.tb << 4 | Cell3<C>::d.tc << 8 | Cell3<C>::d.axis << 12 |
                  Cell3<C>::d.tf << 16, 0) : 0), ...);
  return r;
}
__constant__ int cCell[6] = {cell_code(0, std::make_integer_sequence<int, 6>{}),
                             cell_code(1, std::make_integer_sequence<int, 6>{}),
                             cell_code(2, std::make_integer_sequence<int, 6>{}),
                             cell_code(3, std::make_integer_sequence<int, 6>{}),
                             cell_code(4, std::make_integer_sequence<int, 6>{}),
                             cell_code(5, std::make_integer_sequence<int, 6>{})};

// generic face test from the exact determinant signs: point-in-simplex for the
// face (0, m1, m2): s_k = (-1)^(k+2) sos(rows != k); punctured iff s_0 = s_1 = s_2.
template <int K>
__device__ __forceinline__ void face_test(const i64 (&g)[8][2], const int (&s0k)[8], const int (&sp)[12],
                                          uint32_t exists, uint32_t& pmask) {
  constexpr int m1 = Face3<K>::m1, m2 = Face3<K>::m2;
  if (((exists >> m2) & 1) == 0) return;  // the span's far corner must exist
  const int s0 = sos_sign(sp[K], g[m1][0], g[m1][1], g[m2][0], g[m2][1]);
  const int s1 = -sos_sign(s0k[m2], g[0][0], g[0][1], g[m2][0], g[m2][1]);
  const int s2 = sos_sign(s0k[m1], g[0][0], g[0][1], g[m1][0], g[m1][1]);
  if (s0 == s1 && s1 == s2) pmask |= 1u << K;
}
template <int... K>
__device__ __forceinline__ void all_faces(const i64 (&g)[8][2], const int (&s0k)[8], const int (&sp)[12],
                                          uint32_t exists, uint32_t& pmask, std::integer_sequence<int, K...>) {
  (face_test<K>(g, s0k, sp, exists, pmask), ...);
}
template <bool WIDE>
__device__ __forceinline__ int det_sign(const i64* a, const i64* b) {
  if (WIDE) return sgn128(det2(a[0], a[1], b[0], b[1]));
  return sgn64(a[0] * b[1] - a[1] * b[0]);  // |g| < 2^31: |det| < 2^63
}
template <bool WIDE, int... K>
__device__ __forceinline__ void pair_signs(const i64 (&g)[8][2], int (&sp)[12], std::integer_sequence<int, K...>) {
  ((sp[K] = det_sign<WIDE>(g[Face3<K>::m1], g[Face3<K>::m2])), ...);
}

// Punctured face types of one cube -- the general path: any position (boundary rules, missing
// corners), int64 gradients, int128 determinants when needed, full SoS chains.
template <typename T>
__device__ __noinline__ uint32_t cube_faces_general(const Win<T>& w, const Geo& G, i64 x, i64 y, bool hasB) {
  i64 g[8][2];
  uint32_t exists = 0;
  bool wide = false;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const bool ex = (x + (c & 1) < G.nx) && (y + ((c >> 1) & 1) < G.ny) && ((c >> 2) == 0 || hasB);
    i64 gx, gy;
    corner_grad(w, G, x, y, c, gx, gy);
    g[c][0] = ex ? gx : 0;
    g[c][1] = ex ? gy : 0;
    exists |= (ex ? 1u : 0u) << c;
    wide |= ((gx < 0 ? -gx : gx) | (gy < 0 ? -gy : gy)) >= (1ll << 31);
  }
  int s0k[8], sp[12];
  s0k[0] = 0;
  uint32_t pmask = 0;
  if (!wide) {
#pragma unroll
    for (int k = 1; k < 8; ++k) s0k[k] = det_sign<false>(g[0], g[k]);
    pair_signs<false>(g, sp, std::make_integer_sequence<int, 12>{});
  } else {
#pragma unroll
    for (int k = 1; k < 8; ++k) s0k[k] = det_sign<true>(g[0], g[k]);
    pair_signs<true>(g, sp, std::make_integer_sequence<int, 12>{});
  }
  all_faces(g, s0k, sp, exists, pmask, std::make_integer_sequence<int, 12>{});
  // upper faces of the 6 cells (meaningful for full cubes only)
  uint32_t umask = 0;
#define FTK_UP(C)                                                                                           \
  {                                                                                                         \
    constexpr CellDef d = Cell3<C>::d;                                                                      \
    const int s0 = sos_sign(sp[d.tc], g[d.w2][0], g[d.w2][1], g[7][0], g[7][1]);                            \
    const int s1 = -sos_sign(sp[d.tb], g[d.w1][0], g[d.w1][1], g[7][0], g[7][1]);                           \
    const int s2 = sos_sign(sp[d.ta], g[d.w1][0], g[d.w1][1], g[d.w2][0], g[d.w2][1]);                      \
    umask |= (uint32_t)(s0 == s1 && s1 == s2) << C;                                                         \
  }
  FTK_UP(0) FTK_UP(1) FTK_UP(2) FTK_UP(3) FTK_UP(4) FTK_UP(5)
#undef FTK_UP
  return pmask | umask << 16;
}

// int32 fast path: fast entry (interior cube with both planes, |q| < 2^29), gradients precomputed
// when the window was staged.  Returns false on a zero determinant (the SoS chains are in the general
// path).
__device__ __forceinline__ bool cube_faces_fast(const uint32_t* E, uint32_t& pmask) {
  int g[8][2];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    g[c][0] = (int)E[32 + 2 * c];
    g[c][1] = (int)E[33 + 2 * c];
  }
  // determinants (0, k) and (m1, m2): |g| < 2^30 so |det| < 2^61
  i64 d0[8], dp[12];
#pragma unroll
  for (int k = 1; k < 8; ++k) d0[k] = (i64)g[0][0] * g[k][1] - (i64)g[0][1] * g[k][0];
  bool zero = false;
#pragma unroll
  for (int k = 1; k < 8; ++k) zero |= d0[k] == 0;
#define FTK_DP(K)                                                                                    \
  dp[K] = (i64)g[Face3<K>::m1][0] * g[Face3<K>::m2][1] - (i64)g[Face3<K>::m1][1] * g[Face3<K>::m2][0]; \
  zero |= dp[K] == 0;
  FTK_DP(0) FTK_DP(1) FTK_DP(2) FTK_DP(3) FTK_DP(4) FTK_DP(5)
  FTK_DP(6) FTK_DP(7) FTK_DP(8) FTK_DP(9) FTK_DP(10) FTK_DP(11)
#undef FTK_DP
  if (zero) return false;
  // s0 = sgn D(m1,m2), s1 = -sgn D(0,m2), s2 = sgn D(0,m1): punctured iff all equal
  uint32_t m = 0;
#define FTK_FACE(K)                                                                  \
  {                                                                                  \
    const bool a = dp[K] < 0, b = d0[Face3<K>::m2] > 0, c = d0[Face3<K>::m1] < 0;    \
    m |= (uint32_t)(a == b && b == c) << K;                                          \
  }
  FTK_FACE(0) FTK_FACE(1) FTK_FACE(2) FTK_FACE(3) FTK_FACE(4) FTK_FACE(5)
  FTK_FACE(6) FTK_FACE(7) FTK_FACE(8) FTK_FACE(9) FTK_FACE(10) FTK_FACE(11)
#undef FTK_FACE
  // upper faces (w1, w2, 7) of the 6 cells: s0 = sgn D(w2,7), s1 = -sgn D(w1,7), s2 = sgn D(w1,w2)
#define FTK_UP(C)                                                                            \
  {                                                                                          \
    constexpr CellDef d = Cell3<C>::d;                                                       \
    const bool a = dp[d.tc] < 0, b = dp[d.tb] > 0, c = dp[d.ta] < 0;                         \
    m |= (uint32_t)(a == b && b == c) << (16 + C);                                           \
  }
  FTK_UP(0) FTK_UP(1) FTK_UP(2) FTK_UP(3) FTK_UP(4) FTK_UP(5)
#undef FTK_UP
  pmask = m;
  return true;
}

// int32 fast path for a fast entry on the last timestep (no t + 1 corners, the window's second plane
// repeats the first): only the in-plane faces -- types 0 = (x, x|y) and 3 = (y, x|y) -- exist, and no
// cell.  Returns false on a zero determinant (the SoS chains are in the general path).
__device__ __forceinline__ bool cube_faces_planar(const uint32_t* E, uint32_t& pmask) {
  int g[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    g[c][0] = (int)E[32 + 2 * c];
    g[c][1] = (int)E[33 + 2 * c];
  }
  auto det = [&](int a, int b) { return (i64)g[a][0] * g[b][1] - (i64)g[a][1] * g[b][0]; };
  const i64 d01 = det(0, 1), d02 = det(0, 2), d03 = det(0, 3), d13 = det(1, 3), d23 = det(2, 3);
  if (d01 == 0 || d02 == 0 || d03 == 0 || d13 == 0 || d23 == 0) return false;
  static_assert(Face3<0>::m1 == 1 && Face3<0>::m2 == 3 && Face3<3>::m1 == 2 && Face3<3>::m2 == 3, "in-plane types");
  // s0 = sgn D(m1, 3), s1 = -sgn D(0, 3), s2 = sgn D(0, m1): punctured iff all equal (as cube_faces_fast)
  const bool b = d03 > 0;
  uint32_t m = 0;
  m |= (uint32_t)((d13 < 0) == b && b == (d01 < 0)) << 0;
  m |= (uint32_t)((d23 < 0) == b && b == (d02 < 0)) << 3;
  pmask = m;
  return true;
}

__device__ __forceinline__ double dot3_nofma(const double* mu, double a, double b, double c) {
  return __dadd_rn(__dadd_rn(__dmul_rn(mu[0], a), __dmul_rn(mu[1], b)), __dmul_rn(mu[2], c));
}

// Hessian (4x scale, centre clamped into [1, N-2], R8) straight from global memory;
// used only for partial cubes on the last row/column, whose stencil leaves the 4x4 window.
template <typename T>
__device__ __noinline__ void hessian_global(const ExtractParams& P, const Geo& G, i64 x, i64 y, i64 t, i64* H) {
  const T* base = reinterpret_cast<const T*>(P.field) + (t - P.t0) * G.nx * G.ny;
  auto q = [&](i64 xx, i64 yy) { return quant(base[yy * G.nx + xx], G.scale_f, G.scale); };
  const i64 cx = x < 1 ? 1 : (x > G.nx - 2 ? G.nx - 2 : x);
  const i64 cy = y < 1 ? 1 : (y > G.ny - 2 ? G.ny - 2 : y);
  H[0] = 4 * (q(cx + 1, y) - 2 * q(cx, y) + q(cx - 1, y));
  H[1] = q(cx + 1, cy + 1) - q(cx + 1, cy - 1) - q(cx - 1, cy + 1) + q(cx - 1, cy - 1);
  H[2] = 4 * (q(x, cy + 1) - 2 * q(x, cy) + q(x, cy - 1));
}

// Location (Eq. 2), type and flags of punctured face `ty` of the cube at (x, y, t); writes the record.
#ifndef FTK_K1_REC_NOINLINE
#define FTK_K1_REC_NOINLINE 0
#endif
#if FTK_K1_REC_NOINLINE
#define FTK_REC_INL __noinline__
#else
#define FTK_REC_INL __forceinline__
#endif
template <typename T>
__device__ __noinline__ void emit_record_general(const Win<T>& w, const Geo& G, const ExtractParams& P, i64 x, i64 y,
                                                 i64 t, int ty, unsigned long long slot) {
  int m[3] = {0, 0, 0};
  masks_of(ty, m[1], m[2], std::make_integer_sequence<int, 12>{});
  i64 gv[3][2];
#pragma unroll
  for (int k = 0; k < 3; ++k) corner_grad(w, G, x, y, m[k], gv[k][0], gv[k][1]);
  // mu_k = D_k / sum D, D_k = (-1)^(k+2) det(rows != k)
  const i128 D0 = det2(gv[1][0], gv[1][1], gv[2][0], gv[2][1]);
  const i128 D1 = -det2(gv[0][0], gv[0][1], gv[2][0], gv[2][1]);
  const i128 D2 = det2(gv[0][0], gv[0][1], gv[1][0], gv[1][1]);
  const i128 S = D0 + D1 + D2;
  double mu[3];
  uint32_t flags = 0;
  if (S == 0) {
    mu[0] = mu[1] = mu[2] = 1.0 / 3.0;
    flags |= FTK_CP_DEGENERATE_LOC;
  } else {
    const double s = i128_to_double_rn(S);
    mu[0] = __ddiv_rn(i128_to_double_rn(D0), s);
    mu[1] = __ddiv_rn(i128_to_double_rn(D1), s);
    mu[2] = __ddiv_rn(i128_to_double_rn(D2), s);
  }
  const bool partial = (x == G.nx - 1) || (y == G.ny - 1);  // Hessian stencil leaves the window
  double px[3], py[3], pt[3];
  i64 Hk[3][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int mx = m[k] & 1, my = (m[k] >> 1) & 1, pl = (m[k] >> 2) & 1;
    const i64 vx = x + mx, vy = y + my, vt = t + pl;
    px[k] = (double)vx;
    py[k] = (double)vy;
    pt[k] = (double)vt;
    if (partial) {
      hessian_global<T>(P, G, vx, vy, vt, Hk[k]);
    } else {
      // integer Hessian, 4x scale, centre clamped into [1, N-2] (R8), from the window
      const i64 cxg = vx < 1 ? 1 : (vx > G.nx - 2 ? G.nx - 2 : vx);
      const i64 cyg = vy < 1 ? 1 : (vy > G.ny - 2 ? G.ny - 2 : vy);
      const int cx = (int)(cxg - x) + 1, cy = (int)(cyg - y) + 1, wx = mx + 1, wy = my + 1;
      Hk[k][0] = 4 * (w.q(pl, cx + 1, wy) - 2 * w.q(pl, cx, wy) + w.q(pl, cx - 1, wy));
      Hk[k][1] = w.q(pl, cx + 1, cy + 1) - w.q(pl, cx + 1, cy - 1) - w.q(pl, cx - 1, cy + 1) + w.q(pl, cx - 1, cy - 1);
      Hk[k][2] = 4 * (w.q(pl, wx, cy + 1) - 2 * w.q(pl, wx, cy) + w.q(pl, wx, cy - 1));
    }
  }
  const double lx = dot3_nofma(mu, px[0], px[1], px[2]);
  const double ly = dot3_nofma(mu, py[0], py[1], py[2]);
  const double lt = dot3_nofma(mu, pt[0], pt[1], pt[2]);
  double Hb[3];
#pragma unroll
  for (int e = 0; e < 3; ++e)
    Hb[e] = dot3_nofma(mu, __ll2double_rn(Hk[0][e]), __ll2double_rn(Hk[1][e]), __ll2double_rn(Hk[2][e]));
  // type (R9): sign of the interpolated Hessian's determinant, no tolerance
  const double det = __dsub_rn(__dmul_rn(Hb[0], Hb[2]), __dmul_rn(Hb[1], Hb[1]));
  int type;
  if (det < 0) type = FTK_CP_SADDLE;
  else if (det > 0) type = Hb[0] > 0 ? FTK_CP_MIN : FTK_CP_MAX;
  else type = FTK_CP_DEGENERATE;
  const int span = m[2];
  if (!(span & 4)) flags |= FTK_CP_ORDINAL;
  if (span != 7) {  // closed-form side_of: both parents exist iff v0[c] in [1, N_c - 2]
    const int c = 7 & ~span;
    const i64 vc = c == 1 ? x : (c == 2 ? y : t);
    const i64 Nc = c == 1 ? G.nx : (c == 2 ? G.ny : G.ntg);
    if (vc == 0 || vc == Nc - 1) flags |= FTK_CP_BOUNDARY;
  }
  if (slot < (unsigned long long)P.capacity) {
    ftk_cp* r = P.out + slot;
    r->face_id = ((t * G.ny + y) * G.nx + x) * 12 + ty;
    P.fid[slot] = r->face_id;  // compact face ids for pass 2
    r->label = -1;
    r->x = lx;
    r->y = ly;
    r->z = 0.0;
    r->t = lt;
    r->type = type;
    r->flags = flags;
  }
}

__device__ __forceinline__ void store_record(const ExtractParams& P, unsigned long long slot, long long fid, double lx,
                                             double ly, double lt, int type, uint32_t flags) {
  if (slot < (unsigned long long)P.capacity) {
    ftk_cp* r = P.out + slot;
    r->face_id = fid;
    P.fid[slot] = fid;  // compact face ids for pass 2
    r->label = -1;
    r->x = lx;
    r->y = ly;
    r->z = 0.0;
    r->t = lt;
    r->type = type;
    r->flags = flags;
  }
}

// Record of a punctured face: fast entries (interior cube, |g| < 2^30) in int64 -- |D_k| < 2^61 and
// |sum D| < 2^63, converted exactly as the int128 path would -- else the general int128 path.
template <typename T>
__device__ __forceinline__ void emit_record(const Win<T>& w, const Geo& G, const ExtractParams& P, i64 x, i64 y, i64 t,
                                            int ty, unsigned long long slot) {
  if (!w.isq) {
    emit_record_general<T>(w, G, P, x, y, t, ty, slot);
    return;
  }
  int m[3] = {0, 0, 0};
  masks_of(ty, m[1], m[2], std::make_integer_sequence<int, 12>{});
  int g[3][2];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    g[k][0] = (int)w.W[32 + 2 * m[k]];
    g[k][1] = (int)w.W[33 + 2 * m[k]];
  }
  // mu_k = D_k / sum D, D_k = (-1)^(k+2) det(rows != k)
  const i64 D0 = (i64)g[1][0] * g[2][1] - (i64)g[1][1] * g[2][0];
  const i64 D1 = (i64)g[0][1] * g[2][0] - (i64)g[0][0] * g[2][1];
  const i64 D2 = (i64)g[0][0] * g[1][1] - (i64)g[0][1] * g[1][0];
  const i64 S = D0 + D1 + D2;
  double mu[3];
  uint32_t flags = 0;
  if (S == 0) {
    mu[0] = mu[1] = mu[2] = 1.0 / 3.0;
    flags |= FTK_CP_DEGENERATE_LOC;
  } else {
    const double sd = __ll2double_rn(S);
    mu[0] = __ddiv_rn(__ll2double_rn(D0), sd);
    mu[1] = __ddiv_rn(__ll2double_rn(D1), sd);
    mu[2] = __ddiv_rn(__ll2double_rn(D2), sd);
  }
  double px[3], py[3], pt[3], Hd[3][3];
  const int* q = reinterpret_cast<const int*>(w.W);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int mx = m[k] & 1, my = (m[k] >> 1) & 1, pl = (m[k] >> 2) & 1;
    px[k] = (double)(x + mx);
    py[k] = (double)(y + my);
    pt[k] = (double)(t + pl);
    // interior vertex: the Hessian stencil centre is the vertex itself, window (mx+1, my+1)
    const int* Q = q + pl * 16 + (my + 1) * 4 + (mx + 1);
    // |q| < 2^29 on the fast path: every second difference fits int32, and the 4x scale is an exact
    // FP64 multiply (the same values as the int64 expressions of the general path)
    Hd[k][0] = __dmul_rn(4.0, __int2double_rn(Q[1] - 2 * Q[0] + Q[-1]));
    Hd[k][1] = __int2double_rn(Q[5] - Q[-3] - Q[3] + Q[-5]);
    Hd[k][2] = __dmul_rn(4.0, __int2double_rn(Q[4] - 2 * Q[0] + Q[-4]));
  }
  const double lx = dot3_nofma(mu, px[0], px[1], px[2]);
  const double ly = dot3_nofma(mu, py[0], py[1], py[2]);
  const double lt = dot3_nofma(mu, pt[0], pt[1], pt[2]);
  const double a = dot3_nofma(mu, Hd[0][0], Hd[1][0], Hd[2][0]);
  const double b = dot3_nofma(mu, Hd[0][1], Hd[1][1], Hd[2][1]);
  const double d = dot3_nofma(mu, Hd[0][2], Hd[1][2], Hd[2][2]);
  const double det = __dsub_rn(__dmul_rn(a, d), __dmul_rn(b, b));
  const int type = det < 0 ? FTK_CP_SADDLE : (det > 0 ? (a > 0 ? FTK_CP_MIN : FTK_CP_MAX) : FTK_CP_DEGENERATE);
  const int span = m[2];
  if (!(span & 4)) flags |= FTK_CP_ORDINAL;
  if (span != 7) {  // interior in x and y: only t can be on the boundary
    const int c = 7 & ~span;
    if (c == 4 && (t == 0 || t == G.ntg - 1)) flags |= FTK_CP_BOUNDARY;
  }
  store_record(P, slot, ((t * G.ny + y) * G.nx + x) * 12 + ty, lx, ly, lt, type, flags);
}

// in-cube union-find over the 12 face types: 4-bit parent fields, the root is the smallest type of
// its component (= the smallest face id)
__device__ __forceinline__ int lfind(unsigned long long lp, int ty) {
  int p = (int)((lp >> (4 * ty)) & 15);
  while (p != ty) {
    ty = p;
    p = (int)((lp >> (4 * ty)) & 15);
  }
  return ty;
}

// One batch of 32 entries (one cube per lane): face tests, the 6 cells of every cube, slot
// reservation, then the punctured faces spread over the lanes for the record stage.
template <typename T>
__device__ void process_batch(const BatchBuf& bb, const Geo& G, const ExtractParams& P, Prof& pf) {
  const int lane = threadIdx.x & 31;
  const int qtv = bb.qt[lane];
  const bool valid = qtv != -1;
  const i64 x = bb.qx[lane], y = bb.qy[lane], t = qtv & 0x3fffffff;
  const bool hasB = (qtv >> 31) & 1;
  const uint32_t* E = bb.ring + lane * ws_words<T>();
  const bool isq = (qtv >> 30) & 1;
  uint32_t m = 0;
  if (valid) {
    const bool done = isq && (hasB ? cube_faces_fast(E, m) : cube_faces_planar(E, m));
    if (!done) m = cube_faces_general<T>(Win<T>{E, isq, G.scale_f, G.scale}, G, x, y, hasB);
  }
  const uint32_t pmask = m & 0xFFFu, umask = m >> 16;
  pf.lap(PF_EXFACE);
  // pass 2 for the 6 cells anchored at this cube: every cell lies inside one
  // cube, so its 4 faces are tested right here; a cell holds 0 or 2 punctured faces under SoS
  // (PAPER.md:437, 467).  Two own faces are joined in the cube's union-find (opm: such cells); a pair
  // with the upper face (owned by the neighbour cube) becomes a trajectory-graph edge (edm).
  const bool full = valid && x + 1 < G.nx && y + 1 < G.ny && hasB;
  uint32_t opm = 0, edm = 0;
  int bad = 0;
#define FTK_CELLCNT(C)                                                                                   \
  {                                                                                                      \
    constexpr CellDef d = Cell3<C>::d;                                                                   \
    const uint32_t bits = ((pmask >> d.ta) & 1u) | (((pmask >> d.tb) & 1u) << 1) |                        \
                          (((pmask >> d.tc) & 1u) << 2) | (((umask >> C) & 1u) << 3);                     \
    const int k = __popc(bits);                                                                          \
    if (k == 2) (bits & 8u ? edm : opm) |= 1u << C;                                                      \
    bad += (k != 0 && k != 2) ? 1 : 0;                                                                   \
  }
  if (full) {
    FTK_CELLCNT(0) FTK_CELLCNT(1) FTK_CELLCNT(2) FTK_CELLCNT(3) FTK_CELLCNT(4) FTK_CELLCNT(5)
  }
#undef FTK_CELLCNT
  if (bad) atomicAdd(&P.counters[CNT_INVARIANT], (unsigned long long)bad);
  // record and edge slots: one warp scan of both counts (<= 12 and <= 6 per lane), one atomic each
  const int cnt = __popc(pmask), ecnt = __popc(edm);
  int incl = cnt | (ecnt << 16);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int tot = __shfl_sync(0xffffffffu, incl, 31);
  const int total = tot & 0xFFFF, etotal = tot >> 16;
  if (total == 0) return;
  const int rstart = (incl & 0xFFFF) - cnt, estart = (incl >> 16) - ecnt;
  unsigned long long obase = 0, ebase = 0;
  if (lane == 0) {
    obase = atomicAdd(&P.counters[CNT_NOUT], (unsigned long long)total);
    if (etotal) ebase = atomicAdd(&P.counters[CNT_EDGES], (unsigned long long)etotal);
  }
  // own-own pairs, while the atomics are in flight
  unsigned long long lp = 0xBA9876543210ull;
  for (uint32_t mm = opm; mm; mm &= mm - 1) {
    const int cd = cCell[__ffs(mm) - 1];  // ta | tb << 4 | tc << 8 | axis << 12 | tf << 16
    const int ta = cd & 15, tb = (cd >> 4) & 15, tc = (cd >> 8) & 15;
    const int t1 = ((pmask >> ta) & 1u) ? ta : tb;
    const int t2 = ((pmask >> tc) & 1u) ? tc : tb;
    const int r1 = lfind(lp, t1), r2 = lfind(lp, t2);
    const int lo = min(r1, r2), hi = max(r1, r2);
    lp = (lp & ~(15ull << (4 * hi))) | ((unsigned long long)lo << (4 * hi));
  }
  bb.lp[lane] = lp;
  bb.pm[lane] = pmask;
  bb.rs[lane] = rstart;
  FTK_ASSERT(total <= MAXITEMS && rstart + cnt <= total);
  {
    int pos = rstart;
    for (uint32_t pm = pmask; pm; pm &= pm - 1) bb.items[pos++] = (uint16_t)(lane | ((__ffs(pm) - 1) << 5));
  }
  obase = __shfl_sync(0xffffffffu, obase, 0);
  ebase = __shfl_sync(0xffffffffu, ebase, 0);
  if (edm) {
    unsigned long long eslot = ebase + (unsigned long long)estart;
    const long long rbase = (long long)obase + rstart;
    for (uint32_t mm = edm; mm; mm &= mm - 1, ++eslot) {
      const int cd = cCell[__ffs(mm) - 1];
      const int ta = cd & 15, tb = (cd >> 4) & 15, tc = (cd >> 8) & 15;
      const int ty = ((pmask >> ta) & 1u) ? ta : (((pmask >> tb) & 1u) ? tb : tc);
      const long long a = rbase + __popc(pmask & ((1u << ty) - 1u));
      const int axis = (cd >> 12) & 7, tf = (cd >> 16) & 15;
      const i64 fx = x + (axis & 1), fy = y + ((axis >> 1) & 1), ft = t + ((axis >> 2) & 1);
      const long long b = -1 - (((ft * G.ny + fy) * G.nx + fx) * 12 + tf);
      if (eslot < (unsigned long long)P.capacity) {
        P.edges[2 * eslot] = a;
        P.edges[2 * eslot + 1] = b;
      }
    }
  }
  __syncwarp();
  for (int i = lane; i < total; i += 32) {
    const int it = bb.items[i];
    const int le = it & 31, ty = it >> 5;
    FTK_ASSERT(ty < 12 && ((bb.pm[le] >> ty) & 1u) && bb.qt[le] != -1);
    const int lqt = bb.qt[le];
    const Win<T> w2{bb.ring + le * ws_words<T>(), ((lqt >> 30) & 1) != 0, G.scale_f, G.scale};
    const unsigned long long slot = obase + i;
    emit_record<T>(w2, G, P, bb.qx[le], bb.qy[le], lqt & 0x3fffffff, ty, slot);
    // union-find parent: the in-cube root of ty (its smallest punctured type)
    if (P.parent && slot < (unsigned long long)P.capacity) {
      const int root = lfind(bb.lp[le], ty);
      P.parent[slot] = (int)((long long)obase + bb.rs[le] + __popc(bb.pm[le] & ((1u << root) - 1u)));
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------------------------
// Scan
//
// Code layout: position i (0..3) of a lane lives in byte i; the byte's top nibble holds, from bit 7
// down, (dx > thr), (dx < -thr), (dy > thr), (dy < -thr) -- the sign bits of thr - dx, dx + thr,
// thr - dy, dy + thr (1 = that strict sign of the gradient component is established).  ANDing the
// codes over a cube's corners leaves a bit set iff that component has that sign on every corner, so
// the cubes to keep are the ones whose byte is ZERO after the AND (found with the exact zero-byte
// test below: low nibbles repeat bit 4, so no byte lies in 1..15).  Positions outside the grid get 0xF0 (AND-neutral).
// ---------------------------------------------------------------------------------------------
struct ScanCtx {
  int srow0;       // smem row of the warp's first anchor row
  int lane;
  int rpos;        // position (0..3) of x = nx - 1 in this lane, else -1
  bool lpat;       // x = 0 is this lane's position 0
  bool xe_out;     // column x0 + 128 is outside the grid
  bool xe_last;    // column x0 + 128 is x = nx - 1
  uint32_t xmask;  // top-nibble mask of the lane's in-grid positions (0xF0 per in-grid byte)
  long long gy0;   // global y of the warp's first anchor row
  long long ny;
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

// gather the sign bits of the 4 conditions x 4 positions into the byte-top-nibble layout
// (FTK_GATHER_SR: bits 3..0 repeat bit 4, so a byte is zero iff its four condition bits are, and no
// byte lies in 0x01..0x0F -- the per-byte zero test stays exact)
__device__ __forceinline__ uint32_t gather_code(const f2 (&c)[8]) {
  // c[2*j] = condition j for positions 0,1; c[2*j+1] = condition j for positions 2,3
  if constexpr (FTK_GATHER_SR) {
    // per condition: two sign-replicating PRMTs (positions 0, 1 and 2, 3) and two bit-selects
    uint32_t acc = bitsel(prmt_sr(lo32(c[0]), hi32(c[0])), prmt_sr(lo32(c[1]), hi32(c[1])), 0xFFFF0000u);
#pragma unroll
    for (int j = 1; j < 4; ++j) {
      const uint32_t m = j < 3 ? (0x80808080u >> j) : 0x1F1F1F1Fu;
      acc = bitsel(acc, prmt_sr(lo32(c[2 * j]), hi32(c[2 * j])), m & 0x0000FFFFu);
      acc = bitsel(acc, prmt_sr(lo32(c[2 * j + 1]), hi32(c[2 * j + 1])), m & 0xFFFF0000u);
    }
    return acc;
  } else {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t p01 = __byte_perm(lo32(c[2 * j]), hi32(c[2 * j]), 0x0073);
      const uint32_t p23 = __byte_perm(lo32(c[2 * j + 1]), hi32(c[2 * j + 1]), 0x0073);
      w[j] = __byte_perm(p01, p23, 0x5410);
    }
    return (w[0] & 0x80808080u) | ((w[1] >> 1) & 0x40404040u) | ((w[2] >> 2) & 0x20202020u) |
           ((w[3] >> 3) & 0x10101010u);
  }
}

__device__ __forceinline__ uint32_t code_f32(const float4 u, const float4 v, const float4 d, float l, float r,
                                             f2 thr2, f2 nthr2) {
  // x differences in scalar FADDs (their operands are not register-pair aligned; the results are
  // placed in pairs by the register allocator), y differences in paired FADD2s
  const f2 dx01 = pack2(__fsub_rn(v.y, l), __fsub_rn(v.z, v.x));
  const f2 dx23 = pack2(__fsub_rn(v.w, v.y), __fsub_rn(r, v.z));
  const f2 dy01 = sub2(pack2(d.x, d.y), pack2(u.x, u.y));
  const f2 dy23 = sub2(pack2(d.z, d.w), pack2(u.z, u.w));
  f2 c[8];
  c[0] = sub2(thr2, dx01);   // thr - dx < 0  <=>  dx > thr
  c[1] = sub2(thr2, dx23);
  c[2] = sub2(dx01, nthr2);  // dx + thr < 0  <=>  dx < -thr
  c[3] = sub2(dx23, nthr2);
  c[4] = sub2(thr2, dy01);
  c[5] = sub2(thr2, dy23);
  c[6] = sub2(dy01, nthr2);
  c[7] = sub2(dy23, nthr2);
  return gather_code(c);
}


// Scan one plane (fp32): all RW+3 rows are loaded first (independent shared loads and shuffles),
// then the RW+1 code rows, then the squares Sq[r] (OR over the 4 corners of each square, per
// position).  One-sided differences at the grid boundary by patching neighbour values; MODE 0:
// interior tile, 1: x boundary only, 2: y boundary (and possibly x).
template <int MODE>
__device__ __forceinline__ void scan_plane_f32(const float* S, const ScanCtx& c, f2 thr2, f2 nthr2,
                                               uint32_t (&Sq)[RW], uint32_t& maxb) {
  constexpr bool XE = MODE >= 1, EDGE = MODE >= 2;
  // rows srow0-1 .. srow0+RW+1, rolled through a 3-row window: code row k needs rows k (up), k+1
  // (centre, with its x neighbours l, r) and k+2 (down); square row k ANDs code rows k, k+1
  const bool lane0 = c.lane == 0, lane31 = c.lane == 31;
  const int hcol = lane0 ? XOFF - 1 : XOFF + LX;
  auto load = [&](int i, float4& v, float& l, float& r) {
    const int row = c.srow0 - 1 + i;
    FTK_ASSERT(row >= 0 && row < ROWS);
    v = *reinterpret_cast<const float4*>(S + row * PITCH + XOFF + 4 * c.lane);
    const float h = S[row * PITCH + hcol];  // tile halo (used by lanes 0 and 31)
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
  // computes code row k (centre smem row srow0 + k), Ye = the y-pair of code rows k, k + 1
  uint32_t Ye;
  {
    const int k = min(c.lane, RW);
    const float* p = S + (c.srow0 + k) * PITCH + XOFF + LX;
    const float ctr = p[0], l = p[-1];
    float r = p[1], u = p[-PITCH], d = p[PITCH];
    bool out = false;
    if (XE) {
      if (c.xe_last) r = ctr;
      out = c.xe_out;
    }
    if (EDGE) {
      const long long gy = c.gy0 + k;
      if (gy == 0) u = ctr;
      if (gy == c.ny - 1) d = ctr;
      out = out || gy >= c.ny;
    }
    const float thr = __uint_as_float(lo32(thr2));
    const float dx = __fsub_rn(r, l), dy = __fsub_rn(d, u);
    const uint32_t ce = out ? 0xF0u
                            : ((__float_as_uint(__fsub_rn(thr, dx)) >> 31) << 7) |
                                  ((__float_as_uint(__fadd_rn(dx, thr)) >> 31) << 6) |
                                  ((__float_as_uint(__fsub_rn(thr, dy)) >> 31) << 5) |
                                  ((__float_as_uint(__fadd_rn(dy, thr)) >> 31) << 4);
    Ye = ce & __shfl_down_sync(0xffffffffu, ce, 1);
  }
  float4 v0, v1, v2;
  float l0, r0, l1, r1, l2, r2;
  load(0, v0, l0, r0);
  load(1, v1, l1, r1);
  uint32_t Cprev = 0;
#pragma unroll
  for (int k = 0; k <= RW; ++k) {
    load(k + 2, v2, l2, r2);
    if (k < RW) maxb = max_abs_bits(maxb, v1.x, v1.y, v1.z, v1.w);  // centre rows k = 0..RW-1 are owned
    uint32_t C;
    if (EDGE) {
      const long long gy = c.gy0 + k;
      const float4 u = gy == 0 ? v1 : v0;
      const float4 d = gy == c.ny - 1 ? v1 : v2;
      C = gy >= c.ny ? 0xF0F0F0F0u : code_f32(u, v1, d, l1, r1, thr2, nthr2) | (~c.xmask & 0xF0F0F0F0u);
    } else if (XE) {
      C = code_f32(v0, v1, v2, l1, r1, thr2, nthr2) | (~c.xmask & 0xF0F0F0F0u);
    } else {
      C = code_f32(v0, v1, v2, l1, r1, thr2, nthr2);
    }
    if (k >= 1) {
      const uint32_t Y = Cprev & C;                             // y-pair
      uint32_t nb = __shfl_down_sync(0xffffffffu, Y, 1);  // next lane's position 0
      const uint32_t ne = __shfl_sync(0xffffffffu, Ye, k - 1);  // column x0 + 128
      if (c.lane == 31) nb = ne;
      Sq[k - 1] = Y & ((Y >> 8) | (nb << 24));                 // x-pair
    }
    Cprev = C;
    v0 = v1; l0 = l1; r0 = r1;
    v1 = v2; l1 = l2; r1 = r2;
  }
}

// fp64 input: same layout, scalar arithmetic
__device__ __forceinline__ uint32_t sbit(double v) { return (uint32_t)((unsigned long long)__double_as_longlong(v) >> 63); }
template <bool EDGE>
__device__ __forceinline__ void scan_plane_f64(const double* S, const ScanCtx& c, double thr, uint32_t (&Sq)[RW],
                                               double& maxd) {
  constexpr int NR = RW + 3;
  double f[NR][6];  // f[x-1], f[x..x+3], f[x+4]
  const int hcol = c.lane == 0 ? XOFF - 1 : XOFF + LX;
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    const double* p = S + (c.srow0 - 1 + i) * PITCH;
    const double2 a = *reinterpret_cast<const double2*>(p + XOFF + 4 * c.lane);
    const double2 b = *reinterpret_cast<const double2*>(p + XOFF + 4 * c.lane + 2);
    const double h = p[hcol];
    f[i][1] = a.x; f[i][2] = a.y; f[i][3] = b.x; f[i][4] = b.y;
    const double up = __shfl_up_sync(0xffffffffu, b.y, 1);
    const double dn = __shfl_down_sync(0xffffffffu, a.x, 1);
    f[i][0] = c.lane == 0 ? h : up;
    f[i][5] = c.lane == 31 ? h : dn;
    if (EDGE) {
      if (c.lpat) f[i][0] = f[i][1];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c.rpos == q) f[i][q + 2] = f[i][q + 1];
    }
  }
#pragma unroll
  for (int i = 1; i <= RW; ++i)
#pragma unroll
    for (int q = 1; q <= 4; ++q) {
      const double a = fabs(f[i][q]);
      maxd = (a != a || maxd != maxd) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(maxd, a);
    }
  // codes of column x0 + 128 (as in scan_plane_f32)
  uint32_t Ye;
  {
    const int k = min(c.lane, RW);
    const double* p = S + (c.srow0 + k) * PITCH + XOFF + LX;
    const double ctr = p[0], l = p[-1];
    double r = p[1], u = p[-PITCH], d = p[PITCH];
    bool out = false;
    if (EDGE) {
      const long long gy = c.gy0 + k;
      if (c.xe_last) r = ctr;
      if (gy == 0) u = ctr;
      if (gy == c.ny - 1) d = ctr;
      out = c.xe_out || gy >= c.ny;
    }
    const double dx = r - l, dy = d - u;
    const uint32_t ce = out ? 0xF0u : (sbit(thr - dx) << 7) | (sbit(dx + thr) << 6) | (sbit(thr - dy) << 5) | (sbit(dy + thr) << 4);
    Ye = ce & __shfl_down_sync(0xffffffffu, ce, 1);
  }
  uint32_t C[RW + 1];
#pragma unroll
  for (int k = 0; k <= RW; ++k) {
    const long long gy = c.gy0 + k;
    const int iu = (EDGE && gy == 0) ? k + 1 : k, id = (EDGE && gy == c.ny - 1) ? k + 1 : k + 2;
    uint32_t W = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double dx = f[k + 1][q + 2] - f[k + 1][q], dy = f[id][q + 1] - f[iu][q + 1];
      const uint32_t nib = (sbit(thr - dx) << 3) | (sbit(dx + thr) << 2) | (sbit(thr - dy) << 1) | sbit(dy + thr);
      W |= nib << (8 * q + 4);
    }
    C[k] = (EDGE && gy >= c.ny) ? 0xF0F0F0F0u : (EDGE ? W | (~c.xmask & 0xF0F0F0F0u) : W);
  }
#pragma unroll
  for (int k = 0; k < RW; ++k) {
    const uint32_t Y = C[k] & C[k + 1];
    uint32_t nb = __shfl_down_sync(0xffffffffu, Y, 1);  // next lane's position 0
    const uint32_t ne = __shfl_sync(0xffffffffu, Ye, k);  // column x0 + 128
    if (c.lane == 31) nb = ne;
    Sq[k] = Y & ((Y >> 8) | (nb << 24));
  }
}

// ---------------------------------------------------------------------------------------------
// K1a: the scan kernel
// ---------------------------------------------------------------------------------------------
template <typename T, bool TMA>
__global__ void __launch_bounds__(NTHREADS, FTK_K1_MINB)
    k_scan2d(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ ExtractParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t mis = smem_u32(smem_raw) & 127u;  // dynamic smem is only 16-byte aligned
  ScanSmem<T>& sm = *reinterpret_cast<ScanSmem<T>*>(smem_raw + (mis ? 128 - mis : 0));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NSTAGE = ScanSmem<T>::NSTAGE;

  const i64 nx = P.nx, ny = P.ny;
  constexpr uint32_t STAGE_BYTES = ROWS * PITCH * sizeof(T);
  const int ntx = (int)((nx + TX - 1) / TX), nty = (int)((ny + TY - 1) / TY);
  const int tch = (int)P.tchunk;
  const int ntz = (int)((P.tb - P.ta + tch - 1) / tch);
  const long long nitems = (long long)ntx * nty * ntz;

  if (tid == 0) {
    sm.surv = 0;
    sm.maxbits32 = 0;
    sm.maxbits64 = 0;
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], NSW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  Prof pf;
#pragma unroll
  for (int i = 0; i < PF_N; ++i) pf.acc[i] = 0;
  pf.start();

  if (warp == PRODUCER) {
    // ------------------------------------------------------------------ producer warp
    const T* field = reinterpret_cast<const T*>(P.field);
    int gk = 0;  // planes issued so far (ring position)
    auto acquire = [&](int s) {
      pf.lap(PF_OTHER);
      if (gk >= NSTAGE) mbar_wait_sleep(&sm.empty[s], (uint32_t)((gk / NSTAGE - 1) & 1), 1, gk);
      pf.lap(PF_PRODWAIT);
    };
    while (true) {
      long long item = 0;
      if (lane == 0) item = (long long)atomicAdd(&P.counters[CNT_WORK], 1ull);
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item >= nitems) break;
      const int tx = (int)(item % ntx), ty_ = (int)((item / ntx) % nty), tz = (int)(item / ((long long)ntx * nty));
      const i64 x0 = (i64)tx * TX, y0 = (i64)ty_ * TY;
      const i64 ta = P.ta + (i64)tz * tch;
      const i64 tb = min(ta + tch, P.tb);
      const i64 plast = min(tb, P.nt_global - 1);
      const int np = (int)(plast - ta + 1);
      for (int k = 0; k < np; ++k, ++gk) {
        const int s = gk % NSTAGE;
        acquire(s);
        if (lane == 0) {
          StageMeta& m = sm.meta[s];
          m.x0 = (int)x0;
          m.y0 = (int)y0;
          m.p = (int)(ta + k);
          m.k = k;
          m.nplanes = np;
          m.tb = (int)tb;
          m.done = 0;
        }
        if (TMA) {
          if (lane == 0) {
            mbar_expect_tx(&sm.full[s], STAGE_BYTES);
            tma_load_3d(sm.plane[s], &tmap, &sm.full[s], (int)(x0 - XOFF), (int)(y0 - YOFF), (int)(ta + k - P.t0));
          }
        } else {
          // generic loader for unaligned shapes: guarded element loads (zero outside the grid)
          const T* src = field + (ta + k - P.t0) * nx * ny;
          T* dst = sm.plane[s];
          for (int idx = lane; idx < ROWS * PITCH; idx += 32) {
            const int rr = idx / PITCH, cc = idx - rr * PITCH;
            const i64 yy = y0 - YOFF + rr, xx = x0 - XOFF + cc;
            dst[idx] = (yy >= 0 && yy < ny && xx >= 0 && xx < nx) ? src[yy * nx + xx] : (T)0;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.full[s]);
        }
      }
    }
    // end-of-work marker
    const int s = gk % NSTAGE;
    acquire(s);
    if (lane == 0) {
      sm.meta[s].done = 1;
      mbar_arrive(&sm.full[s]);
    }
  } else {
    // ------------------------------------------------------------------ scan warps
    const T thr = (T)P.thr;
    const f2 thr2 = pack2((float)P.thr, (float)P.thr);
    const f2 nthr2 = pack2(-(float)P.thr, -(float)P.thr);
    uint32_t maxb32 = 0;
    double maxd = 0.0;
    unsigned long long mysurv = 0;
    uint32_t prevSq[RW];
    const int sw = warp;                 // scan-warp index: anchor rows sw*RW .. sw*RW + RW - 1
    const int srow0 = YOFF + sw * RW;    // smem row of this warp's first anchor row
    // the warp's current chunk of the window buffer: entries [cur, end)
    long long cur = 0, end = 0;

    // Hand the survivors to K1b as group entries: one per lane with surviving cubes, holding the
    // lane's first anchor (x0 + 4 lane, first anchor row of the warp), the plane flag and the lane's
    // 32-bit survivor mask (bit 8i + r <-> position i, anchor row r); K1b expands the masks and
    // fetches the cube windows from the field.  Entries are reserved in chunks of CHUNK with one
    // global atomic per warp and chunk.
    const uint32_t lt_mask = (1u << lane) - 1u;
    auto enqueue = [&](uint32_t mask, int tflag, int x0, int y0) {
      const uint32_t bal = __ballot_sync(0xffffffffu, mask != 0);
      if (bal == 0u) return;
      const int n = __popc(bal), rank = __popc(bal & lt_mask);
      const int avail = (int)(end - cur);
      long long e = cur + rank;
      if (n > avail) {  // the chunk runs out: the rest goes to a fresh chunk (n <= 32 = CHUNK)
        long long c = 0;
        if (lane == 0) c = (long long)atomicAdd(&P.counters[CNT_WIN], (unsigned long long)CHUNK);
        c = __shfl_sync(0xffffffffu, c, 0);
        if (rank >= avail) e = c + (rank - avail);
        cur = c + (n - avail);
        end = c + CHUNK;
      } else {
        cur += n;
      }
      if (mask != 0u && e < P.wcap) {
        P.wx[e] = x0 + 4 * lane;
        P.wy[e] = y0 + sw * RW;
        P.wt[e] = tflag;
        P.wz[e] = (int)mask;
      }
      mysurv += __popc(mask);
    };
    static_assert(CHUNK >= 32, "one fresh chunk must hold a whole warp's group entries");

    int gk = 0;
    int x0 = -1, y0 = -1;
    int mode = 0;
    int chk_k = -1, chk_p = -1;  // FTK_CHECKS: the previous plane of the item
    ScanCtx sc;
    sc.srow0 = srow0;
    sc.lane = lane;
    sc.ny = ny;
    sc.rpos = -1;
    sc.lpat = false;
    sc.xe_out = false;
    sc.xe_last = false;
    sc.xmask = 0xF0F0F0F0u;
    sc.gy0 = 0;
    while (true) {
      const int s = gk % NSTAGE;
      pf.lap(PF_OTHER);
      if (FTK_K1_SCANSLEEP) mbar_wait_sleep(&sm.full[s], (uint32_t)((gk / NSTAGE) & 1), 3, gk);
      else mbar_wait(&sm.full[s], (uint32_t)((gk / NSTAGE) & 1), 3, gk, FTK_K1_MBSLEEP);
      pf.lap(PF_WFULL);
      const StageMeta m = sm.meta[s];
      if (m.done) break;
      // protocol: within a work item the planes arrive in order (a stage refilled too early shows here)
      FTK_ASSERT(m.k == 0 || (m.k == chk_k + 1 && m.p == chk_p + 1));
      FTK_ASSERT(m.k < m.nplanes && m.x0 >= 0 && m.y0 >= 0);
      chk_k = m.k;
      chk_p = m.p;
      if (m.k == 0) {
        x0 = m.x0;
        y0 = m.y0;
        const i64 gx = (i64)x0 + 4 * lane;
        sc.gy0 = (i64)y0 + sw * RW;
        const bool xedge = x0 < 1 || x0 + LX + 2 > nx, yedge = sc.gy0 < 1 || sc.gy0 + RW + 2 > ny;
        mode = yedge ? 2 : (xedge ? 1 : 0);
        sc.xe_out = x0 + LX >= nx;
        sc.xe_last = x0 + LX == nx - 1;
        sc.lpat = gx == 0;
        sc.rpos = (nx - 1 >= gx && nx - 1 <= gx + 3) ? (int)(nx - 1 - gx) : -1;
        sc.xmask = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (gx + i < nx) sc.xmask |= 0xF0u << (8 * i);
      }
      const T* S = sm.plane[s];
      uint32_t Sq[RW];
      if constexpr (sizeof(T) == 4) {
        if (mode == 2) scan_plane_f32<2>(S, sc, thr2, nthr2, Sq, maxb32);
        else if (mode == 1) scan_plane_f32<1>(S, sc, thr2, nthr2, Sq, maxb32);
        else scan_plane_f32<0>(S, sc, thr2, nthr2, Sq, maxb32);
      } else {
        if (mode) scan_plane_f64<true>(S, sc, (double)thr, Sq, maxd);
        else scan_plane_f64<false>(S, sc, (double)thr, Sq, maxd);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);  // the plane is no longer needed by this warp
      pf.lap(PF_SCAN);
      // survivors: zero bytes after the AND over the cube's corners (exact zero-byte test: the
      // low nibbles repeat bit 4 or are zero, so no borrow can flag a nonzero byte); bit 8i + r <-> position i,
      // anchor row r
      auto survivors_of = [&](const uint32_t* K) {
        uint32_t mask = 0;
#pragma unroll
        for (int r = 0; r < RW; ++r) mask |= (((K[r] - 0x01010101u) & ~K[r] & 0x80808080u) >> (7 - r));
        return mask;
      };
      // pass 0: anchors at p-1 (cube = planes p-1, p); pass 1: anchors on the last timestep (no
      // t+1 corners: the AND runs over the plane only)
      const bool lastg = m.p == P.nt_global - 1 && m.p < m.tb;
#pragma unroll 1
      for (int pass = (m.k > 0 ? 0 : 1); pass < (lastg ? 2 : 1); ++pass) {
        uint32_t K[RW];
#pragma unroll
        for (int r = 0; r < RW; ++r) K[r] = pass == 0 ? (prevSq[r] & Sq[r]) : Sq[r];
        enqueue(survivors_of(K), pass == 0 ? (int)((uint32_t)(m.p - 1) | 0x80000000u) : m.p, x0, y0);
      }
      pf.lap(PF_ENQ);
#pragma unroll
      for (int r = 0; r < RW; ++r) prevSq[r] = Sq[r];
      ++gk;
    }
    // the unused rest of the warp's chunk holds no cube
    for (long long e = cur + lane; e < end; e += 32)
      if (e < P.wcap) P.wz[e] = 0;

    // statistics
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mysurv += __shfl_xor_sync(0xffffffffu, mysurv, o);  // survivors were counted per lane
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
  if (FTK_K1_PROF && lane == 0) {
    pf.lap(PF_OTHER);
#pragma unroll
    for (int i = 0; i < PF_N; ++i) atomicAdd(&P.counters[CNT_PROF + i], pf.acc[i]);
  }
  __syncthreads();
  if (tid == 0) {
    atomicAdd(&P.counters[CNT_SURVIVORS], sm.surv);
    atomicMax(&P.counters[CNT_MAXBITS], sizeof(T) == 4 ? (unsigned long long)sm.maxbits32 : sm.maxbits64);
  }
}

// Between K1a and K1b: expand the group entries (one per scan lane with surviving cubes: first
// anchor, plane flag, 32-bit survivor mask) into the dense cube list K1b takes in batches of 32.
// A block takes EXPI x 256 consecutive entries (EXPI per thread), block-wide exclusive scan of the
// survivor counts, one global atomic per block.
constexpr int EXPI = 4;
__global__ void __launch_bounds__(256) k_expand2d(const __grid_constant__ ExtractParams P) {
  __shared__ int wsum[8];
  __shared__ unsigned long long bbase;
  const long long ng = min((long long)P.counters[CNT_WIN], (long long)P.wcap);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (long long t0 = (long long)blockIdx.x * 256 * EXPI; t0 < ng; t0 += (long long)gridDim.x * 256 * EXPI) {
    const long long e0 = t0 + (long long)threadIdx.x * EXPI;
    uint32_t m[EXPI];
    int cnt = 0;
#pragma unroll
    for (int i = 0; i < EXPI; ++i) {
      m[i] = e0 + i < ng ? (uint32_t)P.wz[e0 + i] : 0u;
      cnt += __popc(m[i]);
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    int wex = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int v = wsum[k];
      wex += k < wid ? v : 0;
      tot += v;
    }
    if (threadIdx.x == 0) bbase = tot ? atomicAdd(&P.counters[CNT_CUBES], (unsigned long long)tot) : 0ull;
    __syncthreads();
    long long o = (long long)bbase + wex + incl - cnt;
#pragma unroll
    for (int i = 0; i < EXPI; ++i) {
      uint32_t mm = m[i];
      if (!mm) continue;
      const long long e = e0 + i;
      const int x = P.wx[e], y = P.wy[e], t = P.wt[e];
      for (; mm; mm &= mm - 1, ++o) {
        const int bit = __ffs(mm) - 1;
        if (o < P.wcap) {
          P.cx[o] = x + (bit >> 3);
          P.cy[o] = y + (bit & 7);
          P.ct[o] = t;
        }
      }
    }
    __syncthreads();  // wsum / bbase are rewritten by the next tile
  }
}

// ---------------------------------------------------------------------------------------------
// K1b: the exact kernel -- one warp per batch of 32 window-buffer entries (claimed dynamically, the entry
// count is read from the device counter K1a left behind)
// ---------------------------------------------------------------------------------------------
// window of a cube on the spatial boundary (zero outside the grid), raw values; out of line -- rare,
// and it keeps the guarded loads out of the kernel's hot code
template <typename T>
__device__ __noinline__ void load_window_edge(T* dst, const T* field, i64 t0, const Geo& G, int x, int y, int et) {
  const T* pa = field + ((i64)(et & 0x3fffffff) - t0) * G.nx * G.ny;
  const T* pb = et < 0 ? pa + G.nx * G.ny : pa;
#pragma unroll 1
  for (int k = 0; k < 32; ++k) {
    const i64 xx = x - 1 + (k & 3), yy = y - 1 + ((k >> 2) & 3);
    dst[k] = (xx >= 0 && xx < G.nx && yy >= 0 && yy < G.ny) ? __ldg((k < 16 ? pa : pb) + yy * G.nx + xx) : (T)0;
  }
}

template <typename T>
__global__ void __launch_bounds__(EXW * 32, FTK_X_MINB) k_exact2d(const __grid_constant__ ExtractParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ExSmem<T>& sm = *reinterpret_cast<ExSmem<T>*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Geo G;
  G.nx = P.nx;
  G.ny = P.ny;
  G.ntg = P.nt_global;
  G.scale = P.scale;
  G.scale_f = (float)P.scale;
  G.qmax = ldexp(1.0, 29) / P.scale - 1.0 / P.scale;  // |f| < qmax -> |rint(f 2^s)| < 2^29
  const float qmaxf = (float)G.qmax;
  BatchBuf bb{sm.ring + w * 32 * ws_words<T>(), sm.qx + w * 32, sm.qy + w * 32, sm.qt + w * 32, sm.items[w],
              sm.lp + w * 32, sm.pm + w * 32, sm.rs + w * 32};
  const long long nwin = min((long long)*(volatile unsigned long long*)&P.counters[CNT_CUBES], (long long)P.wcap);
  const long long nbat = (nwin + 31) / 32;
  const T* field = reinterpret_cast<const T*>(P.field);
  Prof pf;
#pragma unroll
  for (int i = 0; i < PF_N; ++i) pf.acc[i] = 0;
  pf.start();
  // Each lane's cube of the batch in flight: its list entry and (interior cubes) its raw 4x4x2 window.
  // The next batch's loads are issued before this batch's exact stage (fp32), so the window fetch
  // overlaps the face tests and records instead of stalling the warp.
  constexpr bool PREFETCH = sizeof(T) == 4;
  int et = -1, cxv = 0, cyv = 0;
  bool inner = false;
  T v[32];
  auto fetch = [&](long long b) {
    const long long e = b * 32 + lane;
    et = e < nwin ? P.ct[e] : -1;
    inner = false;
    if (et != -1) {
      cxv = P.cx[e];
      cyv = P.cy[e];
      inner = cxv >= 1 && cxv + 2 < G.nx && cyv >= 1 && cyv + 2 < G.ny;
      if (inner) {
        // the cube's 4x4x2 window (planes t and t+1; t again when t+1 is not in the domain)
        const T* pa = field + ((i64)(et & 0x3fffffff) - P.t0) * G.nx * G.ny + (i64)(cyv - 1) * G.nx + (cxv - 1);
        const T* pb = et < 0 ? pa + G.nx * G.ny : pa;
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = __ldg((k < 16 ? pa : pb) + ((k >> 2) & 3) * G.nx + (k & 3));
      }
    }
  };
  // batches are claimed dynamically (one atomic per batch and warp): their cost varies with the
  // punctured faces they hold, and a static stride leaves the slowest warps as a tail
  auto claim = [&]() -> long long {
    long long c = 0;
    if (lane == 0) c = (long long)atomicAdd(&P.counters[CNT_XBATCH], 1ull);
    return __shfl_sync(0xffffffffu, c, 0);
  };
  long long b = claim();
  if (b < nbat) fetch(b);
  while (b < nbat) {
    const long long bn = claim();
    uint32_t* ent = bb.ring + lane * ws_words<T>();
    bool fast = false;
    if (et != -1) {
      if (inner) {
        if constexpr (sizeof(T) == 4) {
          float mx = 0.f;
#pragma unroll
          for (int k = 0; k < 32; ++k) mx = fmaxf(mx, fabsf(v[k]));
          fast = mx < qmaxf;  // last-timestep cubes too (the second plane repeats the first)
        }
        if (fast) {
          int qv[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            qv[k] = __float2int_rn(__fmul_rn((float)v[k], G.scale_f));  // |v 2^s| < 2^29: exact
            ent[k] = (uint32_t)qv[k];
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) {  // central differences at corner c: window (cx+1, cy+1)
            const int cx = c & 1, cy = (c >> 1) & 1, pl = c >> 2;
            ent[32 + 2 * c] = (uint32_t)(qv[pl * 16 + (cy + 1) * 4 + cx + 2] - qv[pl * 16 + (cy + 1) * 4 + cx]);
            ent[33 + 2 * c] = (uint32_t)(qv[pl * 16 + (cy + 2) * 4 + cx + 1] - qv[pl * 16 + cy * 4 + cx + 1]);
          }
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) reinterpret_cast<T*>(ent)[k] = v[k];
        }
      } else {
        load_window_edge<T>(reinterpret_cast<T*>(ent), field, P.t0, G, cxv, cyv, et);
      }
      bb.qx[lane] = cxv;
      bb.qy[lane] = cyv;
    }
    bb.qt[lane] = et == -1 ? -1 : (et | (fast ? 0x40000000 : 0));
    __syncwarp();
    if (PREFETCH && bn < nbat) fetch(bn);
    pf.lap(PF_EXLOAD);
    process_batch<T>(bb, G, P, pf);
    __syncwarp();
    if (!PREFETCH && bn < nbat) fetch(bn);
    pf.lap(PF_EXREC);
    b = bn;
  }
  if (FTK_K1_PROF && lane == 0) {
#pragma unroll
    for (int i = 0; i < PF_N; ++i) atomicAdd(&P.counters[CNT_PROF + i], pf.acc[i]);
  }
}

}  // namespace k2d

// ---------------------------------------------------------------------------------------------
// Host launcher
// ---------------------------------------------------------------------------------------------
using sm100::get_encode;

template <typename T, bool TMA>
static int launch_t(const ExtractParams& P, cudaStream_t stream) {
  using namespace k2d;
  CUtensorMap map;
  memset(&map, 0, sizeof map);
  if (TMA) {
    EncodeTiledFn enc = get_encode();
    const cuuint64_t dims[3] = {(cuuint64_t)P.nx, (cuuint64_t)P.ny, (cuuint64_t)P.nt_buf};
    const cuuint64_t strides[2] = {(cuuint64_t)P.nx * sizeof(T), (cuuint64_t)P.nx * P.ny * sizeof(T)};
    const cuuint32_t box[3] = {PITCH, ROWS, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&map, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                     const_cast<void*>(P.field), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return launch_t<T, false>(P, stream);
  }
  const size_t smem = sizeof(ScanSmem<T>) + 128;
  auto kern = k_scan2d<T, TMA>;
  const sm100::LaunchGeom lg = sm100::launch_geom(kern, NTHREADS, smem);
  if (lg.err != cudaSuccess) return set_cuda_error(lg.err, "k_scan2d launch geometry");
  const int sms = lg.sms, per_sm = lg.per_sm;
  const long long tiles = ((P.nx + TX - 1) / TX) * ((P.ny + TY - 1) / TY);
  const long long slots = (long long)sms * std::max(per_sm, 1);
  ExtractParams Q = P;
  Q.tchunk = TCHUNK;
  if (tiles * ((P.tb - P.ta + TCHUNK - 1) / TCHUNK) < 16 * slots) Q.tchunk = TCHUNK / 2;
  const long long items = tiles * ((P.tb - P.ta + Q.tchunk - 1) / Q.tchunk);
  if (items <= 0) return FTK_OK;
  const long long grid = std::min<long long>(items, slots);
  kern<<<(unsigned)grid, NTHREADS, smem, stream>>>(map, Q);
  FTK_CUDA_TRY(cudaGetLastError());
  if (P.ev_mid) FTK_CUDA_TRY(cudaEventRecord(reinterpret_cast<cudaEvent_t>(P.ev_mid), stream));
  {
    const int st = launch_expand2d(P, stream, sms);
    if (st) return st;
  }
  // K1b: persistent grid over the cube list
  const size_t xsmem = sizeof(ExSmem<T>);
  auto xk = k_exact2d<T>;
  const sm100::LaunchGeom xg = sm100::launch_geom(xk, EXW * 32, xsmem);
  if (xg.err != cudaSuccess) return set_cuda_error(xg.err, "k_exact2d launch geometry");
  const int xper = xg.per_sm;
  xk<<<(unsigned)(sms * std::max(xper, 1)), EXW * 32, xsmem, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

int launch_expand2d(const ExtractParams& P, cudaStream_t stream, int sms) {
  k2d::k_expand2d<<<(unsigned)(sms * 8), 256, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

int launch_extract2d(const ExtractParams& P, cudaStream_t stream) {
  const size_t esz = P.dtype == FTK_F32 ? 4 : 8;
  const bool aligned = (reinterpret_cast<uintptr_t>(P.field) % 16 == 0) && ((P.nx * esz) % 16 == 0);
  const bool tma = aligned && get_encode() != nullptr && !P.force_generic;
  if (P.nx >= (1ll << 31) - 256 || P.ny >= (1ll << 31) - 64 || P.nt_global >= (1ll << 30)) return FTK_ERR_INVALID_ARG;
  if (P.dtype == FTK_F32) return tma ? launch_t<float, true>(P, stream) : launch_t<float, false>(P, stream);
  return tma ? launch_t<double, true>(P, stream) : launch_t<double, false>(P, stream);
}

}  // namespace ftk
