// extract2d.cu -- K1: pass 1 of Alg. 1 for 2D+t on sm_100a.
//
// One CTA owns a 124 x 32 tile of anchors (x, y) and a chunk of anchor timesteps.  It marches t:
//
//   TMA (cp.async.bulk.tensor, mbarrier ring of NSTAGE planes) stages the plane tile with a halo
//   (x0-4 .. x0+131, y0-2 .. y0+34) in shared memory, so every vertex is read from HBM once and
//   reused by all 12 faces of the 8 cubes it belongs to (north_star (2)).
//
//   Scan (all warps, lane = 4 consecutive x, warp = 8 rows): a CONSERVATIVE sign prefilter on the
//   raw field values.  For gradient component g_a = q[+a] - q[-a] (q = rint(f 2^s)), the float
//   test (f[+a] - f[-a]) >= 2^(1-s) implies g_a > 0 exactly.  Four bits
//   per vertex (x+, x-, y+, y-) are ANDed over the 8 corners of each spacetime cube; a cube whose
//   AND is nonzero has a gradient component of one strict sign on all corners, so no face inside
//   it can contain the origin -- even under SoS (the perturbation is infinitesimal).  Survivors
//   (about 0.5% of cubes on the woven field) go to a CTA queue.
//
//   Exact stage (survivor queue, 32 cubes per warp at a time, data from shared memory): quantize,
//   exact int64 gradients, per-face exact sign reject, SoS point-in-simplex with exact 2x2
//   determinants (int64, or int128 when |g| >= 2^31), Eq. 2 location and the Hessian type in
//   fixed-order FP64 (no FMA), ballot/prefix-sum compaction with one global atomic per warp batch.
#include <cuda.h>

#include <cstring>
#include <utility>

#include "common.cuh"
#include "extract2d.cuh"
#include "kuhn.cuh"

namespace ftk {
namespace k2d {

// ---------------------------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  long long spins = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (++spins > (1ll << 26)) __trap();  // never hang the GPU on a lost transaction
  }
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---------------------------------------------------------------------------------------------
// Tile geometry
// ---------------------------------------------------------------------------------------------
constexpr int LX = 128;             // x positions scanned per warp row (32 lanes x 4)
constexpr int TX = 124;             // anchors owned per CTA in x: lane 31 is a halo lane whose
                                    // codes only complete lane 30's cubes (a cube needs x+1)
constexpr int RW = 8;               // anchor rows per warp
constexpr int NWARP = 4;            // warps per CTA
constexpr int TY = RW * NWARP;      // 32 anchor rows per CTA
constexpr int XOFF = 4;             // smem column of x0
constexpr int YOFF = 2;             // smem row of y0
constexpr int PITCH = LX + 8;       // x0-4 .. x0+131
constexpr int ROWS = TY + 5;        // y0-2 .. y0+34
constexpr int NSTAGE = 4;
constexpr int QCAP = TX * TY;       // survivor queue capacity (one plane step)

// one stage = the plane tile, padded to a multiple of 128 bytes (TMA destination alignment)
template <typename T>
constexpr int stage_elems() {
  return (ROWS * PITCH * (int)sizeof(T) + 127) / 128 * 128 / (int)sizeof(T);
}

template <typename T>
struct alignas(128) Smem {
  T plane[NSTAGE][stage_elems<T>()];
  uint64_t full[NSTAGE];
  uint16_t queue[QCAP];
  int qn[2];
  unsigned long long surv;
  unsigned long long maxbits;
};

template <typename T>
struct Bits;
template <>
struct Bits<float> {
  using U = uint32_t;
  __device__ static U absbits(float v) { return __float_as_uint(v) & 0x7fffffffu; }
};
template <>
struct Bits<double> {
  using U = unsigned long long;
  __device__ static U absbits(double v) { return (U)__double_as_longlong(v) & 0x7fffffffffffffffull; }
};

// ---------------------------------------------------------------------------------------------
// Exact stage helpers
// ---------------------------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ i64 quant(T f, double scale) {
  // q = rint(f * 2^s): (double)f * 2^s is exact (power-of-two scale), __double2ll_rn rounds half-even
  return __double2ll_rn(__dmul_rn((double)f, scale));
}

// SoS sign of the 2x2 determinant | ua va ; ub vb | with rows a < b (global vertex order) and
// perturbation eps_{r,j} = eps^(2^(2r+j)) (R4).  Leading terms of det(M + E) in
// decreasing magnitude: det, +v_b, -u_b, -v_a, then -1 (a constant: the chain always ends).
template <bool WIDE>
__device__ __forceinline__ int sos2(i64 ua, i64 va, i64 ub, i64 vb) {
  int s;
  if (WIDE) {
    s = sgn128(det2(ua, va, ub, vb));
  } else {
    s = sgn64(ua * vb - va * ub);  // |g| < 2^31: |det| < 2^63
  }
  if (s) return s;
  if (vb) return vb > 0 ? 1 : -1;
  if (ub) return ub > 0 ? -1 : 1;
  if (va) return va > 0 ? -1 : 1;
  return -1;
}

// Point-in-simplex for the face with vertex gradients g0 < g1 < g2:
// s_k = (-1)^(k+2) sos(rows != k); punctured iff s_0 = s_1 = s_2.
template <bool WIDE>
__device__ __forceinline__ bool punctured3(const i64* g0, const i64* g1, const i64* g2) {
  const int s0 = sos2<WIDE>(g1[0], g1[1], g2[0], g2[1]);
  const int s1 = -sos2<WIDE>(g0[0], g0[1], g2[0], g2[1]);
  if (s0 != s1) return false;
  const int s2 = sos2<WIDE>(g0[0], g0[1], g1[0], g1[1]);
  return s0 == s2;
}

struct Geo {
  i64 nx, ny, ntg;   // grid extents (t = global)
  i64 x0, y0;        // tile origin
  double scale;
};

template <typename T>
__device__ __forceinline__ i64 qs(const T* P, const Geo& G, i64 x, i64 y) {
  return quant(P[(int)(y - G.y0 + YOFF) * PITCH + (int)(x - G.x0 + XOFF)], G.scale);
}

// exact gradient (2x the derivative; one-sided doubled at the spatial boundary, R7)
template <typename T>
__device__ __forceinline__ void grad_exact(const T* P, const Geo& G, i64 x, i64 y, i64* g) {
  if (x == 0) g[0] = 2 * (qs(P, G, 1, y) - qs(P, G, 0, y));
  else if (x == G.nx - 1) g[0] = 2 * (qs(P, G, x, y) - qs(P, G, x - 1, y));
  else g[0] = qs(P, G, x + 1, y) - qs(P, G, x - 1, y);
  if (y == 0) g[1] = 2 * (qs(P, G, x, 1) - qs(P, G, x, 0));
  else if (y == G.ny - 1) g[1] = 2 * (qs(P, G, x, y) - qs(P, G, x, y - 1));
  else g[1] = qs(P, G, x, y + 1) - qs(P, G, x, y - 1);
}

// integer Hessian, 4x scale, stencil centre clamped into [1, N-2] (R8); xx, xy, yy
template <typename T>
__device__ __forceinline__ void hessian_exact(const T* P, const Geo& G, i64 x, i64 y, i64* H) {
  const i64 cx = x < 1 ? 1 : (x > G.nx - 2 ? G.nx - 2 : x);
  const i64 cy = y < 1 ? 1 : (y > G.ny - 2 ? G.ny - 2 : y);
  H[0] = 4 * (qs(P, G, cx + 1, y) - 2 * qs(P, G, cx, y) + qs(P, G, cx - 1, y));
  H[1] = qs(P, G, cx + 1, cy + 1) - qs(P, G, cx + 1, cy - 1) - qs(P, G, cx - 1, cy + 1) + qs(P, G, cx - 1, cy - 1);
  H[2] = 4 * (qs(P, G, x, cy + 1) - 2 * qs(P, G, x, cy) + qs(P, G, x, cy - 1));
}

__device__ __forceinline__ double fma_free_dot3(const double* mu, double a, double b, double c) {
  return __dadd_rn(__dadd_rn(__dmul_rn(mu[0], a), __dmul_rn(mu[1], b)), __dmul_rn(mu[2], c));
}

// one face type, compile-time masks (the 12 canonical 2D+t types, kuhn.cuh)
template <int TY, bool WIDE>
__device__ __forceinline__ void face_test(const i64 (&g)[8][2], uint32_t exists, uint32_t& pmask) {
  constexpr int m1 = kKuhn3.masks[TY][0];
  constexpr int m2 = kKuhn3.masks[TY][1];
  if (((exists >> m2) & 1) == 0) return;  // the span's far corner must exist
  const i64* g0 = g[0];
  const i64* g1 = g[m1];
  const i64* g2 = g[m2];
  // exact per-face reject: a component of one strict sign on all three vertices
  bool rej = false;
#pragma unroll
  for (int j = 0; j < 2; ++j)
    rej |= (g0[j] > 0 && g1[j] > 0 && g2[j] > 0) || (g0[j] < 0 && g1[j] < 0 && g2[j] < 0);
  if (rej) return;
  if (punctured3<WIDE>(g0, g1, g2)) pmask |= 1u << TY;
}

template <bool WIDE, int... TY>
__device__ __forceinline__ void all_faces(const i64 (&g)[8][2], uint32_t exists, uint32_t& pmask,
                                          std::integer_sequence<int, TY...>) {
  (face_test<TY, WIDE>(g, exists, pmask), ...);
}

template <int K>
struct Face3 {
  static constexpr int m1 = kKuhn3.masks[K][0];
  static constexpr int m2 = kKuhn3.masks[K][1];
};
template <int... K>
__device__ __forceinline__ void masks_of(int ty, int& m1, int& m2, std::integer_sequence<int, K...>) {
  ((ty == K ? (m1 = Face3<K>::m1, m2 = Face3<K>::m2, 0) : 0), ...);
}

// g[c] for a runtime corner index without dynamic register indexing
__device__ __forceinline__ void sel_corner(const i64 (&g)[8][2], int c, i64* out) {
  out[0] = g[0][0];
  out[1] = g[0][1];
#pragma unroll
  for (int k = 1; k < 8; ++k)
    if (c == k) {
      out[0] = g[k][0];
      out[1] = g[k][1];
    }
}

// Process one surviving cube anchored at (x, y, t): test its 12 faces exactly and write records.
// A = plane t, B = plane t+1 (nullptr when t is the last global timestep).  All lanes of the warp
// call this together (valid = false lanes contribute nothing) for the warp-aggregated atomic.
template <typename T>
__device__ void process_cube(const T* A, const T* B, const Geo& G, i64 x, i64 y, i64 t, bool valid,
                             const ExtractParams& P) {
  const int lane = threadIdx.x & 31;
  i64 g[8][2];
  uint32_t exists = 0;   // corner existence
  uint32_t pmask = 0;    // punctured face types
  bool wide = false;
  if (valid) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const i64 cx = x + (c & 1), cy = y + ((c >> 1) & 1);
      const bool has_t = !(c & 4) || B != nullptr;
      if (cx < G.nx && cy < G.ny && has_t) {
        grad_exact((c & 4) ? B : A, G, cx, cy, g[c]);
        exists |= 1u << c;
        const i64 m = (g[c][0] < 0 ? -g[c][0] : g[c][0]) | (g[c][1] < 0 ? -g[c][1] : g[c][1]);
        wide |= m >= (1ll << 31);
      } else {
        g[c][0] = g[c][1] = 0;
      }
    }
    if (wide) all_faces<true>(g, exists, pmask, std::make_integer_sequence<int, 12>{});
    else all_faces<false>(g, exists, pmask, std::make_integer_sequence<int, 12>{});
  }
  // warp-aggregated reservation of output slots (one global atomic per warp batch)
  const int cnt = __popc(pmask);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (total == 0) return;
  unsigned long long base = 0;
  if (lane == 31) base = atomicAdd(&P.counters[CNT_NOUT], (unsigned long long)total);
  base = __shfl_sync(0xffffffffu, base, 31);
  unsigned long long slot = base + (unsigned long long)(incl - cnt);

  while (pmask) {
    const int ty = __ffs(pmask) - 1;
    pmask &= pmask - 1;
    int m[3] = {0, 0, 0};
    masks_of(ty, m[1], m[2], std::make_integer_sequence<int, 12>{});
    i64 gv[3][2];
    sel_corner(g, 0, gv[0]);
    sel_corner(g, m[1], gv[1]);
    sel_corner(g, m[2], gv[2]);
    // Eq. 2: mu_k = D_k / sum D, D_k = (-1)^(k+2) det(rows != k)
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
    double px[3], py[3], pt[3];
    double Hb[3] = {0, 0, 0};
    i64 Hk[3][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const i64 vx = x + (m[k] & 1), vy = y + ((m[k] >> 1) & 1), vt = t + ((m[k] >> 2) & 1);
      px[k] = (double)vx;
      py[k] = (double)vy;
      pt[k] = (double)vt;
      hessian_exact((m[k] & 4) ? B : A, G, vx, vy, Hk[k]);
    }
    const double lx = fma_free_dot3(mu, px[0], px[1], px[2]);
    const double ly = fma_free_dot3(mu, py[0], py[1], py[2]);
    const double lt = fma_free_dot3(mu, pt[0], pt[1], pt[2]);
#pragma unroll
    for (int e = 0; e < 3; ++e)
      Hb[e] = fma_free_dot3(mu, __ll2double_rn(Hk[0][e]), __ll2double_rn(Hk[1][e]), __ll2double_rn(Hk[2][e]));
    // type (R9): det of the interpolated Hessian, no tolerance
    const double det = __dsub_rn(__dmul_rn(Hb[0], Hb[2]), __dmul_rn(Hb[1], Hb[1]));
    int type;
    if (det < 0) type = FTK_CP_SADDLE;
    else if (det > 0) type = Hb[0] > 0 ? FTK_CP_MIN : FTK_CP_MAX;
    else type = FTK_CP_DEGENERATE;
    const int span = m[2];
    if (!(span & 4)) flags |= FTK_CP_ORDINAL;
    if (span != 7) {  // closed-form side_of: parents exist iff v0[c] in [1, N_c - 2]
      const int c = 7 & ~span;
      const i64 vc = c == 1 ? x : (c == 2 ? y : t);
      const i64 Nc = c == 1 ? G.nx : (c == 2 ? G.ny : G.ntg);
      if (vc == 0 || vc == Nc - 1) flags |= FTK_CP_BOUNDARY;
    }
    if (slot < (unsigned long long)P.capacity) {
      ftk_cp* r = P.out + slot;
      r->face_id = ((t * G.ny + y) * G.nx + x) * 12 + ty;
      r->label = -1;
      r->x = lx;
      r->y = ly;
      r->z = 0.0;
      r->t = lt;
      r->type = type;
      r->flags = flags;
    }
    ++slot;
  }
}

// ---------------------------------------------------------------------------------------------
// Scan helpers
// ---------------------------------------------------------------------------------------------
template <typename T>
struct Row {
  T l, a, b, c, d, r;  // f[x-1], f[x..x+3], f[x+4]
};

template <typename T>
__device__ __forceinline__ Row<T> load_row(const T* S, int srow, int lane) {
  Row<T> w;
  const T* p = S + srow * PITCH + XOFF + 4 * lane;
  if constexpr (sizeof(T) == 4) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    w.a = v.x; w.b = v.y; w.c = v.z; w.d = v.w;
  } else {
    const double2 v0 = *reinterpret_cast<const double2*>(p);
    const double2 v1 = *reinterpret_cast<const double2*>(p + 2);
    w.a = v0.x; w.b = v0.y; w.c = v1.x; w.d = v1.y;
  }
  T up = __shfl_up_sync(0xffffffffu, w.d, 1);
  T dn = __shfl_down_sync(0xffffffffu, w.a, 1);
  // lanes 0 and 31 take the tile halo from shared memory (one predicated load)
  if (lane == 0 || lane == 31) {
    const T h = S[srow * PITCH + (lane == 0 ? XOFF - 1 : XOFF + LX)];
    if (lane == 0) up = h; else dn = h;
  }
  w.l = up;
  w.r = dn;
  return w;
}

// 4-bit sign code of one vertex: bit0 dx >= thr, bit1 dx <= -thr, bit2 dy >= thr, bit3 dy <= -thr.
template <typename T>
__device__ __forceinline__ uint32_t code4(T dx, T dy, T thr) {
  return (uint32_t)(dx >= thr) | ((uint32_t)(dx <= -thr) << 1) | ((uint32_t)(dy >= thr) << 2) |
         ((uint32_t)(dy <= -thr) << 3);
}

// codes of the lane's 4 positions on one row (16 bits).  EDGE: apply the one-sided boundary rule
// and neutral codes (0xF) outside the grid.
template <typename T, bool EDGE>
__device__ __forceinline__ uint32_t row_codes(const Row<T>& up, const Row<T>& cur, const Row<T>& dn, T thr,
                                              i64 gx, i64 gy, i64 nx, i64 ny) {
  const T f[6] = {cur.l, cur.a, cur.b, cur.c, cur.d, cur.r};
  const T fu[4] = {up.a, up.b, up.c, up.d};
  const T fd[4] = {dn.a, dn.b, dn.c, dn.d};
  uint32_t C = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    T lo = f[i], hi = f[i + 2], ylo = fu[i], yhi = fd[i];
    if (EDGE) {
      const i64 x = gx + i;
      if (x == 0) lo = f[i + 1];
      if (x == nx - 1) hi = f[i + 1];
      if (gy == 0) ylo = f[i + 1];
      if (gy == ny - 1) yhi = f[i + 1];
    }
    uint32_t c = code4(hi - lo, yhi - ylo, thr);
    if (EDGE && (gx + i >= nx || gy >= ny)) c = 0xF;
    C |= c << (4 * i);
  }
  return C;
}

// ---------------------------------------------------------------------------------------------
// The kernel
// ---------------------------------------------------------------------------------------------
template <typename T, bool TMA>
__global__ void __launch_bounds__(NWARP * 32, 2)
    k_extract2d(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ ExtractParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // the dynamic shared window is only guaranteed 16-byte alignment: round up to 128
  const uint32_t mis = smem_u32(smem_raw) & 127u;
  Smem<T>& sm = *reinterpret_cast<Smem<T>*>(smem_raw + (mis ? 128 - mis : 0));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  Geo G;
  G.nx = P.nx;
  G.ny = P.ny;
  G.ntg = P.nt_global;
  G.x0 = (i64)blockIdx.x * TX;
  G.y0 = (i64)blockIdx.y * TY;
  G.scale = P.scale;
  const i64 ta = P.ta + (i64)blockIdx.z * P.tchunk;
  const i64 tb = min(ta + P.tchunk, P.tb);           // anchor planes [ta, tb)
  const i64 plast = min(tb, P.nt_global - 1);         // planes ta .. plast are loaded
  const int nplanes = (int)(plast - ta + 1);
  const T* field = reinterpret_cast<const T*>(P.field);
  const T thr = (T)P.thr;

  if (tid == 0) {
    sm.qn[0] = sm.qn[1] = 0;
    sm.surv = 0;
    sm.maxbits = 0;
    if (TMA) {
      for (int s = 0; s < NSTAGE; ++s) mbar_init(&sm.full[s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  constexpr uint32_t STAGE_BYTES = ROWS * PITCH * sizeof(T);
  if (TMA && tid == 0) {
    for (int k = 0; k < NSTAGE && k < nplanes; ++k) {
      mbar_expect_tx(&sm.full[k], STAGE_BYTES);
      tma_load_3d(sm.plane[k], &tmap, &sm.full[k], (int)(G.x0 - XOFF), (int)(G.y0 - YOFF), (int)(ta + k - P.t0));
    }
  }

  const bool edge = G.x0 < 1 || G.x0 + LX + 1 > G.nx || G.y0 < 1 || G.y0 + TY + 2 > G.ny;
  const i64 gx = G.x0 + 4 * lane;            // first x of this lane
  const i64 gy0 = G.y0 + warp * RW;          // first anchor row of this warp
  const int srow0 = YOFF + warp * RW;        // its smem row
  typename Bits<T>::U maxb = 0;
  uint32_t prevSq[RW];
#pragma unroll
  for (int r = 0; r < RW; ++r) prevSq[r] = 0xFFFFu;

  auto scan_plane = [&](const T* S, uint32_t* Sq) {
    Row<T> up = load_row<T>(S, srow0 - 1, lane);
    Row<T> cur = load_row<T>(S, srow0, lane);
    uint32_t Cprev = 0;
#pragma unroll
    for (int r = 0; r <= RW; ++r) {
      const Row<T> dn = load_row<T>(S, srow0 + r + 1, lane);
      if (r < RW) {
        maxb = max(maxb, max(max(Bits<T>::absbits(cur.a), Bits<T>::absbits(cur.b)),
                             max(Bits<T>::absbits(cur.c), Bits<T>::absbits(cur.d))));
      }
      const uint32_t C = edge ? row_codes<T, true>(up, cur, dn, thr, gx, gy0 + r, G.nx, G.ny)
                              : row_codes<T, false>(up, cur, dn, thr, gx, gy0 + r, G.nx, G.ny);
      if (r > 0) {
        uint32_t Y = Cprev & C;                                   // y-pair AND (per position)
        // x-pair AND; position 4 = the next lane's position 0 (lane 31's cubes are not owned:
        // its x+1 corners are unknown here, and unknown corners must NOT enter the AND)
        const uint32_t nb = __shfl_down_sync(0xffffffffu, Y, 1) & 0xFu;
        Sq[r - 1] = Y & ((Y >> 4) | (nb << 12));
      }
      Cprev = C;
      up = cur;
      cur = dn;
    }
  };

  // push the survivors of anchor plane (given by their 32-bit mask: bit 4r+i) to the CTA queue
  auto push = [&](uint32_t mask, int qsel) {
    const int cnt = __popc(mask);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) return;
    int base = 0;
    if (lane == 31) base = atomicAdd(&sm.qn[qsel], total);
    base = __shfl_sync(0xffffffffu, base, 31);
    int pos = base + incl - cnt;
    while (mask) {
      const int b = __ffs(mask) - 1;
      mask &= mask - 1;
      const int r = b >> 2, i = b & 3;
      sm.queue[pos++] = (uint16_t)((4 * lane + i) | ((warp * RW + r) << 7));
    }
  };

  auto survivors_of = [&](const uint32_t* K) {
    uint32_t mask = 0;
    if (lane == 31) return mask;  // halo lane owns no anchors
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      uint32_t z = K[r] | (K[r] >> 1);
      z |= z >> 2;
      const uint32_t m = ~z & 0x1111u;                 // nibble == 0  ->  survivor
      mask |= (((m * 0x249u) >> 9) & 0xFu) << (4 * r); // gather bits 0,4,8,12 -> 0..3
    }
    return mask;
  };

  auto process_queue = [&](const T* A, const T* B, i64 t, int n) {
    for (int e0 = warp * 32; e0 < n; e0 += NWARP * 32) {
      const int e = e0 + lane;
      const bool valid = e < n;
      const uint32_t code = valid ? sm.queue[e] : 0u;
      const i64 x = G.x0 + (code & 127u), y = G.y0 + (code >> 7);
      process_cube<T>(A, B, G, x, y, t, valid, P);
    }
  };

  for (int k = 0; k < nplanes; ++k) {
    const i64 p = ta + k;
    const int s = k % NSTAGE;
    T* S = sm.plane[s];
    if (TMA) {
      mbar_wait(&sm.full[s], (uint32_t)((k / NSTAGE) & 1));
    } else {
      // generic loader: guarded element loads of the plane tile (zero outside the grid)
      const T* src = field + (p - P.t0) * G.nx * G.ny;
      for (int idx = tid; idx < ROWS * PITCH; idx += NWARP * 32) {
        const int rr = idx / PITCH, cc = idx % PITCH;
        const i64 yy = G.y0 - YOFF + rr, xx = G.x0 - XOFF + cc;
        S[idx] = (yy >= 0 && yy < G.ny && xx >= 0 && xx < G.nx) ? src[yy * G.nx + xx] : (T)0;
      }
      __syncthreads();
    }
    uint32_t Sq[RW];
    scan_plane(S, Sq);
    const int qsel = k & 1;
    if (k > 0) {
      uint32_t K[RW];
#pragma unroll
      for (int r = 0; r < RW; ++r) K[r] = prevSq[r] & Sq[r];
      push(survivors_of(K), qsel);
    }
#pragma unroll
    for (int r = 0; r < RW; ++r) prevSq[r] = Sq[r];
    const bool last_global = (p == P.nt_global - 1) && (p < tb);  // anchors on the last timestep
    __syncthreads();  // (A) queue complete
    const int n1 = sm.qn[qsel];
    if (k > 0) process_queue(sm.plane[(k - 1) % NSTAGE], S, p - 1, n1);
    int n2 = 0;
    if (last_global) {
      __syncthreads();  // queue entries consumed
      uint32_t K[RW];
#pragma unroll
      for (int r = 0; r < RW; ++r) K[r] = Sq[r];  // no t+1 corners: AND over the plane only
      push(survivors_of(K), qsel ^ 1);
      __syncthreads();
      n2 = sm.qn[qsel ^ 1];
      process_queue(S, nullptr, p, n2);
    }
    __syncthreads();  // (B) plane p-1 is free, every reader of the counters is done
    if (tid == 0) {
      sm.surv += (unsigned long long)(n1 + n2);
      sm.qn[qsel] = 0;
      if (last_global) sm.qn[qsel ^ 1] = 0;
    }
    if (TMA && tid == 0 && k >= 1 && k - 1 + NSTAGE < nplanes) {
      const int kn = k - 1 + NSTAGE;
      const int sn = kn % NSTAGE;
      fence_proxy_async();
      mbar_expect_tx(&sm.full[sn], STAGE_BYTES);
      tma_load_3d(sm.plane[sn], &tmap, &sm.full[sn], (int)(G.x0 - XOFF), (int)(G.y0 - YOFF), (int)(ta + kn - P.t0));
    }
  }

  // block-level reductions of the statistics
  if constexpr (sizeof(T) == 4) {
    uint32_t m = maxb;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) atomicMax(&sm.maxbits, (unsigned long long)m);
  } else {
    unsigned long long m = maxb;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) atomicMax(&sm.maxbits, m);
  }
  __syncthreads();
  if (tid == 0) {
    atomicAdd(&P.counters[CNT_SURVIVORS], sm.surv);
    atomicMax(&P.counters[CNT_MAXBITS], sm.maxbits);
  }
}

}  // namespace k2d

// ---------------------------------------------------------------------------------------------
// Host launcher
// ---------------------------------------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

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
  const size_t smem = sizeof(Smem<T>) + 128;
  auto kern = k_extract2d<T, TMA>;
  FTK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const dim3 grid((unsigned)((P.nx + TX - 1) / TX), (unsigned)((P.ny + TY - 1) / TY),
                  (unsigned)((P.tb - P.ta + P.tchunk - 1) / P.tchunk));
  if (grid.z == 0) return FTK_OK;
  kern<<<grid, NWARP * 32, smem, stream>>>(map, P);
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

int launch_extract2d(const ExtractParams& P, cudaStream_t stream) {
  const size_t esz = P.dtype == FTK_F32 ? 4 : 8;
  const bool aligned = (reinterpret_cast<uintptr_t>(P.field) % 16 == 0) && ((P.nx * esz) % 16 == 0) &&
                       P.nx < (1ll << 31) && P.ny < (1ll << 31) && P.nt_buf < (1ll << 31);
  const bool tma = aligned && get_encode() != nullptr && !P.force_generic;
  if (P.dtype == FTK_F32) return tma ? launch_t<float, true>(P, stream) : launch_t<float, false>(P, stream);
  return tma ? launch_t<double, true>(P, stream) : launch_t<double, false>(P, stream);
}

}  // namespace ftk
