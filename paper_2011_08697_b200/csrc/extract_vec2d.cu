// extract_vec2d.cu -- pass 1 of Alg. 1 for a 2D time-varying VECTOR field
// (the zeros of v itself are tracked; types from the Jacobian's eigensystem).
//
// Same mesh, predicates and record/edge contract as the scalar 2D path (extract2d.cu), without the
// gradient stencil: the tracked vector of a vertex is its own quantized value, q_j = rint(v_j 2^s).
//
//   K1a k_scanvec2d -- one warp per work item (128 x 8 anchor tile x a chunk of timesteps), items
//     pulled from a global counter.  Per vertex a 4-bit "strict sign holds" code: u > thr, u < -thr,
//     v > thr, v < -thr with thr = 2^-s, which implies the exact q_u > 0 (u 2^s > 1 > 1/2, so the
//     round-half-even integer is >= 1), etc.  ANDed over the 8 corners of each spacetime cube (y-pair
//     across the warp's code rows, x-pair by one shuffle plus the codes of column x0 + 128, t-pair
//     with the previous plane's squares in registers); a zero byte is a survivor.  No stencil means
//     no halo beyond the cubes' own +1 row / column: each vertex is read from HBM once, with the
//     9th code row of a warp (1/8 of the rows) re-read from L2.  Survivors leave as group entries
//     (as in 2D): first anchor of the lane, plane flag, 32-bit survivor mask.
//   k_expand2d (extract2d.cu) -- group entries -> cube list.
//   K1b k_exactvec2d -- one thread per surviving cube: exact int64 corner vectors, the 12 face tests
//     (2x2 determinants in int128, SoS chain of DESIGN.md R4), the 6 cells (0 or 2 punctured sides,
//     PAPER.md:437) emitted as trajectory edges (both ends as records, or the neighbour cube's upper
//     face by id), Eq. 2 location and the Jacobian type (R17) of every
//     punctured face, in the same fixed-order FP64 as the oracle.
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "extract2d.cuh"
#include "kuhn.cuh"
#include "sm100.cuh"

namespace ftk {
namespace kv2 {

constexpr int LX = 128;   // anchors per tile row (32 lanes x 4 positions)
constexpr int RW = 8;     // anchor rows per work item (one warp)
constexpr int CHUNK = 32; // group entries a warp reserves at a time
constexpr uint32_t NEUTRAL = 0xF0F0F0F0u;

__constant__ KuhnTables<3> cK3 = kKuhn3;

// code byte (bits 7..4 = u > thr, u < -thr, v > thr, v < -thr) of one vertex
template <typename T>
__device__ __forceinline__ uint32_t vcode(T u, T v, T thr) {
  if constexpr (sizeof(T) == 4) {
    return ((__float_as_uint(__fsub_rn(thr, u)) >> 31) << 7) | ((__float_as_uint(__fadd_rn(u, thr)) >> 31) << 6) |
           ((__float_as_uint(__fsub_rn(thr, v)) >> 31) << 5) | ((__float_as_uint(__fadd_rn(v, thr)) >> 31) << 4);
  } else {
    auto sb = [](double a) { return (uint32_t)((unsigned long long)__double_as_longlong(a) >> 63); };
    return (sb(thr - u) << 7) | (sb(u + thr) << 6) | (sb(thr - v) << 5) | (sb(v + thr) << 4);
  }
}

template <typename T>
__device__ __forceinline__ uint32_t absbits(T a) {
  if constexpr (sizeof(T) == 4) return __float_as_uint(a) & 0x7fffffffu;
  else return 0u;
}

// The lane's 4 positions x0 + 4 lane + i of row y: code word (byte i = position i), 0xF0 outside.
template <typename T>
__device__ __forceinline__ uint32_t row_code(const T* plane, long long nx, long long ny, long long y, long long xl,
                                             T thr, bool pairs_aligned, uint32_t& maxb, double& maxd) {
  if (y >= ny) return NEUTRAL;
  const T* r = plane + 2 * (y * nx + xl);
  T u[4], v[4];
  if (xl + 3 < nx) {
    if constexpr (sizeof(T) == 4) {
      if (pairs_aligned) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(r));
        const float4 b = __ldg(reinterpret_cast<const float4*>(r + 4));
        u[0] = a.x; v[0] = a.y; u[1] = a.z; v[1] = a.w; u[2] = b.x; v[2] = b.y; u[3] = b.z; v[3] = b.w;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 p = __ldg(reinterpret_cast<const float2*>(r + 2 * i));
          u[i] = p.x;
          v[i] = p.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double2 p = __ldg(reinterpret_cast<const double2*>(r + 2 * i));
        u[i] = p.x;
        v[i] = p.y;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool in = xl + i < nx;
      u[i] = in ? __ldg(r + 2 * i) : (T)0;
      v[i] = in ? __ldg(r + 2 * i + 1) : (T)0;
    }
  }
  uint32_t c = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool in = xl + i < nx;
    c |= (in ? vcode<T>(u[i], v[i], thr) : 0xF0u) << (8 * i);
    if (in) {
      if constexpr (sizeof(T) == 4) {
        maxb = max(maxb, max(absbits(u[i]), absbits(v[i])));
      } else {
        const double a = fabs((double)u[i]), b = fabs((double)v[i]);
        if (a != a || b != b || maxd != maxd) maxd = __longlong_as_double(0x7ff8000000000000ll);
        else maxd = fmax(maxd, fmax(a, b));
      }
    }
  }
  return c;
}

#ifndef FTK_V_MINB
#define FTK_V_MINB 4  // 4 blocks of 8 warps per SM (64 registers, measured best on V2: 1.49 -> 1.06 ms)
#endif
template <typename T>
__global__ void __launch_bounds__(256, FTK_V_MINB) k_scanvec2d(const __grid_constant__ ExtractParams P) {
  const int lane = threadIdx.x & 31;
  const i64 nx = P.nx, ny = P.ny;
  const int ntx = (int)((nx + LX - 1) / LX), nty = (int)((ny + RW - 1) / RW);
  const int tch = (int)P.tchunk;
  const int ntz = (int)((P.tb - P.ta + tch - 1) / tch);
  const long long nitems = (long long)ntx * nty * ntz;
  const T thr = (T)P.thr;
  const T* F = reinterpret_cast<const T*>(P.field);
  const bool aligned = sizeof(T) == 4 && (nx % 2 == 0) && ((reinterpret_cast<uintptr_t>(F) & 15) == 0);
  const uint32_t lt_mask = (1u << lane) - 1u;
  long long cur = 0, end = 0;
  unsigned long long mysurv = 0;
  uint32_t maxb = 0;
  double maxd = 0.0;
  auto enqueue = [&](uint32_t mask, int tflag, int xl, int y0) {
    const uint32_t bal = __ballot_sync(0xffffffffu, mask != 0);
    if (bal == 0u) return;
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
    if (mask != 0u && e < P.wcap) {
      P.wx[e] = xl;
      P.wy[e] = y0;
      P.wt[e] = tflag;
      P.wz[e] = (int)mask;
    }
    mysurv += __popc(mask);
  };
  while (true) {
    long long item = 0;
    if (lane == 0) item = (long long)atomicAdd(&P.counters[CNT_WORK], 1ull);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= nitems) break;
    const int tx = (int)(item % ntx), ty = (int)((item / ntx) % nty), tz = (int)(item / ((long long)ntx * nty));
    const i64 x0 = (i64)tx * LX, y0 = (i64)ty * RW;
    const i64 ta = P.ta + (i64)tz * tch, tb = min(ta + tch, P.tb);
    const i64 plast = min(tb, P.nt_global - 1);
    const i64 xl = x0 + 4 * lane;
    uint32_t prevSq[RW];
    for (i64 p = ta; p <= plast; ++p) {
      const T* plane = F + (p - P.t0) * nx * ny * 2;
      uint32_t C[RW + 1];
#pragma unroll
      for (int r = 0; r <= RW; ++r) C[r] = row_code<T>(plane, nx, ny, y0 + r, xl, thr, aligned, maxb, maxd);
      // codes of column x0 + 128 (lane k: code row k), y-paired
      uint32_t Ye;
      {
        const int k = min(lane, RW);
        const i64 y = y0 + k, x = x0 + LX;
        uint32_t ce = 0xF0u;
        if (x < nx && y < ny) {
          const T* q = plane + 2 * (y * nx + x);
          ce = vcode<T>(__ldg(q), __ldg(q + 1), thr);
        }
        Ye = ce & __shfl_down_sync(0xffffffffu, ce, 1);
      }
      uint32_t Sq[RW];
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        const uint32_t Y = C[r] & C[r + 1];
        uint32_t nb = __shfl_down_sync(0xffffffffu, Y, 1);
        const uint32_t ne = __shfl_sync(0xffffffffu, Ye, r);
        if (lane == 31) nb = ne;
        Sq[r] = Y & ((Y >> 8) | (nb << 24));
      }
      auto survivors_of = [&](const uint32_t* K) {
        uint32_t mask = 0;
#pragma unroll
        for (int r = 0; r < RW; ++r) mask |= (((K[r] - 0x01010101u) & ~K[r] & 0x80808080u) >> (7 - r));
        return mask;
      };
      if (p > ta) {  // cubes anchored at p - 1 (planes p - 1, p)
        uint32_t K[RW];
#pragma unroll
        for (int r = 0; r < RW; ++r) K[r] = prevSq[r] & Sq[r];
        enqueue(survivors_of(K), (int)((uint32_t)(p - 1) | 0x80000000u), (int)xl, (int)y0);
      }
      if (p == P.nt_global - 1 && p < tb) enqueue(survivors_of(Sq), (int)p, (int)xl, (int)y0);  // last timestep
#pragma unroll
      for (int r = 0; r < RW; ++r) prevSq[r] = Sq[r];
    }
  }
  for (long long e = cur + lane; e < end; e += 32)
    if (e < P.wcap) P.wz[e] = 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mysurv += __shfl_xor_sync(0xffffffffu, mysurv, o);
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

// ------------------------------------------------------------------------------ K1b
template <typename T>
__device__ __forceinline__ i64 quantv(T f, double scale) { return __double2ll_rn(__dmul_rn((double)f, scale)); }

// SoS sign of | ua va ; ub vb | (rows a < b in global vertex order); R4: the leading terms
// of det(M + E) in decreasing magnitude are det, +v_b, -u_b, -v_a, then the constant -1
__device__ __forceinline__ int sos2(const i64* a, const i64* b) {
  const i128 d = (i128)a[0] * b[1] - (i128)a[1] * b[0];
  if (d != 0) return d > 0 ? 1 : -1;
  if (b[1]) return b[1] > 0 ? 1 : -1;
  if (b[0]) return b[0] > 0 ? -1 : 1;
  if (a[1]) return a[1] > 0 ? -1 : 1;
  return -1;
}

// zero inside the triangle g0 g1 g2 (chain order): s_k = (-1)^(k+2) sos(rows != k) all equal
__device__ __forceinline__ bool punctured3(const i64* g0, const i64* g1, const i64* g2) {
  const int s0 = sos2(g1, g2);
  const int s1 = -sos2(g0, g2);
  if (s0 != s1) return false;
  return sos2(g0, g1) == s0;
}

struct VCell {  // the 6 cells (axis permutations) of a cube, chain 0 < w1 < w2 < 7
  int8_t w1, w2;
  int8_t ta, tb, tc;  // own faces dropping 7, w2, w1: (w1, w2), (w1, 7), (w2, 7)
  int8_t up;          // type of the upper face (w1, w2, 7) relative to its anchor v + w1
};
struct VCells {
  VCell c[6];
};
constexpr VCells make_vcells() {
  VCells t{};
  const int ax[3] = {1, 2, 4};
  int n = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      if (i == j) continue;
      const int w1 = ax[i], w2 = w1 | ax[j];
      VCell& c = t.c[n++];
      c.w1 = (int8_t)w1;
      c.w2 = (int8_t)w2;
      c.ta = kKuhn3.type_of[w1 | w2 << 4];
      c.tb = kKuhn3.type_of[w1 | 7 << 4];
      c.tc = kKuhn3.type_of[w2 | 7 << 4];
      c.up = kKuhn3.type_of[(w2 ^ w1) | (7 ^ w1) << 4];
    }
  return t;
}
__constant__ VCells cVCells = make_vcells();

// Jacobian at vertex (x, y, t) (R17: the gradient rule of R7 applied to both components,
// one-sided doubled at the spatial boundary); order u_x, u_y, v_x, v_y
template <typename T>
__device__ void jacobian(const ExtractParams& P, i64 x, i64 y, i64 t, double scale, i64* J) {
  const T* pl = reinterpret_cast<const T*>(P.field) + (t - P.t0) * P.nx * P.ny * 2;
  auto q = [&](i64 xx, i64 yy, int j) { return quantv<T>(__ldg(pl + 2 * (yy * P.nx + xx) + j), scale); };
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    {
      i64 lo = x - 1, hi = x + 1, f = 1;
      if (x == 0) { lo = 0; hi = 1; f = 2; }
      else if (x == P.nx - 1) { lo = P.nx - 2; hi = P.nx - 1; f = 2; }
      J[2 * j] = f * (q(hi, y, j) - q(lo, y, j));
    }
    {
      i64 lo = y - 1, hi = y + 1, f = 1;
      if (y == 0) { lo = 0; hi = 1; f = 2; }
      else if (y == P.ny - 1) { lo = P.ny - 2; hi = P.ny - 1; f = 2; }
      J[2 * j + 1] = f * (q(x, hi, j) - q(x, lo, j));
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_exactvec2d(const __grid_constant__ ExtractParams P) {
  const long long ncube = min((long long)*(volatile unsigned long long*)&P.counters[CNT_CUBES], (long long)P.wcap);
  const T* F = reinterpret_cast<const T*>(P.field);
  const i64 nx = P.nx, ny = P.ny, plane = nx * ny;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ncube;
       e += (long long)gridDim.x * blockDim.x) {
    const int et = P.ct[e];
    const i64 x = P.cx[e], y = P.cy[e];
    const bool hasB = et < 0;
    const i64 t = et & 0x3fffffff;
    i64 g[8][2];
    uint32_t ex = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const i64 vx = x + (c & 1), vy = y + ((c >> 1) & 1);
      const int pl = c >> 2;
      g[c][0] = g[c][1] = 0;
      if (vx < nx && vy < ny && (pl == 0 || hasB)) {
        const T* q = F + ((t + pl - P.t0) * plane + vy * nx + vx) * 2;
        g[c][0] = quantv<T>(__ldg(q), P.scale);
        g[c][1] = quantv<T>(__ldg(q + 1), P.scale);
        ex |= 1u << c;
      }
    }
    uint32_t pmask = 0;
#pragma unroll
    for (int ty = 0; ty < 12; ++ty) {
      const int m1 = cK3.masks[ty][0], m2 = cK3.masks[ty][1];
      if (((ex >> m2) & 1u) && punctured3(g[0], g[m1], g[m2])) pmask |= 1u << ty;
    }
    const int npunct = __popc(pmask);
    unsigned long long rbase = 0;
    if (npunct) rbase = atomicAdd(&P.counters[CNT_NOUT], (unsigned long long)npunct);
    auto rec_of = [&](int ty) { return (long long)(rbase + __popc(pmask & ((1u << ty) - 1u))); };
    // cells: only full cubes have cells anchored here
    if (ex == 0xFFu) {
#pragma unroll
      for (int C = 0; C < 6; ++C) {
        const VCell cd = cVCells.c[C];
        const bool pa = (pmask >> cd.ta) & 1u, pb = (pmask >> cd.tb) & 1u, pc = (pmask >> cd.tc) & 1u;
        const bool pu = punctured3(g[cd.w1], g[cd.w2], g[7]);
        const int k = (int)pa + (int)pb + (int)pc + (int)pu;
        if (k != 0 && k != 2) atomicAdd(&P.counters[CNT_INVARIANT], 1ull);
        if (k != 2) continue;
        long long a, b;
        if (pu) {
          a = rec_of(pa ? cd.ta : (pb ? cd.tb : cd.tc));
          const i64 fx = x + (cd.w1 & 1), fy = y + ((cd.w1 >> 1) & 1), ft = t + ((cd.w1 >> 2) & 1);
          b = -1 - (((ft * ny + fy) * nx + fx) * 12 + cd.up);
        } else {
          a = rec_of(pa ? cd.ta : cd.tb);
          b = rec_of(pc ? cd.tc : cd.tb);
        }
        const unsigned long long es = atomicAdd(&P.counters[CNT_EDGES], 1ull);
        if (es < (unsigned long long)P.capacity) {
          P.edges[2 * es] = a;
          P.edges[2 * es + 1] = b;
        }
      }
    }
    // records: Eq. 2 location and Jacobian type
    uint32_t pm = pmask;
    while (pm) {
      const int ty = __ffs(pm) - 1;
      pm &= pm - 1;
      const unsigned long long slot = (unsigned long long)rec_of(ty);
      const int m[3] = {0, cK3.masks[ty][0], cK3.masks[ty][1]};
      const i64* r0 = g[m[0]];
      const i64* r1 = g[m[1]];
      const i64* r2 = g[m[2]];
      // D_k = (-1)^(k+2) det(rows != k)
      const i128 D0 = (i128)r1[0] * r2[1] - (i128)r1[1] * r2[0];
      const i128 D1 = -((i128)r0[0] * r2[1] - (i128)r0[1] * r2[0]);
      const i128 D2 = (i128)r0[0] * r1[1] - (i128)r0[1] * r1[0];
      const i128 S = D0 + D1 + D2;
      double mu[3];
      uint32_t flags = 0;
      if (S == 0) {
        mu[0] = mu[1] = mu[2] = 1.0 / 3.0;
        flags |= FTK_CP_DEGENERATE_LOC;
      } else {
        const double sd = i128_to_double_rn(S);
        mu[0] = __ddiv_rn(i128_to_double_rn(D0), sd);
        mu[1] = __ddiv_rn(i128_to_double_rn(D1), sd);
        mu[2] = __ddiv_rn(i128_to_double_rn(D2), sd);
      }
      double pos[3], Jb[4];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const i64 vx = x + (m[k] & 1), vy = y + ((m[k] >> 1) & 1), vt = t + ((m[k] >> 2) & 1);
        const double p3[3] = {(double)vx, (double)vy, (double)vt};
        i64 J[4];
        jacobian<T>(P, vx, vy, vt, P.scale, J);
#pragma unroll
        for (int a = 0; a < 3; ++a) pos[a] = k == 0 ? __dmul_rn(mu[0], p3[a]) : __dadd_rn(pos[a], __dmul_rn(mu[k], p3[a]));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double term = __dmul_rn(mu[k], __ll2double_rn(J[q]));
          Jb[q] = k == 0 ? term : __dadd_rn(Jb[q], term);
        }
      }
      const double det = __dsub_rn(__dmul_rn(Jb[0], Jb[3]), __dmul_rn(Jb[1], Jb[2]));
      const double tr = __dadd_rn(Jb[0], Jb[3]);
      const int type = det < 0 ? FTK_CP_SADDLE
                               : (det > 0 ? (tr > 0 ? FTK_CP_SOURCE : (tr < 0 ? FTK_CP_SINK : FTK_CP_CENTER))
                                          : FTK_CP_DEGENERATE);
      const int span = m[2];
      if (!(span & 4)) flags |= FTK_CP_ORDINAL;
      if (span != 7) {  // the two parent cells differ along the one missing axis
        const int c = 7 & ~span;
        const i64 vc = c == 1 ? x : (c == 2 ? y : t);
        const i64 Nc = c == 1 ? nx : (c == 2 ? ny : P.nt_global);
        if (vc == 0 || vc == Nc - 1) flags |= FTK_CP_BOUNDARY;
      }
      if (slot < (unsigned long long)P.capacity) {
        ftk_cp* r = P.out + slot;
        r->face_id = ((t * ny + y) * nx + x) * 12 + ty;
        P.fid[slot] = r->face_id;
        r->label = -1;
        r->x = pos[0];
        r->y = pos[1];
        r->z = 0.0;
        r->t = pos[2];
        r->type = type;
        r->flags = flags;
      }
    }
  }
}

template <typename T>
static int launch_t(const ExtractParams& P, cudaStream_t stream) {
  auto scan = k_scanvec2d<T>;
  const sm100::LaunchGeom lg = sm100::launch_geom(scan, 256, 0);
  if (lg.err != cudaSuccess) return set_cuda_error(lg.err, "k_scanvec2d launch geometry");
  const long long tiles = ((P.nx + LX - 1) / LX) * ((P.ny + RW - 1) / RW);
  const long long warps = (long long)lg.sms * lg.per_sm * 8;
  ExtractParams Q = P;
  Q.tchunk = 32;
  while (Q.tchunk > 4 && tiles * ((P.tb - P.ta + Q.tchunk - 1) / Q.tchunk) < 4 * warps) Q.tchunk /= 2;
  const long long items = tiles * ((P.tb - P.ta + Q.tchunk - 1) / Q.tchunk);
  if (items <= 0) return FTK_OK;
  const long long blocks = std::min<long long>((items + 7) / 8, (long long)lg.sms * lg.per_sm);
  scan<<<(unsigned)blocks, 256, 0, stream>>>(Q);
  FTK_CUDA_TRY(cudaGetLastError());
  if (P.ev_mid) FTK_CUDA_TRY(cudaEventRecord(reinterpret_cast<cudaEvent_t>(P.ev_mid), stream));
  int st = launch_expand2d(P, stream, lg.sms);
  if (st) return st;
  k_exactvec2d<T><<<(unsigned)(lg.sms * 8), 256, 0, stream>>>(P);
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

}  // namespace kv2

int launch_extract_vec2d(const ExtractParams& P, cudaStream_t stream) {
  if (P.nx >= (1ll << 31) - 256 || P.ny >= (1ll << 31) - 64 || P.nt_global >= (1ll << 30)) return FTK_ERR_INVALID_ARG;
  return P.dtype == FTK_F32 ? kv2::launch_t<float>(P, stream) : kv2::launch_t<double>(P, stream);
}

}  // namespace ftk
