// iso.cu -- isovolume tracking (Alg. 1 right) on the
// Kuhn spacetime mesh of a 2D+t / 3D+t scalar field.
//
// k_iso_scan<D> -- the sign scan: warp tasks of 32 columns x 8 rows [x one z-slice] x 32 timesteps;
//   each vertex row is loaded once per task (coalesced) and its signs g >= 0 (g = q - rint(c 2^s), q =
//   rint(f 2^s); 0 counts as positive, the +eps of the 1D SoS test) are balloted into 32-bit
//   words; a cube whose 2^D corners share one sign holds no crossed edge, cell crossing, simplex or
//   link, and is dropped with a few bitwise operations per 32 cubes; the rest (and the cubes on the
//   grid's last column / row / slice / timestep) go to a candidate list.
// k_iso_cube<D> -- one thread per candidate cube (warp-uniform loop):
//   * the 2^D corners, quantized;
//   * edge pass: the 2^D - 1 edges anchored at v (v -> v + m) whose two signs differ are crossed: one
//     record each, located by Eq. 2 with n = 1 (mu_a = -g_b / (g_a - g_b), mu_b = g_a / (g_a - g_b),
//     FP64 without FMA), id = I(v) (2^D - 1) + m - 1, type 1 if g increases along the edge, flags
//     ordinal when m has no t bit;
//   * cell pass (full cubes): the D! cells (axis permutations) of the cube; the crossed edges of each
//     (0, D or 2 (D - 1) of them -- cases I and II, else FTK_ERR_INVARIANT) are united in a
//     cube-local union-find over the cube's comparable corner pairs, and every local component is
//     emitted as trajectory-graph links (representative, member) -- an end is a record index when the
//     edge is anchored at v, else -1 - edge id (resolved by pass 2 through the hash);
//   * mesh (optional): the cells' isovolume simplices (staircase triangulation) as tuples of
//     crossed-edge ids.
// Pass 2 (track.cu: hash of every record, links, lock-free union-find, min-id labels) is shared.
#include <cstdio>

#include "common.cuh"
#include "extract2d.cuh"
#include "sm100.cuh"

namespace ftk {
namespace iso {

// comparable corner pairs (a subset of b, a != b) of the D-cube, and the slot of each
template <int D>
struct Pairs {
  static constexpr int NC = 1 << D;
  int n;
  int8_t a[81], b[81];
  int8_t slot[NC][NC];  // -1 if not comparable
};
template <int D>
constexpr Pairs<D> make_pairs() {
  Pairs<D> p{};
  p.n = 0;
  for (int a = 0; a < (1 << D); ++a)
    for (int b = 0; b < (1 << D); ++b) {
      p.slot[a][b] = -1;
      if (a != b && (a & ~b) == 0) {
        p.a[p.n] = (int8_t)a;
        p.b[p.n] = (int8_t)b;
        p.slot[a][b] = (int8_t)p.n;
        ++p.n;
      }
    }
  return p;
}
static_assert(make_pairs<3>().n == 19 && make_pairs<4>().n == 65, "comparable corner pairs");
__constant__ Pairs<3> cP3 = make_pairs<3>();
__constant__ Pairs<4> cP4 = make_pairs<4>();

template <int D>
struct Perms {
  int n;
  int8_t p[24][4];
};
template <int D>
constexpr Perms<D> make_perms() {
  Perms<D> r{};
  r.n = 0;
  int a[4] = {0, 1, 2, 3};
  // lexicographic permutations of 0..D-1
  for (int i0 = 0; i0 < D; ++i0)
    for (int i1 = 0; i1 < D; ++i1)
      for (int i2 = 0; i2 < (D > 2 ? D : 1); ++i2)
        for (int i3 = 0; i3 < (D > 3 ? D : 1); ++i3) {
          const int idx[4] = {i0, i1, i2, i3};
          bool ok = true;
          for (int x = 0; x < D; ++x)
            for (int y = x + 1; y < D; ++y)
              if (idx[x] == idx[y]) ok = false;
          if (!ok) continue;
          for (int x = 0; x < D; ++x) r.p[r.n][x] = (int8_t)a[idx[x]];
          ++r.n;
        }
  return r;
}
__constant__ Perms<3> cPm3 = make_perms<3>();
__constant__ Perms<4> cPm4 = make_perms<4>();

template <int D>
__device__ __forceinline__ const Pairs<D>& pairs() {
  if constexpr (D == 3) return cP3;
  else return cP4;
}
template <int D>
__device__ __forceinline__ const Perms<D>& perms() {
  if constexpr (D == 3) return cPm3;
  else return cPm4;
}

// The cube anchored at vertex i (one per lane, `active` lanes only; warp-uniform: the record, link and
// simplex slots are reserved with one atomic per warp): crossed edges, cells, mesh, links.
template <typename T, int D>
__device__ __forceinline__ void iso_cube(const ExtractParams& P, long long cq, const i64 (&ext)[4], int4 vc, bool active,
                                      uint32_t& maxb, double& maxd) {
  constexpr int NC = 1 << D, E = NC - 1, NP = D == 3 ? 19 : 65;
  const T* F = reinterpret_cast<const T*>(P.field);
  const int lane = threadIdx.x & 31;
  {
    // the anchor's coordinates (x, y, [z,] t)
    const i64 v[4] = {active ? vc.x : 0, active ? vc.y : 0, active ? vc.z : 0, active ? vc.w : 0};
    // corner values
    i64 g[NC];
    uint32_t exist = 0, pos = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      bool in = true;
      i64 off = 0, stride = 1;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const i64 w = v[a] + ((c >> a) & 1);
        in = in && w < ext[a];
        off += w * stride;
        stride *= ext[a];
      }
      g[c] = 0;
      if (in && active) {
        const T f = __ldg(F + off);
        if (c == 0) {
          if constexpr (sizeof(T) == 4) maxb = max(maxb, __float_as_uint(f) & 0x7fffffffu);
          else {
            const double x = fabs((double)f);
            maxd = (x != x || maxd != maxd) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(maxd, x);
          }
        }
        g[c] = __double2ll_rn(__dmul_rn((double)f, P.scale)) - cq;
        exist |= 1u << c;
        pos |= (g[c] >= 0 ? 1u : 0u) << c;
      }
    }
    const bool mixed = !(pos == 0 || pos == exist);  // one sign on every corner: nothing crosses this cube
    // edge pass: crossed edges anchored at v
    uint32_t emask = 0;
    const uint32_t s0 = pos & 1u;
    if (mixed) {
#pragma unroll
      for (int m = 1; m < NC; ++m)
        if (((exist >> m) & 1u) && (((pos >> m) & 1u) != s0)) emask |= 1u << m;
    }
    const int nrec = __popc(emask);
    auto warp_reserve = [&](int n, int ctr) -> unsigned long long {
      int incl = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      unsigned long long b0 = 0;
      if (lane == 31 && total) b0 = atomicAdd(&P.counters[ctr], (unsigned long long)total);
      b0 = __shfl_sync(0xffffffffu, b0, 31);
      return b0 + (unsigned long long)(incl - n);
    };
    const unsigned long long rbase = warp_reserve(nrec, CNT_NOUT);
    i64 vid = 0;
    {
      i64 stride = 1;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        vid += v[a] * stride;
        stride *= ext[a];
      }
    }
    auto rec_of = [&](int m) { return (long long)(rbase + __popc(emask & ((1u << m) - 1u))); };
    uint32_t em = emask;
    while (em) {
      const int m = __ffs(em) - 1;
      em &= em - 1;
      const unsigned long long slot = (unsigned long long)rec_of(m);
      const i64 ga = g[0], gb = g[m];
      const i64 D0 = -gb, D1 = ga, S = D0 + D1;
      const double sd = __ll2double_rn(S);
      const double mu0 = __ddiv_rn(__ll2double_rn(D0), sd), mu1 = __ddiv_rn(__ll2double_rn(D1), sd);
      double p[4];
#pragma unroll
      for (int a = 0; a < D; ++a)
        p[a] = __dadd_rn(__dmul_rn(mu0, (double)v[a]), __dmul_rn(mu1, (double)(v[a] + ((m >> a) & 1))));
      if (slot < (unsigned long long)P.capacity) {
        ftk_cp* r = P.out + slot;
        r->face_id = vid * E + (m - 1);
        P.fid[slot] = r->face_id;
        r->label = -1;
        r->x = p[0];
        r->y = p[1];
        r->z = D == 4 ? p[2] : 0.0;
        r->t = p[D - 1];
        r->type = gb >= 0 ? 1 : 0;
        r->flags = ((m >> (D - 1)) & 1) ? 0u : FTK_CP_ORDINAL;
      }
    }
    // cell pass (full cubes only)
    const bool cells = mixed && exist == (1u << NC) - 1u;
    const Pairs<D>& PR = pairs<D>();
    const Perms<D>& PM = perms<D>();
    int8_t up[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) up[k] = (int8_t)k;
    auto find = [&](int k) {
      while (up[k] != k) k = up[k];
      return k;
    };
    for (int pi = 0; cells && pi < PM.n; ++pi) {
      int chain[D + 1];
      chain[0] = 0;
#pragma unroll
      for (int k = 1; k <= D; ++k) chain[k] = chain[k - 1] | (1 << PM.p[pi][k - 1]);
      int first = -1, cnt = 0;
#pragma unroll
      for (int a = 0; a <= D; ++a)
#pragma unroll
        for (int b = a + 1; b <= D; ++b) {
          const int ca = chain[a], cb = chain[b];
          if (((pos >> ca) & 1u) == ((pos >> cb) & 1u)) continue;
          ++cnt;
          const int sl = PR.slot[ca][cb];
          if (first < 0) {
            first = sl;
          } else {
            const int r1 = find(first), r2 = find(sl);
            if (r1 != r2) up[max(r1, r2)] = (int8_t)min(r1, r2);
          }
        }
      if (cnt != 0 && cnt != D && cnt != 2 * (D - 1)) atomicAdd(&P.counters[CNT_INVARIANT], 1ull);
    }
    // isovolume mesh: per crossed cell, the staircase triangulation of simplex(P) x
    // simplex(M) -- P / M the cell's positive / negative chain vertices -- one D-vertex simplex per
    // monotone lattice path, its vertices the crossed edges along the path (edge ids); C(|P| + |M| - 2,
    // |P| - 1) of them: 1 in case I, 3 tetrahedra for ++--- (3D+t), 2 triangles for ++-- (2D+t)
    if (P.mesh) {
      constexpr int NB[5][5] = {{0, 0, 0, 0, 0}, {0, 1, 1, 1, 1}, {0, 1, 2, 3, 4}, {0, 1, 3, 6, 10}, {0, 1, 4, 10, 20}};
      int nel = 0;
      for (int pi = 0; cells && pi < PM.n; ++pi) {
        int np = 0, c = 0;
#pragma unroll
        for (int k = 0; k <= D; ++k) {
          if (k) c |= 1 << PM.p[pi][k - 1];
          np += (pos >> c) & 1u;
        }
        if (np > 0 && np <= D) nel += NB[np][D + 1 - np];  // C(np - 1 + nm - 1, np - 1), nm = D + 1 - np
      }
      unsigned long long el = warp_reserve(nel, CNT_ELEMS);
      for (int pi = 0; cells && pi < PM.n; ++pi) {
        int chain[D + 1], Pv[D + 1], Mv[D + 1], np = 0, nm = 0;
        chain[0] = 0;
#pragma unroll
        for (int k = 1; k <= D; ++k) chain[k] = chain[k - 1] | (1 << PM.p[pi][k - 1]);
#pragma unroll
        for (int k = 0; k <= D; ++k) {
          if ((pos >> chain[k]) & 1u) Pv[np++] = k;
          else Mv[nm++] = k;
        }
        if (np == 0 || nm == 0) continue;
        const int steps = np + nm - 2;
        for (int code = 0; code < (1 << steps); ++code) {
          if (__popc(code) != np - 1) continue;
          if (el < (unsigned long long)P.elem_cap) {
            long long* out = P.elems + el * D;
            int ip = 0, im = 0;
            for (int st = -1; st < steps; ++st) {
              if (st >= 0) {
                if ((code >> (steps - 1 - st)) & 1) ++ip;
                else ++im;
              }
              const int a = min(Pv[ip], Mv[im]), b = max(Pv[ip], Mv[im]);
              const int ca = chain[a], cb = chain[b];
              i64 id = 0, stride = 1;
#pragma unroll
              for (int x = 0; x < D; ++x) {
                id += (v[x] + ((ca >> x) & 1)) * stride;
                stride *= ext[x];
              }
              out[st + 1] = id * E + ((cb ^ ca) - 1);
            }
          }
          ++el;
        }
      }
    }
    // links: every crossed slot of a local component to the component's root slot
    auto end_of = [&](int sl) -> long long {
      const int ca = PR.a[sl], cb = PR.b[sl];
      if (ca == 0) return rec_of(cb);
      i64 id = 0, stride = 1;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        id += (v[a] + ((ca >> a) & 1)) * stride;
        stride *= ext[a];
      }
      return -1 - (id * E + ((cb ^ ca) - 1));
    };
    int nlink = 0;
    for (int k = 0; cells && k < NP; ++k) nlink += up[k] != k;
    unsigned long long es = warp_reserve(nlink, CNT_EDGES);
    for (int k = 0; cells && k < NP; ++k) {
      if (up[k] == k) continue;  // roots and untouched slots
      const int r = find(k);
      if (es < (unsigned long long)P.capacity) {
        P.edges[2 * es] = end_of(r);
        P.edges[2 * es + 1] = end_of(k);
      }
      ++es;
    }
  }
}

// sign of g = rint(f 2^s) - rint(c 2^s) >= 0 (the SoS sign of the 1D test), as iso_cube
// computes it
template <typename T>
__device__ __forceinline__ bool iso_pos(T f, double scale, float scale_f, long long cq) {
  // fp32: f 2^s is exact in fp32 as in FP64, so rint of either is the same integer
  if constexpr (sizeof(T) == 4) return __float2ll_rn(__fmul_rn(f, scale_f)) >= cq;
  else return __double2ll_rn(__dmul_rn(f, scale)) >= cq;
}

// k_iso_scan<D>: warp tasks = 32 columns x RB anchor rows [x one z-slice] x a chunk of TCI timesteps.
// Per timestep the warp loads the task's vertex rows (coalesced) and ballots their signs into one
// 32-bit word per row (plus the sign of column x0 + 32); a cube whose corners (x, x + 1 within the
// words, the row pairs, [the slice pair,] the plane pair) all share one sign holds no crossed edge, no
// cell crossing, no simplex and no link, and is skipped; the others (and every cube on the grid's last
// column, row, slice or timestep, whose corners are partly outside) are appended to the candidate list
// (the survivor-list region: anchors in wx, wy, wz, wt; one atomic per warp and 32-entry chunk) for
// k_iso_cube.  Every vertex of the grid is loaded here (range statistics).
constexpr int RB = 8, TCI = 32;
template <typename T, int D>
__global__ void __launch_bounds__(256, 3) k_iso_scan(const __grid_constant__ ExtractParams P, long long cq) {
  constexpr int NS = D == 4 ? 2 : 1;  // slices per task (z0, z0 + 1)
  const i64 nx = P.nx, ny = P.ny, nz = D == 4 ? P.nz : 1, nt = P.nt_global;
  const T* F = reinterpret_cast<const T*>(P.field);
  const float scale_f = (float)P.scale;
  uint32_t maxb = 0;
  double maxd = 0.0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const i64 ntx = (nx + 31) / 32, nty = (ny + RB - 1) / RB, ntc = (nt + TCI - 1) / TCI, ntasks = ntx * nty * nz * ntc;
  long long cur = 0, end = 0;  // the warp's current chunk of the candidate list
  for (i64 task = (i64)blockIdx.x * 8 + wid; task < ntasks; task += (i64)gridDim.x * 8) {
    const i64 tx = task % ntx, ty = (task / ntx) % nty, tz = (task / (ntx * nty)) % nz, tc = task / (ntx * nty * nz);
    const i64 x0 = tx * 32, y0 = ty * RB, z0 = tz;
    const i64 x = x0 + lane;
    // anchor timesteps [tc TCI, min(tc TCI + TCI, nt)): planes up to the chunk end, inclusive
    const i64 tlo = tc * TCI, thi = min(tlo + TCI, nt - 1);
    uint32_t Wp[NS][RB + 1], Ep[NS];  // previous plane's row sign words; Ep / Ex: bit r = column x0 + 32
    for (i64 t = tlo; t <= thi; ++t) {
      uint32_t W[NS][RB + 1], Ex[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        uint32_t eb = 0;
#pragma unroll
        for (int r = 0; r <= RB; ++r) {
          const i64 y = y0 + r, z = z0 + s;
          const bool rowin = y < ny && z < nz;
          const T* row = F + ((t * nz + z) * ny + y) * nx;
          bool p = false, pe = false;
          if (rowin && x < nx) {
            const T f = __ldg(row + x);
            if constexpr (sizeof(T) == 4) maxb = max(maxb, __float_as_uint(f) & 0x7fffffffu);
            else {
              const double a = fabs((double)f);
              maxd = (a != a || maxd != maxd) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(maxd, a);
            }
            p = iso_pos<T>(f, P.scale, scale_f, cq);
          }
          if (lane == 0 && rowin && x0 + 32 < nx) pe = iso_pos<T>(__ldg(row + x0 + 32), P.scale, scale_f, cq);
          W[s][r] = __ballot_sync(0xffffffffu, p);
          eb |= (pe ? 1u : 0u) << r;
        }
        Ex[s] = __shfl_sync(0xffffffffu, eb, 0);
      }
      // the cubes anchored at plane t - 1 (both planes), and at t itself when it is the last
      for (int pass = t > tlo ? 0 : 1; pass < (t == nt - 1 ? 2 : 1); ++pass) {
        const i64 ta = pass == 0 ? t - 1 : t;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const i64 y = y0 + r;
          uint32_t band = 0xffffffffu, bor = 0u;
          auto take = [&](uint32_t w, uint32_t e) {
            const uint32_t sh = (w >> 1) | (e << 31);
            band &= w & sh;
            bor |= w | sh;
          };
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            take(W[s][r], (Ex[s] >> r) & 1u);
            take(W[s][r + 1], (Ex[s] >> (r + 1)) & 1u);
            if (pass == 0) {
              take(Wp[s][r], (Ep[s] >> r) & 1u);
              take(Wp[s][r + 1], (Ep[s] >> (r + 1)) & 1u);
            }
          }
          // anchors in the grid; cubes with corners outside it are always candidates
          const bool anchor = x < nx && y < ny && z0 < nz;
          const bool edge = x == nx - 1 || y == ny - 1 || (D == 4 && z0 == nz - 1) || ta == nt - 1;
          const bool cand = anchor && (edge || ((bor & ~band) >> lane & 1u));
          const uint32_t m = __ballot_sync(0xffffffffu, cand);
          if (m) {
            const int n = __popc(m), rank = __popc(m & lt);
            const int avail = (int)(end - cur);
            long long e = cur + rank;
            if (n > avail) {  // the chunk runs out: the rest goes to a fresh one (n <= 32)
              long long c = 0;
              if (lane == 0) c = (long long)atomicAdd(&P.counters[CNT_WIN], 32ull);
              c = __shfl_sync(0xffffffffu, c, 0);
              if (rank >= avail) e = c + (rank - avail);
              cur = c + (n - avail);
              end = c + 32;
            } else {
              cur += n;
            }
            if (cand && e < P.wcap) {
              P.wx[e] = (int)x;
              P.wy[e] = (int)y;
              P.wz[e] = (int)z0;
              P.wt[e] = (int)ta;
            }
          }
        }
      }
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        Ep[s] = Ex[s];
#pragma unroll
        for (int r = 0; r <= RB; ++r) Wp[s][r] = W[s][r];
      }
    }
  }
  for (long long e = cur + lane; e < end; e += 32)  // the unused rest of the warp's chunk: no cube
    if (e < P.wcap) P.wt[e] = -1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    maxb = max(maxb, __shfl_xor_sync(0xffffffffu, maxb, o));
    const double od = __shfl_xor_sync(0xffffffffu, maxd, o);
    maxd = (od != od || maxd != maxd) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(maxd, od);
  }
  if (lane == 0)
    atomicMax(&P.counters[CNT_MAXBITS],
              sizeof(T) == 4 ? (unsigned long long)maxb : (unsigned long long)__double_as_longlong(maxd));
}

// k_iso_cube<D>: the candidate cubes, one per thread (warp-uniform loop: the record, link and simplex
// slots are reserved with one atomic per warp)
template <typename T, int D>
__global__ void __launch_bounds__(256) k_iso_cube(const __grid_constant__ ExtractParams P, long long cq) {
  const i64 ext[4] = {P.nx, P.ny, D == 4 ? P.nz : P.nt_global, P.nt_global};
  const long long n = min((long long)*(volatile unsigned long long*)&P.counters[CNT_WIN], (long long)P.wcap);
  uint32_t maxb = 0;
  double maxd = 0.0;
  const int lane = threadIdx.x & 31;
  for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n;
       base += (long long)gridDim.x * blockDim.x) {
    const long long e = base + lane;
    const int t = e < n ? P.wt[e] : -1;
    const bool active = t >= 0;
    int4 vc = make_int4(0, 0, 0, 0);
    if (active) vc = D == 4 ? make_int4(P.wx[e], P.wy[e], P.wz[e], t) : make_int4(P.wx[e], P.wy[e], t, 0);
    iso_cube<T, D>(P, cq, ext, vc, active, maxb, maxd);
  }
}

template <typename T>
static int launch_t(const ExtractParams& P, long long cq, int ndim, cudaStream_t stream) {
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (ndim == 2) {
    k_iso_scan<T, 3><<<sms * 8, 256, 0, stream>>>(P, cq);
    k_iso_cube<T, 3><<<sms * 8, 256, 0, stream>>>(P, cq);
  } else {
    k_iso_scan<T, 4><<<sms * 8, 256, 0, stream>>>(P, cq);
    k_iso_cube<T, 4><<<sms * 8, 256, 0, stream>>>(P, cq);
  }
  FTK_CUDA_TRY(cudaGetLastError());
  return FTK_OK;
}

}  // namespace iso

int launch_iso(const ExtractParams& P, long long cq, int ndim, cudaStream_t stream) {
  return P.dtype == FTK_F32 ? iso::launch_t<float>(P, cq, ndim, stream) : iso::launch_t<double>(P, cq, ndim, stream);
}

}  // namespace ftk
