/*
 * oracle/ftk_oracle.c -- TEST INFRASTRUCTURE, not product code.
 *
 * The independent CPU oracle for the FTK critical-point tracking hot path
 * (Guo et al., "FTK: A Simplicial Spacetime Meshing Framework for Robust and
 * Scalable Feature Tracking", arXiv 2011.08697; "P:<line>" = /root/reference/PAPER.md line).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library.  It shares no code, header, table or constant generator with the CUDA
 * product path (paper_2011_08697_b200/), and it includes nothing from include/.
 *
 * It is deliberately plain and slow: brute-force loops in the order of Alg. 1, left column
 * (P:350-369), generalised to n = 2, 3 spatial dimensions:
 *
 *   step 1  quantize      q = rint(f * 2^s), round-half-even            (reading R6)
 *   step 2  gradient      central differences, one-sided doubled at the spatial boundary
 *                         ("gradients based on central-differences"; reading R7)
 *   step 3  faces         every n-simplex of the Kuhn subdivision of the (n+1)-D regular grid
 *                         (P:301-345); the oracle enumerates the chains itself (nested subsets)
 *   step 4  test          0 in the interior of conv{g_0..g_n} (Bhatia criterion) decided
 *                         with Simulation of Simplicity: the n+1
 *                         barycentric numerators D_k of Eq. 2, each an n x n
 *                         determinant, must share one SoS sign.  The SoS sign is found by
 *                         enumerating every epsilon-monomial of det(M + E) (all partial
 *                         permutations) sorted by magnitude -- no unrolled table.
 *   step 5  location      mu_k = D_k / sum D (Eq. 2), x_c = sum mu_k p_k (reading R11)
 *   step 6  type          integer Hessian interpolated with mu, eigen-signs (reading R8/R9)
 *   step 7  cells         every (n+1)-simplex: T = S cap sides(cell); UF.unite(T)
 *   step 8  labels        label = minimum face_id of the component (reading R13)
 *
 * Exactness: all integer work is int64 / __int128 (ranges checked: |q| < 2^59 in 2D, < 2^38 in
 * 3D, else FTKO_RANGE).  FP64 steps use a fixed left-to-right order; this file must be compiled
 * with -ffp-contract=off (no FMA contraction) and without -ffast-math.
 *
 * Parity-pin status: Kuhn tables, counts, SoS, face test,
 * 0/2 invariant, location (closed forms), woven census and labels are pinned by tests under
 * tests/test_oracle_*.py; tests/test_bruteforce_pin.py re-derives labels, locations and the 2D and
 * 3D Hessian types (3D by Sylvester inertia of the exact rational Hessian) on tiny grids.  Hessian
 * types within a relative 1e-9 of exact degeneracy are "parity unpinned" beyond the closed-form and
 * census pins.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __int128 i128;

/* status codes (values chosen to match the C-ABI's documented meanings; defined independently) */
enum { FTKO_OK = 0, FTKO_INVALID_ARG = 1, FTKO_RANGE = 2, FTKO_CAPACITY = 3,
       FTKO_INVARIANT = 6, FTKO_NOMEM = 7 };
/* critical point types (maxima, minima, saddles of the gradient field; sources, sinks and
 * saddles of a vector field, with centres where the Jacobian's trace vanishes) */
enum { CP_DEGENERATE = 0, CP_MIN = 1, CP_SADDLE = 2, CP_SADDLE1 = 3, CP_SADDLE2 = 4, CP_MAX = 5,
       CP_SOURCE = 6, CP_SINK = 7, CP_CENTER = 8 };
/* record flags */
enum { FL_ORDINAL = 1, FL_BOUNDARY = 2, FL_DEGEN_LOC = 4 };

typedef struct {
  int32_t ndim;      /* n = 2 or 3 spatial dimensions */
  int32_t dtype;     /* 0 = float32, 1 = float64; layout [t][z][y][x], x fastest */
  int64_t n[3];      /* nx, ny, nz (nz = 1 in 2D) */
  int64_t nt;        /* planes in the buffer */
  int64_t t0;        /* global index of the buffer's first plane */
  int64_t nt_global; /* global number of timesteps */
  int32_t scale_log2;
  int32_t nthreads;  /* 0 = OpenMP default */
  int32_t kind;      /* 0 = scalar field (its gradient is tracked); 1 = vector field: n
                        components per vertex, interleaved ([t][y][x][n]), tracked as given; 2D only */
  int32_t pad_;
} ftko_desc;

typedef struct {     /* 56 bytes */
  int64_t face_id;
  int64_t label;
  double x, y, z, t;
  int32_t type;
  int32_t flags;
} ftko_cp;

/* ------------------------------------------------------------------------------------------ */
/* Kuhn subdivision tables, built by enumeration.                                   */
/* Axis bit a: bit0 = x, bit1 = y, [bit2 = z,] top bit = t.                                     */
/* A k-simplex of the subdivided d-cube is a chain v0 < v0+m1 < ... < v0+mk with nested masks   */
/* m1 ⊊ m2 ⊊ ... ⊊ mk (each listed simplex adds coordinates one step at a time).     */
/* A face (n-simplex, d = n+1) has d-1 masks.  Canonical type id = rank in the lexicographic    */
/* order of the mask tuples (reading R2: the paper leaves the numbering open).           */
/* ------------------------------------------------------------------------------------------ */
#define MAXD 4
#define MAXT 64
static int g_ntypes[MAXD + 1];
static int g_masks[MAXD + 1][MAXT][MAXD]; /* [d][type][i] = m_{i+1}, i < d-1 */
static int g_nperm[MAXD + 1];
static int g_perm[MAXD + 1][24][MAXD];    /* axis permutations = the d! cells of a cube */
static int g_perm_sign[MAXD + 1][24];
static int g_tables_built = 0;

static void enum_chains(int d, int level, int prev, int* cur) {
  int full = (1 << d) - 1;
  for (int m = 1; m <= full; m++) {
    if ((m & prev) != prev || m == prev) continue; /* strictly nested */
    cur[level] = m;
    if (level == d - 2) {
      int t = g_ntypes[d]++;
      for (int i = 0; i < d - 1; i++) g_masks[d][t][i] = cur[i];
    } else {
      enum_chains(d, level + 1, m, cur);
    }
  }
}

static void enum_perms(int d, int k, int* a) {
  if (k == d) {
    int idx = g_nperm[d]++;
    int inv = 0;
    for (int i = 0; i < d; i++) {
      g_perm[d][idx][i] = a[i];
      for (int j = i + 1; j < d; j++) inv += a[i] > a[j];
    }
    g_perm_sign[d][idx] = (inv & 1) ? -1 : 1;
    return;
  }
  for (int v = 0; v < d; v++) {
    int used = 0;
    for (int i = 0; i < k; i++) used |= a[i] == v;
    if (used) continue;
    a[k] = v;
    enum_perms(d, k + 1, a);
  }
}

/* SoS epsilon-monomials of an n x n determinant (Edelsbrunner-Muecke, cited at P:129).
 * Entry (r, j) of the row-sorted matrix is perturbed by eps_{r,j} = eps^(2^(n*r+j)) (reading R4:
 * lower (vertex, component) = larger perturbation).  Each monomial prod_{r in R} eps_{r,sigma(r)}
 * is a partial permutation sigma; its exponent is sum 2^(n*r+sigma(r)), a bit set `key`, and a
 * smaller exponent means a larger term.  The unperturbed determinant is the empty sigma (key 0). */
typedef struct { int col[3]; uint32_t key; } pperm_t;
static pperm_t g_pp[4][64];
static int g_npp[4];

static void build_pperms(int n) {
  int total = 1;
  for (int r = 0; r < n; r++) total *= n + 1;
  int cnt = 0;
  for (int code = 0; code < total; code++) {
    pperm_t p;
    int c = code, used = 0, ok = 1;
    p.key = 0;
    for (int r = 0; r < 3; r++) p.col[r] = -1;
    for (int r = 0; r < n; r++) {
      p.col[r] = c % (n + 1) - 1;
      c /= n + 1;
      if (p.col[r] >= 0) {
        if (used & (1 << p.col[r])) ok = 0;
        used |= 1 << p.col[r];
        p.key |= 1u << (n * r + p.col[r]);
      }
    }
    if (ok) g_pp[n][cnt++] = p;
  }
  /* insertion sort by key: increasing exponent = decreasing magnitude */
  for (int i = 1; i < cnt; i++) {
    pperm_t x = g_pp[n][i];
    int j = i - 1;
    while (j >= 0 && g_pp[n][j].key > x.key) { g_pp[n][j + 1] = g_pp[n][j]; j--; }
    g_pp[n][j + 1] = x;
  }
  g_npp[n] = cnt;
}

static void build_tables(void) {
  if (g_tables_built) return;
  for (int d = 2; d <= MAXD; d++) {
    int cur[MAXD];
    g_ntypes[d] = 0;
    enum_chains(d, 0, 0, cur);
    int a[MAXD];
    g_nperm[d] = 0;
    enum_perms(d, 0, a);
  }
  build_pperms(2);
  build_pperms(3);
  g_tables_built = 1;
}

/* ------------------------------------------------------------------------------------------ */
/* Exact SoS sign of det(M + E(eps)) for a row-sorted n x n integer matrix.                     */
/* Coefficient of a monomial = sum over full permutations pi extending sigma of                 */
/* sgn(pi) * prod_{r not in R} M[r][pi(r)]  (expansion of the Leibniz formula).                 */
/* ------------------------------------------------------------------------------------------ */
static i128 monomial_coef(int n, const int64_t M[3][3], const pperm_t* p) {
  i128 sum = 0;
  int d = n; /* permutations of n columns: reuse the axis-permutation table of size n */
  for (int k = 0; k < g_nperm[d]; k++) {
    const int* pi = g_perm[d][k];
    int ok = 1;
    i128 prod = 1;
    for (int r = 0; r < n && ok; r++) {
      if (p->col[r] >= 0) {
        if (pi[r] != p->col[r]) ok = 0;
      } else {
        prod *= (i128)M[r][pi[r]];
      }
    }
    if (ok) sum += g_perm_sign[d][k] > 0 ? prod : -prod;
  }
  return sum;
}

static i128 det_exact(int n, const int64_t M[3][3]) { return monomial_coef(n, M, &g_pp[n][0]); }

static int sos_sign(int n, const int64_t M[3][3]) {
  for (int i = 0; i < g_npp[n]; i++) {
    i128 c = monomial_coef(n, M, &g_pp[n][i]);
    if (c > 0) return 1;
    if (c < 0) return -1;
  }
  return 0; /* unreachable: a full permutation has coefficient +-1 */
}

/* Point-in-simplex with SoS.  G = n+1 rows (vertices in global-id order) of n
 * gradient components.  D_k = (-1)^(k+n) det(rows != k) are the numerators of mu_k in Eq. 2
 * (Cramer's rule on the (n+1)x(n+1) system with the row of ones); 0 is interior iff all D_k have
 * one (SoS) sign. */
static int punctured(int n, const int64_t G[4][3]) {
  int s0 = 0;
  for (int k = 0; k <= n; k++) {
    int64_t M[3][3];
    int r = 0;
    for (int i = 0; i <= n; i++) {
      if (i == k) continue;
      for (int j = 0; j < n; j++) M[r][j] = G[i][j];
      r++;
    }
    int s = sos_sign(n, M);
    if ((k + n) & 1) s = -s;
    if (k == 0) s0 = s;
    else if (s != s0) return 0;
  }
  return 1;
}

/* int128 -> double, correctly rounded (round-half-even) by the C conversion. */
static double cvt(i128 v) { return (double)v; }

/* ------------------------------------------------------------------------------------------ */
/* Grid helpers.  Coordinates c[0..d-1] in axis order x, y, [z,] t (t global).                  */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  const ftko_desc* D;
  int n, d, T;
  int64_t ext[MAXD];     /* grid extents, t = nt_global */
  int64_t* q;            /* quantized buffer */
  int64_t* g;            /* gradient buffer, n per vertex */
} ctx_t;

static int64_t vid(const ctx_t* C, const int64_t* c) {
  /* I = x + nx*(y + ny*(z + nz*t)) (reading R3, global t) */
  const ftko_desc* D = C->D;
  int64_t z = C->n == 3 ? c[2] : 0, t = c[C->d - 1];
  return c[0] + D->n[0] * (c[1] + D->n[1] * (z + D->n[2] * t));
}

static int64_t bidx(const ctx_t* C, const int64_t* c) {
  const ftko_desc* D = C->D;
  int64_t z = C->n == 3 ? c[2] : 0, t = c[C->d - 1] - D->t0;
  return c[0] + D->n[0] * (c[1] + D->n[1] * (z + D->n[2] * t));
}

static int in_buffer_t(const ctx_t* C, int64_t t) { return t >= C->D->t0 && t < C->D->t0 + C->D->nt; }

static int64_t qat(const ctx_t* C, const int64_t* c) { return C->q[bidx(C, c)]; }
/* vector fields: component j of the quantized vector at c */
static int64_t qcomp(const ctx_t* C, const int64_t* c, int j) { return C->q[bidx(C, c) * C->n + j]; }

/* step 1: quantize the whole buffer */
static int quantize_all(ctx_t* C, const void* field) {
  const ftko_desc* D = C->D;
  int64_t nv = D->n[0] * D->n[1] * D->n[2] * D->nt * (D->kind == 1 ? C->n : 1); /* values */
  double bound = ldexp(1.0, C->n == 2 ? 59 : 38);
  int bad = 0;
#pragma omp parallel for reduction(| : bad) schedule(static)
  for (int64_t i = 0; i < nv; i++) {
    double f = D->dtype == 0 ? (double)((const float*)field)[i] : ((const double*)field)[i];
    double v = nearbyint(ldexp(f, D->scale_log2)); /* exact scaling by a power of two, then RNE */
    if (!(fabs(v) < bound)) { bad |= 1; continue; }
    C->q[i] = (int64_t)v;
  }
  return bad ? FTKO_RANGE : FTKO_OK;
}

/* step 2: gradient, 2x the derivative (positive scale; signs and zeros unchanged) */
static void gradient_all(ctx_t* C) {
  const ftko_desc* D = C->D;
  int n = C->n;
  int64_t nz = D->n[2];
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t tt = 0; tt < D->nt; tt++)
    for (int64_t z = 0; z < nz; z++)
      for (int64_t y = 0; y < D->n[1]; y++)
        for (int64_t x = 0; x < D->n[0]; x++) {
          int64_t c[MAXD] = {x, y, 0, 0};
          if (n == 3) { c[2] = z; c[3] = D->t0 + tt; } else { c[2] = D->t0 + tt; }
          int64_t base = bidx(C, c);
          for (int a = 0; a < n; a++) {
            int64_t N = D->n[a];
            int64_t lo[MAXD], hi[MAXD];
            memcpy(lo, c, sizeof lo);
            memcpy(hi, c, sizeof hi);
            int64_t gv;
            if (c[a] == 0) { hi[a] = 1; lo[a] = 0; gv = 2 * (qat(C, hi) - qat(C, lo)); }
            else if (c[a] == N - 1) { hi[a] = N - 1; lo[a] = N - 2; gv = 2 * (qat(C, hi) - qat(C, lo)); }
            else { hi[a] = c[a] + 1; lo[a] = c[a] - 1; gv = qat(C, hi) - qat(C, lo); }
            C->g[base * n + a] = gv;
          }
        }
}

/* Hessian at a vertex (reading R8): compact integer second differences, 4x scale; the stencil
 * centre is clamped into [1, N-2] along each differentiated axis.  Order: xx, xy, [xz,] yy, [yz,] zz */
static void hessian(const ctx_t* C, const int64_t* c, int64_t* H) {
  int n = C->n;
  int k = 0;
  for (int a = 0; a < n; a++)
    for (int b = a; b < n; b++) {
      int64_t cc[MAXD];
      memcpy(cc, c, sizeof cc);
      int64_t Na = C->D->n[a], Nb = C->D->n[b];
      cc[a] = cc[a] < 1 ? 1 : (cc[a] > Na - 2 ? Na - 2 : cc[a]);
      cc[b] = cc[b] < 1 ? 1 : (cc[b] > Nb - 2 ? Nb - 2 : cc[b]);
      if (a == b) {
        int64_t p[MAXD], m[MAXD];
        memcpy(p, cc, sizeof p); memcpy(m, cc, sizeof m);
        p[a] += 1; m[a] -= 1;
        H[k++] = 4 * (qat(C, p) - 2 * qat(C, cc) + qat(C, m));
      } else {
        int64_t pp[MAXD], pm[MAXD], mp[MAXD], mm[MAXD];
        memcpy(pp, cc, sizeof pp); memcpy(pm, cc, sizeof pm);
        memcpy(mp, cc, sizeof mp); memcpy(mm, cc, sizeof mm);
        pp[a] += 1; pp[b] += 1;
        pm[a] += 1; pm[b] -= 1;
        mp[a] -= 1; mp[b] += 1;
        mm[a] -= 1; mm[b] -= 1;
        H[k++] = qat(C, pp) - qat(C, pm) - qat(C, mp) + qat(C, mm);
      }
    }
}

/* Vector fields: Jacobian at a vertex ("the (spatial) Jacobian"), the gradient rule of step
 * 2 applied to every component: J[j][a] = q_j[+a] - q_j[-a] (2x the derivative), one-sided doubled
 * at the spatial boundary.  Order J[j * n + a]: u_x, u_y, v_x, v_y. */
static void jacobian(const ctx_t* C, const int64_t* c, int64_t* J) {
  int n = C->n;
  for (int j = 0; j < n; j++)
    for (int a = 0; a < n; a++) {
      int64_t N = C->D->n[a];
      int64_t lo[MAXD], hi[MAXD];
      memcpy(lo, c, sizeof lo);
      memcpy(hi, c, sizeof hi);
      int64_t f = 1;
      if (c[a] == 0) { hi[a] = 1; lo[a] = 0; f = 2; }
      else if (c[a] == N - 1) { hi[a] = N - 1; lo[a] = N - 2; f = 2; }
      else { hi[a] = c[a] + 1; lo[a] = c[a] - 1; }
      J[j * n + a] = f * (qcomp(C, hi, j) - qcomp(C, lo, j));
    }
}

/* Vector-field type from the mu-interpolated Jacobian ("sources, sinks, and saddles"; reading
 * R17).  2D: det < 0 saddle; det > 0: trace > 0 source, trace < 0 sink, trace == 0 centre; det == 0
 * degenerate.  3D: the number of eigenvalues with positive real part from the Routh-Hurwitz array of
 * det(lambda I - J) = lambda^3 + a1 lambda^2 + a2 lambda + a3 (a1 = -tr, a2 = sum of the principal 2x2
 * minors, a3 = -det): first column 1, a1, (a1 a2 - a3) / a1, a3, counted by sign changes -- 0 sink,
 * 3 source, else saddle; det == 0 degenerate; zero pivots as below.  No tolerance. */
static int classify_vec(int n, const double* Jb) {
  if (n == 2) {
    double a = Jb[0], b = Jb[1], c = Jb[2], d = Jb[3];
    double det = a * d - b * c;
    double tr = a + d;
    if (det < 0) return CP_SADDLE;
    if (det > 0) return tr > 0 ? CP_SOURCE : (tr < 0 ? CP_SINK : CP_CENTER);
    return CP_DEGENERATE;
  }
  double a = Jb[0], b = Jb[1], c = Jb[2], d = Jb[3], e = Jb[4], f = Jb[5], g = Jb[6], h = Jb[7], k = Jb[8];
  double tr = (a + e) + k;
  double m2 = ((a * e - b * d) + (a * k - c * g)) + (e * k - f * h);
  double det = (a * (e * k - f * h) - b * (d * k - f * g)) + c * (d * h - e * g);
  if (det == 0) return CP_DEGENERATE;
  double a1 = -tr, a2 = m2, a3 = -det;
  double r3 = a1 * a2 - a3; /* third Routh entry times a1 */
  /* zero pivots: a1 == 0 (eigenvalues sum to zero, det != 0) is a saddle (Routh's epsilon rule);
   * r3 == 0 factors p = (lambda + a1)(lambda^2 + a2): an imaginary pair (a2 > 0, centre) or a
   * real pair +-sqrt(-a2) (saddle) */
  if (a1 == 0) return CP_SADDLE;
  if (r3 == 0) return a2 > 0 ? CP_CENTER : CP_SADDLE;
  int s[4] = {1, a1 > 0 ? 1 : -1, (r3 > 0) == (a1 > 0) ? 1 : -1, a3 > 0 ? 1 : -1};
  int changes = 0;
  for (int i = 1; i < 4; i++) changes += s[i] != s[i - 1];
  return changes == 0 ? CP_SINK : (changes == 3 ? CP_SOURCE : CP_SADDLE);
}

/* step 6: type from the mu-interpolated Hessian ("based on the eigensystem"; reading R9) */
static int classify(int n, const double* Hb) {
  if (n == 2) {
    double a = Hb[0], b = Hb[1], d = Hb[2];
    double det = a * d - b * b;
    if (det < 0) return CP_SADDLE;
    if (det > 0) return a > 0 ? CP_MIN : CP_MAX;
    return CP_DEGENERATE;
  } else {
    double a = Hb[0], b = Hb[1], c = Hb[2], d = Hb[3], e = Hb[4], f = Hb[5];
    double c2 = (a + d) + f;
    double c1 = ((a * d - b * b) + (a * f - c * c)) + (d * f - e * e);
    double c0 = (a * (d * f - e * e) - b * (b * f - c * e)) + c * (b * e - c * d);
    if (c0 == 0) return CP_DEGENERATE;
    /* det(lambda I - H) = lambda^3 - c2 lambda^2 + c1 lambda - c0; Descartes' rule of signs on
     * (1, -c2, c1, -c0) counts the positive eigenvalues of a real-rooted (symmetric) matrix. */
    double seq[4] = {1.0, -c2, c1, -c0};
    int changes = 0, last = 1;
    for (int i = 1; i < 4; i++) {
      if (seq[i] == 0) continue;
      int s = seq[i] > 0 ? 1 : -1;
      if (s != last) changes++;
      last = s;
    }
    switch (changes) {
      case 3: return CP_MIN;
      case 2: return CP_SADDLE1;
      case 1: return CP_SADDLE2;
      default: return CP_MAX;
    }
  }
}

/* Brute-force count of the cells (d-simplices) that contain a face (P:280 side_of): a containing
 * cell's anchor w satisfies v_last - 1 <= w <= v0, so try all w = v0 - delta, delta in {0,1}^d,
 * and every axis permutation, and test vertex-set inclusion. */
static int face_cell_count(const ctx_t* C, const int64_t verts[MAXD][MAXD]) {
  int d = C->d, count = 0;
  for (int delta = 0; delta < (1 << d); delta++) {
    int64_t w[MAXD];
    int ok = 1;
    for (int a = 0; a < d; a++) {
      w[a] = verts[0][a] - ((delta >> a) & 1);
      if (w[a] < 0 || w[a] > C->ext[a] - 2) ok = 0;
    }
    if (!ok) continue;
    for (int p = 0; p < g_nperm[d]; p++) {
      int64_t chain[MAXD + 1][MAXD];
      memcpy(chain[0], w, sizeof w);
      for (int i = 1; i <= d; i++) {
        memcpy(chain[i], chain[i - 1], sizeof w);
        chain[i][g_perm[d][p][i - 1]] += 1;
      }
      int all = 1;
      for (int i = 0; i < d && all; i++) {
        int found = 0;
        for (int j = 0; j <= d && !found; j++) found = memcmp(verts[i], chain[j], sizeof(int64_t) * d) == 0;
        all = found;
      }
      count += all;
    }
  }
  return count;
}

/* steps 3-6 for one face; returns 1 and fills rec if punctured */
static int test_face(const ctx_t* C, const int64_t* anchor, int type, ftko_cp* rec) {
  int n = C->n, d = C->d;
  int span = g_masks[d][type][d - 2];
  for (int a = 0; a < d; a++)
    if (anchor[a] + ((span >> a) & 1) > C->ext[a] - 1) return -1; /* face does not exist */
  int64_t verts[MAXD][MAXD];
  int64_t G[4][3];
  for (int i = 0; i < d; i++) {
    int m = i == 0 ? 0 : g_masks[d][type][i - 1];
    for (int a = 0; a < d; a++) verts[i][a] = anchor[a] + ((m >> a) & 1);
    int64_t b = bidx(C, verts[i]);
    for (int j = 0; j < n; j++) G[i][j] = C->g[b * n + j];
  }
  if (!punctured(n, G)) return 0;

  /* step 5: location from Eq. 2 */
  i128 Dk[4], sumD = 0;
  for (int k = 0; k <= n; k++) {
    int64_t M[3][3];
    int r = 0;
    for (int i = 0; i <= n; i++) {
      if (i == k) continue;
      for (int j = 0; j < n; j++) M[r][j] = G[i][j];
      r++;
    }
    i128 det = det_exact(n, M);
    Dk[k] = ((k + n) & 1) ? -det : det;
    sumD += Dk[k];
  }
  double mu[4];
  int flags = 0;
  if (sumD == 0) {
    for (int k = 0; k <= n; k++) mu[k] = 1.0 / (double)(n + 1);
    flags |= FL_DEGEN_LOC;
  } else {
    double s = cvt(sumD);
    for (int k = 0; k <= n; k++) mu[k] = cvt(Dk[k]) / s;
  }
  double pos[MAXD];
  for (int a = 0; a < d; a++) {
    double acc = mu[0] * (double)verts[0][a];
    for (int k = 1; k <= n; k++) acc = acc + mu[k] * (double)verts[k][a];
    pos[a] = acc;
  }
  /* step 6: type */
  const int vec = C->D->kind == 1;
  int nh = vec ? n * n : (n == 2 ? 3 : 6);
  double Hb[9];
  for (int k = 0; k <= n; k++) {
    int64_t H[9];
    if (vec) jacobian(C, verts[k], H);
    else hessian(C, verts[k], H);
    for (int e = 0; e < nh; e++) {
      double term = mu[k] * (double)H[e];
      Hb[e] = k == 0 ? term : Hb[e] + term;
    }
  }
  if (!((span >> (d - 1)) & 1)) flags |= FL_ORDINAL;
  if (face_cell_count(C, verts) < 2) flags |= FL_BOUNDARY;

  rec->face_id = vid(C, anchor) * C->T + type;
  rec->label = -1;
  rec->x = pos[0];
  rec->y = pos[1];
  rec->z = n == 3 ? pos[2] : 0.0;
  rec->t = pos[d - 1];
  rec->type = vec ? classify_vec(n, Hb) : classify(n, Hb);
  rec->flags = flags;
  return 1;
}

/* ------------------------------------------------------------------------------------------ */
typedef struct { ftko_cp* v; int64_t n, cap; } vec_t;
static int vec_push(vec_t* a, const ftko_cp* r) {
  if (a->n == a->cap) {
    int64_t nc = a->cap ? a->cap * 2 : 64;
    ftko_cp* nv = (ftko_cp*)realloc(a->v, (size_t)nc * sizeof(ftko_cp));
    if (!nv) return 0;
    a->v = nv;
    a->cap = nc;
  }
  a->v[a->n++] = *r;
  return 1;
}

static int check_desc(const ftko_desc* D) {
  if (!D || (D->ndim != 2 && D->ndim != 3) || (D->dtype != 0 && D->dtype != 1)) return 0;
  if (D->n[0] < 3 || D->n[1] < 3) return 0;
  if (D->ndim == 3 ? D->n[2] < 3 : D->n[2] != 1) return 0;
  if (D->nt < 1 || D->t0 < 0 || D->t0 + D->nt > D->nt_global) return 0;
  if (D->scale_log2 < -64 || D->scale_log2 > 64) return 0;
  if (D->kind != 0 && D->kind != 1) return 0;
  return 1;
}

static int setup(ctx_t* C, const ftko_desc* D, const void* field) {
  build_tables();
  memset(C, 0, sizeof *C);
  C->D = D;
  C->n = D->ndim;
  C->d = D->ndim + 1;
  C->T = g_ntypes[C->d];
  for (int a = 0; a < C->n; a++) C->ext[a] = D->n[a];
  C->ext[C->d - 1] = D->nt_global;
#ifdef _OPENMP
  if (D->nthreads > 0) omp_set_num_threads(D->nthreads);
#endif
  int64_t nv = D->n[0] * D->n[1] * D->n[2] * D->nt;
  if (D->kind == 1) {
    /* vector field: the quantized components ARE the tracked field (no gradient step) */
    C->q = (int64_t*)malloc((size_t)nv * C->n * sizeof(int64_t));
    if (!C->q) return FTKO_NOMEM;
    C->g = C->q;
    return quantize_all(C, field);
  }
  C->q = (int64_t*)malloc((size_t)nv * sizeof(int64_t));
  C->g = (int64_t*)malloc((size_t)nv * C->n * sizeof(int64_t));
  if (!C->q || !C->g) return FTKO_NOMEM;
  int st = quantize_all(C, field);
  if (st != FTKO_OK) return st;
  gradient_all(C);
  return FTKO_OK;
}

static void teardown(ctx_t* C) {
  if (C->g != C->q) free(C->g);
  free(C->q);
}

/* Pass 1 over anchors with global t in [ta, tb): all faces in canonical order. */
static int pass1(const ctx_t* C, int64_t ta, int64_t tb, vec_t* out, int64_t* n_faces) {
  const ftko_desc* D = C->D;
  int d = C->d;
  int64_t ntw = tb - ta;
  vec_t* per = (vec_t*)calloc((size_t)(ntw > 0 ? ntw : 1), sizeof(vec_t));
  int64_t nf = 0;
  int fail = 0;
  if (!per) return FTKO_NOMEM;
#pragma omp parallel for reduction(+ : nf) reduction(| : fail) schedule(dynamic, 1)
  for (int64_t it = 0; it < ntw; it++) {
    int64_t t = ta + it;
    for (int64_t z = 0; z < D->n[2]; z++)
      for (int64_t y = 0; y < D->n[1]; y++)
        for (int64_t x = 0; x < D->n[0]; x++) {
          int64_t anchor[MAXD] = {x, y, 0, 0};
          if (C->n == 3) { anchor[2] = z; anchor[3] = t; } else { anchor[2] = t; }
          for (int type = 0; type < C->T; type++) {
            ftko_cp rec;
            int r = test_face(C, anchor, type, &rec);
            if (r < 0) continue;
            nf++;
            if (r == 1 && !vec_push(&per[it], &rec)) fail |= 1;
          }
        }
  }
  (void)d;
  for (int64_t it = 0; it < ntw && !fail; it++)
    for (int64_t i = 0; i < per[it].n; i++)
      if (!vec_push(out, &per[it].v[i])) fail = 1;
  for (int64_t it = 0; it < ntw; it++) free(per[it].v);
  free(per);
  *n_faces = nf;
  return fail ? FTKO_NOMEM : FTKO_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Public entry points                                                                        */
/* ------------------------------------------------------------------------------------------ */

int ftko_face_types(int d, int32_t* masks_out) {
  build_tables();
  if (d < 2 || d > MAXD) return -1;
  if (masks_out)
    for (int t = 0; t < g_ntypes[d]; t++)
      for (int i = 0; i < d - 1; i++) masks_out[t * (d - 1) + i] = g_masks[d][t][i];
  return g_ntypes[d];
}

int ftko_cell_perms(int d, int32_t* perms_out) {
  build_tables();
  if (d < 2 || d > MAXD) return -1;
  if (perms_out)
    for (int p = 0; p < g_nperm[d]; p++)
      for (int i = 0; i < d; i++) perms_out[p * d + i] = g_perm[d][p][i];
  return g_nperm[d];
}

/* SoS sign of an n x n row-sorted matrix (row-major int64) */
int ftko_sos_sign(int n, const int64_t* M) {
  build_tables();
  int64_t A[3][3] = {{0}};
  for (int i = 0; i < n; i++)
    for (int j = 0; j < n; j++) A[i][j] = M[i * n + j];
  return sos_sign(n, A);
}

/* SoS epsilon-order: writes the partial permutations in order (col[r] or -1), returns count */
int ftko_sos_order(int n, int32_t* cols_out) {
  build_tables();
  for (int i = 0; i < g_npp[n]; i++)
    for (int r = 0; r < n; r++) cols_out[i * n + r] = g_pp[n][i].col[r];
  return g_npp[n];
}

/* point-in-simplex for n+1 rows of n components (row-major int64), rows in global order */
int ftko_punctured(int n, const int64_t* G) {
  build_tables();
  int64_t A[4][3] = {{0}};
  for (int i = 0; i <= n; i++)
    for (int j = 0; j < n; j++) A[i][j] = G[i * n + j];
  return punctured(n, A);
}

/* correctly-rounded int128 -> double, for pinning the conversion used in step 5 */
double ftko_cvt(int64_t hi, uint64_t lo) {
  i128 v = ((i128)hi << 64) | (i128)lo;
  return cvt(v);
}

/* Pass 1 only (extraction) over anchors with global t in [ta, tb).  Records sorted by face_id,
 * label = -1.  The buffer must hold every plane the window's faces touch. */
int ftko_extract(const ftko_desc* D, const void* field, int64_t ta, int64_t tb, ftko_cp* out,
                 int64_t capacity, int64_t* n_out, int64_t* n_faces) {
  if (!check_desc(D) || !field || !n_out) return FTKO_INVALID_ARG;
  if (ta < D->t0 || tb > D->t0 + D->nt || ta > tb) return FTKO_INVALID_ARG;
  if (tb < D->nt_global && !(tb < D->t0 + D->nt)) return FTKO_INVALID_ARG; /* needs plane tb */
  ctx_t C;
  int st = setup(&C, D, field);
  if (st != FTKO_OK) { teardown(&C); return st; }
  vec_t v = {0, 0, 0};
  int64_t nf = 0;
  st = pass1(&C, ta, tb, &v, &nf);
  if (n_faces) *n_faces = nf;
  if (st == FTKO_OK) {
    *n_out = v.n;
    if (v.n > capacity) st = FTKO_CAPACITY;
    else if (out) memcpy(out, v.v, (size_t)v.n * sizeof(ftko_cp));
  }
  free(v.v);
  teardown(&C);
  return st;
}

static int64_t uf_find(int64_t* parent, int64_t i) {
  while (parent[i] != i) { parent[i] = parent[parent[i]]; i = parent[i]; }
  return i;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : x > y;
}

/* Type id of the chain u_0..u_{d-1} (coordinates), by scanning the face-type table. */
static int chain_type(int d, int64_t u[MAXD][MAXD]) {
  int m[MAXD];
  for (int i = 1; i < d; i++) {
    m[i - 1] = 0;
    for (int a = 0; a < d; a++) m[i - 1] |= (int)(u[i][a] - u[0][a]) << a;
  }
  for (int t = 0; t < g_ntypes[d]; t++) {
    int eq = 1;
    for (int i = 0; i < d - 1; i++) eq &= g_masks[d][t][i] == m[i];
    if (eq) return t;
  }
  return -1;
}

/* Full two-pass tracking (Alg. 1 left) on the whole buffer, which must be the whole domain
 * (t0 = 0, nt = nt_global).  stats (optional, 4 entries): cells visited, cells with a punctured
 * count not in {0, 2}, components, united pairs. */
int ftko_track(const ftko_desc* D, const void* field, ftko_cp* out, int64_t capacity,
               int64_t* n_out, int64_t* n_faces, int64_t* stats) {
  if (!check_desc(D) || !field || !n_out) return FTKO_INVALID_ARG;
  if (D->t0 != 0 || D->nt != D->nt_global) return FTKO_INVALID_ARG;
  ctx_t C;
  int st = setup(&C, D, field);
  if (st != FTKO_OK) { teardown(&C); return st; }
  vec_t S = {0, 0, 0};
  int64_t nf = 0;
  st = pass1(&C, 0, D->nt_global, &S, &nf);
  if (n_faces) *n_faces = nf;
  if (st != FTKO_OK) { free(S.v); teardown(&C); return st; }

  int64_t P = S.n;
  int64_t* ids = (int64_t*)malloc((size_t)(P ? P : 1) * sizeof(int64_t));
  int64_t* parent = (int64_t*)malloc((size_t)(P ? P : 1) * sizeof(int64_t));
  for (int64_t i = 0; i < P; i++) { ids[i] = S.v[i].face_id; parent[i] = i; }

  /* pass 2: every cell (d-simplex) of the mesh */
  int d = C.d;
  int64_t ncells = 0, nbad = 0, npairs = 0;
  int64_t ntc = D->nt_global - 1;
  int64_t (*pairs)[2] = NULL;
  int64_t npairs_cap = 0;
#pragma omp parallel
  {
    int64_t (*lp)[2] = NULL;
    int64_t ln = 0, lcap = 0, lcells = 0, lbad = 0;
#pragma omp for schedule(dynamic, 1)
    for (int64_t t = 0; t < ntc; t++)
      for (int64_t z = 0; z < (C.n == 3 ? D->n[2] - 1 : 1); z++)
        for (int64_t y = 0; y < D->n[1] - 1; y++)
          for (int64_t x = 0; x < D->n[0] - 1; x++) {
            int64_t w[MAXD + 1][MAXD];
            w[0][0] = x; w[0][1] = y;
            if (C.n == 3) { w[0][2] = z; w[0][3] = t; } else { w[0][2] = t; }
            for (int p = 0; p < g_nperm[d]; p++) {
              for (int i = 1; i <= d; i++) {
                memcpy(w[i], w[i - 1], sizeof w[0]);
                w[i][g_perm[d][p][i - 1]] += 1;
              }
              lcells++;
              int64_t hit[MAXD + 1];
              int nh = 0;
              for (int j = 0; j <= d; j++) { /* sides(cell): drop vertex j */
                int64_t u[MAXD][MAXD];
                int r = 0;
                for (int i = 0; i <= d; i++) {
                  if (i == j) continue;
                  memcpy(u[r++], w[i], sizeof w[0]);
                }
                int type = chain_type(d, u);
                int64_t fid = vid(&C, u[0]) * C.T + type;
                int64_t* f = (int64_t*)bsearch(&fid, ids, (size_t)P, sizeof(int64_t), cmp_i64);
                if (f) hit[nh++] = f - ids;
              }
              if (nh != 0 && nh != 2) lbad++;
              if (nh == 2) {
                if (ln == lcap) {
                  lcap = lcap ? 2 * lcap : 256;
                  lp = (int64_t(*)[2])realloc(lp, (size_t)lcap * sizeof *lp);
                }
                lp[ln][0] = hit[0];
                lp[ln][1] = hit[1];
                ln++;
              }
            }
          }
#pragma omp critical
    {
      ncells += lcells;
      nbad += lbad;
      if (npairs + ln > npairs_cap) {
        npairs_cap = (npairs + ln) * 2 + 16;
        pairs = (int64_t(*)[2])realloc(pairs, (size_t)npairs_cap * sizeof *pairs);
      }
      memcpy(pairs + npairs, lp, (size_t)ln * sizeof *lp);
      npairs += ln;
    }
    free(lp);
  }
  /* UF.unite: hook the root with the larger face_id under the smaller one, so every
   * component's final root is its minimum face_id (records are sorted by face_id). */
  for (int64_t k = 0; k < npairs; k++) {
    int64_t a = uf_find(parent, pairs[k][0]), b = uf_find(parent, pairs[k][1]);
    if (a == b) continue;
    if (a < b) parent[b] = a; else parent[a] = b;
  }
  int64_t ncomp = 0;
  for (int64_t i = 0; i < P; i++) {
    int64_t r = uf_find(parent, i);
    S.v[i].label = ids[r];
    ncomp += r == i;
  }
  if (stats) { stats[0] = ncells; stats[1] = nbad; stats[2] = ncomp; stats[3] = npairs; }
  *n_out = P;
  if (nbad) st = FTKO_INVARIANT;
  if (P > capacity) st = st == FTKO_OK ? FTKO_CAPACITY : st;
  else if (out) memcpy(out, S.v, (size_t)P * sizeof(ftko_cp));
  free(pairs);
  free(ids);
  free(parent);
  free(S.v);
  teardown(&C);
  return st;
}

/* ------------------------------------------------------------------------------------------ */
/* Isovolume tracking (Alg. 1 right): the level set f = c of a 2D+t / 3D+t scalar     */
/* field on the same Kuhn spacetime mesh.                                                      */
/*   edge pass   every spacetime edge (1-simplex, anchor v, mask m != 0) is tested: with        */
/*               g = q - rint(c 2^s), the 1D SoS point-in-simplex test of P:640 reduces to      */
/*               "the two SoS signs differ", the SoS sign of a single value being its sign with */
/*               0 counted as positive (the +eps of the only row); location by Eq. 2 (n = 1).   */
/*   cell pass   every cell (d-simplex) of the mesh: its crossed edges (0, d or 2(d-1) of them, */
/*               P:629-633 cases I / II) are united; label = minimum edge id of the component.  */
/* Edge id = I(anchor) * (2^d - 1) + (m - 1).  Record type: 1 if g increases along the edge     */
/* (g_a < 0 <= g_b), else 0; flags: ordinal (m has no t bit).                                   */
/* ------------------------------------------------------------------------------------------ */
int ftko_iso_track(const ftko_desc* D, const void* field, double isovalue, ftko_cp* out, int64_t capacity,
                   int64_t* n_out, int64_t* n_edges, int64_t* stats) {
  if (!check_desc(D) || D->kind != 0 || !field || !n_out) return FTKO_INVALID_ARG;
  if (D->t0 != 0 || D->nt != D->nt_global) return FTKO_INVALID_ARG;
  ctx_t C;
  memset(&C, 0, sizeof C);
  C.D = D;
  C.n = D->ndim;
  C.d = D->ndim + 1;
  for (int a = 0; a < C.n; a++) C.ext[a] = D->n[a];
  C.ext[C.d - 1] = D->nt_global;
#ifdef _OPENMP
  if (D->nthreads > 0) omp_set_num_threads(D->nthreads);
#endif
  int64_t nv = D->n[0] * D->n[1] * D->n[2] * D->nt;
  C.q = (int64_t*)malloc((size_t)nv * sizeof(int64_t));
  if (!C.q) return FTKO_NOMEM;
  int st = quantize_all(&C, field);
  double cqd = nearbyint(ldexp(isovalue, D->scale_log2));
  if (st == FTKO_OK && !(fabs(cqd) < ldexp(1.0, C.n == 2 ? 59 : 38))) st = FTKO_RANGE;
  if (st != FTKO_OK) { free(C.q); return st; }
  const int64_t cq = (int64_t)cqd;
  const int d = C.d, E = (1 << d) - 1;
  vec_t S = {0, 0, 0};
  int64_t ne = 0;
  /* edge pass, anchors in id order */
  for (int64_t i = 0; i < nv; i++) {
    int64_t v[MAXD], rem = i;
    for (int a = 0; a < d; a++) {
      int64_t N = C.ext[a];
      v[a] = a < d - 1 ? rem % N : rem;
      rem = a < d - 1 ? rem / N : 0;
    }
    for (int m = 1; m <= E; m++) {
      int64_t b[MAXD];
      int ok = 1;
      for (int a = 0; a < d; a++) {
        b[a] = v[a] + ((m >> a) & 1);
        if (b[a] > C.ext[a] - 1) ok = 0;
      }
      if (!ok) continue;
      ne++;
      int64_t ga = C.q[bidx(&C, v)] - cq, gb = C.q[bidx(&C, b)] - cq;
      if ((ga >= 0) == (gb >= 0)) continue;
      i128 D0 = -(i128)gb, D1 = (i128)ga, Ssum = D0 + D1;
      double s = cvt(Ssum), mu0 = cvt(D0) / s, mu1 = cvt(D1) / s;
      double pos[MAXD];
      for (int a = 0; a < d; a++) pos[a] = mu0 * (double)v[a] + mu1 * (double)b[a];
      ftko_cp r;
      r.face_id = vid(&C, v) * E + (m - 1);
      r.label = -1;
      r.x = pos[0];
      r.y = pos[1];
      r.z = C.n == 3 ? pos[2] : 0.0;
      r.t = pos[d - 1];
      r.type = gb >= 0 ? 1 : 0;
      r.flags = ((m >> (d - 1)) & 1) ? 0 : FL_ORDINAL;
      if (!vec_push(&S, &r)) { free(S.v); free(C.q); return FTKO_NOMEM; }
    }
  }
  if (n_edges) *n_edges = ne;
  /* cell pass */
  build_tables();
  int64_t P = S.n;
  int64_t* ids = (int64_t*)malloc((size_t)(P ? P : 1) * sizeof(int64_t));
  int64_t* parent = (int64_t*)malloc((size_t)(P ? P : 1) * sizeof(int64_t));
  for (int64_t i = 0; i < P; i++) { ids[i] = S.v[i].face_id; parent[i] = i; } /* ascending already */
  int64_t ncells = 0, nbad = 0;
  int64_t ncube = 1;
  for (int a = 0; a < d; a++) ncube *= C.ext[a] - 1;
  for (int64_t i = 0; i < ncube; i++) {
    int64_t w0[MAXD], rem = i;
    for (int a = 0; a < d; a++) { w0[a] = rem % (C.ext[a] - 1); rem /= (C.ext[a] - 1); }
    for (int p = 0; p < g_nperm[d]; p++) {
      int64_t w[MAXD + 1][MAXD];
      memcpy(w[0], w0, sizeof w0);
      for (int k = 1; k <= d; k++) {
        memcpy(w[k], w[k - 1], sizeof w0);
        w[k][g_perm[d][p][k - 1]] += 1;
      }
      ncells++;
      int64_t hit[16];
      int nh = 0;
      for (int a = 0; a <= d; a++)
        for (int b = a + 1; b <= d; b++) {
          int m = 0;
          for (int x = 0; x < d; x++) m |= (int)(w[b][x] - w[a][x]) << x;
          int64_t key = vid(&C, w[a]) * E + (m - 1);
          int64_t* f = (int64_t*)bsearch(&key, ids, (size_t)P, sizeof(int64_t), cmp_i64);
          if (f) hit[nh++] = f - ids;
        }
      if (!(nh == 0 || nh == d || nh == 2 * (d - 1))) nbad++;
      for (int k = 1; k < nh; k++) {
        int64_t ra = uf_find(parent, hit[0]), rb = uf_find(parent, hit[k]);
        if (ra != rb) { if (ra < rb) parent[rb] = ra; else parent[ra] = rb; }
      }
    }
  }
  int64_t ncomp = 0;
  for (int64_t i = 0; i < P; i++) {
    int64_t r = uf_find(parent, i);
    S.v[i].label = ids[r]; /* roots are component minima: ids ascend with the index */
    ncomp += r == i;
  }
  if (stats) { stats[0] = ncells; stats[1] = nbad; stats[2] = ncomp; stats[3] = 0; }
  *n_out = P;
  st = nbad ? FTKO_INVARIANT : FTKO_OK;
  if (P > capacity) st = FTKO_CAPACITY;
  else if (out && P) memcpy(out, S.v, (size_t)P * sizeof(ftko_cp));
  free(ids); free(parent); free(S.v); free(C.q);
  return st;
}

/*
 * Isovolume mesh ("Two-pass isovolume reconstruction").
 *
 * The isovolume f = c inside one cell (an (n+1)-simplex of the spacetime mesh: a pentachoron in 3D+t,
 * a tetrahedron in 2D+t) is fixed by the signs of its n+2 vertices (g = rint(f 2^s) - rint(c 2^s),
 * g >= 0 counting as positive -- the SoS reading of P:640, as in ftko_iso_track).  With P the positive
 * and M the negative vertices (|P| + |M| = n + 2, both non-empty), the crossed edges are the |P| |M|
 * pairs (p, m), and the piece is the product polytope simplex(P) x simplex(M): case I (|P| = 1 or |M| =
 * 1) is a single n-simplex ("the single tetrahedron consisting of the four intersections");
 * case II (++--- in 3D+t) is the prism simplex_1 x simplex_2, tessellated "with the same staircase
 * triangulation" into three tetrahedra.  The staircase triangulation of simplex_a x simplex_b
 * (vertices ordered by the global vertex order, i.e. the chain order of the cell) takes one n-simplex
 * per monotone lattice path from (p_0, m_0) to (p_last, m_last): C(a + b, a) simplices, each with
 * a + b + 1 = n + 1 vertices -- crossed edges, identified by their edge ids (I(lower end) (2^(n+1) - 1)
 * + mask - 1, as the records of ftko_iso_track).
 *
 * Output: elements [n_out][n + 1] int64 edge ids, cells in id order (anchor, permutation), paths in
 * lexicographic order (an "m-step" before a "p-step"), vertices along the path.
 */
int ftko_iso_mesh(const ftko_desc* D, const void* field, double isovalue, int64_t* elems, int64_t capacity,
                  int64_t* n_out) {
  if (!check_desc(D) || D->kind != 0 || !field || !n_out) return FTKO_INVALID_ARG;
  if (D->t0 != 0 || D->nt != D->nt_global) return FTKO_INVALID_ARG;
  ctx_t C;
  memset(&C, 0, sizeof C);
  C.D = D;
  C.n = D->ndim;
  C.d = D->ndim + 1;
  for (int a = 0; a < C.n; a++) C.ext[a] = D->n[a];
  C.ext[C.d - 1] = D->nt_global;
  int64_t nv = D->n[0] * D->n[1] * D->n[2] * D->nt;
  C.q = (int64_t*)malloc((size_t)nv * sizeof(int64_t));
  if (!C.q) return FTKO_NOMEM;
  int st = quantize_all(&C, field);
  double cqd = nearbyint(ldexp(isovalue, D->scale_log2));
  if (st == FTKO_OK && !(fabs(cqd) < ldexp(1.0, C.n == 2 ? 59 : 38))) st = FTKO_RANGE;
  if (st != FTKO_OK) { free(C.q); return st; }
  const int64_t cq = (int64_t)cqd;
  const int d = C.d, E = (1 << d) - 1;
  build_tables();
  int64_t cnt = 0;
  int64_t ncube = 1;
  for (int a = 0; a < d; a++) ncube *= C.ext[a] - 1;
  for (int64_t i = 0; i < ncube; i++) {
    int64_t w0[MAXD], rem = i;
    for (int a = 0; a < d; a++) { w0[a] = rem % (C.ext[a] - 1); rem /= (C.ext[a] - 1); }
    for (int p = 0; p < g_nperm[d]; p++) {
      /* the cell's vertices in chain order */
      int64_t w[MAXD + 1][MAXD];
      memcpy(w[0], w0, sizeof w0);
      for (int k = 1; k <= d; k++) {
        memcpy(w[k], w[k - 1], sizeof w0);
        w[k][g_perm[d][p][k - 1]] += 1;
      }
      int Pv[MAXD + 1], Mv[MAXD + 1], np = 0, nm = 0;
      for (int k = 0; k <= d; k++) {
        if (C.q[bidx(&C, w[k])] - cq >= 0) Pv[np++] = k;
        else Mv[nm++] = k;
      }
      if (np == 0 || nm == 0) continue;
      /* monotone lattice paths from (0, 0) to (np - 1, nm - 1): choose which of the np + nm - 2 steps
       * advance in P, in lexicographic order of the step strings (M-step = 0 < P-step = 1) */
      const int steps = np + nm - 2;
      for (int code = 0; code < (1 << steps); code++) {
        if (__builtin_popcount((unsigned)code) != np - 1) continue;
        /* read the steps most significant first so that the codes ascend lexicographically */
        int64_t el[MAXD + 1];
        int ip = 0, im = 0, k = 0;
        for (int s = -1; s < steps; s++) {
          if (s >= 0) {
            if ((code >> (steps - 1 - s)) & 1) ip++;
            else im++;
          }
          const int a = Pv[ip] < Mv[im] ? Pv[ip] : Mv[im];
          const int b = Pv[ip] < Mv[im] ? Mv[im] : Pv[ip];
          int m = 0;
          for (int x = 0; x < d; x++) m |= (int)(w[b][x] - w[a][x]) << x;
          el[k++] = vid(&C, w[a]) * E + (m - 1);
        }
        if (elems && cnt < capacity)
          for (int x = 0; x < d; x++) elems[cnt * d + x] = el[x];
        cnt++;
      }
    }
  }
  free(C.q);
  *n_out = cnt;
  return cnt > capacity ? FTKO_CAPACITY : FTKO_OK;
}
