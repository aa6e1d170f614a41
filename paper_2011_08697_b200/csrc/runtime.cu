// runtime.cu -- host side of the C-ABI (include/ftk_cp.h): validation, workspace layout, stream
// ordering of K1 (pass 1) and pass 2, error mapping, profiling events.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <unordered_map>
#include <vector>
#include <cstring>
#include <memory>
#include <new>
#include <string>

#include "common.cuh"
#include "extract2d.cuh"
#include "kuhn.cuh"
#include "sort.cuh"
#include "track.cuh"

namespace ftk {

static thread_local std::string g_last_error;
static thread_local int g_profiling = 0;
static thread_local uint32_t g_debug = 0;  // ftk_set_debug: FTK_DEBUG_* testing switches
static thread_local float g_ms[4] = {0, 0, 0, 0};
static thread_local int64_t g_stats[3] = {0, 0, 0};

int set_cuda_error(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return FTK_ERR_CUDA;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Layout {
  size_t counters, table, edges, fid, parent, cross, exportA, exportB, map, win, wx, wy, wt, wz, cx, cy, ct, total;
  u64 hcap;
  i64 wcap;
};

// survivor-list entries (2D K1a -> K1b): prefilter survivors run at about 0.45 per punctured face on
// smooth fields; more survivors than capacity -> FTK_ERR_CAPACITY + retry
static i64 window_cap(i64 capacity) { return std::max<i64>(1024, capacity); }

static Layout layout(i64 capacity, int esz = 8) {
  (void)esz;
  Layout L;
  u64 h = 1024;
  while (h < (u64)(capacity + capacity / 2)) h <<= 1;
  L.hcap = h;
  size_t off = 0;
  L.counters = off;
  off = align_up(off + CNT_N * sizeof(u64), 256);
  L.table = off;
  off = align_up(off + h * sizeof(int), 256);
  L.edges = off;
  off = align_up(off + (size_t)capacity * 2 * sizeof(long long), 256);
  L.fid = off;
  off = align_up(off + (size_t)capacity * sizeof(i64), 256);
  L.parent = off;
  off = align_up(off + (size_t)capacity * sizeof(int), 256);
  L.cross = off;  // slab stitch lists, [capacity][2] each
  off = align_up(off + (size_t)capacity * 2 * sizeof(long long), 256);
  L.exportA = off;
  off = align_up(off + (size_t)capacity * 2 * sizeof(long long), 256);
  L.exportB = off;
  off = align_up(off + (size_t)capacity * 2 * sizeof(long long), 256);
  L.map = off;  // relabel map: [2 capacity] old labels, then [2 capacity] new labels
  off = align_up(off + (size_t)capacity * 4 * sizeof(long long), 256);
  L.wcap = window_cap(capacity);
  L.win = off;
  L.wx = off;
  off = align_up(off + (size_t)L.wcap * 4, 256);
  L.wy = off;
  off = align_up(off + (size_t)L.wcap * 4, 256);
  L.wt = off;
  off = align_up(off + (size_t)L.wcap * 4, 256);
  L.wz = off;
  off = align_up(off + (size_t)L.wcap * 4, 256);
  L.cx = off;  // 2D cube list
  off = align_up(off + (size_t)L.wcap * 4, 256);
  L.cy = off;
  off = align_up(off + (size_t)L.wcap * 4, 256);
  L.ct = off;
  off = align_up(off + (size_t)L.wcap * 4, 256);
  L.total = off;
  return L;
}

// record slots, union-find parents and hash slots are int32: capacity stays below 2^31 - 1
static constexpr int64_t kMaxCapacity = (1ll << 31) - 2;

static int esz_of(const ftk_desc* d) { return d->dtype == FTK_F32 ? 4 : 8; }
static bool is_vector(const ftk_desc* d) { return (d->flags & FTK_VECTOR_FIELD) != 0; }
// bytes of one vertex's values (2 interleaved components for a vector field)
static size_t vertex_bytes(const ftk_desc* d) { return (size_t)esz_of(d) * (is_vector(d) ? d->ndim : 1); }

// Face types an edge can look up: the upper face of a cell, seen from the neighbour cube that owns
// it, is the chain (0, p2, p2|p3[, p2|p3|p4]) -- its last mask misses exactly one axis.  The other
// types are only ever reached through in-cube pairs.
template <int D>
static constexpr unsigned long long upper_types(const KuhnTables<D>& K) {
  unsigned long long m = 0;
  for (int t = 0; t < KuhnTables<D>::NT; ++t) {
    int pc = 0;
    for (int b = 0; b < D; ++b) pc += (K.masks[t][D - 2] >> b) & 1;
    if (pc == D - 1) m |= 1ull << t;
  }
  return m;
}
static_assert(__builtin_popcountll(upper_types<3>(kKuhn3)) == 6, "6 upper face types in 2D+t");
static_assert(__builtin_popcountll(upper_types<4>(kKuhn4)) == 24, "24 upper face types in 3D+t");

static int validate(const ftk_desc* d) {
  if (!d) return FTK_ERR_INVALID_ARG;
  if (d->ndim != 2 && d->ndim != 3) return FTK_ERR_INVALID_ARG;
  if (d->dtype != FTK_F32 && d->dtype != FTK_F64) return FTK_ERR_INVALID_ARG;
  if (d->n[0] < 3 || d->n[1] < 3) return FTK_ERR_INVALID_ARG;
  if (d->ndim == 3 ? d->n[2] < 3 : d->n[2] != 1) return FTK_ERR_INVALID_ARG;
  if (d->nt < 1 || d->t0 < 0 || d->t0 + d->nt > d->nt_global) return FTK_ERR_INVALID_ARG;
  if (d->scale_log2 < -64 || d->scale_log2 > 64) return FTK_ERR_INVALID_ARG;
  if ((d->flags & FTK_GHOST_PLANE) && d->nt < 2) return FTK_ERR_INVALID_ARG;
  if (d->flags & ~(FTK_GHOST_PLANE | FTK_SORTED | FTK_VECTOR_FIELD)) return FTK_ERR_INVALID_ARG;
  if (d->n[0] * d->n[1] * d->n[2] > (1ll << 40)) return FTK_ERR_INVALID_ARG;
  return FTK_OK;
}

// owned anchor timesteps [ta, tb)
static void owned_range(const ftk_desc* d, i64& ta, i64& tb) {
  ta = d->t0;
  tb = d->t0 + d->nt - ((d->flags & FTK_GHOST_PLANE) ? 1 : 0);
}

static int range_status(const ftk_desc* d, unsigned long long maxbits) {
  double m;
  if (d->dtype == FTK_F32) {
    uint32_t b = (uint32_t)maxbits;
    float f;
    memcpy(&f, &b, 4);
    m = f;
  } else {
    memcpy(&m, &maxbits, 8);
  }
  if (!std::isfinite(m)) return FTK_ERR_RANGE;
  const double q = std::nearbyint(std::ldexp(m, d->scale_log2));
  const double bound = std::ldexp(1.0, d->ndim == 2 ? 59 : 38);
  return q < bound ? FTK_OK : FTK_ERR_RANGE;
}

static thread_local float g_kms[4] = {0, 0, 0, 0};  // K1a, K1b, pass 2, stitch

struct Events {  // profiling events, created once per host thread and device, and reused
  cudaEvent_t* e = nullptr;  // 4: between K1a and K1b
  bool on = false;
  Events() {
    thread_local std::unordered_map<int, std::vector<cudaEvent_t>> pools;
    int dev = 0;
    if (g_profiling && cudaGetDevice(&dev) == cudaSuccess) {
      std::vector<cudaEvent_t>& pool = pools[dev];
      if (pool.empty()) {
        pool.resize(5);
        for (auto& x : pool) cudaEventCreate(&x);
      }
      e = pool.data();
      on = true;
    }
  }
  void rec(int i, cudaStream_t s) {
    if (on) cudaEventRecord(e[i], s);
  }
};

// Pinned host copy of the device counters (one per host thread): the end-of-call read is a true
// asynchronous D2H copy followed by one stream synchronisation (a pageable destination would stage).
static unsigned long long* pinned_counters() {
  thread_local unsigned long long* p = nullptr;
  thread_local unsigned long long fallback[CNT_N];
  if (!p && cudaHostAlloc(reinterpret_cast<void**>(&p), CNT_N * sizeof(unsigned long long), cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    p = fallback;
  }
  return p;
}

static ExtractParams extract_params(const ftk_desc* desc, const void* d_field, ftk_cp* d_out, int64_t capacity,
                                    char* ws, const Layout& L, unsigned long long* counters, bool track) {
  ExtractParams EP;
  memset(&EP, 0, sizeof EP);
  EP.field = d_field;
  EP.dtype = desc->dtype;
  EP.nx = desc->n[0];
  EP.ny = desc->n[1];
  EP.nz = desc->n[2];
  EP.nt_buf = desc->nt;
  EP.t0 = desc->t0;
  EP.nt_global = desc->nt_global;
  owned_range(desc, EP.ta, EP.tb);
  EP.tchunk = 32;
  EP.scale = std::ldexp(1.0, desc->scale_log2);
  // prefilter threshold on raw values: 2^(1-s) for the differences of the gradient stencil, 2^-s for
  // vector components (u > 2^-s => u 2^s > 1 => rint(u 2^s) >= 1)
  EP.thr = std::ldexp(1.0, (is_vector(desc) ? 0 : 1) - desc->scale_log2);
  EP.out = d_out;
  EP.capacity = capacity;
  EP.counters = counters;
  EP.edges = reinterpret_cast<long long*>(ws + L.edges);
  EP.fid = reinterpret_cast<long long*>(ws + L.fid);
  EP.parent = reinterpret_cast<int*>(ws + L.parent);
  EP.wx = reinterpret_cast<int*>(ws + L.wx);
  EP.wy = reinterpret_cast<int*>(ws + L.wy);
  EP.wt = reinterpret_cast<int*>(ws + L.wt);
  EP.wz = reinterpret_cast<int*>(ws + L.wz);
  EP.cx = reinterpret_cast<int*>(ws + L.cx);
  EP.cy = reinterpret_cast<int*>(ws + L.cy);
  EP.ct = reinterpret_cast<int*>(ws + L.ct);
  EP.wcap = L.wcap;
  EP.force_generic = (g_debug & FTK_DEBUG_FORCE_GENERIC) != 0;
  return EP;
}

static TrackParams track_params(const ftk_desc* desc, ftk_cp* d_out, int64_t capacity, char* ws, const Layout& L,
                                unsigned long long* counters) {
  TrackParams TP;
  TP.rec = d_out;
  TP.capacity = capacity;
  TP.counters = counters;
  TP.table = reinterpret_cast<int*>(ws + L.table);
  TP.table_cap = L.hcap;
  TP.edges = reinterpret_cast<const long long*>(ws + L.edges);
  TP.verify = (g_debug & FTK_DEBUG_VERIFY_LINK) != 0;
  TP.prelinked = desc->ndim == 2 && !is_vector(desc);  // the vector kernel emits all pairs as edges
  TP.lookup_types = TP.verify ? ~0ull : (desc->ndim == 2 ? upper_types<3>(kKuhn3) : upper_types<4>(kKuhn4));
  TP.fid = reinterpret_cast<i64*>(ws + L.fid);
  TP.parent = reinterpret_cast<int*>(ws + L.parent);
  // the relabel-map region is dead during pass 2 (the stitch and post-processing use it afterwards)
  TP.lab = reinterpret_cast<long long*>(ws + L.map);
  TP.root = reinterpret_cast<int*>(ws + L.map + (size_t)capacity * sizeof(long long));
  TP.uf_by_id = (g_debug & FTK_DEBUG_UF_BY_ID) != 0;
  TP.T = desc->ndim == 2 ? 12 : 60;
  TP.plane = desc->n[0] * desc->n[1] * desc->n[2];
  TP.ndim = desc->ndim;
  TP.ext[0] = desc->n[0];
  TP.ext[1] = desc->n[1];
  TP.ext[2] = desc->n[2];
  TP.ext[3] = desc->nt_global;
  TP.inv[0] = 1.0 / TP.T;
  TP.inv[1] = 1.0 / (double)desc->n[0];
  TP.inv[2] = 1.0 / (double)desc->n[1];
  TP.inv[3] = 1.0 / (double)desc->n[2];
  TP.ghost_t = (desc->flags & FTK_GHOST_PLANE) ? desc->t0 + desc->nt - 1 : -1;
  TP.first_t = desc->t0 > 0 ? desc->t0 : -1;
  TP.cross = reinterpret_cast<long long*>(ws + L.cross);
  TP.exportA = reinterpret_cast<long long*>(ws + L.exportA);
  TP.exportB = reinterpret_cast<long long*>(ws + L.exportB);
  return TP;
}

// status of a finished call from its device counters (range, capacities, the 0/2 invariant)
static int result_status(const ftk_desc* desc, const unsigned long long* host_cnt, const Layout& L, int64_t capacity,
                         int64_t* n_out) {
  int st;
  st = range_status(desc, host_cnt[CNT_MAXBITS]);
  if (st) return st;
  const unsigned long long wmax = std::max(std::max(host_cnt[CNT_WIN], host_cnt[CNT_CUBES]), host_cnt[CNT_WIN_MAX]);
  if ((i64)wmax > L.wcap) {  // survivors beyond the survivor / cube lists were not tested
    *n_out = std::max<int64_t>(*n_out, (int64_t)wmax);
    return FTK_ERR_CAPACITY;
  }
  if ((i64)host_cnt[CNT_NOUT] > capacity || (i64)host_cnt[CNT_EDGES] > capacity ||
      (i64)host_cnt[CNT_CROSS] > capacity || (i64)host_cnt[CNT_EXPORT_B] > capacity)
    return FTK_ERR_CAPACITY;
  if (host_cnt[CNT_INVARIANT]) {
    g_last_error = "cells with a punctured-face count not in {0, 2}: " + std::to_string(host_cnt[CNT_INVARIANT]);
    return FTK_ERR_INVARIANT;
  }
  return FTK_OK;
}

// CUDA graphs of the launch sequence of a call (counter reset, extraction kernels, pass 2, export),
// replayed when the same call repeats -- same descriptor, pointers, capacity, workspace and debug
// switches (the kernels' parameters, the TMA descriptor and every grid size derive from these alone) --
// so a step costs one graph launch instead of ~8 kernel launches (fixed per-step
// overheads).  Not used while profiling events are recorded (they time individual kernels) or under
// FTK_DEBUG_NO_GRAPH.
struct GraphKey {
  ftk_desc desc;
  const void* field;
  const void* out;
  const void* ws;
  int64_t capacity;
  uint32_t debug;
  int32_t track;
  int32_t dev;
  int32_t pad;
};
struct GraphEnt {
  GraphKey key;
  cudaGraphExec_t exec;
};
static std::vector<GraphEnt>& graph_cache() {
  thread_local std::vector<GraphEnt> cache;  // per host thread; the key holds the device
  return cache;
}

static int enqueue_call(const ftk_desc* desc, const void* d_field, ftk_cp* d_out, int64_t capacity, char* ws,
                        const Layout& L, unsigned long long* counters, cudaStream_t stream, bool track, Events& ev);
static int finish_call(const ftk_desc* desc, const Layout& L, int64_t capacity, int64_t* n_out,
                       unsigned long long* counters, cudaStream_t stream, Events& ev);

// the stream graphs are captured on (per host thread and device): capture needs a stream other than the
// legacy default stream, which callers (torch's default) often pass; the captured work does not run there
static cudaStream_t capture_stream(int dev) {
  thread_local std::unordered_map<int, cudaStream_t> streams;
  cudaStream_t& s = streams[dev];
  if (!s && cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    s = nullptr;
  }
  return s;
}

template <typename F>
static int launch_graphed(const GraphKey& key, cudaStream_t stream, F&& enqueue) {
  std::vector<GraphEnt>& cache = graph_cache();
  for (GraphEnt& g : cache)
    if (memcmp(&g.key, &key, sizeof key) == 0) {
      FTK_CUDA_TRY(cudaGraphLaunch(g.exec, stream));
      return FTK_OK;
    }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  FTK_CUDA_TRY(cudaStreamIsCapturing(stream, &cs));
  const cudaStream_t cap = capture_stream(key.dev);
  if (cs != cudaStreamCaptureStatusNone || !cap) return enqueue(stream);  // caller capturing: plain launches
  FTK_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  const int st = enqueue(cap);
  cudaGraph_t graph = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(cap, &graph);
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = (st == FTK_OK && ce == cudaSuccess) ? cudaGraphInstantiate(&exec, graph, 0) : ce;
  if (graph) cudaGraphDestroy(graph);
  if (st == FTK_OK && ie != cudaSuccess) {
    // the sequence could not be captured or instantiated: run it directly (nothing of it ran yet)
    cudaGetLastError();
    return enqueue(stream);
  }
  if (st) return st;
  if (cache.size() >= 8) {  // a few live configurations per thread; the oldest goes
    cudaGraphExecDestroy(cache.front().exec);
    cache.erase(cache.begin());
  }
  cache.push_back(GraphEnt{key, exec});
  FTK_CUDA_TRY(cudaGraphLaunch(exec, stream));
  return FTK_OK;
}

static int run(const ftk_desc* desc, const void* d_field, ftk_cp* d_out, int64_t capacity, int64_t* n_out,
               void* d_ws, size_t ws_bytes, cudaStream_t stream, bool track) {
  int st = validate(desc);
  if (st) return st;
  if (!d_field || !n_out || !d_ws || capacity < 0 || capacity > kMaxCapacity || (capacity > 0 && !d_out))
    return FTK_ERR_INVALID_ARG;
  const Layout L = layout(capacity, esz_of(desc));
  if (ws_bytes < L.total) return FTK_ERR_INVALID_ARG;
  char* ws = static_cast<char*>(d_ws);
  auto* counters = reinterpret_cast<unsigned long long*>(ws + L.counters);
  Events ev;
  if (!ev.on && !(g_debug & FTK_DEBUG_NO_GRAPH)) {
    GraphKey key;
    memset(&key, 0, sizeof key);
    key.desc = *desc;
    key.field = d_field;
    key.out = d_out;
    key.ws = d_ws;
    key.capacity = capacity;
    key.debug = g_debug;
    key.track = track;
    FTK_CUDA_TRY(cudaGetDevice(&key.dev));
    st = launch_graphed(key, stream, [&](cudaStream_t sq) {
      return enqueue_call(desc, d_field, d_out, capacity, ws, L, counters, sq, track, ev);
    });
  } else {
    st = enqueue_call(desc, d_field, d_out, capacity, ws, L, counters, stream, track, ev);
  }
  if (st) return st;
  return finish_call(desc, L, capacity, n_out, counters, stream, ev);
}

static int enqueue_call(const ftk_desc* desc, const void* d_field, ftk_cp* d_out, int64_t capacity, char* ws,
                        const Layout& L, unsigned long long* counters, cudaStream_t stream, bool track, Events& ev) {
  int st;
  ev.rec(0, stream);
  FTK_CUDA_TRY(cudaMemsetAsync(counters, 0, CNT_N * sizeof(u64), stream));

  ExtractParams EP = extract_params(desc, d_field, d_out, capacity, ws, L, counters, track);
  EP.ev_mid = ev.on ? (void*)ev.e[4] : nullptr;
  if (ev.on) cudaEventRecord(ev.e[4], stream);  // a recorded default for paths that skip K1a
  ev.rec(1, stream);
  st = is_vector(desc) ? (desc->ndim == 2 ? launch_extract_vec2d(EP, stream) : launch_extract_vec3d(EP, stream))
                       : (desc->ndim == 2 ? launch_extract2d(EP, stream) : launch_extract3d(EP, stream));
  if (st) return st;
  ev.rec(2, stream);
  if (track) {
    TrackParams TP = track_params(desc, d_out, capacity, ws, L, counters);
    const i64 ext[4] = {desc->n[0], desc->n[1], desc->n[2], desc->nt_global};
    st = launch_track(TP, desc->ndim, ext, stream);
    if (st) return st;
    if (TP.ghost_t >= 0 || TP.first_t >= 0) {
      st = launch_export(TP, stream);
      if (st) return st;
    }
  }
  ev.rec(3, stream);
  return FTK_OK;
}

static int finish_call(const ftk_desc* desc, const Layout& L, int64_t capacity, int64_t* n_out,
                       unsigned long long* counters, cudaStream_t stream, Events& ev) {
  unsigned long long* host_cnt = pinned_counters();
  FTK_CUDA_TRY(cudaMemcpyAsync(host_cnt, counters, CNT_N * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
  FTK_CUDA_TRY(cudaStreamSynchronize(stream));
  *n_out = (int64_t)host_cnt[CNT_NOUT];
  if (ev.on) {
    cudaEventElapsedTime(&g_ms[0], ev.e[1], ev.e[2]);
    cudaEventElapsedTime(&g_ms[1], ev.e[2], ev.e[3]);
    g_ms[2] = 0.f;
    cudaEventElapsedTime(&g_ms[3], ev.e[0], ev.e[3]);
    if (cudaEventQuery(ev.e[4]) == cudaSuccess) {
      cudaEventElapsedTime(&g_kms[0], ev.e[1], ev.e[4]);
      cudaEventElapsedTime(&g_kms[1], ev.e[4], ev.e[2]);
    } else {
      g_kms[0] = g_ms[0];
      g_kms[1] = 0.f;
    }
    g_kms[2] = g_ms[1];
    g_kms[3] = 0.f;
  }
  ftk_num_faces(desc, &g_stats[0]);
  g_stats[1] = (int64_t)host_cnt[CNT_SURVIVORS];
  g_stats[2] = (int64_t)host_cnt[CNT_NOUT];
  return result_status(desc, host_cnt, L, capacity, n_out);
}


// ------------------------------------------------------------------------------ slab stitch
// Host resolver: A = (face id F owned by another slab, label of its partner), B = (face id F, label of F
// on its owner slab), gathered from every slab.  Every A pair joins its label with the owner's label
// of F; labels are face ids, so the union keeps the minimum = the min face id of the global component.
static int stitch_resolve(const long long* A, i64 nA, const long long* B, i64 nB, const long long* mine, i64 nmine,
                          long long* map_old, long long* map_new, i64* nmap) {
  std::unordered_map<long long, long long> owner;
  owner.reserve((size_t)nB * 2 + 16);
  for (i64 i = 0; i < nB; ++i) owner[B[2 * i]] = B[2 * i + 1];
  std::unordered_map<long long, long long> parent;
  parent.reserve((size_t)(nA + nB) * 2 + 16);
  auto find = [&](long long x) {
    auto it = parent.find(x);
    if (it == parent.end()) return x;
    long long r = x;
    while (true) {
      auto jt = parent.find(r);
      if (jt == parent.end() || jt->second == r) break;
      r = jt->second;
    }
    while (x != r) {  // path compression
      long long& px = parent[x];
      const long long nx = px;
      px = r;
      x = nx;
    }
    return r;
  };
  int bad = 0;
  for (i64 i = 0; i < nA; ++i) {
    auto it = owner.find(A[2 * i]);
    if (it == owner.end()) {
      ++bad;
      continue;
    }
    const long long a = find(A[2 * i + 1]), b = find(it->second);
    if (a == b) continue;
    if (a < b) parent[b] = a; else parent[a] = b;
  }
  std::vector<std::pair<long long, long long>> m;
  m.reserve((size_t)nmine);
  for (i64 i = 0; i < nmine; ++i) {
    const long long r = find(mine[i]);
    if (r != mine[i]) m.emplace_back(mine[i], r);
  }
  std::sort(m.begin(), m.end());
  m.erase(std::unique(m.begin(), m.end()), m.end());
  for (size_t i = 0; i < m.size(); ++i) {
    map_old[i] = m[i].first;
    map_new[i] = m[i].second;
  }
  *nmap = (i64)m.size();
  if (bad) {
    g_last_error = "slab stitch: " + std::to_string(bad) + " cross faces without an owner record";
    return FTK_ERR_INVARIANT;
  }
  return FTK_OK;
}

static int read_exports(const ftk_desc* desc, void* d_ws, int64_t capacity, std::vector<long long>& A,
                        std::vector<long long>& B, cudaStream_t s) {
  const Layout L = layout(capacity);
  char* ws = static_cast<char*>(d_ws);
  unsigned long long cnt[CNT_N];
  FTK_CUDA_TRY(cudaMemcpyAsync(cnt, ws + L.counters, sizeof cnt, cudaMemcpyDeviceToHost, s));
  FTK_CUDA_TRY(cudaStreamSynchronize(s));
  const i64 nA = (i64)cnt[CNT_CROSS], nB = (i64)cnt[CNT_EXPORT_B];
  if (nA > capacity || nB > capacity) return FTK_ERR_CAPACITY;
  A.resize((size_t)nA * 2);
  B.resize((size_t)nB * 2);
  if (nA) FTK_CUDA_TRY(cudaMemcpyAsync(A.data(), ws + L.exportA, A.size() * 8, cudaMemcpyDeviceToHost, s));
  if (nB) FTK_CUDA_TRY(cudaMemcpyAsync(B.data(), ws + L.exportB, B.size() * 8, cudaMemcpyDeviceToHost, s));
  FTK_CUDA_TRY(cudaStreamSynchronize(s));
  (void)desc;
  return FTK_OK;
}

static int apply_map(ftk_cp* d_out, i64 n, void* d_ws, int64_t capacity, const long long* map_old,
                     const long long* map_new, i64 nmap, cudaStream_t s) {
  if (nmap <= 0) return FTK_OK;
  if (nmap > 2 * capacity) return FTK_ERR_CAPACITY;
  const Layout L = layout(capacity);
  char* ws = static_cast<char*>(d_ws);
  long long* d_old = reinterpret_cast<long long*>(ws + L.map);
  long long* d_new = d_old + 2 * capacity;
  FTK_CUDA_TRY(cudaMemcpyAsync(d_old, map_old, (size_t)nmap * 8, cudaMemcpyHostToDevice, s));
  FTK_CUDA_TRY(cudaMemcpyAsync(d_new, map_new, (size_t)nmap * 8, cudaMemcpyHostToDevice, s));
  int st = launch_relabel(d_out, n, d_old, d_new, nmap, s);
  if (st) return st;
  FTK_CUDA_TRY(cudaStreamSynchronize(s));
  return FTK_OK;
}

// ---- NCCL, loaded at ftk_comm_init (torch's libnccl.so.2 when torch is already loaded)
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool load() {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      g_last_error = std::string("dlopen libnccl.so.2: ") + dlerror();
      return false;
    }
    getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    allGather = (decltype(allGather))dlsym(h, "ncclAllGather");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    getErrorString = (decltype(getErrorString))dlsym(h, "ncclGetErrorString");
    return getUniqueId && commInitRank && allGather && commDestroy && getErrorString;
  }
};
static NcclApi g_nccl;

// seam pairs per list the communicator's blocks hold from ftk_comm_init on (a seam plane carries
// about one ordinal face per critical point: ~4.2e4 on C4); larger lists take the host path once,
// which grows the blocks (or call ftk_comm_reserve)
static constexpr long long kDefaultSeamPairs = 1ll << 17;

}  // namespace ftk

struct ftk_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
  long long* d_send = nullptr;  // host-path exchange buffers (list overflow only), grown on demand
  long long* d_recv = nullptr;
  size_t cap_pairs = 0;
  long long seam_cap = 0;       // pairs per list of a packed seam block
  long long* d_gather = nullptr;  // world packed seam blocks (in-place allgather)
  char* d_scratch = nullptr;    // device resolve tables (SeamScratch), sized for world * seam_cap
  size_t scratch_bytes = 0;
};

namespace ftk {

static int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return FTK_OK;
  g_last_error = std::string(what) + ": " + (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "nccl error");
  return FTK_ERR_NCCL;
}

// ------------------------------------------------------------------ device seam path
// resolve tables for world * cap pairs per list, carved from `base` (bytes: seam_scratch_bytes)
static size_t seam_scratch_bytes(int world, long long cap) {
  const u64 hb = hash_slots(2 * (long long)world * cap, 1ull << 40);
  const u64 hl = hash_slots(4 * (long long)world * cap, 1ull << 40);
  return hb * 16 + hl * 12 + 64;
}
static void seam_scratch_carve(char* base, int world, long long cap, SeamScratch& S) {
  const u64 hb = hash_slots(2 * (long long)world * cap, 1ull << 40);
  const u64 hl = hash_slots(4 * (long long)world * cap, 1ull << 40);
  S.hb_key = reinterpret_cast<long long*>(base);
  S.hb_val = S.hb_key + hb;
  S.hb_mask = hb - 1;
  S.hl_key = S.hb_val + hb;
  S.hl_mask = hl - 1;
  S.flags = reinterpret_cast<unsigned long long*>(S.hl_key + hl);
  S.hl_parent = reinterpret_cast<int*>(S.flags + 4);
}

// scratch of the stand-alone ftk_seam_resolve (virtual slabs): library-owned per host thread and
// device, grown on demand
static int seam_scratch(int world, long long cap, SeamScratch& S) {
  struct Buf {
    char* base = nullptr;
    size_t bytes = 0;
  };
  thread_local std::unordered_map<int, Buf> bufs;
  int dev = 0;
  FTK_CUDA_TRY(cudaGetDevice(&dev));
  Buf& b = bufs[dev];
  const size_t need = seam_scratch_bytes(world, cap);
  if (need > b.bytes) {
    if (b.base) cudaFree(b.base);
    b.base = nullptr;
    b.bytes = 0;
    FTK_CUDA_TRY(cudaMalloc(&b.base, need));
    b.bytes = need;
  }
  seam_scratch_carve(b.base, world, cap, S);
  return FTK_OK;
}

static int seam_pack(void* d_ws, int64_t capacity, long long* block, long long cap, cudaStream_t s) {
  const Layout L = layout(capacity);
  char* ws = static_cast<char*>(d_ws);
  TrackParams TP;
  memset(&TP, 0, sizeof TP);
  TP.counters = reinterpret_cast<unsigned long long*>(ws + L.counters);
  TP.exportA = reinterpret_cast<long long*>(ws + L.exportA);
  TP.exportB = reinterpret_cast<long long*>(ws + L.exportB);
  TP.capacity = capacity;
  return launch_seam_pack(TP, block, cap, s);
}

// resolve all packed blocks on the device and relabel d_out; fl = the resolve's flags (overflow,
// unmatched A faces, failed-slab code)
static int seam_resolve_flags(const long long* all, int world, long long cap, const SeamScratch& S, ftk_cp* d_out,
                              i64 n, cudaStream_t s, unsigned long long (&fl)[3]) {
  int st = launch_seam_resolve(all, world, cap, S, d_out, n, s);
  if (st) return st;
  FTK_CUDA_TRY(cudaMemcpyAsync(fl, S.flags, sizeof fl, cudaMemcpyDeviceToHost, s));
  FTK_CUDA_TRY(cudaStreamSynchronize(s));
  return FTK_OK;
}

// FTK_ERR_CAPACITY when a list did not fit its block (nothing relabelled), FTK_ERR_INVARIANT for an A
// face no slab exported
static int seam_resolve(const long long* all, int world, long long cap, ftk_cp* d_out, i64 n, cudaStream_t s) {
  SeamScratch S;
  int st = seam_scratch(world, cap, S);
  if (st) return st;
  unsigned long long fl[3];
  st = seam_resolve_flags(all, world, cap, S, d_out, n, s, fl);
  if (st) return st;
  if (fl[0]) return FTK_ERR_CAPACITY;
  if (fl[1]) {
    g_last_error = "seam faces without a partner slab: " + std::to_string(fl[1]);
    return FTK_ERR_INVARIANT;
  }
  return FTK_OK;
}

// size the communicator's seam buffers for `cap` pairs per list (outside the hot path)
static int comm_reserve(ftk_comm* c, long long cap) {
  const size_t gather = (size_t)seam_stride(cap) * c->world;
  const size_t scratch = seam_scratch_bytes(c->world, cap);
  cudaFree(c->d_gather);
  cudaFree(c->d_scratch);
  c->d_gather = nullptr;
  c->d_scratch = nullptr;
  c->seam_cap = 0;
  FTK_CUDA_TRY(cudaMalloc(&c->d_gather, gather * sizeof(long long)));
  FTK_CUDA_TRY(cudaMalloc(&c->d_scratch, scratch));
  c->scratch_bytes = scratch;
  c->seam_cap = cap;
  return FTK_OK;
}

// status code a failed slab publishes in its block header (as -code): every other error outranks a
// capacity shortfall, so all ranks agree on one status and either all retry or all give up
static long long fail_code(int st) { return st == FTK_ERR_CAPACITY ? st : st + 16; }
static int code_status(unsigned long long code) { return code >= 16 ? (int)code - 16 : (int)code; }

// Device path: pack this slab's lists (or, if its track failed, the failure code) into its block of
// the pre-sized gather buffer, one in-place NCCL allgather of the fixed-size blocks, resolve and
// relabel on the device -- no allocation and no host round trip except the final flag read.
// Returns the agreed status; *overflow when some slab's list outgrew the blocks.
static int stitch_device(ftk_comm* c, int local_st, ftk_cp* d_out, i64 n, void* d_ws, int64_t capacity,
                         cudaStream_t s, bool* overflow) {
  *overflow = false;
  const long long stride = seam_stride(c->seam_cap);
  long long* mine = c->d_gather + (size_t)c->rank * stride;
  int st;
  if (local_st) {
    const long long hdr[2] = {-fail_code(local_st), 0};
    FTK_CUDA_TRY(cudaMemcpyAsync(mine, hdr, sizeof hdr, cudaMemcpyHostToDevice, s));
  } else {
    st = seam_pack(d_ws, capacity, mine, c->seam_cap, s);
    if (st) return st;
  }
  st = nccl_check(g_nccl.allGather(mine, c->d_gather, (size_t)stride, ncclInt64, c->comm, s), "ncclAllGather(seams)");
  if (st) return st;
  SeamScratch S;
  seam_scratch_carve(c->d_scratch, c->world, c->seam_cap, S);
  unsigned long long fl[3];
  st = seam_resolve_flags(c->d_gather, c->world, c->seam_cap, S, d_out, local_st ? 0 : n, s, fl);
  if (st) return st;
  if (fl[2]) {
    if (local_st) return local_st;
    g_last_error = "the track of another time slab failed";
    return code_status(fl[2]);
  }
  if (fl[0]) {
    *overflow = true;
    return FTK_OK;
  }
  if (fl[1]) {
    g_last_error = "seam faces without a partner slab: " + std::to_string(fl[1]);
    return FTK_ERR_INVARIANT;
  }
  return FTK_OK;
}

// Exchange this slab's A and B lists with every slab over NVLink, resolve, relabel.  Every rank
// calls this after its local track, failed or not (local_st), so the collectives always match: the
// device path carries the failure codes and all ranks return the same status.  Only when some list
// outgrew the pre-sized blocks (every rank sees it) do all ranks take the host path, which also
// re-sizes the blocks for the next calls.
static int stitch_nccl(ftk_comm* c, int local_st, const ftk_desc* desc, ftk_cp* d_out, i64 n, void* d_ws,
                       int64_t capacity, cudaStream_t s) {
  // testing (FTK_DEBUG_STITCH_HOST): the device exchange only agrees on the status, then the host path
  const bool force_host = (g_debug & FTK_DEBUG_STITCH_HOST) != 0;
  bool overflow = false;
  {
    const int st = stitch_device(c, local_st, d_out, force_host ? 0 : n, d_ws, capacity, s, &overflow);
    if (st || (!overflow && !force_host)) return st;
  }
  std::vector<long long> A, B;
  int st = read_exports(desc, d_ws, capacity, A, B, s);
  if (st) return st;
  const long long nA = (long long)A.size() / 2, nB = (long long)B.size() / 2;
  // counts
  if (c->cap_pairs < 1) {
    c->cap_pairs = 1024;
    FTK_CUDA_TRY(cudaMalloc(&c->d_send, c->cap_pairs * 2 * 8));
    FTK_CUDA_TRY(cudaMalloc(&c->d_recv, c->cap_pairs * 2 * 8 * c->world));
  }
  long long mycnt[2] = {nA, nB};
  FTK_CUDA_TRY(cudaMemcpyAsync(c->d_send, mycnt, 16, cudaMemcpyHostToDevice, s));
  st = nccl_check(g_nccl.allGather(c->d_send, c->d_recv, 2, ncclInt64, c->comm, s), "ncclAllGather(counts)");
  if (st) return st;
  std::vector<long long> counts((size_t)c->world * 2);
  FTK_CUDA_TRY(cudaMemcpyAsync(counts.data(), c->d_recv, counts.size() * 8, cudaMemcpyDeviceToHost, s));
  FTK_CUDA_TRY(cudaStreamSynchronize(s));
  long long maxA = 0, maxB = 0;
  for (int r = 0; r < c->world; ++r) {
    maxA = std::max(maxA, counts[2 * r]);
    maxB = std::max(maxB, counts[2 * r + 1]);
  }
  // every rank sees the same counts: size the device path's blocks for the next calls
  const long long want = ((std::max(maxA, maxB) * 3 / 2 + 1024) + 4095) / 4096 * 4096;
  if (want > c->seam_cap) {
    st = comm_reserve(c, want);
    if (st) return st;
  }
  const size_t per = (size_t)(maxA + maxB);  // pairs per rank, padded
  if (per > c->cap_pairs) {
    cudaFree(c->d_send);
    cudaFree(c->d_recv);
    c->cap_pairs = per * 2;
    FTK_CUDA_TRY(cudaMalloc(&c->d_send, c->cap_pairs * 2 * 8));
    FTK_CUDA_TRY(cudaMalloc(&c->d_recv, c->cap_pairs * 2 * 8 * c->world));
  }
  std::vector<long long> sendbuf(per * 2, -1);
  std::copy(A.begin(), A.end(), sendbuf.begin());
  std::copy(B.begin(), B.end(), sendbuf.begin() + (size_t)maxA * 2);
  if (per) {
    FTK_CUDA_TRY(cudaMemcpyAsync(c->d_send, sendbuf.data(), per * 16, cudaMemcpyHostToDevice, s));
    st = nccl_check(g_nccl.allGather(c->d_send, c->d_recv, per * 2, ncclInt64, c->comm, s), "ncclAllGather(pairs)");
    if (st) return st;
  }
  std::vector<long long> all(per * 2 * c->world);
  if (per) FTK_CUDA_TRY(cudaMemcpyAsync(all.data(), c->d_recv, all.size() * 8, cudaMemcpyDeviceToHost, s));
  FTK_CUDA_TRY(cudaStreamSynchronize(s));
  std::vector<long long> GA, GB;
  for (int r = 0; r < c->world; ++r) {
    const long long* base = all.data() + (size_t)r * per * 2;
    GA.insert(GA.end(), base, base + counts[2 * r] * 2);
    GB.insert(GB.end(), base + maxA * 2, base + maxA * 2 + counts[2 * r + 1] * 2);
  }
  std::vector<long long> mine;
  for (long long i = 0; i < nA; ++i) mine.push_back(A[2 * i + 1]);
  for (long long i = 0; i < nB; ++i) mine.push_back(B[2 * i + 1]);
  std::vector<long long> mo(mine.size() + 1), mn(mine.size() + 1);
  i64 nmap = 0;
  st = stitch_resolve(GA.data(), (i64)GA.size() / 2, GB.data(), (i64)GB.size() / 2, mine.data(), (i64)mine.size(),
                      mo.data(), mn.data(), &nmap);
  if (st) return st;
  return apply_map(d_out, n, d_ws, capacity, mo.data(), mn.data(), nmap, s);
}

}  // namespace ftk

using namespace ftk;


// ------------------------------------------------------------------------------ streaming ingestion
// push_field_data (traversal of the spacetime mesh one timestep after another):
// the caller pushes timesteps one at a time; the tracker stages them in a window of W + 1 planes and
// runs pass 1 (K1) on every full window -- anchors [t0, t0 + W) with plane t0 + W as the ghost plane,
// exactly the time-slab rule of DESIGN.md 7 -- then keeps the last plane as the first of the next
// window.  Records, their compact face ids, in-cube unions and trajectory edges accumulate in the
// caller's buffers across windows (record indices are global), so finish() runs pass 2 once over
// everything: the labels equal those of one ftk_cp_track over the whole field, while the field
// itself never has to be resident.
struct ftk_tracker {
  ftk_desc desc;        // spatial extents, dtype, scale; nt / t0 / nt_global / flags set per window
  int window;
  ftk_cp* out;
  int64_t capacity;
  char* ws;
  Layout L;
  char* buf;            // window + 1 planes, contiguous in time
  size_t plane_bytes;
  int64_t buf_t0;       // global timestep of buffer plane 0
  int nbuf;             // planes in the buffer
  int64_t pushed;       // timesteps pushed so far
  cudaStream_t stream;
  int error;            // first error of an enqueue (sticky, reported by finish)
};

static constexpr int64_t kOpenEnd = (1ll << 30) - 2;  // nt_global of a window that is not the last

// per-window survivor-list counters: fold into the sticky maximum, then reset
__global__ void k_window_reset(unsigned long long* c) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const unsigned long long w = c[CNT_WIN] > c[CNT_CUBES] ? c[CNT_WIN] : c[CNT_CUBES];
    if (w > c[CNT_WIN_MAX]) c[CNT_WIN_MAX] = w;
    c[CNT_WORK] = 0;
    c[CNT_WIN] = 0;
    c[CNT_CUBES] = 0;
    c[CNT_XBATCH] = 0;
  }
}

static size_t tracker_ws(const ftk_desc* d, int64_t capacity, int window) {
  const size_t plane = (size_t)d->n[0] * d->n[1] * d->n[2] * vertex_bytes(d);
  return align_up(layout(capacity, esz_of(d)).total, 256) + (size_t)(window + 1) * plane;
}

// pass 1 over the staged planes: a ghost window (not last) or the final window
static int tracker_window(ftk_tracker* tr, bool last) {
  ftk_desc c = tr->desc;
  c.t0 = tr->buf_t0;
  c.nt = tr->nbuf;
  c.nt_global = last ? tr->pushed : kOpenEnd;
  c.flags = (tr->desc.flags & FTK_VECTOR_FIELD) | (last ? 0u : FTK_GHOST_PLANE);
  auto* counters = reinterpret_cast<unsigned long long*>(tr->ws + tr->L.counters);
  k_window_reset<<<1, 32, 0, tr->stream>>>(counters);
  FTK_CUDA_TRY(cudaGetLastError());
  ExtractParams EP = extract_params(&c, tr->buf, tr->out, tr->capacity, tr->ws, tr->L, counters, true);
  int st = is_vector(&c) ? (c.ndim == 2 ? launch_extract_vec2d(EP, tr->stream) : launch_extract_vec3d(EP, tr->stream))
                         : (c.ndim == 2 ? launch_extract2d(EP, tr->stream) : launch_extract3d(EP, tr->stream));
  if (st) return st;
  if (!last) {  // the ghost plane becomes plane 0 of the next window
    FTK_CUDA_TRY(cudaMemcpyAsync(tr->buf, tr->buf + (size_t)(tr->nbuf - 1) * tr->plane_bytes, tr->plane_bytes,
                                 cudaMemcpyDeviceToDevice, tr->stream));
    tr->buf_t0 += tr->nbuf - 1;
    tr->nbuf = 1;
  }
  return FTK_OK;
}

extern "C" {

int ftk_abi_version(void) { return FTK_ABI_VERSION; }

const char* ftk_strerror(int s) {
  switch (s) {
    case FTK_OK: return "ok";
    case FTK_ERR_INVALID_ARG: return "invalid argument";
    case FTK_ERR_RANGE: return "quantized value out of the exact range (or non-finite input)";
    case FTK_ERR_CAPACITY: return "output capacity exceeded";
    case FTK_ERR_CUDA: return "CUDA error";
    case FTK_ERR_NCCL: return "NCCL error";
    case FTK_ERR_INVARIANT: return "0/2 cell invariant violated";
    case FTK_ERR_NOMEM: return "out of memory";
    default: return "unknown status";
  }
}

const char* ftk_last_error(void) { return g_last_error.c_str(); }

int ftk_num_faces(const ftk_desc* d, int64_t* n_faces) {
  int st = validate(d);
  if (st) return st;
  if (!n_faces) return FTK_ERR_INVALID_ARG;
  i64 ta, tb;
  owned_range(d, ta, tb);
  const int D = d->ndim + 1;
  const i64 ext[4] = {d->n[0], d->n[1], d->ndim == 3 ? d->n[2] : d->nt_global, d->nt_global};
  // sum over the face types of prod_a (N_a - s_a), restricted to owned anchor timesteps;
  // a type spans D-1 or D axes
  const int T = D == 3 ? kNT3() : kNT4();
  i64 total = 0;
  for (int ty = 0; ty < T; ++ty) {
    const int span = face_span(D, ty);
    i64 c = 1;
    for (int a = 0; a < D - 1; ++a) c *= ext[a] - ((span >> a) & 1);
    const int st_ = (span >> (D - 1)) & 1;
    const i64 t_hi = std::min<i64>(tb, d->nt_global - st_);  // anchors t with t + st <= nt_global - 1
    c *= std::max<i64>(0, t_hi - ta);
    total += c;
  }
  *n_faces = total;
  return FTK_OK;
}

int ftk_workspace_size(const ftk_desc* d, int64_t capacity, size_t* bytes) {
  int st = validate(d);
  if (st) return st;
  if (!bytes || capacity < 0 || capacity > kMaxCapacity) return FTK_ERR_INVALID_ARG;
  *bytes = layout(capacity, esz_of(d)).total;
  return FTK_OK;
}

// FTK_SORTED: records in face-id order (sort.cu), scratch from the workspace regions that are dead
// once the labels are final (stitch lists, relabel map, survivor lists and windows)
static int sort_output(const ftk_desc* desc, ftk_cp* d_out, int64_t n, void* d_ws, size_t ws_bytes, int64_t capacity,
                       cudaStream_t s) {
  if (!(desc->flags & FTK_SORTED) || n <= 1) return FTK_OK;
  const Layout L = layout(capacity, esz_of(desc));
  char* ws = static_cast<char*>(d_ws);
  if (L.cross + sort_scratch_bytes(n) > ws_bytes) return FTK_ERR_INVALID_ARG;  // cannot happen: n <= capacity
  const int T = desc->ndim == 2 ? 12 : 60;
  const unsigned long long maxfid = (unsigned long long)T * desc->n[0] * desc->n[1] * desc->n[2] * desc->nt_global - 1;
  const int bits = 64 - __builtin_clzll(maxfid | 1ull);
  const SortScratch S = sort_scratch(ws + L.cross, n);
  int st = launch_sort_records(d_out, reinterpret_cast<const long long*>(ws + L.fid), n, bits, S, s);
  if (st) return st;
  FTK_CUDA_TRY(cudaStreamSynchronize(s));
  return FTK_OK;
}

int ftk_cp_extract(const ftk_desc* desc, const void* d_field, ftk_cp* d_out, int64_t capacity, int64_t* n_out,
                   void* d_ws, size_t ws_bytes, ftk_stream stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int st = run(desc, d_field, d_out, capacity, n_out, d_ws, ws_bytes, s, false);
  if (st) return st;
  return sort_output(desc, d_out, *n_out, d_ws, ws_bytes, capacity, s);
}

int ftk_cp_track(const ftk_desc* desc, const void* d_field, ftk_cp* d_out, int64_t capacity, int64_t* n_out,
                 void* d_ws, size_t ws_bytes, ftk_stream stream, ftk_comm* comm) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int st = run(desc, d_field, d_out, capacity, n_out, d_ws, ws_bytes, s, true);
  if (comm && comm->world > 1) {
    // every rank enters the exchange, so a failure on one slab cannot leave its peers waiting in
    // NCCL: the failure codes travel in the seam blocks and all ranks return the agreed status
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (g_profiling) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
    }
    const int local = st;
    st = stitch_nccl(comm, local, desc, d_out, local ? 0 : *n_out, d_ws, capacity, s);
    if (g_profiling) {
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&g_ms[2], e0, e1);
      g_ms[3] += g_ms[2];
      g_kms[3] = g_ms[2];
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
  }
  if (st) return st;
  return sort_output(desc, d_out, *n_out, d_ws, ws_bytes, capacity, s);
}

int ftk_stitch_export(const ftk_desc* desc, void* d_ws, size_t ws_bytes, int64_t capacity, int64_t* h_A,
                      int64_t capA, int64_t* nA, int64_t* h_B, int64_t capB, int64_t* nB, ftk_stream stream) {
  int st = validate(desc);
  if (st) return st;
  if (!d_ws || !nA || !nB || ws_bytes < layout(capacity, esz_of(desc)).total) return FTK_ERR_INVALID_ARG;
  std::vector<long long> A, B;
  st = read_exports(desc, d_ws, capacity, A, B, reinterpret_cast<cudaStream_t>(stream));
  if (st) return st;
  *nA = (int64_t)A.size() / 2;
  *nB = (int64_t)B.size() / 2;
  if (*nA > capA || *nB > capB) return FTK_ERR_CAPACITY;
  if (h_A) std::copy(A.begin(), A.end(), h_A);
  if (h_B) std::copy(B.begin(), B.end(), h_B);
  return FTK_OK;
}

int ftk_stitch_resolve(const int64_t* A, int64_t nA, const int64_t* B, int64_t nB, const int64_t* mine,
                       int64_t nmine, int64_t* map_old, int64_t* map_new, int64_t* nmap) {
  if ((nA && !A) || (nB && !B) || (nmine && !mine) || !nmap || (nmine && (!map_old || !map_new)))
    return FTK_ERR_INVALID_ARG;
  i64 n = 0;
  const int st = stitch_resolve(reinterpret_cast<const long long*>(A), nA, reinterpret_cast<const long long*>(B), nB,
                                reinterpret_cast<const long long*>(mine), nmine,
                                reinterpret_cast<long long*>(map_old), reinterpret_cast<long long*>(map_new), &n);
  *nmap = n;
  return st;
}

int ftk_relabel(ftk_cp* d_out, int64_t n, const int64_t* h_map_old, const int64_t* h_map_new, int64_t nmap,
                void* d_ws, size_t ws_bytes, int64_t capacity, ftk_stream stream) {
  if (!d_ws || ws_bytes < layout(capacity).win || (nmap && (!h_map_old || !h_map_new))) return FTK_ERR_INVALID_ARG;
  return apply_map(d_out, n, d_ws, capacity, reinterpret_cast<const long long*>(h_map_old),
                   reinterpret_cast<const long long*>(h_map_new), nmap, reinterpret_cast<cudaStream_t>(stream));
}

int ftk_cp_track_host(const ftk_desc* desc, const void* h_field, void* d_stage, ftk_cp* d_out, ftk_cp* h_out,
                      int64_t capacity, int64_t* n_out, void* d_ws, size_t ws_bytes, ftk_stream stream) {
  int st = validate(desc);
  if (st) return st;
  if (!h_field || !d_stage || !h_out || !n_out) return FTK_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t esz = desc->dtype == FTK_F32 ? 4 : 8;
  const size_t bytes = (size_t)desc->n[0] * desc->n[1] * desc->n[2] * desc->nt * esz * (is_vector(desc) ? desc->ndim : 1);
  FTK_CUDA_TRY(cudaMemcpyAsync(d_stage, h_field, bytes, cudaMemcpyHostToDevice, s));
  st = run(desc, d_stage, d_out, capacity, n_out, d_ws, ws_bytes, s, true);
  if (st) return st;
  FTK_CUDA_TRY(cudaMemcpyAsync(h_out, d_out, (size_t)*n_out * sizeof(ftk_cp), cudaMemcpyDeviceToHost, s));
  FTK_CUDA_TRY(cudaStreamSynchronize(s));
  return FTK_OK;
}

int ftk_tracker_workspace_size(const ftk_desc* desc, int64_t capacity, int32_t window, size_t* bytes) {
  if (!desc || !bytes || window < 1 || capacity < 0 || capacity > kMaxCapacity) return FTK_ERR_INVALID_ARG;
  ftk_desc c = *desc;
  c.t0 = 0;
  c.nt = 2;
  c.nt_global = 2;
  c.flags &= FTK_VECTOR_FIELD;
  const int st = validate(&c);
  if (st) return st;
  *bytes = tracker_ws(&c, capacity, window);
  return FTK_OK;
}

int ftk_tracker_begin(ftk_tracker** out, const ftk_desc* desc, int32_t window, ftk_cp* d_out, int64_t capacity,
                      void* d_ws, size_t ws_bytes, ftk_stream stream) {
  size_t need = 0;
  if (!out) return FTK_ERR_INVALID_ARG;
  int st = ftk_tracker_workspace_size(desc, capacity, window, &need);
  if (st) return st;
  if (!d_ws || ws_bytes < need || (capacity > 0 && !d_out)) return FTK_ERR_INVALID_ARG;
  auto* tr = new (std::nothrow) ftk_tracker();
  if (!tr) return FTK_ERR_NOMEM;
  tr->desc = *desc;
  tr->desc.t0 = 0;
  tr->desc.flags &= FTK_VECTOR_FIELD;
  tr->window = window;
  tr->out = d_out;
  tr->capacity = capacity;
  tr->ws = static_cast<char*>(d_ws);
  tr->L = layout(capacity, esz_of(desc));
  tr->buf = tr->ws + align_up(tr->L.total, 256);
  tr->plane_bytes = (size_t)desc->n[0] * desc->n[1] * desc->n[2] * vertex_bytes(desc);
  tr->stream = reinterpret_cast<cudaStream_t>(stream);
  auto* counters = reinterpret_cast<unsigned long long*>(tr->ws + tr->L.counters);
  const cudaError_t e = cudaMemsetAsync(counters, 0, CNT_N * sizeof(u64), tr->stream);
  if (e != cudaSuccess) {
    delete tr;
    return set_cuda_error(e, "ftk_tracker_begin");
  }
  *out = tr;
  return FTK_OK;
}

int ftk_tracker_push(ftk_tracker* tr, const void* plane) {
  if (!tr || !plane) return FTK_ERR_INVALID_ARG;
  if (tr->error) return tr->error;
  if (tr->pushed + 1 >= kOpenEnd) return FTK_ERR_INVALID_ARG;
  cudaError_t e = cudaMemcpyAsync(tr->buf + (size_t)tr->nbuf * tr->plane_bytes, plane, tr->plane_bytes,
                                  cudaMemcpyDefault, tr->stream);
  if (e != cudaSuccess) return tr->error = set_cuda_error(e, "ftk_tracker_push");
  ++tr->nbuf;
  ++tr->pushed;
  if (tr->nbuf == tr->window + 1) {
    const int st = tracker_window(tr, false);
    if (st) return tr->error = st;
  }
  return FTK_OK;
}

int ftk_tracker_finish(ftk_tracker* tr, int64_t* n_out) {
  if (!tr || !n_out) return FTK_ERR_INVALID_ARG;
  std::unique_ptr<ftk_tracker> own(tr);
  if (tr->error) return tr->error;
  if (tr->pushed < 2) return FTK_ERR_INVALID_ARG;  // tracking needs two timesteps
  int st = tracker_window(tr, true);
  if (st) return st;
  ftk_desc f = tr->desc;
  f.t0 = 0;
  f.nt = tr->pushed;
  f.nt_global = tr->pushed;
  f.flags = tr->desc.flags & FTK_VECTOR_FIELD;
  auto* counters = reinterpret_cast<unsigned long long*>(tr->ws + tr->L.counters);
  TrackParams TP = track_params(&f, tr->out, tr->capacity, tr->ws, tr->L, counters);
  const i64 ext[4] = {f.n[0], f.n[1], f.n[2], f.nt_global};
  st = launch_track(TP, f.ndim, ext, tr->stream);
  if (st) return st;
  unsigned long long* host_cnt = pinned_counters();
  FTK_CUDA_TRY(cudaMemcpyAsync(host_cnt, counters, CNT_N * sizeof(unsigned long long), cudaMemcpyDeviceToHost, tr->stream));
  FTK_CUDA_TRY(cudaStreamSynchronize(tr->stream));
  *n_out = (int64_t)host_cnt[CNT_NOUT];
  ftk_num_faces(&f, &g_stats[0]);
  g_stats[1] = (int64_t)host_cnt[CNT_SURVIVORS];
  g_stats[2] = (int64_t)host_cnt[CNT_NOUT];
  return result_status(&f, host_cnt, tr->L, tr->capacity, n_out);
}

int ftk_tracker_abort(ftk_tracker* tr) {
  delete tr;
  return FTK_OK;
}

// ------------------------------------------------------------------------------ post-processing
static int post_setup(const ftk_desc* desc, int64_t n, void* d_ws, size_t ws_bytes, int64_t capacity, Layout& L) {
  int st = validate(desc);
  if (st) return st;
  if (!d_ws || n < 0 || capacity < 0 || capacity > kMaxCapacity || n > capacity) return FTK_ERR_INVALID_ARG;
  L = layout(capacity, esz_of(desc));
  if (ws_bytes < L.total) return FTK_ERR_INVALID_ARG;
  return FTK_OK;
}

int ftk_post_adjacency(const ftk_desc* desc, const ftk_cp* d_rec, int64_t n, int64_t* d_nbr, void* d_ws,
                       size_t ws_bytes, int64_t capacity, ftk_stream stream) {
  Layout L;
  int st = post_setup(desc, n, d_ws, ws_bytes, capacity, L);
  if (st) return st;
  if (n > 0 && (!d_rec || !d_nbr)) return FTK_ERR_INVALID_ARG;
  char* ws = static_cast<char*>(d_ws);
  auto* counters = reinterpret_cast<unsigned long long*>(ws + L.counters);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  TrackParams TP = track_params(desc, const_cast<ftk_cp*>(d_rec), n, ws, L, counters);
  FTK_CUDA_TRY(cudaMemsetAsync(counters + CNT_INVARIANT, 0, sizeof(u64), s));
  const i64 ext[4] = {desc->n[0], desc->n[1], desc->n[2], desc->nt_global};
  st = launch_post_adjacency(TP, desc->ndim, ext, n, reinterpret_cast<long long*>(d_nbr), s);
  if (st) return st;
  unsigned long long bad = 0;
  FTK_CUDA_TRY(cudaMemcpyAsync(&bad, counters + CNT_INVARIANT, sizeof bad, cudaMemcpyDeviceToHost, s));
  FTK_CUDA_TRY(cudaStreamSynchronize(s));
  if (bad) {
    g_last_error = "post_adjacency: parent cells without exactly one partner: " + std::to_string(bad);
    return FTK_ERR_INVARIANT;
  }
  return FTK_OK;
}

static int post_op(int op, const ftk_desc* desc, ftk_cp* d_rec, const int64_t* d_nbr, int64_t n, double t0,
                   double dmin, int drop_loops, int half_window, ftk_cp* d_out, int64_t cap, int64_t* n_out,
                   void* d_ws, size_t ws_bytes, int64_t capacity, ftk_stream stream, double tau = 0.0) {
  Layout L;
  int st = post_setup(desc, n, d_ws, ws_bytes, capacity, L);
  if (st) return st;
  if (n > 0 && (!d_rec || !d_nbr)) return FTK_ERR_INVALID_ARG;
  const bool in_place = op == 2 || op == 3;
  if (!in_place && (!n_out || cap < 0 || (cap > 0 && !d_out))) return FTK_ERR_INVALID_ARG;
  char* ws = static_cast<char*>(d_ws);
  auto* counters = reinterpret_cast<unsigned long long*>(ws + L.counters);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  TrackParams TP = track_params(desc, d_rec, n, ws, L, counters);
  PostCall c;
  c.rec = d_rec;
  c.rec_mut = d_rec;
  c.nbr = reinterpret_cast<const long long*>(d_nbr);
  c.n = n;
  c.out = d_out;
  c.cap = cap;
  c.count = counters + CNT_POST;
  c.scratch = reinterpret_cast<long long*>(ws + L.map);
  c.t0 = t0;
  c.dmin = dmin;
  c.drop_loops = drop_loops;
  c.half_window = half_window;
  c.tau = tau;
  FTK_CUDA_TRY(cudaMemsetAsync(counters + CNT_POST, 0, sizeof(u64), s));
  if (n > 0) {
    st = launch_post(TP, op, c, s);
    if (st) return st;
  }
  unsigned long long cnt = 0;
  FTK_CUDA_TRY(cudaMemcpyAsync(&cnt, counters + CNT_POST, sizeof cnt, cudaMemcpyDeviceToHost, s));
  FTK_CUDA_TRY(cudaStreamSynchronize(s));
  if (in_place) return FTK_OK;
  *n_out = (int64_t)cnt;
  return (int64_t)cnt > cap ? FTK_ERR_CAPACITY : FTK_OK;
}

int ftk_post_slice(const ftk_desc* desc, const ftk_cp* d_rec, const int64_t* d_nbr, int64_t n, double t0,
                   ftk_cp* d_out, int64_t cap, int64_t* n_out, void* d_ws, size_t ws_bytes, int64_t capacity,
                   ftk_stream stream) {
  if (!(t0 == t0)) return FTK_ERR_INVALID_ARG;
  return post_op(0, desc, const_cast<ftk_cp*>(d_rec), d_nbr, n, t0, 0.0, 0, 0, d_out, cap, n_out, d_ws, ws_bytes,
                 capacity, stream);
}

int ftk_post_filter(const ftk_desc* desc, const ftk_cp* d_rec, const int64_t* d_nbr, int64_t n, double min_duration,
                    int32_t drop_loops, ftk_cp* d_out, int64_t cap, int64_t* n_out, void* d_ws, size_t ws_bytes,
                    int64_t capacity, ftk_stream stream) {
  if (!(min_duration == min_duration)) return FTK_ERR_INVALID_ARG;
  return post_op(1, desc, const_cast<ftk_cp*>(d_rec), d_nbr, n, 0.0, min_duration, drop_loops != 0, 0, d_out, cap,
                 n_out, d_ws, ws_bytes, capacity, stream);
}

int ftk_post_smooth_types(const ftk_desc* desc, ftk_cp* d_rec, const int64_t* d_nbr, int64_t n, int32_t half_window,
                          void* d_ws, size_t ws_bytes, int64_t capacity, ftk_stream stream) {
  if (half_window < 1) return FTK_ERR_INVALID_ARG;
  return post_op(2, desc, d_rec, d_nbr, n, 0.0, 0.0, 0, half_window, nullptr, 0, nullptr, d_ws, ws_bytes, capacity,
                 stream);
}

int ftk_post_simplify_types(const ftk_desc* desc, ftk_cp* d_rec, const int64_t* d_nbr, int64_t n, double tau,
                            void* d_ws, size_t ws_bytes, int64_t capacity, ftk_stream stream) {
  if (!(tau == tau)) return FTK_ERR_INVALID_ARG;
  return post_op(3, desc, d_rec, d_nbr, n, 0.0, 0.0, 0, 0, nullptr, 0, nullptr, d_ws, ws_bytes, capacity, stream,
                 tau);
}

// ------------------------------------------------------------------------------ isovolume tracking
static int iso_run(const ftk_desc* desc, double isovalue, const void* d_field, ftk_cp* d_out, int64_t capacity,
                   int64_t* n_out, bool mesh, int64_t* d_elems, int64_t elem_cap, int64_t* n_elems, void* d_ws,
                   size_t ws_bytes, ftk_stream stream_) {
  int st = validate(desc);
  if (st) return st;
  if (is_vector(desc) || (desc->flags & FTK_GHOST_PLANE) || desc->t0 != 0 || desc->nt != desc->nt_global || desc->nt < 2)
    return FTK_ERR_INVALID_ARG;
  if (desc->n[0] >= (1ll << 31) || desc->n[1] >= (1ll << 31) || desc->n[2] >= (1ll << 31) || desc->nt >= (1ll << 31))
    return FTK_ERR_INVALID_ARG;  // k_iso queues anchors as int32 coordinates
  if (!d_field || !n_out || !d_ws || capacity < 0 || capacity > kMaxCapacity || (capacity > 0 && !d_out) ||
      !(isovalue == isovalue))
    return FTK_ERR_INVALID_ARG;
  const Layout L = layout(capacity, esz_of(desc));
  if (ws_bytes < L.total) return FTK_ERR_INVALID_ARG;
  const double cqd = std::nearbyint(std::ldexp(isovalue, desc->scale_log2));
  if (!(std::fabs(cqd) < std::ldexp(1.0, desc->ndim == 2 ? 59 : 38))) return FTK_ERR_RANGE;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  char* ws = static_cast<char*>(d_ws);
  auto* counters = reinterpret_cast<unsigned long long*>(ws + L.counters);
  FTK_CUDA_TRY(cudaMemsetAsync(counters, 0, CNT_N * sizeof(u64), stream));
  ExtractParams EP = extract_params(desc, d_field, d_out, capacity, ws, L, counters, false);
  EP.mesh = mesh;
  EP.elems = reinterpret_cast<long long*>(d_elems);
  EP.elem_cap = elem_cap;
  st = launch_iso(EP, (long long)cqd, desc->ndim, stream);
  if (st) return st;
  TrackParams TP = track_params(desc, d_out, capacity, ws, L, counters);
  TP.T = desc->ndim == 2 ? 7 : 15;           // edge types per cube
  TP.inv[0] = 1.0 / TP.T;
  TP.lookup_types = (1ull << TP.T) - 1ull;   // links may name any edge
  TP.prelinked = false;
  TP.verify = false;
  TP.ghost_t = -1;
  TP.first_t = -1;
  const i64 ext[4] = {desc->n[0], desc->n[1], desc->n[2], desc->nt_global};
  st = launch_track(TP, desc->ndim, ext, stream);
  if (st) return st;
  unsigned long long* host_cnt = pinned_counters();
  FTK_CUDA_TRY(cudaMemcpyAsync(host_cnt, counters, CNT_N * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
  FTK_CUDA_TRY(cudaStreamSynchronize(stream));
  *n_out = (int64_t)host_cnt[CNT_NOUT];
  if (n_elems) *n_elems = (int64_t)host_cnt[CNT_ELEMS];
  st = range_status(desc, host_cnt[CNT_MAXBITS]);
  if (st) return st;
  if ((i64)host_cnt[CNT_NOUT] > capacity || (i64)host_cnt[CNT_EDGES] > capacity || (i64)host_cnt[CNT_WIN] > L.wcap) {
    // records, links, or candidate cubes (k_iso_scan's list, wcap = max(1024, capacity) entries)
    *n_out = std::max<int64_t>(std::max<int64_t>((int64_t)host_cnt[CNT_NOUT], (int64_t)host_cnt[CNT_EDGES]),
                               (int64_t)host_cnt[CNT_WIN]);
    return FTK_ERR_CAPACITY;
  }
  if (mesh && (int64_t)host_cnt[CNT_ELEMS] > elem_cap) return FTK_ERR_CAPACITY;  // *n_elems = the need
  if (host_cnt[CNT_INVARIANT]) {
    g_last_error = "isovolume cells with a crossed-edge count not in {0, d, 2(d-1)}: " + std::to_string(host_cnt[CNT_INVARIANT]);
    return FTK_ERR_INVARIANT;
  }
  return FTK_OK;
}

int ftk_iso_track(const ftk_desc* desc, double isovalue, const void* d_field, ftk_cp* d_out, int64_t capacity,
                  int64_t* n_out, void* d_ws, size_t ws_bytes, ftk_stream stream) {
  return iso_run(desc, isovalue, d_field, d_out, capacity, n_out, false, nullptr, 0, nullptr, d_ws, ws_bytes, stream);
}

int ftk_iso_track_mesh(const ftk_desc* desc, double isovalue, const void* d_field, ftk_cp* d_out, int64_t capacity,
                       int64_t* n_out, int64_t* d_elems, int64_t elem_cap, int64_t* n_elems, void* d_ws,
                       size_t ws_bytes, ftk_stream stream) {
  if (!n_elems || elem_cap < 0 || (elem_cap > 0 && !d_elems)) return FTK_ERR_INVALID_ARG;
  return iso_run(desc, isovalue, d_field, d_out, capacity, n_out, true, d_elems, elem_cap, n_elems, d_ws, ws_bytes,
                 stream);
}

int ftk_set_profiling(int enable) {
  g_profiling = enable;
  return FTK_OK;
}

int ftk_last_kernel_timings(float* ms, int n) {
  if (!ms || n < 0) return FTK_ERR_INVALID_ARG;
  for (int i = 0; i < n && i < 4; ++i) ms[i] = g_kms[i];
  return FTK_OK;
}

int ftk_last_timings(float* ms4, int64_t* stats3) {
  if (ms4)
    for (int i = 0; i < 4; ++i) ms4[i] = g_ms[i];
  if (stats3)
    for (int i = 0; i < 3; ++i) stats3[i] = g_stats[i];
  return FTK_OK;
}

int ftk_comm_get_unique_id(uint8_t id[128]) {
  if (!id) return FTK_ERR_INVALID_ARG;
  if (!g_nccl.load()) return FTK_ERR_NCCL;
  ncclUniqueId u;
  const int st = nccl_check(g_nccl.getUniqueId(&u), "ncclGetUniqueId");
  if (st) return st;
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id, &u, 128);
  return FTK_OK;
}

int ftk_seam_pack(const ftk_desc* desc, void* d_ws, size_t ws_bytes, int64_t capacity, int64_t* d_block,
                  int64_t cap, ftk_stream stream) {
  int st = validate(desc);
  if (st) return st;
  if (!d_ws || !d_block || cap < 1 || ws_bytes < layout(capacity, esz_of(desc)).total) return FTK_ERR_INVALID_ARG;
  return seam_pack(d_ws, capacity, reinterpret_cast<long long*>(d_block), cap, reinterpret_cast<cudaStream_t>(stream));
}

int ftk_seam_resolve(const int64_t* d_all, int world, int64_t cap, ftk_cp* d_out, int64_t n, ftk_stream stream) {
  if (!d_all || world < 1 || cap < 1 || n < 0 || (n > 0 && !d_out)) return FTK_ERR_INVALID_ARG;
  return seam_resolve(reinterpret_cast<const long long*>(d_all), world, cap, d_out, n,
                      reinterpret_cast<cudaStream_t>(stream));
}

int ftk_comm_init(ftk_comm** comm, int rank, int world, const uint8_t id[128]) {
  if (!comm || !id || world < 1 || rank < 0 || rank >= world) return FTK_ERR_INVALID_ARG;
  if (!g_nccl.load()) return FTK_ERR_NCCL;
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ftk_comm* c = new ftk_comm();
  c->rank = rank;
  c->world = world;
  int st = FTK_OK;
  const cudaError_t de = cudaGetDevice(&c->device);
  if (de != cudaSuccess) st = set_cuda_error(de, "cudaGetDevice");
  if (!st) st = nccl_check(g_nccl.commInitRank(&c->comm, world, u, rank), "ncclCommInitRank");
  // the seam blocks and resolve tables are allocated here, not in ftk_cp_track
  if (!st && world > 1) st = comm_reserve(c, kDefaultSeamPairs);
  if (st) {
    ftk_comm_destroy(c);
    return st;
  }
  *comm = c;
  return FTK_OK;
}

int ftk_comm_reserve(ftk_comm* comm, int64_t seam_pairs) {
  if (!comm || seam_pairs < 1) return FTK_ERR_INVALID_ARG;
  if (comm->world <= 1 || seam_pairs <= comm->seam_cap) return FTK_OK;
  return comm_reserve(comm, seam_pairs);
}

int ftk_comm_destroy(ftk_comm* comm) {
  if (!comm) return FTK_OK;
  if (comm->comm && g_nccl.commDestroy) g_nccl.commDestroy(comm->comm);
  cudaFree(comm->d_send);
  cudaFree(comm->d_recv);
  cudaFree(comm->d_gather);
  cudaFree(comm->d_scratch);
  delete comm;
  return FTK_OK;
}

int ftk_set_debug(uint32_t flags) {
  if (flags & ~(uint32_t)(FTK_DEBUG_FORCE_GENERIC | FTK_DEBUG_VERIFY_LINK | FTK_DEBUG_STITCH_HOST | FTK_DEBUG_NO_GRAPH |
                          FTK_DEBUG_UF_BY_ID))
    return FTK_ERR_INVALID_ARG;
  g_debug = flags;
  return FTK_OK;
}

}  // extern "C"
