// runtime.cu -- host side of the C-ABI (include/ftk_cp.h): validation, workspace layout, stream
// ordering of K1 (pass 1) and pass 2, error mapping, profiling events.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "extract2d.cuh"
#include "track.cuh"
#include "kuhn.cuh"
#include <algorithm>

namespace ftk {

static thread_local std::string g_last_error;
static thread_local int g_profiling = 0;
static thread_local float g_ms[4] = {0, 0, 0, 0};
static thread_local int64_t g_stats[3] = {0, 0, 0};

int set_cuda_error(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return FTK_ERR_CUDA;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Layout {
  size_t counters, table, edges, fid, parent, total;
  u64 hcap;
};

static Layout layout(i64 capacity) {
  Layout L;
  u64 h = 1024;
  while (h < (u64)(capacity + capacity / 2)) h <<= 1;
  L.hcap = h;
  size_t off = 0;
  L.counters = off;
  off = align_up(off + CNT_N * sizeof(u64), 256);
  L.table = off;
  off = align_up(off + h * sizeof(HashSlot), 256);
  L.edges = off;
  off = align_up(off + (size_t)capacity * 2 * sizeof(long long), 256);
  L.fid = off;
  off = align_up(off + (size_t)capacity * sizeof(i64), 256);
  L.parent = off;
  off = align_up(off + (size_t)capacity * sizeof(int), 256);
  L.total = off;
  return L;
}

static int validate(const ftk_desc* d) {
  if (!d) return FTK_ERR_INVALID_ARG;
  if (d->ndim != 2 && d->ndim != 3) return FTK_ERR_INVALID_ARG;
  if (d->dtype != FTK_F32 && d->dtype != FTK_F64) return FTK_ERR_INVALID_ARG;
  if (d->n[0] < 3 || d->n[1] < 3) return FTK_ERR_INVALID_ARG;
  if (d->ndim == 3 ? d->n[2] < 3 : d->n[2] != 1) return FTK_ERR_INVALID_ARG;
  if (d->nt < 1 || d->t0 < 0 || d->t0 + d->nt > d->nt_global) return FTK_ERR_INVALID_ARG;
  if (d->scale_log2 < -64 || d->scale_log2 > 64) return FTK_ERR_INVALID_ARG;
  if ((d->flags & FTK_GHOST_PLANE) && d->nt < 2) return FTK_ERR_INVALID_ARG;
  if (d->flags & ~(FTK_GHOST_PLANE | FTK_SORTED)) return FTK_ERR_INVALID_ARG;
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

struct Events {
  cudaEvent_t e[4] = {nullptr, nullptr, nullptr, nullptr};
  bool on = false;
  Events() {
    if (g_profiling) {
      on = true;
      for (auto& x : e) cudaEventCreate(&x);
    }
  }
  ~Events() {
    for (auto& x : e)
      if (x) cudaEventDestroy(x);
  }
  void rec(int i, cudaStream_t s) {
    if (on) cudaEventRecord(e[i], s);
  }
};

static int run(const ftk_desc* desc, const void* d_field, ftk_cp* d_out, int64_t capacity, int64_t* n_out,
               void* d_ws, size_t ws_bytes, cudaStream_t stream, bool track) {
  int st = validate(desc);
  if (st) return st;
  if (!d_field || !n_out || !d_ws || capacity < 0 || (capacity > 0 && !d_out)) return FTK_ERR_INVALID_ARG;
  const Layout L = layout(capacity);
  if (ws_bytes < L.total) return FTK_ERR_INVALID_ARG;
  char* ws = static_cast<char*>(d_ws);
  auto* counters = reinterpret_cast<unsigned long long*>(ws + L.counters);
  Events ev;
  ev.rec(0, stream);
  FTK_CUDA_TRY(cudaMemsetAsync(counters, 0, CNT_N * sizeof(u64), stream));

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
  EP.thr = std::ldexp(1.0, 1 - desc->scale_log2);
  EP.out = d_out;
  EP.capacity = capacity;
  EP.counters = counters;
  EP.edges = reinterpret_cast<long long*>(ws + L.edges);
  EP.force_generic = getenv("FTK_FORCE_GENERIC") != nullptr;
  ev.rec(1, stream);
  st = desc->ndim == 2 ? launch_extract2d(EP, stream) : launch_extract3d(EP, stream);
  if (st) return st;
  ev.rec(2, stream);
  if (track) {
    TrackParams TP;
    TP.rec = d_out;
    TP.capacity = capacity;
    TP.counters = counters;
    TP.table = reinterpret_cast<HashSlot*>(ws + L.table);
    TP.table_cap = L.hcap;
    TP.edges = reinterpret_cast<const long long*>(ws + L.edges);
    TP.verify = getenv("FTK_VERIFY_LINK") != nullptr;
    TP.fid = reinterpret_cast<i64*>(ws + L.fid);
    TP.parent = reinterpret_cast<int*>(ws + L.parent);
    const i64 ext[4] = {desc->n[0], desc->n[1], desc->n[2], desc->nt_global};
    st = launch_track(TP, desc->ndim, ext, stream);
    if (st) return st;
  }
  ev.rec(3, stream);
  unsigned long long host_cnt[CNT_N];
  FTK_CUDA_TRY(cudaMemcpyAsync(host_cnt, counters, sizeof host_cnt, cudaMemcpyDeviceToHost, stream));
  FTK_CUDA_TRY(cudaStreamSynchronize(stream));
  *n_out = (int64_t)host_cnt[CNT_NOUT];
  if (getenv("FTK_PRINT_PROF")) {
    const char* names[] = {"scan", "wait_full", "enqueue", "wait_ring", "exact_wait", "exact_faces",
                           "exact_records", "producer_wait", "other"};
    fprintf(stderr, "K1 cycle accounting (sum over warps, Gcycles):");
    for (int i = 0; i < 9; ++i) fprintf(stderr, " %s=%.3f", names[i], host_cnt[CNT_PROF + i] * 1e-9);
    fprintf(stderr, " edges=%llu\n", host_cnt[CNT_EDGES]);
  }
  if (ev.on) {
    cudaEventElapsedTime(&g_ms[0], ev.e[1], ev.e[2]);
    cudaEventElapsedTime(&g_ms[1], ev.e[2], ev.e[3]);
    g_ms[2] = 0.f;
    cudaEventElapsedTime(&g_ms[3], ev.e[0], ev.e[3]);
  }
  ftk_num_faces(desc, &g_stats[0]);
  g_stats[1] = (int64_t)host_cnt[CNT_SURVIVORS];
  g_stats[2] = (int64_t)host_cnt[CNT_NOUT];
  st = range_status(desc, host_cnt[CNT_MAXBITS]);
  if (st) return st;
  if ((i64)host_cnt[CNT_NOUT] > capacity) return FTK_ERR_CAPACITY;
  if (host_cnt[CNT_INVARIANT]) {
    g_last_error = "cells with a punctured-face count not in {0, 2}: " + std::to_string(host_cnt[CNT_INVARIANT]);
    return FTK_ERR_INVARIANT;
  }
  return FTK_OK;
}


}  // namespace ftk

using namespace ftk;

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
  if (!bytes || capacity < 0) return FTK_ERR_INVALID_ARG;
  *bytes = layout(capacity).total;
  return FTK_OK;
}

int ftk_cp_extract(const ftk_desc* desc, const void* d_field, ftk_cp* d_out, int64_t capacity, int64_t* n_out,
                   void* d_ws, size_t ws_bytes, ftk_stream stream) {
  return run(desc, d_field, d_out, capacity, n_out, d_ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), false);
}

int ftk_cp_track(const ftk_desc* desc, const void* d_field, ftk_cp* d_out, int64_t capacity, int64_t* n_out,
                 void* d_ws, size_t ws_bytes, ftk_stream stream, ftk_comm* comm) {
  if (comm) {
    g_last_error = "multi-GPU stitch not built yet";
    return FTK_ERR_NCCL;
  }
  return run(desc, d_field, d_out, capacity, n_out, d_ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), true);
}

int ftk_cp_track_host(const ftk_desc* desc, const void* h_field, void* d_stage, ftk_cp* d_out, ftk_cp* h_out,
                      int64_t capacity, int64_t* n_out, void* d_ws, size_t ws_bytes, ftk_stream stream) {
  int st = validate(desc);
  if (st) return st;
  if (!h_field || !d_stage || !h_out || !n_out) return FTK_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t esz = desc->dtype == FTK_F32 ? 4 : 8;
  const size_t bytes = (size_t)desc->n[0] * desc->n[1] * desc->n[2] * desc->nt * esz;
  FTK_CUDA_TRY(cudaMemcpyAsync(d_stage, h_field, bytes, cudaMemcpyHostToDevice, s));
  st = run(desc, d_stage, d_out, capacity, n_out, d_ws, ws_bytes, s, true);
  if (st) return st;
  FTK_CUDA_TRY(cudaMemcpyAsync(h_out, d_out, (size_t)*n_out * sizeof(ftk_cp), cudaMemcpyDeviceToHost, s));
  FTK_CUDA_TRY(cudaStreamSynchronize(s));
  return FTK_OK;
}

int ftk_set_profiling(int enable) {
  g_profiling = enable;
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
  (void)id;
  g_last_error = "NCCL communicator not built yet";
  return FTK_ERR_NCCL;
}
int ftk_comm_init(ftk_comm** comm, int rank, int world, const uint8_t id[128]) {
  (void)comm; (void)rank; (void)world; (void)id;
  g_last_error = "NCCL communicator not built yet";
  return FTK_ERR_NCCL;
}
int ftk_comm_destroy(ftk_comm* comm) {
  (void)comm;
  return FTK_OK;
}

}  // extern "C"
