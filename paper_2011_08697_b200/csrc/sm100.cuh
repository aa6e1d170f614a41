// sm100.cuh -- sm_100a device helpers shared by the pass-1 kernels: mbarrier waits, TMA tile loads,
// packed f32x2 arithmetic, the globaltimer watchdog.  Product path only.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <unordered_map>

namespace ftk {
namespace sm100 {

// ---------------------------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA + packed fp32
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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar, uint32_t count = 1) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
#ifndef FTK_K1_HINT
#define FTK_K1_HINT 0
#endif
#ifndef FTK_K1_MBSLEEP
#define FTK_K1_MBSLEEP 32     // scan warps waiting for a plane
#endif
#ifndef FTK_K1_SCANSLEEP
#define FTK_K1_SCANSLEEP 0    // scan warps wait for a plane with the suspend-time hint too
#endif
#ifndef FTK_K1_PRODSLEEP
#define FTK_K1_PRODSLEEP 256  // the producer waiting for a free stage
#endif
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  if (FTK_K1_HINT) {  // suspend-time hint (ns)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"((uint32_t)FTK_K1_HINT)
        : "memory");
  } else {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
  return done != 0;
}
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Watchdog: a wait longer than FTK_WAIT_WATCHDOG_NS of wall-clock (%globaltimer) reports where it is
// stuck and traps instead of hanging the GPU.  The default (60 s) is far beyond any valid wait, also
// under compute-sanitizer or time-slicing; build with -DFTK_WAIT_WATCHDOG_NS=0 to compile it out.
#ifndef FTK_WAIT_WATCHDOG_NS
#define FTK_WAIT_WATCHDOG_NS 60000000000ull
#endif
static __device__ __noinline__ void wait_timeout(int what, int a, int b) {
  if ((threadIdx.x & 31) == 0)
    printf("ftk k_extract2d: wait timeout what=%d a=%d b=%d block=%d warp=%d\n", what, a, b, blockIdx.x,
           threadIdx.x >> 5);
  __trap();
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, int what, int a, int sleep_ns) {
  if (mbar_try(bar, parity)) return;
  // back off: a spinning warp takes issue slots from the scan warps on its SMSP
  const unsigned long long t0 = gtimer_ns();
  int spins = 0;
  while (!mbar_try(bar, parity)) {
    __nanosleep(sleep_ns);
    if (FTK_WAIT_WATCHDOG_NS && (++spins & 15) == 0) {
      if (gtimer_ns() - t0 > FTK_WAIT_WATCHDOG_NS) wait_timeout(what, a, (int)parity);
    }
  }
}
// the producer's wait for a free stage: try_wait with a suspend-time hint, so the warp sleeps in
// hardware until the phase completes (no issue slots spent) -- bounded by the same 2 s trap
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, int what, int a) {
  const unsigned long long t0 = gtimer_ns();
  int spins = 0;
  while (true) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
    if (done) return;
    if (FTK_WAIT_WATCHDOG_NS && (++spins & 15) == 0) {
      if (gtimer_ns() - t0 > FTK_WAIT_WATCHDOG_NS) wait_timeout(what, a, (int)parity);
    }
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

// optional cycle accounting (build with -DFTK_K1_PROF=1): per role, cycles spent per activity
#ifndef FTK_K1_PROF
#define FTK_K1_PROF 0
#endif
enum ProfSlot { PF_SCAN = 0, PF_WFULL, PF_ENQ, PF_WRING, PF_EXWAIT, PF_EXLOAD, PF_EXFACE, PF_EXREC, PF_PRODWAIT, PF_OTHER, PF_N };
struct Prof {
  unsigned long long acc[PF_N];
  unsigned long long t;
  __device__ void start() {
    if (FTK_K1_PROF) t = clock64();
  }
  __device__ void lap(int slot) {
    if (FTK_K1_PROF) {
      const unsigned long long n = clock64();
      acc[slot] += n - t;
      t = n;
    }
  }
};

struct f2 {
  unsigned long long v;
};
__device__ __forceinline__ f2 pack2(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ uint32_t lo32(f2 a) { return (uint32_t)a.v; }
__device__ __forceinline__ uint32_t hi32(f2 a) { return (uint32_t)(a.v >> 32); }
// push the sign bit of `bits` into the low end of W
__device__ __forceinline__ uint32_t push_sign(uint32_t W, uint32_t bits) { return __funnelshift_l(bits, W, 1); }


// |.|-max of four values into the running max (as float bits), NaN-propagating (range check)
__device__ __forceinline__ uint32_t max_abs_bits(uint32_t m, float a, float b, float c, float d) {
  float r = __uint_as_float(m), t1, t2;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(t1) : "f"(fabsf(a)), "f"(fabsf(b)));
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(t2) : "f"(fabsf(c)), "f"(fabsf(d)));
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(t1) : "f"(t1), "f"(t2));
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(r), "f"(t1));
  return __float_as_uint(r);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn get_encode() {
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

// Per-thread cache of the launch geometry of a kernel on the current device: SM count and resident
// blocks per SM (the dynamic-smem attribute is set on the first call).  Keeps the per-call host
// overhead of the persistent launches to a lookup.
struct LaunchGeom {
  int sms = 0, per_sm = 0;
  cudaError_t err = cudaSuccess;
};
template <typename K>
inline LaunchGeom launch_geom(K kern, int threads, size_t smem) {
  thread_local std::unordered_map<unsigned long long, LaunchGeom> cache;
  int dev = 0;
  LaunchGeom g;
  if ((g.err = cudaGetDevice(&dev)) != cudaSuccess) return g;
  const unsigned long long key = reinterpret_cast<unsigned long long>(reinterpret_cast<const void*>(kern)) ^
                                 ((unsigned long long)dev << 56) ^ ((unsigned long long)smem << 40) ^ (unsigned)threads;
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (smem > 48 * 1024 &&
      (g.err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
    return g;
  if ((g.err = cudaDeviceGetAttribute(&g.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return g;
  if ((g.err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g.per_sm, kern, threads, smem)) != cudaSuccess) return g;
  if (g.per_sm < 1) g.per_sm = 1;
  cache[key] = g;
  return g;
}

}  // namespace sm100
}  // namespace ftk
