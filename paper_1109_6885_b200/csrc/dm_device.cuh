// dm_device.cuh -- device-side helpers shared by the dictmerge kernels (sm_100a only).
//
// Key traits (8-byte unsigned integers, 16-byte memcmp-ordered strings), PTX
// wrappers for TMA bulk copies / mbarriers / cache policies, and a warp-parallel
// decoupled look-back used by every single-pass scan in the library (the GPU
// form of the paper's counter array + prefix sum).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "dm_internal.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "dictmerge is written for sm_100a (B200) only"
#endif

// DM_CHECK builds (debugging only, see build.build_check): device-side bounds
// assertions that print and trap.
#ifdef DM_CHECK
#include <cstdio>
#define DM_ASSERT(cond, ...)                                                    \
  do {                                                                          \
    if (!(cond)) {                                                              \
      printf("DM_ASSERT %s:%d block %d thread %d: ", __FILE__, __LINE__, (int)blockIdx.x, (int)threadIdx.x); \
      printf(__VA_ARGS__);                                                      \
      printf("\n");                                                             \
      __trap();                                                                 \
    }                                                                           \
  } while (0)
#else
#define DM_ASSERT(cond, ...) \
  do {                       \
  } while (0)
#endif

namespace dm {

constexpr unsigned FULL = 0xffffffffu;

// Programmatic dependent launch (every kernel is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, see launch_k): a kernel
// is pre-launched while its predecessor in the stream runs; this prologue, the
// first statement of every kernel, waits until the predecessor grid has
// completed and its memory is visible (a no-op without PDL).  Measured: eager
// launches gain (cfg2 Step 1(a) 0.160 -> 0.145 ms, cfg1 0.110 -> 0.091 ms);
// CUDA-graph replay is unchanged.  An early `griddepcontrol.launch_dependents`
// (DM_PDL_TRIGGER=1) made graph replay much slower (cfg2 0.68 -> 1.04 ms), so
// the dependents launch at the predecessor's exit.
#ifndef DM_PDL_TRIGGER
#define DM_PDL_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_prologue() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if DM_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// ----------------------------------------------------------------------------- keys
// 8-byte keys: little-endian u64, unsigned numeric order (reading A5).
struct KeyU64 {
  using K = uint64_t;           // numeric (sortable) form
  static constexpr int kBytes = 8;
  static constexpr int kPasses = 8;
  __device__ __forceinline__ static K load(const void* p, uint64_t i) {
    return __ldg(static_cast<const uint64_t*>(p) + i);
  }
  __device__ __forceinline__ static void store(void* p, uint64_t i, K k) {
    static_cast<uint64_t*>(p)[i] = k;
  }
  // read-only load with an L2 eviction-priority hint (createpolicy); streaming store
  __device__ __forceinline__ static K load_hint(const void* p, uint64_t i, uint64_t pol) {
    K v;
    asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;"
                 : "=l"(v) : "l"(static_cast<const uint64_t*>(p) + i), "l"(pol));
    return v;
  }
  __device__ __forceinline__ static void store_cs(void* p, uint64_t i, K k) {
    __stcs(reinterpret_cast<unsigned long long*>(static_cast<uint64_t*>(p) + i), (unsigned long long)k);
  }
  // coherent (L2) load of a value written by another SM in the same kernel
  __device__ __forceinline__ static K load_cg(const void* p, uint64_t i) {
    return __ldcg(static_cast<const uint64_t*>(p) + i);
  }
  __device__ __forceinline__ static uint32_t digit(K k, int pass) {
    return (uint32_t)(k >> (8 * pass)) & 0xffu;
  }
  __device__ __forceinline__ static bool lt(K a, K b) { return a < b; }
  __device__ __forceinline__ static bool eq(K a, K b) { return a == b; }
  __device__ __forceinline__ static bool le(K a, K b) { return a <= b; }
  __device__ __forceinline__ static K shfl_up(K v, unsigned d) { return __shfl_up_sync(0xffffffffu, v, d); }
  // raw input and numeric workspace layouts coincide for u64 keys
  __device__ __forceinline__ static K ld_any(const void* p, uint64_t i, bool /*raw*/) {
    return static_cast<const uint64_t*>(p)[i];
  }
};

// 4-byte keys (NEXT4, the paper's E = 4 of Fig 8): little-endian u32,
// unsigned numeric order.
struct KeyU32 {
  using K = uint32_t;
  static constexpr int kBytes = 4;
  static constexpr int kPasses = 4;
  __device__ __forceinline__ static K load(const void* p, uint64_t i) {
    return __ldg(static_cast<const uint32_t*>(p) + i);
  }
  __device__ __forceinline__ static void store(void* p, uint64_t i, K k) { static_cast<uint32_t*>(p)[i] = k; }
  __device__ __forceinline__ static K load_hint(const void* p, uint64_t i, uint64_t pol) {
    K v;
    asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v) : "l"(static_cast<const uint32_t*>(p) + i), "l"(pol));
    return v;
  }
  __device__ __forceinline__ static void store_cs(void* p, uint64_t i, K k) { __stcs(static_cast<uint32_t*>(p) + i, k); }
  __device__ __forceinline__ static K load_cg(const void* p, uint64_t i) {
    return __ldcg(static_cast<const uint32_t*>(p) + i);
  }
  __device__ __forceinline__ static uint32_t digit(K k, int pass) { return (k >> (8 * pass)) & 0xffu; }
  __device__ __forceinline__ static bool lt(K a, K b) { return a < b; }
  __device__ __forceinline__ static bool eq(K a, K b) { return a == b; }
  __device__ __forceinline__ static bool le(K a, K b) { return a <= b; }
  __device__ __forceinline__ static K shfl_up(K v, unsigned d) { return __shfl_up_sync(0xffffffffu, v, d); }
  __device__ __forceinline__ static K ld_any(const void* p, uint64_t i, bool /*raw*/) {
    return static_cast<const uint32_t*>(p)[i];
  }
};

// 16-byte keys: raw bytes compared with memcmp (reading A5).  The numeric form
// is the big-endian (hi, lo) pair, so (hi, lo) lexicographic == memcmp order.
struct K128 {
  uint64_t hi, lo;
};
struct KeyB16 {
  using K = K128;
  static constexpr int kBytes = 16;
  static constexpr int kPasses = 16;
  __device__ __forceinline__ static uint64_t bswap(uint64_t x) {
    uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    return ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32) | __byte_perm(hi, 0, 0x0123);
  }
  __device__ __forceinline__ static K load(const void* p, uint64_t i) {
    const ulonglong2 v = __ldg(static_cast<const ulonglong2*>(p) + i);
    return K{bswap(v.x), bswap(v.y)};
  }
  __device__ __forceinline__ static void store(void* p, uint64_t i, K k) {
    static_cast<ulonglong2*>(p)[i] = make_ulonglong2(bswap(k.hi), bswap(k.lo));
  }
  __device__ __forceinline__ static K load_hint(const void* p, uint64_t i, uint64_t pol) {
    uint64_t x, y;
    asm volatile("ld.global.nc.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;"
                 : "=l"(x), "=l"(y) : "l"(static_cast<const ulonglong2*>(p) + i), "l"(pol));
    return K{bswap(x), bswap(y)};
  }
  __device__ __forceinline__ static void store_cs(void* p, uint64_t i, K k) {
    const uint64_t a = bswap(k.hi), b = bswap(k.lo);
    __stcs(reinterpret_cast<uint4*>(static_cast<ulonglong2*>(p) + i),
           make_uint4((uint32_t)a, (uint32_t)(a >> 32), (uint32_t)b, (uint32_t)(b >> 32)));
  }
  __device__ __forceinline__ static K load_cg(const void* p, uint64_t i) {
    const ulonglong2 v = __ldcg(static_cast<const ulonglong2*>(p) + i);
    return K{bswap(v.x), bswap(v.y)};
  }
  __device__ __forceinline__ static uint32_t digit(K k, int pass) {
    return pass < 8 ? (uint32_t)(k.lo >> (8 * pass)) & 0xffu : (uint32_t)(k.hi >> (8 * (pass - 8))) & 0xffu;
  }
  __device__ __forceinline__ static bool lt(K a, K b) { return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo); }
  __device__ __forceinline__ static bool eq(K a, K b) { return a.hi == b.hi && a.lo == b.lo; }
  __device__ __forceinline__ static K shfl_up(K v, unsigned d) {
    return K128{__shfl_up_sync(0xffffffffu, v.hi, d), __shfl_up_sync(0xffffffffu, v.lo, d)};
  }
  __device__ __forceinline__ static bool le(K a, K b) { return !lt(b, a); }
  // one 16-byte load; raw (input) layout converted to the numeric (hi, lo) form
  __device__ __forceinline__ static K ld_any(const void* p, uint64_t i, bool raw) {
    const ulonglong2 v = static_cast<const ulonglong2*>(p)[i];
    return raw ? K{bswap(v.x), bswap(v.y)} : K{v.x, v.y};
  }
};

// Numeric-form storage used inside the workspace (ping-pong sort buffers).
template <class KT>
struct NumStore;
template <>
struct NumStore<KeyU64> {
  __device__ __forceinline__ static uint64_t ld(const void* p, uint64_t i) { return static_cast<const uint64_t*>(p)[i]; }
  __device__ __forceinline__ static void st(void* p, uint64_t i, uint64_t k) { static_cast<uint64_t*>(p)[i] = k; }
};
template <>
struct NumStore<KeyU32> {
  __device__ __forceinline__ static uint32_t ld(const void* p, uint64_t i) { return static_cast<const uint32_t*>(p)[i]; }
  __device__ __forceinline__ static void st(void* p, uint64_t i, uint32_t k) { static_cast<uint32_t*>(p)[i] = k; }
};
template <>
struct NumStore<KeyB16> {
  __device__ __forceinline__ static K128 ld(const void* p, uint64_t i) {
    ulonglong2 v = static_cast<const ulonglong2*>(p)[i];
    return K128{v.x, v.y};
  }
  __device__ __forceinline__ static void st(void* p, uint64_t i, K128 k) {
    static_cast<ulonglong2*>(p)[i] = make_ulonglong2(k.hi, k.lo);
  }
};

// ----------------------------------------------------------------------------- misc
__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ uint32_t umin32(uint32_t a, uint32_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ uint32_t umax32(uint32_t a, uint32_t b) { return a > b ? a : b; }
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
// Shifts that clamp (PTX semantics: amounts >= 32 give 0), so callers can use
// data-dependent amounts without C++ undefined behaviour.
__device__ __forceinline__ uint32_t shl32(uint32_t x, uint32_t s) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
  return r;
}
__device__ __forceinline__ uint32_t shr32(uint32_t x, uint32_t s) {
  uint32_t r;
  asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
  return r;
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// ----------------------------------------------------------------- decoupled look-back
// Status word (u64): bits 63..62 = flag (0 empty, 1 aggregate, 2 inclusive prefix),
// bits 61..0 = value.  Called by ALL 32 lanes of one warp; returns the exclusive
// prefix of `tile` (same value in every lane).  Tiles must be claimed in
// increasing order (dynamic tile ids) so predecessors always make progress.
constexpr uint64_t LB_AGG = 1ull << 62;
constexpr uint64_t LB_PRE = 2ull << 62;
constexpr uint64_t LB_VAL = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t lookback_exclusive(uint64_t* status, uint64_t tile, uint64_t aggregate) {
  const unsigned lane = lane_id();
  if (tile == 0) {
    if (lane == 0) st_volatile_u64(&status[0], LB_PRE | aggregate);
    return 0;
  }
  if (lane == 0) st_volatile_u64(&status[tile], LB_AGG | aggregate);
  uint64_t excl = 0;
  int64_t base = (int64_t)tile - 1;
  while (true) {
    const int64_t idx = base - (int64_t)lane;
    uint64_t s = idx >= 0 ? ld_volatile_u64(&status[idx]) : LB_PRE;
    while (__any_sync(FULL, (s >> 62) == 0)) {
      if ((s >> 62) == 0) s = ld_volatile_u64(&status[idx]);
    }
    const unsigned pmask = __ballot_sync(FULL, (s >> 62) == 2);
    if (pmask) {
      const unsigned first = __ffs(pmask) - 1;  // nearest tile holding an inclusive prefix
      excl += warp_sum<uint64_t>(lane <= first ? (s & LB_VAL) : 0);
      break;
    }
    excl += warp_sum<uint64_t>(s & LB_VAL);
    base -= 32;
  }
  if (lane == 0) st_volatile_u64(&status[tile], LB_PRE | (excl + aggregate));
  return excl;
}

// Block-wide exclusive scan of one u32 per thread (NT threads, NT/32 warps).
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp /*[NT/32]*/, uint32_t& total) {
  const unsigned lane = lane_id(), w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= (unsigned)o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < NT / 32 ? s_warp[lane] : 0;
    uint32_t u = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(FULL, u, o);
      if (lane >= (unsigned)o) u += y;
    }
    if (lane < NT / 32) s_warp[lane] = u - t;  // exclusive warp offsets
    if (lane == NT / 32 - 1) s_warp[NT / 32] = u;
  }
  __syncthreads();
  total = s_warp[NT / 32];
  const uint32_t r = s_warp[w] + x - v;
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------ TMA / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// Shared-memory loads by 32-bit shared address; the predicated form compiles to
// one predicated LDS (no branch) and yields 0 when `pred` is false.  Only for
// data that is read-only after a barrier (the address depends on loaded data,
// so the compiler cannot hoist these above the barrier).
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32_if(uint32_t a, bool pred) {
  uint32_t v = 0;
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.u32 %0, [%1];\n}" : "+r"(v) : "r"(a), "r"((uint32_t)pred));
  return v;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_parity(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_parity(bar, parity)) {
  }
}
// As mbar_wait_parity, with a suspend-time hint: the thread sleeps in the
// try_wait until the phase completes or ~`ns` elapse, instead of re-issuing
// it (each retry costs issue slots the streaming kernels need).
__device__ __forceinline__ void mbar_wait_parity_sleep(uint64_t* bar, uint32_t parity, uint32_t ns = 20000) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Bulk (non-tensor) TMA copy global -> shared, completing on an mbarrier.
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// Bulk TMA copy shared -> global (bulk-group completion).
__device__ __forceinline__ void tma_store_1d(void* dst_gmem, const void* src_smem, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst_gmem),
               "r"(smem_u32(src_smem)), "r"(bytes), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void tma_store_wait_all() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Read-only gather with an L2 evict-last hint (translation tables).
__device__ __forceinline__ uint32_t ld_gather_u32(const uint32_t* p, uint64_t policy) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy));
  return v;
}

}  // namespace dm
