// microbench_gather2.cu -- random 4-byte lookups from a 40 MB L2-resident table (cfg2's X_M):
//   (a) LSU gather, default caching        (b) LSU gather, L1::no_allocate
//   (c) TMA tile::gather4, deep pipeline (each warp keeps 8 gather4 batches in flight)
//   (d) (a) and (c) concurrently in one kernel (half the warps each)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_gather2 microbench_gather2.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return (uint32_t)x;
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool NOALLOC>
__device__ __forceinline__ uint32_t ldg(const uint32_t* p) {
  uint32_t v;
  if (NOALLOC)
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <bool NOALLOC>
__device__ void lsu_part(const uint32_t* t, uint32_t n, uint64_t seed, int iters, uint32_t& acc) {
  for (int r = 0; r < iters; ++r) {
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ldg<NOALLOC>(t + hash32(seed + r * 8 + k) % n);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k];
  }
}

// TMA part: a warp owns NSLOT slots of 32 lanes x 64 B; lane l issues one gather4 per slot.
constexpr int NSLOT = 4;
__device__ void tma_part(const CUtensorMap* tm, uint32_t nrows, uint64_t seed, int iters, uint32_t& acc,
                         uint32_t* wbuf /*NSLOT*32*32 u32*/, uint64_t* bars /*NSLOT*/, int* err) {
  const unsigned lane = threadIdx.x & 31;
  if (lane == 0)
    for (int s = 0; s < NSLOT; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  auto issue = [&](int r) {
    const int s = r % NSLOT;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[s])),
                   "r"(32 * 64));
    __syncwarp();
    int32_t rows[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) rows[k] = (int32_t)(hash32(seed + r * 4 + k) % nrows);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(su32(&wbuf[(s * 32 + lane) * 32])),
        "l"(tm), "r"(0), "r"(rows[0]), "r"(rows[1]), "r"(rows[2]), "r"(rows[3]), "r"(su32(&bars[s]))
        : "memory");
  };
  for (int r = 0; r < NSLOT && r < iters; ++r) issue(r);
  for (int r = 0; r < iters; ++r) {
    const int s = r % NSLOT;
    uint32_t ok = 0;
    for (int spin = 0; spin < (1 << 22) && !ok; ++spin)
      asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0,1,0,P;}"
                   : "=r"(ok) : "r"(su32(&bars[s])), "r"((uint32_t)((r / NSLOT) & 1)) : "memory");
    if (!ok) { atomicExch(err, 1); return; }
    acc += wbuf[(s * 32 + lane) * 32] + wbuf[(s * 32 + lane) * 32 + 4];
    __syncwarp();
    if (r + NSLOT < iters) issue(r + NSLOT);
  }
}

// mode 0: LSU, 1: LSU no_allocate, 2: TMA, 3: half LSU half TMA (by warp parity)
__global__ void __launch_bounds__(256) k_mix(const uint32_t* t, uint32_t n, const __grid_constant__ CUtensorMap tm,
                                             int mode, int lsu_iters, int tma_iters, uint32_t* out, int* err) {
  extern __shared__ __align__(128) uint32_t sm[];
  __shared__ __align__(8) uint64_t bars[8][NSLOT];
  const unsigned w = threadIdx.x >> 5;
  uint32_t acc = 0;
  const uint64_t seed = (blockIdx.x * 256ull + threadIdx.x) * 0x9E3779B97F4A7C15ull;
  const bool use_tma = mode == 2 || (mode == 3 && (w & 1));
  if (use_tma)
    tma_part(&tm, n / 4, seed, tma_iters, acc, sm + w * NSLOT * 32 * 32, bars[w], err);
  else if (mode == 1)
    lsu_part<true>(t, n, seed, lsu_iters, acc);
  else
    lsu_part<false>(t, n, seed, lsu_iters, acc);
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  uint32_t* out; int* err; CK(cudaMalloc(&out, 4)); CK(cudaMalloc(&err, 4)); cudaMemset(err, 0, 4);
  const uint64_t tb = 40ull << 20;
  const uint32_t n = (uint32_t)(tb / 4);
  uint32_t* t; CK(cudaMalloc(&t, tb)); cudaMemset(t, 1, tb);
  CUtensorMap tm;
  const cuuint64_t gdim[2] = {4, tb / 16};
  const cuuint64_t gstr[1] = {16};
  const cuuint32_t box[2] = {4, 1};
  const cuuint32_t est[2] = {1, 1};
  if (cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, t, gdim, gstr, box, est,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  const size_t smem = 8 * NSLOT * 32 * 32 * 4;  // 8 warps x NSLOT x 32 lanes x 128 B = 256 KB too big -> use 4 slots
  (void)smem;
  const size_t dsmem = 8 * NSLOT * 32 * 32 * 4 / 2;
  CK(cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int blocks = sms * 1;
  for (int mode = 0; mode < 4; ++mode) {
    const int lsu_iters = 256, tma_iters = 512;
    float bm = 1e9;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(a);
      k_mix<<<blocks, 256, 8 * NSLOT * 32 * 32 * 4>>>(
          t, n, tm, mode, lsu_iters, tma_iters, out, err);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < bm) bm = ms;
    }
    double lookups = 0;
    for (int w = 0; w < 8; ++w) {
      const bool tma = mode == 2 || (mode == 3 && (w & 1));
      lookups += tma ? 32.0 * tma_iters * 4 : 32.0 * lsu_iters * 8;
    }
    lookups *= blocks;
    int herr; cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost);
    printf("{\"mode\": %d, \"lookups_per_s\": %.3e, \"err\": %d}\n", mode, lookups / (bm * 1e-3), herr);
    fflush(stdout);
  }
  (void)dsmem;
  return 0;
}
