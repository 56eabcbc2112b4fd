// microbench_tma.cu -- random lookups by TMA tile::gather4 and from shared memory (B200).
// Decides where Step 2's translation-table lookups should come from when the table
// does not fit on chip (cfg2: 40 MB X_M).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_tma microbench_tma.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return (uint32_t)x;
}
__device__ __forceinline__ uint32_t smem_u32p(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Each thread issues one gather4 (4 random 16-B rows) per round into its own 64-B slot.
__global__ void k_tma_gather4(const __grid_constant__ CUtensorMap tm, uint32_t nrows, int rounds, uint32_t* out,
                              int* err, uint32_t expect_per_thread) {
  __shared__ __align__(128) uint32_t buf[2][128 * 32];
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32p(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t acc = 0;
  const uint64_t base = (blockIdx.x * 128ull + threadIdx.x) * 0x9E3779B97F4A7C15ull;
  for (int r = 0; r < rounds; ++r) {
    const int s = r & 1;
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32p(&bar[s])),
                   "r"(128 * expect_per_thread));
    __syncthreads();
    int32_t rows[4];
    for (int k = 0; k < 4; ++k) rows[k] = (int32_t)(hash32(base + r * 4 + k) % nrows);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(smem_u32p(&buf[s][threadIdx.x * 32])),
        "l"(&tm), "r"(0), "r"(rows[0]), "r"(rows[1]), "r"(rows[2]), "r"(rows[3]), "r"(smem_u32p(&bar[s]))
        : "memory");
    uint32_t ok = 0;
    for (int spin = 0; spin < (1 << 20) && !ok; ++spin)
      asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0,1,0,P;}"
                   : "=r"(ok) : "r"(smem_u32p(&bar[s])), "r"((uint32_t)((r >> 1) & 1)) : "memory");
    if (!ok) { atomicExch(err, 1); return; }
    acc += buf[s][threadIdx.x * 32] + buf[s][threadIdx.x * 32 + 4] + buf[s][threadIdx.x * 32 + 8] +
           buf[s][threadIdx.x * 32 + 12];
    __syncthreads();
  }
  if (acc == 0x12345678) out[0] = acc;
}

// Random lookups into a shared-memory table of `entries` u32 (per-lane random index).
__global__ void k_smem_lookup(const uint32_t* __restrict__ t, uint32_t entries, int rounds, uint32_t* out) {
  extern __shared__ uint32_t st[];
  for (uint32_t i = threadIdx.x; i < entries; i += blockDim.x) st[i] = t[i];
  __syncthreads();
  uint32_t acc = 0, x = hash32(blockIdx.x * 1024 + threadIdx.x);
  for (int r = 0; r < rounds; ++r) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x = x * 1664525u + 1013904223u;
      acc += st[(x >> 8) % entries];
    }
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  uint32_t* out; int* err; CK(cudaMalloc(&out, 4)); CK(cudaMalloc(&err, 4));
  for (uint32_t expect : {64u}) {
    for (uint64_t tb : {4ull << 20, 40ull << 20, 4ull << 30}) {
      cudaMemset(err, 0, 4);
      uint32_t* t; CK(cudaMalloc(&t, tb)); cudaMemset(t, 1, tb);
      CUtensorMap tm;
      const cuuint64_t gdim[2] = {4, tb / 16};
      const cuuint64_t gstr[1] = {16};
      const cuuint32_t box[2] = {4, 1};
      const cuuint32_t est[2] = {1, 1};
      CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, t, gdim, gstr, box, est,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) { printf("{\"tma_encode_error\": %d}\n", (int)cr); return 1; }
      const int rounds = 64, blocks = sms * 8;
      float bm = 1e9;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        k_tma_gather4<<<blocks, 128>>>(tm, (uint32_t)(tb / 16), rounds, out, err, expect);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < bm) bm = ms;
      }
      int herr; cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost);
      const double rows = (double)blocks * 128 * rounds * 4;
      printf("{\"tma_gather4_table_bytes\": %llu, \"rows_per_s\": %.3e, \"err\": %d}\n", (unsigned long long)tb,
             rows / (bm * 1e-3), herr);
      fflush(stdout);
      cudaFree(t);
    }
  }
  for (uint32_t entries : {1024u, 16384u, 49152u}) {
    uint32_t* t; CK(cudaMalloc(&t, entries * 4)); cudaMemset(t, 1, entries * 4);
    CK(cudaFuncSetAttribute(k_smem_lookup, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    const int rounds = 4096, blocks = sms * 1;
    float bm = 1e9;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(a); k_smem_lookup<<<blocks, 1024, entries * 4>>>(t, entries, rounds, out); cudaEventRecord(b);
      CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < bm) bm = ms;
    }
    printf("{\"smem_lookup_entries\": %u, \"lookups_per_s\": %.3e}\n", entries,
           (double)blocks * 1024 * rounds * 8 / (bm * 1e-3));
    cudaFree(t);
  }
  CK(cudaGetLastError());
  return 0;
}
