// microbench.cu -- B200 memory microbenchmarks that set the Step-2 bounds (SURVEY K8';
// the GPU analogue of the paper's streaming / random bandwidth micro-benchmarks).
//   copy      : 16-byte vector copy, GB/s (read + write bytes)
//   gather    : random 4-byte gathers from tables of 4 KB .. 4 GB, G gathers/s
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__global__ void k_copy(const int4* __restrict__ a, int4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

__device__ __forceinline__ uint32_t hash32(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return (uint32_t)x;
}

// each thread does ITER independent gathers per round (MLP), mask = table entries - 1 (power of 2)
template <int ITER>
__global__ void k_gather(const uint32_t* __restrict__ t, uint32_t mask, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
  for (size_t i = tid; i < n; i += nt * ITER) {
    uint32_t v[ITER];
#pragma unroll
    for (int k = 0; k < ITER; ++k) v[k] = __ldg(t + (hash32(i + k * nt) & mask));
#pragma unroll
    for (int k = 0; k < ITER; ++k) acc += v[k];
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const size_t cbytes = 2ull << 30;
  int4 *x, *y; CK(cudaMalloc(&x, cbytes)); CK(cudaMalloc(&y, cbytes));
  cudaMemset(x, 1, cbytes);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); k_copy<<<sms * 8, 512>>>(x, y, cbytes / 16); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  printf("{\"copy_GBps\": %.1f}\n", 2.0 * cbytes / best / 1e6);
  cudaFree(y);
  uint32_t* out; CK(cudaMalloc(&out, 4));
  const size_t n = 1ull << 28;  // gathers per run
  for (uint64_t tb = 1ull << 12; tb <= (4ull << 30); tb <<= 1) {
    const uint32_t* t = reinterpret_cast<const uint32_t*>(x);
    uint32_t* big = nullptr;
    if (tb > cbytes) { CK(cudaMalloc(&big, tb)); cudaMemset(big, 1, tb); t = big; }
    const uint32_t mask = (uint32_t)(tb / 4 - 1);
    float bm = 1e9;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(a); k_gather<8><<<sms * 8, 256>>>(t, mask, n, out); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < bm) bm = ms;
    }
    printf("{\"table_bytes\": %llu, \"gathers_per_s\": %.3e, \"sector_GBps\": %.1f}\n", (unsigned long long)tb,
           n / (bm * 1e-3), n * 32.0 / (bm * 1e-3) / 1e9);
    if (big) cudaFree(big);
  }
  CK(cudaGetLastError());
  return 0;
}
