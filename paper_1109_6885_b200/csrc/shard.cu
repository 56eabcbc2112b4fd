// shard.cu -- small kernels of the sharded Step 1(b).
//
// The merge of U_M with U_D is split by value ranges: U_M is cut at
// superblock-aligned positions a_g, U_D at the first value >= U_M[a_g]
// (k_lower_bound).  Every range merges independently (Step 1(b) is a merge of
// two sorted sequences; its parallel form splits both inputs at
// matching quantiles); the only cross-range quantities are the counts
// of earlier ranges -- |U'| and the number of new values -- which rebase the
// range's translation tables (k_add_u32) and its XC records (k_xc_rebase).
#include <algorithm>

#include "dm_device.cuh"

namespace dm {
namespace {

template <class KT>
__global__ void __launch_bounds__(256) k_lower_bound(const void* __restrict__ sorted, uint64_t n,
                                                     const void* __restrict__ values, uint64_t nv,
                                                     uint64_t* __restrict__ pos) {
  pdl_prologue();
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const auto v = KT::load(values, i);
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (KT::lt(KT::load(sorted, mid), v)) lo = mid + 1; else hi = mid;
  }
  pos[i] = lo;
}

__global__ void __launch_bounds__(256) k_add_u32(uint32_t* __restrict__ x, uint64_t n, uint32_t add) {
  pdl_prologue();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    x[i] += add;
}

// XC record word 0 = R | flag << 31: add to R, keep the flag
__global__ void __launch_bounds__(256) k_xc_rebase(uint2* __restrict__ rec, uint64_t n, uint32_t add) {
  pdl_prologue();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = rec[i].x;
    rec[i].x = (x & 0x80000000u) | ((x & 0x7fffffffu) + add);
  }
}

__global__ void k_set_delta_len(dm_header* hdr, uint64_t n) {
  pdl_prologue(); hdr->delta_dict_len = n; }

unsigned grid_for(uint64_t n) { return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

cudaError_t launch_lower_bound(int key, const void* sorted, uint64_t n, const void* values, uint64_t nv,
                               uint64_t* pos, cudaStream_t st) {
  if (nv == 0) return cudaSuccess;
  const unsigned g = (unsigned)((nv + 255) / 256);
  switch (key) {
    case DM_KEY_U64: launch_k(k_lower_bound<KeyU64>, g, 256, 0, st, sorted, n, values, nv, pos); break;
    case DM_KEY_U32: launch_k(k_lower_bound<KeyU32>, g, 256, 0, st, sorted, n, values, nv, pos); break;
    default: launch_k(k_lower_bound<KeyB16>, g, 256, 0, st, sorted, n, values, nv, pos);
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_add_u32(uint32_t* x, uint64_t n, uint32_t add, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  launch_k(k_add_u32, grid_for(n), 256, 0, st, x, n, add);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_xc_rebase(void* rec, uint64_t n, uint32_t add, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  launch_k(k_xc_rebase, grid_for(n), 256, 0, st, static_cast<uint2*>(rec), n, add);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_set_delta_len(dm_header* hdr, uint64_t n, cudaStream_t st) {
  launch_k(k_set_delta_len, 1, 1, 0, st, hdr, n);
  note_launch();
  return cudaGetLastError();
}

}  // namespace dm
