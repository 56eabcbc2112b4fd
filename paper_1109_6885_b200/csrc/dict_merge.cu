// dict_merge.cu -- Step 1(b) and Step 2(a) on the GPU: merge U_M with U_D.
//
// Paper, Step 1(b): walk the two sorted dictionaries with two
// pointers, append the smaller value, record its output index in X_M or X_D;
// equal heads are appended once and both tables get the same index.  Parallel
// form: split both inputs at quantiles, merge locally while dropping
// the duplicate that can straddle a split, count the uniques per thread,
// prefix-sum the counts, then re-merge writing at the offsets.
//
// GPU form (one pass instead of the paper's three):
//   k_partition  merge-path co-ranks at every 2048-element diagonal (the paper's
//                quantile split, [8][5] in P:302)
//   k_merge      per tile: stage both ranges in shared memory, per-thread
//                co-rank + 8-step serial merge; a U_D element equal to the U_M
//                element immediately before it in merged order is the duplicate
//                (ties take U_M first -- the GPU form of P:304's boundary check);
//                duplicate counts are prefix-summed across tiles with a
//                decoupled look-back (P:306's counter array, done in one pass);
//                U', X_M, X_D are staged in shared memory and written coalesced.
//                The tile that ends the merge writes |U'| and b' = w(|U'|)
//                (Eq 4) to the result header.
#include "dm_device.cuh"

namespace dm {
namespace {

__device__ __forceinline__ uint32_t dev_width(uint64_t n) { return n <= 1 ? 1u : 64u - __clzll(n - 1); }

template <class KT>
__device__ __forceinline__ uint64_t corank(const void* A, uint64_t nA, const void* B, uint64_t nB, uint64_t d) {
  // Number of U_M elements among the first d merged elements (U_M first on ties).
  uint64_t lo = d > nB ? d - nB : 0, hi = d < nA ? d : nA;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (KT::le(KT::load(A, mid), KT::load(B, d - mid - 1)))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

template <class KT>
__global__ void __launch_bounds__(256) k_partition(const void* __restrict__ A, uint64_t nA,
                                                   const void* __restrict__ B, const dm_header* __restrict__ hdr,
                                                   uint64_t nparts, uint64_t* __restrict__ part) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= nparts) return;
  const uint64_t nB = hdr->delta_dict_len;
  const uint64_t total = nA + nB;
  const uint64_t d = umin64(t * (uint64_t)kMergeTile, total);
  part[t] = corank<KT>(A, nA, B, nB, d);
}

template <class KT>
__global__ void __launch_bounds__(kMergeThreads) k_merge(const void* __restrict__ A, uint64_t nA,
                                                         const void* __restrict__ B, const uint64_t* __restrict__ part,
                                                         void* __restrict__ U, uint32_t* __restrict__ XM,
                                                         uint32_t* __restrict__ XD, uint64_t* status,
                                                         uint32_t* counter, dm_header* hdr) {
  using K = typename KT::K;
  constexpr int T = kMergeTile;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* s_in = reinterpret_cast<K*>(smem_raw);                       // [T + 1]: A[i0-1 .. i1) then B[j0 .. j1)
  K* s_out = s_in + (T + 1);                                        // [T] U' staging
  uint32_t* s_x = reinterpret_cast<uint32_t*>(s_out + T);          // [T] X_M then X_D staging
  __shared__ uint32_t s_warp[kMergeThreads / 32 + 1];
  __shared__ uint64_t s_excl;
  __shared__ uint32_t s_tile;
  __shared__ int s_unsorted;

  if (threadIdx.x == 0) {
    s_tile = atomicAdd(counter, 1u);
    s_unsorted = 0;
  }
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t nB = hdr->delta_dict_len;
  const uint64_t total = nA + nB;
  const uint64_t d0 = tile * T;
  if (d0 >= total && tile != 0) return;
  const uint64_t d1 = umin64(d0 + T, total);
  const uint64_t i0 = part[tile], i1 = part[tile + 1];
  const uint64_t j0 = d0 - i0, j1 = d1 - i1;
  const uint32_t na = (uint32_t)(i1 - i0), nb = (uint32_t)(j1 - j0);
  K* sA = s_in;           // sA[k] = A[i0 + k - 1], k = 0 .. na
  K* sB = s_in + na + 1;  // sB[k] = B[j0 + k]
  for (uint32_t k = threadIdx.x; k <= na; k += kMergeThreads) {
    if (k > 0 || i0 > 0) sA[k] = KT::load(A, i0 + k - 1);
  }
  for (uint32_t k = threadIdx.x; k < nb; k += kMergeThreads) sB[k] = KT::load(B, j0 + k);
  __syncthreads();
  // Strictly-increasing check of U_M over the pairs this tile owns.
  for (uint32_t k = threadIdx.x; k + 1 <= na; k += kMergeThreads) {
    if ((k > 0 || i0 > 0) && !KT::lt(sA[k], sA[k + 1])) s_unsorted = 1;
  }

  // Per-thread co-rank inside the tile, then an ITEMS-step serial merge.
  const uint32_t n_loc = na + nb;
  const uint32_t dd0 = umin32(threadIdx.x * kMergeItems, n_loc);
  uint32_t lo = dd0 > nb ? dd0 - nb : 0, hi = dd0 < na ? dd0 : na;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (KT::le(sA[mid + 1], sB[dd0 - mid - 1]))
      lo = mid + 1;
    else
      hi = mid;
  }
  uint32_t ia = lo, ib = dd0 - lo;
  uint32_t rec[kMergeItems];  // bit31: from B; bit30: duplicate; low bits: local index
  uint32_t ndup = 0;
#pragma unroll
  for (int k = 0; k < kMergeItems; ++k) {
    rec[k] = 0xffffffffu;
    if (dd0 + k < n_loc) {
      const bool takeA = ib >= nb || (ia < na && KT::le(sA[ia + 1], sB[ib]));
      if (takeA) {
        rec[k] = ia++;
      } else {
        const bool dup = (i0 + ia > 0) && KT::eq(sA[ia], sB[ib]);
        rec[k] = (1u << 31) | ((uint32_t)dup << 30) | ib++;
        ndup += dup;
      }
    }
  }
  uint32_t tile_dups;
  const uint32_t texcl = block_exclusive_scan<kMergeThreads>(ndup, s_warp, tile_dups);
  if (threadIdx.x < 32) {
    const uint64_t e = lookback_exclusive(status, tile, tile_dups);
    if (threadIdx.x == 0) s_excl = e;
  }
  __syncthreads();
  const uint64_t D0 = s_excl;
  const uint64_t out_base = d0 - D0;  // first U' index this tile writes
  uint64_t dups_before = D0 + texcl;
#pragma unroll
  for (int k = 0; k < kMergeItems; ++k) {
    if (rec[k] == 0xffffffffu) continue;
    const uint64_t p = d0 + dd0 + k;
    if (rec[k] & (1u << 31)) {
      const uint32_t jb = rec[k] & 0x3fffffffu;
      if (rec[k] & (1u << 30)) {
        s_x[na + jb] = (uint32_t)(p - 1 - dups_before);  // same index as its U_M twin
        ++dups_before;
      } else {
        const uint64_t o = p - dups_before;
        s_out[o - out_base] = sB[jb];
        s_x[na + jb] = (uint32_t)o;
      }
    } else {
      const uint64_t o = p - dups_before;
      s_out[o - out_base] = sA[rec[k] + 1];
      s_x[rec[k]] = (uint32_t)o;
    }
  }
  __syncthreads();
  const uint32_t n_out = (uint32_t)(n_loc - tile_dups);
  for (uint32_t k = threadIdx.x; k < n_out; k += kMergeThreads) KT::store(U, out_base + k, s_out[k]);
  for (uint32_t k = threadIdx.x; k < na; k += kMergeThreads) XM[i0 + k] = s_x[k];
  for (uint32_t k = threadIdx.x; k < nb; k += kMergeThreads) XD[j0 + k] = s_x[na + k];
  if (threadIdx.x == 0) {
    if (s_unsorted) atomicMin(&hdr->status, (int)DM_E_UNSORTED);
    if (d1 == total) {
      const uint64_t m = total - (D0 + tile_dups);
      hdr->merged_dict_len = m;
      hdr->merged_bits = dev_width(m);
      if (m > (1ull << 32)) atomicMin(&hdr->status, (int)DM_E_TOO_WIDE);
    }
  }
}

template <class KT>
cudaError_t run(const dm_column_in* in, char* ws, const WsLayout& L, const void* udict, void* U, uint32_t* xm,
                uint32_t* xd, dm_header* hdr, cudaStream_t st) {
  using K = typename KT::K;
  const uint64_t nparts = L.ntiles_merge + 1;
  uint64_t* part = reinterpret_cast<uint64_t*>(ws + L.part);
  k_partition<KT><<<(unsigned)((nparts + 255) / 256), 256, 0, st>>>(in->main_dict, in->dict_len, udict, hdr, nparts,
                                                                      part);
  const size_t dsmem = sizeof(K) * (2 * kMergeTile + 1) + sizeof(uint32_t) * kMergeTile;
  cudaFuncSetAttribute(k_merge<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem);
  k_merge<KT><<<(unsigned)L.ntiles_merge, kMergeThreads, dsmem, st>>>(
      in->main_dict, in->dict_len, udict, part, U, xm, xd, reinterpret_cast<uint64_t*>(ws + L.status_merge),
      reinterpret_cast<uint32_t*>(ws + L.counters) + CNT_MERGE, hdr);
  note_launch(2);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_dictionary_merge(const dm_column_in* in, const dm_column_out* out, char* ws, const WsLayout& L,
                                    const void* udict, uint32_t* xm, uint32_t* xd, dm_header* hdr, cudaStream_t st) {
  return in->key == DM_KEY_U64 ? run<KeyU64>(in, ws, L, udict, out->merged_dict, xm, xd, hdr, st)
                               : run<KeyB16>(in, ws, L, udict, out->merged_dict, xm, xd, hdr, st);
}

}  // namespace dm
