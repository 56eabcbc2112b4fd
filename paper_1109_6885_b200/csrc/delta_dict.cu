// delta_dict.cu -- Step 1(a) on the GPU: the delta dictionary U_D and per-tuple ranks.
//
// Paper: "Extracting the unique values from the delta partition D to form the
// corresponding sorted dictionary U_D" and "replace the uncompressed
// values in the delta partition with their respective indices in the
// dictionary".  The paper gets U_D in order by walking the leaves of
// the CSB+ tree it maintains at insert time; here the delta is a
// raw insertion-order array (BASELINE.json north_star), so the sort happens at
// merge time:
//
//   k_hist       one read of D: all digit histograms (8 or 16 passes) at once
//   k_plan       exclusive digit offsets per pass; passes whose digit is constant
//                over every key are skipped (device-decided, no host sync)
//   k_onesweep   one LSD pass: stable warp-multisplit ranking in shared memory,
//                per-digit decoupled look-back across tiles, coalesced scatter
//   k_unique     head flags over the sorted keys, single-pass scan (look-back) ->
//                U_D[rank] and r[original index] = rank
#include "dm_device.cuh"

namespace dm {
namespace {

template <class KT>
__global__ void __launch_bounds__(256) k_hist(const void* __restrict__ D, uint64_t n, uint32_t* __restrict__ hist) {
  constexpr int P = KT::kPasses;
  __shared__ uint32_t s_h[P][256];
  for (int i = threadIdx.x; i < P * 256; i += blockDim.x) (&s_h[0][0])[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const typename KT::K k = KT::load(D, i);
#pragma unroll
    for (int p = 0; p < P; ++p) atomicAdd(&s_h[p][KT::digit(k, p)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P * 256; i += blockDim.x) {
    const uint32_t c = (&s_h[0][0])[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

__global__ void __launch_bounds__(256) k_plan(const uint32_t* __restrict__ hist, uint64_t n, int npass,
                                              SortPlan* __restrict__ plan) {
  __shared__ uint32_t s_warp[9];
  __shared__ int s_active[16];
  const int t = threadIdx.x;
  for (int p = 0; p < npass; ++p) {
    const uint32_t c = hist[p * 256 + t];
    const int full = __syncthreads_or(c == (uint32_t)n);
    uint32_t total;
    const uint32_t ex = block_exclusive_scan<256>(c, s_warp, total);
    plan->digit_base[p][t] = ex;
    if (t == 0) s_active[p] = !full;
  }
  __syncthreads();
  if (t == 0) {
    int cur = SEL_INPUT, na = 0;
    for (int p = 0; p < 16; ++p) {
      const int a = p < npass ? s_active[p] : 0;
      plan->active[p] = a;
      plan->src[p] = cur;
      if (a) {
        const int nxt = (cur == SEL_BUF0) ? SEL_BUF1 : SEL_BUF0;
        plan->dst[p] = nxt;
        cur = nxt;
        ++na;
      } else {
        plan->dst[p] = cur;
      }
    }
    plan->final_sel = cur;
    plan->n_active = na;
  }
}

// One stable LSD radix pass over (key, original-index) pairs.
template <class KT, int ITEMS>
__global__ void __launch_bounds__(kSortThreads) k_onesweep(const void* __restrict__ D, void* kbuf0, void* kbuf1,
                                                          uint32_t* vbuf0, uint32_t* vbuf1, uint64_t n, int pass,
                                                          const SortPlan* __restrict__ plan, uint32_t* status,
                                                          uint32_t* counter) {
  using K = typename KT::K;
  constexpr int W = kSortThreads / 32;
  constexpr int TILE = kSortThreads * ITEMS;
  if (!plan->active[pass]) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* s_keys = reinterpret_cast<K*>(smem_raw);
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(smem_raw + sizeof(K) * TILE);
  __shared__ uint32_t s_whist[W][257];
  __shared__ uint32_t s_bstart[256];
  __shared__ uint32_t s_gofs[256];
  __shared__ uint32_t s_warp[W + 1];
  __shared__ uint32_t s_tile;

  const unsigned lane = lane_id(), w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < W * 257; i += kSortThreads) (&s_whist[0][0])[i] = 0;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * TILE;
  const int src = plan->src[pass];
  const void* ksrc = src == SEL_BUF0 ? kbuf0 : kbuf1;
  const uint32_t* vsrc = src == SEL_BUF0 ? vbuf0 : vbuf1;
  void* kdst = plan->dst[pass] == SEL_BUF0 ? kbuf0 : kbuf1;
  uint32_t* vdst = plan->dst[pass] == SEL_BUF0 ? vbuf0 : vbuf1;

  K key[ITEMS];
  uint32_t val[ITEMS];
  uint32_t dig[ITEMS];
  uint32_t rnk[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t idx = base + (uint64_t)w * 32 * ITEMS + (uint64_t)i * 32 + lane;
    if (idx < n) {
      if (src == SEL_INPUT) {
        key[i] = KT::load(D, idx);
        val[i] = (uint32_t)idx;
      } else {
        key[i] = NumStore<KT>::ld(ksrc, idx);
        val[i] = vsrc[idx];
      }
      dig[i] = KT::digit(key[i], pass);
    } else {
      dig[i] = 256;  // out of range: private bucket, never published
    }
  }
  // Stable warp-level multisplit: keys are ranked in (warp, item, lane) order,
  // which is their input order.
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const unsigned peers = __match_any_sync(FULL, dig[i]);
    const unsigned leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (lane == leader) {
      old = s_whist[w][dig[i]];
      s_whist[w][dig[i]] = old + __popc(peers);
    }
    old = __shfl_sync(FULL, old, leader);
    rnk[i] = old + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  // Per digit: exclusive offsets across warps, the tile's count, the look-back.
  const int d = threadIdx.x;  // kSortThreads == 256 digits
  uint32_t run = 0;
#pragma unroll
  for (int ww = 0; ww < W; ++ww) {
    const uint32_t c = s_whist[ww][d];
    s_whist[ww][d] = run;
    run += c;
  }
  const uint32_t tile_cnt = run;
  uint32_t* my = status + tile * 256 + d;
  uint32_t excl = 0;
  if (tile == 0) {
    st_volatile_u32(my, kRadixFlagPre | tile_cnt);
  } else {
    st_volatile_u32(my, kRadixFlagAgg | tile_cnt);
    // Look back LB predecessors per round trip (independent loads in flight),
    // so a first wave of T tiles resolves in ~T/LB round trips, not T.
    constexpr int LB = 32;
    bool done = false;
    for (int64_t t0 = (int64_t)tile - 1; !done; t0 -= LB) {
      uint32_t s[LB];
#pragma unroll
      for (int j = 0; j < LB; ++j)
        s[j] = t0 - j >= 0 ? ld_volatile_u32(status + (uint64_t)(t0 - j) * 256 + d) : kRadixFlagPre;
#pragma unroll
      for (int j = 0; j < LB; ++j) {
        if (!done) {
          while ((s[j] >> 30) == 0) s[j] = ld_volatile_u32(status + (uint64_t)(t0 - j) * 256 + d);
          excl += s[j] & kRadixValMask;
          done = (s[j] >> 30) == 2;
        }
      }
    }
    st_volatile_u32(my, kRadixFlagPre | (excl + tile_cnt));
  }
  uint32_t tot;
  const uint32_t bstart = block_exclusive_scan<kSortThreads>(tile_cnt, s_warp, tot);
  s_bstart[d] = bstart;
  s_gofs[d] = plan->digit_base[pass][d] + excl - bstart;
  __syncthreads();
  // Local reorder into shared memory (block-sorted by digit), then coalesced-ish writes.
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (dig[i] < 256) {
      const uint32_t pos = s_bstart[dig[i]] + s_whist[w][dig[i]] + rnk[i];
      s_keys[pos] = key[i];
      s_vals[pos] = val[i];
    }
  }
  __syncthreads();
  const uint32_t valid = (uint32_t)umin64(TILE, n - base);
  for (uint32_t j = threadIdx.x; j < valid; j += kSortThreads) {
    const K k = s_keys[j];
    const uint32_t dst = s_gofs[KT::digit(k, pass)] + j;
    NumStore<KT>::st(kdst, dst, k);
    vdst[dst] = s_vals[j];
  }
}

// Head flags + single-pass scan over the sorted keys -> U_D and r.
template <class KT>
__global__ void __launch_bounds__(kUniqThreads) k_unique(const void* __restrict__ D, const void* kbuf0,
                                                        const void* kbuf1, const uint32_t* vbuf0,
                                                        const uint32_t* vbuf1, uint64_t n,
                                                        const SortPlan* __restrict__ plan, uint64_t* status,
                                                        uint32_t* counter, void* __restrict__ udict,
                                                        uint32_t* __restrict__ rank, dm_header* hdr) {
  using K = typename KT::K;
  constexpr int TILE = kUniqThreads * kUniqItems;
  __shared__ uint32_t s_warp[kUniqThreads / 32 + 1];
  __shared__ uint64_t s_excl;
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const int sel = plan->final_sel;
  const void* ks = sel == SEL_BUF0 ? kbuf0 : kbuf1;
  const uint32_t* vs = sel == SEL_BUF0 ? vbuf0 : vbuf1;
  auto key_at = [&](uint64_t p) -> K { return sel == SEL_INPUT ? KT::load(D, p) : NumStore<KT>::ld(ks, p); };
  auto val_at = [&](uint64_t p) -> uint32_t { return sel == SEL_INPUT ? (uint32_t)p : vs[p]; };

  const uint64_t p0 = tile * TILE + (uint64_t)threadIdx.x * kUniqItems;
  K key[kUniqItems];
  uint32_t head = 0;  // bitmask over items
  uint32_t cnt = 0;
  K prev;
  if (p0 < n && p0 > 0) prev = key_at(p0 - 1);
#pragma unroll
  for (int i = 0; i < kUniqItems; ++i) {
    const uint64_t p = p0 + i;
    if (p < n) {
      key[i] = key_at(p);
      const bool h = (p == 0) || !KT::eq(key[i], prev);
      head |= (uint32_t)h << i;
      cnt += h;
      prev = key[i];
    }
  }
  uint32_t tile_cnt;
  const uint32_t texcl = block_exclusive_scan<kUniqThreads>(cnt, s_warp, tile_cnt);
  if (threadIdx.x < 32) {
    const uint64_t e = lookback_exclusive(status, tile, tile_cnt);
    if (threadIdx.x == 0) s_excl = e;
  }
  __syncthreads();
  uint64_t r = s_excl + texcl;  // number of heads strictly before p0
#pragma unroll
  for (int i = 0; i < kUniqItems; ++i) {
    const uint64_t p = p0 + i;
    if (p < n) {
      if ((head >> i) & 1) {
        KT::store(udict, r, key[i]);
        ++r;
      }
      rank[val_at(p)] = (uint32_t)(r - 1);
      if (p == n - 1) hdr->delta_dict_len = r;
    }
  }
}

template <class KT, int ITEMS>
cudaError_t run(const dm_column_in* in, char* ws, const WsLayout& L, void* udict, uint32_t* rank, dm_header* hdr,
                cudaStream_t st) {
  const uint64_t n = in->n_delta;
  uint32_t* counters = reinterpret_cast<uint32_t*>(ws + L.counters);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist);
  SortPlan* plan = reinterpret_cast<SortPlan*>(ws + L.plan);
  const int hist_blocks = (int)std::min<uint64_t>((n + 4095) / 4096, 148 * 4);
  k_hist<KT><<<hist_blocks, 256, 0, st>>>(in->delta, n, hist);
  k_plan<<<1, 256, 0, st>>>(hist, n, KT::kPasses, plan);
  note_launch(2);
  using K = typename KT::K;
  constexpr int TILE = kSortThreads * ITEMS;
  const size_t dsmem = (sizeof(K) + sizeof(uint32_t)) * TILE;
  cudaFuncSetAttribute(k_onesweep<KT, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem);
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  for (int p = 0; p < KT::kPasses; ++p) {
    uint32_t* status = reinterpret_cast<uint32_t*>(ws + L.status_sort) + (uint64_t)p * ntiles * 256;
    k_onesweep<KT, ITEMS><<<(unsigned)ntiles, kSortThreads, dsmem, st>>>(
        in->delta, ws + L.keys0, ws + L.keys1, reinterpret_cast<uint32_t*>(ws + L.vals0),
        reinterpret_cast<uint32_t*>(ws + L.vals1), n, p, plan, status, counters + CNT_SORT + p);
    note_launch();
  }
  const uint64_t utiles = (n + kUniqThreads * kUniqItems - 1) / (kUniqThreads * kUniqItems);
  k_unique<KT><<<(unsigned)utiles, kUniqThreads, 0, st>>>(
      in->delta, ws + L.keys0, ws + L.keys1, reinterpret_cast<const uint32_t*>(ws + L.vals0),
      reinterpret_cast<const uint32_t*>(ws + L.vals1), n, plan, reinterpret_cast<uint64_t*>(ws + L.status_unique),
      counters + CNT_UNIQUE, udict, rank, hdr);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_delta_dictionary(const dm_column_in* in, char* ws, const WsLayout& L, void* udict, uint32_t* rank,
                                    dm_header* hdr, cudaStream_t st) {
  if (in->n_delta == 0) return cudaSuccess;
  return in->key == DM_KEY_U64 ? run<KeyU64, kSortItemsU64>(in, ws, L, udict, rank, hdr, st)
                               : run<KeyB16, kSortItemsB16>(in, ws, L, udict, rank, hdr, st);
}

}  // namespace dm
