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
// Two sorting paths with the same result (U_D sorted and distinct, r[k] =
// rank of tuple k's value): for 2^11 <= N_D <= 2^23 the bucket path (k_bk_*,
// below: one counting pass into ~N_D/4 buckets by the keys' top varying bits,
// then a rank among the bucket mates) and otherwise, or when a bucket
// overflows (skewed keys; decided on the device), the LSD radix passes:
//   k_hist       one read of D: all digit histograms (8 or 16 byte passes) at
//                once; the last block to finish turns them into the pass plan:
//                exclusive digit offsets, and passes whose byte is constant over
//                every key are skipped (device-decided, no host sync)
//   k_onesweep   one stable LSD pass: warp-multisplit ranking (match.any) in
//                shared memory, local reorder, per-digit decoupled look-back
//                across tiles (32 predecessors per round trip), scatter
//   k_unique     head flags over the sorted keys (warp ballots), single-pass
//                scan with look-back -> U_D[rank] and r[original index] = rank
#include <algorithm>

#include <cooperative_groups.h>

#include "dm_device.cuh"

namespace cg = cooperative_groups;

#ifdef DM_TRACE
__device__ unsigned long long dm_trace_buf[8 * 32];
extern "C" int dm_debug_trace(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, dm_trace_buf, sizeof(dm_trace_buf));
}
__device__ __forceinline__ void dm_trace(int slot) {
  // blocks 0, S, 2S, ... (S = gridDim/8 rounded up): first wave and steady state
  const unsigned stride = (gridDim.x + 7) / 8;
  if (threadIdx.x == 0 && blockIdx.x % stride == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    dm_trace_buf[(blockIdx.x / stride) * 32 + slot] = t;
  }
}
#define DM_T(slot) dm_trace(slot)
#else
#define DM_T(slot)
#endif

namespace dm {
namespace {

__device__ void build_plan(const uint32_t* hist, uint64_t n, int npass, SortPlan* plan) {
  // Called by one block of 256 threads (the last k_hist block).
  __shared__ uint32_t s_warp[9];
  __shared__ int s_active[16];
  const int t = threadIdx.x;
  for (int p = 0; p < npass; ++p) {
    const uint32_t c = t < 256 ? __ldcg(hist + p * 256 + t) : 0u;
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

template <class KT>
__global__ void __launch_bounds__(256) k_hist(const void* __restrict__ D, uint64_t n_host,
                                              const unsigned long long* __restrict__ n_dev,
                                              uint32_t* __restrict__ hist, uint32_t* done,
                                              SortPlan* __restrict__ plan, const BucketState* __restrict__ gate) {
  pdl_prologue();
  if (gate && !gate->overflow) return;  // the bucket path sorted D (its plan stands)
  constexpr int P = KT::kPasses;
  const uint64_t n = n_dev ? (uint64_t)*n_dev : n_host;
  __shared__ uint32_t s_h[P][256];
  __shared__ bool s_last;
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
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    __threadfence();
    build_plan(hist, n, P, plan);
  }
}

// One stable LSD radix pass over (key, original-index) pairs.  NT threads,
// ITEMS keys per thread, tile = NT * ITEMS keys in (warp, item, lane) order.
// One tile of one pass (claimed in order from `counter`); false once the tiles
// run past n.  Shared by the per-pass kernel and the cooperative all-passes one.
template <class KT, int NT, int ITEMS>
__device__ __forceinline__ bool onesweep_tile(const void* __restrict__ D, void* kbuf0, void* kbuf1, uint32_t* vbuf0,
                                              uint32_t* vbuf1, uint64_t n, int pass,
                                              const SortPlan* __restrict__ plan, uint32_t* status,
                                              uint32_t* counter) {
  using K = typename KT::K;
  constexpr int W = NT / 32;
  constexpr int TILE = NT * ITEMS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* s_keys = reinterpret_cast<K*>(smem_raw);
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(smem_raw + sizeof(K) * TILE);
  __shared__ uint32_t s_whist[W][257];
  __shared__ uint32_t s_bstart[256];
  __shared__ uint32_t s_gofs[256];
  __shared__ uint32_t s_tcnt[256];
  __shared__ uint32_t s_warp[W + 1];
  __shared__ uint32_t s_tile;

  const unsigned lane = lane_id(), w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < W * 257; i += NT) (&s_whist[0][0])[i] = 0;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  DM_T(2);
  const uint64_t tile = s_tile;
  const uint64_t base = tile * TILE;
  if (base >= n) return false;
  const int src = plan->src[pass];
  const void* ksrc = src == SEL_BUF0 ? kbuf0 : kbuf1;
  const uint32_t* vsrc = src == SEL_BUF0 ? vbuf0 : vbuf1;
  void* kdst = plan->dst[pass] == SEL_BUF0 ? kbuf0 : kbuf1;
  uint32_t* vdst = plan->dst[pass] == SEL_BUF0 ? vbuf0 : vbuf1;

  K key[ITEMS];
  uint32_t val[ITEMS];
  uint32_t dig[ITEMS];
  uint32_t rnk[ITEMS];
  // All loads first, branch-free (clamped index), so they are in flight together.
  const bool from_input = src == SEL_INPUT;
  const void* kp = from_input ? D : ksrc;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t idx = base + (uint64_t)w * 32 * ITEMS + (uint64_t)i * 32 + lane;
    const uint64_t ic = idx < n ? idx : n - 1;
    key[i] = KT::ld_any(kp, ic, from_input);
    val[i] = from_input ? (uint32_t)idx : vsrc[ic];
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t idx = base + (uint64_t)w * 32 * ITEMS + (uint64_t)i * 32 + lane;
    dig[i] = idx < n ? KT::digit(key[i], pass) : 256u;  // 256: private bucket, never published
  }
  DM_T(3);
  // Stable warp-level multisplit: ranks in (warp, item, lane) order = input order.
  // Peers (lanes with the same digit) from 8 bit-plane ballots -- far cheaper
  // than match.any, which measured as the pass's throughput limiter -- then a
  // short per-item chain: every lane reads its digit's running count, the
  // digit's leader adds the item's population.
  const unsigned lt = lanemask_lt();
  unsigned peers[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    unsigned p = __ballot_sync(FULL, dig[i] < 256);  // valid lanes only
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const unsigned bit = (dig[i] >> b) & 1u;
      const unsigned v = __ballot_sync(FULL, bit);
      p &= bit ? v : ~v;
    }
    peers[i] = dig[i] < 256 ? p : (1u << lane);  // invalid lanes: private bucket 256
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t old = s_whist[w][dig[i]];
    const unsigned below = peers[i] & lt;
    if (below == 0) s_whist[w][dig[i]] = old + __popc(peers[i]);  // the leader (lowest lane)
    rnk[i] = old + __popc(below);
    __syncwarp();
  }
  __syncthreads();
  DM_T(4);
  // Per digit: exclusive offsets across warps and the tile's count; publish the
  // aggregate right away so successors can start their look-back.
  const int d = threadIdx.x;
  uint32_t tile_cnt = 0;
  if (d < 256) {
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < W; ++ww) {
      const uint32_t c = s_whist[ww][d];
      s_whist[ww][d] = run;
      run += c;
    }
    tile_cnt = run;
    s_tcnt[d] = run;
    st_volatile_u32(status + tile * 256 + d, (tile == 0 ? kRadixFlagPre : kRadixFlagAgg) | tile_cnt);
  }
  uint32_t tot;
  const uint32_t bstart = block_exclusive_scan<NT>(d < 256 ? tile_cnt : 0u, s_warp, tot);
  if (d < 256) s_bstart[d] = bstart;
  __syncthreads();
  DM_T(5);
  // Local reorder into shared memory (block-sorted by digit): frees the registers
  // before the look-back.
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (dig[i] < 256) {
      const uint32_t pos = s_bstart[dig[i]] + s_whist[w][dig[i]] + rnk[i];
      s_keys[pos] = key[i];
      s_vals[pos] = val[i];
    }
  }
  DM_T(6);
  if (d < 256) {
    uint32_t excl = 0;
    if (tile > 0) {
      // LB predecessors per round trip: a first wave of T tiles resolves in ~T/LB trips.
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
      st_volatile_u32(status + tile * 256 + d, kRadixFlagPre | (excl + s_tcnt[d]));
    }
    s_gofs[d] = plan->digit_base[pass][d] + excl - s_bstart[d];
  }
  __syncthreads();
  DM_T(7);
  const uint32_t valid = (uint32_t)umin64(TILE, n - base);
#pragma unroll 4
  for (uint32_t j = threadIdx.x; j < valid; j += NT) {
    const K k = s_keys[j];
    const uint32_t dst = s_gofs[KT::digit(k, pass)] + j;
    NumStore<KT>::st(kdst, dst, k);
    vdst[dst] = s_vals[j];
  }
  DM_T(8);
  __syncthreads();  // the shared tile is reused by the next claim
  return true;
}

template <class KT, int NT, int ITEMS>
__global__ void __launch_bounds__(NT) k_onesweep(const void* __restrict__ D, void* kbuf0, void* kbuf1,
                                                uint32_t* vbuf0, uint32_t* vbuf1, uint64_t n_host,
                                                const unsigned long long* __restrict__ n_dev, int pass,
                                                const SortPlan* __restrict__ plan, uint32_t* status,
                                                uint32_t* counter) {
  pdl_prologue();
  // n_dev: the key count is only known on the device (deduplicated delta); the
  // grid covers n_host >= n and tiles past n exit (nothing waits on them)
  const uint64_t n = n_dev ? (uint64_t)*n_dev : n_host;
  DM_T(0);
  if (!plan->active[pass]) return;
  DM_T(1);
  onesweep_tile<KT, NT, ITEMS>(D, kbuf0, kbuf1, vbuf0, vbuf1, n, pass, plan, status, counter);
}

// All LSD passes in one cooperative, persistent launch: the CTAs claim the tiles
// of each active pass in order (the per-digit look-back needs every claimed
// predecessor running -- a cooperative grid is co-resident) and meet at a grid
// barrier between passes.  One launch instead of one per byte: the bucket path's
// gated fallback (the passes only run when a bucket overflowed) then costs a
// single early-exit launch per merge, not 8 or 16.
template <class KT, int NT, int ITEMS>
__global__ void __launch_bounds__(NT) k_onesweep_all(const void* __restrict__ D, void* kbuf0, void* kbuf1,
                                                    uint32_t* vbuf0, uint32_t* vbuf1, uint64_t n_host,
                                                    const unsigned long long* __restrict__ n_dev,
                                                    const SortPlan* __restrict__ plan, uint32_t* status_base,
                                                    uint64_t status_stride, uint32_t* counters) {
  const uint64_t n = n_dev ? (uint64_t)*n_dev : n_host;
  cg::grid_group grid = cg::this_grid();
  for (int p = 0; p < KT::kPasses; ++p) {
    if (!plan->active[p]) continue;  // uniform: every CTA reads the same plan
    while (onesweep_tile<KT, NT, ITEMS>(D, kbuf0, kbuf1, vbuf0, vbuf1, n, p, plan,
                                        status_base + (uint64_t)p * status_stride, counters + p)) {
    }
    grid.sync();
  }
}

// Head flags + single-pass scan over the sorted keys -> U_D and r.
// Warp-striped layout: element (w, i, l) is position base + w*32*ITEMS + i*32 + l.
template <class KT>
__global__ void __launch_bounds__(kUniqThreads) k_unique(const void* __restrict__ D, const void* kbuf0,
                                                        const void* kbuf1, const uint32_t* vbuf0,
                                                        const uint32_t* vbuf1, uint64_t n_host,
                                                        const unsigned long long* __restrict__ n_dev,
                                                        const SortPlan* __restrict__ plan, uint64_t* status,
                                                        uint32_t* counter, void* __restrict__ udict,
                                                        uint32_t* __restrict__ rank, dm_header* hdr) {
  pdl_prologue();
  using K = typename KT::K;
  constexpr int NT = kUniqThreads, ITEMS = kUniqItems, W = NT / 32;
  constexpr int TILE = NT * ITEMS;
  __shared__ uint32_t s_warp[W + 1];
  __shared__ uint64_t s_excl;
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t n = n_dev ? (uint64_t)*n_dev : n_host;
  if (tile * TILE >= n) return;
  const int sel = plan->final_sel;
  const void* ks = sel == SEL_BUF0 ? kbuf0 : kbuf1;
  const uint32_t* vs = sel == SEL_BUF0 ? vbuf0 : vbuf1;
  const bool from_input = sel == SEL_INPUT;
  const void* kp = from_input ? D : ks;
  auto val_at = [&](uint64_t p) -> uint32_t { return from_input ? (uint32_t)p : vs[p]; };

  const unsigned lane = lane_id(), w = threadIdx.x >> 5;
  const uint64_t wbase = tile * TILE + (uint64_t)w * 32 * ITEMS;
  K key[ITEMS];
  uint32_t hb[ITEMS];  // head ballots per item
  uint32_t wcount = 0;
  // the element just before this warp's first element (branch-free, clamped)
  K before = KT::ld_any(kp, wbase > 0 ? umin64(wbase - 1, n - 1) : 0, from_input);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t p = wbase + (uint64_t)i * 32 + lane;
    key[i] = KT::ld_any(kp, p < n ? p : n - 1, from_input);
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t p = wbase + (uint64_t)i * 32 + lane;
    // previous element: lane-1 of this item, lane 31 of the previous item, or `before`
    K prev;
    if constexpr (sizeof(K) <= 8) {
      uint64_t up = __shfl_up_sync(FULL, (uint64_t)key[i], 1);
      uint64_t last = i > 0 ? __shfl_sync(FULL, (uint64_t)key[i > 0 ? i - 1 : 0], 31) : (uint64_t)before;
      if (i == 0) last = __shfl_sync(FULL, (uint64_t)before, 0);
      prev = (K)(lane == 0 ? last : up);
    } else {
      K128 kk = *reinterpret_cast<K128*>(&key[i]);
      K128 pk = *reinterpret_cast<K128*>(&key[i > 0 ? i - 1 : 0]);
      K128 bk = *reinterpret_cast<K128*>(&before);
      uint64_t uh = __shfl_up_sync(FULL, kk.hi, 1), ul = __shfl_up_sync(FULL, kk.lo, 1);
      uint64_t lh = i > 0 ? __shfl_sync(FULL, pk.hi, 31) : __shfl_sync(FULL, bk.hi, 0);
      uint64_t ll = i > 0 ? __shfl_sync(FULL, pk.lo, 31) : __shfl_sync(FULL, bk.lo, 0);
      K128 r = lane == 0 ? K128{lh, ll} : K128{uh, ul};
      prev = *reinterpret_cast<K*>(&r);
    }
    const bool h = p < n && (p == 0 || !KT::eq(key[i], prev));
    hb[i] = __ballot_sync(FULL, h);
    wcount += __popc(hb[i]);
  }
  // block scan over warp counts (lane 0 of each warp contributes)
  uint32_t tile_cnt;
  const uint32_t wex = block_exclusive_scan<NT>(lane == 0 ? wcount : 0u, s_warp, tile_cnt);
  const uint32_t wexcl = __shfl_sync(FULL, wex, 0);
  if (threadIdx.x < 32) {
    const uint64_t e = lookback_exclusive(status, tile, tile_cnt);
    if (threadIdx.x == 0) s_excl = e;
  }
  __syncthreads();
  uint64_t run = s_excl + wexcl;  // heads strictly before this warp's first element
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t p = wbase + (uint64_t)i * 32 + lane;
    const uint64_t r = run + __popc(hb[i] & lt);  // heads before p
    const bool h = (hb[i] >> lane) & 1;
    if (p < n) {
      if (h) KT::store(udict, r, key[i]);
      rank[val_at(p)] = (uint32_t)(r + h - 1);
      if (p == n - 1) hdr->delta_dict_len = r + h;
    }
    run += __popc(hb[i]);
  }
}

// ------------------------------------------------------------ bucket path
// Step 1(a) for N_D <= 2^23 without LSD passes.  Each LSD pass over ~10^6 keys is
// a latency-bound kernel of ~16 us (look-back chain, one tile per SM), and a
// 48-bit key needs six of them.  Instead, one counting pass places every key in
// one of B ~ N_D / 4 buckets by the top log2 B bits below the prefix shared by
// all keys (so bucket order = key order), and each key then finds its final
// position inside its (small) bucket by comparing with its bucket mates:
//   k_bk_range    OR of (k ^ k0) over D -> the highest differing bit h; digit =
//                 bits [h + 1 - log2 B, h]; zeroes the counts
//   k_bk_count    counts per bucket (global atomics)
//   k_bk_scan     exclusive offsets (single pass, decoupled look-back); a bucket
//                 above kBkMaxBucket raises the overflow flag
//   k_bk_scatter  key -> its bucket (slot from an atomic cursor: unordered)
//   k_bk_local    rank among the bucket mates by (key, index) -> sorted order
// then k_unique as after the LSD passes.  Skewed key sets (a dense cluster, an
// outlier, heavy repeats without the dedup front end) overflow a bucket: the
// bucket kernels stop and the LSD passes, launched behind them and gated on
// the flag, sort instead.
template <class KT>
struct Bits128;
template <>
struct Bits128<KeyU64> {
  __device__ __forceinline__ static void get(uint64_t k, uint64_t& hi, uint64_t& lo) { hi = 0; lo = k; }
};
template <>
struct Bits128<KeyU32> {
  __device__ __forceinline__ static void get(uint32_t k, uint64_t& hi, uint64_t& lo) { hi = 0; lo = k; }
};
template <>
struct Bits128<KeyB16> {
  __device__ __forceinline__ static void get(K128 k, uint64_t& hi, uint64_t& lo) { hi = k.hi; lo = k.lo; }
};
template <class KT>
__device__ __forceinline__ uint32_t bk_digit(typename KT::K k, uint32_t s, uint32_t mask) {
  uint64_t hi, lo;
  Bits128<KT>::get(k, hi, lo);
  const uint64_t v = s >= 64 ? hi >> (s - 64) : s == 0 ? lo : (lo >> s) | (hi << (64 - s));
  return (uint32_t)v & mask;
}

template <class KT>
__global__ void __launch_bounds__(256) k_bk_range(const void* __restrict__ D, uint64_t n_host,
                                                  const unsigned long long* __restrict__ n_dev,
                                                  BucketState* st, uint32_t* __restrict__ cnt, uint32_t bits,
                                                  SortPlan* __restrict__ plan) {  // cnt: the counts to zero
  pdl_prologue();
  const uint64_t n = n_dev ? (uint64_t)*n_dev : n_host;
  const uint64_t nb = 1ull << bits;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, nthr = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = tid; i < nb; i += nthr) cnt[i] = 0;
  uint64_t h0 = 0, l0 = 0, dh = 0, dl = 0;
  if (n) Bits128<KT>::get(KT::load(D, 0), h0, l0);
  for (uint64_t i = tid; i < n; i += nthr) {
    uint64_t h, l;
    Bits128<KT>::get(KT::load(D, i), h, l);
    dh |= h ^ h0;
    dl |= l ^ l0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dh |= __shfl_xor_sync(FULL, dh, o);
    dl |= __shfl_xor_sync(FULL, dl, o);
  }
  __shared__ unsigned long long s_h, s_l;
  __shared__ bool s_last;
  if (threadIdx.x == 0) s_h = s_l = 0;
  __syncthreads();
  if (lane_id() == 0) {
    atomicOr(&s_h, (unsigned long long)dh);
    atomicOr(&s_l, (unsigned long long)dl);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // one global atomic per block and word
    if (s_h) atomicOr(&st->diff_hi, s_h);
    if (s_l) atomicOr(&st->diff_lo, s_l);
    __threadfence();
    s_last = atomicAdd(&st->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  const uint64_t H = __ldcg(&st->diff_hi), Lo = __ldcg(&st->diff_lo);
  const int h = H ? 127 - __clzll((long long)H) : Lo ? 63 - __clzll((long long)Lo) : -1;
  st->shift = h + 1 > (int)bits ? (uint32_t)(h + 1 - (int)bits) : 0u;
  // the LSD passes stay idle unless a bucket overflows (k_hist then rebuilds
  // this plan and k_unique runs)
  for (int p = 0; p < 16; ++p) plan->active[p] = 0;
  plan->final_sel = SEL_BUF0;
  plan->n_active = 0;
}

template <class KT>
__global__ void __launch_bounds__(256) k_bk_count(const void* __restrict__ D, uint64_t n_host,
                                                  const unsigned long long* __restrict__ n_dev,
                                                  const BucketState* __restrict__ st, uint32_t* __restrict__ off,
                                                  uint32_t bits) {
  pdl_prologue();
  const uint64_t n = n_dev ? (uint64_t)*n_dev : n_host;
  const uint32_t s = st->shift, mask = (uint32_t)((1ull << bits) - 1);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(off + bk_digit<KT>(KT::load(D, i), s, mask), 1u);
}

// In place: off[d] = #keys in buckets < d (off[B] = n), cur[d] = off[d]; a
// bucket above kBkMaxBucket keys raises the overflow flag.
__global__ void __launch_bounds__(256) k_bk_scan(uint32_t* __restrict__ off, uint32_t* __restrict__ cur,
                                                 uint64_t nb, uint64_t* status, uint32_t* counter,
                                                 BucketState* st) {
  pdl_prologue();
  constexpr int ITEMS = kBkScanItems, TILE = 256 * ITEMS;
  __shared__ uint32_t s_warp[9];
  __shared__ uint64_t s_excl;
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t p0 = tile * TILE + threadIdx.x * ITEMS;  // nb is a multiple of TILE
  uint32_t v[ITEMS], sum = 0, mx = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; i += 4) {
    const uint4 q = *reinterpret_cast<const uint4*>(off + p0 + i);
    v[i] = q.x, v[i + 1] = q.y, v[i + 2] = q.z, v[i + 3] = q.w;
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    sum += v[i];
    mx = v[i] > mx ? v[i] : mx;
  }
  if (__any_sync(FULL, mx > kBkMaxBucket) && lane_id() == 0) atomicOr(&st->overflow, 1u);
  uint32_t tile_sum;
  const uint32_t texcl = block_exclusive_scan<256>(sum, s_warp, tile_sum);
  if (threadIdx.x < 32) {
    const uint64_t e = lookback_exclusive(status, tile, tile_sum);
    if (threadIdx.x == 0) s_excl = e;
  }
  __syncthreads();
  uint32_t run = (uint32_t)(s_excl + texcl);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t x = v[i];
    v[i] = run;
    run += x;
  }
#pragma unroll
  for (int i = 0; i < ITEMS; i += 4) {
    *reinterpret_cast<uint4*>(off + p0 + i) = make_uint4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    *reinterpret_cast<uint4*>(cur + p0 + i) = make_uint4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  }
  if ((tile + 1) * TILE >= nb && threadIdx.x == 255) off[nb] = run;
}

template <class KT>
__global__ void __launch_bounds__(256) k_bk_scatter(const void* __restrict__ D, uint64_t n_host,
                                                    const unsigned long long* __restrict__ n_dev,
                                                    const BucketState* __restrict__ st, uint32_t* __restrict__ cur,
                                                    uint32_t bits, void* __restrict__ kout,
                                                    uint32_t* __restrict__ vout) {
  pdl_prologue();
  if (st->overflow) return;
  const uint64_t n = n_dev ? (uint64_t)*n_dev : n_host;
  const uint32_t s = st->shift, mask = (uint32_t)((1ull << bits) - 1);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const typename KT::K k = KT::load(D, i);
    const uint32_t pos = atomicAdd(cur + bk_digit<KT>(k, s, mask), 1u);
    DM_ASSERT(pos < n, "bucket scatter pos %u n %llu", pos, (unsigned long long)n);
    if constexpr (KT::kBytes <= 8) {  // one 16-byte (key, index) record: one scattered store
      const uint64_t k64 = (uint64_t)k;
      static_cast<uint4*>(kout)[pos] = make_uint4((uint32_t)k64, (uint32_t)(k64 >> 32), (uint32_t)i, 0u);
    } else {
      NumStore<KT>::st(kout, pos, k);
      vout[pos] = (uint32_t)i;
    }
  }
}

// Final position of each key: its bucket's offset + #{bucket mates ordered
// before it by (key, original index)} -- a permutation, sorted by key.
template <class KT>
__global__ void __launch_bounds__(256) k_bk_local(const void* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                  uint64_t n_host, const unsigned long long* __restrict__ n_dev,
                                                  const BucketState* __restrict__ st,
                                                  const uint32_t* __restrict__ off, uint32_t bits,
                                                  void* __restrict__ kout, uint32_t* __restrict__ vout) {
  pdl_prologue();
  if (st->overflow) return;
  using K = typename KT::K;
  const uint64_t n = n_dev ? (uint64_t)*n_dev : n_host;
  const uint32_t s = st->shift, mask = (uint32_t)((1ull << bits) - 1);
  // 4/8-byte keys arrive as 16-byte (key, index) records (k_bk_scatter)
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    K k;
    uint32_t id;
    if constexpr (KT::kBytes <= 8) {
      const uint4 v = static_cast<const uint4*>(kin)[p];
      k = (K)(((uint64_t)v.y << 32) | v.x);
      id = v.z;
    } else {
      k = NumStore<KT>::ld(kin, p);
      id = vin[p];
    }
    const uint32_t d = bk_digit<KT>(k, s, mask);
    const uint32_t lo = off[d], hi = off[d + 1];
    DM_ASSERT(lo <= p && p < hi && hi <= n, "bucket local p %llu lo %u hi %u n %llu", (unsigned long long)p, lo, hi,
              (unsigned long long)n);
    uint32_t r = lo;
    for (uint32_t q = lo; q < hi; ++q) {
      if constexpr (KT::kBytes <= 8) {
        const uint4 v = static_cast<const uint4*>(kin)[q];
        const K kq = (K)(((uint64_t)v.y << 32) | v.x);
        r += KT::lt(kq, k) ? 1u : (KT::eq(kq, k) && v.z < id) ? 1u : 0u;
      } else {
        const K kq = NumStore<KT>::ld(kin, q);
        r += KT::lt(kq, k) ? 1u : (KT::eq(kq, k) && vin[q] < id) ? 1u : 0u;
      }
    }
    NumStore<KT>::st(kout, r, k);
    vout[r] = id;
  }
}

// ------------------------------------------------------------ dedup front end
// NEXT1: the paper gets U_D by "extracting the unique values"
// from a tree it maintained at insert time; a delta with many
// repeated values (cfg3's Zipf reuse: 5e6 tuples, ~1.5e6 distinct) would spend
// the 16 radix passes mostly on repeats.  So: insert every tuple into an
// open-addressing hash table first -- the first inserter of a value claims a
// slot, takes the next distinct id and stores the value at dkeys[id] -- then
// sort only the distinct values (count known on the device only) and map each
// tuple's id to its rank.  Same U_D and r as sorting all of D.
__device__ __forceinline__ uint64_t dd_mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}
__device__ __forceinline__ uint64_t dd_hash(uint64_t k) { return dd_mix(k); }
__device__ __forceinline__ uint64_t dd_hash(K128 k) { return dd_mix(k.hi ^ dd_mix(k.lo + 0x9e3779b97f4a7c15ull)); }
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One 8-byte slot per entry: low word = tag (0 empty; (h & ~3) | 1 claimed;
// | 3 ready), high word = the distinct id once ready, so a probe reads tag and id
// in one access.  Probes and the spin read relaxed (no L1 invalidation); one
// acquire load once a matching tag is ready orders the value read after it.
// The claimant's release store orders its value write before (id, ready)
// (measured: a __threadfence there and acquire probes took ~60% of the
// kernel's stall samples on cfg3).
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <class KT>
__global__ void __launch_bounds__(256) k_dedup_insert(const void* __restrict__ D, uint64_t n,
                                                      uint64_t* __restrict__ slots, uint64_t mask,
                                                      void* __restrict__ dkeys, uint32_t* __restrict__ tid,
                                                      unsigned long long* n_dist) {
  pdl_prologue();
  using K = typename KT::K;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const K k = KT::load(D, i);
    const uint64_t h = dd_hash(k);
    uint64_t slot = (h >> 32) & mask;
    const uint32_t tg = ((uint32_t)h & ~3u) | 1u;
    uint32_t id = 0;
    for (;;) {
      uint64_t sv = ld_relaxed_u64(slots + slot);
      if ((uint32_t)sv == 0) {
        sv = atomicCAS(reinterpret_cast<unsigned long long*>(slots + slot), 0ull, (unsigned long long)tg);
        if (sv == 0) {  // claimed: publish the value, then (id, ready)
          // ids for all lanes that claimed in this step: one atomic per warp, not per value
          const unsigned m = __activemask();
          const int leader = __ffs(m) - 1;
          unsigned long long b0 = 0;
          if ((int)lane_id() == leader) b0 = atomicAdd(n_dist, (unsigned long long)__popc(m));
          b0 = __shfl_sync(m, b0, leader);
          id = (uint32_t)(b0 + __popc(m & lanemask_lt()));
          KT::store(dkeys, id, k);
          st_release_u64(slots + slot, ((uint64_t)id << 32) | tg | 2u);
          break;
        }
      }
      if (((uint32_t)sv | 2u) == (tg | 2u)) {  // same hash tag: wait until ready, compare the value
        while (!((uint32_t)sv & 2u)) sv = ld_relaxed_u64(slots + slot);
        sv = ld_acquire_u64(slots + slot);
        const uint32_t cid = (uint32_t)(sv >> 32);
        if (KT::eq(KT::load_cg(dkeys, cid), k)) {
          id = cid;
          break;
        }
      }
      slot = (slot + 1) & mask;
    }
    tid[i] = id;
  }
}

// ---------------------------------------------------------- probe-first (NEXT1)
// "The delta partition's dictionary U_D ... is merged with U_M": a
// delta value already in U_M needs no sorting -- its new code is X_M at its U_M
// position.  U_M's positions go into an open-addressing table keyed by value
// (k_pf_build; U_M is distinct, so inserts never contend), then every tuple
// probes it (k_pf_probe): the table and U_M are read-only by then, so the probes
// go through L1 and a skewed reuse (cfg3's Zipf) hits cache instead of hammering
// one hash slot.  Found -> src = position (and its bit in the "used" bitmap, for
// |U_D|); not found -> compacted (warp-aggregated atomic) into the keys Step
// 1(a)'s sort sees.  (A binary search of U_M with a shared-memory sample was
// measured first: ~10 dependent L2 round trips per tuple, 0.60 ms on cfg3.)
// Table entries are (tag | position): the position in the low pos_bits =
// ceil(log2 |U_M|) bits, the value hash's low bits above them (the lowest tag
// bit cleared, so no entry equals the empty word), so a probe loads U_M only
// when the tag matches.  Measured on cfg3 before the tags (load factor 1/2,
// every probe loading U_M): a warp walked ~6.8 probe steps per tuple batch (the
// longest chain of its 32 lanes), each two dependent loads -- 152 us for 5e6 tuples.
constexpr uint32_t kPfEmpty = 0xffffffffu;
struct PfTag {
  uint32_t pos_mask, tag_mask;
  __host__ __device__ static PfTag make(uint64_t nM) {
    uint32_t b = 1;
    while (b < 32 && (1ull << b) < nM) ++b;
    const uint32_t pm = b >= 32 ? 0xffffffffu : (1u << b) - 1u;
    return PfTag{pm, b >= 32 ? 0u : ~pm & ~(1u << b)};
  }
  __device__ __forceinline__ uint32_t tag(uint64_t h) const { return (uint32_t)h & tag_mask; }
};
template <class KT>
__global__ void __launch_bounds__(256) k_pf_build(const void* __restrict__ UM, uint64_t nM, uint32_t* __restrict__ table,
                                                  uint64_t mask, PfTag tg) {
  pdl_prologue();
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nM; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = dd_hash(KT::load(UM, p));
    uint64_t slot = (h >> 32) & mask;
    const uint32_t e = (uint32_t)p | tg.tag(h);
    while (atomicCAS(table + slot, kPfEmpty, e) != kPfEmpty) slot = (slot + 1) & mask;
  }
}

// Each block takes 1024 tuples per round: one atomic per block and round
// claims the compacted slots of its new values (a per-warp atomic on one counter
// serialised ~1.6e5 warps on cfg3), and a tuple whose "used" bit is already set
// (a Zipf-hot value) skips its atomicOr.
constexpr int kPfThreads = 256, kPfItems = 4;
template <class KT>
__global__ void __launch_bounds__(kPfThreads) k_pf_probe(const void* __restrict__ UM,
                                                         const uint32_t* __restrict__ table, uint64_t mask,
                                                         const void* __restrict__ D, uint64_t n,
                                                         uint32_t* __restrict__ src, void* __restrict__ newkeys,
                                                         unsigned long long* n_new, uint32_t* used, PfTag tg) {
  pdl_prologue();
  using K = typename KT::K;
  constexpr int TILE = kPfThreads * kPfItems;
  __shared__ uint32_t s_warp[kPfThreads / 32 + 1];
  __shared__ unsigned long long s_base;
  for (uint64_t base = (uint64_t)blockIdx.x * TILE; base < n; base += (uint64_t)gridDim.x * TILE) {
    K v[kPfItems];
    uint32_t p[kPfItems];
    uint32_t nnew = 0;
    // the kPfItems probes of a thread as independent loads, step by step (key,
    // first slot, candidate's U_M value); an item whose first slot holds another
    // value continues alone in a loop
    uint64_t h[kPfItems];
    uint32_t q[kPfItems];
#pragma unroll
    for (int r = 0; r < kPfItems; ++r) {
      const uint64_t i = base + (uint64_t)r * kPfThreads + threadIdx.x;
      v[r] = KT::load(D, i < n ? i : n - 1);
      h[r] = dd_hash(v[r]);
    }
#pragma unroll
    for (int r = 0; r < kPfItems; ++r) q[r] = __ldg(table + ((h[r] >> 32) & mask));
    bool hit[kPfItems];
#pragma unroll
    for (int r = 0; r < kPfItems; ++r) {
      const bool cand = q[r] != kPfEmpty && (q[r] & tg.tag_mask) == tg.tag(h[r]);
      hit[r] = cand && KT::eq(KT::load(UM, cand ? q[r] & tg.pos_mask : 0u), v[r]);
    }
#pragma unroll
    for (int r = 0; r < kPfItems; ++r) {
      const uint64_t i = base + (uint64_t)r * kPfThreads + threadIdx.x;
      p[r] = kPfEmpty;
      if (i < n) {
        if (hit[r]) {
          p[r] = q[r] & tg.pos_mask;
        } else if (q[r] != kPfEmpty) {  // the first slot holds another value: walk on
          const uint32_t tag = tg.tag(h[r]);
          uint64_t slot = (h[r] >> 32) & mask;
          for (;;) {
            slot = (slot + 1) & mask;
            const uint32_t e = __ldg(table + slot);
            if (e == kPfEmpty) break;
            if ((e & tg.tag_mask) == tag && KT::eq(KT::load(UM, e & tg.pos_mask), v[r])) {
              p[r] = e & tg.pos_mask;
              break;
            }
          }
        }
      }
    }
    uint32_t uw[kPfItems];  // the "used" words, loaded together
#pragma unroll
    for (int r = 0; r < kPfItems; ++r) uw[r] = p[r] != kPfEmpty ? used[p[r] >> 5] : 0xffffffffu;
#pragma unroll
    for (int r = 0; r < kPfItems; ++r) {
      const uint64_t i = base + (uint64_t)r * kPfThreads + threadIdx.x;
      if (i >= n) continue;
      if (p[r] == kPfEmpty) {
        ++nnew;
      } else {
        src[i] = p[r];
        const uint32_t bit = 1u << (p[r] & 31);
        if (!(uw[r] & bit)) atomicOr(&used[p[r] >> 5], bit);
      }
    }
    uint32_t tot;
    uint32_t off = block_exclusive_scan<kPfThreads>(nnew, s_warp, tot);
    if (threadIdx.x == 0) s_base = tot ? atomicAdd(n_new, (unsigned long long)tot) : 0ull;
    __syncthreads();
    const unsigned long long b0 = s_base;
#pragma unroll
    for (int r = 0; r < kPfItems; ++r) {
      const uint64_t i = base + (uint64_t)r * kPfThreads + threadIdx.x;
      if (i < n && p[r] == kPfEmpty) {
        const uint64_t j = b0 + off++;
        KT::store(newkeys, j, v[r]);
        src[i] = kPfNew | (uint32_t)j;
      }
    }
    __syncthreads();  // s_base / s_warp reused next round
  }
}

// After Step 1(b) over (U_M, U_new): the tuples' final codes, and |U_D| = |U_new|
// + #distinct found values (the used bitmap's population, block-reduced).
__global__ void __launch_bounds__(256) k_pf_codes(const uint32_t* __restrict__ src, uint64_t n,
                                                  const uint32_t* __restrict__ rank_new,
                                                  const uint32_t* __restrict__ xm, const uint32_t* __restrict__ xd,
                                                  uint32_t* __restrict__ codes, const uint32_t* __restrict__ used,
                                                  uint64_t nwords, dm_header* hdr) {
  pdl_prologue();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t s = src[i];
    codes[i] = (s & kPfNew) ? __ldg(xd + __ldg(rank_new + (s & ~kPfNew))) : __ldg(xm + s);
  }
  uint32_t c = 0;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) c += __popc(used[w]);
  c = warp_sum<uint32_t>(c);
  if (lane_id() == 0 && c) atomicAdd(reinterpret_cast<unsigned long long*>(&hdr->delta_dict_len), (unsigned long long)c);
}

// r[k] = rank of tuple k's distinct value = rank_of_id[tid[k]].
__global__ void __launch_bounds__(256) k_dedup_ranks(const uint32_t* __restrict__ tid,
                                                     const uint32_t* __restrict__ rank_of_id, uint64_t n,
                                                     uint32_t* __restrict__ rank) {
  pdl_prologue();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    rank[i] = __ldg(rank_of_id + __ldg(tid + i));
}

// DM_SORT_COOP=0: one launch per pass (the round-1 form; experiments)
bool onesweep_coop() {
  static const bool v = [] {
    const char* e = std::getenv("DM_SORT_COOP");
    return !(e && e[0] == '0');
  }();
  return v;
}

template <class KT, int NT, int ITEMS>
void launch_passes(const void* D, uint64_t n, const unsigned long long* n_dev, char* ws, const WsLayout& L,
                   SortPlan* plan, uint32_t* counters, cudaStream_t st) {
  using K = typename KT::K;
  constexpr int TILE = NT * ITEMS;
  const size_t dsmem = (sizeof(K) + sizeof(uint32_t)) * TILE;
  ensure_smem((const void*)k_onesweep<KT, NT, ITEMS>);
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  if (onesweep_coop()) {  // one cooperative launch for all passes
    auto kern = k_onesweep_all<KT, NT, ITEMS>;
    ensure_smem((const void*)kern);
    const int occ = occupancy((const void*)kern, NT, dsmem);
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ntiles, (uint64_t)device_sms() * occ));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = NT;
    cfg.dynamicSmemBytes = dsmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, D, (void*)(ws + L.keys0), (void*)(ws + L.keys1),
                       reinterpret_cast<uint32_t*>(ws + L.vals0), reinterpret_cast<uint32_t*>(ws + L.vals1), n,
                       n_dev, (const SortPlan*)plan, reinterpret_cast<uint32_t*>(ws + L.status_sort),
                       (uint64_t)ntiles * 256, counters + CNT_SORT);
    note_launch();
    return;
  }
  for (int p = 0; p < KT::kPasses; ++p) {
    uint32_t* status = reinterpret_cast<uint32_t*>(ws + L.status_sort) + (uint64_t)p * ntiles * 256;
    launch_k(k_onesweep<KT, NT, ITEMS>, (unsigned)ntiles, NT, dsmem, st, 
        D, ws + L.keys0, ws + L.keys1, reinterpret_cast<uint32_t*>(ws + L.vals0),
        reinterpret_cast<uint32_t*>(ws + L.vals1), n, n_dev, p, plan, status, counters + CNT_SORT + p);
    note_launch();
  }
}

template <class KT>
cudaError_t run(const dm_column_in* in, char* ws, const WsLayout& L, void* udict, uint32_t* rank, dm_header* hdr,
                cudaStream_t st, bool probe) {
  const uint64_t n = in->n_delta;
  uint32_t* counters = reinterpret_cast<uint32_t*>(ws + L.counters);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist);
  SortPlan* plan = reinterpret_cast<SortPlan*>(ws + L.plan);
  // Sorted input: D itself, or (dedup) its distinct values dkeys, whose count
  // n_dist exists on the device only; ranks then go to rank_of_id first.
  const void* D = in->delta;
  const unsigned long long* n_dev = nullptr;
  uint32_t* sort_rank = rank;
  if (probe) {  // NEXT1: only the values not in U_M are sorted
    unsigned long long* n_new = reinterpret_cast<unsigned long long*>(counters + CNT_PROBE);
    const int sms = device_sms();
    uint32_t* table = reinterpret_cast<uint32_t*>(ws + L.pf_table);
    cudaMemsetAsync(table, 0xff, L.pf_cap * 4, st);
    const PfTag tg = PfTag::make(in->dict_len);
    launch_k(k_pf_build<KT>, (unsigned)std::min<uint64_t>((in->dict_len + 255) / 256, (uint64_t)sms * 8), 256, 0, st,
             in->main_dict, in->dict_len, table, L.pf_cap - 1, tg);
    launch_k(k_pf_probe<KT>, (unsigned)std::min<uint64_t>((n + 1023) / 1024, (uint64_t)sms * 8), kPfThreads, 0, st,
             in->main_dict, (const uint32_t*)table, L.pf_cap - 1, in->delta, n,
             reinterpret_cast<uint32_t*>(ws + L.pf_src), (void*)(ws + L.pf_keys), n_new,
             reinterpret_cast<uint32_t*>(ws + L.pf_used), tg);
    note_launch(2);
    D = ws + L.pf_keys;
    n_dev = n_new;
    sort_rank = reinterpret_cast<uint32_t*>(ws + L.pf_rank);
  } else if (L.dedup) {
    unsigned long long* n_dist = reinterpret_cast<unsigned long long*>(counters + CNT_DEDUP);
    const int sms = device_sms();
    launch_k(k_dedup_insert<KT>, (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 8), 256, 0, st, 
        in->delta, n, reinterpret_cast<uint64_t*>(ws + L.dd_slots), L.dd_cap - 1, ws + L.dd_keys,
        reinterpret_cast<uint32_t*>(ws + L.dd_tid), n_dist);
    note_launch();
    D = ws + L.dd_keys;
    n_dev = n_dist;
    sort_rank = reinterpret_cast<uint32_t*>(ws + L.dd_rank);
  }
  const BucketState* gate = nullptr;
  if (L.bucket) {
    BucketState* bst = reinterpret_cast<BucketState*>(ws + L.bk_state);
    uint32_t* off = reinterpret_cast<uint32_t*>(ws + L.bk_off);
    uint32_t* cur = reinterpret_cast<uint32_t*>(ws + L.bk_cur);
    const uint64_t nb = 1ull << L.bk_bits;
    const int sms = device_sms();
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 8));
    const unsigned g_range = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((std::max<uint64_t>(n, nb) + 255) / 256, (uint64_t)sms * 8));
    launch_k(k_bk_range<KT>, g_range, 256, 0, st, D, n, n_dev, bst, off, L.bk_bits, plan);
    launch_k(k_bk_count<KT>, g, 256, 0, st, D, n, n_dev, (const BucketState*)bst, off, L.bk_bits);
    launch_k(k_bk_scan, (unsigned)(nb / (256 * kBkScanItems)), 256, 0, st, off, cur, nb,
             reinterpret_cast<uint64_t*>(ws + L.bk_status), counters + CNT_BKSCAN, bst);
    void* const scat = KT::kBytes <= 8 ? (void*)(ws + L.bk_pairs) : (void*)(ws + L.keys1);
    launch_k(k_bk_scatter<KT>, g, 256, 0, st, D, n, n_dev, (const BucketState*)bst, cur, L.bk_bits,
             scat, reinterpret_cast<uint32_t*>(ws + L.vals1));
    launch_k(k_bk_local<KT>, g, 256, 0, st, (const void*)scat,
             reinterpret_cast<const uint32_t*>(ws + L.vals1), n, n_dev, (const BucketState*)bst,
             (const uint32_t*)off, L.bk_bits, (void*)(ws + L.keys0), reinterpret_cast<uint32_t*>(ws + L.vals0));
    note_launch(5);
    gate = bst;
  }
  const int hist_blocks = (int)std::min<uint64_t>((n + 4095) / 4096, 148 * 4);
  launch_k(k_hist<KT>, hist_blocks, 256, 0, st, D, n, n_dev, hist, counters + CNT_HIST, plan, gate);
  note_launch();
  constexpr bool U64 = KT::kBytes <= 8;  // tile shape: 8-byte and 4-byte keys alike
  switch (sort_variant()) {  // must match sort_tile_keys() (workspace layout)
    case 1: launch_passes<KT, 256, U64 ? 16 : 8>(D, n, n_dev, ws, L, plan, counters, st); break;
    case 2: launch_passes<KT, 256, U64 ? 8 : 4>(D, n, n_dev, ws, L, plan, counters, st); break;
    case 3: launch_passes<KT, 1024, U64 ? 8 : 4>(D, n, n_dev, ws, L, plan, counters, st); break;
    default: launch_passes<KT, 512, U64 ? 16 : 8>(D, n, n_dev, ws, L, plan, counters, st); break;
  }
  const uint64_t utiles = (n + kUniqThreads * kUniqItems - 1) / (kUniqThreads * kUniqItems);
  launch_k(k_unique<KT>, (unsigned)utiles, kUniqThreads, 0, st, 
      D, ws + L.keys0, ws + L.keys1, reinterpret_cast<const uint32_t*>(ws + L.vals0),
      reinterpret_cast<const uint32_t*>(ws + L.vals1), n, n_dev, plan,
      reinterpret_cast<uint64_t*>(ws + L.status_unique), counters + CNT_UNIQUE, udict, sort_rank, hdr);
  note_launch();
  if (L.dedup && !probe) {
    const int sms = device_sms();
    launch_k(k_dedup_ranks, (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 8), 256, 0, st, 
        reinterpret_cast<const uint32_t*>(ws + L.dd_tid), sort_rank, n, rank);
    note_launch();
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_delta_dictionary(const dm_column_in* in, char* ws, const WsLayout& L, void* udict, uint32_t* rank,
                                    dm_header* hdr, cudaStream_t st, bool probe) {
  if (in->n_delta == 0) return cudaSuccess;
  switch (in->key) {
    case DM_KEY_U64: return run<KeyU64>(in, ws, L, udict, rank, hdr, st, probe);
    case DM_KEY_U32: return run<KeyU32>(in, ws, L, udict, rank, hdr, st, probe);
    default: return run<KeyB16>(in, ws, L, udict, rank, hdr, st, probe);
  }
}

cudaError_t launch_probe_codes(const dm_column_in* in, char* ws, const WsLayout& L, const uint32_t* xm,
                               const uint32_t* xd, dm_header* hdr, cudaStream_t st) {
  if (in->n_delta == 0) return cudaSuccess;
  const uint64_t nwords = (in->dict_len + 31) / 32;
  const unsigned g = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>((std::max<uint64_t>(in->n_delta, nwords) + 255) / 256, (uint64_t)device_sms() * 8));
  launch_k(k_pf_codes, g, 256, 0, st, reinterpret_cast<const uint32_t*>(ws + L.pf_src), in->n_delta,
           reinterpret_cast<const uint32_t*>(ws + L.pf_rank), xm, xd, reinterpret_cast<uint32_t*>(ws + L.pf_codes),
           reinterpret_cast<const uint32_t*>(ws + L.pf_used), nwords, hdr);
  note_launch();
  return cudaGetLastError();
}

}  // namespace dm
