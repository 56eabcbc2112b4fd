// dict_merge.cu -- Step 1(b) and Step 2(a) on the GPU: merge U_M with U_D.
//
// Paper, Step 1(b): walk the two sorted dictionaries with two
// pointers, append the smaller value, record its output index in X_M or X_D;
// equal heads are appended once and both tables get the same index.  Parallel
// form: split both inputs at quantiles, merge locally while dropping
// the duplicate that can straddle a split, count the uniques per thread,
// prefix-sum the counts, then re-merge writing at the offsets.
//
// GPU form -- the paper's three phases with 2048-element merge-path tiles in
// place of threads:
//   k_partition    merge-path co-ranks at every tile diagonal (the quantile
//                  split, [8][5] in P:302), one warp per boundary, 32-way search
//   k_merge_count  phase 1: per tile, stage both ranges in shared memory and
//                  rank the smaller side inside the larger (TileRank below); a
//                  U_D value equal to the U_M value right before it in merged
//                  order is the duplicate (ties take U_M first -- the GPU form of
//                  P:304's boundary check); the tile's duplicate count is stored
//   k_scan_counts  phase 2: prefix sum of the counts; writes |U'|, b'
//   k_merge_write  phase 3: rank again and write U', X_M, X_D at the offsets
// Measured alternatives: a per-thread co-rank + serial merge (the CPU pattern)
// cost ~160 instructions per element; a single pass with decoupled look-back
// was 1% faster on cfg2 but 11% slower on cfg5 (look-back chains at 5e5 tiles).
#include <algorithm>

#include "dm_device.cuh"

namespace dm {
namespace {

__device__ __forceinline__ uint32_t dev_width(uint64_t n) { return n <= 1 ? 1u : 64u - __clzll(n - 1); }

// Merge-path co-rank of diagonal d by one warp: number of U_M elements among the
// first d merged elements (U_M first on ties).  32 probes per round (ballot), so a
// 2^24-wide range resolves in ~5 dependent round trips instead of 24.
template <class KT>
__global__ void __launch_bounds__(256) k_partition(const void* __restrict__ A, uint64_t nA,
                                                   const void* __restrict__ B, const dm_header* __restrict__ hdr,
                                                   uint64_t nparts, uint64_t* __restrict__ part) {
  pdl_prologue();
  const uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const unsigned lane = lane_id();
  if (t >= nparts) return;
  const uint64_t nB = hdr->delta_dict_len;
  const uint64_t d = umin64(t * (uint64_t)kMergeTile, nA + nB);
  uint64_t lo = d > nB ? d - nB : 0, hi = d < nA ? d : nA;
  while (hi > lo) {
    const uint64_t span = hi - lo;
    const uint64_t ik = lo + span * lane / 32;
    const bool cond = KT::le(KT::load(A, ik), KT::load(B, d - ik - 1));
    const unsigned c = __popc(__ballot_sync(FULL, cond));
    const uint64_t nlo = c ? lo + span * (c - 1) / 32 + 1 : lo;
    const uint64_t nhi = c < 32 ? lo + span * c / 32 : hi;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) part[t] = lo;
}

// ---------------------------------------------------------------- tile ranking
// One merge-path tile = A[i0, i1) (U_M) and B[j0, j1) (U_D): exactly the
// elements at merged positions [d0, d1).  Instead of a serial per-thread merge,
// each tile ranks its SMALLER side inside the larger one by binary search, and
// one shared-memory scan over the larger side turns those ranks into every
// element's merged position.  Equal values: U_M first; a U_D
// value whose twin is the U_M element right before it in merged order is a
// duplicate -- dropped from U', its X_D is the twin's index.  For U_D-sparse
// tiles (cfg2, cfg5) the work per U_M element is a few instructions.
//
//   q_j   = #{tile A <= B[j]}          (tile U_M elements merged before B[j])
//   nB(a) = #{tile B <  A[a]}          (tile U_D elements merged before A[a])
//   dup_j = B[j] equals a U_M value (in the tile, or A[i0-1] for j = 0)
//   E[j]  = #{dup_k : k < j}           (exclusive; E[nb] = the tile's duplicates)
//   pos(A[a]) = d0 + a + nB(a) - D0 - #{dup B < A[a]}
//   pos(B[j]) = d0 + j + q_j  - D0 - E[j]          (non-duplicate)
//   X_D[j]    = d0 + j + q_j - 1 - D0 - E[j]       (duplicate: its twin's index)
// with D0 = duplicates dropped by earlier tiles (phase 2's prefix sum).
__device__ __forceinline__ uint32_t odd_seg(uint32_t n, uint32_t nt) {
  const uint32_t s = (n + nt - 1) / nt;
  return s | 1u;  // odd segment length: conflict-free blocked access
}

// In-place block scan of n u32 in shared memory (NT threads).  exclusive: a[n]
// receives the total (the array must have n + 1 slots).
template <int NT>
__device__ __forceinline__ void smem_scan(uint32_t* a, uint32_t n, bool exclusive, uint32_t* s_warp) {
  const uint32_t seg = odd_seg(n, NT);
  const uint32_t b0 = umin32(threadIdx.x * seg, n), b1 = umin32(b0 + seg, n);
  uint32_t sum = 0;
  for (uint32_t k = b0; k < b1; ++k) sum += a[k];
  uint32_t total;
  uint32_t run = block_exclusive_scan<NT>(sum, s_warp, total);
  for (uint32_t k = b0; k < b1; ++k) {
    const uint32_t v = a[k];
    a[k] = exclusive ? run : run + v;
    run += v;
  }
  if (exclusive && threadIdx.x == 0) a[n] = total;
  __syncthreads();
}

template <class KT>
struct TileRank {
  using K = typename KT::K;
  uint64_t d0, i0, j0;
  uint32_t na, nb;
  bool has_prev, small_b;
  K* sk;         // [0] = A[i0-1], [1 .. na] = A tile, [na+1 .. na+nb] = B tile
  uint32_t* sc;  // small_b: packed (#B | #dupB << 16) scan over A slots; else #A scan over B slots
  uint32_t* sq;  // small_b: q_j per B; else c_a = #{tile B < A[a]} per A
  uint32_t* se;  // dup flags over B, then their exclusive scan (nb + 1 slots)

  __device__ __forceinline__ K A_(uint32_t a) const { return sk[1 + a]; }
  __device__ __forceinline__ K B_(uint32_t j) const { return sk[1 + na + j]; }

  // smem: keys (kMergeTile + 1), then three u32 arrays of (kMergeTile + 2)
  __device__ __forceinline__ bool setup(const void* A, uint64_t nA, const void* B, uint64_t nB,
                                        const uint64_t* part, uint64_t tile, unsigned char* smem,
                                        uint32_t* s_warp) {
    constexpr uint32_t T = kMergeTile;
    const uint64_t total = nA + nB;
    d0 = tile * T;
    if (d0 >= total) return false;
    const uint64_t d1 = umin64(d0 + T, total);
    i0 = part[tile];
    const uint64_t i1 = part[tile + 1];
    j0 = d0 - i0;
    na = (uint32_t)(i1 - i0);
    nb = (uint32_t)((d1 - i1) - j0);
    has_prev = i0 > 0;
    small_b = nb <= na;
    sk = reinterpret_cast<K*>(smem);
    sc = reinterpret_cast<uint32_t*>(sk + (T + 1));
    sq = sc + (T + 2);
    se = sq + (T + 2);
    if (threadIdx.x == 0 && has_prev) sk[0] = KT::load(A, i0 - 1);
    {
      // na + nb <= kMergeTile: at most kMergeItems strided slots per thread; all
      // loads are issued before the first shared store (branch-free, clamped).
      K v[kMergeItems];
#pragma unroll
      for (int r = 0; r < kMergeItems; ++r) {
        const uint32_t k = threadIdx.x + r * kMergeThreads;
        const bool in_a = k < na || nb == 0;  // tile is non-empty, so one side exists
        v[r] = in_a ? KT::load(A, i0 + umin32(k, na - 1)) : KT::load(B, j0 + umin32(k - na, nb - 1));
      }
#pragma unroll
      for (int r = 0; r < kMergeItems; ++r) {
        const uint32_t k = threadIdx.x + r * kMergeThreads;
        if (k < na + nb) sk[1 + k] = v[r];
      }
    }
    const uint32_t nc = (small_b ? na : nb) + 1;
    for (uint32_t k = threadIdx.x; k < nc; k += kMergeThreads) sc[k] = 0;
    for (uint32_t k = threadIdx.x; k <= nb; k += kMergeThreads) se[k] = 0;
    __syncthreads();
    if (small_b) {
      for (uint32_t j = threadIdx.x; j < nb; j += kMergeThreads) {
        const K v = B_(j);
        uint32_t lo = 0, hi = na;  // upper bound: #{A <= v}
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (KT::le(A_(mid), v))
            lo = mid + 1;
          else
            hi = mid;
        }
        const bool dup = lo > 0 ? KT::eq(A_(lo - 1), v) : (has_prev && KT::eq(sk[0], v));
        sq[j] = lo;
        se[j] = dup;
        atomicAdd(&sc[lo], 1u + ((uint32_t)dup << 16));
      }
      __syncthreads();
      smem_scan<kMergeThreads>(sc, na + 1, false, s_warp);
    } else {
      for (uint32_t a = threadIdx.x; a < na; a += kMergeThreads) {
        const K v = A_(a);
        uint32_t lo = 0, hi = nb;  // lower bound: #{B < v}
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (KT::lt(B_(mid), v))
            lo = mid + 1;
          else
            hi = mid;
        }
        sq[a] = lo;
        if (lo < nb && KT::eq(B_(lo), v)) se[lo] = 1;
        atomicAdd(&sc[lo], 1u);
      }
      if (threadIdx.x == 0 && has_prev && nb > 0 && KT::eq(B_(0), sk[0])) se[0] = 1;
      __syncthreads();
      smem_scan<kMergeThreads>(sc, nb, false, s_warp);
    }
    smem_scan<kMergeThreads>(se, nb, true, s_warp);
    return true;
  }
  __device__ __forceinline__ uint32_t dups() const { return se[nb]; }
  // tile U_D elements (all / duplicates) merged before A[a]
  __device__ __forceinline__ void a_rank(uint32_t a, uint32_t& nbb, uint32_t& dupb) const {
    if (small_b) {
      const uint32_t x = sc[a];
      nbb = x & 0xffffu;
      dupb = x >> 16;
    } else {
      nbb = sq[a];
      dupb = se[nbb];
    }
  }
  __device__ __forceinline__ uint32_t b_q(uint32_t j) const { return small_b ? sq[j] : sc[j]; }
};

__device__ __forceinline__ size_t tile_smem_bytes(size_t key_bytes) {
  return key_bytes * (kMergeTile + 1) + 3 * sizeof(uint32_t) * (kMergeTile + 2);
}

// Phase 1: per tile, the number of duplicates it drops.
template <class KT>
__global__ void __launch_bounds__(kMergeThreads) k_merge_count(const void* __restrict__ A, uint64_t nA,
                                                               const void* __restrict__ B,
                                                               const uint64_t* __restrict__ part,
                                                               const dm_header* __restrict__ hdr,
                                                               uint32_t* __restrict__ cnt) {
  pdl_prologue();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_warp[kMergeThreads / 32 + 1];
  TileRank<KT> tr;
  const uint64_t tile = blockIdx.x;
  if (!tr.setup(A, nA, B, hdr->delta_dict_len, part, tile, smem_raw, s_warp)) {
    if (threadIdx.x == 0) cnt[tile] = 0;
    return;
  }
  if (threadIdx.x == 0) cnt[tile] = tr.dups();
}

// Phase 2: exclusive prefix sum of the per-tile counts (single pass,
// decoupled look-back over 2048-count blocks); the block holding the last count
// writes |U'| and b' = w(|U'|) (Eq 4) into the result header.
__global__ void __launch_bounds__(256) k_scan_counts(const uint32_t* __restrict__ cnt, uint64_t n,
                                                     uint64_t* __restrict__ excl, uint64_t* status, uint32_t* counter,
                                                     uint64_t nA, dm_header* hdr) {
  pdl_prologue();
  constexpr int ITEMS = 8, TILE = 256 * ITEMS;
  __shared__ uint32_t s_warp[9];
  __shared__ uint64_t s_excl;
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t p0 = tile * TILE + threadIdx.x * ITEMS;
  uint32_t v[ITEMS], sum = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    v[i] = p0 + i < n ? cnt[p0 + i] : 0u;
    sum += v[i];
  }
  uint32_t tile_sum;
  const uint32_t texcl = block_exclusive_scan<256>(sum, s_warp, tile_sum);
  if (threadIdx.x < 32) {
    const uint64_t e = lookback_exclusive(status, tile, tile_sum);
    if (threadIdx.x == 0) s_excl = e;
  }
  __syncthreads();
  uint64_t run = s_excl + texcl;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (p0 + i < n) excl[p0 + i] = run;
    run += v[i];
  }
  if ((tile + 1) * TILE >= n && threadIdx.x == 255) {  // the block holding the last count
    const uint64_t m = nA + hdr->delta_dict_len - run;
    hdr->merged_dict_len = m;
    hdr->merged_bits = dev_width(m);
    if (m > (1ull << 32)) atomicMin(&hdr->status, (int)DM_E_TOO_WIDE);
  }
}

// Phase 3: rank each tile again and write U', X_M, X_D at the offsets.
template <class KT>
__global__ void __launch_bounds__(kMergeThreads) k_merge_write(const void* __restrict__ A, uint64_t nA,
                                                               const void* __restrict__ B,
                                                               const uint64_t* __restrict__ part,
                                                               const uint64_t* __restrict__ excl,
                                                               void* __restrict__ U, uint32_t* __restrict__ XM,
                                                               uint32_t* __restrict__ XD, dm_header* hdr,
                                                               uint32_t* __restrict__ rblk,
                                                               uint8_t* __restrict__ offs, uint32_t xs) {
  pdl_prologue();
  using K = typename KT::K;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_warp[kMergeThreads / 32 + 1];
  TileRank<KT> tr;
  const uint64_t tile = blockIdx.x;
  const uint64_t D0 = excl[tile];  // issued early; consumed after the ranking
  if (!tr.setup(A, nA, B, hdr->delta_dict_len, part, tile, smem_raw, s_warp)) return;
  const uint64_t base = tr.d0 - D0;  // first U' index this tile writes
  // U' is written directly: consecutive U_M elements land at consecutive slots
  // except at the (few, for U_D-sparse tiles) insertion points.
  bool unsorted = false;
  for (uint32_t a = threadIdx.x; a < tr.na; a += kMergeThreads) {
    uint32_t nbb, dupb;
    tr.a_rank(a, nbb, dupb);
    const uint32_t o = a + nbb - dupb;  // tile-local U' slot
    const K v = tr.A_(a);
    const uint64_t i = tr.i0 + a, u = base + o;
    KT::store(U, u, v);
    XM[i] = (uint32_t)u;
    if (rblk) {
      // XC: R(g) = #{new values with insertion point p <= 256g} = X_M[256g] - 256g,
      // and after the last main entry (the end of the last list).
      if ((i & ((1u << xs) - 1)) == 0) rblk[i >> xs] = (uint32_t)(u - i);
      if (i == nA - 1) rblk[(nA + (1u << xs) - 1) >> xs] = (uint32_t)(u - i);
    }
    // strictly increasing U_M over the pairs this tile owns
    if ((a > 0 || tr.has_prev) && !KT::lt(a > 0 ? tr.A_(a - 1) : tr.sk[0], v)) unsorted = true;
  }
  for (uint32_t j = threadIdx.x; j < tr.nb; j += kMergeThreads) {
    const uint32_t e = tr.se[j];
    const bool dup = tr.se[j + 1] != e;
    const uint32_t o = j + tr.b_q(j) - e;  // tile-local merged slot minus earlier drops
    if (dup) {
      XD[tr.j0 + j] = (uint32_t)(base + o - 1);  // its U_M twin's index
    } else {
      KT::store(U, base + o, tr.B_(j));
      XD[tr.j0 + j] = (uint32_t)(base + o);
      if (offs) {
        // a new value: inserted before U_M[p], p = #U_M below it; it is the
        // (u - p)-th new value in sorted order.  It raises X_M[c] for c >= p;
        // stored in the list of the block holding p - 1 (blocks own (256g, 256g+256])
        const uint64_t p = tr.i0 + tr.b_q(j);
        offs[base + o - p] = (uint8_t)((p - 1) & ((1u << xs) - 1));
      }
    }
  }
  if (__any_sync(FULL, unsorted) && lane_id() == 0) atomicMin(&hdr->status, (int)DM_E_UNSORTED);
}

// ------------------------------------------------------------ single-pass merge
// One merge-path tile per CTA (tiles claimed in order), all of Step 1(b) in one
// pass: the tile's smaller side S is binary-searched in its larger side G
// (q = #G before it), which fixes every S element's slot in the tile's share
// of U'; those slots are set in a 2048-bit bitmap, and the G elements fill the
// remaining slots in order -- slot p holds G element p - #{S slots < p}, one
// popcount per element.  The tile's duplicate count (a U_D value equal to a
// U_M value) is published as soon as it is known and the
// exclusive count of earlier tiles arrives by decoupled look-back (the GPU
// form of P:302-308's counts + prefix sum, without the second pass).
//   small side B (U_D sparse; cfg2, cfg5): q_j = #{A <= B_j}, dup_j = B_j equals
//       the A before it; E = exclusive scan of dup over B; slot(B_j) = j + q_j - E_j
//   small side A (U_D dense): l_a = #{B < A_a}; B_l is a dup if it equals A_a;
//       E over B as above; slot(A_a) = a + l_a - E[l_a]; non-dup B fill the rest
// MODE 0: single pass (look-back); 1: count pass only (writes cnt[tile]);
// 2: write pass with the exclusive counts excl[] of k_scan_counts.
template <class KT, int MODE>
__global__ void __launch_bounds__(kMergeThreads) k_merge(const void* __restrict__ A, uint64_t nA,
                                                         const void* __restrict__ B,
                                                         const uint64_t* __restrict__ part, uint64_t ntiles,
                                                         uint64_t* status, uint32_t* counter,
                                                         uint32_t* __restrict__ cnt,
                                                         const uint64_t* __restrict__ excl,
                                                         void* __restrict__ U, uint32_t* __restrict__ XM,
                                                         uint32_t* __restrict__ XD, dm_header* hdr,
                                                         uint32_t* __restrict__ rblk, uint8_t* __restrict__ offs,
                                                         uint32_t xs) {
  pdl_prologue();
  using K = typename KT::K;
  constexpr uint32_t T = kMergeTile, NT = kMergeThreads, IT = kMergeItems, NW = T / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* sk = reinterpret_cast<K*>(smem_raw);                      // [0] = A[i0-1], A tile, B tile
  uint32_t* sq = reinterpret_cast<uint32_t*>(sk + (T + 1));    // per S element: q (or l)
  uint32_t* se = sq + T;                                       // dup flags over B -> exclusive scan (+1)
  uint32_t* snd = se + (T + 1);                                // dense case: non-dup B indices
  __shared__ uint32_t s_bm[NW], s_wpre[NW];
  __shared__ uint32_t s_warp[NT / 32 + 1];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_D0;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;

  if (MODE == 0 && threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  for (uint32_t w = threadIdx.x; w < NW; w += NT) s_bm[w] = 0;
  __syncthreads();
  const uint64_t tile = MODE == 0 ? (uint64_t)s_tile : (uint64_t)blockIdx.x;
  const uint64_t nB = hdr->delta_dict_len, total = nA + nB;
  // the grid is sized from N_D >= |U_D|: surplus CTAs claim the last ids, after
  // every real tile, so nothing waits on them
  const uint64_t nreal = (total + T - 1) / T;
  if (tile >= nreal) {
    if (MODE == 1 && threadIdx.x == 0) cnt[tile] = 0;
    return;
  }
  const uint64_t d0 = tile * T, d1 = umin64(d0 + T, total);
  const uint64_t i0 = part[tile], i1 = part[tile + 1], j0 = d0 - i0;
  const uint32_t na = (uint32_t)(i1 - i0), nb = (uint32_t)((d1 - i1) - j0);
  DM_ASSERT(tile < ntiles && nreal <= ntiles && i1 >= i0 && i1 <= nA && d1 >= i1 + j0 && na + nb <= T && j0 + nb <= nB,
            "tile %llu i0 %llu i1 %llu j0 %llu na %u nb %u nA %llu nB %llu", (unsigned long long)tile,
            (unsigned long long)i0, (unsigned long long)i1, (unsigned long long)j0, na, nb, (unsigned long long)nA,
            (unsigned long long)nB);
  const bool has_prev = i0 > 0;
  auto A_ = [&](uint32_t a) -> K { return sk[1 + a]; };
  auto B_ = [&](uint32_t j) -> K { return sk[1 + na + j]; };
  {
    K v[IT];
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      const uint32_t k = threadIdx.x + r * NT;
      const bool in_a = k < na || nb == 0;
      v[r] = (na + nb == 0) ? K{} : in_a ? KT::load(A, i0 + umin32(k, na - 1)) : KT::load(B, j0 + umin32(k - na, nb - 1));
    }
    if (threadIdx.x == 0 && has_prev) sk[0] = KT::load(A, i0 - 1);
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      const uint32_t k = threadIdx.x + r * NT;
      if (k < na + nb) sk[1 + k] = v[r];
    }
  }
  const bool small_b = nb <= na;
  if constexpr (MODE == 1) {
    // count pass: only the tile's duplicate count (each U_D value matches at
    // most one U_M value) -- no slot arrays, so the launch takes the key
    // staging only and more tiles are resident per SM
    __syncthreads();
    uint32_t c = 0;
    if (small_b) {
      for (uint32_t j = threadIdx.x; j < nb; j += NT) {
        const K v = B_(j);
        uint32_t lo = 0, hi = na;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (KT::le(A_(mid), v)) lo = mid + 1; else hi = mid;
        }
        c += (lo > 0 ? KT::eq(A_(lo - 1), v) : (has_prev && KT::eq(sk[0], v))) ? 1u : 0u;
      }
    } else {
      for (uint32_t a = threadIdx.x; a < na; a += NT) {
        const K v = A_(a);
        uint32_t lo = 0, hi = nb;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (KT::lt(B_(mid), v)) lo = mid + 1; else hi = mid;
        }
        c += (lo < nb && KT::eq(B_(lo), v)) ? 1u : 0u;
      }
      if (threadIdx.x == 0 && has_prev && nb > 0 && KT::eq(B_(0), sk[0])) ++c;
    }
    uint32_t tot;
    block_exclusive_scan<NT>(c, s_warp, tot);
    if (threadIdx.x == 0) cnt[tile] = tot;
    return;
  }
  for (uint32_t k = threadIdx.x; k <= nb; k += NT) se[k] = 0;
  __syncthreads();
  if (small_b) {
    for (uint32_t j = threadIdx.x; j < nb; j += NT) {
      const K v = B_(j);
      uint32_t lo = 0, hi = na;  // upper bound: #{A <= v}
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (KT::le(A_(mid), v)) lo = mid + 1; else hi = mid;
      }
      sq[j] = lo;
      se[j] = lo > 0 ? KT::eq(A_(lo - 1), v) : (has_prev && KT::eq(sk[0], v));
    }
  } else {
    for (uint32_t a = threadIdx.x; a < na; a += NT) {
      const K v = A_(a);
      uint32_t lo = 0, hi = nb;  // lower bound: #{B < v}
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (KT::lt(B_(mid), v)) lo = mid + 1; else hi = mid;
      }
      sq[a] = lo;
      if (lo < nb && KT::eq(B_(lo), v)) se[lo] = 1;
    }
    if (threadIdx.x == 0 && has_prev && nb > 0 && KT::eq(B_(0), sk[0])) se[0] = 1;
  }
  __syncthreads();
  // exclusive scan of the dup flags over B (blocked, IT per thread); se[nb] = total
  {
    const uint32_t b0 = umin32(threadIdx.x * IT, nb), b1 = umin32(b0 + IT, nb);
    uint32_t f[IT], sum = 0;
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      f[r] = b0 + r < b1 ? se[b0 + r] : 0u;
      sum += f[r];
    }
    uint32_t tot;
    uint32_t run = block_exclusive_scan<NT>(sum, s_warp, tot);
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      if (b0 + r < b1) se[b0 + r] = run;
      run += f[r];
    }
    if (threadIdx.x == 0) se[nb] = tot;
  }
  __syncthreads();
  const uint32_t dups = se[nb];
  if (MODE == 0 && warp == 0) {
    const uint64_t e = lookback_exclusive(status, tile, dups);
    if (lane == 0) s_D0 = e;
  }
  if (MODE == 2 && threadIdx.x == 0) s_D0 = excl[tile];
  // meanwhile: the small side's slots into the bitmap (independent of D0)
  if (small_b) {
    for (uint32_t j = threadIdx.x; j < nb; j += NT) {
      if (se[j + 1] == se[j]) {
        const uint32_t slot = j + sq[j] - se[j];
        atomicOr(&s_bm[slot >> 5], 1u << (slot & 31));
      }
    }
  } else {
    for (uint32_t a = threadIdx.x; a < na; a += NT) {
      const uint32_t l = sq[a], slot = a + l - se[l];
      atomicOr(&s_bm[slot >> 5], 1u << (slot & 31));
    }
    for (uint32_t j = threadIdx.x; j < nb; j += NT)
      if (se[j + 1] == se[j]) snd[j - se[j]] = j;
  }
  __syncthreads();
  if (warp == 1 || (NT == 32)) {  // word prefix of the bitmap (NW = 64 words, 2 per lane)
    const uint32_t c0 = __popc(s_bm[2 * lane]), c1 = __popc(s_bm[2 * lane + 1]);
    uint32_t x = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= (unsigned)o) x += y;
    }
    s_wpre[2 * lane] = x - c0 - c1;
    s_wpre[2 * lane + 1] = x - c1;
  }
  __syncthreads();
  const uint64_t D0 = s_D0;
  const uint64_t base = d0 - D0;  // U' index of the tile's first slot
  const uint32_t nU = na + nb - dups;
  DM_ASSERT(D0 <= j0 && dups <= nb, "tile %llu D0 %llu j0 %llu dups %u nb %u", (unsigned long long)tile,
            (unsigned long long)D0, (unsigned long long)j0, dups, nb);
  const unsigned lt = lanemask_lt();
  bool unsorted = false;
  // 32-bit per-element index math from tile-base pointers (U', X_M) and
  // per-tile constants (the write pass is issue-bound); sk[g] is the element
  // before A_(g) (sk[0] = A[i0 - 1]), so the sortedness check needs no select
  void* const Ub = static_cast<char*>(U) + base * (uint64_t)KT::kBytes;  // U' from the tile's first slot
  uint32_t* const XMt = XM + i0;  // XM == nullptr: X_M is not materialised (see launch_dictionary_merge)
  const uint32_t bmask = (1u << xs) - 1, i0lo = (uint32_t)i0, ub32 = (uint32_t)base;
  const uint32_t dU = (uint32_t)(base - i0);  // U' index - U_M index of the tile's first A slot
  const uint32_t glast = nA > i0 && nA <= i1 ? (uint32_t)(nA - 1 - i0) : 0xffffffffu;
  const uint32_t hp = has_prev ? 1u : 0u;
  auto sample = [&](uint32_t a, uint32_t r32) {  // XC block samples R(g) = X_M[256 g] - 256 g
    if (((i0lo + a) & bmask) == 0) rblk[(i0 + a) >> xs] = r32;
    if (a == glast) rblk[(nA + bmask) >> xs] = r32;
  };
  // fill: slot p not taken by S holds the (p - #S slots before p)-th G element
  if (small_b) {
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      const uint32_t p = r * NT + threadIdx.x;
      if (p >= nU) break;
      const uint32_t bits = s_bm[p >> 5];
      if ((bits >> lane) & 1u) continue;
      const uint32_t g = p - (s_wpre[p >> 5] + __popc(bits & lt));  // minus the S slots before p
      DM_ASSERT(g < na, "fill tile %llu p %u g %u na %u", (unsigned long long)tile, p, g, na);
      const K v = sk[1 + g];
      KT::store(Ub, p, v);
      if (XM) XMt[g] = ub32 + p;
      if (rblk) sample(g, dU + p - g);
      if ((g | hp) && !KT::lt(sk[g], v)) unsorted = true;
    }
  } else {
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      const uint32_t p = r * NT + threadIdx.x;
      if (p >= nU) break;
      const uint32_t bits = s_bm[p >> 5];
      if ((bits >> lane) & 1u) continue;
      const uint32_t before = s_wpre[p >> 5] + __popc(bits & lt);  // S slots before p
      const uint32_t g = p - before;
      DM_ASSERT(g < nb - dups, "fill tile %llu p %u g %u nb %u dups %u", (unsigned long long)tile, p, g, nb, dups);
      const uint32_t j = snd[g];
      KT::store(Ub, p, B_(j));
      XD[j0 + j] = ub32 + p;
      if (offs) offs[(uint64_t)(dU + p - before)] = (uint8_t)((i0lo + before - 1) & bmask);  // P = i0 + before
    }
  }
  // the small side
  if (small_b) {
    for (uint32_t j = threadIdx.x; j < nb; j += NT) {
      const uint32_t e = se[j];
      if (se[j + 1] != e) {
        XD[j0 + j] = (uint32_t)(base + sq[j] - 1 + (j - e));  // its U_M twin's slot
      } else {
        const uint32_t slot = j + sq[j] - e;
        const uint64_t u = base + slot;
        KT::store(U, u, B_(j));
        XD[j0 + j] = (uint32_t)u;
        if (offs) {
          const uint64_t P = i0 + sq[j];
          offs[u - P] = (uint8_t)((P - 1) & ((1u << xs) - 1));
        }
      }
    }
  } else {
    for (uint32_t a = threadIdx.x; a < na; a += NT) {
      const uint32_t l = sq[a], slot = a + l - se[l];
      const K v = sk[1 + a];
      KT::store(Ub, slot, v);
      if (XM) XMt[a] = ub32 + slot;
      if (l < nb && se[l + 1] != se[l] && KT::eq(B_(l), v)) XD[j0 + l] = ub32 + slot;
      if (rblk) sample(a, dU + slot - a);
      if ((a | hp) && !KT::lt(sk[a], v)) unsorted = true;
    }
    if (threadIdx.x == 0 && has_prev && nb > 0 && KT::eq(B_(0), sk[0])) XD[j0] = (uint32_t)(base - 1);
  }
  if (__any_sync(FULL, unsorted) && lane == 0) atomicMin(&hdr->status, (int)DM_E_UNSORTED);
  if (tile == nreal - 1 && threadIdx.x == 0) {
    const uint64_t m = total - (D0 + dups);
    hdr->merged_dict_len = m;
    hdr->merged_bits = dev_width(m);
    if (m > (1ull << 32)) atomicMin(&hdr->status, (int)DM_E_TOO_WIDE);
  }
}

// ------------------------------------------------- sparse deltas: U_M tiles
// When U_D is much smaller than U_M (cfg2: 1e6 vs 1e7; cfg5: 5e7 vs 1.07e9),
// the merge is a copy of U_M with a few insertions.  Tile over U_M alone: tile
// t = U_M[a, a + T) and the U_D values in [U_M[a], U_M[a + T)) (its "slice",
// found by k_sp_partition; the first tile also takes the values below U_M[0],
// the last the values above U_M[N-1]).  The paper's merge then
// reduces, per tile, to:
//   p_j   = #{tile U_M < B[j]} (binary search in the staged tile), found_j =
//           U_M[a + p_j] == B[j] (a duplicate: appended once);
//   cnt[p] = #{new j : p_j = p}, shift(i) = sum_{p <= i} cnt[p];
//   E_t   = #{new values in earlier tiles} (decoupled look-back: the paper's
//           counts + prefix sum, one pass);
//   U_M[a+i] -> U'[a + E_t + i + shift(i)] = X_M[a+i];
//   new B[j] -> U'[a + E_t + p_j + newrank_j] = X_D[j] (newrank_j = new values
//           of the slice before j); a duplicate takes its twin's X_M.
// Three phases like the paper's: k_sp_count ranks each slice in its
// staged tile (p_j | found_j saved, 4 bytes per U_D value) and counts the
// tile's duplicates; k_scan_counts prefix-sums them (E_t = lo_t - dups before
// t); k_sp_write copies U_M with gaps straight from global memory and inserts
// the new values -- no merge-path ranking of both sides.  A single pass with
// decoupled look-back was slower (cfg2 0.131 vs 0.100 ms, cfg5 12.3 vs 7.6 ms):
// the look-back serialised the concurrently resident tiles.
#ifndef DM_SP_TILE
#define DM_SP_TILE 2048
#endif
constexpr uint32_t kSpTile = DM_SP_TILE, kSpThreads = 256, kSpItems = kSpTile / kSpThreads, kSpChunk = 512;
static_assert(kSpItems % 4 == 0, "the shift prefix reads 4 positions per 16-byte load");

// Grid of the persistent sparse kernels (knob 7): 0 one resident wave (SMs x
// occupancy), 1 one CTA per tile (non-persistent), 2 three CTAs (tests: long
// tile walks).
unsigned sp_grid(const void* func, size_t smem, uint64_t ntiles) {
  const int k = tuning(7);
  const uint64_t g = k == 1 ? ntiles : k == 2 ? 3 : (uint64_t)device_sms() * occupancy(func, kSpThreads, smem);
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, ntiles));
}

template <class KT>
__global__ void __launch_bounds__(256) k_sp_partition(const void* __restrict__ A, uint64_t nA,
                                                      const void* __restrict__ B, const dm_header* __restrict__ hdr,
                                                      uint64_t ntiles, uint64_t* __restrict__ part) {
  pdl_prologue();
  const uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const unsigned lane = lane_id();
  if (t > ntiles) return;
  const uint64_t nB = hdr->delta_dict_len;
  if (t == 0 || t == ntiles) {
    if (lane == 0) part[t] = t == 0 ? 0 : nB;
    return;
  }
  const auto v = KT::load(A, t * kSpTile);
  uint64_t lo = 0, hi = nB;  // lower bound of v in B, 32 probes per round
  while (hi > lo) {
    const uint64_t span = hi - lo;
    const uint64_t ik = lo + span * lane / 32;
    const bool cond = KT::lt(KT::load(B, ik), v);
    const unsigned c = __popc(__ballot_sync(FULL, cond));
    const uint64_t nlo = c ? lo + span * (c - 1) / 32 + 1 : lo;
    const uint64_t nhi = c < 32 ? lo + span * c / 32 : hi;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) part[t] = lo;
}

// Phase 1: rank the tile's slice inside the staged tile; pf[j] = p_j | found << 31,
// cnt[t] = the tile's duplicates (k_scan_counts turns them into prefix sums).
template <class KT>
__global__ void __launch_bounds__(kSpThreads) k_sp_count(const void* __restrict__ A, uint64_t nA,
                                                         const void* __restrict__ B,
                                                         const uint64_t* __restrict__ part, uint64_t ntiles,
                                                         uint32_t* __restrict__ pf, uint32_t* __restrict__ cnt) {
  pdl_prologue();
  using K = typename KT::K;
  constexpr uint32_t T = kSpTile, NT = kSpThreads, IT = kSpItems;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* sk = reinterpret_cast<K*>(smem_raw);
  __shared__ uint32_t s_warp[NT / 32 + 1];
  // (measured: an evict-last hint here, evict-first / streaming in the write pass,
  // made Step 1(b) slower: cfg2 0.100 -> 0.103 ms, cfg5 7.56 -> 8.81 ms)
  // Persistent over tiles t = blockIdx.x + k * gridDim.x: the next tile's U_M
  // values are loaded into registers while the current one is searched, so the
  // HBM reads of the resident CTAs do not all fall in one phase.
  K nx[IT];
  auto fetch = [&](uint64_t tt) {
    const uint64_t a = tt * T;
    const uint32_t na = (uint32_t)umin64(T, nA - a);
#pragma unroll
    for (uint32_t r = 0; r < IT; ++r) {
      const uint32_t i = threadIdx.x + r * NT;
      if (i < na) nx[r] = KT::load(A, a + i);
    }
  };
  if (blockIdx.x < ntiles) fetch(blockIdx.x);
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t a = t * T;
    const uint32_t na = (uint32_t)umin64(T, nA - a);
    const uint64_t lo = part[t], nb = part[t + 1] - lo;
#pragma unroll
    for (uint32_t r = 0; r < IT; ++r) {
      const uint32_t i = threadIdx.x + r * NT;
      if (i < na) sk[i] = nx[r];
    }
    __syncthreads();
    if (t + gridDim.x < ntiles) fetch(t + gridDim.x);
    uint32_t dups = 0;
    for (uint64_t j = threadIdx.x; j < nb; j += NT) {
      const K v = KT::load(B, lo + j);
      uint32_t l = 0, h = na;  // #{tile A < v}
      while (l < h) {
        const uint32_t m = (l + h) >> 1;
        if (KT::lt(sk[m], v)) l = m + 1; else h = m;
      }
      const bool found = l < na && KT::eq(sk[l], v);
      dups += found ? 1u : 0u;
      pf[lo + j] = l | (found ? 0x80000000u : 0u);
    }
    uint32_t tot;
    block_exclusive_scan<NT>(dups, s_warp, tot);  // ends with a barrier: sk is free again
    if (threadIdx.x == 0) cnt[t] = tot;
  }
}

// Phase 3: E_t = part[t] - excl[t] new values precede the tile; copy U_M with
// gaps (straight from global memory, coalesced), insert the new values, write
// X_M / X_D and the XC inputs.
template <class KT>
__global__ void __launch_bounds__(kSpThreads) k_sp_write(const void* __restrict__ A, uint64_t nA,
                                                         const void* __restrict__ B,
                                                         const uint64_t* __restrict__ part, uint64_t ntiles,
                                                         const uint32_t* __restrict__ pf,
                                                         const uint64_t* __restrict__ excl, void* __restrict__ U,
                                                         uint32_t* __restrict__ XM, uint32_t* __restrict__ XD,
                                                         dm_header* hdr, uint32_t* __restrict__ rblk,
                                                         uint8_t* __restrict__ offs, uint32_t xs) {
  pdl_prologue();
  using K = typename KT::K;
  constexpr uint32_t T = kSpTile, NT = kSpThreads, IT = kSpItems, C = kSpChunk, JT = C / NT;
  __shared__ __align__(16) uint32_t scnt[T + 4];  // cnt[p], then the inclusive shift(i)
  __shared__ uint32_t s_warp[NT / 32 + 1];
  const unsigned lane = lane_id();
  // Persistent over tiles (as k_sp_count): the next tile's U_M values are loaded
  // into registers while the current tile is written.
  K nx[IT];
  auto fetch = [&](uint64_t tt) {
    const uint64_t a = tt * T;
    const uint32_t na = (uint32_t)umin64(T, nA - a);
#pragma unroll
    for (uint32_t r = 0; r < IT; ++r) {
      const uint32_t i = threadIdx.x + r * NT;
      if (i < na) nx[r] = KT::load(A, a + i);
    }
  };
  if (blockIdx.x < ntiles) fetch(blockIdx.x);
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t a = t * T;
    const uint32_t na = (uint32_t)umin64(T, nA - a);
    const uint64_t lo = part[t], nb = part[t + 1] - lo;
    const uint64_t E = lo - excl[t];  // new values of earlier tiles
    const uint64_t base = a + E;
    __syncthreads();  // the previous tile's readers of scnt are done
    for (uint32_t i = threadIdx.x; i < T / 4 + 1; i += NT) reinterpret_cast<uint4*>(scnt)[i] = make_uint4(0, 0, 0, 0);
    // the tile's U_M values (registers; the copy needs no staging)
    K v[IT];
#pragma unroll
    for (uint32_t r = 0; r < IT; ++r) v[r] = nx[r];
    if (t + gridDim.x < ntiles) fetch(t + gridDim.x);
    __syncthreads();
    for (uint64_t j = threadIdx.x; j < nb; j += NT) {
      const uint32_t w = pf[lo + j];
      if (!(w >> 31)) atomicAdd(&scnt[w], 1u);
    }
    __syncthreads();
    {  // inclusive prefix over positions [0, na); a thread's IT positions as 16-byte
       // loads / stores (the scalar stride-IT form was an IT-way bank conflict)
      const uint32_t i0 = threadIdx.x * IT;
      uint32_t c[IT], sum = 0;
      uint4* s4 = reinterpret_cast<uint4*>(scnt + i0);
#pragma unroll
      for (uint32_t q = 0; q < IT / 4; ++q) {
        const uint4 x = s4[q];
        c[4 * q] = x.x; c[4 * q + 1] = x.y; c[4 * q + 2] = x.z; c[4 * q + 3] = x.w;
      }
#pragma unroll
      for (uint32_t r = 0; r < IT; ++r) {
        if (i0 + r >= na) c[r] = 0u;
        sum += c[r];
      }
      uint32_t tot;
      uint32_t run = block_exclusive_scan<NT>(sum, s_warp, tot);
#pragma unroll
      for (uint32_t r = 0; r < IT; ++r) {
        run += c[r];
        c[r] = run;  // positions >= na are never read as shifts
      }
#pragma unroll
      for (uint32_t q = 0; q < IT / 4; ++q) s4[q] = make_uint4(c[4 * q], c[4 * q + 1], c[4 * q + 2], c[4 * q + 3]);
    }
    __syncthreads();
    const uint32_t bmask = (1u << xs) - 1;
    bool unsorted = false;
#pragma unroll
    for (uint32_t r = 0; r < IT; ++r) {
      const uint32_t i = threadIdx.x + r * NT;
      // predecessor for the sortedness check: the lane below, or a load at warp edges
      // (every lane shuffles: no lane leaves the loop early)
      const K prev_l = KT::shfl_up(v[r], 1);
      if (i >= na) continue;
      const uint32_t sh = scnt[i];
      const uint64_t out = base + i + sh;
      KT::store(U, out, v[r]);
      if (XM) XM[a + i] = (uint32_t)out;
      if (rblk) {  // XC block samples R(g) = X_M[2^xs g] - 2^xs g
        if (((a + i) & bmask) == 0) rblk[(a + i) >> xs] = (uint32_t)(E + sh);
        if (a + i == nA - 1) rblk[(nA + bmask) >> xs] = (uint32_t)(E + sh);
      }
      if (a + i > 0) {
        const K prev = lane > 0 ? prev_l : KT::load(A, a + i - 1);
        if (!KT::lt(prev, v[r])) unsorted = true;
      }
    }
    if (__any_sync(FULL, unsorted) && lane == 0) atomicMin(&hdr->status, (int)DM_E_UNSORTED);
    // the slice: new values into their slots, X_D for all (blocked chunks of C for the new-rank scan)
    uint32_t run_new = 0;
    for (uint64_t c0 = 0; c0 < nb; c0 += C) {
      const uint32_t cn = (uint32_t)umin64(C, nb - c0);
      const uint32_t j0 = threadIdx.x * JT;
      uint32_t w[JT], cntn = 0;
#pragma unroll
      for (uint32_t r = 0; r < JT; ++r) {
        w[r] = j0 + r < cn ? pf[lo + c0 + j0 + r] : 0x80000000u;
        cntn += (w[r] >> 31) ? 0u : 1u;
      }
      uint32_t tot;
      uint32_t nr = run_new + block_exclusive_scan<NT>(cntn, s_warp, tot);
#pragma unroll
      for (uint32_t r = 0; r < JT; ++r) {
        const uint32_t j = j0 + r;
        if (j >= cn) break;
        const uint32_t p = w[r] & 0x7fffffffu;
        if (w[r] >> 31) {  // duplicate: its U_M twin's index
          XD[lo + c0 + j] = (uint32_t)(base + p + scnt[p]);
        } else {
          const uint64_t u = base + p + nr;
          KT::store(U, u, KT::load(B, lo + c0 + j));
          XD[lo + c0 + j] = (uint32_t)u;
          if (offs) offs[E + nr] = (uint8_t)((a + p - 1) & bmask);
          ++nr;
        }
      }
      run_new += tot;
    }
  }
}

// XC superblock records (NEXT3) from the block samples R(g) = rblk[g]:
// {R(4s) | flag << 31, cum bytes 0..3}, cum[t] = R(4s+t+1) - R(4s).  Flag = the
// counts do not fit a byte, or one block holds more than kXcMaxBlock
// insertions (bounds the per-lookup scan); flagged superblocks are looked up
// in the plain X_M.
__global__ void __launch_bounds__(256) k_xc_records(const uint32_t* __restrict__ rblk, uint64_t nblk, uint64_t nsb,
                                                    uint2* __restrict__ rec) {
  pdl_prologue();
  const uint64_t sb = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (sb >= nsb) return;
  constexpr uint32_t BPS = 4;
  const uint64_t g0 = sb * BPS;
  const uint32_t R0 = rblk[g0];
  uint32_t prev = 0, cum = 0, flag = R0 >> 31;
#pragma unroll
  for (uint32_t t = 0; t < BPS; ++t) {
    const uint32_t c = rblk[umin64(g0 + t + 1, nblk)] - R0;
    if (c > 255u || c - prev > kXcMaxBlock) flag = 1;
    cum |= (c & 255u) << (8 * t);
    prev = c;
  }
  rec[sb] = make_uint2(R0 | (flag << 31), cum);
}

// X_M for the flagged superblocks only, when the merge does not materialise X_M
// (nobody asked for it and Step 2(b) reads XC from L2, which falls back to
// X_M on flagged superblocks alone): X_M[c] = c + R(g) + #{entries of block g
// below c mod 2^xs} with g = c's block -- the closed form XC encodes,
// the list binary-searched (sorted: new values in order).  One warp per superblock.
__global__ void __launch_bounds__(256) k_xm_flagged(const uint2* __restrict__ rec, uint64_t nsb, uint32_t xs,
                                                    uint64_t dict_len, const uint32_t* __restrict__ rblk,
                                                    uint64_t nblk, const uint8_t* __restrict__ offs,
                                                    uint32_t* __restrict__ xm) {
  pdl_prologue();
  const unsigned lane = lane_id();
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t bmask = (1u << xs) - 1;
  for (uint64_t sb = warp0; sb < nsb; sb += nwarps) {
    if (!(rec[sb].x >> 31)) continue;
    const uint64_t c0 = sb << (xs + 2), c1 = umin64(c0 + (4ull << xs), dict_len);
    for (uint64_t c = c0 + lane; c < c1; c += 32) {
      const uint64_t g = c >> xs;
      const uint32_t lo = rblk[g], hi = rblk[umin64(g + 1, nblk)], o = (uint32_t)c & bmask;
      uint32_t a = lo, b = hi;  // first entry >= o
      while (a < b) {
        const uint32_t m = (a + b) >> 1;
        if (offs[m] < o) a = m + 1; else b = m;
      }
      xm[c] = (uint32_t)c + a;  // c + R(g) + (a - lo), R(g) = lo
    }
  }
}

// XC exception list (row-sharded Step 2): one warp per superblock; a flagged
// superblock's X_M slice (4 * 2^xs entries) moves between X_M and a compact
// slices[] array at slot ids[] (gather: slot from an atomic counter).
__global__ void __launch_bounds__(256) k_xc_exceptions(bool gather, const uint2* __restrict__ rec, uint64_t nsb,
                                                       uint32_t xs, uint64_t dict_len, uint32_t* __restrict__ xm,
                                                       uint32_t* __restrict__ ids, uint32_t* __restrict__ slices,
                                                       unsigned long long* d_count, uint64_t count) {
  pdl_prologue();
  const unsigned lane = lane_id();
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t SB = 4ull << xs;
  const uint64_t n_items = gather ? nsb : count;
  for (uint64_t w = warp0; w < n_items; w += nwarps) {
    uint64_t sb, slot;
    if (gather) {
      if (!(rec[w].x >> 31)) continue;
      unsigned long long sl = 0;
      if (lane == 0) sl = atomicAdd(d_count, 1ull);
      if (!slices) continue;  // count only (the caller sizes the slices from the count)
      slot = __shfl_sync(FULL, sl, 0);
      sb = w;
      if (lane == 0) ids[slot] = (uint32_t)sb;
    } else {
      slot = w;
      sb = ids[w];
    }
    const uint64_t c0 = sb * SB, n = umin64(SB, dict_len - c0);
    for (uint64_t i = lane; i < n; i += 32) {
      if (gather)
        slices[slot * SB + i] = xm[c0 + i];
      else
        xm[c0 + i] = slices[slot * SB + i];
    }
  }
}

__global__ void k_empty_header(dm_header* hdr) {
  pdl_prologue();
  // |U_M| + |U_D| == 0: U' is empty and b' = 1 (reading A1)
  if (hdr->delta_dict_len == 0) {
    hdr->merged_dict_len = 0;
    hdr->merged_bits = 1;
  }
}

template <class KT>
cudaError_t run(const dm_column_in* in, char* ws, const WsLayout& L, const void* udict, void* U, uint32_t* xm,
                uint32_t* xd, dm_header* hdr, cudaStream_t st, bool force_xc, bool xm_requested) {
  using K = typename KT::K;
  if (in->dict_len + in->n_delta == 0) {
    launch_k(k_empty_header, 1, 1, 0, st, hdr);
    note_launch();
    return cudaGetLastError();
  }
  const uint64_t nt = L.ntiles_merge;
  uint64_t* part = reinterpret_cast<uint64_t*>(ws + L.part);
  const bool xc = xc_wanted(in) || (force_xc && in->dict_len > 0);
  uint32_t* rblk = xc ? reinterpret_cast<uint32_t*>(ws + L.xc_rblk) : nullptr;
  uint8_t* offs = xc ? reinterpret_cast<uint8_t*>(ws + L.xc_offs) : nullptr;
  const uint32_t xs = xc_shift(in);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(ws + L.mcount);
  uint64_t* excl = reinterpret_cast<uint64_t*>(ws + L.mexcl);
  uint64_t* status = reinterpret_cast<uint64_t*>(ws + L.status_merge);
  uint32_t* counter = reinterpret_cast<uint32_t*>(ws + L.counters) + CNT_MERGE;
  const int variant = sp_wanted(in) ? 3 : tuning(1) == 3 ? 0 : tuning(1);
  // X_M need not be materialised when nobody asked for it and Step 2(b) will
  // read XC from L2 (that kernel falls back to X_M on flagged superblocks only,
  // filled by k_xm_flagged): cfg5 skips 4.3 GB of writes
  const int xknob = tuning(0);
  const bool skip_xm = xc && !force_xc && !xm_requested && (variant == 0 || variant == 2 || variant == 3) &&
                       (xknob == 2 || xknob == 3 || (xknob == 0 && in->dict_len * 4 > kXcGlobalMinBytes));
  uint32_t* xm_w = skip_xm ? nullptr : xm;
  if (variant == 3) {  // sparse deltas: U_M tiles with their U_D slices, one pass (sp_wanted)
    const uint64_t ntiles = (in->dict_len + kSpTile - 1) / kSpTile;
    launch_k(k_sp_partition<KT>, (unsigned)((ntiles + 1 + 7) / 8), 256, 0, st, in->main_dict, in->dict_len, udict, hdr,
                                                                        ntiles, part);
    uint32_t* pf = reinterpret_cast<uint32_t*>(ws + L.vals0);  // Step 1(a) scratch, free by now (>= N_D u32)
    if (sizeof(K) * kSpTile > 48 * 1024) ensure_smem((const void*)k_sp_count<KT>);
    // persistent grids (sp_grid): every resident CTA walks tiles t, t + grid, ...
    const unsigned g_count = sp_grid((const void*)k_sp_count<KT>, sizeof(K) * kSpTile, ntiles);
    const unsigned g_write = sp_grid((const void*)k_sp_write<KT>, 0, ntiles);
    launch_k(k_sp_count<KT>, g_count, kSpThreads, sizeof(K) * kSpTile, st, in->main_dict, in->dict_len, udict,
                                                              part, ntiles, pf, cnt);
    launch_k(k_scan_counts, (unsigned)((ntiles + 2047) / 2048), 256, 0, st, cnt, ntiles, excl, status, counter,
                                                                  in->dict_len, hdr);
    launch_k(k_sp_write<KT>, g_write, kSpThreads, 0, st, in->main_dict, in->dict_len, udict, part, ntiles,
                                                              (const uint32_t*)pf, (const uint64_t*)excl, U, xm_w, xd,
                                                              hdr, rblk, offs, xs);
    note_launch(4);
  } else if (variant == 0 || variant == 2) {  // lean tiles: two passes (default) or single pass
    launch_k(k_partition<KT>, (unsigned)((nt + 1 + 7) / 8), 256, 0, st, in->main_dict, in->dict_len, udict, hdr, nt + 1,
                                                                     part);
    const size_t smem = sizeof(K) * (kMergeTile + 1) + sizeof(uint32_t) * (3 * kMergeTile + 1);
    auto go = [&](auto kern, size_t sm) {
      ensure_smem((const void*)kern, true);
      launch_k(kern, (unsigned)nt, kMergeThreads, sm, st, in->main_dict, in->dict_len, udict, part, nt, status, counter,
                                                      cnt, excl, U, xm_w, xd, hdr, rblk, offs, xs);
    };
    if (variant == 2) {
      go(k_merge<KT, 0>, smem);
      note_launch(2);
    } else {
      go(k_merge<KT, 1>, sizeof(K) * (kMergeTile + 1));  // count pass: key staging only
      launch_k(k_scan_counts, (unsigned)((nt + 2047) / 2048), 256, 0, st, cnt, nt, excl, status, counter, in->dict_len,
                                                                    hdr);
      go(k_merge<KT, 2>, smem);
      note_launch(4);
    }
  } else {
  uint32_t* cnt = reinterpret_cast<uint32_t*>(ws + L.mcount);
  uint64_t* excl = reinterpret_cast<uint64_t*>(ws + L.mexcl);
  launch_k(k_partition<KT>, (unsigned)((nt + 1 + 7) / 8), 256, 0, st, in->main_dict, in->dict_len, udict, hdr, nt + 1,
                                                                   part);
  const size_t smem_count = sizeof(K) * (kMergeTile + 1) + 3 * sizeof(uint32_t) * (kMergeTile + 2);
  ensure_smem((const void*)k_merge_count<KT>, true);
  launch_k(k_merge_count<KT>, (unsigned)nt, kMergeThreads, smem_count, st, in->main_dict, in->dict_len, udict, part, hdr,
                                                                     cnt);
  launch_k(k_scan_counts, (unsigned)((nt + 2047) / 2048), 256, 0, st, 
      cnt, nt, excl, reinterpret_cast<uint64_t*>(ws + L.status_merge),
      reinterpret_cast<uint32_t*>(ws + L.counters) + CNT_MERGE, in->dict_len, hdr);
  const size_t smem_write = smem_count;
  ensure_smem((const void*)k_merge_write<KT>, true);
  launch_k(k_merge_write<KT>, (unsigned)nt, kMergeThreads, smem_write, st, in->main_dict, in->dict_len, udict, part, excl,
                                                                     U, xm, xd, hdr, rblk, offs, xs);
  note_launch(4);
  }
  if (xc) {
    const uint64_t nsb = xc_nsb(in->dict_len, xs);
    launch_k(k_xc_records, (unsigned)((nsb + 255) / 256), 256, 0, st, rblk, xc_nblk(in->dict_len, xs), nsb,
                                                                reinterpret_cast<uint2*>(ws + L.xc_rec));
    note_launch();
    if (skip_xm) {
      const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nsb + 7) / 8, (uint64_t)device_sms() * 8));
      launch_k(k_xm_flagged, g, 256, 0, st, reinterpret_cast<const uint2*>(ws + L.xc_rec), nsb, xs, in->dict_len,
               (const uint32_t*)rblk, xc_nblk(in->dict_len, xs), (const uint8_t*)offs, xm);
      note_launch();
    }
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_xc_exceptions(bool gather, const uint2* rec, uint64_t nsb, uint32_t xs, uint64_t dict_len,
                                 uint32_t* xm, uint32_t* ids, uint32_t* slices, unsigned long long* d_count,
                                 uint64_t count, cudaStream_t st) {
  const uint64_t items = gather ? nsb : count;
  if (items == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<uint64_t>((items + 7) / 8, (uint64_t)device_sms() * 16);
  launch_k(k_xc_exceptions, grid, 256, 0, st, gather, rec, nsb, xs, dict_len, xm, ids, slices, d_count, count);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_dictionary_merge(const dm_column_in* in, const dm_column_out* out, char* ws, const WsLayout& L,
                                    const void* udict, uint32_t* xm, uint32_t* xd, dm_header* hdr, cudaStream_t st,
                                    bool force_xc, bool need_xm) {
  const bool want_xm = out->x_main != nullptr || need_xm;
  switch (in->key) {
    case DM_KEY_U64: return run<KeyU64>(in, ws, L, udict, out->merged_dict, xm, xd, hdr, st, force_xc, want_xm);
    case DM_KEY_U32: return run<KeyU32>(in, ws, L, udict, out->merged_dict, xm, xd, hdr, st, force_xc, want_xm);
    default: return run<KeyB16>(in, ws, L, udict, out->merged_dict, xm, xd, hdr, st, force_xc, want_xm);
  }
}

}  // namespace dm
