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
                                                               uint8_t* __restrict__ offs) {
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
      if ((i & (kXcBlock - 1)) == 0) rblk[i / kXcBlock] = (uint32_t)(u - i);
      if (i == nA - 1) rblk[(nA + kXcBlock - 1) / kXcBlock] = (uint32_t)(u - i);
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
        offs[base + o - p] = (uint8_t)((p - 1) & (kXcBlock - 1));
      }
    }
  }
  if (__any_sync(FULL, unsorted) && lane_id() == 0) atomicMin(&hdr->status, (int)DM_E_UNSORTED);
}

// XC superblock records (NEXT3) from the block samples R(g) = rblk[g]:
// {R(4s) | flag << 31, cum bytes 0..3}, cum[t] = R(4s+t+1) - R(4s).  Flag = the
// counts do not fit a byte, or one block holds more than kXcMaxBlock
// insertions (bounds the per-lookup scan); flagged superblocks are looked up
// in the plain X_M.
__global__ void __launch_bounds__(256) k_xc_records(const uint32_t* __restrict__ rblk, uint64_t nblk, uint64_t nsb,
                                                    uint2* __restrict__ rec) {
  const uint64_t sb = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (sb >= nsb) return;
  constexpr uint32_t BPS = kXcSuper / kXcBlock;
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

__global__ void k_empty_header(dm_header* hdr) {
  // |U_M| + |U_D| == 0: U' is empty and b' = 1 (reading A1)
  if (hdr->delta_dict_len == 0) {
    hdr->merged_dict_len = 0;
    hdr->merged_bits = 1;
  }
}

template <class KT>
cudaError_t run(const dm_column_in* in, char* ws, const WsLayout& L, const void* udict, void* U, uint32_t* xm,
                uint32_t* xd, dm_header* hdr, cudaStream_t st) {
  using K = typename KT::K;
  if (in->dict_len + in->n_delta == 0) {
    k_empty_header<<<1, 1, 0, st>>>(hdr);
    note_launch();
    return cudaGetLastError();
  }
  const uint64_t nt = L.ntiles_merge;
  uint64_t* part = reinterpret_cast<uint64_t*>(ws + L.part);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(ws + L.mcount);
  uint64_t* excl = reinterpret_cast<uint64_t*>(ws + L.mexcl);
  k_partition<KT><<<(unsigned)((nt + 1 + 7) / 8), 256, 0, st>>>(in->main_dict, in->dict_len, udict, hdr, nt + 1,
                                                                   part);
  const size_t smem_count = sizeof(K) * (kMergeTile + 1) + 3 * sizeof(uint32_t) * (kMergeTile + 2);
  ensure_smem((const void*)k_merge_count<KT>, true);
  k_merge_count<KT><<<(unsigned)nt, kMergeThreads, smem_count, st>>>(in->main_dict, in->dict_len, udict, part, hdr,
                                                                     cnt);
  k_scan_counts<<<(unsigned)((nt + 2047) / 2048), 256, 0, st>>>(
      cnt, nt, excl, reinterpret_cast<uint64_t*>(ws + L.status_merge),
      reinterpret_cast<uint32_t*>(ws + L.counters) + CNT_MERGE, in->dict_len, hdr);
  const size_t smem_write = smem_count;
  ensure_smem((const void*)k_merge_write<KT>, true);
  const bool xc = xc_wanted(in->dict_len);
  uint32_t* rblk = xc ? reinterpret_cast<uint32_t*>(ws + L.xc_rblk) : nullptr;
  uint8_t* offs = xc ? reinterpret_cast<uint8_t*>(ws + L.xc_offs) : nullptr;
  k_merge_write<KT><<<(unsigned)nt, kMergeThreads, smem_write, st>>>(in->main_dict, in->dict_len, udict, part, excl,
                                                                     U, xm, xd, hdr, rblk, offs);
  note_launch(4);
  if (xc) {
    const uint64_t nsb = xc_nsb(in->dict_len);
    k_xc_records<<<(unsigned)((nsb + 255) / 256), 256, 0, st>>>(rblk, xc_nblk(in->dict_len), nsb,
                                                                reinterpret_cast<uint2*>(ws + L.xc_rec));
    note_launch();
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_dictionary_merge(const dm_column_in* in, const dm_column_out* out, char* ws, const WsLayout& L,
                                    const void* udict, uint32_t* xm, uint32_t* xd, dm_header* hdr, cudaStream_t st) {
  return in->key == DM_KEY_U64 ? run<KeyU64>(in, ws, L, udict, out->merged_dict, xm, xd, hdr, st)
                               : run<KeyB16>(in, ws, L, udict, out->merged_dict, xm, xd, hdr, st);
}

}  // namespace dm
