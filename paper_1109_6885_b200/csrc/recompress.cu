// recompress.cu -- Step 2(b) on the GPU: recompress the main codes through X_M at
// the new width and append the delta tuples through X_D.
//
// Paper: "computing the new compressed value for the main (or delta) table
// reduces to reading the old compressed value K_C^i and retrieving the value
// stored at K_C^i th index of the corresponding auxiliary structure X_M^j or
// X_D^j"; M'[i] <- X_M[M[i]] (Eq 11), executed for each main
// element "and similar for the delta partition", the delta appended
// after the main.  The paper splits the N' tuples evenly over threads
// (P:324); its time is the stream of the packed vectors plus the X gathers,
// which hit the cache when X fits on die.
//
// GPU form: a persistent kernel, one CTA per SM slot.  The output rows are cut
// into 4096-row chunks; a 32-row group is exactly b input u32 words and b'
// output u32 words for every width, so chunks are word-aligned at both widths.
//   * the main words of each chunk arrive by bulk TMA (cp.async.bulk, L2
//     evict-first) into a 4-stage shared-memory ring guarded by mbarriers;
//   * each warp handles whole 32-row groups: lane l unpacks row l with two
//     conflict-free shared loads and a funnel shift, gathers X_M[code] through
//     the read-only path with an L2 evict-last hint (X_M stays L2-resident
//     while the streams flow past it), delta rows gather X_D[r[k]];
//   * lane k builds output word k of the group from the <= ceil((b'+31)/b')
//     codes that overlap it, fetched by warp shuffles (funnel packing across
//     word boundaries), into a shared staging buffer;
//   * the staged chunk leaves by bulk TMA store (L2 evict-first).
// b' is only known on the device (no host sync): the host launches the width
// specialisations that |U'|'s bounds allow and each exits unless it matches.
#include <algorithm>
#include <array>
#include <utility>

#include "dm_device.cuh"

namespace dm {
namespace {

__device__ __forceinline__ uint64_t dwords(uint64_t n, uint32_t bits) { return (n * bits + 63) >> 6; }

template <int NB>
__device__ __forceinline__ uint32_t warp_pack(uint32_t v, uint32_t nb, uint32_t r0, uint32_t op) {
  constexpr int TMAX = NB ? (2 * NB + 30) / NB : 32;
  const int tmax = NB ? TMAX : (int)((2 * nb + 30) / nb);
  uint32_t word = 0;
#pragma unroll
  for (int t = 0; t < TMAX; ++t) {
    if (!NB && t >= tmax) break;
    const uint32_t c = __shfl_sync(FULL, v, (r0 + t) & 31);
    word |= (t == 0) ? shr32(c, op) : shl32(c, t * nb - op);
  }
  return word;
}

// Warp-specialised: warp kRecConsumerWarps is the TMA producer, warps
// 0..kRecConsumerWarps-1 consume.  full[s] completes when stage s holds its
// chunk's main words; empty[s] completes when every consumer warp is done with
// stage s.  No CTA-wide barrier after the prologue.  XS: X_M staged in shared
// memory (tables up to kRecSmemXBytes), else gathered through L2.
template <int NB, bool XS>
__global__ void __launch_bounds__(kRecThreads) k_recompress(const uint64_t* __restrict__ M, uint64_t n_main, uint32_t b,
                                                            uint64_t dict_len, const uint32_t* __restrict__ XM,
                                                            const uint32_t* __restrict__ XD,
                                                            const uint32_t* __restrict__ rank, uint64_t n_delta,
                                                            uint64_t* __restrict__ Mout, dm_header* hdr,
                                                            uint32_t in_stage_bytes, uint32_t fixed_bits) {
  constexpr int G = kRecGroups;
  constexpr int S = kRecStages;
  constexpr int CW = kRecConsumerWarps;
  constexpr int U = G / CW;  // groups per consumer warp per chunk, all in flight together
  static_assert(G % CW == 0, "groups must split evenly over consumer warps");
  const uint32_t hb = fixed_bits ? fixed_bits : hdr->merged_bits;
  if (NB && hb != (uint32_t)NB) return;
  const uint32_t nb = NB ? (uint32_t)NB : hb;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + S;
  unsigned char* in_ring = smem_raw + 128;
  uint32_t* sx = reinterpret_cast<uint32_t*>(in_ring + (size_t)S * in_stage_bytes);  // XS only

  const uint64_t n_total = n_main + n_delta;
  const uint64_t R = 32ull * G;
  const uint64_t nchunks = (n_total + R - 1) / R;
  const uint64_t main_bytes = dwords(n_main, b) * 8;
  const uint64_t nw32 = 2 * dwords(n_total, nb);
  const uint32_t chunk_in = G * b * 4;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_mbar_init();
  }
  if (XS) {
    for (uint32_t i = threadIdx.x; i < dict_len; i += blockDim.x) sx[i] = __ldg(XM + i);
  }
  __syncthreads();

  if (warp == CW) {  // ---------------------------------------------------- producer
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();
      for (uint64_t k = 0;; ++k) {
        const uint64_t c = blockIdx.x + k * gridDim.x;
        if (c >= nchunks) break;
        const int s = (int)(k % S);
        if (k >= S) mbar_wait_parity(&empty[s], (uint32_t)(((k / S) - 1) & 1));
        unsigned char* dst = in_ring + (size_t)s * in_stage_bytes;
        const uint64_t start = c * (uint64_t)chunk_in;
        const uint32_t len = start < main_bytes ? (uint32_t)umin64(chunk_in, main_bytes - start) : 0u;
        const uint32_t tl = len & ~15u;
        if (len > tl)  // 8-byte tail the bulk copy cannot take; published by the arrive (release)
          *reinterpret_cast<uint64_t*>(dst + tl) =
              *reinterpret_cast<const uint64_t*>(reinterpret_cast<const unsigned char*>(M) + start + tl);
        mbar_arrive_expect_tx(&full[s], tl);
        if (tl) tma_load_1d(dst, reinterpret_cast<const unsigned char*>(M) + start, tl, &full[s], pol_stream);
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  const uint64_t pol_x = policy_evict_last();
  const uint32_t us = lane * b, uw0 = us >> 5, uo = us & 31;
  const uint32_t umask = b == 32 ? 0xffffffffu : ((1u << b) - 1);
  const uint32_t pr0 = (32 * lane) / nb, pop = 32 * lane - pr0 * nb;
  uint32_t* out32 = reinterpret_cast<uint32_t*>(Mout);
  bool bad = false;

  for (uint64_t k = 0;; ++k) {
    const uint64_t c = blockIdx.x + k * gridDim.x;
    if (c >= nchunks) break;
    const int s = (int)(k % S);
    mbar_wait_parity(&full[s], (uint32_t)((k / S) & 1));
    const uint32_t* sin = reinterpret_cast<const uint32_t*>(in_ring + (size_t)s * in_stage_bytes);
    const uint64_t row_base = c * R;
    uint32_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int g = warp + CW * u;
      const uint64_t row = row_base + (uint64_t)g * 32 + lane;
      if (row < n_main) {
        const uint32_t lo = sin[g * b + uw0], hi = sin[g * b + uw0 + 1];
        uint32_t code = __funnelshift_r(lo, hi, uo) & umask;
        if (code >= dict_len) {
          bad = true;
          code = 0;
        }
        v[u] = XS ? sx[code] : ld_gather_u32(XM + code, pol_x);
      } else if (row < n_total) {
        v[u] = __ldg(XD + __ldg(rank + (row - n_main)));
      } else {
        v[u] = 0;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // stage s fully read by this warp
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int g = warp + CW * u;
      const uint32_t word = warp_pack<NB>(v[u], nb, pr0, pop);
      const uint64_t ow = (c * G + g) * nb + lane;
      if (lane < nb && ow < nw32) __stcs(out32 + ow, word);
    }
  }
  if (__any_sync(FULL, bad) && lane == 0) atomicMin(&hdr->status, (int)DM_E_CODE_RANGE);
}

__global__ void __launch_bounds__(256) k_pack(const uint32_t* __restrict__ codes, uint64_t n, uint32_t bits,
                                              uint32_t* __restrict__ words32, uint64_t nw32) {
  const unsigned lane = lane_id();
  const uint32_t mask = bits == 32 ? 0xffffffffu : ((1u << bits) - 1);
  const uint32_t pr0 = (32 * lane) / bits, pop = 32 * lane - pr0 * bits;
  const uint64_t ngroups = (n + 31) / 32;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t g = warp; g < ngroups; g += nwarps) {
    const uint64_t row = g * 32 + lane;
    const uint32_t v = row < n ? (codes[row] & mask) : 0u;
    const uint32_t word = warp_pack<0>(v, bits, pr0, pop);
    const uint64_t widx = g * bits + lane;
    // lanes >= bits of the last group zero the pad half-word of the final u64
    if ((lane < bits || g + 1 == ngroups) && widx < nw32) words32[widx] = lane < bits ? word : 0u;
  }
}

__global__ void __launch_bounds__(256) k_unpack(const uint32_t* __restrict__ words32, uint64_t nw32, uint64_t n,
                                                uint32_t bits, uint32_t* __restrict__ codes) {
  const uint32_t mask = bits == 32 ? 0xffffffffu : ((1u << bits) - 1);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = i * bits;
    const uint64_t w = s >> 5;
    const uint32_t lo = words32[w], hi = (w + 1 < nw32) ? words32[w + 1] : 0u;
    codes[i] = __funnelshift_r(lo, hi, (uint32_t)(s & 31)) & mask;
  }
}

template <int NB>
cudaError_t launch_nb(const dm_column_in* in, const dm_column_out* out, const uint32_t* xm, const uint32_t* xd,
                      const uint32_t* rank, dm_header* hdr, cudaStream_t st, uint32_t nb_cap, uint32_t fixed_bits) {
  (void)nb_cap;
  const uint32_t in_stage = kRecGroups * in->main_bits * 4 + 16;
  const bool xs = in->dict_len * 4 <= kRecSmemXBytes;
  const size_t smem = 128 + (size_t)kRecStages * in_stage + (xs ? in->dict_len * 4 : 0);
  const int sms = device_sms();
  const uint64_t n_total = in->n_main + in->n_delta;
  const uint64_t nchunks = (n_total + 32ull * kRecGroups - 1) / (32ull * kRecGroups);
  auto go = [&](auto kern) {
    const int occ = occupancy((const void*)kern, kRecThreads, smem);
    const unsigned grid = (unsigned)std::min<uint64_t>(nchunks, (uint64_t)sms * occ);
    kern<<<grid, kRecThreads, smem, st>>>(in->main_codes, in->n_main, in->main_bits, in->dict_len, xm, xd, rank,
                                          in->n_delta, out->merged_codes, hdr, in_stage, fixed_bits);
  };
  if (xs)
    go(k_recompress<NB, true>);
  else
    go(k_recompress<NB, false>);
  note_launch();
  return cudaGetLastError();
}

using LaunchFn = cudaError_t (*)(const dm_column_in*, const dm_column_out*, const uint32_t*, const uint32_t*,
                                 const uint32_t*, dm_header*, cudaStream_t, uint32_t, uint32_t);
template <int... I>
constexpr auto make_table(std::integer_sequence<int, I...>) {
  return std::array<LaunchFn, sizeof...(I)>{&launch_nb<I>...};
}

}  // namespace

cudaError_t launch_recompress(const dm_column_in* in, const dm_column_out* out, const uint32_t* xm,
                              const uint32_t* xd, const uint32_t* rank, dm_header* hdr, cudaStream_t st,
                              uint32_t fixed_bits) {
  if (in->n_main + in->n_delta == 0) return cudaSuccess;
  static const auto table = make_table(std::make_integer_sequence<int, 33>{});  // [0] = runtime width
  if (fixed_bits) return table[fixed_bits](in, out, xm, xd, rank, hdr, st, fixed_bits, fixed_bits);
  const uint64_t lo_len = std::max<uint64_t>(in->dict_len, in->n_delta ? 1 : 0);
  const uint32_t nb_lo = host_width(lo_len), nb_hi = host_width(in->dict_len + in->n_delta);
  if (nb_hi > 32) return cudaErrorInvalidValue;  // caller checks DM_E_TOO_WIDE first
  if (nb_hi - nb_lo <= 2) {
    for (uint32_t nb = nb_lo; nb <= nb_hi; ++nb) {
      cudaError_t e = table[nb](in, out, xm, xd, rank, hdr, st, nb_hi, 0);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  return table[0](in, out, xm, xd, rank, hdr, st, nb_hi, 0);
}

cudaError_t launch_pack(const uint32_t* codes, uint64_t n, uint32_t bits, uint64_t* words, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const uint64_t groups = (n + 31) / 32;
  const unsigned grid = (unsigned)std::min<uint64_t>((groups + 7) / 8, 148 * 16);
  k_pack<<<grid, 256, 0, st>>>(codes, n, bits, reinterpret_cast<uint32_t*>(words), 2 * host_words(n, bits));
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_unpack(const uint64_t* words, uint64_t n, uint32_t bits, uint32_t* codes, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  k_unpack<<<grid, 256, 0, st>>>(reinterpret_cast<const uint32_t*>(words), 2 * host_words(n, bits), n, bits, codes);
  note_launch();
  return cudaGetLastError();
}

}  // namespace dm
