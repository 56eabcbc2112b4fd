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
// GPU form: a persistent, warp-specialised kernel, one CTA per SM slot.  The
// output rows are cut into chunks of 32-row groups; a group is exactly b input
// u32 words and b' output u32 words for every width, so chunks are
// word-aligned at both widths.
//   * one producer warp brings the main words of each chunk by bulk TMA
//     (cp.async.bulk, L2 evict-first) into a 4-stage shared-memory ring guarded
//     by mbarriers (full / empty per stage);
//   * each consumer warp handles whole 32-row groups: lane l unpacks row l with
//     two conflict-free shared loads and a funnel shift and translates it --
//     plain X_M staged in shared memory (<= 96 KB), the compact table XC in
//     shared memory (lean lookup below), plain X_M gathered through L2
//     (evict-last: it stays resident while the streams flow past), or XC
//     through L2; delta rows gather X_D[r[k]];
//   * lane k builds output word k of the group from the <= ceil((b'+31)/b')
//     codes that overlap it, fetched by warp shuffles (funnel packing across
//     word boundaries), and writes it with a streaming store (coalesced per
//     group).
// b' is only known on the device (no host sync): the host launches the width
// specialisations that |U'|'s bounds allow and each exits unless it matches
// (wide ranges: one runtime-width kernel, see launch_recompress).
#include <algorithm>
#include <array>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "dm_device.cuh"

namespace dm {
namespace {

__device__ __forceinline__ uint64_t dwords(uint64_t n, uint32_t bits) { return (n * bits + 63) >> 6; }

// NB > 0: b' = NB at compile time.  NB <= 0: b' at run time, with at most -NB
// codes per output word (NB = 0: any width, up to 32).
// Exact maximum number of b'-bit codes overlapping one 32-bit output word (the
// pattern repeats every b' words): e.g. 2 for b' = 24, whose code offsets are
// multiples of 8 (the generic bound (2b' + 30) / b' says 3).
__host__ __device__ constexpr int pack_tmax(int nb) {
  int mx = 0;
  for (int k = 0; k < nb; ++k) {
    int c = 0;
    for (int j = 0; j < 32; ++j) c += (j * nb < 32 * k + 32 && (j + 1) * nb > 32 * k) ? 1 : 0;
    mx = c > mx ? c : mx;
  }
  return mx;
}
template <int NB>
__device__ __forceinline__ uint32_t warp_pack(uint32_t v, uint32_t nb, uint32_t r0, uint32_t op) {
  constexpr int TMAX = NB > 0 ? pack_tmax(NB) : NB < 0 ? -NB : 32;
  const int tmax = NB > 0 ? TMAX : (int)((2 * nb + 30) / nb);
  uint32_t word = 0;
  if constexpr (NB == 0) {  // any width: a rolled loop (unrolling 32 steps behind a break only spills)
#pragma unroll 1
    for (int t = 0; t < tmax; ++t) {
      const uint32_t c = __shfl_sync(FULL, v, (r0 + t) & 31);
      word |= (t == 0) ? shr32(c, op) : shl32(c, t * nb - op);
    }
  } else {
#pragma unroll
    for (int t = 0; t < TMAX; ++t) {
      if (NB <= 0 && t >= tmax) break;
      const uint32_t c = __shfl_sync(FULL, v, (r0 + t) & 31);
      word |= (t == 0) ? shr32(c, op) : shl32(c, t * nb - op);
    }
  }
  return word;
}

// Warp packing on the FMA pipe (widths with at most 5 codes per output word):
// the codes overlapping a word occupy disjoint bits, so the word is a SUM of
// shifted codes, and every shift is by a per-lane constant -- a multiply by a
// per-lane power of two.  word = hi(c_0 * 2^(32-op)) [op > 0] + c_0 [op = 0]
// + sum_{t >= 1} c_t * 2^(t b' - op) [t b' - op < 32], all IMAD / IMAD.HI:
// the ALU pipe, which the lookups saturate, is left alone (B300 microarch
// notes: ALU and FMA pipes each take one warp instruction per 2 cycles).
template <int NB>
struct FmaPack {
  static constexpr int T = pack_tmax(NB);
  uint32_t src[T], mul[T], m0hi;
  __device__ __forceinline__ FmaPack(uint32_t lane) {
    const uint32_t r0 = (32 * lane) / NB, op = 32 * lane - r0 * NB;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      src[t] = (r0 + t) & 31;
      const uint32_t a = t * NB - op;  // t >= 1: shift left by a
      mul[t] = t == 0 ? (op == 0 ? 1u : 0u) : (a < 32 ? (1u << a) : 0u);
    }
    m0hi = op == 0 ? 0u : (1u << (32 - op));
  }
  __device__ __forceinline__ uint32_t pack(uint32_t v) const {
    uint32_t c[T];
#pragma unroll
    for (int t = 0; t < T; ++t) c[t] = __shfl_sync(FULL, v, src[t]);
    uint32_t acc = 0;
#pragma unroll
    for (int t = 0; t < T; ++t) acc += c[t] * mul[t];
    uint32_t w;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(w) : "r"(c[0]), "r"(m0hi), "r"(acc));
    return w;
  }
};
#ifndef DM_PACK_FMA
#define DM_PACK_FMA 1
#endif
template <int NB>
__host__ __device__ constexpr bool use_fma_pack() { return DM_PACK_FMA && NB >= 8; }

// Compact X_M lookup (XC, NEXT3; layout in dm_internal.h):
//   X_M[c] = c + start + #{entries of c's 256-block with offset < c mod 256}
// where start = R + cum[t-1] = #{new values with insertion point p <= 256g}
// (g = c's block) and the block's n entries are the new values with p in
// (256g, 256g + 256], stored as (p - 1) mod 256: bytes [start, start + n).
// Branch-free common case: the two words holding bytes [start & ~3, +8) cover
// the first k = min(n, 8 - start % 4) >= 5 entries, counted with a SIMD byte
// compare; longer lists (rare: n <= kXcMaxBlock) finish in a loop.  SM: tables
// in shared memory; else through L2 (evict-last).  Flagged superblocks use the
// plain X_M.
__device__ __forceinline__ uint2 ld_gather_v2(const uint2* p, uint64_t policy) {
  uint2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p), "l"(policy));
  return v;
}
template <bool SM>
__device__ __forceinline__ uint32_t xc_word(const uint32_t* p, uint64_t pol) {
  return SM ? *p : ld_gather_u32(p, pol);
}
__device__ __forceinline__ uint4 ld_gather_v4(const uint4* p, uint64_t policy) {
  uint4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(policy));
  return v;
}
// #{bytes b of word w at window positions [4i, 4i+4) with lo <= pos < hi and b < o}, x8
__device__ __forceinline__ uint32_t count_lt(uint32_t w, uint32_t ob, int i, uint32_t lo, uint32_t hi) {
  const uint32_t a = lo > 4u * i ? lo - 4u * i : 0u, z = hi > 4u * i ? hi - 4u * i : 0u;  // byte range [a, z)
  const uint32_t m = shl32(0xffffffffu, 8 * a) & (z >= 4 ? 0xffffffffu : shl32(1u, 8 * z) - 1u);
  return __popc(__vcmpltu4(w, ob) & m);
}
// Per-byte x < y over four packed bytes, as the byte's most significant bit
// (no cross-byte borrow: each byte of (x | 0x80) - (y & 0x7f) stays >= 1).
__device__ __forceinline__ uint32_t bytes_lt_msb(uint32_t x, uint32_t y, uint32_t y7) {
  const uint32_t z = (x | 0x80808080u) - y7;  // byte msb = (x & 0x7f) >= (y & 0x7f)
  // borrow out of x - y: (~x & y) | (~(x ^ y) & ~z), per byte msb
  return ((~x & y) | (~(x ^ y) & ~z)) & 0x80808080u;
}

// Shared-memory lookup (blocks of 256 codes, xs = 8).  The staging copy turns
// every 8-byte superblock record of the global XC into two 4-byte records, one
// per pair of 256-code blocks (512 codes): bits [0,7) = c1 = entries of the
// first block, [7,14) = c2 = entries of both blocks, [14,32) = R' = #new values
// inserted at or before the pair's first code (= the list start of the pair).
// A 4-byte random shared load costs fewer bank-conflict wavefronts than the
// 8-byte one, and the list window is read as one word plus two words predicated
// on the list actually reaching them (~2.6 entries per block on cfg2), so idle
// lanes take no bank slots.  Lists longer than 8 and flagged superblocks
// (rewritten as c1 = 127, c2 = 0: n = c2 - c1 wraps, so the fast path needs no
// flag test) report `slow`; the caller resolves them in one rare pass after all
// of a warp's lookups (xc4_slow), so the fast path is straight-line code whose
// loads the compiler can overlap across rows.  Counts are those of xc_lookup.
#ifndef DM_XC_HYB
#define DM_XC_HYB 0  // experiments: rows per lane and chunk translated by an L2 gather of X_M instead
#endif
constexpr uint32_t kXc4Flag = 127u;      // c1 = 127, c2 = 0: flagged superblock
constexpr uint32_t kXc4MaxStart = 1u << 18;
constexpr uint32_t kXcSmemSlack = 272;  // window reads up to start + 11 with start <= n_new + 127
__device__ __forceinline__ uint32_t xc4_fast(uint32_t code, uint32_t rec4_sa, uint32_t offs_sa, uint32_t& slow) {
  const uint32_t w = lds_u32(rec4_sa + ((code >> 9) << 2));
  const bool hi = (code & 256u) != 0u;
  const uint32_t c1 = w & 127u, c2 = (w >> 7) & 127u;
  const uint32_t s_rel = hi ? c1 : 0u, e_rel = hi ? c2 : c1;
  const uint32_t start = (w >> 14) + s_rel;
  const uint32_t n = e_rel - s_rel;  // wraps (huge) for a flagged record
  const uint32_t s3 = start & 3u, ns = n + s3;
  const uint32_t pa = offs_sa + (start & ~3u);
  const uint32_t w0 = lds_u32(pa);
  const uint32_t w1 = lds_u32_if(pa + 4, ns > 4u);
  const uint32_t w2 = lds_u32_if(pa + 8, ns > 8u);
  const uint32_t sh = 8u * s3;
  const uint32_t a = __funnelshift_r(w0, w1, sh), b = __funnelshift_r(w1, w2, sh);  // bytes [start, start + 8)
  const uint32_t y = (code & 255u) * 0x01010101u, y7 = y & 0x7f7f7f7fu;
  const uint32_t k8 = 8u * umin32(n, 8u);
  const uint32_t ma = ~shl32(0xffffffffu, k8), mb = shr32(0xffffffffu, 64u - k8);
  slow = n > 8u;
  return code + start + __popc(bytes_lt_msb(a, y, y7) & ma) + __popc(bytes_lt_msb(b, y, y7) & mb);
}
// The same lookup rebalanced for the pipes (the kernel is bound by the ALU pipe,
// ~75% busy, while the FMA pipe idles): shifts by constants become IMAD.HI /
// IMAD by runtime powers of two (k.m23 = 2^23, k.m18 = 2^18, kept opaque so
// ptxas cannot turn them back into shifts), the byte masks for the list length
// come from a 9-entry shared-memory table (one conflict-free LDS.64 instead of
// four ALU ops), and the window start is formed with adds.
struct Xc4Consts {
  uint32_t rec_sa, offs_sa, lut_sa, m23, m18, kpop, four, eight;
};
#ifndef DM_POPC_FMA
#define DM_POPC_FMA 0
#endif
__device__ __forceinline__ uint32_t mad_hi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint2 lds_u64(uint32_t a) {
  uint2 v;
  asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t xc4_fast2(uint32_t code, const Xc4Consts& k, uint32_t& slow) {
  const uint32_t ridx = __umulhi(code, k.m23);  // code >> 9
  const uint32_t w = lds_u32(ridx * k.four + k.rec_sa);
  const bool hi = (code & 256u) != 0u;
  const uint32_t c1 = w & 127u, c2 = (w >> 7) & 127u;
  const uint32_t s_rel = hi ? c1 : 0u, e_rel = hi ? c2 : c1;
  const uint32_t start = mad_hi(w, k.m18, s_rel);  // (w >> 14) + s_rel
  const uint32_t n = e_rel - s_rel;  // wraps (huge) for a flagged record
  const uint32_t s3 = start & 3u, ns = n + s3;
  const uint32_t pa = k.offs_sa + (start - s3);
  const uint32_t w0 = lds_u32(pa), w1 = lds_u32(pa + 4);
  const uint32_t w2 = lds_u32_if(pa + 8, ns > 8u);
  const uint2 m = lds_u64(umin32(n, 8u) * k.eight + k.lut_sa);  // byte-MSB masks of the first min(n, 8) bytes
  const uint32_t sh = 8u * s3;
  const uint32_t a = __funnelshift_r(w0, w1, sh), b = __funnelshift_r(w1, w2, sh);  // bytes [start, start + 8)
  const uint32_t y = __byte_perm(code, 0u, 0u), y7 = y & 0x7f7f7f7fu;
  const uint32_t za = (a | 0x80808080u) - y7, zb = (b | 0x80808080u) - y7;
  const uint32_t lta = ((~a & y) | (~(a ^ y) & ~za)) & m.x, ltb = ((~b & y) | (~(b ^ y) & ~zb)) & m.y;
  slow = n > 8u;
#if DM_POPC_FMA
  return code + start + (mad_hi(lta, k.kpop, __umulhi(ltb, k.kpop)) & 255u);
#else
  return code + start + __popc(lta) + __popc(ltb);
#endif
}

// The same lookup for the thread-per-group kernel, balanced for the two integer
// pipes (ALU: LOP3 / SHF / ISETP / PRMT; FMA: IMAD / IMAD.HI, each one warp
// instruction per 2 cycles per SM sub-partition): the record fields and the
// window arithmetic are multiply(-high)s by powers of two held in registers
// (opaque to ptxas, so they stay on the FMA pipe), the list words past the
// first are loaded only by lanes whose list reaches them, and the byte masks
// come from a 128-entry table indexed by n mod 128.
struct TpgK {  // powers of two (and -2) passed as kernel parameters, so ptxas cannot turn the multiplies into shifts
  uint32_t m23, m18, m25, m30, two, four, eight, m5, m7, m10, neg2;
  uint32_t xs;  // XC block shift (XC read through L2)
};
struct TpgXc {
  uint32_t rec_sa, offs_sa, lut_sa;
  TpgK c;
};
__device__ __forceinline__ uint32_t lds_u32_pred(uint32_t a, bool pred) {  // no value when !pred (masked later)
  uint32_t v;
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.u32 %0, [%1];\n}" : "=r"(v) : "r"(a), "r"((uint32_t)pred));
  return v;
}
__device__ __forceinline__ uint32_t xc4_tpg(uint32_t code, const TpgXc& k, bool& slow) {
  const TpgK& c = k.c;
  const uint32_t w = lds_u32(__umulhi(code, c.m23) * c.four + k.rec_sa);  // pair record of code >> 9
  const uint32_t hb = __umulhi(code * c.m23, c.two);                     // code bit 8: the second block
  const uint32_t c1 = w & 127u;                                           // entries of the first block
  const uint32_t c2 = __umulhi(w * c.m18, c.m7);                          // of both: bits [7, 14)
  const uint32_t start = __umulhi(w, c.m18) + c1 * hb;                    // R' + (hb ? c1 : 0)
  const uint32_t n = hb * (c1 * c.neg2 + c2) + c1;                        // wraps (huge) when flagged
  const uint32_t pa = __umulhi(start, c.m30) * c.four + k.offs_sa;        // word holding entry `start`
  const uint32_t sh = __umulhi(start * c.m30, c.m5);                      // 8 (start mod 4)
  const uint32_t ns8 = n * c.eight + sh;
  const uint32_t w0 = lds_u32(pa);
  const uint32_t w1 = lds_u32_pred(pa + 4, ns8 > 32u);
  const uint32_t w2 = lds_u32_pred(pa + 8, ns8 > 64u);
  const uint2 m = lds_u64(__umulhi(n * c.m25, c.m10) + k.lut_sa);        // masks of min(n mod 128, 8) bytes
  const uint32_t a = __funnelshift_r(w0, w1, sh), b = __funnelshift_r(w1, w2, sh);  // bytes [start, start + 8)
  const uint32_t y = __byte_perm(code, 0u, 0u), y7 = y & 0x7f7f7f7fu;
  const uint32_t za = (~a & 0x7f7f7f7fu) + y7, zb = (~b & 0x7f7f7f7fu) + y7;  // per byte: ~((a | 0x80) - y7)
  const uint32_t lta = ((~a & y) | (~(a ^ y) & za)) & m.x, ltb = ((~b & y) | (~(b ^ y) & zb)) & m.y;
  slow = n > 8u;
  return code + start + __popc(lta) + __popc(ltb);
}

// The rare case: a list longer than 8 entries (counted in a loop) or a flagged
// superblock (the plain X_M, global).
__device__ __noinline__ uint32_t xc4_slow(uint32_t code, const uint32_t* __restrict__ rec4,
                                          const uint32_t* __restrict__ offs32, const uint32_t* __restrict__ XM) {
  const uint32_t w = rec4[code >> 9];
  const uint32_t c1 = w & 127u, c2 = (w >> 7) & 127u;
  if (c1 == kXc4Flag && c2 == 0u) return __ldg(XM + code);
  const bool hi = (code & 256u) != 0u;
  const uint32_t s_rel = hi ? c1 : 0u, e_rel = hi ? c2 : c1;
  const uint32_t start = (w >> 14) + s_rel, o = code & 255u;
  DM_ASSERT(e_rel - s_rel <= 2 * kXcMaxBlock, "xc4 list n %u", e_rel - s_rel);
  uint32_t cnt = 0;
  for (uint32_t q = start; q < start + (e_rel - s_rel); ++q) cnt += ((offs32[q >> 2] >> (8 * (q & 3u))) & 255u) < o;
  return code + start + cnt;
}
// Staging: the 4-byte pair record h from the global 8-byte superblock record.
__device__ __forceinline__ uint32_t xc4_record(uint2 r, uint32_t half) {
  const uint32_t R = r.x & 0x7fffffffu;
  const uint32_t b0 = r.y & 255u, b1 = (r.y >> 8) & 255u, b2 = (r.y >> 16) & 255u, b3 = r.y >> 24;
  const uint32_t base = half ? b1 : 0u, c1 = half ? b2 - b1 : b0, c2 = half ? b3 - b1 : b1;
  const uint32_t Rp = R + base;
  if ((r.x >> 31) || c2 > 126u || Rp >= kXc4MaxStart) return (umin32(Rp, kXc4MaxStart - 1) << 14) | kXc4Flag;
  return (Rp << 14) | (c2 << 7) | c1;
}

// xs: block shift (blocks of 2^xs codes, superblocks of 4 blocks).
template <bool SM>
__device__ __forceinline__ uint32_t xc_lookup(uint32_t code, uint32_t xs, const uint2* __restrict__ rec,
                                              const uint32_t* __restrict__ offs32, const uint32_t* __restrict__ XM,
                                              uint64_t pol) {
  const uint32_t sb = code >> (xs + 2), t8 = 8 * ((code >> xs) & 3u), o = code & ((1u << xs) - 1u);
  const uint2 r = SM ? rec[sb] : ld_gather_v2(rec + sb, pol);
  const bool flagged = r.x >> 31;
  const uint32_t xm_flagged = flagged ? __ldg(XM + code) : 0u;  // predicated, no divergence
  const uint32_t s_rel = ((r.y << 8) >> t8) & 255u, e_rel = (r.y >> t8) & 255u;
  const uint32_t start = (r.x & 0x7fffffffu) + s_rel, n = flagged ? 0u : e_rel - s_rel;
  const uint32_t ob = o * 0x01010101u;
  uint32_t cnt, k;
  if constexpr (SM) {
    // shared memory: the two words holding bytes [start & ~3, +8)
    const uint32_t wi = start >> 2, sh = 8 * (start & 3u);
    const uint32_t w0 = offs32[wi], w1 = offs32[wi + 1];
    const uint32_t a = __funnelshift_r(w0, w1, sh), b = w1 >> sh;  // bytes start.., start+4..
    k = umin32(n, 8u - (start & 3u));
    const uint32_t ka = umin32(k, 4u);
    cnt = __popc(__vcmpltu4(a, ob) & (shl32(1u, 8 * ka) - 1u)) +
          __popc(__vcmpltu4(b, ob) & (shl32(1u, 8 * (k - ka)) - 1u));
  } else {
    // L2: the aligned 16-byte window holding start, and (predicated, issued
    // together, no dependent round trip) the next one when the list crosses it
    const uint32_t s0 = start & 15u;
    const uint4* base4 = reinterpret_cast<const uint4*>(offs32) + (start >> 4);
    const uint4 v = ld_gather_v4(base4, pol);
    const uint4 w = s0 + n > 16u ? ld_gather_v4(base4 + 1, pol) : make_uint4(0, 0, 0, 0);
    k = umin32(n, 32u - s0);
    const uint32_t e0 = s0 + k;
    cnt = count_lt(v.x, ob, 0, s0, e0) + count_lt(v.y, ob, 1, s0, e0) + count_lt(v.z, ob, 2, s0, e0) +
          count_lt(v.w, ob, 3, s0, e0) + count_lt(w.x, ob, 4, s0, e0) + count_lt(w.y, ob, 5, s0, e0) +
          count_lt(w.z, ob, 6, s0, e0) + count_lt(w.w, ob, 7, s0, e0);
  }
  if (__builtin_expect(n > k, 0)) {
    for (uint32_t q = start + k; q < start + n; ++q) {  // rare tail (n <= kXcMaxBlock)
      const uint32_t w = xc_word<SM>(offs32 + (q >> 2), pol);
      cnt += ((w >> (8 * (q & 3u))) & 255u) < o ? 8u : 0u;
    }
  }
  return flagged ? xm_flagged : code + start + (cnt >> 3);
}

// xc_lookup<false> without its tail loop, for the thread-per-group kernel: `slow`
// when the list runs past the two 16-byte windows (rare: > 16 entries from the
// window start); the caller finishes those rows after the straight-line pass.
__device__ __forceinline__ uint32_t xc_l2_fast(uint32_t code, uint32_t xs, const uint2* __restrict__ rec,
                                               const uint32_t* __restrict__ offs32, const uint32_t* __restrict__ XM,
                                               uint64_t pol, bool& slow) {
  const uint32_t sb = code >> (xs + 2), t8 = 8 * ((code >> xs) & 3u), o = code & ((1u << xs) - 1u);
  const uint2 r = ld_gather_v2(rec + sb, pol);
  const bool flagged = r.x >> 31;
  const uint32_t xm_flagged = flagged ? __ldg(XM + code) : 0u;
  const uint32_t s_rel = ((r.y << 8) >> t8) & 255, e_rel = (r.y >> t8) & 255;
  const uint32_t start = (r.x & 0x7fffffffu) + s_rel, n = flagged ? 0u : e_rel - s_rel;
  const uint32_t ob = o * 0x01010101u;
  const uint32_t s0 = start & 15u;
  const uint4* base4 = reinterpret_cast<const uint4*>(offs32) + (start >> 4);
  const uint4 v = ld_gather_v4(base4, pol);
  const uint4 w = s0 + n > 16u ? ld_gather_v4(base4 + 1, pol) : make_uint4(0, 0, 0, 0);
  const uint32_t k = umin32(n, 32u - s0), e0 = s0 + k;
  const uint32_t cnt = count_lt(v.x, ob, 0, s0, e0) + count_lt(v.y, ob, 1, s0, e0) + count_lt(v.z, ob, 2, s0, e0) +
                       count_lt(v.w, ob, 3, s0, e0) + count_lt(w.x, ob, 4, s0, e0) + count_lt(w.y, ob, 5, s0, e0) +
                       count_lt(w.z, ob, 6, s0, e0) + count_lt(w.w, ob, 7, s0, e0);
  slow = n > k;
  return flagged ? xm_flagged : code + start + (cnt >> 3);
}

template <int XMODE>
__host__ __device__ constexpr int rec_consumer_warps() { return XMODE == XM_XC_SMEM ? 28 : kRecConsumerWarps; }
// 32-row groups per chunk: a multiple of 4 (16-byte aligned chunks at any width)
// and of the consumer warp count
template <int XMODE>
__host__ __device__ constexpr int rec_groups() { return XMODE == XM_XC_SMEM ? 112 : kRecGroups; }
template <int XMODE>
__host__ __device__ constexpr int rec_threads() { return 32 * (rec_consumer_warps<XMODE>() + 1); }

template <int NB, int XMODE>
__global__ void __launch_bounds__(rec_threads<XMODE>(), XMODE == XM_XC_SMEM ? 1 : 2) k_recompress(const uint64_t* __restrict__ M, uint64_t n_main, uint32_t b,
                                                            uint64_t dict_len, const uint32_t* __restrict__ XM,
                                                            const uint32_t* __restrict__ XD,
                                                            const uint32_t* __restrict__ rank, uint64_t n_delta,
                                                            uint64_t* __restrict__ Mout, dm_header* hdr,
                                                            uint32_t in_stage_bytes, uint32_t fixed_bits,
                                                            const uint2* __restrict__ xrec,
                                                            const uint8_t* __restrict__ xoffs, uint32_t xc_budget,
                                                            uint32_t xc_dens, uint32_t xs) {
  pdl_prologue();
  constexpr int G = rec_groups<XMODE>();
  constexpr int S = XMODE == XM_XC_SMEM ? kRecStagesXc : kRecStages;
  constexpr int CW = rec_consumer_warps<XMODE>();
  constexpr int U = G / CW;  // groups per consumer warp per chunk, all in flight together
  constexpr bool XS = XMODE == XM_RAW_SMEM;
  static_assert(G % CW == 0, "groups must split evenly over consumer warps");
  const uint32_t hb = fixed_bits ? fixed_bits : hdr->merged_bits;
  if (NB > 0 && hb != (uint32_t)NB) return;
  const uint32_t nb = NB > 0 ? (uint32_t)NB : hb;
  const uint64_t nsb = (dict_len + (4ull << xs) - 1) >> (xs + 2);
  uint64_t xc_offs_bytes = 0;
  if (xc_budget) {
    const uint64_t n_new = hdr->merged_dict_len - dict_len;
    xc_offs_bytes = (n_new + 15) & ~15ull;
    // + slack: the window reads past the last entry (kXcSmemSlack)
    // xc_dens (auto mode): also require n_new * 2^xc_dens <= |U_M|, i.e. short
    // lists (cfg2: 2.6 entries per 256-code block), else the L2 companion runs
    // (and n_new < 2^18: the 4-byte shared-memory records hold list starts in 18 bits)
    const bool fits = ((nsb * kXcRecBytes + 15) & ~15ull) + xc_offs_bytes + kXcSmemSlack <= xc_budget &&
                      (xc_dens == 0 || (n_new << xc_dens) <= dict_len) && n_new < kXc4MaxStart;
    if ((XMODE == XM_XC_SMEM) != fits) return;
  }

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + S;
  uint2* lut = reinterpret_cast<uint2*>(smem_raw + 128);  // XC list masks by length (xc4_fast2)
  unsigned char* in_ring = smem_raw + kRecHdrBytes;
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
  if (threadIdx.x < 9) {  // lut[n]: MSB of each of the first min(n, 8) bytes of an 8-byte window
    const uint32_t n = threadIdx.x;
    lut[n] = make_uint2(0x80808080u & (n >= 4 ? 0xffffffffu : (1u << (8 * n)) - 1u),
                        0x80808080u & (n >= 8 ? 0xffffffffu : n <= 4 ? 0u : (1u << (8 * (n - 4))) - 1u));
  }
  if (XS) {
    for (uint32_t i = threadIdx.x; i < dict_len; i += blockDim.x) sx[i] = __ldg(XM + i);
  }
  const uint32_t* srec4 = sx;
  const uint64_t rec_pad = (nsb * kXcRecBytes + 15) & ~15ull;
  const uint32_t* soffs = reinterpret_cast<const uint32_t*>(reinterpret_cast<unsigned char*>(sx) + rec_pad);
  if (XMODE == XM_XC_SMEM) {
    // one bulk copy of the records and one of the lists (the global arrays are
    // padded to 16 bytes), then two 8-byte records -> four 4-byte ones in place
    uint64_t* stage_bar = empty + S;  // header bytes [64, 72): after full[4], empty[4]
    static_assert(2 * S * 8 + 8 <= 128, "staging barrier fits before the mask table");
    if (threadIdx.x == 0) {
      mbar_init(stage_bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(stage_bar, (uint32_t)(rec_pad + xc_offs_bytes));
      tma_load_1d(sx, xrec, (uint32_t)rec_pad, stage_bar, policy_evict_last());
      if (xc_offs_bytes)
        tma_load_1d(reinterpret_cast<unsigned char*>(sx) + rec_pad, xoffs, (uint32_t)xc_offs_bytes, stage_bar,
                    policy_evict_last());
    }
    mbar_wait_parity(stage_bar, 0);
    uint4* d = reinterpret_cast<uint4*>(sx);
    for (uint32_t i = threadIdx.x; i < rec_pad / 16; i += blockDim.x) {
      const uint4 v = d[i];
      d[i] = make_uint4(xc4_record(make_uint2(v.x, v.y), 0), xc4_record(make_uint2(v.x, v.y), 1),
                        xc4_record(make_uint2(v.z, v.w), 0), xc4_record(make_uint2(v.z, v.w), 1));
    }
  }
  __syncthreads();

  if (warp == CW) {  // ---------------------------------------------------- producer
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();
      for (uint64_t k = 0;; ++k) {
        const uint64_t c = blockIdx.x + k * gridDim.x;
        if (c >= nchunks) break;
        const int s = (int)(k % S);
        if (k >= S) mbar_wait_parity_sleep(&empty[s], (uint32_t)(((k / S) - 1) & 1));
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
  const uint32_t srec4_sa = smem_u32(srec4), soffs_sa = smem_u32(soffs);
  const Xc4Consts xk{srec4_sa, soffs_sa, smem_u32(lut), 1u << (xs + 15), 1u << (xs + 10), 0x02020202u + (xs - 8),
                     xs - 4, xs};  // xs = 8 here: four = 4, eight = 8, opaque to ptxas (IMAD, not LEA)
  const uint32_t us = lane * b, uw0 = us >> 5, uo = us & 31;
  const uint32_t umask = b == 32 ? 0xffffffffu : ((1u << b) - 1);
  const uint32_t pr0 = (32 * lane) / nb, pop = 32 * lane - pr0 * nb;
  const FmaPack<use_fma_pack<NB>() ? NB : 8> fpk(lane);
  auto pack = [&](uint32_t x) -> uint32_t {
    if constexpr (use_fma_pack<NB>())
      return fpk.pack(x);
    else
      return warp_pack<NB>(x, nb, pr0, pop);
  };
  uint32_t* out32 = reinterpret_cast<uint32_t*>(Mout);
  // codes >= |U_M| are clamped (reads stay in the table) and reported once at
  // the end through the running maximum: two ALU ops per row
  const uint32_t dict_last = (uint32_t)dict_len - 1u;  // |U_M| >= 1 when N_M > 0 (validated by the ABI)
  uint32_t code_max = 0;

  // chunks [0, n_fast) are all-main and lie wholly inside M': no per-row bounds
  // and no per-word store predicate beyond lane < b'
  const uint64_t n_fast = umin64(n_main / R, nw32 / ((uint64_t)G * nb));
  int s = 0;
  uint32_t phase = 0;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    mbar_wait_parity_sleep(&full[s], phase);
    const uint32_t* sin = reinterpret_cast<const uint32_t*>(in_ring + (size_t)s * in_stage_bytes);
    uint32_t v[U];
    auto translate = [&](uint32_t code) -> uint32_t {
      code_max = umax32(code_max, code);
      code = umin32(code, dict_last);
      if constexpr (XMODE == XM_RAW_SMEM)
        return sx[code];
      else if constexpr (XMODE == XM_XC_SMEM) {
        uint32_t slow;
        const uint32_t x = xc4_fast2(code, xk, slow);
        return slow ? xc4_slow(code, srec4, soffs, XM) : x;
      }
      else if constexpr (XMODE == XM_XC_GLOBAL)
        return xc_lookup<false>(code, xs, xrec, reinterpret_cast<const uint32_t*>(xoffs), XM, pol_x);
      else
        return ld_gather_u32(XM + code, pol_x);
    };
    const bool fast = c < n_fast;
    if (fast) {
      if constexpr (XMODE == XM_XC_SMEM) {
        // straight-line fast lookups for all U rows of this lane, then one rare
        // pass for the long lists / flagged superblocks
        uint32_t cd[U], slow = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int g = warp + CW * u;
          const uint32_t lo = sin[g * b + uw0], hi = sin[g * b + uw0 + 1];
          const uint32_t code = __funnelshift_r(lo, hi, uo) & umask;
          code_max = umax32(code_max, code);
          cd[u] = umin32(code, dict_last);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (u >= U - DM_XC_HYB) {  // experiment: some rows gather the plain X_M through L2 (LSU, not ALU)
            v[u] = ld_gather_u32(XM + cd[u], pol_x);
            continue;
          }
          uint32_t su;
          v[u] = xc4_fast2(cd[u], xk, su);
          slow |= su << u;
        }
        if (__builtin_expect(slow != 0u, 0)) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (slow & (1u << u)) v[u] = xc4_slow(cd[u], srec4, soffs, XM);
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int g = warp + CW * u;
          const uint32_t lo = sin[g * b + uw0], hi = sin[g * b + uw0 + 1];
          v[u] = translate(__funnelshift_r(lo, hi, uo) & umask);
        }
      }
    } else {
      const uint64_t row_base = c * R;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int g = warp + CW * u;
        const uint64_t row = row_base + (uint64_t)g * 32 + lane;
        if (row < n_main) {
          const uint32_t lo = sin[g * b + uw0], hi = sin[g * b + uw0 + 1];
          v[u] = translate(__funnelshift_r(lo, hi, uo) & umask);
        } else if (row < n_total) {
          v[u] = __ldg(XD + (rank ? __ldg(rank + (row - n_main)) : (uint32_t)(row - n_main)));
        } else {
          v[u] = 0;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // stage s fully read by this warp
    if (++s == S) s = 0, phase ^= 1u;
    // output: group g of chunk c is words [(c G + g) b', +b'); lane k < b' writes word k
    uint32_t* outc = out32 + (c * G + warp) * (uint64_t)nb + lane;
    if ((c + 1) * G * (uint64_t)nb <= nw32) {  // the whole chunk is inside M' (all but the last)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t word = pack(v[u]);
        if (lane < nb) __stcs(outc + (size_t)CW * u * nb, word);
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int g = warp + CW * u;
        const uint32_t word = pack(v[u]);
        const uint64_t ow = (c * G + g) * nb + lane;
        if (lane < nb && ow < nw32) __stcs(out32 + ow, word);
      }
    }
  }
  const bool bad = n_main > 0 && code_max > dict_last;
  if (__any_sync(FULL, bad) && lane == 0) atomicMin(&hdr->status, (int)DM_E_CODE_RANGE);
}

// ---------------------------------------------------------------------------
// Step 2(b), thread-per-group form (XC in shared memory).  The warp-per-group
// kernel above spends ~35 of its ~80 instructions per row on the streaming
// structure (two unpack loads, funnel, shuffle-pack, per-chunk 64-bit index
// math) around the XC lookup (ncu r02: 259M warp instructions for cfg2, issue
// active 75%).  Here lane l owns a whole 32-row group of a tile of 32 groups
// (1024 rows): it reads the group's b input words from shared memory with
// 16-byte loads, extracts the 32 codes with compile-time shifts, translates
// them, and assembles the b' output words in registers (compile-time shifts,
// disjoint bits: multiply-adds on the FMA pipe) -- no shuffles, ~5 instructions
// per row of streaming work.  b and b' are template parameters (b' - b in
// {0, 1}, the usual growth); other width pairs keep the warp-per-group kernel.
//   * every warp runs its own pipeline over tiles: kTpgSlots shared-memory
//     slots, each filled by one bulk TMA copy of the tile (128 b bytes) that
//     completes on the slot's mbarrier;
//   * the output words go back into the same slot (in place, after a
//     __syncwarp: every lane holds its input in registers) and leave by one
//     bulk TMA store; the slot is refilled once that store has read it
//     (bulk-group wait at the top of the next tile);
//   * the rare lookups the fast path cannot finish (a list longer than 8, a
//     flagged superblock) read the plain X_M, which is whole whenever this
//     kernel runs (its L2 companion is the plain-X_M kernel);
//   * tiles holding delta rows or the ragged end keep the lane-per-group
//     layout with run-time row checks: input words and ranks from global, all
//     32 gathers of a lane independent.
// XC is staged by two bulk copies and converted to the 4-byte pair records in
// place.  The number of warps per CTA follows from the shared memory XC leaves
// (decided on the device from |U'|, like the XC fit itself).
// Measured (cfg2, B200): 0.298 ms vs 0.312 ms for the warp-per-group kernel,
// 169M vs 259M warp instructions; with the lookup replaced by the identity
// (DM_TPG_NOLOOKUP, timing only) 0.127 ms = 0.79 of the HBM copy peak: the
// stream is no longer the limit, the ~45 instructions and ~13 shared-memory
// wavefronts per 32 lookups are.
#ifndef DM_TPG_DIRECT
#define DM_TPG_DIRECT 1  // XC in smem: no tile slots -- input words straight into registers, output by 16-byte stores
#endif
#ifndef DM_TPG_V8
#define DM_TPG_V8 1  // direct form: 32-byte global loads / stores when b, b' are multiples of 8 and M, M' are 32-byte aligned (checked at run time: the ABI asks for 16)
#endif
// 256-bit global accesses (sm_100: LDG.E.ENL2.256 / STG.E.ENL2.256)
__device__ __forceinline__ void ld_v8_na(const void* p, uint32_t* v) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "l"(p));
}
__device__ __forceinline__ void st_v8_cs(void* p, const uint32_t* v) {
  asm volatile("st.global.cs.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
template <int B, int NB>
struct Tpg {
  static constexpr uint32_t slot_bytes = 128u * (B > NB ? B : NB);  // one tile in, then out (in place)
};
#ifndef DM_TPG_PATCH
#define DM_TPG_PATCH 1  // XC in smem: slow rows patched after the pass (1) or a predicated X_M read per row (0)
#endif
#ifndef DM_TPG_NOLOOKUP
#define DM_TPG_NOLOOKUP 0
#endif
#ifndef DM_TPG_SLOTS
#define DM_TPG_SLOTS 2
#endif
#ifndef DM_TPG_WARPS
#define DM_TPG_WARPS 8
#endif
// Two slots per warp (the next tile loads while this one is translated) and up
// to 8 warps.  Measured on cfg2 (B200): 2 x 8 0.298 ms; 1 slot x 16 warps (the
// load of the next tile waits for the store of this one) 0.314-0.321 ms.
constexpr int kTpgSlots = DM_TPG_SLOTS;
constexpr int kTpgWarps = DM_TPG_WARPS;
constexpr int kTpgMinWarps = 4;
constexpr int kTpgMinWidth = 15;  // XC in shared memory needs |U_M| > 24576
constexpr int kTpgBarBytes = (kTpgWarps * kTpgSlots * 8 + 127) / 128 * 128;  // slot mbarriers
constexpr int kTpgHdrBytes = kTpgBarBytes + 128 * 8 + 128;  // slot mbarriers, the 128-entry list-mask table, the staging mbarrier

template <int B>
__device__ __forceinline__ uint32_t tpg_code(const uint32_t (&w)[B], int r) {
  constexpr uint32_t mask = B == 32 ? 0xffffffffu : (1u << B) - 1u;
  const int s = r * B, i = s >> 5, o = s & 31;
  if (o + B <= 32) return (w[i] >> o) & mask;
  return __funnelshift_r(w[i], w[i + 1], o) & mask;
}
template <int NB>
__device__ __forceinline__ void tpg_put(uint32_t (&o)[NB], int r, uint32_t v) {
  const int s = r * NB, i = s >> 5, sh = s & 31;
  o[i] += v * (1u << sh);  // the codes of a word occupy disjoint bits (IMAD / IMAD.HI: the FMA pipe)
  if (sh + NB > 32) o[i + 1] = mad_hi(v, 1u << sh, o[i + 1]);
}

template <int B, int NB, int XMODE>
__global__ void __launch_bounds__(32 * kTpgWarps, 1)
    k_recompress_tpg(const uint64_t* __restrict__ M, uint64_t n_main, uint64_t dict_len,
                     const uint32_t* __restrict__ XM, const uint32_t* __restrict__ XD,
                     const uint32_t* __restrict__ rank, uint64_t n_delta, uint64_t* __restrict__ Mout,
                     dm_header* hdr, uint32_t fixed_bits, const uint2* __restrict__ xrec,
                     const uint8_t* __restrict__ xoffs, uint32_t xc_budget, uint32_t xc_dens, TpgK kc,
                     uint32_t smem_bytes) {
  pdl_prologue();
  using T = Tpg<B, NB>;
  constexpr bool XCS = XMODE == XM_XC_SMEM, XS = XMODE == XM_RAW_SMEM;
  const uint32_t hb = fixed_bits ? fixed_bits : hdr->merged_bits;
  if (hb != (uint32_t)NB) return;
  // the XC fit: the same rule (and budget) for the shared-memory kernel and its
  // L2 companion (exactly one of them runs)
  const uint64_t nsb = (dict_len + 1023) >> 10;
  const uint64_t n_new = hdr->merged_dict_len - dict_len;
  const uint64_t xc_offs_bytes = (n_new + 15) & ~15ull;
  const uint64_t rec_pad = (nsb * kXcRecBytes + 15) & ~15ull;
  const uint64_t xc_bytes = rec_pad + xc_offs_bytes + kXcSmemSlack;
  if (xc_budget) {
    const bool fits = xc_bytes <= xc_budget && (xc_dens == 0 || (n_new << xc_dens) <= dict_len) && n_new < kXc4MaxStart;
    if (XCS != fits) return;
  }

  extern __shared__ __align__(128) unsigned char smem_raw[];
  // XC in shared memory: the tiles bypass shared memory (DM_TPG_DIRECT); the
  // other modes stage them in per-warp slots filled / drained by bulk copies
  constexpr bool DIR = DM_TPG_DIRECT && XCS;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);          // kTpgWarps x kTpgSlots
  uint2* lut = reinterpret_cast<uint2*>(smem_raw + kTpgBarBytes);   // 128 entries
  uint32_t* sx = reinterpret_cast<uint32_t*>(smem_raw + kTpgHdrBytes);
  const uint64_t table_bytes = XCS ? xc_bytes : XS ? dict_len * 4 : 0;
  const uint32_t slot0 = (uint32_t)((kTpgHdrBytes + table_bytes + 127) & ~127ull);
  const int W = DIR ? (int)(blockDim.x >> 5) : (int)umin32(blockDim.x >> 5, (smem_bytes - slot0) / (kTpgSlots * T::slot_bytes));

  if (!DIR && threadIdx.x == 0) {
    for (int i = 0; i < kTpgWarps * kTpgSlots; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  if (XCS && threadIdx.x < 128) {  // lut[n]: MSB of each of the first min(n, 8) bytes of an 8-byte window
    const uint32_t n = umin32(threadIdx.x, 8u);
    lut[threadIdx.x] = make_uint2(0x80808080u & (n >= 4 ? 0xffffffffu : (1u << (8 * n)) - 1u),
                                  0x80808080u & (n >= 8 ? 0xffffffffu : n <= 4 ? 0u : (1u << (8 * (n - 4))) - 1u));
  }
  if constexpr (XCS) {
    // XC staging: one bulk copy of the records and one of the lists (the global
    // arrays are padded to 16 bytes), then every 8-byte superblock record becomes
    // two 4-byte pair records in place (same size)
    uint64_t* stage_bar = reinterpret_cast<uint64_t*>(smem_raw + kTpgBarBytes + 128 * 8);
    if (threadIdx.x == 0) {
      mbar_init(stage_bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(stage_bar, (uint32_t)(rec_pad + xc_offs_bytes));
      tma_load_1d(sx, xrec, (uint32_t)rec_pad, stage_bar, policy_evict_last());
      if (xc_offs_bytes)
        tma_load_1d(reinterpret_cast<unsigned char*>(sx) + rec_pad, xoffs, (uint32_t)xc_offs_bytes, stage_bar,
                    policy_evict_last());
    }
    mbar_wait_parity(stage_bar, 0);
    uint4* d = reinterpret_cast<uint4*>(sx);
    for (uint32_t i = threadIdx.x; i < rec_pad / 16; i += blockDim.x) {
      const uint4 v = d[i];
      d[i] = make_uint4(xc4_record(make_uint2(v.x, v.y), 0), xc4_record(make_uint2(v.x, v.y), 1),
                        xc4_record(make_uint2(v.z, v.w), 0), xc4_record(make_uint2(v.z, v.w), 1));
    }
  } else if constexpr (XS) {
    for (uint32_t i = threadIdx.x; i < dict_len; i += blockDim.x) sx[i] = __ldg(XM + i);
  }
  __syncthreads();
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  if ((int)warp >= W) return;

  const uint32_t* srec4 = sx;
  const uint32_t* soffs = reinterpret_cast<const uint32_t*>(reinterpret_cast<unsigned char*>(sx) + rec_pad);
  const TpgXc xk{smem_u32(srec4), smem_u32(soffs), smem_u32(lut), kc};
  const uint64_t pol_x = policy_evict_last();
  // X_M[cc]; XC in shared memory: `slow` set when the fast lookup cannot finish
  // (a list longer than 8, a flagged superblock) -- then the plain X_M, which is
  // whole whenever this kernel runs (its L2 companion is the plain-X_M kernel)
  auto translate = [&](uint32_t cc, bool& slow) -> uint32_t {
    slow = false;
#if DM_TPG_NOLOOKUP  // timing experiment only (wrong results): the streaming structure alone
    return cc;
#endif
    if constexpr (XCS)
      return xc4_tpg(cc, xk, slow);
    else if constexpr (XS)
      return sx[cc];
    else if constexpr (XMODE == XM_XC_GLOBAL)
      return xc_l2_fast(cc, kc.xs, xrec, reinterpret_cast<const uint32_t*>(xoffs), XM, pol_x, slow);
    else
      return ld_gather_u32(XM + cc, pol_x);
  };
  auto exact = [&](uint32_t cc) -> uint32_t {  // the rare rows `translate` could not finish
    if constexpr (XMODE == XM_XC_GLOBAL)
      return xc_lookup<false>(cc, kc.xs, xrec, reinterpret_cast<const uint32_t*>(xoffs), XM, pol_x);
    else
      return __ldg(XM + cc);  // XC in smem: the plain X_M is whole whenever that kernel runs
  };
  constexpr bool XCG = XMODE == XM_XC_GLOBAL;
  const uint32_t dict_last = (uint32_t)dict_len - 1u;
  uint32_t code_max = 0;
  const uint64_t n_total = n_main + n_delta;
  const uint64_t n_tiles = (n_total + 1023) >> 10;
  const uint64_t n_fast = n_main >> 10;  // tiles of main rows only: input and output wholly inside M, M'
  const uint64_t gw = (uint64_t)blockIdx.x * W + warp, GW = (uint64_t)gridDim.x * W;
  uint64_t* full = bars + warp * kTpgSlots;
  unsigned char* slots = smem_raw + slot0 + (size_t)warp * kTpgSlots * T::slot_bytes;
  const uint64_t pol = policy_evict_first();
  const unsigned char* Mb = reinterpret_cast<const unsigned char*>(M);
  unsigned char* Ob = reinterpret_cast<unsigned char*>(Mout);

  if constexpr (DIR) {
  // No slots: a lane's b input words come straight from global memory into
  // registers (16-byte loads; the next tile's are in flight while this one is
  // translated) and its b' output words leave by 16-byte streaming stores, so
  // shared memory holds only the table and the CTA can run more warps.
  uint32_t wn[B];
  // 32-byte accesses (every one a whole sector; cfg2 Step 2(b) 0.278 -> 0.275 ms) need M and M'
  // 32-byte aligned: a tile starts at a multiple of 128 b bytes and a lane's words at 4 b l
  const bool al32 = ((reinterpret_cast<uintptr_t>(M) | reinterpret_cast<uintptr_t>(Mout)) & 31u) == 0;
  auto gload = [&](uint64_t t) {
    const unsigned char* src = Mb + t * (uint64_t)(128 * B) + lane * (B * 4);
    if constexpr (B % 8 == 0 && DM_TPG_V8) {
      if (al32) {
#pragma unroll
        for (int i = 0; i < B / 8; ++i) ld_v8_na(src + 32 * i, &wn[8 * i]);
        return;
      }
    }
    if constexpr (B % 4 == 0) {
#pragma unroll
      for (int i = 0; i < B / 4; ++i) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + i);
        wn[4 * i] = v.x, wn[4 * i + 1] = v.y, wn[4 * i + 2] = v.z, wn[4 * i + 3] = v.w;
      }
    } else if constexpr (B % 2 == 0) {
#pragma unroll
      for (int i = 0; i < B / 2; ++i) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(src) + i);
        wn[2 * i] = v.x, wn[2 * i + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < B; ++i) wn[i] = __ldg(reinterpret_cast<const uint32_t*>(src) + i);
    }
  };
#ifndef DM_TPG_PREFETCH
#define DM_TPG_PREFETCH 1  // 0: the tile's words loaded at its start (fewer registers, more warps hide the latency)
#endif
  if (DM_TPG_PREFETCH && gw < n_fast) gload(gw);
  for (uint64_t t = gw; t < n_fast; t += GW) {
    if (!DM_TPG_PREFETCH) gload(t);
    uint32_t w[B];
#pragma unroll
    for (int i = 0; i < B; ++i) w[i] = wn[i];
    if (DM_TPG_PREFETCH && t + GW < n_fast) gload(t + GW);
    uint32_t o[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) o[i] = 0;
    uint32_t smask = 0;
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const uint32_t c = tpg_code<B>(w, r);
      code_max = umax32(code_max, c);
      const uint32_t cc = umin32(c, dict_last);
      bool su;
      const uint32_t v = translate(cc, su);
      if (XCG || (XCS && DM_TPG_PATCH)) smask |= (uint32_t)su << r;
      tpg_put<NB>(o, r, (XCS && !DM_TPG_PATCH && su) ? __ldg(XM + cc) : v);
    }
    unsigned char* dst = Ob + t * (uint64_t)(128 * NB) + lane * (NB * 4);
    bool stored = false;
    if constexpr (NB % 8 == 0 && DM_TPG_V8) {
      if (al32) {
#pragma unroll
        for (int i = 0; i < NB / 8; ++i) st_v8_cs(dst + 32 * i, &o[8 * i]);
        stored = true;
      }
    }
    if (stored) {
    } else if constexpr (NB % 4 == 0) {
#pragma unroll
      for (int i = 0; i < NB / 4; ++i)
        __stcs(reinterpret_cast<uint4*>(dst) + i, make_uint4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]));
    } else if constexpr (NB % 2 == 0) {
#pragma unroll
      for (int i = 0; i < NB / 2; ++i) __stcs(reinterpret_cast<uint2*>(dst) + i, make_uint2(o[2 * i], o[2 * i + 1]));
    } else {
#pragma unroll
      for (int i = 0; i < NB; ++i) __stcs(reinterpret_cast<uint32_t*>(dst) + i, o[i]);
    }
    if ((XCG || (XCS && DM_TPG_PATCH)) && smask) {  // rare, per lane: exact values patched into the lane's own words
      uint32_t* ow = reinterpret_cast<uint32_t*>(dst);
      const uint32_t* M32 = reinterpret_cast<const uint32_t*>(M);
      constexpr uint32_t cmask = B == 32 ? 0xffffffffu : (1u << B) - 1u;
      constexpr uint64_t vmask = NB == 32 ? 0xffffffffull : (1ull << NB) - 1ull;
      do {
        const uint32_t r = __ffs(smask) - 1;
        smask &= smask - 1;
        const uint64_t bi = ((t * 32 + lane) * 32 + r) * (uint64_t)B;
        const uint64_t wi = bi >> 5;
        const uint32_t hi = wi + 1 < 2 * dwords(n_main, B) ? __ldg(M32 + wi + 1) : 0u;
        const uint32_t c = __funnelshift_r(__ldg(M32 + wi), hi, (uint32_t)(bi & 31)) & cmask;
        const uint64_t v = exact(umin32(c, dict_last));
        const uint32_t ob = r * NB, i = ob >> 5, sh = ob & 31;
        uint64_t x = ow[i] | (i + 1 < (uint32_t)NB ? (uint64_t)ow[i + 1] << 32 : 0ull);
        x = (x & ~(vmask << sh)) | (v << sh);
        ow[i] = (uint32_t)x;
        if (i + 1 < (uint32_t)NB) ow[i + 1] = (uint32_t)(x >> 32);
      } while (smask);
    }
  }
  } else {
  auto issue = [&](uint64_t t, int k) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&full[k], 128u * B);
      tma_load_1d(slots + k * T::slot_bytes, Mb + t * (uint64_t)(128 * B), 128u * B, &full[k], pol);
    }
  };
#pragma unroll
  for (int k = 0; k < kTpgSlots; ++k)
    if (gw + k * GW < n_fast) issue(gw + k * GW, k);

  uint64_t j = 0;
  for (uint64_t t = gw; t < n_fast; t += GW, ++j) {
    const int k = (int)(j % kTpgSlots);
    if (j > 0) {  // the previous tile's store has read its slot: refill it
      tma_store_wait_read<0>();
      __syncwarp();
      const uint64_t tn = t + (kTpgSlots - 1) * GW;
      if (tn < n_fast) issue(tn, (int)((j - 1) % kTpgSlots));
    }
    mbar_wait_parity_sleep(&full[k], (uint32_t)((j / kTpgSlots) & 1));
    unsigned char* sl = slots + k * T::slot_bytes;
    uint32_t w[B];
    if constexpr (B % 4 == 0) {
      const uint4* p = reinterpret_cast<const uint4*>(sl + lane * (B * 4));
#pragma unroll
      for (int i = 0; i < B / 4; ++i) {
        const uint4 v = p[i];
        w[4 * i] = v.x, w[4 * i + 1] = v.y, w[4 * i + 2] = v.z, w[4 * i + 3] = v.w;
      }
    } else if constexpr (B % 2 == 0) {
      const uint2* p = reinterpret_cast<const uint2*>(sl + lane * (B * 4));
#pragma unroll
      for (int i = 0; i < B / 2; ++i) {
        const uint2 v = p[i];
        w[2 * i] = v.x, w[2 * i + 1] = v.y;
      }
    } else {
      const uint32_t* p = reinterpret_cast<const uint32_t*>(sl) + lane * B;
#pragma unroll
      for (int i = 0; i < B; ++i) w[i] = p[i];
    }
    __syncwarp();  // every lane holds its input: the slot takes the output
    uint32_t o[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) o[i] = 0;
    uint32_t smask = 0;  // XC through L2: rows whose list runs past the read windows
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const uint32_t c = tpg_code<B>(w, r);
      code_max = umax32(code_max, c);
      const uint32_t cc = umin32(c, dict_last);
      bool su;
      const uint32_t v = translate(cc, su);
      if (XCG || (XCS && DM_TPG_PATCH)) smask |= (uint32_t)su << r;
      tpg_put<NB>(o, r, (XCS && !DM_TPG_PATCH && su) ? __ldg(XM + cc) : v);
    }
    if constexpr (NB % 4 == 0) {
      uint4* d = reinterpret_cast<uint4*>(sl + lane * (NB * 4));
#pragma unroll
      for (int i = 0; i < NB / 4; ++i) d[i] = make_uint4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
    } else if constexpr (NB % 2 == 0) {
      uint2* d = reinterpret_cast<uint2*>(sl + lane * (NB * 4));
#pragma unroll
      for (int i = 0; i < NB / 2; ++i) d[i] = make_uint2(o[2 * i], o[2 * i + 1]);
    } else {
      uint32_t* d = reinterpret_cast<uint32_t*>(sl) + lane * NB;
#pragma unroll
      for (int i = 0; i < NB; ++i) d[i] = o[i];
    }
    if ((XCG || (XCS && DM_TPG_PATCH)) && smask) {  // rare, per lane: exact values patched into the staged output
      uint32_t* ow = reinterpret_cast<uint32_t*>(sl) + lane * NB;
      const uint32_t* M32 = reinterpret_cast<const uint32_t*>(M);
      constexpr uint32_t cmask = B == 32 ? 0xffffffffu : (1u << B) - 1u;
      constexpr uint64_t vmask = NB == 32 ? 0xffffffffull : (1ull << NB) - 1ull;
      do {
        const uint32_t r = __ffs(smask) - 1;
        smask &= smask - 1;
        const uint64_t bi = ((t * 32 + lane) * 32 + r) * (uint64_t)B;  // the row's bit offset in M
        const uint64_t wi = bi >> 5;
        const uint32_t hi = wi + 1 < 2 * dwords(n_main, B) ? __ldg(M32 + wi + 1) : 0u;
        const uint32_t c = __funnelshift_r(__ldg(M32 + wi), hi, (uint32_t)(bi & 31)) & cmask;
        const uint64_t v = exact(umin32(c, dict_last));
        const uint32_t ob = r * NB, i = ob >> 5, sh = ob & 31;
        uint64_t x = ow[i] | (i + 1 < (uint32_t)NB ? (uint64_t)ow[i + 1] << 32 : 0ull);
        x = (x & ~(vmask << sh)) | (v << sh);
        ow[i] = (uint32_t)x;
        if (i + 1 < (uint32_t)NB) ow[i + 1] = (uint32_t)(x >> 32);
      } while (smask);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_1d(Ob + t * (uint64_t)(128 * NB), sl, 128u * NB, pol);
      tma_store_commit();
    }
  }
  tma_store_wait_all<0>();
  }

  // tiles holding delta rows or the ragged end: lane l still owns group l, its
  // input words read from global (bounded), every row checked at run time; the
  // 32 gathers of a lane (X_D through r, or the main lookups) are independent,
  // so a tile costs a few round trips, not 32
  if (n_fast < n_tiles) {
    const uint32_t* M32 = reinterpret_cast<const uint32_t*>(M);
    const uint64_t nw_in32 = 2 * dwords(n_main, B), nw32 = 2 * dwords(n_total, NB);
    uint32_t* out32 = reinterpret_cast<uint32_t*>(Mout);
    for (uint64_t t = n_fast + gw; t < n_tiles; t += GW) {
      const uint64_t g = t * 32 + lane, row0 = g * 32;
      uint32_t w[B];
#pragma unroll
      for (int i = 0; i < B; ++i) {
        const uint64_t wi = g * B + i;
        w[i] = wi < nw_in32 ? __ldg(M32 + wi) : 0u;
      }
      uint32_t o[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) o[i] = 0;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const uint64_t row = row0 + r;
        uint32_t v = 0;
        if (row < n_main) {
          const uint32_t c = tpg_code<B>(w, r);
          code_max = umax32(code_max, c);
          const uint32_t cc = umin32(c, dict_last);
          bool su;
          v = translate(cc, su);
          if (su) v = exact(cc);
        } else if (row < n_total) {
          v = __ldg(XD + (rank ? __ldg(rank + (row - n_main)) : (uint32_t)(row - n_main)));
        }
        tpg_put<NB>(o, r, v);
      }
#pragma unroll
      for (int i = 0; i < NB; ++i)
        if (g * NB + i < nw32) out32[g * NB + i] = o[i];
    }
  }
  const bool bad = n_main > 0 && code_max > dict_last;
  if (__any_sync(FULL, bad) && lane == 0) atomicMin(&hdr->status, (int)DM_E_CODE_RANGE);
}

// Naive Step 2 -- the paper's unoptimized algorithm ("UnOpt" of
// Fig 7/8): for every tuple take its value (U_M[M[i]] for a main row, D[k] for
// a delta row) and binary-search it in the merged dictionary U'.  No
// translation tables; log2|U'| dependent gathers per tuple.  Kept as the
// baseline for the optimized Step 2 (NEXT4, the paper's 9-10x claim).
// One warp per 32-row group (grid-stride), codes packed by warp shuffles.
template <class KT>
__global__ void __launch_bounds__(256) k_naive_step2(const uint64_t* __restrict__ M, uint64_t n_main, uint32_t b,
                                                     const void* __restrict__ UM, uint64_t dict_len,
                                                     const void* __restrict__ D, uint64_t n_delta,
                                                     const void* __restrict__ Up, uint64_t* __restrict__ Mout,
                                                     dm_header* hdr) {
  pdl_prologue();
  using K = typename KT::K;
  const uint32_t nb = hdr->merged_bits;
  const uint64_t nU = hdr->merged_dict_len, n_total = n_main + n_delta, ngroups = (n_total + 31) / 32;
  const unsigned lane = lane_id();
  const uint32_t pr0 = (32 * lane) / nb, pop = 32 * lane - pr0 * nb;
  const uint32_t umask = b == 32 ? 0xffffffffu : ((1u << b) - 1);
  const uint32_t* M32 = reinterpret_cast<const uint32_t*>(M);
  const uint64_t nw32_in = 2 * dwords(n_main, b), nw32 = 2 * dwords(n_total, nb);
  uint32_t* out32 = reinterpret_cast<uint32_t*>(Mout);
  bool bad = false;
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t g = warp0; g < ngroups; g += nwarps) {
    const uint64_t row = g * 32 + lane;
    K v{};
    if (row < n_main) {
      const uint64_t s0 = row * b, w = s0 >> 5;
      const uint32_t lo = M32[w], hi = w + 1 < nw32_in ? M32[w + 1] : 0u;
      uint32_t code = __funnelshift_r(lo, hi, (uint32_t)(s0 & 31)) & umask;
      if (code >= dict_len) {
        bad = true;
        code = 0;
      }
      v = KT::load(UM, code);
    } else if (row < n_total) {
      v = KT::load(D, row - n_main);
    }
    uint64_t lo = 0, hi = nU;  // lower_bound(U', v)
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (KT::lt(KT::load(Up, mid), v)) lo = mid + 1; else hi = mid;
    }
    const uint32_t c = row < n_total ? (uint32_t)lo : 0u;
    const uint32_t word = warp_pack<0>(c, nb, pr0, pop);
    const uint64_t ow = g * nb + lane;
    if (lane < nb && ow < nw32) out32[ow] = word;
  }
  if (__any_sync(FULL, bad) && lane == 0) atomicMin(&hdr->status, (int)DM_E_CODE_RANGE);
}

__global__ void __launch_bounds__(256) k_pack(const uint32_t* __restrict__ codes, uint64_t n, uint32_t bits,
                                              uint32_t* __restrict__ words32, uint64_t nw32) {
  pdl_prologue();
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
  pdl_prologue();
  const uint32_t mask = bits == 32 ? 0xffffffffu : ((1u << bits) - 1);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = i * bits;
    const uint64_t w = s >> 5;
    const uint32_t lo = words32[w], hi = (w + 1 < nw32) ? words32[w + 1] : 0u;
    codes[i] = __funnelshift_r(lo, hi, (uint32_t)(s & 31)) & mask;
  }
}

// Share of the SM slots a recompress launch may take: all of them for one
// column; a quarter inside dm_merge_table, where other columns' latency-bound
// Step 1 kernels then co-run (cfg4: 15.3 -> 14.6 ms; 50%: 14.8 ms).
// DM_REC_GRID_PCT (1..100) overrides both (experiments).
static thread_local bool t_table_merge = false;
static int rec_grid_percent() {
  static const int v = [] {
    const char* e = std::getenv("DM_REC_GRID_PCT");
    const int x = e ? std::atoi(e) : 0;
    return (x >= 1 && x <= 100) ? x : 0;
  }();
  return v ? v : t_table_merge ? 25 : 100;
}

// Experiments: DM_TPG_TABLE=1 lets dm_merge_table use the thread-per-group kernel too.
static bool tpg_in_tables() {
  static const bool v = [] {
    const char* e = std::getenv("DM_TPG_TABLE");
    return e && e[0] == '1';
  }();
  return v;
}

// Shared-memory bytes left for XC next to a kRecStagesXc-deep ring.
static uint32_t xc_smem_budget(uint32_t in_stage) {
  static int optin = [] {
    int d = 0, v = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
    return v;
  }();
  const int64_t b = (int64_t)optin - 1024 - kRecHdrBytes - (int64_t)kRecStagesXc * in_stage;
  return b > 0 ? (uint32_t)(b & ~15ll) : 0u;
}

// Thread-per-group Step 2(b): dynamic shared memory (the device maximum) and
// the XC budget that leaves room for kTpgMinWarps warps' slots.
static uint32_t tpg_smem() {
  static int optin = [] {
    int d = 0, v = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
    return v;
  }();
  return optin > 1024 ? (uint32_t)(optin - 1024) : 0u;
}
// XC budget that leaves room for kTpgMinWarps warps' slots (slots: 128 b' bytes for b' - b in {0, 1})
template <int NB>
uint32_t tpg_budget() {
  const int64_t b = (int64_t)tpg_smem() - kTpgHdrBytes - 128 -
                    (DM_TPG_DIRECT ? 0 : (int64_t)kTpgMinWarps * kTpgSlots * Tpg<NB, NB>::slot_bytes);
  return b > 0 ? (uint32_t)(b & ~15ll) : 0u;
}
// Which (b', mode) pairs use the thread-per-group kernel: XC in shared memory
// and the plain X_M through L2 (b, b' >= 15: |U_M| * 4 > 96 KB).  Measured and
// not used: XC through L2 (cfg5 Step 2(b): 39.2 vs 11.9 ms with the looping
// lookup inside the 32-row pass; 16.6 ms with the straight-line `xc_l2_fast`
// and the rare long lists patched afterwards -- DM_TPG_XCL2=1) and the plain
// X_M in shared memory (cfg1 0.031 vs 0.017 ms: a small column is
// latency-bound on the per-CTA staging and the few tiles).
// cfg3 (plain X_M through L2): 0.298 vs 0.318 ms.
#ifndef DM_TPG_XCL2
#define DM_TPG_XCL2 0  // experiments: XC through L2 (cfg5 Step 2(b) 16.6 vs 11.9 ms, not used)
#endif
template <int NB, int XMODE>
constexpr bool tpg_has() {
  return NB >= kTpgMinWidth && NB <= 32 &&
         (XMODE == XM_XC_SMEM || XMODE == XM_RAW_GLOBAL || (DM_TPG_XCL2 && XMODE == XM_XC_GLOBAL));
}
template <int B, int NB, int XMODE>
void launch_tpg(const dm_column_in* in, const dm_column_out* out, const uint32_t* xm, const uint32_t* xd,
                const uint32_t* rank, dm_header* hdr, cudaStream_t st, uint32_t fixed_bits, const uint2* xrec,
                const uint8_t* xoffs, uint32_t budget, uint32_t dens, uint32_t xs) {
  auto kern = k_recompress_tpg<B, NB, XMODE>;
  constexpr uint32_t slots = kTpgWarps * kTpgSlots * Tpg<B, NB>::slot_bytes;  // (unused by XC in smem, DM_TPG_DIRECT)
  const uint32_t smem = XMODE == XM_XC_SMEM ? tpg_smem()
                        : XMODE == XM_RAW_SMEM
                            ? (uint32_t)((kTpgHdrBytes + in->dict_len * 4 + 127) & ~127ull) + slots
                            : kTpgHdrBytes + slots;
  ensure_smem((const void*)kern);
  const uint64_t tiles = (in->n_main + in->n_delta + 1023) / 1024;
  const unsigned grid = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>(tiles, (uint64_t)device_sms() * rec_grid_percent() / 100));
  const TpgK kc{1u << 23, 1u << 18, 1u << 25, 1u << 30, 2u, 4u, 8u, 32u, 128u, 1024u, 0xfffffffeu, xs};
  launch_k(kern, grid, 32 * kTpgWarps, smem, st, in->main_codes, in->n_main, in->dict_len, xm, xd, rank, in->n_delta,
           out->merged_codes, hdr, fixed_bits, xrec, xoffs, budget, dens, kc, smem);
  note_launch();
}
// The thread-per-group kernel for b' = NB and the caller's b when one exists
// (knob 6 = 0, b' - b in {0, 1}); false: the caller launches the warp-per-group kernel.
template <int NB, int XMODE>
bool try_tpg(const dm_column_in* in, const dm_column_out* out, const uint32_t* xm, const uint32_t* xd,
             const uint32_t* rank, dm_header* hdr, cudaStream_t st, uint32_t fixed_bits, const uint2* xrec,
             const uint8_t* xoffs, uint32_t budget, uint32_t dens, uint32_t xs) {
  if constexpr (!tpg_has<NB, XMODE>()) {
    return false;
  } else {
    // not inside dm_merge_table: there the capped Step 2(b) grids co-run with other
    // columns' Step 1 kernels, and the warp-per-group kernel measured faster
    // (cfg4 13.99 vs 14.31 ms)
    if (tuning(6) != 0 || (t_table_merge && !tpg_in_tables())) return false;
    if (in->main_bits == (uint32_t)NB)
      launch_tpg<NB, NB, XMODE>(in, out, xm, xd, rank, hdr, st, fixed_bits, xrec, xoffs, budget, dens, xs);
    else if (in->main_bits + 1 == (uint32_t)NB)
      launch_tpg<NB - 1, NB, XMODE>(in, out, xm, xd, rank, hdr, st, fixed_bits, xrec, xoffs, budget, dens, xs);
    else
      return false;
    return true;
  }
}

template <int NB>
cudaError_t launch_nb(const dm_column_in* in, const dm_column_out* out, const uint32_t* xm, const uint32_t* xd,
                      const uint32_t* rank, dm_header* hdr, cudaStream_t st, uint32_t fixed_bits, const uint2* xrec,
                      const uint8_t* xoffs, uint32_t xs, bool xc_only) {
  const uint32_t in_stage = kRecGroups * in->main_bits * 4 + 16;
  const uint32_t in_stage_xc = rec_groups<XM_XC_SMEM>() * in->main_bits * 4 + 16;
  const int sms = device_sms();
  const uint64_t n_total = in->n_main + in->n_delta;
  uint32_t dens = 0;
  auto go = [&](auto kern, size_t smem, uint32_t budget, int threads = kRecThreads, int groups = kRecGroups) {
    const uint64_t nchunks = (n_total + 32ull * groups - 1) / (32ull * groups);
    const int occ = occupancy((const void*)kern, threads, smem);
    const unsigned grid = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>(nchunks, (uint64_t)sms * occ * rec_grid_percent() / 100));
    launch_k(kern, grid, threads, smem, st, in->main_codes, in->n_main, in->main_bits, in->dict_len, xm, xd, rank,
                                          in->n_delta, out->merged_codes, hdr,
                                          groups == kRecGroups ? in_stage : in_stage_xc, fixed_bits, xrec, xoffs,
                                          budget, dens, xs);
    note_launch();
  };
  const size_t ring = kRecHdrBytes + (size_t)kRecStages * in_stage;
  auto tpg = [&](auto mode, uint32_t budget) {
    if constexpr (NB <= 0)
      return false;
    else
      return try_tpg<NB, decltype(mode)::value>(in, out, xm, xd, rank, hdr, st, fixed_bits, xrec, xoffs, budget, dens,
                                                xs);
  };
  using RawSmem = std::integral_constant<int, XM_RAW_SMEM>;
  using RawGlobal = std::integral_constant<int, XM_RAW_GLOBAL>;
  using XcSmem = std::integral_constant<int, XM_XC_SMEM>;
  using XcGlobal = std::integral_constant<int, XM_XC_GLOBAL>;
  if (in->dict_len * 4 <= kRecSmemXBytes) {
    if (!tpg(RawSmem{}, 0)) go(k_recompress<NB, XM_RAW_SMEM>, ring + in->dict_len * 4, 0);
    return cudaGetLastError();
  }
  const int knob = tuning(0);
  if constexpr (NB < 0) {  // bounded runtime-width kernels exist for the plain-X_M modes only
    if (xrec && knob != 1)
      return launch_nb<0>(in, out, xm, xd, rank, hdr, st, fixed_bits, xrec, xoffs, xs, xc_only);
    go(k_recompress<NB, XM_RAW_GLOBAL>, ring, 0);
    return cudaGetLastError();
  } else {
  if (!xrec || knob == 1) {
    if (!tpg(RawGlobal{}, 0)) go(k_recompress<NB, XM_RAW_GLOBAL>, ring, 0);
    return cudaGetLastError();
  }
  // compact table available: the smem variant (if its records can fit at all)
  // plus an L2 companion; which one runs is decided on the device from |U'|
  const bool auto_smem = knob == 0 && xc_smem_candidate(in);
  const bool want_smem = (knob == 2 || auto_smem) && xs == 8;
  if (auto_smem) dens = 6;  // <= 4 entries per 256-code block on average
  if (knob == 0 && !auto_smem && !xc_only && in->dict_len * 4 <= kXcGlobalMinBytes) {
    if (!tpg(RawGlobal{}, 0)) go(k_recompress<NB, XM_RAW_GLOBAL>, ring, 0);
    return cudaGetLastError();
  }
  const uint32_t budget0 = want_smem ? xc_smem_budget(in_stage_xc) : 0u;
  uint32_t budget = (uint64_t)xc_nsb(in->dict_len, xs) * kXcRecBytes + 16 <= budget0 ? budget0 : 0u;
  const bool xc_l2 = xc_only || knob == 2 || knob == 3 || in->dict_len * 4 > kXcGlobalMinBytes;
  bool tpg_smem_run = false;
  if constexpr (NB >= kTpgMinWidth) {  // thread-per-group form for b' - b in {0, 1} (knob 6); its rare
    // lookups read the plain X_M, which is whole when the companion is the plain-X_M kernel
    if (want_smem && !xc_l2 && tpg_has<NB, XM_XC_SMEM>() && tuning(6) == 0 && (!t_table_merge || tpg_in_tables()) &&
        (in->main_bits == (uint32_t)NB || in->main_bits + 1 == (uint32_t)NB)) {
      const uint32_t bt = tpg_budget<NB>();
      if ((uint64_t)xc_nsb(in->dict_len, xs) * kXcRecBytes + 16 <= bt) {
        budget = bt;
        tpg_smem_run = tpg(XcSmem{}, budget);
      }
    }
  }
  if (budget && !tpg_smem_run)
    go(k_recompress<NB, XM_XC_SMEM>, kRecHdrBytes + (size_t)kRecStagesXc * in_stage_xc + budget, budget,
       rec_threads<XM_XC_SMEM>(), rec_groups<XM_XC_SMEM>());
  // (A persisting L2 access-policy window over XC was measured: no gain on
  // cfg5's Step 2(b), and the set-aside slowed Steps 1(a)/1(b) by 40%.)
  if (xc_l2) {
    if (!tpg(XcGlobal{}, budget)) go(k_recompress<NB, XM_XC_GLOBAL>, ring, budget);
  } else {
    if (!tpg(RawGlobal{}, budget)) go(k_recompress<NB, XM_RAW_GLOBAL>, ring, budget);
  }
  return cudaGetLastError();
  }
}

using XcKernel = void (*)(const uint64_t*, uint64_t, uint32_t, uint64_t, const uint32_t*, const uint32_t*,
                         const uint32_t*, uint64_t, uint64_t*, dm_header*, uint32_t, uint32_t, const uint2*,
                         const uint8_t*, uint32_t, uint32_t, uint32_t);
template <int... I>
constexpr auto make_xc_table(std::integer_sequence<int, I...>) {
  return std::array<XcKernel, sizeof...(I)>{&k_recompress<I, XM_XC_GLOBAL>...};
}

using LaunchFn = cudaError_t (*)(const dm_column_in*, const dm_column_out*, const uint32_t*, const uint32_t*,
                                 const uint32_t*, dm_header*, cudaStream_t, uint32_t, const uint2*, const uint8_t*, uint32_t,
                                 bool);
template <int... I>
constexpr auto make_table(std::integer_sequence<int, I...>) {
  return std::array<LaunchFn, sizeof...(I)>{&launch_nb<I>...};
}

}  // namespace

void set_table_merge(bool on) { t_table_merge = on; }

cudaError_t launch_recompress(const dm_column_in* in, const dm_column_out* out, const uint32_t* xm,
                              const uint32_t* xd, const uint32_t* rank, dm_header* hdr, cudaStream_t st,
                              uint32_t fixed_bits, const uint2* xc_rec, const uint8_t* xc_offs, uint32_t xc_shift,
                              bool xc_only) {
  if (in->n_main + in->n_delta == 0) return cudaSuccess;
  static const auto table = make_table(std::make_integer_sequence<int, 33>{});  // [0] = runtime width
  // fixed b' (dm_recompress, the host path's row chunks): XC when the caller has
  // one (its shared-memory variant reads n_new from the merge's header)
  if (fixed_bits)
    return table[fixed_bits](in, out, xm, xd, rank, hdr, st, fixed_bits, xc_rec, xc_offs, xc_shift, xc_only);
  const uint64_t lo_len = std::max<uint64_t>(in->dict_len, in->n_delta ? 1 : 0);
  const uint32_t nb_lo = host_width(lo_len), nb_hi = host_width(in->dict_len + in->n_delta);
  if (nb_hi > 32) return cudaErrorInvalidValue;  // caller checks DM_E_TOO_WIDE first
  // b' is only known on the device: launch every width-specialised kernel |U'|'s
  // bounds allow (the others exit at once, ~2 us each) while that is cheaper
  // than the runtime-width kernel (its shuffle-pack loop and spills)
  if (nb_hi - nb_lo <= 3) {
    for (uint32_t nb = nb_lo; nb <= nb_hi; ++nb) {
      cudaError_t e = table[nb](in, out, xm, xd, rank, hdr, st, 0, xc_rec, xc_offs, xc_shift, xc_only);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  // wider ranges: a runtime-width kernel whose pack loop is bounded by the
  // narrowest candidate (codes per output word = 2 + 30 / b', non-increasing in
  // b'), so small-dictionary columns with large deltas keep a short, unspilled loop
  static const LaunchFn classes[] = {&launch_nb<-2>, &launch_nb<-3>, &launch_nb<-4>, &launch_nb<-5>,
                                     &launch_nb<-6>, &launch_nb<-7>, &launch_nb<-8>, &launch_nb<-9>,
                                     &launch_nb<-12>, &launch_nb<-17>};
  static const int bound[] = {2, 3, 4, 5, 6, 7, 8, 9, 12, 17};
  const int tm = (int)((2 * nb_lo + 30) / nb_lo);
  for (int c = 0; c < 10; ++c)
    if (tm <= bound[c]) return classes[c](in, out, xm, xd, rank, hdr, st, 0, xc_rec, xc_offs, xc_shift, xc_only);
  return table[0](in, out, xm, xd, rank, hdr, st, 0, xc_rec, xc_offs, xc_shift, xc_only);
}

cudaError_t launch_recompress_xc(const dm_column_in* in, const dm_column_out* out, const uint32_t* xm,
                                 const uint32_t* xd, const uint32_t* rank, dm_header* hdr, cudaStream_t st,
                                 uint32_t bits, const uint2* xc_rec, const uint8_t* xc_offs, uint32_t xs) {
  if (in->n_main + in->n_delta == 0) return cudaSuccess;
  const uint32_t in_stage = kRecGroups * in->main_bits * 4 + 16;
  const size_t smem = kRecHdrBytes + (size_t)kRecStages * in_stage;
  const uint64_t n_total = in->n_main + in->n_delta;
  const uint64_t nchunks = (n_total + 32ull * kRecGroups - 1) / (32ull * kRecGroups);
  static const auto xc_table = make_xc_table(std::make_integer_sequence<int, 33>{});
  auto kern = xc_table[bits <= 32 ? bits : 0];  // width-specialised (same instantiations as launch_nb)
  const int occ = occupancy((const void*)kern, kRecThreads, smem);
  const unsigned grid = (unsigned)std::min<uint64_t>(nchunks, (uint64_t)device_sms() * occ);
  launch_k(kern, grid, kRecThreads, smem, st, in->main_codes, in->n_main, in->main_bits, in->dict_len, xm, xd, rank,
                                        in->n_delta, out->merged_codes, hdr, in_stage, bits, xc_rec, xc_offs, 0u, 0,
                                        xs);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_naive_step2(const dm_column_in* in, const dm_column_out* out, dm_header* hdr, cudaStream_t st) {
  const uint64_t n_total = in->n_main + in->n_delta;
  if (n_total == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<uint64_t>((n_total + 255) / 256, (uint64_t)device_sms() * 16);
  switch (in->key) {
    case DM_KEY_U64:
      launch_k(k_naive_step2<KeyU64>, grid, 256, 0, st, in->main_codes, in->n_main, in->main_bits, in->main_dict,
                                                  in->dict_len, in->delta, in->n_delta, out->merged_dict,
                                                  out->merged_codes, hdr);
      break;
    case DM_KEY_U32:
      launch_k(k_naive_step2<KeyU32>, grid, 256, 0, st, in->main_codes, in->n_main, in->main_bits, in->main_dict,
                                                  in->dict_len, in->delta, in->n_delta, out->merged_dict,
                                                  out->merged_codes, hdr);
      break;
    default:
      launch_k(k_naive_step2<KeyB16>, grid, 256, 0, st, in->main_codes, in->n_main, in->main_bits, in->main_dict,
                                                  in->dict_len, in->delta, in->n_delta, out->merged_dict,
                                                  out->merged_codes, hdr);
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pack(const uint32_t* codes, uint64_t n, uint32_t bits, uint64_t* words, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const uint64_t groups = (n + 31) / 32;
  const unsigned grid = (unsigned)std::min<uint64_t>((groups + 7) / 8, 148 * 16);
  launch_k(k_pack, grid, 256, 0, st, codes, n, bits, reinterpret_cast<uint32_t*>(words), 2 * host_words(n, bits));
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_unpack(const uint64_t* words, uint64_t n, uint32_t bits, uint32_t* codes, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  launch_k(k_unpack, grid, 256, 0, st, reinterpret_cast<const uint32_t*>(words), 2 * host_words(n, bits), n, bits, codes);
  note_launch();
  return cudaGetLastError();
}

}  // namespace dm
