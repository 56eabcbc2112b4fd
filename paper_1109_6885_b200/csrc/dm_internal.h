// dm_internal.h -- host/device shared internals of libdictmerge (not part of the ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/dictmerge.h"

namespace dm {

// ---- tiling constants
// Onesweep tile shapes (threads x keys per thread); variant chosen by sort_variant().
struct SortShape {
  int threads, items_u64, items_b16;
};
constexpr SortShape kSortShapes[4] = {{512, 16, 8}, {256, 16, 8}, {256, 8, 4}, {1024, 8, 4}};
int sort_variant();  // DM_SORT_CFG environment override (experiments), default 0
uint64_t sort_tile_keys(int key);
#ifndef DM_UNIQ_THREADS
#define DM_UNIQ_THREADS 512
#endif
constexpr int kUniqThreads = DM_UNIQ_THREADS;
constexpr int kUniqItems = 8;                            // 4096 per tile
constexpr int kMergeThreads = 256;
constexpr int kMergeItems = 8;                           // 2048 merged-diagonal elements per tile
constexpr int kMergeTile = kMergeThreads * kMergeItems;
constexpr int kRecConsumerWarps = 16;                    // recompress: consumer warps per CTA
constexpr int kRecThreads = 32 * (kRecConsumerWarps + 1);  // + one TMA producer warp
constexpr int kRecGroups = 128;                          // 32-row groups per chunk (4096 rows)
constexpr int kRecStages = 4;                            // TMA input ring depth
constexpr uint32_t kRecSmemXBytes = 96 * 1024;           // X_M staged in shared memory up to this size
constexpr int kRecHdrBytes = 256;                        // recompress smem head: mbarriers + XC mask table
constexpr int kRecStagesXc = 4;                          // ring depth when the compact X_M takes the smem

// Compact translation table "XC": X_M[c] = c + #{new values
// inserted at or before main position c} (insertion point p of a new value =
// #U_M below it; it raises X_M[c] for c >= p).  Blocks of 2^xs codes (xs = 7 or
// 8, chosen per column from N_D / |U_M| so a block holds a few entries), four
// blocks per superblock s, one 8-byte record per superblock: word 0 = R =
// #{p <= 4s 2^xs} (bit 31: flag), word 1 = four bytes cum[t] = #{p in the
// superblock's first t+1 blocks, (4s 2^xs, ...]}; per new value (sorted order)
// one byte, (p - 1) mod 2^xs.  A superblock whose counts do not fit (> 255, or
// > kXcMaxBlock in one block) is flagged and its lookups read the plain X_M.
constexpr uint32_t kXcMaxBlock = 32;
constexpr uint32_t kXcRecBytes = 8;
constexpr uint32_t kXcMinShift = 7;
constexpr uint64_t kXcGlobalMinBytes = 64ull << 20;     // plain X_M above this: use XC from L2
inline uint64_t xc_nblk(uint64_t dict_len, uint32_t xs) { return (dict_len + (1ull << xs) - 1) >> xs; }
inline uint64_t xc_nsb(uint64_t dict_len, uint32_t xs) { return (dict_len + (4ull << xs) - 1) >> (xs + 2); }
enum XMode { XM_RAW_GLOBAL = 0, XM_RAW_SMEM = 1, XM_XC_SMEM = 2, XM_XC_GLOBAL = 3 };
// Tuning knobs (dm_set_tuning): index 0 = X_M placement (0 auto, 1 plain only,
// 2 compact (smem if it fits, else L2), 3 compact from L2); index 1 = Step 1(b)
// variant (0 lean two-pass, 1 first three-phase form, 2 lean single pass);
// index 2 = Step 1(a) dedup front end (0 auto, 1 off, 2 on); index 3 = Step 2
// variant (0 optimized, 1 naive binary search, the paper's UnOpt baseline).
int tuning(int knob);
// Whether a merge builds XC at all: only when the plain X_M is too big for smem.
inline bool xc_enabled(uint64_t dict_len) { return dict_len * 4 > kRecSmemXBytes; }
// Auto mode, plain X_M between kRecSmemXBytes and kXcGlobalMinBytes: build XC
// with 256-code blocks when its records leave room in shared memory for the
// lists; Step 2(b) then decodes it from shared memory if the lists turn out
// short (decided on the device from |U'|), else gathers the plain X_M from L2.
constexpr uint64_t kXcSmemRecMax = 112 * 1024;
inline bool xc_smem_candidate(const dm_column_in* in) {
  return tuning(0) == 0 && in->dict_len * 4 > kRecSmemXBytes && in->dict_len * 4 <= kXcGlobalMinBytes &&
         xc_nsb(in->dict_len, 8) * kXcRecBytes <= kXcSmemRecMax;
}
// Whether this merge builds XC: auto when the plain X_M exceeds kXcGlobalMinBytes
// or XC may fit in shared memory.
inline bool xc_wanted(const dm_column_in* in) {
  const int k = tuning(0);
  return k == 1 ? false : k == 0 ? in->dict_len * 4 > kXcGlobalMinBytes || xc_smem_candidate(in)
                                 : xc_enabled(in->dict_len);
}
// Step 1(a) dedup front end (NEXT1): knob 2 = 0 auto (16-byte keys with
// N_D >= 2^16: 16 radix passes make repeats expensive), 1 off, 2 on.
// Step 1(a) sort (knob 5): 0 auto = the bucket path (below) for 2^11 <= N_D <=
// 2^23, else the LSD passes; 1 LSD only; 2 bucket path for any N_D >= 1.
constexpr uint64_t kBkMinN = 1ull << 11, kBkMaxN = 1ull << 23;
constexpr uint32_t kBkMaxBucket = 256;  // a larger bucket sends the merge to the LSD passes
constexpr int kBkScanItems = 16;        // counts per thread in k_bk_scan (tile = 4096 buckets)
inline bool bucket_wanted(const dm_column_in* in) {
  const int k = tuning(5);
  if (in->n_delta == 0 || k == 1) return false;
  return k == 2 || (in->n_delta >= kBkMinN && in->n_delta <= kBkMaxN);
}
// log2 of the bucket count: about four keys per bucket
inline uint32_t bucket_bits(uint64_t n) {
  uint32_t b = 0;
  while ((1ull << b) < n) ++b;
  return b < 14 ? 12u : b > 26 ? 24u : b - 2;  // >= one k_bk_scan tile
}
inline bool dedup_wanted(const dm_column_in* in) {
  const int k = tuning(2);
  if (in->n_delta == 0 || k == 1 || k == 3) return false;
  // 16-byte keys with many tuples (16 radix passes), or -- for the bucket path,
  // whose buckets must stay small -- a delta that must repeat values heavily
  // (at most |U_M| of its distinct values can be old ones)
  return k == 2 || (in->key == DM_KEY_B16 && in->n_delta >= (1u << 16)) ||
         (bucket_wanted(in) && in->dict_len * 4 < in->n_delta);
}
// Probe-first Step 1(a) (knob 2 = 3; auto for 16-byte keys with
// N_D >= 2^16 and U_M <= 64 MB): every delta value is first looked up in U_M
// (a hash table of U_M's positions, read-only while probed); only the values
// not found are sorted into U_new, and U' = merge(U_M, U_new).  Runs only when
// the caller asked for none of U_D / X_D / r (their index space is U_D's).
constexpr uint32_t kPfNew = 0x80000000u;
inline bool probe_possible(const dm_column_in* in) {
  const int k = tuning(2);
  if (in->n_delta == 0 || in->dict_len == 0 || k == 1 || k == 2) return false;
  return k == 3 || (in->key == DM_KEY_B16 && in->n_delta >= (1u << 16) && in->dict_len * 16 <= (64ull << 20));
}

// Block shift: 256-code blocks when N_D / |U_M| promises <= 6 entries per block
// (and always for the shared-memory variant, knob 2), else 128-code blocks.
int xc_shift_override();  // knob 4 / DM_XC_SHIFT: 7 or 8, 0 = none (a thread override first)
void set_xc_shift_override(int xs);  // this thread only; 0 clears (the library's sharded Step 1(b))
inline uint32_t xc_shift(const dm_column_in* in) {
  if (const int o = xc_shift_override()) return (uint32_t)o;
  if (tuning(0) == 2 || xc_smem_candidate(in)) return 8;
  return in->n_delta * 256 <= 6 * in->dict_len ? 8u : 7u;
}

// Step 1(b) sparse-delta tiles (knob 1 = 3, auto when N_D <= |U_M| / 8): U_M
// tiles of 2048 with the U_D values falling into them (k_sp_merge).  Needs
// |U_M| > 0; ws status_merge / part hold >= |U_M| / 2048 + 1 entries.
inline bool sp_wanted(const dm_column_in* in) {
  const int k = tuning(1);
  if (in->dict_len == 0) return false;
  return k == 3 || (k == 0 && in->n_delta * 8 <= in->dict_len);
}

constexpr uint32_t kRadixFlagAgg = 1u << 30;
constexpr uint32_t kRadixFlagPre = 2u << 30;
constexpr uint32_t kRadixValMask = (1u << 30) - 1;

// Device-computed radix plan (pass skipping: a pass whose digit is constant
// over all keys is skipped; src/dst select the ping-pong buffers).
enum { SEL_INPUT = 0, SEL_BUF0 = 1, SEL_BUF1 = 2 };
struct SortPlan {
  int32_t active[16];
  int32_t src[16];
  int32_t dst[16];
  int32_t final_sel;
  int32_t n_active;
  int32_t pad[2];
  uint32_t digit_base[16][256];
};
// Bucket path state (zeroed per call): OR of (key ^ key[0]) over all keys, the
// grid-done counter, the overflow flag (a bucket > kBkMaxBucket keys: the LSD passes
// run instead) and the digit shift.
struct BucketState {
  unsigned long long diff_hi, diff_lo;
  uint32_t done, overflow, shift, pad;
};

// Workspace layout (byte offsets).  [0, zero_bytes) is memset to 0 per call.
struct WsLayout {
  size_t hdr;            // dm_header used by the synchronous entry points
  size_t counters;       // u32[64]: tile counters (16 sort passes, unique, merge, ...)
  size_t hist;           // u32[16][256] global digit histograms
  size_t status_sort;    // u32[npass][ntiles_sort][256]
  size_t status_unique;  // u64[ntiles_unique]
  size_t status_merge;   // u64[ntiles_merge]
  size_t zero_bytes;
  size_t plan;           // SortPlan
  size_t keys0, keys1;   // numeric keys, n_delta each
  size_t vals0, vals1;   // u32, n_delta each
  size_t udict;          // U_D raw keys, n_delta
  size_t rank;           // r: u32 n_delta
  size_t part;           // u64[ntiles_merge + 1] merge-path co-ranks
  size_t mcount;         // u32[ntiles_merge] duplicates dropped per merge tile
  size_t mexcl;          // u64[ntiles_merge] exclusive prefix of mcount
  size_t xm;             // X_M u32[dict_len]
  size_t xd;             // X_D u32[n_delta]
  size_t xc_rblk;        // XC: u32[nblk + 1], new values inserted before each 256-block
  size_t xc_rec;         // XC: uint2[nsb] superblock records
  size_t xc_offs;        // XC: u8[n_delta] insertion position mod 256 per new value
  size_t pf_used;        // probe-first (NEXT1): bitmap over U_M positions hit by the delta (zeroed region)
  size_t pf_src;         // probe-first: u32[n_delta] per tuple: U_M position, or kPfNew | compacted index
  size_t pf_keys;        // probe-first: the delta values not found in U_M (raw layout), n_delta capacity
  size_t pf_rank;        // probe-first: u32[n_delta] rank of each compacted value among the new values
  size_t pf_codes;       // probe-first: u32[n_delta] the delta tuples' final codes (Step 2(b) input)
  size_t pf_table;       // probe-first: u32[pf_cap] (hash tag | U_M position) by value hash (0xff.. = empty)
  uint64_t pf_cap;       // probe-first: table slots (power of two >= 4 |U_M|)
  bool probe;            // probe-first buffers laid out (probe_possible)
  size_t dd_slots;       // dedup (NEXT1): u64[dd_cap] (tag | id << 32) slots (memset per call)
  size_t dd_keys;        // dedup: distinct values, raw layout, n_delta capacity
  size_t dd_tid;         // dedup: u32[n_delta] distinct id per tuple
  size_t dd_rank;        // dedup: u32[n_delta] rank of each distinct id
  uint64_t dd_cap;       // dedup: table slots (power of two >= 2 n_delta), 0 = no dedup
  bool dedup;
  bool bucket;           // Step 1(a) bucket path
  uint32_t bk_bits;      // log2 bucket count
  size_t bk_state;       // BucketState (zeroed region)
  size_t bk_status;      // u64[scan tiles + 1] look-back (zeroed region)
  size_t bk_off;         // u32[B + 1]: counts, then exclusive offsets
  size_t bk_pairs;       // 4/8-byte keys: 16-byte (key, index) records, n_delta
  size_t bk_cur;         // u32[B]: scatter cursors
  size_t total;
  uint64_t ntiles_sort, ntiles_unique, ntiles_merge;
  int npass;
};

enum { CNT_SORT = 0, CNT_UNIQUE = 16, CNT_MERGE = 17, CNT_HIST = 18, CNT_DEDUP = 20 /* u64, 2 slots */, CNT_BKSCAN = 22,
       CNT_PROBE = 24 /* u64, 2 slots */ };

WsLayout ws_layout(const dm_column_in* in);
inline size_t key_bytes(int key) { return key == DM_KEY_U64 ? 8 : key == DM_KEY_U32 ? 4 : 16; }
uint32_t host_width(uint64_t n);
uint64_t host_words(uint64_t n, uint32_t bits);

// ---- launches: cudaLaunchKernelEx with programmatic dependent launch (PDL,
// see pdl_prologue in dm_device.cuh); DM_PDL=0 turns the attribute off.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  static_assert(sizeof...(KArgs) == sizeof...(Args), "kernel argument count");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- launch bookkeeping (host; cached so a merge issues no per-launch driver queries)
void note_launch(int n = 1);
// Raise the dynamic shared memory limit of `func` to the device maximum, once per device.
void ensure_smem(const void* func, bool max_carveout = false);
int device_sms();
int occupancy(const void* func, int threads, size_t smem);
cudaError_t last_error_check();

// ---- kernel launchers (each .cu file)
// Step 1(a): sort + unique of D -> U_D (udict), r (rank), hdr->delta_dict_len.
// probe: the probe-first front end (L.probe, no U_D / X_D / r requested): U_new
// into udict, the new values' ranks into L.pf_rank, hdr->delta_dict_len = |U_new|
// until launch_probe_codes adds the distinct found values.
cudaError_t launch_delta_dictionary(const dm_column_in* in, char* ws, const WsLayout& L, void* udict, uint32_t* rank,
                                    dm_header* hdr, cudaStream_t st, bool probe = false);
// Probe-first, after Step 1(b): codes[k] = X_M[p] (found) or X_D[rank_new] (new);
// hdr->delta_dict_len += #distinct found values (|U_D| = |U_new| + that).
cudaError_t launch_probe_codes(const dm_column_in* in, char* ws, const WsLayout& L, const uint32_t* xm,
                               const uint32_t* xd, dm_header* hdr, cudaStream_t st);
// Step 1(b) + 2(a): merge-path merge -> U', X_M, X_D, hdr->merged_dict_len / merged_bits.
// When xc_enabled(dict_len), also builds the compact table XC in the workspace.
// force_xc: build XC whenever xc_enabled (the row-sharded root exports it).
// need_xm: materialise X_M even where Step 2(b) would not read it (probe-first).
cudaError_t launch_dictionary_merge(const dm_column_in* in, const dm_column_out* out, char* ws, const WsLayout& L,
                                    const void* udict, uint32_t* xm, uint32_t* xd, dm_header* hdr, cudaStream_t st,
                                    bool force_xc = false, bool need_xm = false);
// Step 2(b): recompress main through X_M and append delta through X_D.
// fixed_bits != 0: b' given by the caller (dm_recompress); else read from hdr->merged_bits.
// xc_rec / xc_offs: the compact table (NULL: plain X_M only).
// rank NULL: delta row k takes xd[k] (the codes themselves).  xc_only: the caller
// holds XC but not the plain X_M (beyond flagged superblocks): never pick a
// plain-X_M kernel (requires |U_M| * 4 > kRecSmemXBytes).
cudaError_t launch_recompress(const dm_column_in* in, const dm_column_out* out, const uint32_t* xm,
                              const uint32_t* xd, const uint32_t* rank, dm_header* hdr, cudaStream_t st,
                              uint32_t fixed_bits = 0, const uint2* xc_rec = nullptr,
                              const uint8_t* xc_offs = nullptr, uint32_t xc_shift = 8, bool xc_only = false);
// dm_merge_table marks its launches (this thread) so Step 2(b) leaves SMs to
// the other columns' kernels.
void set_table_merge(bool on);
// Step 2(b) of a row shard through XC read from L2 (dm_recompress_xc).
cudaError_t launch_recompress_xc(const dm_column_in* in, const dm_column_out* out, const uint32_t* xm,
                                 const uint32_t* xd, const uint32_t* rank, dm_header* hdr, cudaStream_t st,
                                 uint32_t bits, const uint2* xc_rec, const uint8_t* xc_offs, uint32_t xc_shift);
// XC exception list: the X_M slices of flagged superblocks (gather on the root,
// scatter on the receiving ranks).
cudaError_t launch_xc_exceptions(bool gather, const uint2* rec, uint64_t nsb, uint32_t xs, uint64_t dict_len,
                                 uint32_t* xm, uint32_t* ids, uint32_t* slices, unsigned long long* d_count,
                                 uint64_t count, cudaStream_t st);
// Sharded Step 1(b) helpers (shard.cu, NEXT2).
cudaError_t launch_lower_bound(int key, const void* sorted, uint64_t n, const void* values, uint64_t nv,
                               uint64_t* pos, cudaStream_t st);
cudaError_t launch_add_u32(uint32_t* x, uint64_t n, uint32_t add, cudaStream_t st);
cudaError_t launch_xc_rebase(void* rec, uint64_t n, uint32_t add, cudaStream_t st);
cudaError_t launch_set_delta_len(dm_header* hdr, uint64_t n, cudaStream_t st);
// Naive Step 2: binary-search every tuple's value in U' (baseline).
cudaError_t launch_naive_step2(const dm_column_in* in, const dm_column_out* out, dm_header* hdr, cudaStream_t st);
cudaError_t launch_pack(const uint32_t* codes, uint64_t n, uint32_t bits, uint64_t* words, cudaStream_t st);
cudaError_t launch_unpack(const uint64_t* words, uint64_t n, uint32_t bits, uint32_t* codes, cudaStream_t st);

}  // namespace dm
