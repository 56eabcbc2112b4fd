/*
 * dictmerge.h -- C ABI of libdictmerge, a B200-native (sm_100a) implementation
 * of the online merge for dictionary-encoded column stores of Krueger et al.,
 * "Fast Updates on Read-Optimized Databases Using Multi-Core CPUs"
 * (arXiv 1109.6885, PVLDB 5(1)).  "P:n" = line n of the paper text.
 *
 * What one merge computes (Sec 5).  Per column, inputs are the main
 * partition -- a sorted dictionary U_M and the bit-packed code
 * vector M whose codes are positions in U_M -- and the delta partition D, raw
 * values in insertion order.  Outputs are the merged dictionary
 * U' = sorted distinct (U_M u D) (Eq 3) and the merged code vector M' of
 * N' = N_M + N_D rows (Eq 2): main rows first, then delta rows in
 * insertion order, each the position of its value in U', packed at
 * the new width b' = ceil(log2 |U'|) (Eq 4).  The path is the paper's
 * optimized merge:
 *   Step 1(a)  sorted distinct delta values U_D and per-tuple ranks
 *   Step 1(b)  merge U_M with U_D, dropping duplicates, emitting the
 *              translation tables X_M (old main code -> new code) and X_D
 *              (delta-dictionary rank -> new code)
 *   Step 2(a)  b' = ceil(log2 |U'|)                            (Eq 4)
 *   Step 2(b)  M'[i] = X_M[M[i]] for main rows (Eq 11), and the delta
 *              rows appended through X_D.
 *
 * Conventions (DESIGN.md "Readings" A1-A5):
 *   - width(n) = max(1, ceil(log2 n)); width(0) = width(1) = 1.
 *   - codes are 0-based dictionary positions.
 *   - a packed code vector of n codes at b bits (1 <= b <= 32) is an LSB-first
 *     bitstream held in little-endian u64 words: code i occupies stream bits
 *     [i*b, (i+1)*b), stream bit s is bit s%64 of word s/64.  Exactly
 *     dm_words(n, b) words are significant and their pad bits are zero.
 *   - DM_KEY_U64 (DM_KEY_U32) keys are little-endian u64 (u32) compared as
 *     unsigned integers.
 *     DM_KEY_B16 keys are 16 raw bytes compared bytewise (memcmp) over all 16
 *     bytes; zero padding takes part in the order.
 *
 * Memory and ownership.  Every pointer in dm_column_in / dm_column_out is a
 * DEVICE pointer (current CUDA device) unless the function says "host".  The
 * caller allocates every buffer (PyTorch in the Python binding) and owns it;
 * the library never frees caller memory and never writes its inputs.  All
 * device buffers must be 16-byte aligned.  One workspace (dm_workspace_bytes)
 * per concurrent call.  Calls are stream-ordered on the given cudaStream_t
 * (NULL = legacy default stream).
 *
 * Errors.  Host-detectable argument errors return before any launch.
 * Data-dependent errors (a main code >= |U_M|, an unsorted main dictionary,
 * |U'| > 2^32) are detected on the device, recorded in dm_header.status and
 * returned by the synchronous entry points; outputs are then unspecified but
 * the inputs are untouched (outputs always go to separate buffers, so a
 * failed merge leaves the table as it was).
 */
#ifndef DICTMERGE_H
#define DICTMERGE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DM_OK = 0,
  DM_E_INVALID = -1,     /* bad argument: NULL, misaligned, width out of range, ... */
  DM_E_CAPACITY = -2,    /* an output or workspace capacity is too small          */
  DM_E_TOO_WIDE = -3,    /* |U'| > 2^32: b' would exceed 32 bits                   */
  DM_E_UNSORTED = -4,    /* main dictionary not strictly increasing               */
  DM_E_CODE_RANGE = -5,  /* some main code >= |U_M|                               */
  DM_E_CUDA = -6,        /* a CUDA runtime call failed (dm_last_cuda_error)       */
  DM_E_NCCL = -7         /* reserved for the sharded variant                      */
} dm_status;

/* Value types: 8-byte unsigned integers, 16-byte memcmp-ordered strings, and
 * 4-byte unsigned integers (the paper's E = 4 of Fig 8). */
typedef enum { DM_KEY_U64 = 0, DM_KEY_B16 = 1, DM_KEY_U32 = 2 } dm_key;

/* One column's merge inputs.  All device pointers, read-only. */
typedef struct {
  int32_t key;                  /* dm_key                                            */
  const void* main_dict;        /* U_M: dict_len keys, strictly increasing           */
  uint64_t dict_len;            /* |U_M|  (< 2^32)                                   */
  const uint64_t* main_codes;   /* M: dm_words(n_main, main_bits) words              */
  uint64_t n_main;              /* N_M                                               */
  uint32_t main_bits;           /* b: width(dict_len) <= b <= 32 (reading A15)       */
  const void* delta;            /* D: n_delta keys, insertion order                  */
  uint64_t n_delta;             /* N_D  (< 2^30)                                     */
} dm_column_in;

/* One column's merge outputs: caller-allocated device buffers. */
typedef struct {
  void* merged_dict;               /* U': capacity merged_dict_cap keys               */
  uint64_t merged_dict_cap;        /* >= dict_len + n_delta                           */
  uint64_t* merged_codes;          /* M': capacity merged_codes_cap_words u64 words   */
  uint64_t merged_codes_cap_words; /* >= dm_merged_codes_cap_words(in)                */
  uint32_t* x_main;                /* optional (NULL = workspace): X_M, dict_len u32  */
  uint32_t* x_delta;               /* optional: X_D, capacity n_delta u32 (|U_D| used) */
  void* delta_dict;                /* optional: U_D, capacity n_delta keys            */
  uint32_t* delta_rank;            /* optional: r[k] = rank of D[k] in U_D, n_delta   */
  /* results, written (host side) by the synchronous entry points */
  uint64_t merged_dict_len;        /* |U'|                                            */
  uint64_t delta_dict_len;         /* |U_D|                                           */
  uint32_t merged_bits;            /* b'                                              */
} dm_column_out;

/* Result header, written on the device by dm_merge_column_async. */
typedef struct {
  uint64_t merged_dict_len;  /* |U'|                       */
  uint64_t delta_dict_len;   /* |U_D|                      */
  uint32_t merged_bits;      /* b'                         */
  int32_t status;            /* 0 or a negative dm_status  */
} dm_header;

/* width(n) = max(1, ceil(log2 n)) (Eq 4; reading A1).  Host, pure. */
uint32_t dm_width(uint64_t n);
/* ceil(n*bits/64): significant u64 words of a packed vector.  Host, pure. */
uint64_t dm_words(uint64_t n, uint32_t bits);
/* dm_words(n_main + n_delta, width(dict_len + n_delta)): an M' capacity that
 * fits every possible merge result of `in`.  Host, pure. */
uint64_t dm_merged_codes_cap_words(const dm_column_in* in);
/* Workspace bytes needed by dm_merge_column[_async] for `in`.  Host, pure. */
size_t dm_workspace_bytes(const dm_column_in* in);

/* Merge one column, stream-ordered, without any host synchronisation
 * (capturable in a CUDA graph).  Results land in *d_header (device memory,
 * 16-byte aligned) when the stream reaches that point.  Returns DM_OK or a
 * host-detectable error; data-dependent errors appear in d_header->status. */
dm_status dm_merge_column_async(const dm_column_in* in, const dm_column_out* out, void* ws, size_t ws_bytes,
                                dm_header* d_header, void* cuda_stream);

/* As dm_merge_column_async, and additionally records four caller-created
 * cudaEvent_t on the stream: events[0] before Step 1(a) (workspace reset
 * included), events[1] before Step 1(b), events[2] before Step 2(b),
 * events[3] after Step 2(b).  Used to time each step on the launching stream. */
dm_status dm_merge_column_async_ev(const dm_column_in* in, const dm_column_out* out, void* ws, size_t ws_bytes,
                                   dm_header* d_header, void* cuda_stream, void* const* events);

/* As above, then waits for the stream and fills out->merged_dict_len,
 * out->delta_dict_len, out->merged_bits; returns the device status. */
dm_status dm_merge_column(const dm_column_in* in, dm_column_out* out, void* ws, size_t ws_bytes, void* cuda_stream);

/* Merge `ncols` independent columns (a wide table) on one device.
 * ws[c] / ws_bytes[c] is column c's workspace.  Columns run concurrently on an
 * internal stream pool forked from and joined back into `cuda_stream`.
 * Synchronous: fills every out[c] result field; returns the worst status. */
dm_status dm_merge_table(int ncols, const dm_column_in* in, dm_column_out* out, void* const* ws,
                         const size_t* ws_bytes, void* cuda_stream);
/* As dm_merge_table without the host synchronisation: column c's results land
 * in d_headers[c] (device memory).  Stream-ordered, graph-capturable. */
dm_status dm_merge_table_async(int ncols, const dm_column_in* in, const dm_column_out* out, void* const* ws,
                               const size_t* ws_bytes, dm_header* const* d_headers, void* cuda_stream);

/* Steps 1(a), 1(b) and 2(a) only (no M'): U', X_M, X_D, U_D, r, the header
 * and (when |U_M| > 0) the compact table XC in the workspace.
 * out->x_main, out->x_delta and out->delta_rank must be non-NULL;
 * out->merged_codes is ignored.  Used by the row-sharded Step 2 (each device
 * then runs dm_recompress on its row range).  Stream-ordered. */
dm_status dm_dictionary_merge_async(const dm_column_in* in, const dm_column_out* out, void* ws, size_t ws_bytes,
                                    dm_header* d_header, void* cuda_stream);

/* Step 1(a) alone: U_D into out->delta_dict and r into out->delta_rank (both
 * required when n_delta > 0), |U_D| into d_header.  The root's part of the
 * sharded Step 1(b).  Stream-ordered. */
dm_status dm_delta_dictionary_async(const dm_column_in* in, const dm_column_out* out, void* ws, size_t ws_bytes,
                                    dm_header* d_header, void* cuda_stream);

/* Steps 1(b) and 2(a) for a delta that already IS its dictionary: in->delta
 * holds U_D itself (sorted, distinct -- the paper reads it off the CSB+ tree's
 * leaves; the caller's promise, not checked).  X_D is over in->delta;
 * out->delta_rank is not used; out->x_main and out->x_delta are required.
 * Builds XC like dm_dictionary_merge_async.  One value range of the sharded
 * Step 1(b) (NEXT2).  Stream-ordered. */
dm_status dm_dictionary_merge_sorted_async(const dm_column_in* in, const dm_column_out* out, void* ws,
                                           size_t ws_bytes, dm_header* d_header, void* cuda_stream);

/* Sharded Step 1(b) helpers (NEXT2), stream-ordered, device pointers:
 * pos[i] = #{sorted[j] < values[i]} (lower bound) for n_values values of type
 * `key`; x[i] += add for n u32 entries (rebasing a range's X_M / X_D by the
 * |U'| of earlier ranges); R += add in n_records XC records, flags kept
 * (rebasing by the new values of earlier ranges). */
dm_status dm_lower_bound_async(int key, const void* sorted, uint64_t n, const void* values, uint64_t n_values,
                               uint64_t* pos, void* cuda_stream);
dm_status dm_rebase_async(uint32_t* x, uint64_t n, uint32_t add, void* cuda_stream);
dm_status dm_xc_rebase_async(void* records, uint64_t n_records, uint32_t add, void* cuda_stream);

/* Step 2(b) alone (Eq 11): given translation tables, write
 * M'[i] = x_main[M[i]] for i < n_main and M'[n_main + k] = x_delta[delta_rank[k]]
 * for k < n_delta, packed at new_bits (1..32) into dm_words(n_main + n_delta,
 * new_bits) words of out_codes (capacity out_cap_words).  Every table value must
 * be < 2^new_bits.  main_codes at main_bits (1..32), codes < dict_len (else
 * DM_E_CODE_RANGE, reported after a stream synchronisation).  With n_main > 0,
 * 1 <= dict_len < 2^32 and main_bits >= dm_width(dict_len), else DM_E_INVALID.  Device pointers,
 * 16-byte aligned.  Synchronous. */
dm_status dm_recompress(const uint64_t* main_codes, uint64_t n_main, uint32_t main_bits, uint64_t dict_len,
                        const uint32_t* x_main, const uint32_t* x_delta, const uint32_t* delta_rank,
                        uint64_t n_delta, uint32_t new_bits, uint64_t* out_codes, uint64_t out_cap_words,
                        void* cuda_stream);

/* Compact translation table XC (X_M[c] = c + #{new values
 * inserted at or before main position c}, the closed form of X_M).
 * Used by the row-sharded Step 2: the root's XC (|U_M|/2^(shift+2)
 * 8-byte records + one byte per new value, ~67 MB for cfg5) is broadcast
 * instead of X_M (4.3 GB).  Layout: record s = {u32 R | flag << 31, u32 four
 * cumulative per-block counts}, R = #{new values with insertion point
 * p <= s * 4 * 2^shift}; offsets[k] = (p_k - 1) mod 2^shift for the k-th new
 * value in sorted order.  A flagged record (counts too large) means: read the
 * plain X_M for that superblock. */
typedef struct {
  const void* records;     /* device, n_records * 8 bytes, 16-byte aligned      */
  uint64_t n_records;      /* ceil(dict_len / (4 << shift))                      */
  const uint8_t* offsets;  /* device, |U'| - |U_M| bytes used, 16-byte aligned  */
  uint64_t offsets_cap;    /* bytes readable (n_delta + 16)                      */
  uint32_t shift;          /* block = 2^shift codes (7 or 8)                     */
  int32_t built;           /* 1 if a merge with this workspace builds XC        */
} dm_xc;
/* Describe the XC inside a workspace after dm_dictionary_merge_async or
 * dm_dictionary_merge_sorted_async (which always build it when |U_M| > 0) --
 * pointers into `ws`, valid while it lives and until the next call on it.
 * Host, pure. */
dm_status dm_xc_export(const dm_column_in* in, const void* ws, size_t ws_bytes, dm_xc* xc);
/* Gather the X_M slices of flagged superblocks: for each, ids[slot] = its
 * record index and slices[slot * 4 << shift ...] = its X_M entries; *d_count
 * (device u64) = number of slots.  Capacities: ids >= count, slices >=
 * count * (4 << shift).  ids = slices = NULL: count only (x_main may be NULL);
 * a caller sizes the buffers from that count first.  Stream-ordered. */
dm_status dm_xc_exceptions_gather(const dm_xc* xc, uint64_t dict_len, const uint32_t* x_main, uint32_t* ids,
                                  uint32_t* slices, uint64_t* d_count, void* cuda_stream);
/* The inverse on a receiving rank: write the `count` slices into x_main (a
 * dict_len-entry buffer whose other entries are never read).  Stream-ordered. */
dm_status dm_xc_exceptions_scatter(const dm_xc* xc, uint64_t dict_len, const uint32_t* ids, const uint32_t* slices,
                                   uint64_t count, uint32_t* x_main, void* cuda_stream);
/* dm_recompress with the main translation read from XC (L2); x_main is read
 * only for flagged superblocks.  Same arguments and errors otherwise.
 * Synchronous. */
dm_status dm_recompress_xc(const uint64_t* main_codes, uint64_t n_main, uint32_t main_bits, uint64_t dict_len,
                           const dm_xc* xc, const uint32_t* x_main, const uint32_t* x_delta,
                           const uint32_t* delta_rank, uint64_t n_delta, uint32_t new_bits, uint64_t* out_codes,
                           uint64_t out_cap_words, void* cuda_stream);

/* ---------------------------------------------------------------- sharded merge
 * One column's merge spread over the ranks of a communicator, one GPU per rank
 * (SURVEY §8e).  The paper splits Step 2 over threads by tuples, "the N' tuples
 * are evenly split between the threads", every thread translating its
 * own range through the shared tables (Eq 11); here the threads are GPUs
 * and the tables cross NVLink once.  Output rows [0, N') are cut into one
 * contiguous range per rank (dm_plan_row_shards); rank g holds the packed main
 * codes of its range's main rows and writes its range's M' words.
 *
 * Transport: dm_comm, either NCCL (dm_comm_init_nccl; the library resolves
 * ncclBroadcast / ncclAllGather / ncclSend / ncclRecv at run time from the
 * process's libnccl.so.2) or caller-supplied callbacks over HOST buffers
 * (dm_comm_init_callbacks: any process-group library; the library stages device
 * data through pinned host memory and synchronises around each call).  Every
 * rank calls the collectives in the same order; callbacks return 0 on success. */
typedef struct dm_comm dm_comm;
typedef struct {
  /* buf: `bytes` host bytes; on `root` the data, elsewhere filled in */
  int (*broadcast)(void* buf, uint64_t bytes, int root, void* user);
  /* recv: nranks * bytes host bytes, rank g's `send` at offset g * bytes */
  int (*allgather)(const void* send, void* recv, uint64_t bytes, void* user);
  /* is_send = 1: send `bytes` of buf to `peer`; 0: receive them from `peer` into buf */
  int (*sendrecv)(void* buf, uint64_t bytes, int peer, int is_send, void* user);
  void* user;
} dm_comm_callbacks;
/* 128 bytes: a fresh NCCL unique id for rank 0 to hand to every rank (host).
 * DM_E_NCCL when no NCCL library can be loaded. */
dm_status dm_comm_nccl_unique_id(void* id_out);
/* Collective over the nranks processes; `device` becomes the current device.
 * NULL on failure. */
dm_comm* dm_comm_init_nccl(const void* id, int nranks, int rank, int device);
/* The callbacks struct is copied; it must stay valid (its `user`) for the comm's life. */
dm_comm* dm_comm_init_callbacks(const dm_comm_callbacks* cb, int nranks, int rank);
void dm_comm_destroy(dm_comm* comm);
int dm_comm_rank(const dm_comm* comm);
int dm_comm_size(const dm_comm* comm);
/* Host-only self-test of a callback transport (no GPU): broadcast from every
 * root, an all-gather in rank order and a rank 0 -> last rank transfer.
 * Collective.  DM_OK, or DM_E_NCCL if any byte arrived wrong. */
dm_status dm_comm_selftest_host(dm_comm* comm);

/* cuts[0..nranks]: rank g owns output rows [cuts[g], cuts[g+1]) of the
 * N' = n_main + n_delta rows (main rows first, then delta rows);
 * every cut but the last is a multiple of 4096, so every range starts on a u64
 * word at both widths.  Host, pure. */
void dm_plan_row_shards(uint64_t n_main, uint64_t n_delta, int nranks, uint64_t* cuts);
/* u64 words rank `rank`'s M' range can need: its rows at the widest possible
 * b' = width(dict_len + n_delta).  Host, pure. */
uint64_t dm_sharded_codes_cap_words(uint64_t dict_len, uint64_t n_main, uint64_t n_delta, int nranks, int rank);

/* U_M value ranges for DM_STEP1B_RANGES: cuts[0..nranks], rank g holds
 * U_M[cuts[g], cuts[g+1]); every cut but the last a multiple of 1024 (whole XC
 * superblocks).  Host, pure. */
void dm_plan_dict_ranges(uint64_t dict_len, int nranks, uint64_t* cuts);

enum { DM_TABLES_XC = 0, DM_TABLES_PLAIN = 1 };
enum { DM_STEP1B_ROOT = 0, DM_STEP1B_RANGES = 1 };
typedef struct {
  int32_t key;                 /* dm_key, the same on every rank                         */
  int32_t tables;              /* DM_TABLES_XC: broadcast the compact table XC (NEXT3)   *
                                * (+ the X_M slices of flagged superblocks); PLAIN: the  *
                                * literal X_M (SURVEY §8e's control design)              */
  int32_t root;                /* rank that holds D and runs Step 1(a) (and, ROOT mode,  *
                                * Step 1(b))                                             */
  int32_t step1b;              /* DM_STEP1B_ROOT: the root merges the whole dictionary;  *
                                * DM_STEP1B_RANGES (the paper's        *
                                * quantile-split parallel merge, one level up):*
                                * rank g merges its U_M value range with the U_D values  *
                                * that fall into it, an all-gather of (|U'_g|, new       *
                                * values_g) rebases every range's tables; XC only        *
                                * (tables = DM_TABLES_XC, 128-code blocks)               */
  const void* main_dict;       /* ROOT: the root's U_M (device), strictly increasing;    *
                                * RANGES: this rank's range U_M[range_begin, +range_len) */
  uint64_t dict_len;           /* |U_M| (every rank)                                     */
  uint64_t range_begin;        /* RANGES: dm_plan_dict_ranges(dict_len, nranks)[g]       */
  uint64_t range_len;          /* RANGES: the range's length (> 0)                       */
  const void* delta;           /* root: D (device), insertion order; others ignored      */
  uint64_t n_delta;            /* N_D (every rank)                                       */
  const uint64_t* main_codes;  /* this rank's main rows [min(cuts[g], N_M),              *
                                * min(cuts[g+1], N_M)) packed at main_bits from bit 0    *
                                * (device, 16-byte aligned)                              */
  uint64_t n_main;             /* N_M, the whole column (every rank)                     */
  uint32_t main_bits;          /* b (every rank)                                         */
} dm_sharded_in;
typedef struct {
  void* merged_dict;               /* ROOT: the root's U' (device), capacity             *
                                    * merged_dict_cap keys; RANGES: this rank's slice of  *
                                    * U' (its range's values and the new ones among them) */
  uint64_t merged_dict_cap;        /* ROOT (root): >= dict_len + n_delta; RANGES (every   *
                                    * rank): >= range_len + n_delta                       */
  uint64_t* merged_codes;          /* this rank's M' words: rows [cuts[g], cuts[g+1])    *
                                    * at b' from bit 0 (device, 16-byte aligned)         */
  uint64_t merged_codes_cap_words; /* >= dm_sharded_codes_cap_words(...)                 */
  uint64_t merged_dict_len;        /* out (every rank): |U'|                            */
  uint32_t merged_bits;            /* out (every rank): b'                              */
  uint64_t merged_dict_offset;     /* out, RANGES: U' index of this rank's slice; its   *
                                    * length = merged_slice_len                         */
  uint64_t merged_slice_len;       /* out, RANGES: entries in this rank's U' slice      */
} dm_sharded_out;
/* Collective, synchronous.  1. every rank's descriptor (key, tables, root,
 * |U_M|, N_M, N_D, b) must agree (all-gather; else DM_E_INVALID everywhere);
 * 2. root: Steps 1(a)-2(a); 3. broadcast of the result
 * header; 4. broadcast of XC (or X_M); 5. root computes the delta rows' codes
 * X_D[r[k]] and sends each owner its slice; 6. every rank:
 * Step 2(b) of its rows (Eq 11).  Concatenating the ranks' M' words in
 * rank order gives the merged code vector of dm_merge_column, bit for bit.
 * DM_STEP1B_RANGES replaces 2-4 by: all-gather of every range's first value,
 * the root cuts U_D there (lower bound) and broadcasts U_D and the cuts; every
 * rank merges its range (Steps 1(b)-2(a)); all-gather of (|U'_g|, new_g); every
 * rank rebases its X_M / X_D / XC records by the counts of earlier ranges; the
 * XC pieces and the flagged superblocks' X_M slices are all-gathered (rank =
 * value order), the X_D pieces gathered on the root.  Concatenating the ranks'
 * U' slices in rank order gives U'.
 * Temporaries come from the device's stream-ordered memory pool and are
 * released before return (a non-root rank holding flagged-superblock slices
 * allocates a sparse |U_M|-entry X_M).  Returns the worst status of all ranks;
 * DM_E_NCCL for a failed transport call. */
dm_status dm_merge_column_sharded(dm_comm* comm, const dm_sharded_in* in, dm_sharded_out* out, void* cuda_stream);

/* Pack n u32 codes (each < 2^bits) into dm_words(n, bits) words at `bits`
 * (device pointers; words need not be zeroed).  Stream-ordered. */
dm_status dm_pack_codes(const uint32_t* codes, uint64_t n, uint32_t bits, uint64_t* words, void* cuda_stream);
/* Unpack n codes at `bits` into u32.  Stream-ordered. */
dm_status dm_unpack_codes(const uint64_t* words, uint64_t n, uint32_t bits, uint32_t* codes, void* cuda_stream);

/* Host-buffer entry point (end-to-end use).  `in` and `out` hold HOST pointers
 * (checked before any copy: a NULL input with a non-zero length or a NULL
 * merged_dict / merged_codes gives DM_E_INVALID; merged_dict_cap < dict_len +
 * n_delta or merged_codes_cap_words < dm_merged_codes_cap_words(in) gives
 * DM_E_CAPACITY; the optional x_main / x_delta / delta_dict / delta_rank
 * buffers must hold dict_len / n_delta entries)
 * (pinned memory gives full PCIe bandwidth and copy/compute overlap); the
 * context owns device staging buffers, grows them on demand and reuses them
 * across calls.  Pipelined over three streams: U_M and D are uploaded first and
 * Steps 1(a)-2(a) start while M is still uploading in row chunks; Step 2(b)
 * runs chunk by chunk as M arrives (rows are independent, Eq 11) and each M'
 * chunk is downloaded while later chunks upload; U' (and any requested X_M /
 * X_D / U_D / r) download during the M upload.  Synchronises and fills the
 * result fields. */
typedef struct dm_ctx dm_ctx;
dm_ctx* dm_ctx_create(int device);
void dm_ctx_destroy(dm_ctx* ctx);
dm_status dm_merge_column_host(dm_ctx* ctx, const dm_column_in* in, dm_column_out* out);

/* Process-wide tuning knobs (they never change results, only which kernels
 * run).  knob 0 = placement of the main translation table in Step 2(b):
 *   0 auto (default): plain X_M in shared memory when it fits (<= 96 KB);
 *     else the compact table XC (per 4 blocks of 128 or 256
 *     codes an 8-byte record, per new dictionary value one byte; X_M[c] = c +
 *     #{new values inserted at or before main position c}
 *     restated): staged in shared memory when X_M is at most 64 MB, its
 *     records fit and the device finds few new values per block, read through
 *     L2 when X_M exceeds 64 MB (it would not stay L2-resident); else the plain
 *     X_M through L2.  When XC is read through L2 and X_M was not requested
 *     (out->x_main NULL), X_M is only filled for the superblocks XC flags;
 *   1 plain X_M only;  2 XC, staged in shared memory when it fits, else L2;
 *   3 XC through L2.
 * knob 1 = Step 1(b) variant: 0 (default) auto -- sparse-delta tiles when
 *   N_D <= |U_M| / 8, else bitmap-slot tiles in two passes (count, prefix sum,
 *   write: P:302-314); 1 the first GPU form (rank tiles, three kernels); 2
 *   bitmap-slot tiles in one pass with decoupled look-back; 3 sparse-delta
 *   tiles always (|U_M| > 0): U_M tiles of 2048 with the U_D values that fall
 *   into them, one pass (copy U_M with gaps, insert the new values).
 * knob 2 = Step 1(a) front end: 0 (default) auto --
 *   probe-first for 16-byte keys with N_D >= 65536 and |U_M| * 16 <= 64 MB when
 *   no U_D / X_D / r output is requested, else hash deduplication of D before
 *   the sort for 16-byte keys with N_D >= 65536 and for bucket-path deltas with
 *   N_D > 4 |U_M| (they must repeat values); 1 neither; 2 hash deduplication
 *   always (insert every tuple into a device hash table, sort only the distinct
 *   values, map each tuple to its value's rank: same U_D and r); 3 probe-first
 *   whenever |U_M| > 0 and no U_D / X_D / r output is requested (look every
 *   delta value up in U_M -- binary search -- and sort only the values not
 *   found: U' = merge(U_M, U_new), a found value's code is X_M at its U_M
 *   position; |U_D| is still reported).  Changes the workspace size:
 *   call dm_workspace_bytes after setting it.
 * knob 3 = Step 2(b) variant: 0 (default) the optimized recompression through
 *   X_M / X_D (Eq 11); 1 the paper's unoptimized form:
 *   every tuple's value binary-searched in U' -- a measured baseline only.
 * knob 4 = XC block shift: 0 (default) per column from N_D / |U_M|; 7 or 8
 *   fixed (the sharded Step 1(b) needs one shift for all value ranges).
 * knob 5 = Step 1(a) sort: 0 (default) auto -- the bucket path for
 *   2^11 <= N_D <= 2^23 (one counting pass into ~N_D/4 buckets by the top bits
 *   below the keys' common prefix, then each key ranked among its bucket mates),
 *   else the LSD radix passes; 1 LSD passes only; 2 bucket path for any N_D.  A
 *   skewed key set (a bucket above 256 keys) falls back to the LSD passes on the
 *   device.  Same U_D and r either way.  Changes the workspace size.
 * knob 6 = Step 2(b) kernel form when XC sits in shared memory: 0 (default)
 *   thread-per-group (a lane owns a 32-row group: unpack, translate and pack
 *   in registers with compile-time widths; used when b' - b is 0 or 1 and the
 *   plain X_M is whole), 1 the warp-per-group kernel (a lane per row, shuffle
 *   packing) for every width pair.  Same M' either way.
 * knob 7 = grid of the sparse-delta Step 1(b) kernels (knob 1 = 3), which walk
 *   U_M tiles t, t + grid, ... and load the next tile while working on the
 *   current one: 0 (default) one resident wave (SMs x occupancy), 1 one CTA per
 *   tile, 2 three CTAs (tests).  Same outputs either way.
 * The process starts with knobs 0..7 = $DM_XMODE / $DM_MERGE / $DM_DEDUP /
 * $DM_STEP2 / $DM_XC_SHIFT / $DM_SORT1A / $DM_TPG / $DM_SP_GRID when set
 * (experiments), else 0.
 * Returns DM_OK, or DM_E_INVALID for an unknown knob or value.  Affects calls
 * made after it returns (a captured CUDA graph keeps the kernels it recorded). */
int dm_set_tuning(int knob, int value);
/* Current value of a knob (>= 0), or DM_E_INVALID for an unknown knob.  Lets a
 * caller that changes a knob restore it afterwards. */
int dm_get_tuning(int knob);

/* Number of library kernels launched by this process so far (monotone). */
uint64_t dm_launch_count(void);
/* Last CUDA error code seen by the library (cudaError_t as int). */
int dm_last_cuda_error(void);
const char* dm_status_str(int status);

#ifdef __cplusplus
}
#endif
#endif
