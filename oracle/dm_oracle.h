/*
 * dm_oracle.h -- plain, slow, single-threaded CPU oracle for the online
 * dictionary merge of Krueger et al., "Fast Updates on Read-Optimized
 * Databases Using Multi-Core CPUs" (arXiv 1109.6885, PVLDB 5(1)).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA library
 * (paper_1109_6885_b200/csrc, include/dictmerge.h) and neither includes the
 * other.
 *
 * Citations: "P:n" = line n of the paper text.  Readings of
 * silent/garbled passages are the DESIGN.md table "Readings" (A1..A16).
 *
 * Conventions (readings A1-A5):
 *   - code width w(n) = max(1, ceil(log2 n))             (Eq 4; A1)
 *   - codes are 0-based dictionary positions              (A2)
 *   - packed vectors are LSB-first bitstreams in little-endian u64 words,
 *     exactly ceil(n*w/64) words, pad bits zero            (A4)
 *   - 4- and 8-byte keys: unsigned integers; 16-byte keys: raw bytes compared
 *     with memcmp over all 16 bytes                        (A5)
 */
#ifndef DM_ORACLE_H
#define DM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DMO_OK = 0,
  DMO_E_INVALID = -1,   /* bad sizes / widths / null pointers            */
  DMO_E_TOO_WIDE = -3,  /* |U'| > 2^32                                   */
  DMO_E_UNSORTED = -4,  /* main dictionary not strictly increasing       */
  DMO_E_CODE_RANGE = -5 /* some main code >= |U_M|                       */
};

typedef struct {
  uint32_t key_bytes;          /* 4, 8 or 16                                   */
  const void* main_dict;       /* |U_M| keys, strictly increasing              */
  uint64_t dict_len;           /* |U_M|                                        */
  const uint64_t* main_words;  /* M packed at main_bits, ceil(n_main*b/64) words */
  uint64_t n_main;             /* N_M                                          */
  uint32_t main_bits;          /* b, w(|U_M|) <= b <= 32                        */
  const void* delta;           /* D, N_D keys in insertion order               */
  uint64_t n_delta;            /* N_D                                          */
} dmo_in;

typedef struct {
  void* merged_dict;           /* U', capacity dict_len + n_delta keys          */
  uint64_t merged_len;         /* out: |U'|                                     */
  uint32_t merged_bits;        /* out: b' = w(|U'|)                             */
  uint64_t* merged_words;      /* M', capacity ceil(N'*w(dict_len+n_delta)/64)  */
  uint32_t* x_main;            /* X_M, dict_len entries (may be NULL)           */
  uint32_t* x_delta;           /* X_D, n_delta capacity (may be NULL)           */
  void* delta_dict;            /* U_D, n_delta capacity (may be NULL)           */
  uint64_t delta_dict_len;     /* out: |U_D|                                    */
  uint32_t* delta_rank;        /* r[k] = index of D[k] in U_D (linear mode; may be NULL) */
  double seconds[4];           /* out: step 1(a), 1(b), 2(a), 2(b) wall times   */
} dmo_out;

uint32_t dmo_width(uint64_t n);
uint64_t dmo_words(uint64_t n, uint32_t bits);
/* Pack n codes at `bits` into dmo_words(n,bits) words (zeroed first). */
int dmo_pack(const uint32_t* codes, uint64_t n, uint32_t bits, uint64_t* words);
/* Unpack n codes at `bits`. */
int dmo_unpack(const uint64_t* words, uint64_t n, uint32_t bits, uint32_t* codes);

/* The paper's optimized merge, serial, in its own order:
 * Step 1(a) sort+unique D with ranks,
 * Step 1(b) two-pointer merge emitting X_M / X_D,
 * Step 2(a) width (Eq 4), Step 2(b) M'[i] = X_M[M[i]] (Eq 11),
 * delta appended through X_D. */
int dmo_merge_linear(const dmo_in* in, dmo_out* out);

/* The plain definition (Eqs 2-4):
 * V = decode(M) ++ D, U' = sorted distinct (U_M u D), b' = w(|U'|),
 * M'[i] = position of V[i] in U' by binary search; X_M / X_D likewise. */
int dmo_merge_definitional(const dmo_in* in, dmo_out* out);

/* Definitional codes for given values (for sampled-row checks of very large
 * merges): U' = std::set_union(U_M, sorted distinct D) (Eq 3), then
 * codes[i] = position of values[i] in U' by binary search.
 * Every value must occur in U_M or D (DMO_E_CODE_RANGE otherwise).
 * *merged_len receives |U'|. */
int dmo_codes_at(uint32_t key_bytes, const void* main_dict, uint64_t dict_len, const void* delta,
                 uint64_t n_delta, const void* values, uint64_t n_values, uint32_t* codes,
                 uint64_t* merged_len);

#ifdef __cplusplus
}
#endif
#endif
