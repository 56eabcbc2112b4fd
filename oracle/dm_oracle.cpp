// dm_oracle.cpp -- plain CPU oracle for the online dictionary merge (arXiv 1109.6885).
//
// TEST INFRASTRUCTURE ONLY (see dm_oracle.h).  Deliberately simple: std::sort,
// std::unique, std::lower_bound, a textbook two-pointer merge and scalar bit
// packing.  No blocking, no fusion, no threads.  Each function cites the paper
// passage it follows ("P:n" = PAPER.md line n).
#include "dm_oracle.h"

#include <algorithm>
#include <iterator>
#include <chrono>
#include <cstring>
#include <utility>
#include <vector>

namespace {

using clk = std::chrono::steady_clock;
double secs(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

// 16-byte key compared bytewise over all 16 bytes (reading A5).
struct K16 {
  unsigned char b[16];
  bool operator<(const K16& o) const { return std::memcmp(b, o.b, 16) < 0; }
  bool operator==(const K16& o) const { return std::memcmp(b, o.b, 16) == 0; }
};

// ---------------------------------------------------------------- codec
// LSB-first bitstream in little-endian u64 words (reading A4): code i occupies
// bits [i*bits, (i+1)*bits) of the stream; bit s lives in word s/64 at bit s%64.
uint64_t code_at(const uint64_t* W, uint64_t i, uint32_t bits) {
  uint64_t s = i * (uint64_t)bits;  // 64-bit bit offset
  uint64_t w = s >> 6;
  uint32_t o = (uint32_t)(s & 63);
  uint64_t v = W[w] >> o;
  if (o + bits > 64) v |= W[w + 1] << (64 - o);
  return v & ((bits == 64) ? ~0ull : ((1ull << bits) - 1));
}

void put_code(uint64_t* W, uint64_t i, uint64_t c, uint32_t bits) {
  uint64_t s = i * (uint64_t)bits;
  uint64_t w = s >> 6;
  uint32_t o = (uint32_t)(s & 63);
  W[w] |= c << o;
  if (o + bits > 64) W[w + 1] |= c >> (64 - o);
}

uint32_t width_of(uint64_t n) {
  // Eq 4: E'_C = ceil(log2 |U'|); 1-bit minimum for |U'| <= 1 (reading A1).
  uint32_t w = 1;
  while (w < 64 && (1ull << w) < n) ++w;
  return w;
}

uint64_t words_of(uint64_t n, uint32_t bits) { return (n * (uint64_t)bits + 63) / 64; }

template <class K>
int validate(const dmo_in* in, const K* UM) {
  if (in->n_main > 0 && in->dict_len == 0) return DMO_E_INVALID;
  if (in->main_bits < 1 || in->main_bits > 32) return DMO_E_INVALID;
  if (in->dict_len > 0 && in->main_bits < width_of(in->dict_len)) return DMO_E_INVALID;
  // "sorted unique values": strictly increasing.
  for (uint64_t i = 1; i < in->dict_len; ++i)
    if (!(UM[i - 1] < UM[i])) return DMO_E_UNSORTED;
  for (uint64_t i = 0; i < in->n_main; ++i)
    if (code_at(in->main_words, i, in->main_bits) >= in->dict_len) return DMO_E_CODE_RANGE;
  return DMO_OK;
}

// ------------------------------------------------------------- linear mode
template <class K>
int merge_linear(const dmo_in* in, dmo_out* out) {
  const K* UM = static_cast<const K*>(in->main_dict);
  const K* D = static_cast<const K*>(in->delta);
  int st = validate<K>(in, UM);
  if (st != DMO_OK) return st;
  const uint64_t nM = in->n_main, nD = in->n_delta, nUM = in->dict_len;

  // Step 1(a): sorted distinct delta values U_D and
  // each delta tuple replaced by its index in U_D.
  auto t0 = clk::now();
  std::vector<std::pair<K, uint64_t>> kv(nD);
  for (uint64_t k = 0; k < nD; ++k) kv[k] = {D[k], k};
  std::sort(kv.begin(), kv.end(), [](const std::pair<K, uint64_t>& a, const std::pair<K, uint64_t>& b) {
    if (a.first < b.first) return true;
    if (b.first < a.first) return false;
    return a.second < b.second;
  });
  std::vector<K> UD;
  std::vector<uint32_t> r(nD);
  for (uint64_t p = 0; p < nD; ++p) {
    if (p == 0 || !(kv[p].first == kv[p - 1].first)) UD.push_back(kv[p].first);
    r[kv[p].second] = (uint32_t)(UD.size() - 1);
  }
  auto t1 = clk::now();

  // Step 1(b): two pointers; append the smaller value and
  // record its output index in X_M or X_D; equal heads are appended once and
  // both tables get the same index.
  const uint64_t nUD = UD.size();
  std::vector<K> U;
  U.reserve(nUM + nUD);
  std::vector<uint32_t> XM(nUM), XD(nUD);
  uint64_t i = 0, j = 0;
  while (i < nUM && j < nUD) {
    if (UM[i] < UD[j]) {
      XM[i++] = (uint32_t)U.size();
      U.push_back(UM[i - 1]);
    } else if (UD[j] < UM[i]) {
      XD[j++] = (uint32_t)U.size();
      U.push_back(UD[j - 1]);
    } else {
      XM[i++] = (uint32_t)U.size();
      XD[j++] = (uint32_t)U.size();
      U.push_back(UM[i - 1]);
    }
  }
  while (i < nUM) { XM[i++] = (uint32_t)U.size(); U.push_back(UM[i - 1]); }
  while (j < nUD) { XD[j++] = (uint32_t)U.size(); U.push_back(UD[j - 1]); }
  auto t2 = clk::now();
  if (U.size() > (1ull << 32)) return DMO_E_TOO_WIDE;

  // Step 2(a) (Eq 4).
  const uint32_t nb = width_of(U.size());
  auto t3 = clk::now();

  // Step 2(b) (Eq 11): M'[i] = X_M[M[i]]; then the delta
  // tuples appended through X_D.
  const uint64_t nW = words_of(nM + nD, nb);
  std::memset(out->merged_words, 0, nW * sizeof(uint64_t));
  for (uint64_t row = 0; row < nM; ++row)
    put_code(out->merged_words, row, XM[code_at(in->main_words, row, in->main_bits)], nb);
  for (uint64_t k = 0; k < nD; ++k) put_code(out->merged_words, nM + k, XD[r[k]], nb);
  auto t4 = clk::now();

  std::memcpy(out->merged_dict, U.data(), U.size() * sizeof(K));
  out->merged_len = U.size();
  out->merged_bits = nb;
  out->delta_dict_len = nUD;
  if (out->x_main) std::memcpy(out->x_main, XM.data(), nUM * sizeof(uint32_t));
  if (out->x_delta) std::memcpy(out->x_delta, XD.data(), nUD * sizeof(uint32_t));
  if (out->delta_dict) std::memcpy(out->delta_dict, UD.data(), nUD * sizeof(K));
  if (out->delta_rank) std::memcpy(out->delta_rank, r.data(), nD * sizeof(uint32_t));
  out->seconds[0] = secs(t0, t1);
  out->seconds[1] = secs(t1, t2);
  out->seconds[2] = secs(t2, t3);
  out->seconds[3] = secs(t3, t4);
  return DMO_OK;
}

// -------------------------------------------------------- definitional mode
template <class K>
int merge_definitional(const dmo_in* in, dmo_out* out) {
  const K* UM = static_cast<const K*>(in->main_dict);
  const K* D = static_cast<const K*>(in->delta);
  int st = validate<K>(in, UM);
  if (st != DMO_OK) return st;
  const uint64_t nM = in->n_main, nD = in->n_delta, nUM = in->dict_len;
  auto t0 = clk::now();

  // Output column = main followed by delta, in order (Eq 2).
  std::vector<K> V;
  V.reserve(nM + nD);
  for (uint64_t row = 0; row < nM; ++row) V.push_back(UM[code_at(in->main_words, row, in->main_bits)]);
  for (uint64_t k = 0; k < nD; ++k) V.push_back(D[k]);

  // U' = sorted distinct values of D u U_M (Eq 3).
  std::vector<K> U(UM, UM + nUM);
  U.insert(U.end(), D, D + nD);
  std::sort(U.begin(), U.end());
  U.erase(std::unique(U.begin(), U.end()), U.end());
  if (U.size() > (1ull << 32)) return DMO_E_TOO_WIDE;
  std::vector<K> UD(D, D + nD);
  std::sort(UD.begin(), UD.end());
  UD.erase(std::unique(UD.begin(), UD.end()), UD.end());
  auto t1 = clk::now();

  // b' = ceil(log2 |U'|) (Eq 4).
  const uint32_t nb = width_of(U.size());

  // The code of a value is its position in the sorted dictionary (P:130,
  // P:165), found by binary search.
  const uint64_t nW = words_of(nM + nD, nb);
  std::memset(out->merged_words, 0, nW * sizeof(uint64_t));
  for (uint64_t row = 0; row < nM + nD; ++row) {
    uint64_t pos = (uint64_t)(std::lower_bound(U.begin(), U.end(), V[row]) - U.begin());
    put_code(out->merged_words, row, pos, nb);
  }
  auto t2 = clk::now();

  std::memcpy(out->merged_dict, U.data(), U.size() * sizeof(K));
  out->merged_len = U.size();
  out->merged_bits = nb;
  out->delta_dict_len = UD.size();
  if (out->x_main)
    for (uint64_t i = 0; i < nUM; ++i)
      out->x_main[i] = (uint32_t)(std::lower_bound(U.begin(), U.end(), UM[i]) - U.begin());
  if (out->x_delta)
    for (uint64_t j = 0; j < UD.size(); ++j)
      out->x_delta[j] = (uint32_t)(std::lower_bound(U.begin(), U.end(), UD[j]) - U.begin());
  if (out->delta_dict) std::memcpy(out->delta_dict, UD.data(), UD.size() * sizeof(K));
  if (out->delta_rank)
    for (uint64_t k = 0; k < nD; ++k)
      out->delta_rank[k] = (uint32_t)(std::lower_bound(UD.begin(), UD.end(), D[k]) - UD.begin());
  out->seconds[0] = secs(t0, t1);
  out->seconds[1] = 0;
  out->seconds[2] = 0;
  out->seconds[3] = secs(t1, t2);
  return DMO_OK;
}

template <class K>
int codes_at(const K* UM, uint64_t nUM, const K* D, uint64_t nD, const K* vals, uint64_t nv, uint32_t* codes,
             uint64_t* merged_len) {
  for (uint64_t i = 1; i < nUM; ++i)
    if (!(UM[i - 1] < UM[i])) return DMO_E_UNSORTED;
  std::vector<K> UD(D, D + nD);
  std::sort(UD.begin(), UD.end());
  UD.erase(std::unique(UD.begin(), UD.end()), UD.end());
  std::vector<K> U;
  U.reserve(nUM + UD.size());
  std::set_union(UM, UM + nUM, UD.begin(), UD.end(), std::back_inserter(U));
  *merged_len = U.size();
  for (uint64_t i = 0; i < nv; ++i) {
    auto it = std::lower_bound(U.begin(), U.end(), vals[i]);
    if (it == U.end() || !(*it == vals[i])) return DMO_E_CODE_RANGE;
    codes[i] = (uint32_t)(it - U.begin());
  }
  return DMO_OK;
}

bool args_ok(const dmo_in* in, const dmo_out* out) {
  if (!in || !out) return false;
  if (in->key_bytes != 4 && in->key_bytes != 8 && in->key_bytes != 16) return false;
  if (in->dict_len && !in->main_dict) return false;
  if (in->n_main && !in->main_words) return false;
  if (in->n_delta && !in->delta) return false;
  if ((in->dict_len + in->n_delta) && !out->merged_dict) return false;
  if ((in->n_main + in->n_delta) && !out->merged_words) return false;
  return true;
}

}  // namespace

extern "C" {

uint32_t dmo_width(uint64_t n) { return width_of(n); }
uint64_t dmo_words(uint64_t n, uint32_t bits) { return words_of(n, bits); }

int dmo_pack(const uint32_t* codes, uint64_t n, uint32_t bits, uint64_t* words) {
  if (bits < 1 || bits > 32) return DMO_E_INVALID;
  std::memset(words, 0, words_of(n, bits) * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) {
    if (bits < 32 && (codes[i] >> bits)) return DMO_E_CODE_RANGE;
    put_code(words, i, codes[i], bits);
  }
  return DMO_OK;
}

int dmo_unpack(const uint64_t* words, uint64_t n, uint32_t bits, uint32_t* codes) {
  if (bits < 1 || bits > 32) return DMO_E_INVALID;
  for (uint64_t i = 0; i < n; ++i) codes[i] = (uint32_t)code_at(words, i, bits);
  return DMO_OK;
}

int dmo_merge_linear(const dmo_in* in, dmo_out* out) {
  if (!args_ok(in, out)) return DMO_E_INVALID;
  if (in->key_bytes == 4) return merge_linear<uint32_t>(in, out);
  return in->key_bytes == 8 ? merge_linear<uint64_t>(in, out) : merge_linear<K16>(in, out);
}

int dmo_merge_definitional(const dmo_in* in, dmo_out* out) {
  if (!args_ok(in, out)) return DMO_E_INVALID;
  if (in->key_bytes == 4) return merge_definitional<uint32_t>(in, out);
  return in->key_bytes == 8 ? merge_definitional<uint64_t>(in, out) : merge_definitional<K16>(in, out);
}

int dmo_codes_at(uint32_t key_bytes, const void* main_dict, uint64_t dict_len, const void* delta, uint64_t n_delta,
                 const void* values, uint64_t n_values, uint32_t* codes, uint64_t* merged_len) {
  if (key_bytes == 8)
    return codes_at<uint64_t>(static_cast<const uint64_t*>(main_dict), dict_len,
                              static_cast<const uint64_t*>(delta), n_delta, static_cast<const uint64_t*>(values),
                              n_values, codes, merged_len);
  if (key_bytes == 4)
    return codes_at<uint32_t>(static_cast<const uint32_t*>(main_dict), dict_len,
                              static_cast<const uint32_t*>(delta), n_delta, static_cast<const uint32_t*>(values),
                              n_values, codes, merged_len);
  if (key_bytes == 16)
    return codes_at<K16>(static_cast<const K16*>(main_dict), dict_len, static_cast<const K16*>(delta), n_delta,
                         static_cast<const K16*>(values), n_values, codes, merged_len);
  return DMO_E_INVALID;
}

}  // extern "C"
