// dictmerge.cu -- host side of libdictmerge: the C ABI (include/dictmerge.h),
// argument validation, workspace layout, stream-ordered orchestration of the
// three kernel families, the wide-table entry point and the host-buffer
// context.  Every step of the merge runs in the kernels of delta_dict.cu,
// dict_merge.cu and recompress.cu; this file only plans and launches.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "dm_internal.h"

namespace dm {

static std::atomic<uint64_t> g_launches{0};
static std::atomic<int> g_last_cuda{0};

void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

bool pdl_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("DM_PDL");
    return !(e && e[0] == '0');
  }();
  return v;
}

namespace {
std::mutex g_cache_mu;
struct FuncKey {
  const void* f;
  int dev;
  size_t smem;
  int threads;
  bool operator<(const FuncKey& o) const {
    return std::tie(f, dev, smem, threads) < std::tie(o.f, o.dev, o.smem, o.threads);
  }
};
std::map<FuncKey, int> g_func_cache;
int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
}  // namespace

void ensure_smem(const void* func, bool max_carveout) {
  const FuncKey k{func, current_device(), 0, max_carveout ? -3 : -1};
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (g_func_cache.count(k)) return;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, k.dev);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, func);
  cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  // Full shared-memory carveout on request: otherwise the driver may pick a
  // smaller split and cap residency (k_merge_write ran 3 CTAs/SM instead of 5,
  // ncu r01).  Not for the gather kernels: k_recompress's L2 gathers need the
  // L1 capacity (measured 440 -> 787 us on cfg2 with the full carveout).
  if (max_carveout)
    cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  g_func_cache[k] = 1;
}

int device_sms() {
  const FuncKey k{nullptr, current_device(), 0, -2};
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_func_cache.find(k);
  if (it != g_func_cache.end()) return it->second;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, k.dev);
  g_func_cache[k] = sms;
  return sms;
}

int occupancy(const void* func, int threads, size_t smem) {
  ensure_smem(func);
  const FuncKey k{func, current_device(), smem, threads};
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_func_cache.find(k);
  if (it != g_func_cache.end()) return it->second;
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, func, threads, smem);
  if (occ < 1) occ = 1;
  g_func_cache[k] = occ;
  return occ;
}

uint32_t host_width(uint64_t n) {
  // Eq 4: ceil(log2 n), with a 1-bit minimum (reading A1).
  uint32_t w = 1;
  while (w < 64 && (1ull << w) < n) ++w;
  return w;
}
uint64_t host_words(uint64_t n, uint32_t bits) { return (n * (uint64_t)bits + 63) / 64; }

// Knob defaults may come from the environment (DM_XMODE for knob 0; experiments).
static int env_knob(const char* name, int hi) {
  const char* s = std::getenv(name);
  const int v = s ? std::atoi(s) : 0;
  return (v >= 0 && v <= hi) ? v : 0;
}
static std::atomic<int> g_tuning[8] = {env_knob("DM_XMODE", 3), env_knob("DM_MERGE", 2), env_knob("DM_DEDUP", 2),
                                       env_knob("DM_STEP2", 1), env_knob("DM_XC_SHIFT", 8), env_knob("DM_SORT1A", 2),
                                       env_knob("DM_TPG", 1), env_knob("DM_SP_GRID", 2)};
int tuning(int knob) { return (knob >= 0 && knob < 8) ? g_tuning[knob].load(std::memory_order_relaxed) : 0; }

static thread_local int t_xc_shift = 0;
void set_xc_shift_override(int xs) { t_xc_shift = xs; }
int xc_shift_override() {
  if (t_xc_shift) return t_xc_shift;  // this thread's sharded Step 1(b): one shift for all ranges
  const int x = tuning(4);  // knob 4 (DM_XC_SHIFT)
  return (x == 7 || x == 8) ? x : 0;
}

int sort_variant() {
  static const int v = [] {
    const char* s = std::getenv("DM_SORT_CFG");
    const int x = s ? std::atoi(s) : 0;
    return (x >= 0 && x < 4) ? x : 0;
  }();
  return v;
}

uint64_t sort_tile_keys(int key) {
  const SortShape& s = kSortShapes[sort_variant()];
  return (uint64_t)s.threads * (key == DM_KEY_B16 ? s.items_b16 : s.items_u64);
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

WsLayout ws_layout(const dm_column_in* in) {
  WsLayout L{};
  const size_t E = key_bytes(in->key);
  const uint64_t nD = in->n_delta;
  L.npass = (int)E;
  const uint64_t sort_tile = sort_tile_keys(in->key);
  L.ntiles_sort = (nD + sort_tile - 1) / sort_tile;
  L.ntiles_unique = (nD + kUniqThreads * kUniqItems - 1) / (kUniqThreads * kUniqItems);
  L.ntiles_merge = std::max<uint64_t>(1, (in->dict_len + nD + kMergeTile - 1) / kMergeTile);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  L.hdr = take(sizeof(dm_header));
  L.counters = take(64 * sizeof(uint32_t));
  L.hist = take(16 * 256 * sizeof(uint32_t));
  L.status_sort = take((size_t)L.npass * L.ntiles_sort * 256 * sizeof(uint32_t));
  L.status_unique = take(L.ntiles_unique * sizeof(uint64_t));
  L.status_merge = take((L.ntiles_merge + 1) * sizeof(uint64_t));  // per tile (single-pass look-back)
  L.bucket = bucket_wanted(in);
  L.bk_bits = L.bucket ? bucket_bits(nD) : 0;
  if (L.bucket) {
    L.bk_state = take(sizeof(BucketState));
    L.bk_status = take(((1ull << L.bk_bits) / (256 * kBkScanItems) + 1) * sizeof(uint64_t));
  }
  if (probe_possible(in)) L.pf_used = take(((in->dict_len + 31) / 32) * 4);
  L.zero_bytes = o;
  L.plan = take(sizeof(SortPlan));
  L.keys0 = take(nD * E);
  L.keys1 = take(nD * E);
  L.vals0 = take(nD * 4);
  L.vals1 = take(nD * 4);
  L.udict = take(nD * E);
  L.rank = take(nD * 4);
  L.part = take((L.ntiles_merge + 1) * sizeof(uint64_t));
  L.mcount = take(L.ntiles_merge * sizeof(uint32_t));
  L.mexcl = take(L.ntiles_merge * sizeof(uint64_t));
  L.xm = take(in->dict_len * 4);
  L.xd = take(nD * 4);
  L.xc_rblk = take((xc_nblk(in->dict_len, kXcMinShift) + 1) * 4);  // sized for the smallest blocks
  L.xc_rec = take(xc_nsb(in->dict_len, kXcMinShift) * kXcRecBytes);
  L.xc_offs = take(nD + 16);
  if (L.bucket) {
    L.bk_off = take(((1ull << L.bk_bits) + 1) * 4);
    if (E <= 8) L.bk_pairs = take(nD * 16);
    L.bk_cur = take((1ull << L.bk_bits) * 4);
  }
  L.probe = probe_possible(in);
  if (L.probe) {
    L.pf_src = take(nD * 4);
    L.pf_keys = take(nD * E);
    L.pf_rank = take(nD * 4);
    L.pf_codes = take(nD * 4);
    uint64_t cap = 1024;  // load factor <= 1/4: a warp's longest probe chain stays short
    while (cap < 4 * in->dict_len) cap <<= 1;
    L.pf_cap = cap;
    L.pf_table = take(cap * 4);
  }
  L.dedup = dedup_wanted(in);
  if (L.dedup) {
    uint64_t cap = 1024;
    while (cap < 2 * nD) cap <<= 1;
    L.dd_cap = cap;
    L.dd_slots = take(cap * 8);
    L.dd_keys = take(nD * E);
    L.dd_tid = take(nD * 4);
    L.dd_rank = take(nD * 4);
  }
  L.total = o;
  return L;
}

cudaError_t last_error_check() { return cudaGetLastError(); }

static dm_status cuda_fail(cudaError_t e) {
  g_last_cuda.store((int)e);
  return DM_E_CUDA;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// One NVTX range at a time, popped on every exit path.
struct NvtxSteps {
  bool open = false;
  void next(const char* name) {
    if (open) nvtxRangePop();
    open = name != nullptr;
    if (open) nvtxRangePushA(name);
  }
  ~NvtxSteps() {
    if (open) nvtxRangePop();
  }
};
// Main codes index a dictionary: with N_M > 0, 1 <= |U_M| < 2^32 and b >= width(|U_M|)
// (the recompress kernels clamp codes to |U_M| - 1, so |U_M| = 0 must not reach them).
static bool main_dict_len_ok(uint64_t n_main, uint64_t dict_len, uint32_t main_bits) {
  if (n_main == 0) return dict_len < (1ull << 32);
  return dict_len >= 1 && dict_len < (1ull << 32) && main_bits >= host_width(dict_len);
}

// What one call runs: the whole merge, Steps 1(a)-2(a), Step 1(a) alone, or
// Steps 1(b)-2(a) on a delta that already is U_D (sorted, distinct).
enum MergeMode { MM_FULL = 0, MM_DICT = 1, MM_DELTA = 2, MM_SORTED_DICT = 3 };

static dm_status validate(const dm_column_in* in, const dm_column_out* out, int mode = MM_FULL) {
  const bool with_step2 = mode == MM_FULL;
  if (!in || !out) return DM_E_INVALID;
  if (in->key != DM_KEY_U64 && in->key != DM_KEY_B16 && in->key != DM_KEY_U32) return DM_E_INVALID;
  if (in->main_bits < 1 || in->main_bits > 32) return DM_E_INVALID;
  if (in->dict_len >= (1ull << 32)) return DM_E_INVALID;
  if (in->n_delta >= (1ull << 30)) return DM_E_INVALID;
  if (in->n_main > 0 && in->dict_len == 0) return DM_E_INVALID;
  if (in->dict_len > 0 && in->main_bits < host_width(in->dict_len)) return DM_E_INVALID;
  if (in->dict_len && (!in->main_dict || !aligned16(in->main_dict))) return DM_E_INVALID;
  if (with_step2 && in->n_main && (!in->main_codes || !aligned16(in->main_codes))) return DM_E_INVALID;
  if (in->n_delta && (!in->delta || !aligned16(in->delta))) return DM_E_INVALID;
  const uint64_t dict_cap = in->dict_len + in->n_delta;
  if (dict_cap > (1ull << 32)) return DM_E_TOO_WIDE;  // |U'| <= |U_M| + N_D must stay <= 2^32
  if (dict_cap && (!out->merged_dict || !aligned16(out->merged_dict))) return DM_E_INVALID;
  if (out->merged_dict_cap < dict_cap) return DM_E_CAPACITY;
  if (with_step2) {
    const uint64_t need_words = dm_merged_codes_cap_words(in);
    if (need_words && (!out->merged_codes || !aligned16(out->merged_codes))) return DM_E_INVALID;
    if (out->merged_codes_cap_words < need_words) return DM_E_CAPACITY;
  } else if (mode == MM_DICT) {
    if (in->dict_len && !out->x_main) return DM_E_INVALID;
    if (in->n_delta && (!out->x_delta || !out->delta_rank)) return DM_E_INVALID;
  } else if (mode == MM_DELTA) {
    if (in->n_delta && (!out->delta_dict || !out->delta_rank)) return DM_E_INVALID;
  } else {  // MM_SORTED_DICT
    if (in->dict_len && !out->x_main) return DM_E_INVALID;
    if (in->n_delta && !out->x_delta) return DM_E_INVALID;
  }
  if (out->delta_dict && !aligned16(out->delta_dict)) return DM_E_INVALID;
  return DM_OK;
}

static dm_status merge_async(const dm_column_in* in, const dm_column_out* out, void* ws, size_t ws_bytes,
                             dm_header* d_header, cudaStream_t st, bool zero_header,
                             void* const* events = nullptr, int mode = MM_FULL) {
  const bool with_step2 = mode == MM_FULL;
  dm_status v = validate(in, out, mode);
  if (v != DM_OK) return v;
  const WsLayout L = ws_layout(in);
  if (!ws || ws_bytes < L.total) return DM_E_CAPACITY;
  if (!d_header || !aligned16(d_header)) return DM_E_INVALID;
  char* w = static_cast<char*>(ws);
  // NVTX ranges per step (host enqueue spans; nsys / ncu timelines show them)
  static const char* const kStepNames[3] = {"dm Step 1(a) delta dictionary (P:181, P:218-222)",
                                            "dm Step 1(b) dictionary merge + 2(a) width (P:192, P:224-226, Eq 4)",
                                            "dm Step 2(b) recompress (Eq 11, P:272)"};
  NvtxSteps nv;
  auto mark = [&](int i) {
    if (events && events[i]) cudaEventRecord(static_cast<cudaEvent_t>(events[i]), st);
    nv.next(i < 3 ? kStepNames[i] : nullptr);
  };
  mark(0);
  cudaError_t e = cudaMemsetAsync(w, 0, L.zero_bytes, st);
  if (e == cudaSuccess && L.dedup) e = cudaMemsetAsync(w + L.dd_slots, 0, L.dd_cap * 8, st);
  if (e == cudaSuccess && zero_header) e = cudaMemsetAsync(d_header, 0, sizeof(dm_header), st);
  if (e != cudaSuccess) return cuda_fail(e);
  void* udict = out->delta_dict ? out->delta_dict : (void*)(w + L.udict);
  uint32_t* rank = out->delta_rank ? out->delta_rank : reinterpret_cast<uint32_t*>(w + L.rank);
  uint32_t* xm = out->x_main ? out->x_main : reinterpret_cast<uint32_t*>(w + L.xm);
  uint32_t* xd = out->x_delta ? out->x_delta : reinterpret_cast<uint32_t*>(w + L.xd);
  // DM_SYNC_DEBUG=1: synchronise after each step and report which one faulted (debugging only)
  static const bool sync_debug = std::getenv("DM_SYNC_DEBUG") != nullptr;
  auto dbg = [&](const char* step) -> cudaError_t {
    if (!sync_debug) return cudaSuccess;
    cudaError_t x = cudaStreamSynchronize(st);
    if (x != cudaSuccess) fprintf(stderr, "dictmerge: %s failed: %s\n", step, cudaGetErrorString(x));
    return x;
  };
  // Step 1(a): delta dictionary U_D and ranks r -- or, for a
  // delta that already is U_D (the paper reads it off the CSB+ tree's leaves,
  // P:190), just its length.
  // probe-first (NEXT1) only when nobody asked for U_D / X_D / r, whose index space it skips
  const bool probe = L.probe && mode == MM_FULL && !out->delta_dict && !out->x_delta && !out->delta_rank;
  if (mode == MM_SORTED_DICT) {
    udict = const_cast<void*>(in->delta);
    if ((e = launch_set_delta_len(d_header, in->n_delta, st)) != cudaSuccess) return cuda_fail(e);
  } else if ((e = launch_delta_dictionary(in, w, L, udict, rank, d_header, st, probe)) != cudaSuccess) {
    return cuda_fail(e);
  }
  if ((e = dbg("step 1(a)")) != cudaSuccess) return cuda_fail(e);
  mark(1);
  if (mode == MM_DELTA) return DM_OK;
  // Step 1(b) + 2(a): U', X_M, X_D, b' (Eq 4).
  // (probe-first needs the plain X_M: the found tuples' codes come from it)
  if ((e = launch_dictionary_merge(in, out, w, L, udict, xm, xd, d_header, st, !with_step2, probe)) != cudaSuccess)
    return cuda_fail(e);
  if (probe && (e = launch_probe_codes(in, w, L, xm, xd, d_header, st)) != cudaSuccess) return cuda_fail(e);
  if ((e = dbg("step 1(b)")) != cudaSuccess) return cuda_fail(e);
  mark(2);
  // Step 2(b): M' (Eq 11).
  const bool xc = xc_wanted(in);
  if (with_step2 && tuning(3) == 1) {
    if ((e = launch_naive_step2(in, out, d_header, st)) != cudaSuccess) return cuda_fail(e);
  } else if (with_step2 && (e = launch_recompress(in, out, xm, probe ? reinterpret_cast<const uint32_t*>(w + L.pf_codes) : xd,
                                                  probe ? nullptr : rank, d_header, st, 0,
                                           xc ? reinterpret_cast<const uint2*>(w + L.xc_rec) : nullptr,
                                           xc ? reinterpret_cast<const uint8_t*>(w + L.xc_offs) : nullptr,
                                           xc_shift(in))) !=
                         cudaSuccess)
    return cuda_fail(e);
  mark(3);
  return DM_OK;
}

// Per-device pool of non-blocking streams used by dm_merge_table.
// One caller at a time forks / joins a pool (`mu`): the fork and join events
// are shared, so two host threads (or interleaved captures) on one device must
// not interleave their record / wait pairs.
struct StreamPool {
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> join;
  cudaEvent_t fork = nullptr;
  std::mutex mu;
};
// Stream-pool size for dm_merge_table (DM_TABLE_STREAMS overrides; experiments).
static int table_streams() {
  static const int v = [] {
    const char* e = std::getenv("DM_TABLE_STREAMS");
    const int x = e ? std::atoi(e) : 16;
    return (x >= 1 && x <= 128) ? x : 16;
  }();
  return v;
}

static StreamPool& stream_pool() {
  static std::mutex mu;
  static std::map<int, StreamPool> pools;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  StreamPool& p = pools[dev];
  if (p.streams.empty()) {
    cudaEventCreateWithFlags(&p.fork, cudaEventDisableTiming);
    for (int k = 0; k < table_streams(); ++k) {
      cudaStream_t s;
      cudaEvent_t e;
      if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) break;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      p.streams.push_back(s);
      p.join.push_back(e);
    }
  }
  return p;
}

struct dm_ctx_impl {
  int device = 0;
  cudaStream_t stream = nullptr;    // compute
  cudaStream_t s_in = nullptr;      // host -> device copies
  cudaStream_t s_out = nullptr;     // device -> host copies
  std::vector<cudaEvent_t> events;  // pipeline events, grown on demand
  cudaEvent_t event(size_t i) {
    while (events.size() <= i) {
      cudaEvent_t e = nullptr;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      events.push_back(e);
    }
    return events[i];
  }
  std::vector<std::pair<void*, size_t>> bufs;  // device buffers, grown on demand
  dm_header* host_hdr = nullptr;                // pinned
  void* get(int slot, size_t bytes) {
    if ((int)bufs.size() <= slot) bufs.resize(slot + 1, {nullptr, 0});
    auto& b = bufs[slot];
    if (b.second < bytes) {
      if (b.first) cudaFree(b.first);
      b.first = nullptr;
      b.second = 0;
      if (cudaMalloc(&b.first, std::max<size_t>(bytes, 256)) != cudaSuccess) return nullptr;
      b.second = std::max<size_t>(bytes, 256);
    }
    return b.first;
  }
};

}  // namespace dm

using namespace dm;

struct dm_ctx {
  dm_ctx_impl impl;
};

extern "C" {

int dm_set_tuning(int knob, int value) {
  static const int hi[8] = {3, 3, 3, 1, 8, 2, 1, 2};
  if (knob < 0 || knob > 7 || value < 0 || value > hi[knob]) return DM_E_INVALID;
  if (knob == 4 && value != 0 && value != 7 && value != 8) return DM_E_INVALID;
  g_tuning[knob].store(value);
  return DM_OK;
}

int dm_get_tuning(int knob) { return (knob >= 0 && knob < 8) ? tuning(knob) : DM_E_INVALID; }

uint32_t dm_width(uint64_t n) { return host_width(n); }
uint64_t dm_words(uint64_t n, uint32_t bits) { return host_words(n, bits); }

uint64_t dm_merged_codes_cap_words(const dm_column_in* in) {
  if (!in) return 0;
  return host_words(in->n_main + in->n_delta, std::min<uint32_t>(32, host_width(in->dict_len + in->n_delta)));
}

size_t dm_workspace_bytes(const dm_column_in* in) { return in ? ws_layout(in).total : 0; }

dm_status dm_merge_column_async(const dm_column_in* in, const dm_column_out* out, void* ws, size_t ws_bytes,
                                dm_header* d_header, void* cuda_stream) {
  return merge_async(in, out, ws, ws_bytes, d_header, static_cast<cudaStream_t>(cuda_stream), true);
}

dm_status dm_merge_column_async_ev(const dm_column_in* in, const dm_column_out* out, void* ws, size_t ws_bytes,
                                   dm_header* d_header, void* cuda_stream, void* const* events) {
  return merge_async(in, out, ws, ws_bytes, d_header, static_cast<cudaStream_t>(cuda_stream), true, events);
}

dm_status dm_merge_column(const dm_column_in* in, dm_column_out* out, void* ws, size_t ws_bytes, void* cuda_stream) {
  if (!in) return DM_E_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const WsLayout L = ws_layout(in);
  if (!ws || ws_bytes < L.total) return DM_E_CAPACITY;
  dm_header* d_hdr = reinterpret_cast<dm_header*>(static_cast<char*>(ws) + L.hdr);
  dm_status s = merge_async(in, out, ws, ws_bytes, d_hdr, st, false);  // header lives in the zeroed zone
  if (s != DM_OK) return s;
  dm_header h{};
  cudaError_t e = cudaMemcpyAsync(&h, d_hdr, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e);
  out->merged_dict_len = h.merged_dict_len;
  out->delta_dict_len = h.delta_dict_len;
  out->merged_bits = h.merged_bits;
  return (dm_status)h.status;
}

dm_status dm_merge_table(int ncols, const dm_column_in* in, dm_column_out* out, void* const* ws,
                         const size_t* ws_bytes, void* cuda_stream) {
  if (ncols < 0 || (ncols > 0 && (!in || !out || !ws || !ws_bytes))) return DM_E_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  // Each column is merged separately; the columns are independent
  // tasks.  The GPU form of the paper's task queue: columns, largest
  // first, are dealt round-robin onto a pool of streams forked from (and joined
  // back into) the caller's stream, so one column's latency-bound Step 1
  // kernels overlap other columns' streaming Step 2.
  std::vector<dm_header*> hdrs(ncols);
  for (int c = 0; c < ncols; ++c) {
    const WsLayout L = ws_layout(&in[c]);
    if (!ws[c] || ws_bytes[c] < L.total) return DM_E_CAPACITY;
    hdrs[c] = reinterpret_cast<dm_header*>(static_cast<char*>(ws[c]) + L.hdr);
  }
  dm_status s0 = dm_merge_table_async(ncols, in, out, ws, ws_bytes, hdrs.data(), cuda_stream);
  if (s0 != DM_OK) return s0;
  cudaError_t e = cudaSuccess;
  std::vector<dm_header> h(ncols);
  for (int c = 0; c < ncols && e == cudaSuccess; ++c)
    e = cudaMemcpyAsync(&h[c], hdrs[c], sizeof(dm_header), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e);
  int status = DM_OK;
  for (int c = 0; c < ncols; ++c) {
    out[c].merged_dict_len = h[c].merged_dict_len;
    out[c].delta_dict_len = h[c].delta_dict_len;
    out[c].merged_bits = h[c].merged_bits;
    status = std::min(status, (int)h[c].status);
  }
  return (dm_status)status;
}

dm_status dm_merge_table_async(int ncols, const dm_column_in* in, const dm_column_out* out, void* const* ws,
                               const size_t* ws_bytes, dm_header* const* hdrs, void* cuda_stream) {
  if (ncols < 0 || (ncols > 0 && (!in || !out || !ws || !ws_bytes || !hdrs))) return DM_E_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  for (int c = 0; c < ncols; ++c) {
    dm_status v = validate(&in[c], &out[c]);
    if (v != DM_OK) return v;
    if (!ws[c] || ws_bytes[c] < ws_layout(&in[c]).total) return DM_E_CAPACITY;
  }
  std::vector<int> order(ncols);
  for (int c = 0; c < ncols; ++c) order[c] = c;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return in[a].n_main + in[a].n_delta > in[b].n_main + in[b].n_delta;
  });
  StreamPool& pool = stream_pool();
  std::lock_guard<std::mutex> lk(pool.mu);
  const int K = std::max(1, std::min<int>(ncols, (int)pool.streams.size()));
  cudaError_t e = cudaEventRecord(pool.fork, st);
  for (int k = 0; k < K && e == cudaSuccess; ++k) e = cudaStreamWaitEvent(pool.streams[k], pool.fork, 0);
  if (e != cudaSuccess) return cuda_fail(e);
  dm_status bad = DM_OK;
  set_table_merge(ncols > 1);
  for (int t = 0; t < ncols && bad == DM_OK; ++t) {
    const int c = order[t];
    bad = merge_async(&in[c], &out[c], ws[c], ws_bytes[c], hdrs[c], pool.streams[t % K], true);
  }
  set_table_merge(false);
  // always join every forked stream back (an active graph capture must not end
  // with forked streams, even when a column failed to launch)
  for (int k = 0; k < K; ++k) {
    cudaError_t j = cudaEventRecord(pool.join[k], pool.streams[k]);
    if (j == cudaSuccess) j = cudaStreamWaitEvent(st, pool.join[k], 0);
    if (e == cudaSuccess) e = j;
  }
  if (bad != DM_OK) return bad;
  return e == cudaSuccess ? DM_OK : cuda_fail(e);
}

dm_status dm_dictionary_merge_async(const dm_column_in* in, const dm_column_out* out, void* ws, size_t ws_bytes,
                                    dm_header* d_header, void* cuda_stream) {
  return merge_async(in, out, ws, ws_bytes, d_header, static_cast<cudaStream_t>(cuda_stream), true, nullptr,
                     MM_DICT);
}

dm_status dm_delta_dictionary_async(const dm_column_in* in, const dm_column_out* out, void* ws, size_t ws_bytes,
                                    dm_header* d_header, void* cuda_stream) {
  return merge_async(in, out, ws, ws_bytes, d_header, static_cast<cudaStream_t>(cuda_stream), true, nullptr,
                     MM_DELTA);
}

dm_status dm_dictionary_merge_sorted_async(const dm_column_in* in, const dm_column_out* out, void* ws,
                                           size_t ws_bytes, dm_header* d_header, void* cuda_stream) {
  return merge_async(in, out, ws, ws_bytes, d_header, static_cast<cudaStream_t>(cuda_stream), true, nullptr,
                     MM_SORTED_DICT);
}

dm_status dm_lower_bound_async(int key, const void* sorted, uint64_t n, const void* values, uint64_t n_values,
                               uint64_t* pos, void* cuda_stream) {
  if (key != DM_KEY_U64 && key != DM_KEY_B16 && key != DM_KEY_U32) return DM_E_INVALID;
  if (n_values && (!values || !pos || (n && !sorted))) return DM_E_INVALID;
  cudaError_t e = launch_lower_bound(key, sorted, n, values, n_values, pos, static_cast<cudaStream_t>(cuda_stream));
  return e == cudaSuccess ? DM_OK : cuda_fail(e);
}

dm_status dm_rebase_async(uint32_t* x, uint64_t n, uint32_t add, void* cuda_stream) {
  if (n && !x) return DM_E_INVALID;
  cudaError_t e = launch_add_u32(x, n, add, static_cast<cudaStream_t>(cuda_stream));
  return e == cudaSuccess ? DM_OK : cuda_fail(e);
}

dm_status dm_xc_rebase_async(void* records, uint64_t n_records, uint32_t add, void* cuda_stream) {
  if (n_records && (!records || !aligned16(records))) return DM_E_INVALID;
  cudaError_t e = launch_xc_rebase(records, n_records, add, static_cast<cudaStream_t>(cuda_stream));
  return e == cudaSuccess ? DM_OK : cuda_fail(e);
}

dm_status dm_recompress(const uint64_t* main_codes, uint64_t n_main, uint32_t main_bits, uint64_t dict_len,
                        const uint32_t* x_main, const uint32_t* x_delta, const uint32_t* delta_rank,
                        uint64_t n_delta, uint32_t new_bits, uint64_t* out_codes, uint64_t out_cap_words,
                        void* cuda_stream) {
  if (main_bits < 1 || main_bits > 32 || new_bits < 1 || new_bits > 32) return DM_E_INVALID;
  if (!main_dict_len_ok(n_main, dict_len, main_bits)) return DM_E_INVALID;
  if (n_main && (!main_codes || !x_main || !aligned16(main_codes))) return DM_E_INVALID;
  if (n_delta && (!x_delta || !delta_rank)) return DM_E_INVALID;
  const uint64_t need = host_words(n_main + n_delta, new_bits);
  if (need && (!out_codes || !aligned16(out_codes))) return DM_E_INVALID;
  if (out_cap_words < need) return DM_E_CAPACITY;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  dm_header* d_hdr = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d_hdr), sizeof(dm_header), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_hdr, 0, sizeof(dm_header), st);
  if (e != cudaSuccess) return cuda_fail(e);
  dm_column_in in{};
  in.key = DM_KEY_U64;
  in.dict_len = dict_len;
  in.main_codes = main_codes;
  in.n_main = n_main;
  in.main_bits = main_bits;
  in.n_delta = n_delta;
  dm_column_out out{};
  out.merged_codes = out_codes;
  out.merged_codes_cap_words = out_cap_words;
  e = launch_recompress(&in, &out, x_main, x_delta, delta_rank, d_hdr, st, new_bits);
  dm_header h{};
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d_hdr, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_hdr, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e);
  return (dm_status)h.status;
}

dm_status dm_xc_export(const dm_column_in* in, const void* ws, size_t ws_bytes, dm_xc* xc) {
  if (!in || !xc) return DM_E_INVALID;
  const WsLayout L = ws_layout(in);
  if (!ws || ws_bytes < L.total) return DM_E_CAPACITY;
  const char* w = static_cast<const char*>(ws);
  const uint32_t xs = xc_shift(in);
  xc->records = w + L.xc_rec;
  xc->n_records = xc_nsb(in->dict_len, xs);
  xc->offsets = reinterpret_cast<const uint8_t*>(w + L.xc_offs);
  xc->offsets_cap = in->n_delta + 16;
  xc->shift = xs;
  xc->built = in->dict_len > 0 ? 1 : 0;  // dictionary-only merges always build it
  return DM_OK;
}

dm_status dm_xc_exceptions_gather(const dm_xc* xc, uint64_t dict_len, const uint32_t* x_main, uint32_t* ids,
                                  uint32_t* slices, uint64_t* d_count, void* cuda_stream) {
  if (!xc || !xc->records || (xc->shift != 7 && xc->shift != 8) || !d_count) return DM_E_INVALID;
  if ((ids == nullptr) != (slices == nullptr)) return DM_E_INVALID;  // both NULL: count only
  if (xc->n_records && slices && !x_main) return DM_E_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  cudaError_t e = cudaMemsetAsync(d_count, 0, sizeof(uint64_t), st);
  if (e == cudaSuccess)
    e = launch_xc_exceptions(true, static_cast<const uint2*>(xc->records), xc->n_records, xc->shift, dict_len,
                             const_cast<uint32_t*>(x_main), ids, slices,
                             reinterpret_cast<unsigned long long*>(d_count), 0, st);
  return e == cudaSuccess ? DM_OK : cuda_fail(e);
}

dm_status dm_xc_exceptions_scatter(const dm_xc* xc, uint64_t dict_len, const uint32_t* ids, const uint32_t* slices,
                                   uint64_t count, uint32_t* x_main, void* cuda_stream) {
  if (!xc || (xc->shift != 7 && xc->shift != 8)) return DM_E_INVALID;
  if (count && (!x_main || !ids || !slices)) return DM_E_INVALID;
  cudaError_t e = launch_xc_exceptions(false, nullptr, xc->n_records, xc->shift, dict_len, x_main,
                                       const_cast<uint32_t*>(ids), const_cast<uint32_t*>(slices), nullptr, count,
                                       static_cast<cudaStream_t>(cuda_stream));
  return e == cudaSuccess ? DM_OK : cuda_fail(e);
}

dm_status dm_recompress_xc(const uint64_t* main_codes, uint64_t n_main, uint32_t main_bits, uint64_t dict_len,
                           const dm_xc* xc, const uint32_t* x_main, const uint32_t* x_delta,
                           const uint32_t* delta_rank, uint64_t n_delta, uint32_t new_bits, uint64_t* out_codes,
                           uint64_t out_cap_words, void* cuda_stream) {
  if (main_bits < 1 || main_bits > 32 || new_bits < 1 || new_bits > 32) return DM_E_INVALID;
  if (!main_dict_len_ok(n_main, dict_len, main_bits)) return DM_E_INVALID;
  if (!xc || !xc->built || (xc->shift != 7 && xc->shift != 8)) return DM_E_INVALID;
  if (xc->n_records != xc_nsb(dict_len, xc->shift)) return DM_E_INVALID;
  if (n_main && (!main_codes || !x_main || !xc->records || !xc->offsets || !aligned16(main_codes) ||
                 !aligned16(xc->records) || !aligned16(xc->offsets)))
    return DM_E_INVALID;
  if (n_delta && (!x_delta || !delta_rank)) return DM_E_INVALID;
  const uint64_t need = host_words(n_main + n_delta, new_bits);
  if (need && (!out_codes || !aligned16(out_codes))) return DM_E_INVALID;
  if (out_cap_words < need) return DM_E_CAPACITY;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  dm_header* d_hdr = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d_hdr), sizeof(dm_header), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_hdr, 0, sizeof(dm_header), st);
  if (e != cudaSuccess) return cuda_fail(e);
  dm_column_in in{};
  in.key = DM_KEY_U64;
  in.dict_len = dict_len;
  in.main_codes = main_codes;
  in.n_main = n_main;
  in.main_bits = main_bits;
  in.n_delta = n_delta;
  dm_column_out out{};
  out.merged_codes = out_codes;
  out.merged_codes_cap_words = out_cap_words;
  e = launch_recompress_xc(&in, &out, x_main, x_delta, delta_rank, d_hdr, st, new_bits,
                           static_cast<const uint2*>(xc->records), xc->offsets, xc->shift);
  dm_header h{};
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d_hdr, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_hdr, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e);
  return (dm_status)h.status;
}

dm_status dm_pack_codes(const uint32_t* codes, uint64_t n, uint32_t bits, uint64_t* words, void* cuda_stream) {
  if (bits < 1 || bits > 32) return DM_E_INVALID;
  if (n && (!codes || !words)) return DM_E_INVALID;
  cudaError_t e = launch_pack(codes, n, bits, words, static_cast<cudaStream_t>(cuda_stream));
  return e == cudaSuccess ? DM_OK : cuda_fail(e);
}

dm_status dm_unpack_codes(const uint64_t* words, uint64_t n, uint32_t bits, uint32_t* codes, void* cuda_stream) {
  if (bits < 1 || bits > 32) return DM_E_INVALID;
  if (n && (!codes || !words)) return DM_E_INVALID;
  cudaError_t e = launch_unpack(words, n, bits, codes, static_cast<cudaStream_t>(cuda_stream));
  return e == cudaSuccess ? DM_OK : cuda_fail(e);
}

dm_ctx* dm_ctx_create(int device) {
  if (cudaSetDevice(device) != cudaSuccess) return nullptr;
  dm_ctx* c = new dm_ctx();
  c->impl.device = device;
  if (cudaStreamCreateWithFlags(&c->impl.stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->impl.s_in, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->impl.s_out, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMallocHost(&c->impl.host_hdr, sizeof(dm_header)) != cudaSuccess) {
    delete c;
    return nullptr;
  }
  return c;
}

void dm_ctx_destroy(dm_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->impl.device);
  for (auto& b : c->impl.bufs)
    if (b.first) cudaFree(b.first);
  if (c->impl.host_hdr) cudaFreeHost(c->impl.host_hdr);
  if (c->impl.stream) cudaStreamDestroy(c->impl.stream);
  if (c->impl.s_in) cudaStreamDestroy(c->impl.s_in);
  if (c->impl.s_out) cudaStreamDestroy(c->impl.s_out);
  for (cudaEvent_t ev : c->impl.events) cudaEventDestroy(ev);
  delete c;
}

// dm_merge_column_host's checks of the caller's HOST buffers: the same argument
// rules as the device entry points (validate), minus alignment, and output
// capacities that fit every possible result.
static dm_status validate_host(const dm_column_in* in, const dm_column_out* out) {
  if (in->key != DM_KEY_U64 && in->key != DM_KEY_B16 && in->key != DM_KEY_U32) return DM_E_INVALID;
  if (in->main_bits < 1 || in->main_bits > 32) return DM_E_INVALID;
  if (in->dict_len >= (1ull << 32) || in->n_delta >= (1ull << 30)) return DM_E_INVALID;
  if (!main_dict_len_ok(in->n_main, in->dict_len, in->main_bits)) return DM_E_INVALID;
  if (in->dict_len && !in->main_dict) return DM_E_INVALID;
  if (in->n_main && !in->main_codes) return DM_E_INVALID;
  if (in->n_delta && !in->delta) return DM_E_INVALID;
  const uint64_t dict_cap = in->dict_len + in->n_delta;
  if (dict_cap > (1ull << 32)) return DM_E_TOO_WIDE;
  if (dict_cap && !out->merged_dict) return DM_E_INVALID;
  if (out->merged_dict_cap < dict_cap) return DM_E_CAPACITY;
  const uint64_t need_words = dm_merged_codes_cap_words(in);
  if (need_words && !out->merged_codes) return DM_E_INVALID;
  if (out->merged_codes_cap_words < need_words) return DM_E_CAPACITY;
  return DM_OK;
}

dm_status dm_merge_column_host(dm_ctx* c, const dm_column_in* hin, dm_column_out* hout) {
  // A three-stream pipeline (copy-in, compute, copy-out; B200 has separate copy
  // engines per direction, PCIe is full duplex):
  //   in:      U_M, D  |  M chunk 0 | M chunk 1 | ...
  //   compute:           Steps 1(a)-2(a) | Step 2(b) chunk 0 | chunk 1 | ...
  //   out:                               U' (X_M ...) | M' chunk 0 | chunk 1 | ...
  // Step 2(b) of a row chunk needs only its M words and the translation tables
  // (Eq 11, P:272 is row-local; the paper splits N' over threads the same way,
  // P:324), so the main-code upload overlaps Step 1 and the M' download
  // overlaps the remaining uploads.  One host wait: for b' after Step 2(a).
  if (!c || !hin || !hout) return DM_E_INVALID;
  {  // the host buffers: inputs present, outputs present and large enough (before any copy)
    dm_status v = validate_host(hin, hout);
    if (v != DM_OK) return v;
  }
  cudaSetDevice(c->impl.device);
  auto& I = c->impl;
  cudaStream_t st = I.stream, sin = I.s_in, sout = I.s_out;
  const size_t E = key_bytes(hin->key);
  dm_column_in din = *hin;
  dm_column_out dout = *hout;
  const uint64_t in_words = host_words(hin->n_main, hin->main_bits);
  const uint64_t cap_words = dm_merged_codes_cap_words(hin);
  enum { B_DICT, B_CODES, B_DELTA, B_UOUT, B_MOUT, B_XM, B_XD, B_UD, B_R, B_WS };
  din.main_dict = hin->dict_len ? I.get(B_DICT, hin->dict_len * E) : nullptr;
  din.main_codes = in_words ? static_cast<const uint64_t*>(I.get(B_CODES, in_words * 8)) : nullptr;
  din.delta = hin->n_delta ? I.get(B_DELTA, hin->n_delta * E) : nullptr;
  dout.merged_dict = I.get(B_UOUT, (hin->dict_len + hin->n_delta) * E);
  dout.merged_dict_cap = hin->dict_len + hin->n_delta;
  dout.merged_codes = static_cast<uint64_t*>(I.get(B_MOUT, cap_words * 8));
  dout.merged_codes_cap_words = cap_words;
  // the tables always live on the device (Step 2(b) runs per chunk from them)
  uint32_t* xm = static_cast<uint32_t*>(I.get(B_XM, std::max<uint64_t>(hin->dict_len, 1) * 4));
  uint32_t* xd = static_cast<uint32_t*>(I.get(B_XD, std::max<uint64_t>(hin->n_delta, 1) * 4));
  uint32_t* rk = static_cast<uint32_t*>(I.get(B_R, std::max<uint64_t>(hin->n_delta, 1) * 4));
  dout.x_main = xm;
  dout.x_delta = xd;
  dout.delta_rank = rk;
  dout.delta_dict = hout->delta_dict ? I.get(B_UD, hin->n_delta * E) : nullptr;
  const size_t wsb = dm_workspace_bytes(hin);
  void* ws = I.get(B_WS, wsb);
  if (!ws || !dout.merged_dict || !dout.merged_codes || !xm || !xd || !rk) return cuda_fail(cudaErrorMemoryAllocation);
  if (in_words && !hin->main_codes) return DM_E_INVALID;
  cudaError_t e = cudaSuccess;
  auto h2d = [&](const void* d, const void* h, size_t n) {
    if (n && e == cudaSuccess) e = cudaMemcpyAsync(const_cast<void*>(d), h, n, cudaMemcpyHostToDevice, sin);
  };
  auto d2h = [&](void* hp, const void* dp, size_t n) {
    if (hp && n && e == cudaSuccess) e = cudaMemcpyAsync(hp, dp, n, cudaMemcpyDeviceToHost, sout);
  };
  auto rec = [&](size_t i, cudaStream_t s) {
    if (e == cudaSuccess) e = cudaEventRecord(I.event(i), s);
  };
  auto wait = [&](cudaStream_t s, size_t i) {
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, I.event(i), 0);
  };
  // row chunks of N' at multiples of 4096 rows (word-aligned at b and b'), >= 4M rows each, <= 32
  const uint64_t n_total = hin->n_main + hin->n_delta;
  const uint64_t K = n_total ? std::max<uint64_t>(1, std::min<uint64_t>(32, n_total >> 22)) : 0;
  std::vector<uint64_t> cut(K + 1, 0);
  for (uint64_t k = 1; k < K; ++k) cut[k] = std::max(cut[k - 1], (n_total * k / K) / 4096 * 4096);
  if (K) cut[K] = n_total;
  enum { EV_DICT = 0, EV_S1 = 1, EV_IN0 = 2 };  // then EV_IN0 + k (M chunk k in), EV_IN0 + K + k (M' chunk k out)
  // 1. uploads: U_M and D first, then the main codes chunk by chunk
  h2d(din.main_dict, hin->main_dict, hin->dict_len * E);
  h2d(din.delta, hin->delta, hin->n_delta * E);
  rec(EV_DICT, sin);
  for (uint64_t k = 0; k < K; ++k) {
    const uint64_t m0 = std::min(cut[k], hin->n_main), m1 = std::min(cut[k + 1], hin->n_main);
    if (m1 > m0) {
      const uint64_t w0 = m0 * hin->main_bits / 64, w1 = host_words(m1, hin->main_bits);
      h2d(din.main_codes + w0, hin->main_codes + w0, (w1 - w0) * 8);
    }
    rec(EV_IN0 + k, sin);
  }
  if (e != cudaSuccess) return cuda_fail(e);
  // 2. Steps 1(a)-2(a) as soon as U_M and D are in
  const WsLayout L = ws_layout(hin);
  dm_header* d_hdr = reinterpret_cast<dm_header*>(static_cast<char*>(ws) + L.hdr);
  wait(st, EV_DICT);
  if (e != cudaSuccess) return cuda_fail(e);
  dm_status s = merge_async(&din, &dout, ws, wsb, d_hdr, st, false, nullptr, MM_DICT);
  if (s != DM_OK) {
    cudaStreamSynchronize(sin);
    return s;
  }
  rec(EV_S1, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(I.host_hdr, d_hdr, sizeof(dm_header), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the one host wait: |U'|, b'
  if (e != cudaSuccess) return cuda_fail(e);
  dm_header h = *I.host_hdr;
  if (h.status != DM_OK) {
    cudaStreamSynchronize(sin);
    return (dm_status)h.status;
  }
  const uint32_t nb = h.merged_bits;
  const bool xc_on = din.dict_len > 0;  // MM_DICT builds XC whenever |U_M| > 0 (force_xc)
  const uint2* xc_rec = xc_on ? reinterpret_cast<const uint2*>(static_cast<char*>(ws) + L.xc_rec) : nullptr;
  const uint8_t* xc_offs = xc_on ? reinterpret_cast<const uint8_t*>(static_cast<char*>(ws) + L.xc_offs) : nullptr;
  const uint32_t xs = xc_shift(&din);
  // 3. U' and the requested tables go out while M is still coming in
  wait(sout, EV_S1);
  d2h(hout->merged_dict, dout.merged_dict, h.merged_dict_len * E);
  d2h(hout->x_main, xm, hin->dict_len * 4);
  d2h(hout->x_delta, xd, h.delta_dict_len * 4);
  d2h(hout->delta_dict, dout.delta_dict, h.delta_dict_len * E);
  d2h(hout->delta_rank, rk, hin->n_delta * 4);
  // 4. Step 2(b) chunk by chunk, each M' chunk downloaded as soon as it is written
  for (uint64_t k = 0; k < K && e == cudaSuccess; ++k) {
    const uint64_t r0 = cut[k], r1 = cut[k + 1];
    const uint64_t m0 = std::min(r0, hin->n_main), m1 = std::min(r1, hin->n_main);
    const uint64_t d0 = std::max(r0, hin->n_main) - hin->n_main, d1 = std::max(r1, hin->n_main) - hin->n_main;
    wait(st, EV_IN0 + k);
    dm_column_in cin{};
    cin.key = hin->key;
    cin.dict_len = hin->dict_len;
    cin.main_codes = m1 > m0 ? din.main_codes + m0 * hin->main_bits / 64 : nullptr;
    cin.n_main = m1 - m0;
    cin.main_bits = hin->main_bits;
    cin.n_delta = d1 - d0;
    dm_column_out cout{};
    cout.merged_codes = dout.merged_codes + r0 * nb / 64;
    cout.merged_codes_cap_words = host_words(r1, nb) - r0 * nb / 64;
    // the same translation-table placement as the device entry point: the
    // dictionary merge built XC (force_xc) whenever the plain X_M is too big
    // for shared memory, so each chunk may read it from shared memory or L2
    if (e == cudaSuccess) e = launch_recompress(&cin, &cout, xm, xd, rk + d0, d_hdr, st, nb, xc_rec, xc_offs, xs);
    rec(EV_IN0 + K + k, st);
    wait(sout, EV_IN0 + K + k);
    d2h(hout->merged_codes + r0 * nb / 64, cout.merged_codes, cout.merged_codes_cap_words * 8);
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(I.host_hdr, d_hdr, sizeof(dm_header), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(sout);
  if (e == cudaSuccess) e = cudaStreamSynchronize(sin);
  if (e != cudaSuccess) return cuda_fail(e);
  h = *I.host_hdr;
  hout->merged_dict_len = h.merged_dict_len;
  hout->delta_dict_len = h.delta_dict_len;
  hout->merged_bits = h.merged_bits;
  return (dm_status)h.status;
}

uint64_t dm_launch_count(void) { return g_launches.load(); }
int dm_last_cuda_error(void) { return g_last_cuda.load(); }

const char* dm_status_str(int s) {
  switch (s) {
    case DM_OK: return "ok";
    case DM_E_INVALID: return "invalid argument";
    case DM_E_CAPACITY: return "capacity too small";
    case DM_E_TOO_WIDE: return "merged dictionary exceeds 2^32 entries";
    case DM_E_UNSORTED: return "main dictionary not strictly increasing";
    case DM_E_CODE_RANGE: return "main code out of dictionary range";
    case DM_E_CUDA: return "CUDA error";
    case DM_E_NCCL: return "NCCL error";
    default: return "unknown status";
  }
}

}  // extern "C"
