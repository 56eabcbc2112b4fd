// sharded.cu -- dm_merge_column_sharded: one column's merge spread over the
// ranks of a communicator (include/dictmerge.h).
//
// The paper splits Step 2 over threads by tuples: "the N' tuples are evenly
// split between the threads", every thread recompressing its own
// tuple range through the shared translation tables.  Here the threads are
// GPUs: output rows [0, N') are cut into one contiguous range per rank at
// multiples of 4096 rows (every range starts on a u64 word at both widths),
// each rank holds the packed main codes of its range, and the tables cross
// NVLink once:
//   1. root: Steps 1(a), 1(b), 2(a) (dm_dictionary_merge path) -> U', X_M, X_D,
//      r, |U'|, b' and the compact table XC;
//   2. broadcast of the result header (|U'|, |U_D|, b', ...);
//   3. broadcast of XC -- records + one byte per new value (67 MB for cfg5
//      instead of the 4.3 GB X_M) -- and of the X_M slices of the rare flagged
//      superblocks; `tables = DM_TABLES_PLAIN` broadcasts the literal X_M instead
//      (SURVEY §8e's control design);
//   4. the delta rows' codes c[k] = X_D[r[k]] computed on the
//      root and sent to the rank(s) owning rows >= N_M (point to point);
//   5. every rank: Step 2(b) of its row range (Eq 11).
// Transport: NCCL (resolved at run time from the process's libnccl.so.2, the
// copy torch already loaded) or caller callbacks over host buffers (any
// process-group library -- the multi-process tests use gloo).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "dm_device.cuh"

namespace dm {
namespace {

// ------------------------------------------------------------------ NCCL, resolved at run time
struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi a = [] {
    NcclApi x;
    // the copy already in the process (torch links it) first, then the loader's search
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h && std::getenv("DM_NCCL_LIB")) h = dlopen(std::getenv("DM_NCCL_LIB"), RTLD_NOW);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) return x;
#define DM_SYM(f, n) x.f = reinterpret_cast<decltype(x.f)>(dlsym(h, n))
    DM_SYM(getUniqueId, "ncclGetUniqueId");
    DM_SYM(commInitRank, "ncclCommInitRank");
    DM_SYM(commDestroy, "ncclCommDestroy");
    DM_SYM(broadcast, "ncclBroadcast");
    DM_SYM(allGather, "ncclAllGather");
    DM_SYM(send, "ncclSend");
    DM_SYM(recv, "ncclRecv");
    DM_SYM(groupStart, "ncclGroupStart");
    DM_SYM(groupEnd, "ncclGroupEnd");
#undef DM_SYM
    x.ok = x.getUniqueId && x.commInitRank && x.commDestroy && x.broadcast && x.allGather && x.send && x.recv &&
           x.groupStart && x.groupEnd;
    return x;
  }();
  return a;
}

__global__ void __launch_bounds__(256) k_gather_codes(const uint32_t* __restrict__ xd, const uint32_t* __restrict__ r,
                                                      uint64_t n, uint32_t* __restrict__ c) {
  pdl_prologue();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    c[i] = __ldg(xd + __ldg(r + i));
}

}  // namespace
}  // namespace dm

using namespace dm;

// Opaque transport between the ranks of a sharded merge.
struct dm_comm {
  int nranks = 1, rank = 0;
  bool is_nccl = false;
  ncclComm_t nc = nullptr;
  dm_comm_callbacks cb{};
  void* host = nullptr;  // pinned staging for the callback transport
  size_t host_bytes = 0;
  void* stage(size_t bytes) {
    if (bytes <= host_bytes) return host;
    if (host) cudaFreeHost(host);
    host = nullptr;
    host_bytes = 0;
    if (cudaMallocHost(&host, std::max<size_t>(bytes, 1 << 20)) != cudaSuccess) return nullptr;
    host_bytes = std::max<size_t>(bytes, 1 << 20);
    return host;
  }
};

namespace {

// Device-buffer collectives on the comm (stream-ordered for NCCL; the callback
// transport stages through pinned host memory and synchronises the stream).
// (NCCL runs even at one rank, so a one-GPU run exercises the NCCL calls.)
dm_status c_bcast(dm_comm* c, void* dbuf, size_t bytes, int root, cudaStream_t st) {
  if (bytes == 0 || (c->nranks == 1 && !c->is_nccl)) return DM_OK;
  if (c->is_nccl) {
    return nccl().broadcast(dbuf, dbuf, bytes, ncclUint8, root, c->nc, st) == ncclSuccess ? DM_OK : DM_E_NCCL;
  }
  void* h = c->stage(bytes);
  if (!h) return DM_E_CUDA;
  if (c->rank == root && (cudaMemcpyAsync(h, dbuf, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                          cudaStreamSynchronize(st) != cudaSuccess))
    return DM_E_CUDA;
  if (c->cb.broadcast(h, bytes, root, c->cb.user) != 0) return DM_E_NCCL;
  if (c->rank != root && (cudaMemcpyAsync(dbuf, h, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
                          cudaStreamSynchronize(st) != cudaSuccess))
    return DM_E_CUDA;
  return DM_OK;
}

// Host-value broadcast / all-gather (small descriptors); dev_scratch: >= nranks * bytes device bytes.
dm_status c_bcast_host(dm_comm* c, void* hbuf, size_t bytes, int root, void* dev_scratch, cudaStream_t st) {
  if (c->nranks == 1 && !c->is_nccl) return DM_OK;
  if (!c->is_nccl) return c->cb.broadcast(hbuf, bytes, root, c->cb.user) == 0 ? DM_OK : DM_E_NCCL;
  if (cudaMemcpyAsync(dev_scratch, hbuf, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) return DM_E_CUDA;
  dm_status s = c_bcast(c, dev_scratch, bytes, root, st);
  if (s != DM_OK) return s;
  if (cudaMemcpyAsync(hbuf, dev_scratch, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return DM_E_CUDA;
  return DM_OK;
}

dm_status c_allgather_host(dm_comm* c, const void* hsend, void* hrecv, size_t bytes, void* dev_scratch,
                           cudaStream_t st) {
  if (c->nranks == 1 && !c->is_nccl) {
    std::memcpy(hrecv, hsend, bytes);
    return DM_OK;
  }
  if (!c->is_nccl) return c->cb.allgather(hsend, hrecv, bytes, c->cb.user) == 0 ? DM_OK : DM_E_NCCL;
  char* d = static_cast<char*>(dev_scratch);
  if (cudaMemcpyAsync(d + (size_t)c->rank * bytes, hsend, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return DM_E_CUDA;
  if (nccl().allGather(d + (size_t)c->rank * bytes, d, bytes, ncclUint8, c->nc, st) != ncclSuccess) return DM_E_NCCL;
  if (cudaMemcpyAsync(hrecv, d, bytes * c->nranks, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return DM_E_CUDA;
  return DM_OK;
}

// Point to point: `from` sends `bytes` of its dbuf to `to` (both call it).
dm_status c_p2p(dm_comm* c, void* dbuf, size_t bytes, int from, int to, cudaStream_t st) {
  if (bytes == 0 || from == to || (c->rank != from && c->rank != to)) return DM_OK;
  if (c->is_nccl) {
    auto& N = nccl();
    ncclResult_t r = c->rank == from ? N.send(dbuf, bytes, ncclUint8, to, c->nc, st)
                                     : N.recv(dbuf, bytes, ncclUint8, from, c->nc, st);
    return r == ncclSuccess ? DM_OK : DM_E_NCCL;
  }
  void* h = c->stage(bytes);
  if (!h) return DM_E_CUDA;
  if (c->rank == from) {
    if (cudaMemcpyAsync(h, dbuf, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return DM_E_CUDA;
    return c->cb.sendrecv(h, bytes, to, 1, c->cb.user) == 0 ? DM_OK : DM_E_NCCL;
  }
  if (c->cb.sendrecv(h, bytes, from, 0, c->cb.user) != 0) return DM_E_NCCL;
  if (cudaMemcpyAsync(dbuf, h, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return DM_E_CUDA;
  return DM_OK;
}

// Stream-ordered temporaries, released on every exit path.
struct Temps {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Temps(cudaStream_t s) : st(s) {}
  void* get(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, std::max<size_t>(bytes, 256), st) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return p;
  }
  ~Temps() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

// What every rank must agree on (checked by an all-gather before any data moves).
struct ShardDesc {
  int32_t key, tables, root, pad;
  uint64_t dict_len, n_main, n_delta;
  uint32_t main_bits, pad2;
};

// Header the root broadcasts after Steps 1(a)-2(a).
struct ShardHdr {
  uint64_t merged_len, delta_dict_len, n_records, n_new, n_exc;
  uint32_t merged_bits, xs;
  int32_t status, xc;
};

}  // namespace

extern "C" {

void dm_plan_row_shards(uint64_t n_main, uint64_t n_delta, int nranks, uint64_t* cuts) {
  if (nranks < 1 || !cuts) return;
  const uint64_t total = n_main + n_delta;
  cuts[0] = 0;
  for (int g = 1; g < nranks; ++g) {
    // total * g / nranks without overflow: total < 2^63 / nranks in practice; use 128-bit to be safe
    const unsigned __int128 q = (unsigned __int128)total * (unsigned)g / (unsigned)nranks;
    const uint64_t c = ((uint64_t)q) / 4096 * 4096;
    cuts[g] = std::max(c, cuts[g - 1]);
  }
  cuts[nranks] = total;
}

uint64_t dm_sharded_codes_cap_words(uint64_t dict_len, uint64_t n_main, uint64_t n_delta, int nranks, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return 0;
  std::vector<uint64_t> cuts(nranks + 1);
  dm_plan_row_shards(n_main, n_delta, nranks, cuts.data());
  const uint32_t bw = std::min<uint32_t>(32, host_width(dict_len + n_delta));
  return host_words(cuts[rank + 1], bw) - cuts[rank] * bw / 64;
}

dm_status dm_comm_nccl_unique_id(void* id_out) {
  if (!id_out) return DM_E_INVALID;
  if (!nccl().ok) return DM_E_NCCL;
  ncclUniqueId id;
  if (nccl().getUniqueId(&id) != ncclSuccess) return DM_E_NCCL;
  std::memcpy(id_out, &id, sizeof(id));
  return DM_OK;
}

dm_comm* dm_comm_init_nccl(const void* id, int nranks, int rank, int device) {
  if (!id || nranks < 1 || rank < 0 || rank >= nranks || !nccl().ok) return nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return nullptr;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t nc = nullptr;
  if (nccl().commInitRank(&nc, nranks, uid, rank) != ncclSuccess) return nullptr;
  dm_comm* c = new dm_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->is_nccl = true;
  c->nc = nc;
  return c;
}

dm_comm* dm_comm_init_callbacks(const dm_comm_callbacks* cb, int nranks, int rank) {
  if (!cb || !cb->broadcast || !cb->allgather || !cb->sendrecv || nranks < 1 || rank < 0 || rank >= nranks)
    return nullptr;
  dm_comm* c = new dm_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->cb = *cb;
  return c;
}

void dm_comm_destroy(dm_comm* c) {
  if (!c) return;
  if (c->is_nccl && c->nc) nccl().commDestroy(c->nc);
  if (c->host) cudaFreeHost(c->host);
  delete c;
}

int dm_comm_rank(const dm_comm* c) { return c ? c->rank : -1; }
int dm_comm_size(const dm_comm* c) { return c ? c->nranks : -1; }

dm_status dm_comm_selftest_host(dm_comm* c) {
  // Host-only check of a callback transport (no GPU): broadcast, all-gather and
  // point to point deliver the right bytes in rank order.
  if (!c || c->is_nccl) return DM_E_INVALID;
  const int n = c->nranks, me = c->rank;
  std::vector<uint32_t> b(1024);
  for (int root = 0; root < n; ++root) {
    for (size_t i = 0; i < b.size(); ++i) b[i] = me == root ? (uint32_t)(i * 2654435761u + root) : 0u;
    if (c->cb.broadcast(b.data(), b.size() * 4, root, c->cb.user) != 0) return DM_E_NCCL;
    for (size_t i = 0; i < b.size(); ++i)
      if (b[i] != (uint32_t)(i * 2654435761u + root)) return DM_E_NCCL;
  }
  std::vector<uint64_t> mine(3), all(3 * (size_t)n);
  for (int i = 0; i < 3; ++i) mine[i] = ((uint64_t)me << 32) | (uint64_t)i;
  if (c->cb.allgather(mine.data(), all.data(), 24, c->cb.user) != 0) return DM_E_NCCL;
  for (int g = 0; g < n; ++g)
    for (int i = 0; i < 3; ++i)
      if (all[(size_t)g * 3 + i] != (((uint64_t)g << 32) | (uint64_t)i)) return DM_E_NCCL;
  if (n > 1) {  // rank 0 -> last rank
    std::vector<uint32_t> p(257, me == 0 ? 7u : 0u);
    if (me == 0 && c->cb.sendrecv(p.data(), p.size() * 4, n - 1, 1, c->cb.user) != 0) return DM_E_NCCL;
    if (me == n - 1) {
      if (c->cb.sendrecv(p.data(), p.size() * 4, 0, 0, c->cb.user) != 0) return DM_E_NCCL;
      for (uint32_t v : p)
        if (v != 7u) return DM_E_NCCL;
    }
  }
  return DM_OK;
}

void dm_plan_dict_ranges(uint64_t dict_len, int nranks, uint64_t* cuts) {
  if (nranks < 1 || !cuts) return;
  cuts[0] = 0;
  for (int g = 1; g < nranks; ++g) {
    const unsigned __int128 q = (unsigned __int128)dict_len * (unsigned)g / (unsigned)nranks;
    cuts[g] = std::max<uint64_t>(cuts[g - 1], ((uint64_t)q) / 1024 * 1024);
  }
  cuts[nranks] = dict_len;
}

dm_status dm_merge_column_sharded(dm_comm* comm, const dm_sharded_in* in, dm_sharded_out* out, void* cuda_stream) {
  if (!comm || !in || !out) return DM_E_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const int R = comm->nranks, me = comm->rank, root = in->root;
  if (root < 0 || root >= R) return DM_E_INVALID;
  if (in->tables != DM_TABLES_XC && in->tables != DM_TABLES_PLAIN) return DM_E_INVALID;
  if (in->step1b != DM_STEP1B_ROOT && in->step1b != DM_STEP1B_RANGES) return DM_E_INVALID;
  const bool ranges = in->step1b == DM_STEP1B_RANGES;
  Temps T(st);
  void* scratch = T.get(256 * (size_t)R + 256);
  if (!scratch) return DM_E_CUDA;
  // 1. every rank agrees on the column's shape and the call's options
  ShardDesc mine{in->key, in->tables, root, in->step1b, in->dict_len, in->n_main, in->n_delta, in->main_bits, 0};
  std::vector<ShardDesc> all(R);
  dm_status s = c_allgather_host(comm, &mine, all.data(), sizeof(ShardDesc), scratch, st);
  if (s != DM_OK) return s;
  for (int g = 0; g < R; ++g)
    if (std::memcmp(&all[g], &mine, sizeof(ShardDesc)) != 0) return DM_E_INVALID;
  // argument checks (the same on every rank, so every rank returns the same error)
  if (in->key != DM_KEY_U64 && in->key != DM_KEY_B16 && in->key != DM_KEY_U32) return DM_E_INVALID;
  if (in->main_bits < 1 || in->main_bits > 32 || in->dict_len >= (1ull << 32) || in->n_delta >= (1ull << 30))
    return DM_E_INVALID;
  if (in->n_main > 0 && (in->dict_len == 0 || in->main_bits < host_width(in->dict_len))) return DM_E_INVALID;
  if (in->dict_len + in->n_delta > (1ull << 32)) return DM_E_TOO_WIDE;
  std::vector<uint64_t> rg(2 * (size_t)R);  // RANGES: every rank's (range_begin, range_len)
  if (ranges) {
    const uint64_t mr[2] = {in->range_begin, in->range_len};
    if ((s = c_allgather_host(comm, mr, rg.data(), 16, scratch, st)) != DM_OK) return s;
    if (in->tables != DM_TABLES_XC || in->dict_len == 0) return DM_E_INVALID;
    uint64_t next = 0;
    for (int g = 0; g < R; ++g) {  // ranges tile [0, |U_M|) in rank order, whole superblocks
      if (rg[2 * g] != next || rg[2 * g + 1] == 0 || (rg[2 * g] % 1024) != 0) return DM_E_INVALID;
      next += rg[2 * g + 1];
    }
    if (next != in->dict_len) return DM_E_INVALID;
    if (!in->main_dict || (reinterpret_cast<uintptr_t>(in->main_dict) & 15u)) return DM_E_INVALID;
  }
  std::vector<uint64_t> cuts(R + 1);
  dm_plan_row_shards(in->n_main, in->n_delta, R, cuts.data());
  const uint64_t r0 = cuts[me], r1 = cuts[me + 1];
  const uint64_t m0 = std::min(r0, in->n_main), m1 = std::min(r1, in->n_main);
  const uint64_t d0 = std::max(r0, in->n_main) - in->n_main, d1 = std::max(r1, in->n_main) - in->n_main;
  if (m1 > m0 && (!in->main_codes || (reinterpret_cast<uintptr_t>(in->main_codes) & 15u))) return DM_E_INVALID;
  const uint64_t cap_words = dm_sharded_codes_cap_words(in->dict_len, in->n_main, in->n_delta, R, me);
  if (r1 > r0 && (!out->merged_codes || (reinterpret_cast<uintptr_t>(out->merged_codes) & 15u))) return DM_E_INVALID;
  if (out->merged_codes_cap_words < cap_words) return DM_E_CAPACITY;
  if (ranges && (!out->merged_dict || out->merged_dict_cap < in->range_len + in->n_delta)) return DM_E_CAPACITY;
  const size_t E = key_bytes(in->key);

  ShardHdr H{};
  uint32_t *xm = nullptr, *xd = nullptr, *rk = nullptr, *codes_d = nullptr;
  const uint2* xc_rec = nullptr;
  const uint8_t* xc_offs = nullptr;
  uint32_t* xm_use = nullptr;
  dm_header* d_hdr = reinterpret_cast<dm_header*>(static_cast<char*>(scratch) + 256 * (size_t)R);
  if (!ranges) {
    // ---- 2. root: Steps 1(a), 1(b), 2(a)
    char* ws = nullptr;
    dm_column_in cin{};
    cin.key = in->key;
    cin.main_dict = in->main_dict;
    cin.dict_len = in->dict_len;
    cin.n_main = 0;  // no Step 2 on the root's full column here
    cin.main_bits = in->main_bits;
    cin.delta = in->delta;
    cin.n_delta = in->n_delta;
    if (me == root) {
      dm_column_out cout{};
      cout.merged_dict = out->merged_dict;
      cout.merged_dict_cap = out->merged_dict_cap;
      xm = static_cast<uint32_t*>(T.get(std::max<uint64_t>(in->dict_len, 1) * 4));
      xd = static_cast<uint32_t*>(T.get(std::max<uint64_t>(in->n_delta, 1) * 4));
      rk = static_cast<uint32_t*>(T.get(std::max<uint64_t>(in->n_delta, 1) * 4));
      cout.x_main = xm;
      cout.x_delta = xd;
      cout.delta_rank = rk;
      const size_t wsb = dm_workspace_bytes(&cin);
      ws = static_cast<char*>(T.get(wsb));
      if (!xm || !xd || !rk || !ws) s = DM_E_CUDA;
      if (s == DM_OK) s = dm_dictionary_merge_async(&cin, &cout, ws, wsb, d_hdr, st);
      dm_header h{};
      if (s == DM_OK && (cudaMemcpyAsync(&h, d_hdr, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                         cudaStreamSynchronize(st) != cudaSuccess))
        s = DM_E_CUDA;
      H.status = s != DM_OK ? (int32_t)s : h.status;
      H.merged_len = h.merged_dict_len;
      H.delta_dict_len = h.delta_dict_len;
      H.merged_bits = h.merged_bits;
      // XC only where Step 2(b) would read it: a plain X_M of <= 96 KB is staged in
      // shared memory as it is, and broadcasting it costs nothing
      H.xc = in->tables == DM_TABLES_XC && in->dict_len * 4 > kRecSmemXBytes && s == DM_OK;
      if (H.xc) {
        dm_xc x{};
        dm_xc_export(&cin, ws, wsb, &x);
        xc_rec = static_cast<const uint2*>(x.records);
        xc_offs = x.offsets;
        H.xs = x.shift;
        H.n_records = x.n_records;
        H.n_new = H.merged_len - in->dict_len;
        unsigned long long* cnt = reinterpret_cast<unsigned long long*>(static_cast<char*>(scratch) + 128);
        if (cudaMemsetAsync(cnt, 0, 8, st) != cudaSuccess ||
            launch_xc_exceptions(true, xc_rec, H.n_records, H.xs, in->dict_len, xm, nullptr, nullptr, cnt, 0, st) !=
                cudaSuccess ||
            cudaMemcpyAsync(&H.n_exc, cnt, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
          H.status = DM_E_CUDA;
      }
    }
    // ---- 3. the header to every rank
    if ((s = c_bcast_host(comm, &H, sizeof(H), root, scratch, st)) != DM_OK) return s;
    if (H.status != DM_OK) return (dm_status)H.status;
    // ---- 4. translation tables
    xm_use = xm;
    if (H.xc) {
      // + 64: the L2 lookup reads 16-byte windows past the last entry (zeroed)
      const size_t rec_bytes = H.n_records * 8, offs_bytes = ((H.n_new + 15) / 16) * 16 + 64;
      if (me != root) {
        void* rec = T.get(rec_bytes);
        void* offs = T.get(offs_bytes);
        if (!rec || !offs) return DM_E_CUDA;
        if (cudaMemsetAsync(offs, 0, offs_bytes, st) != cudaSuccess) return DM_E_CUDA;
        xc_rec = static_cast<const uint2*>(rec);
        xc_offs = static_cast<const uint8_t*>(offs);
      }
      if ((s = c_bcast(comm, const_cast<uint2*>(xc_rec), rec_bytes, root, st)) != DM_OK) return s;
      if ((s = c_bcast(comm, const_cast<uint8_t*>(xc_offs), H.n_new, root, st)) != DM_OK) return s;
      if (H.n_exc) {  // X_M slices of flagged superblocks: root gathers, everyone else scatters into a sparse X_M
        const uint64_t SB = 4ull << H.xs;
        uint32_t* ids = static_cast<uint32_t*>(T.get(H.n_exc * 4));
        uint32_t* sl = static_cast<uint32_t*>(T.get(H.n_exc * SB * 4));
        if (!ids || !sl) return DM_E_CUDA;
        if (me == root) {
          unsigned long long* cnt = reinterpret_cast<unsigned long long*>(static_cast<char*>(scratch) + 128);
          if (cudaMemsetAsync(cnt, 0, 8, st) != cudaSuccess ||
              launch_xc_exceptions(true, xc_rec, H.n_records, H.xs, in->dict_len, xm, ids, sl, cnt, 0, st) !=
                  cudaSuccess)
            return DM_E_CUDA;
        }
        if ((s = c_bcast(comm, ids, H.n_exc * 4, root, st)) != DM_OK) return s;
        if ((s = c_bcast(comm, sl, H.n_exc * SB * 4, root, st)) != DM_OK) return s;
        if (me != root) {
          xm_use = static_cast<uint32_t*>(T.get(in->dict_len * 4));  // only the flagged superblocks are written/read
          if (!xm_use) return DM_E_CUDA;
          if (launch_xc_exceptions(false, nullptr, H.n_records, H.xs, in->dict_len, xm_use, ids, sl, nullptr,
                                   H.n_exc, st) != cudaSuccess)
            return DM_E_CUDA;
        }
      } else if (me != root) {
        xm_use = static_cast<uint32_t*>(scratch);  // never read: no flagged superblock
      }
    } else if (in->dict_len) {  // control design: the literal X_M
      if (me != root) {
        xm_use = static_cast<uint32_t*>(T.get(in->dict_len * 4));
        if (!xm_use) return DM_E_CUDA;
      }
      if ((s = c_bcast(comm, xm_use, in->dict_len * 4, root, st)) != DM_OK) return s;
    }
  } else {
    // ---- NEXT2: Step 1(b) by U_M value ranges
    const uint32_t xs = kXcMinShift;  // one block size for every range (128 codes)
    const uint64_t SB = 4ull << xs;
    const uint64_t a = in->range_begin, L = in->range_len;
    // 2a. root: Step 1(a) -> U_D, r, |U_D|
    void* ud = nullptr;
    uint64_t meta[2] = {0, 0};  // |U_D|, status
    if (me == root) {
      dm_column_in cin{};
      cin.key = in->key;
      cin.main_dict = in->main_dict;
      cin.dict_len = L;
      cin.main_bits = in->main_bits;
      cin.delta = in->delta;
      cin.n_delta = in->n_delta;
      dm_column_out cout{};
      ud = T.get(std::max<uint64_t>(in->n_delta, 1) * E);
      rk = static_cast<uint32_t*>(T.get(std::max<uint64_t>(in->n_delta, 1) * 4));
      cout.merged_dict = out->merged_dict;  // not written in this mode
      cout.merged_dict_cap = out->merged_dict_cap;
      cout.delta_dict = ud;
      cout.delta_rank = rk;
      const size_t wsb = dm_workspace_bytes(&cin);
      void* ws = T.get(wsb);
      if (!ud || !rk || !ws) s = DM_E_CUDA;
      if (s == DM_OK) s = dm_delta_dictionary_async(&cin, &cout, ws, wsb, d_hdr, st);
      dm_header h{};
      if (s == DM_OK && (cudaMemcpyAsync(&h, d_hdr, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                         cudaStreamSynchronize(st) != cudaSuccess))
        s = DM_E_CUDA;
      meta[0] = h.delta_dict_len;
      meta[1] = (uint64_t)(int64_t)(s != DM_OK ? (int)s : h.status);
    }
    if ((s = c_bcast_host(comm, meta, 16, root, scratch, st)) != DM_OK) return s;
    if ((int64_t)meta[1] != 0) return (dm_status)(int)(int64_t)meta[1];
    const uint64_t n_ud = meta[0];
    // 2b. every range's first value -> the root cuts U_D there
    char* firsts = static_cast<char*>(T.get(E * (size_t)R));
    std::vector<unsigned char> myfirst(E), allfirst(E * (size_t)R);
    if (!firsts || cudaMemcpyAsync(myfirst.data(), in->main_dict, E, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return DM_E_CUDA;
    if ((s = c_allgather_host(comm, myfirst.data(), allfirst.data(), E, scratch, st)) != DM_OK) return s;
    std::vector<uint64_t> ucut(R + 1, 0);
    ucut[R] = n_ud;
    if (me == root && R > 1) {
      uint64_t* pos = static_cast<uint64_t*>(T.get(8 * (size_t)R));
      if (!pos || cudaMemcpyAsync(firsts, allfirst.data(), E * R, cudaMemcpyHostToDevice, st) != cudaSuccess ||
          launch_lower_bound(in->key, ud, n_ud, firsts + E, R - 1, pos, st) != cudaSuccess ||
          cudaMemcpyAsync(ucut.data() + 1, pos, 8 * (size_t)(R - 1), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess)
        return DM_E_CUDA;
    }
    if ((s = c_bcast_host(comm, ucut.data(), 8 * (size_t)(R + 1), root, scratch, st)) != DM_OK) return s;
    // 2c. U_D to every rank; each keeps its value range (its own 16-byte aligned copy)
    if (me != root) ud = T.get(std::max<uint64_t>(n_ud, 1) * E);
    if (!ud) return DM_E_CUDA;
    if ((s = c_bcast(comm, ud, n_ud * E, root, st)) != DM_OK) return s;
    const uint64_t j0 = ucut[me], nj = ucut[me + 1] - ucut[me];
    void* mine = T.get(std::max<uint64_t>(nj, 1) * E);
    if (!mine || (nj && cudaMemcpyAsync(mine, static_cast<char*>(ud) + j0 * E, nj * E, cudaMemcpyDeviceToDevice,
                                       st) != cudaSuccess))
      return DM_E_CUDA;
    // 2d. this range's merge (Steps 1(b)-2(a)); XC with the common block size
    dm_column_in lin{};
    lin.key = in->key;
    lin.main_dict = in->main_dict;
    lin.dict_len = L;
    lin.main_bits = in->main_bits;
    lin.delta = mine;
    lin.n_delta = nj;
    dm_column_out lout{};
    lout.merged_dict = out->merged_dict;
    lout.merged_dict_cap = out->merged_dict_cap;
    uint32_t* xm_l = static_cast<uint32_t*>(T.get(L * 4));
    uint32_t* xd_l = static_cast<uint32_t*>(T.get(std::max<uint64_t>(nj, 1) * 4));
    lout.x_main = xm_l;
    lout.x_delta = xd_l;
    set_xc_shift_override((int)xs);
    const size_t wsb = dm_workspace_bytes(&lin);
    char* lws = static_cast<char*>(T.get(wsb));
    if (!xm_l || !xd_l || !lws) s = DM_E_CUDA;
    if (s == DM_OK) s = dm_dictionary_merge_sorted_async(&lin, &lout, lws, wsb, d_hdr, st);
    dm_xc lx{};
    if (s == DM_OK) dm_xc_export(&lin, lws, wsb, &lx);
    set_xc_shift_override(0);
    dm_header h{};
    if (s == DM_OK && (cudaMemcpyAsync(&h, d_hdr, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                       cudaStreamSynchronize(st) != cudaSuccess))
      s = DM_E_CUDA;
    // 2e. counts of every range: offsets, |U'|, b' (and every rank's status)
    int64_t cnt3[3] = {(int64_t)h.merged_dict_len, (int64_t)(h.merged_dict_len - L), (int64_t)(s != DM_OK ? (int)s : h.status)};
    std::vector<int64_t> allc(3 * (size_t)R);
    dm_status s2 = c_allgather_host(comm, cnt3, allc.data(), 24, scratch, st);
    if (s2 != DM_OK) return s2;
    uint64_t u_off = 0, new_off = 0, n_u = 0, n_new = 0;
    for (int g = 0; g < R; ++g) {
      if (allc[3 * g + 2] != 0) return (dm_status)allc[3 * g + 2];
      if (g < me) u_off += allc[3 * g], new_off += allc[3 * g + 1];
      n_u += allc[3 * g];
      n_new += allc[3 * g + 1];
    }
    out->merged_dict_offset = u_off;
    out->merged_slice_len = h.merged_dict_len;
    // 2f. rebase this range's tables by the earlier ranges
    if (u_off && (launch_add_u32(xm_l, L, (uint32_t)u_off, st) != cudaSuccess ||
                  launch_add_u32(xd_l, nj, (uint32_t)u_off, st) != cudaSuccess))
      return DM_E_CUDA;
    const uint64_t nrec_l = (L + SB - 1) / SB;
    if (new_off && launch_xc_rebase(const_cast<void*>(lx.records), nrec_l, (uint32_t)new_off, st) != cudaSuccess)
      return DM_E_CUDA;
    H.merged_len = n_u;
    H.delta_dict_len = n_ud;
    H.merged_bits = host_width(n_u);
    // X_D on the root, gathered from the ranges
    if (me == root) {
      xd = static_cast<uint32_t*>(T.get(std::max<uint64_t>(n_ud, 1) * 4));
      if (!xd || (nj && cudaMemcpyAsync(xd + j0, xd_l, nj * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess))
        return DM_E_CUDA;
    }
    {
      const bool grouped = comm->is_nccl && me == root;
      if (grouped && nccl().groupStart() != ncclSuccess) return DM_E_NCCL;
      for (int g = 0; g < R && s == DM_OK; ++g) {
        const uint64_t gn = ucut[g + 1] - ucut[g];
        if (g == root || gn == 0) continue;
        s = c_p2p(comm, me == root ? xd + ucut[g] : xd_l, gn * 4, g, root, st);
      }
      if (grouped && nccl().groupEnd() != ncclSuccess) return DM_E_NCCL;
      if (s != DM_OK) return s;
    }
    if (in->dict_len * 4 <= kRecSmemXBytes) {  // a small X_M is staged in shared memory whole: gather it plainly
      xm_use = static_cast<uint32_t*>(T.get(in->dict_len * 4));
      if (!xm_use || cudaMemcpyAsync(xm_use + a, xm_l, L * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return DM_E_CUDA;
      for (int g = 0; g < R; ++g)
        if ((s = c_bcast(comm, xm_use + rg[2 * g], rg[2 * g + 1] * 4, g, st)) != DM_OK) return s;
      H.xc = 0;
    } else {
    // 2g. the global XC on every rank (rank order = value order)
    H.xc = 1;
    H.xs = xs;
    H.n_records = (in->dict_len + SB - 1) / SB;
    H.n_new = n_new;
    const size_t offs_bytes = ((n_new + 15) / 16) * 16 + 64;
    uint2* grec = static_cast<uint2*>(T.get(H.n_records * 8));
    uint8_t* goffs = static_cast<uint8_t*>(T.get(offs_bytes));
    if (!grec || !goffs || cudaMemsetAsync(goffs, 0, offs_bytes, st) != cudaSuccess) return DM_E_CUDA;
    const uint64_t rec0 = a / SB;
    if (cudaMemcpyAsync(grec + rec0, lx.records, nrec_l * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
        (h.merged_dict_len > L &&
         cudaMemcpyAsync(goffs + new_off, lx.offsets, h.merged_dict_len - L, cudaMemcpyDeviceToDevice, st) !=
             cudaSuccess))
      return DM_E_CUDA;
    uint64_t o_new = 0;
    for (int g = 0; g < R; ++g) {  // all-gather by broadcasts from each rank in turn
      const uint64_t rb = rg[2 * g] / SB, rn = (rg[2 * g + 1] + SB - 1) / SB;
      if ((s = c_bcast(comm, grec + rb, rn * 8, g, st)) != DM_OK) return s;
      if ((s = c_bcast(comm, goffs + o_new, (uint64_t)allc[3 * g + 1], g, st)) != DM_OK) return s;
      o_new += (uint64_t)allc[3 * g + 1];
    }
    xc_rec = grec;
    xc_offs = goffs;
    // 2h. flagged superblocks: every range's X_M slices to every rank
    uint64_t my_exc = 0;
    {
      unsigned long long* cnt = reinterpret_cast<unsigned long long*>(static_cast<char*>(scratch) + 128);
      if (cudaMemsetAsync(cnt, 0, 8, st) != cudaSuccess ||
          launch_xc_exceptions(true, static_cast<const uint2*>(lx.records), nrec_l, xs, L, xm_l, nullptr, nullptr,
                               cnt, 0, st) != cudaSuccess ||
          cudaMemcpyAsync(&my_exc, cnt, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess)
        return DM_E_CUDA;
    }
    std::vector<uint64_t> exc(R);
    if ((s = c_allgather_host(comm, &my_exc, exc.data(), 8, scratch, st)) != DM_OK) return s;
    uint64_t n_exc = 0;
    for (uint64_t x : exc) n_exc += x;
    H.n_exc = n_exc;
    xm_use = static_cast<uint32_t*>(scratch);  // never read without flagged superblocks
    if (n_exc) {
      uint32_t* ids = static_cast<uint32_t*>(T.get(n_exc * 4));
      uint32_t* sl = static_cast<uint32_t*>(T.get(n_exc * SB * 4));
      xm_use = static_cast<uint32_t*>(T.get(in->dict_len * 4));  // sparse: the flagged superblocks only
      if (!ids || !sl || !xm_use) return DM_E_CUDA;
      uint64_t e0 = 0;
      for (int g = 0; g < me; ++g) e0 += exc[g];
      if (my_exc) {
        unsigned long long* cnt = reinterpret_cast<unsigned long long*>(static_cast<char*>(scratch) + 128);
        if (cudaMemsetAsync(cnt, 0, 8, st) != cudaSuccess ||
            launch_xc_exceptions(true, static_cast<const uint2*>(lx.records), nrec_l, xs, L, xm_l, ids + e0,
                                 sl + e0 * SB, cnt, 0, st) != cudaSuccess ||
            launch_add_u32(ids + e0, my_exc, (uint32_t)rec0, st) != cudaSuccess)  // local -> global superblock ids
          return DM_E_CUDA;
      }
      uint64_t o = 0;
      for (int g = 0; g < R; ++g) {
        if ((s = c_bcast(comm, ids + o, exc[g] * 4, g, st)) != DM_OK) return s;
        if ((s = c_bcast(comm, sl + o * SB, exc[g] * SB * 4, g, st)) != DM_OK) return s;
        o += exc[g];
      }
      if (launch_xc_exceptions(false, nullptr, H.n_records, xs, in->dict_len, xm_use, ids, sl, nullptr, n_exc, st) !=
          cudaSuccess)
        return DM_E_CUDA;
    }
    }  // XC
  }
  const uint32_t nb = H.merged_bits;
  out->merged_dict_len = H.merged_len;
  out->merged_bits = nb;
  // a device header with |U'| and b' on every rank (the Step 2(b) kernels read them)
  dm_header hh{H.merged_len, H.delta_dict_len, nb, 0};
  if (cudaMemcpyAsync(d_hdr, &hh, sizeof(hh), cudaMemcpyHostToDevice, st) != cudaSuccess) return DM_E_CUDA;

  // 5. the delta rows' codes c = X_D[r] (root), each owner receives its slice
  if (in->n_delta) {
    if (me == root) {
      codes_d = static_cast<uint32_t*>(T.get(in->n_delta * 4));
      if (!codes_d) return DM_E_CUDA;
      const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((in->n_delta + 255) / 256, 148 * 16));
      launch_k(k_gather_codes, g, 256, 0, st, (const uint32_t*)xd, (const uint32_t*)rk, in->n_delta, codes_d);
      note_launch();
    } else if (d1 > d0) {
      codes_d = static_cast<uint32_t*>(T.get((d1 - d0) * 4));
      if (!codes_d) return DM_E_CUDA;
    }
    const bool grouped = comm->is_nccl && me == root;  // the root's sends to several owners in one group
    if (grouped && nccl().groupStart() != ncclSuccess) return DM_E_NCCL;
    for (int g = 0; g < R && s == DM_OK; ++g) {
      const uint64_t gd0 = std::max(cuts[g], in->n_main) - in->n_main, gd1 = std::max(cuts[g + 1], in->n_main) - in->n_main;
      if (gd1 <= gd0 || g == root) continue;
      uint32_t* buf = me == root ? codes_d + gd0 : codes_d;
      s = c_p2p(comm, buf, (gd1 - gd0) * 4, root, g, st);
    }
    if (grouped && nccl().groupEnd() != ncclSuccess) return DM_E_NCCL;
    if (s != DM_OK) return s;
  }

  // 6. Step 2(b) of this rank's rows
  if (r1 > r0) {
    dm_column_in sin{};
    sin.key = in->key;
    sin.dict_len = in->dict_len;
    sin.main_codes = m1 > m0 ? in->main_codes : nullptr;
    sin.n_main = m1 - m0;
    sin.main_bits = in->main_bits;
    sin.n_delta = d1 - d0;
    dm_column_out sout{};
    sout.merged_codes = out->merged_codes;
    sout.merged_codes_cap_words = out->merged_codes_cap_words;
    const uint32_t* cd = codes_d ? (me == root ? codes_d + d0 : codes_d) : nullptr;
    // delta rows: x_delta = their codes, rank = NULL (identity); (xc_only: ranks
    // other than the root hold XC, not the plain X_M)
    cudaError_t e = launch_recompress(&sin, &sout, xm_use, cd, nullptr, d_hdr, st, nb, H.xc ? xc_rec : nullptr,
                                      H.xc ? xc_offs : nullptr, H.xc ? H.xs : 8, H.xc != 0);
    if (e != cudaSuccess) return DM_E_CUDA;
  }
  // 7. every rank's Step 2(b) status (code range), worst wins
  dm_header fin{};
  if (cudaMemcpyAsync(&fin, d_hdr, sizeof(fin), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return DM_E_CUDA;
  std::vector<int32_t> stats(R);
  s = c_allgather_host(comm, &fin.status, stats.data(), sizeof(int32_t), scratch, st);
  if (s != DM_OK) return s;
  int worst = DM_OK;
  for (int32_t v : stats) worst = std::min(worst, (int)v);
  return (dm_status)worst;
}

}  // extern "C"
