// Library-internal state shared by runtime.cu (context, load, build, results)
// and execute.cu (slots, executor).  Product code.
#pragma once
#include <algorithm>
#include <condition_variable>
#include <functional>
#include <map>
#include <memory>
#include <thread>
#include <mutex>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include <cuda_runtime.h>

#include "gsmart.h"
#include "internal.h"
#include "kernels.h"
#include "nccl_shim.h"

namespace gsm {

enum Kid {
  K_BUILD_PACK = 0, K_BUILD_SORT, K_BUILD_UNIQUE, K_BUILD_ROWPTR, K_SEED, K_FILTER, K_BITMAP, K_COMPACT,
  K_SCAN, K_EXPAND_SEG, K_EXPAND_COUNT, K_EXPAND_EMIT, K_PRUNE, K_ENUMERATE, K_SORT_ROWS, K_COLLECTIVE
};
extern const char* kKernelNames[GSMART_NKERNELS];

// One symmetric region (symheap.cu): rank q's chunk is mapped at va + off[q] on
// every rank; this rank's own chunk is local().
struct SymRegion {
  uint64_t va = 0, total = 0;
  std::vector<uint64_t> off, bytes;
  std::vector<unsigned long long> handles;  // CUmemGenericAllocationHandle per rank
  bool own_only = false;                    // handles shared in-process: release only our own
  int rank = 0;
  char* local() const { return va ? (char*)(va + off[rank]) : nullptr; }
  SymDelta delta(int world) const {         // word (4-byte) distance from our chunk to rank q's
    SymDelta d{};
    for (int q = 0; q < world && q < MAX_WORLD; q++) d.words[q] = ((long long)off[q] - (long long)off[rank]) / 4;
    return d;
  }
};

struct Lspm {
  uint32_t* rp = nullptr;
  uint32_t* col = nullptr;
  void* pred = nullptr;
  uint32_t* lmask = nullptr;  // [N] row label signatures (Fmt::lmask)
  uint64_t nnz = 0;
  bool built = false;
  unsigned long long heavy_rows = 0, heavy_chunks = 0;
  // world > 1: rp/col/pred/lmask point into symmetric regions (global view of
  // every rank's rows); this rank stores rows [row_lo, row_hi) only
  bool sym = false;
  SymRegion s_rp, s_col, s_pred, s_lmask;
  // [l]: rows holding label l, [P + 1 + l]: its entries (empty when P > 4095);
  // entries / rows = the expected fan-out of a pattern from this side
  std::vector<unsigned long long> label_rows;
  // [l] = 1: no row holds two entries with label l (exact, every row): a trie
  // level reached over label l from this format's rows is "functional"
  std::vector<uint8_t> functional;
};

// Label-major entry lists: the kept, de-duplicated triples grouped by predicate,
// (s, o) ascending within a label: entries of label l are [off[l], off[l+1]).
// The push form of the grouped evaluation streams them.
struct LabelMajor {
  uint32_t* s = nullptr;
  uint32_t* o = nullptr;
  std::vector<uint64_t> off;  // host copy, P + 2 entries
  uint64_t M = 0;
  bool built = false;
};

// 1-D vertex-range partition (world > 1): rank q owns rows [v[q], v[q+1]) of
// both formats; split points balance out+in entries, aligned to 2^19 vertices
// (2 MiB of row pointers: the granularity of a symmetric chunk)
constexpr uint32_t PART_ALIGN_ROWS = 1u << 19;
// f4 dictionary (ingest.cu): term bytes stay resident in `text`; per kind
// (0 entity, 1 predicate) the (offset, length) of each id's term and the
// sorted term hashes with their ids (lookups)
struct Dict {
  uint8_t* text = nullptr;
  uint64_t bytes = 0;
  bool valid = false;
  uint32_t n[2] = {0, 0};
  uint64_t* off[2] = {nullptr, nullptr};
  uint32_t* len[2] = {nullptr, nullptr};
  uint64_t* hash[2] = {nullptr, nullptr};
  uint32_t* hid[2] = {nullptr, nullptr};
};

struct Partition {
  std::vector<uint32_t> v;  // world + 1 split points
};

// host side of the ranks-as-processes rendezvous (symheap.cu): a star of
// abstract Unix sockets through rank 0, for small all-gathers and SCM_RIGHTS
// file-descriptor exchange of symmetric chunks
struct SockChan {
  int rank = 0, world = 1;
  int listen_fd = -1;
  std::vector<int> peers;  // rank 0: one socket per peer; others: [0] = socket to rank 0
  ~SockChan();
  bool open(const void* id128, int rank, int world, std::string* err);
  bool allgather(const void* mine, size_t n, void* all);
  bool allgather_fds(int my_fd, std::vector<int>* fds);
};

inline int bits_for(uint64_t v) {  // bits to represent values in [0, v]
  int b = 1;
  while (b < 64 && (v >> b) != 0) b++;
  return b;
}

constexpr uint32_t LB_CAP_TILES = 1u << 22;  // 4M tiles x 1024 entries = the 2^32-entry limit
constexpr uint32_t LB_EPOCHS = 65536;
constexpr uint32_t MAX_SLOTS = 16;
constexpr uint32_t H_EPOCH = 255;  // h_pin slot: look-back epoch base of the running execute
constexpr uint32_t H_BAR = 254;    // h_pin slot: rank-barrier generation base (world > 1)

// One concurrent execution lane: a stream plus everything an in-flight
// execute writes (workspace, look-back state, counters, pinned readback).
struct Slot {
  cudaStream_t st = nullptr;
  bool own_stream = false;
  cudaEvent_t ev = nullptr;
  struct LvBuf {
    uint64_t cap = 0;
    uint32_t *bind = nullptr, *parent = nullptr, *seg_beg = nullptr, *off = nullptr, *newidx = nullptr;
    uint8_t* alive = nullptr;
    uint32_t* anc[MAXANC] = {};  // materialised ancestor bindings (allocated on first use)
  };
  LvBuf lv[GSMART_MAX_LEVELS];
  uint32_t* list[GSMART_MAX_LEVELS] = {};
  uint64_t list_cap[GSMART_MAX_LEVELS] = {};
  unsigned long long* lb_status = nullptr;
  uint32_t* lb_counters = nullptr;
  uint32_t* tile_start = nullptr;      // [LB_CAP_TILES] expansion tile -> first parent
  unsigned long long* om = nullptr;    // f2: (root, binding) key sets of first occurrences with a second one
  uint64_t om_cap = 0;
  uint32_t epoch = 0;
  unsigned long long* d_sz = nullptr;  // [0,32) F_k, [32,64) T_k, [64,96) list len, [96,128) alive, 127 overflow
  int* d_ovf = nullptr;
  unsigned long long* d_ctr = nullptr; // C_NCTR counters, then scratch (flag at 48)
  unsigned long long* h_pin = nullptr; // 256 pinned slots: [0,128) sizes, [128,160) alive, [192,..) counters, H_EPOCH
  uint32_t *heavy_rows = nullptr, *heavy_chunks = nullptr, *heavy_sat = nullptr, *heavy_cnt = nullptr;
  uint64_t heavy_gen = ~0ull;          // LSpM generation the heavy buffers were sized for
  uint32_t* frows = nullptr;           // group filter: compacted candidate rows of the center
  uint64_t frows_cap = 0;
  uint32_t* sat = nullptr;             // push form: two row-mark bitmaps (ping-pong)
  uint64_t sat_cap = 0;
  uint32_t* cand = nullptr;            // candidate bitmaps of the running plan (stable for graph replay)
  uint64_t cand_words = 0;
  OutTab* h_tab = nullptr;             // pinned: this execute's phase-2 output pointers
  OutTab* d_tab = nullptr;             // device copy (copied inside the phase-2 work)
  char* p2 = nullptr;                  // phase-2 scratch (unsorted rows + sort temp), grow-only
  uint64_t p2_cap = 0;
  uint32_t* d_epoch = nullptr;         // device base epoch of the current launch sequence
  uint32_t epoch_next = 1, seq_base = 1, seq_off = 0;
  // world > 1 (peer exchange): candidate bitmaps, change words and barrier flags
  // in a symmetric region; barrier generations base + off (device-resident base)
  SymRegion sym;
  uint64_t sym_cand_words = 0;
  SymRegion gath;                      // world > 1: rows of every rank, read by rank 0
  uint64_t gath_cap = 0;               // bytes per rank
  unsigned long long* d_bar = nullptr;  // device copy of the barrier generation base
  uint64_t bar_next = 1, bar_base = 1;
  uint32_t bar_off = 0;
  uint64_t ws_gen = 0;                 // bumped whenever a workspace buffer moves
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    uint64_t ws_gen = 0, lspm_gen = 0;
    uint32_t flags = 0, n_lb = 0, off0 = 0, n_bar = 0, bar0 = 0;
    std::vector<int> launches;  // kernel launches inside the graph, per kernel class
    uint64_t filter_main = 0, push_and = 0, n_exchanges = 0;
  };
  std::unordered_map<uint64_t, GraphEntry> graphs;  // (plan uid << 3 | phase tag) -> captured work
  std::unordered_set<uint64_t> seen;                // keys run once without capture
};

// Small persistent host thread pool (hostio.cu): run(f) calls f(i) on every
// worker i and waits.  Used for the pageable -> pinned staging memcpys.
struct HostWorkers {
  explicit HostWorkers(int n);
  ~HostWorkers();
  void run(const std::function<void(int)>& f);
  size_t size() const { return th.size(); }
 private:
  void loop(int idx);
  std::vector<std::thread> th;
  std::mutex mu;
  std::condition_variable cv, done_cv;
  std::function<void(int)> job;
  uint64_t gen = 0;
  int pending = 0;
  bool stop = false;
};

// Ring of pinned chunks for H2D of pageable caller arrays (hostio.cu).
struct StageRing {
  static constexpr int K = 4;
  static constexpr size_t CHUNK = 32u << 20;
  void* buf[K] = {};
  cudaEvent_t ev[K] = {};
  bool used[K] = {};
  uint64_t next = 0;
};

// Caching pool of pinned host blocks (power-of-two size classes >= 64 KiB)
// for result rows; bounded, the rest is released.
struct PinnedPool {
  static constexpr size_t CAP = 8ull << 30;
  std::multimap<size_t, void*> free_blocks;
  size_t cached = 0;
  void* get(size_t bytes, size_t* cls);
  void put(void* p, size_t cls);
  void clear();
};

}  // namespace gsm

// In-process communicator: `world` ranks, one host thread each (any devices).
// Collectives rendezvous on a generation barrier and copy device buffers
// directly (cudaMemcpyPeerAsync), standing in for NCCL when all ranks live in
// one process (tests on one GPU, or one process driving several GPUs).
struct gsmart_comm {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptr;
  std::vector<int> dev;
  std::vector<unsigned long long> val;
  std::vector<std::string> blob;  // host all-gather of byte strings
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct gsmart_ctx {
  gsmart_config cfg{};
  cudaStream_t st = nullptr;
  cudaMemPool_t pool = nullptr;  // the context's device memory pool (dalloc)
  bool own_stream = false;
  bool poisoned = false;
  std::string err;
  int sm_count = 148;
  uint32_t N = 0, P = 0;
  uint64_t n_triples = 0;
  uint32_t *d_s = nullptr, *d_p = nullptr, *d_o = nullptr;
  int pred_bytes = 1;
  gsm::Lspm f[2];
  std::vector<uint8_t> keep[2];  // labels each format holds (P + 1 flags) since the last build
  uint64_t* lm_keys = nullptr;    // build-time hand-off: the CSR's unique (s, p, o) keys (label-major source)
  unsigned long long lm_keys_n = 0;
  gsm::LabelMajor lm;
  gsm::LabelMajor lm_in;     // world > 1: label-major entries whose OBJECT is this rank's (stored as (o, s))
  gsm::Partition part;       // world > 1: vertex ranges of the ranks
  gsm::Dict dict;            // f4: terms of the last gsmart_ingest_ntriples
  std::unique_ptr<gsm::SockChan> chan;  // world > 1, ranks are processes
  uint32_t exchange = GSMART_XCHG_PEER;
  bool use_tma = true;        // GSMART_NO_TMA=1: plain loads instead of cp.async.bulk staging (A/B)
  uint64_t push_min = 1ull << 16;  // smallest label streamed by the push form (GSMART_PUSH_MIN, A/B)
  bool l2_persist = false;    // GSMART_L2_PERSIST=1: persisting L2 window over the candidate bitmaps (A/B)
  // push/pull choice per plan (uid -> lspm_gen, per group per edge), DESIGN.md §5
  std::unordered_map<uint64_t, std::pair<uint64_t, std::vector<std::vector<uint8_t>>>> push_cache;
  std::unordered_map<uint64_t, unsigned long long> plan_cost;  // uid -> work of its last execute (batch start order)
  struct P2Guess { uint64_t gen = 0; uint32_t flags = 0; std::vector<uint64_t> F; };
  std::unordered_map<uint64_t, P2Guess> p2_guess;
  uint32_t spec_test = 0;  // GSMART_SPEC_TEST=1: every speculation guesses a wrong row count (tests)  // uid -> level sizes of its last execute (speculative phase 2)
  uint64_t lspm_gen = 0;
  int filter_variant = 6;               // FilterArgs::variant bits + 4: row-list path (GSMART_FILTER_VARIANT)
  unsigned long long* d_ctr = nullptr;  // load/build scratch
  unsigned long long* h_pin = nullptr;
  ncclComm_t comm = nullptr;     // world > 1 with NCCL
  gsmart_comm* lcomm = nullptr;  // world > 1 with an in-process communicator
  int rank = 0, world = 1;
  std::vector<std::unique_ptr<gsm::Slot>> slots;
  std::unique_ptr<gsm::HostWorkers> workers;  // staging memcpy threads (lazy)
  gsm::StageRing ring;                        // pinned H2D staging chunks (lazy)
  gsm::PinnedPool pinned;                     // pinned blocks for result rows
  uint64_t cap() const { return cfg.max_result_rows ? cfg.max_result_rows : 0x7fffffffull; }
};

struct gsmart_result {
  gsmart_ctx* ctx = nullptr;
  cudaStream_t st = nullptr;     // stream the result's memory is ordered on
  uint64_t n_rows = 0;
  uint32_t n_cols = 0;
  std::vector<uint32_t> var_of_col;
  uint32_t* d_rows = nullptr;
  uint32_t* h_rows = nullptr;      // pinned block of ctx->pinned (class h_cls)
  size_t h_cls = 0;
  bool host_valid = false;
  bool count_only = false;
  uint32_t* d_cand = nullptr;
  uint32_t n_words = 0, stride_words = 0;
  std::vector<int32_t> cand_slot;  // vertex -> slot or -1
  struct Lv { uint32_t var; uint64_t n; uint32_t* parent; uint32_t* bind; int32_t parent_level = -2; uint8_t* alive = nullptr; };
  std::vector<Lv> levels;
  std::vector<void*> owned;        // device allocations to free
  gsmart_stats stats{};
};

namespace gsm {

extern thread_local std::string g_static_err;

gsmart_status cuda_fail(gsmart_ctx* ctx, cudaError_t e, const char* what, int line);

#define FAIL(code, msg) \
  do {                  \
    ctx->err = (msg);   \
    return (code);      \
  } while (0)

#define CU(x)                                                         \
  do {                                                                \
    cudaError_t e_ = (x);                                             \
    if (e_ != cudaSuccess) return gsm::cuda_fail(ctx, e_, #x, __LINE__); \
  } while (0)

#define TRY(x)                      \
  do {                              \
    gsmart_status s_ = (x);         \
    if (s_ != GSMART_OK) return s_; \
  } while (0)

// Device memory: the caller's allocator hooks (gsmart_config.alloc/free) when
// given, else the stream-ordered allocator of the device's default pool.
template <typename T>
gsmart_status dalloc(gsmart_ctx* ctx, T** p, uint64_t count, cudaStream_t st) {
  *p = nullptr;
  size_t bytes = std::max<uint64_t>(count, 1) * sizeof(T);
  bytes = (bytes + 255) / 256 * 256;
  if (ctx->cfg.alloc) {
    *p = (T*)ctx->cfg.alloc(bytes, (void*)st, ctx->cfg.alloc_user);
    if (!*p) {
      ctx->err = "allocator hook returned NULL";
      return GSMART_E_OOM;
    }
    return GSMART_OK;
  }
  cudaError_t e = cudaMallocFromPoolAsync((void**)p, bytes, ctx->pool, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMallocFromPoolAsync", __LINE__);
  return GSMART_OK;
}
template <typename T>
gsmart_status dalloc(gsmart_ctx* ctx, T** p, uint64_t count) {
  return dalloc(ctx, p, count, ctx->st);
}

inline void dfree(gsmart_ctx* ctx, cudaStream_t st, void* p) {
  if (!p) return;
  if (ctx->cfg.free) ctx->cfg.free(p, (void*)st, ctx->cfg.alloc_user);
  else cudaFreeAsync(p, st);
}
inline void dfree(gsmart_ctx* ctx, void* p) { dfree(ctx, ctx->st, p); }

// stream-ordered scratch freed at scope exit
struct Scratch {
  gsmart_ctx* ctx;
  cudaStream_t st;
  std::vector<void*> ptrs;
  Scratch(gsmart_ctx* c, cudaStream_t s) : ctx(c), st(s) {}
  explicit Scratch(gsmart_ctx* c) : ctx(c), st(c->st) {}
  ~Scratch() {
    for (void* p : ptrs) dfree(ctx, st, p);
  }
  template <typename T>
  gsmart_status get(T** p, uint64_t count) {
    gsmart_status s = dalloc(ctx, p, count, st);
    if (s == GSMART_OK) ptrs.push_back((void*)*p);
    return s;
  }
};

gsmart_status readback(gsmart_ctx* ctx, cudaStream_t st, unsigned long long* h_pin, const unsigned long long* dev,
                       int n, unsigned long long* host);

void slots_free(gsmart_ctx* ctx);
// ingest.cu: release the dictionary (new data loaded, or destroy)
void dict_free(gsmart_ctx* ctx);
// runtime.cu: release both LSpM formats and the label-major lists
void free_lspm(gsmart_ctx* ctx);
// wait for every stream of this context (ranks sharing a device never wait on each other's streams)
gsmart_status ctx_sync(gsmart_ctx* ctx);

// symheap.cu: host all-gather / barrier over the ranks (in-process comm or
// sockets), symmetric regions, device barrier across ranks
gsmart_status host_allgather(gsmart_ctx* ctx, const void* mine, size_t n, void* all);
gsmart_status host_barrier(gsmart_ctx* ctx);
size_t sym_granularity(gsmart_ctx* ctx);
gsmart_status sym_alloc(gsmart_ctx* ctx, uint64_t my_off, uint64_t my_bytes, SymRegion* out);
void sym_free(gsmart_ctx* ctx, SymRegion* R);

// hostio.cu
bool host_is_pinned(const void* p);
gsmart_status h2d_staged(gsmart_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st);
void stage_ring_free(gsmart_ctx* ctx);
gsmart_status rows_to_host(gsmart_ctx* ctx, gsmart_result* r, cudaStream_t st);

// bitmap words [lo, hi) of rank q's vertex range (empty range: 0, 0)
inline uint32_t part_word_lo(const gsmart_ctx* ctx, int q) {
  return ctx->part.v[q] < ctx->part.v[q + 1] ? ctx->part.v[q] / 32 : 0u;
}
inline uint32_t part_word_hi(const gsmart_ctx* ctx, int q) {
  return ctx->part.v[q] < ctx->part.v[q + 1] ? (ctx->part.v[q + 1] + 31) / 32 : 0u;
}

// ---- collectives of the baseline exchange (NCCL or the in-process communicator), comm.cu
// In-place all-gather of the ranks' word ranges of a replicated bitmap.
gsmart_status coll_allgatherv(gsmart_ctx* ctx, cudaStream_t st, uint32_t* bm);
// Host values of all ranks (blocking).
gsmart_status coll_allgather_host(gsmart_ctx* ctx, cudaStream_t st, unsigned long long v,
                                  std::vector<unsigned long long>* out);
// Rank r's send_bytes[r] bytes land at recv + sum_{q<r} send_bytes[q] on rank 0 (blocking).
gsmart_status coll_gather_root(gsmart_ctx* ctx, cudaStream_t st, const void* send, void* recv,
                               const std::vector<unsigned long long>& send_bytes);

}  // namespace gsm
