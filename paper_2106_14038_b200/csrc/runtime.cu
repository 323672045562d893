// C-ABI implementation: context, device memory, LSpM build orchestration and
// the level-synchronous executor (§5-§8).  Host code only
// sequences kernels from kernels.cu on the ctx stream; every data-path step
// runs on the GPU.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "gsmart.h"
#include "internal.h"
#include "kernels.h"
#include "nccl_shim.h"

using namespace gsm;

#define GSM_STR2(x) #x
#define GSM_STR(x) GSM_STR2(x)

namespace {

enum Kid {
  K_BUILD_PACK = 0, K_BUILD_SORT, K_BUILD_UNIQUE, K_BUILD_ROWPTR, K_SEED, K_FILTER, K_BITMAP, K_COMPACT,
  K_SCAN, K_EXPAND_SEG, K_EXPAND_COUNT, K_EXPAND_EMIT, K_PRUNE, K_ENUMERATE, K_SORT_ROWS, K_COLLECTIVE
};
const char* kKernelNames[GSMART_NKERNELS] = {
    "build_pack", "build_sort", "build_unique", "build_rowptr", "seed", "group_filter", "bitmap",
    "compact", "scan", "expand_seg", "expand_count", "expand_emit", "prune", "enumerate", "sort_rows",
    "collective"};

struct Lspm {
  uint32_t* rp = nullptr;
  uint32_t* col = nullptr;
  void* pred = nullptr;
  uint64_t nnz = 0;
  bool built = false;
  unsigned long long heavy_rows = 0, heavy_chunks = 0;
};

int bits_for(uint64_t v) {  // bits to represent values in [0, v]
  int b = 1;
  while (b < 64 && (v >> b) != 0) b++;
  return b;
}

}  // namespace

struct gsmart_ctx {
  gsmart_config cfg{};
  cudaStream_t st = nullptr;
  bool own_stream = false;
  bool poisoned = false;
  std::string err;
  int sm_count = 148;
  uint32_t N = 0, P = 0;
  uint64_t n_triples = 0;
  uint32_t *d_s = nullptr, *d_p = nullptr, *d_o = nullptr;
  int pred_bytes = 1;
  Lspm f[2];
  unsigned long long* d_ctr = nullptr;  // C_NCTR counters, then scratch slots
  unsigned long long* h_pin = nullptr;  // pinned readback slots
  ncclComm_t comm = nullptr;
  uint64_t cap() const { return cfg.max_result_rows ? cfg.max_result_rows : 0x7fffffffull; }
};

struct gsmart_result {
  gsmart_ctx* ctx = nullptr;
  uint64_t n_rows = 0;
  uint32_t n_cols = 0;
  std::vector<uint32_t> var_of_col;
  uint32_t* d_rows = nullptr;
  std::vector<uint32_t> h_rows;
  bool host_valid = false;
  bool count_only = false;
  uint32_t* d_cand = nullptr;
  uint32_t n_words = 0, stride_words = 0;
  std::vector<int32_t> cand_slot;  // vertex -> slot or -1
  struct Lv { uint32_t var; uint64_t n; uint32_t* parent; uint32_t* bind; };
  std::vector<Lv> levels;
  std::vector<void*> owned;        // device allocations to free
  gsmart_stats stats{};
};

static thread_local std::string g_static_err;

// ------------------------------------------------------------------------ errors / memory
#define FAIL(code, msg)            \
  do {                             \
    ctx->err = (msg);              \
    return (code);                 \
  } while (0)

static gsmart_status cuda_fail(gsmart_ctx* ctx, cudaError_t e, const char* what, int line) {
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    ctx->err = std::string("device out of memory at ") + what;
    return GSMART_E_OOM;
  }
  ctx->poisoned = true;
  ctx->err = std::string("CUDA error '") + cudaGetErrorString(e) + "' at " + what + " (runtime.cu:" +
             std::to_string(line) + ")";
  return GSMART_E_CUDA;
}

#define CU(x)                                                    \
  do {                                                           \
    cudaError_t e_ = (x);                                        \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #x, __LINE__); \
  } while (0)

#define TRY(x)                       \
  do {                               \
    gsmart_status s_ = (x);          \
    if (s_ != GSMART_OK) return s_;  \
  } while (0)

template <typename T>
static gsmart_status dalloc(gsmart_ctx* ctx, T** p, uint64_t count) {
  *p = nullptr;
  size_t bytes = std::max<uint64_t>(count, 1) * sizeof(T);
  bytes = (bytes + 255) / 256 * 256;
  cudaError_t e = cudaMallocAsync((void**)p, bytes, ctx->st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMallocAsync", __LINE__);
  return GSMART_OK;
}

static void dfree(gsmart_ctx* ctx, void* p) {
  if (p) cudaFreeAsync(p, ctx->st);
}

// stream-ordered scratch freed at scope exit
struct Scratch {
  gsmart_ctx* ctx;
  std::vector<void*> ptrs;
  explicit Scratch(gsmart_ctx* c) : ctx(c) {}
  ~Scratch() {
    for (void* p : ptrs) dfree(ctx, p);
  }
  template <typename T>
  gsmart_status get(T** p, uint64_t count) {
    gsmart_status s = dalloc(ctx, p, count);
    if (s == GSMART_OK) ptrs.push_back((void*)*p);
    return s;
  }
};

static gsmart_status readback(gsmart_ctx* ctx, const unsigned long long* dev, int n, unsigned long long* host) {
  CU(cudaMemcpyAsync(ctx->h_pin, dev, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->st));
  CU(cudaStreamSynchronize(ctx->st));
  memcpy(host, ctx->h_pin, n * sizeof(unsigned long long));
  return GSMART_OK;
}

// ------------------------------------------------------------------------ profiling
struct Prof {
  gsmart_ctx* ctx;
  gsmart_stats* st;
  bool on;
  struct Rec { int kid; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  int cur = -1;
  cudaEvent_t cur_a = nullptr;
  Prof(gsmart_ctx* c, gsmart_stats* s, bool enable) : ctx(c), st(s), on(enable) {}
  void begin(int kid) {
    if (!on) return;
    cur = kid;
    cudaEventCreate(&cur_a);
    cudaEventRecord(cur_a, ctx->st);
  }
  void end() {
    if (!on || cur < 0) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, ctx->st);
    recs.push_back({cur, cur_a, b});
    cur = -1;
  }
  void flush() {  // after a stream sync
    for (auto& r : recs) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) st->ms_kernel[r.kid] += ms;
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    recs.clear();
  }
  ~Prof() { flush(); }
};

// ------------------------------------------------------------------------ ABI: misc
extern "C" int gsmart_abi_version(void) { return GSMART_ABI_VERSION; }

extern "C" const char* gsmart_build_info(void) {
  return "gsmart sm_100a build " __DATE__ " " __TIME__ " (cuda " GSM_STR(__CUDACC_VER_MAJOR__) "." GSM_STR(
      __CUDACC_VER_MINOR__) ")";
}

extern "C" const char* gsmart_last_error(const gsmart_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_static_err.c_str();
}

extern "C" gsmart_status gsmart_get_nccl_id(void* out128) {
  if (!out128) return GSMART_E_INVALID_ARG;
  const NcclApi* api = nccl_api();
  if (!api) {
    g_static_err = "NCCL library (libnccl.so.2) not loadable";
    return GSMART_E_NCCL;
  }
  ncclUniqueId id;
  if (api->GetUniqueId(&id) != 0) {
    g_static_err = "ncclGetUniqueId failed";
    return GSMART_E_NCCL;
  }
  memcpy(out128, &id, sizeof(id));
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_create(const gsmart_config* cfg, gsmart_ctx** out) {
  if (!cfg || !out) {
    g_static_err = "null argument";
    return GSMART_E_INVALID_ARG;
  }
  *out = nullptr;
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) {
    g_static_err = "bad rank/world";
    return GSMART_E_INVALID_ARG;
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    g_static_err = std::string("no CUDA device: ") + cudaGetErrorString(e);
    return GSMART_E_CUDA;
  }
  if (cfg->device < 0 || cfg->device >= ndev) {
    g_static_err = "device ordinal out of range";
    return GSMART_E_INVALID_ARG;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess || prop.major != 10) {
    g_static_err = "this library is built for sm_100a only (B200)";
    return GSMART_E_CUDA;
  }
  auto ctx = std::make_unique<gsmart_ctx>();
  ctx->cfg = *cfg;
  ctx->sm_count = prop.multiProcessorCount;
  if (cudaSetDevice(cfg->device) != cudaSuccess) {
    g_static_err = "cudaSetDevice failed";
    return GSMART_E_CUDA;
  }
  if (cfg->stream) {
    ctx->st = (cudaStream_t)cfg->stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking) != cudaSuccess) {
      g_static_err = "stream create failed";
      return GSMART_E_CUDA;
    }
    ctx->own_stream = true;
  }
  // keep freed blocks in the pool (stream-ordered allocator as a caching allocator)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, cfg->device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (cudaMalloc(&ctx->d_ctr, 64 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMallocHost(&ctx->h_pin, 64 * sizeof(unsigned long long)) != cudaSuccess) {
    g_static_err = "context allocation failed";
    return GSMART_E_OOM;
  }
  if (cfg->world > 1) {
    const NcclApi* api = nccl_api();
    if (!api || !cfg->nccl_unique_id) {
      g_static_err = "world > 1 needs NCCL and a unique id";
      return GSMART_E_NCCL;
    }
    ncclUniqueId id;
    memcpy(&id, cfg->nccl_unique_id, sizeof(id));
    if (api->CommInitRank(&ctx->comm, cfg->world, id, cfg->rank) != 0) {
      g_static_err = "ncclCommInitRank failed";
      return GSMART_E_NCCL;
    }
  }
  *out = ctx.release();
  return GSMART_OK;
}

static void free_lspm(gsmart_ctx* ctx) {
  for (auto& f : ctx->f) {
    dfree(ctx, f.rp);
    dfree(ctx, f.col);
    dfree(ctx, f.pred);
    f = Lspm();
  }
}

extern "C" void gsmart_destroy(gsmart_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->cfg.device);
  free_lspm(ctx);
  dfree(ctx, ctx->d_s);
  dfree(ctx, ctx->d_p);
  dfree(ctx, ctx->d_o);
  cudaStreamSynchronize(ctx->st);
  if (ctx->comm) {
    const NcclApi* api = nccl_api();
    if (api) api->CommDestroy(ctx->comm);
  }
  cudaFree(ctx->d_ctr);
  cudaFreeHost(ctx->h_pin);
  if (ctx->own_stream) cudaStreamDestroy(ctx->st);
  delete ctx;
}

// ------------------------------------------------------------------------ load
__global__ void k_validate(const uint32_t* s, const uint32_t* p, const uint32_t* o, uint64_t n, uint32_t N,
                           uint32_t P, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (s[i] >= N || o[i] >= N || p[i] == 0 || p[i] > P) atomicAdd(bad, 1ull);
}

extern "C" gsmart_status gsmart_load_triples(gsmart_ctx* ctx, const uint32_t* s, const uint32_t* p,
                                             const uint32_t* o, uint64_t n, uint32_t n_entities,
                                             uint32_t n_predicates, uint32_t flags) {
  if (!ctx) return GSMART_E_INVALID_ARG;
  if (ctx->poisoned) return GSMART_E_CUDA;
  if (n && (!s || !p || !o)) FAIL(GSMART_E_INVALID_ARG, "null triple arrays");
  if (n_entities == 0 || n_entities >= 0x80000000u) FAIL(GSMART_E_INVALID_ARG, "n_entities must be in [1, 2^31)");
  if (n_predicates == 0 || n_predicates > 65535) FAIL(GSMART_E_INVALID_ARG, "n_predicates must be in [1, 65535]");
  if (n >= 0xffffffffull) FAIL(GSMART_E_INVALID_ARG, "n must be < 2^32 - 1");
  if (flags != GSMART_PTR_HOST && flags != GSMART_PTR_DEVICE) FAIL(GSMART_E_INVALID_ARG, "flags must be PTR_HOST or PTR_DEVICE");
  CU(cudaSetDevice(ctx->cfg.device));
  if (flags == GSMART_PTR_HOST) {
    for (uint64_t i = 0; i < n; i++)
      if (s[i] >= n_entities || o[i] >= n_entities || p[i] == 0 || p[i] > n_predicates)
        FAIL(GSMART_E_INVALID_ARG, "triple id out of range at index " + std::to_string(i));
  }
  free_lspm(ctx);
  dfree(ctx, ctx->d_s);
  dfree(ctx, ctx->d_p);
  dfree(ctx, ctx->d_o);
  ctx->d_s = ctx->d_p = ctx->d_o = nullptr;
  ctx->n_triples = 0;
  TRY(dalloc(ctx, &ctx->d_s, n));
  TRY(dalloc(ctx, &ctx->d_p, n));
  TRY(dalloc(ctx, &ctx->d_o, n));
  cudaMemcpyKind kind = flags == GSMART_PTR_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  if (n) {
    CU(cudaMemcpyAsync(ctx->d_s, s, n * 4, kind, ctx->st));
    CU(cudaMemcpyAsync(ctx->d_p, p, n * 4, kind, ctx->st));
    CU(cudaMemcpyAsync(ctx->d_o, o, n * 4, kind, ctx->st));
  }
  if (flags == GSMART_PTR_DEVICE && n) {
    CU(cudaMemsetAsync(ctx->d_ctr + 32, 0, 8, ctx->st));
    k_validate<<<(unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->sm_count * 16), 256, 0, ctx->st>>>(
        ctx->d_s, ctx->d_p, ctx->d_o, n, n_entities, n_predicates, ctx->d_ctr + 32);
    CU(cudaGetLastError());
    unsigned long long bad = 0;
    TRY(readback(ctx, ctx->d_ctr + 32, 1, &bad));
    if (bad) FAIL(GSMART_E_INVALID_ARG, std::to_string(bad) + " triples with ids out of range");
  }
  ctx->n_triples = n;
  ctx->N = n_entities;
  ctx->P = n_predicates;
  ctx->pred_bytes = n_predicates <= 255 ? 1 : 2;
  CU(cudaStreamSynchronize(ctx->st));  // caller may free / reuse its buffers after return
  return GSMART_OK;
}

// ------------------------------------------------------------------------ build (a1)
static gsmart_status build_format(gsmart_ctx* ctx, int fmt, const uint8_t* d_keep) {
  Lspm& L = ctx->f[fmt];
  const uint64_t n = ctx->n_triples;
  const uint32_t N = ctx->N;
  const int nb = bits_for(N - 1), pb = bits_for(ctx->P);
  const int sh_pred = nb, sh_row = nb + pb, drop_bit = 2 * nb + pb;
  if (drop_bit >= 64) FAIL(GSMART_E_UNSUPPORTED, "packed (row,pred,col) key exceeds 63 bits");
  Scratch sc(ctx);
  uint64_t *keys = nullptr, *keys2 = nullptr;
  uint32_t* flags = nullptr;
  TRY(sc.get(&keys, n));
  TRY(sc.get(&keys2, n));
  TRY(sc.get(&flags, n + 1));
  const uint32_t* rowv = fmt == 0 ? ctx->d_s : ctx->d_o;
  const uint32_t* colv = fmt == 0 ? ctx->d_o : ctx->d_s;
  unsigned long long* tot = ctx->d_ctr + 40;
  if (n) {
    CU(launch_pack_keys(rowv, ctx->d_p, colv, n, d_keep, sh_row, sh_pred, drop_bit, keys, ctx->st));
    size_t tb = sort_keys_tmp_bytes(n, drop_bit + 1);
    void* tmp = nullptr;
    TRY(sc.get((char**)&tmp, tb));
    CU(sort_keys_u64(tmp, tb, keys, keys2, n, drop_bit + 1, ctx->st));
    CU(launch_unique_flags(keys2, n, drop_bit, flags, ctx->st));
    void* stmp = nullptr;
    TRY(sc.get((char**)&stmp, scan_tmp_bytes(n)));
    CU(scan_exclusive_u32(flags, flags, n, tot, stmp, ctx->st, nullptr));
  } else {
    CU(cudaMemsetAsync(tot, 0, 8, ctx->st));
  }
  unsigned long long M = 0;
  TRY(readback(ctx, tot, 1, &M));
  if (M >= 0xffffffffull) FAIL(GSMART_E_UNSUPPORTED, "more than 2^32-2 entries in one LSpM format");
  TRY(dalloc(ctx, &L.rp, (uint64_t)N + 1));
  TRY(dalloc(ctx, &L.col, M));
  TRY(dalloc(ctx, (uint8_t**)&L.pred, M * ctx->pred_bytes));
  CU(cudaMemsetAsync(L.rp, 0, ((uint64_t)N + 1) * 4, ctx->st));
  if (n) CU(launch_unpack(keys2, n, flags, drop_bit, sh_row, sh_pred, L.col, L.pred, ctx->pred_bytes, L.rp, ctx->st));
  {
    void* stmp = nullptr;
    TRY(sc.get((char**)&stmp, scan_tmp_bytes((uint64_t)N + 1)));
    CU(scan_exclusive_u32(L.rp, L.rp, (uint64_t)N + 1, tot, stmp, ctx->st, nullptr));
  }
  CU(cudaMemsetAsync(ctx->d_ctr + 42, 0, 16, ctx->st));
  CU(launch_heavy_stats(L.rp, N, ctx->d_ctr + 42, ctx->st));
  unsigned long long hv[2];
  TRY(readback(ctx, ctx->d_ctr + 42, 2, hv));
  L.heavy_rows = hv[0];
  L.heavy_chunks = hv[1];
  L.nnz = M;
  L.built = true;
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_build_lspm(gsmart_ctx* ctx, const uint32_t* keep_preds, uint32_t n_keep,
                                           uint32_t formats) {
  if (!ctx) return GSMART_E_INVALID_ARG;
  if (ctx->poisoned) return GSMART_E_CUDA;
  if (ctx->N == 0) FAIL(GSMART_E_STATE, "gsmart_load_triples must be called first");
  if (formats == 0 || (formats & ~(GSMART_CSR | GSMART_CSC))) FAIL(GSMART_E_INVALID_ARG, "formats must be CSR|CSC");
  if (n_keep && !keep_preds) FAIL(GSMART_E_INVALID_ARG, "null keep_preds");
  CU(cudaSetDevice(ctx->cfg.device));
  std::vector<uint8_t> keep(ctx->P + 1, n_keep ? 0 : 1);
  keep[0] = 0;
  for (uint32_t i = 0; i < n_keep; i++) {
    if (keep_preds[i] == 0 || keep_preds[i] > ctx->P) FAIL(GSMART_E_INVALID_ARG, "keep_preds id out of range");
    keep[keep_preds[i]] = 1;
  }
  free_lspm(ctx);
  Scratch sc(ctx);
  uint8_t* d_keep = nullptr;
  TRY(sc.get(&d_keep, keep.size()));
  CU(cudaMemcpyAsync(d_keep, keep.data(), keep.size(), cudaMemcpyHostToDevice, ctx->st));
  for (int fmt = 0; fmt < 2; fmt++)
    if (formats & (fmt == 0 ? GSMART_CSR : GSMART_CSC)) TRY(build_format(ctx, fmt, d_keep));
  CU(cudaStreamSynchronize(ctx->st));
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_lspm_get(const gsmart_ctx* ctx, uint32_t format, gsmart_lspm_view* out) {
  if (!ctx || !out || (format != GSMART_CSR && format != GSMART_CSC)) return GSMART_E_INVALID_ARG;
  const Lspm& L = ctx->f[format == GSMART_CSR ? 0 : 1];
  if (!L.built) return GSMART_E_STATE;
  out->n_rows = ctx->N;
  out->nnz = L.nnz;
  out->pred_bytes = (uint32_t)ctx->pred_bytes;
  out->row_ptr = L.rp;
  out->col = L.col;
  out->pred = L.pred;
  return GSMART_OK;
}

// ------------------------------------------------------------------------ plan
extern "C" gsmart_status gsmart_plan(gsmart_ctx* ctx, const gsmart_query* q, uint32_t traversal,
                                     gsmart_plan_t** out) {
  if (!out) return GSMART_E_INVALID_ARG;
  *out = nullptr;
  auto p = std::make_unique<gsmart_plan_t>();
  std::string err;
  gsmart_status s = build_plan(q, traversal, p.get(), &err);
  if (s != GSMART_OK) {
    if (ctx) ctx->err = err; else g_static_err = err;
    return s;
  }
  *out = p.release();
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_plan_describe(const gsmart_plan_t* plan, char* buf, size_t cap, size_t* need) {
  if (!plan) return GSMART_E_INVALID_ARG;
  std::string js = describe_plan(*plan);
  if (need) *need = js.size() + 1;
  if (buf && cap) {
    size_t k = std::min(cap - 1, js.size());
    memcpy(buf, js.data(), k);
    buf[k] = 0;
  }
  return GSMART_OK;
}

extern "C" void gsmart_plan_free(gsmart_plan_t* plan) { delete plan; }

// ------------------------------------------------------------------------ execute (a2..a9)
namespace {

struct Exec {
  gsmart_ctx* ctx;
  const gsmart_plan_t* plan;
  uint32_t flags;
  gsmart_result* R;
  Prof prof;
  Scratch sc;
  uint32_t W = 0, Wpad = 0;
  std::vector<int32_t> slot;  // vertex -> cand slot
  FmtAny fa[2];
  uint32_t *heavy_rows = nullptr, *heavy_chunks = nullptr, *heavy_sat = nullptr, *heavy_cnt = nullptr;
  uint64_t cap_heavy_rows = 0;
  int launches[GSMART_NKERNELS] = {0};

  Exec(gsmart_ctx* c, const gsmart_plan_t*p, uint32_t fl, gsmart_result* r)
      : ctx(c), plan(p), flags(fl), R(r), prof(c, &r->stats, (fl & GSMART_PROFILE) != 0), sc(c) {}

  uint32_t* cand(uint32_t vertex) { return R->d_cand + (uint64_t)slot[vertex] * Wpad; }

  gsmart_status alloc_result(void** p, uint64_t bytes) {
    TRY(dalloc(ctx, (char**)p, bytes));
    R->owned.push_back(*p);
    return GSMART_OK;
  }

  gsmart_status seeds_and_guards(bool* empty) {
    const uint32_t N = ctx->N;
    *empty = false;
    for (auto& sd : plan->seeds)
      if (sd.cid >= N) *empty = true;
    for (auto& g : plan->guards)
      if (g.s >= N || g.o >= N) *empty = true;
    for (auto& sd : plan->seeds)
      if (sd.label > ctx->P) *empty = true;
    for (auto& g : plan->guards)
      if (g.label > ctx->P) *empty = true;
    if (*empty) {  // a constant outside the data: every candidate set is empty (R12)
      if (!plan->vars.empty())
        CU(cudaMemsetAsync(R->d_cand, 0, (size_t)Wpad * plan->vars.size() * 4, ctx->st));
      return GSMART_OK;
    }
    std::vector<int> nseed(plan->n_vertices, 0);
    for (auto& sd : plan->seeds) nseed[sd.var]++;
    prof.begin(K_BITMAP);
    for (uint32_t v : plan->vars) {
      if (nseed[v]) CU(cudaMemsetAsync(cand(v), 0, (size_t)Wpad * 4, ctx->st));
      else { CU(launch_fill_ones(cand(v), Wpad, N, ctx->st)); launches[K_BITMAP]++; }
    }
    prof.end();
    int* flag = (int*)(ctx->d_ctr + 48);
    if (!plan->guards.empty()) {
      int one = 1;
      CU(cudaMemcpyAsync(flag, &one, 4, cudaMemcpyHostToDevice, ctx->st));
      prof.begin(K_SEED);
      for (auto& g : plan->guards) {
        CU(launch_guard(fa[0], ctx->pred_bytes, g.s, g.label, g.o, flag, ctx->st));
        launches[K_SEED]++;
      }
      prof.end();
    }
    uint32_t* tmp = nullptr;
    std::vector<int> done(plan->n_vertices, 0);
    for (auto& sd : plan->seeds) {
      uint32_t* dst = cand(sd.var);
      bool first = done[sd.var]++ == 0;
      if (!first) {
        if (!tmp) TRY(sc.get(&tmp, Wpad));
        CU(cudaMemsetAsync(tmp, 0, (size_t)Wpad * 4, ctx->st));
      }
      prof.begin(K_SEED);
      CU(launch_seed_scatter(fa[sd.dir == OUT ? 0 : 1], ctx->pred_bytes, sd.cid, sd.label, first ? dst : tmp,
                             ctx->d_ctr, ctx->sm_count, ctx->st));
      launches[K_SEED]++;
      prof.end();
      if (!first) {
        prof.begin(K_BITMAP);
        CU(launch_and_inplace(dst, tmp, Wpad, ctx->st));
        launches[K_BITMAP]++;
        prof.end();
      }
    }
    if (!plan->guards.empty() && !plan->vars.empty()) {
      prof.begin(K_BITMAP);
      CU(launch_zero_if_flag(R->d_cand, (uint64_t)Wpad * plan->vars.size(), flag, ctx->st));
      launches[K_BITMAP]++;
      prof.end();
    }
    return GSMART_OK;
  }

  gsmart_status eval_group(const Group& g) {
    // split into launches of <= MAXG edges per direction (AND is associative)
    std::vector<const GroupEdge*> by[2];
    for (auto& e : g.edges) by[e.dir == OUT ? 0 : 1].push_back(&e);
    size_t done[2] = {0, 0};
    while (done[0] < by[0].size() || done[1] < by[1].size() || (by[0].empty() && by[1].empty())) {
      FilterArgs a;
      memset(&a, 0, sizeof a);
      a.f[0] = fa[0];
      a.f[1] = fa[1];
      for (int d = 0; d < 2; d++) {
        while (done[d] < by[d].size() && a.ne[d] < (uint32_t)MAXG) {
          const GroupEdge* e = by[d][done[d]++];
          GEdge& ge = a.e[d][a.ne[d]++];
          ge.label = e->label;
          ge.self = e->nbr == g.center ? 1u : 0u;
          ge.nbr = ge.self ? nullptr : cand(e->nbr);
        }
      }
      a.cand = cand(g.center);
      a.n_words = W;
      a.heavy_rows = heavy_rows;
      a.heavy_chunks = heavy_chunks;
      a.heavy_sat = heavy_sat;
      a.heavy_count = heavy_cnt;
      a.ctr = ctx->d_ctr;
      CU(cudaMemsetAsync(heavy_cnt, 0, 8, ctx->st));
      if (cap_heavy_rows) CU(cudaMemsetAsync(heavy_sat, 0, cap_heavy_rows * 4, ctx->st));
      prof.begin(K_FILTER);
      CU(launch_group_filter(a, ctx->pred_bytes, ctx->sm_count, ctx->st, &launches[K_FILTER]));
      prof.end();
      if (by[0].empty() && by[1].empty()) break;
    }
    return GSMART_OK;
  }

  gsmart_status compact(const uint32_t* bm, uint32_t** ids, uint64_t* count, bool result_owned) {
    void* tmp = nullptr;
    TRY(sc.get((char**)&tmp, compact_tmp_bytes(W)));
    unsigned long long* cnt = ctx->d_ctr + 50;
    prof.begin(K_COMPACT);
    CU(compact_count(bm, W, cnt, tmp, ctx->st, &launches[K_COMPACT]));
    prof.end();
    unsigned long long c = 0;
    TRY(readback(ctx, cnt, 1, &c));
    *count = c;
    if (result_owned) TRY(alloc_result((void**)ids, c * 4));
    else TRY(sc.get(ids, c));
    prof.begin(K_COMPACT);
    CU(compact_emit(bm, W, *ids, tmp, ctx->st, &launches[K_COMPACT]));
    prof.end();
    return GSMART_OK;
  }

  gsmart_status run() {
    const uint32_t N = ctx->N;
    const uint32_t nvar = (uint32_t)plan->vars.size();
    W = (N + 31) / 32;
    Wpad = (W + 31) / 32 * 32;
    R->n_words = W;
    R->stride_words = Wpad;
    slot.assign(plan->n_vertices, -1);
    for (uint32_t i = 0; i < nvar; i++) slot[plan->vars[i]] = (int32_t)i;
    R->cand_slot = slot;
    for (int d = 0; d < 2; d++) {
      fa[d].rp = ctx->f[d].rp;
      fa[d].col = ctx->f[d].col;
      fa[d].pred = ctx->f[d].pred;
    }
    CU(cudaMemsetAsync(ctx->d_ctr, 0, C_NCTR * 8, ctx->st));
    if (nvar) TRY(alloc_result((void**)&R->d_cand, (uint64_t)Wpad * nvar * 4));

    bool empty = false;
    TRY(seeds_and_guards(&empty));
    if (nvar == 0) {  // only guards (or nothing): one empty row iff all hold
      uint64_t rows = 0;
      if (!empty) {
        int flag = 1;
        if (!plan->guards.empty()) {
          CU(cudaMemcpyAsync(&flag, ctx->d_ctr + 48, 4, cudaMemcpyDeviceToHost, ctx->st));
          CU(cudaStreamSynchronize(ctx->st));
        }
        rows = flag ? 1 : 0;
      }
      R->n_rows = rows;
      R->host_valid = true;
      return GSMART_OK;
    }
    if (empty) {
      R->n_rows = 0;
      R->host_valid = true;
      R->stats.n_levels = (uint32_t)plan->levels.size();
      for (auto& L : plan->levels) R->levels.push_back({L.var, 0, nullptr, nullptr});
      return GSMART_OK;
    }

    // ---- a4: grouped incident-edge evaluation, forward then backward (refine)
    cap_heavy_rows = ctx->f[0].heavy_rows + ctx->f[1].heavy_rows;
    uint64_t cap_chunks = ctx->f[0].heavy_chunks + ctx->f[1].heavy_chunks;
    TRY(sc.get(&heavy_cnt, 2));
    TRY(sc.get(&heavy_rows, std::max<uint64_t>(cap_heavy_rows, 1)));
    TRY(sc.get(&heavy_sat, std::max<uint64_t>(cap_heavy_rows, 1)));
    TRY(sc.get(&heavy_chunks, 2 * std::max<uint64_t>(cap_chunks, 1)));
    for (auto& g : plan->groups) TRY(eval_group(g));
    if (!(flags & GSMART_NO_REFINE) && plan->groups.size() > 1)
      for (size_t i = plan->groups.size() - 1; i-- > 0;) TRY(eval_group(plan->groups[i]));

    // ---- a5/a6/a7: trie expansion in visitation order
    const uint32_t L = (uint32_t)plan->levels.size();
    std::vector<uint32_t*> par(L, nullptr), bnd(L, nullptr);
    std::vector<uint64_t> F(L, 0);
    const uint64_t cap = ctx->cap();
    TRY(compact(cand(plan->levels[0].var), &bnd[0], &F[0], false));
    R->stats.n_levels = L;
    R->stats.level_nodes[0] = F[0];
    if (F[0] > cap) {
      R->n_rows = F[0];
      FAIL(GSMART_E_RESULT_OVERFLOW, "trie level 0 exceeds max_result_rows");
    }
    uint32_t built = 1;
    for (uint32_t k = 1; k < L; k++) {
      if (F[k - 1] == 0) break;
      const Level& Lv = plan->levels[k];
      ExpandArgs a;
      memset(&a, 0, sizeof a);
      for (uint32_t j = 0; j < k; j++) {
        a.tab.parent[j] = par[j];
        a.tab.bind[j] = bnd[j];
      }
      a.k = k;
      a.n_parents = (uint32_t)F[k - 1];
      a.tree = Lv.tree_edge >= 0 ? 1 : 0;
      a.parent_level = Lv.parent_level;
      a.label = Lv.label;
      a.dir = Lv.dir == OUT ? 0 : 1;
      a.f[0] = fa[0];
      a.f[1] = fa[1];
      a.cand = cand(Lv.var);
      if (Lv.closing.size() > (size_t)MAXC) FAIL(GSMART_E_UNSUPPORTED, "more than 16 closing edges on one level");
      for (auto& c : Lv.closing) {
        ClosingDev& d = a.cl[a.ncl++];
        d.label = c.label;
        d.other_level = c.other_level;
        d.dir = c.dir == OUT ? 0 : 1;
        d.self = c.other_level == k ? 1u : 0u;
      }
      if (!a.tree) {
        uint32_t* list = nullptr;
        uint64_t ln = 0;
        TRY(compact(cand(Lv.var), &list, &ln, false));
        a.list = list;
        a.list_len = (uint32_t)ln;
      }
      a.ctr = ctx->d_ctr;
      TRY(sc.get(&a.seg_beg, F[k - 1]));
      TRY(sc.get(&a.seg_len, F[k - 1]));
      TRY(sc.get(&a.item_off, F[k - 1] + 1));
      prof.begin(K_EXPAND_SEG);
      CU(launch_expand_seg(a, ctx->pred_bytes, ctx->st));
      launches[K_EXPAND_SEG]++;
      prof.end();
      void* stmp = nullptr;
      TRY(sc.get((char**)&stmp, scan_tmp_bytes(F[k - 1] + 1)));
      unsigned long long* tot = ctx->d_ctr + 52;
      prof.begin(K_SCAN);
      CU(scan_exclusive_u32(a.item_off, a.item_off, F[k - 1], tot, stmp, ctx->st, &launches[K_SCAN]));
      prof.end();
      unsigned long long n_items = 0;
      TRY(readback(ctx, tot, 1, &n_items));
      if (n_items >= 0xffffffffull) FAIL(GSMART_E_RESULT_OVERFLOW, "expansion work items exceed 2^32");
      a.n_items = (uint32_t)n_items;
      TRY(sc.get(&a.item_node, n_items));
      TRY(sc.get(&a.item_cnt, n_items + 1));
      prof.begin(K_EXPAND_SEG);
      CU(launch_items_fill(a, ctx->st));
      launches[K_EXPAND_SEG]++;
      prof.end();
      prof.begin(K_EXPAND_COUNT);
      CU(launch_expand_pass(a, ctx->pred_bytes, false, ctx->sm_count, ctx->st));
      launches[K_EXPAND_COUNT]++;
      prof.end();
      void* stmp2 = nullptr;
      TRY(sc.get((char**)&stmp2, scan_tmp_bytes(n_items + 1)));
      prof.begin(K_SCAN);
      CU(scan_exclusive_u32(a.item_cnt, a.item_cnt, n_items, tot, stmp2, ctx->st, &launches[K_SCAN]));
      prof.end();
      unsigned long long n_child = 0;
      TRY(readback(ctx, tot, 1, &n_child));
      F[k] = n_child;
      R->stats.level_nodes[k] = n_child;
      if (n_child > cap) {
        R->n_rows = n_child;
        FAIL(GSMART_E_RESULT_OVERFLOW, "trie level " + std::to_string(k) + " exceeds max_result_rows");
      }
      TRY(sc.get(&par[k], n_child));
      TRY(sc.get(&bnd[k], n_child));
      a.out_parent = par[k];
      a.out_bind = bnd[k];
      prof.begin(K_EXPAND_EMIT);
      CU(launch_expand_pass(a, ctx->pred_bytes, true, ctx->sm_count, ctx->st));
      launches[K_EXPAND_EMIT]++;
      prof.end();
      built = k + 1;
    }
    for (uint32_t k = built; k < L; k++) F[k] = 0;
    const uint64_t n_rows = F[L - 1];

    // ---- a8: bottom-up pruning + level compaction (pruned trie is a result)
    std::vector<uint8_t*> alive(L, nullptr);
    std::vector<uint32_t*> newpos(L, nullptr);
    std::vector<uint64_t> A(L, 0);
    A[L - 1] = F[L - 1];
    if (n_rows) {
      prof.begin(K_PRUNE);
      for (uint32_t k = 0; k + 1 < L; k++) {
        TRY(sc.get(&alive[k], F[k]));
        CU(cudaMemsetAsync(alive[k], 0, F[k], ctx->st));
      }
      for (uint32_t k = L - 1; k >= 1; k--) {
        CU(launch_prune_mark(par[k], k == L - 1 ? nullptr : alive[k], (uint32_t)F[k], alive[k - 1], ctx->st));
        launches[K_PRUNE]++;
      }
      unsigned long long* tot = ctx->d_ctr + 54;
      for (uint32_t k = 0; k + 1 < L; k++) {
        TRY(sc.get(&newpos[k], F[k] + 1));
        CU(launch_u8_to_u32(alive[k], newpos[k], (uint32_t)F[k], ctx->st));
        void* stmp = nullptr;
        TRY(sc.get((char**)&stmp, scan_tmp_bytes(F[k] + 1)));
        CU(scan_exclusive_u32(newpos[k], newpos[k], F[k], tot, stmp, ctx->st, &launches[K_PRUNE]));
        unsigned long long a = 0;
        TRY(readback(ctx, tot, 1, &a));
        A[k] = a;
        launches[K_PRUNE]++;
      }
      prof.end();
    }
    R->levels.clear();
    LevelTab pt;
    memset(&pt, 0, sizeof pt);
    for (uint32_t k = 0; k < L; k++) {
      R->stats.level_alive[k] = n_rows ? A[k] : 0;
      gsmart_result::Lv lv{plan->levels[k].var, n_rows ? A[k] : 0, nullptr, nullptr};
      if (n_rows) {
        TRY(alloc_result((void**)&lv.bind, A[k] * 4));
        if (k > 0) TRY(alloc_result((void**)&lv.parent, A[k] * 4));
        prof.begin(K_PRUNE);
        CU(launch_compact_level(k > 0 ? par[k] : nullptr, bnd[k], k + 1 < L ? alive[k] : nullptr,
                                k + 1 < L ? newpos[k] : nullptr, k > 0 ? newpos[k - 1] : nullptr, (uint32_t)F[k],
                                lv.parent, lv.bind, ctx->st));
        launches[K_PRUNE]++;
        prof.end();
      }
      pt.parent[k] = lv.parent;
      pt.bind[k] = lv.bind;
      R->levels.push_back(lv);
    }
    R->n_rows = n_rows;

    // ---- a9: rows (variable-index column order), lexicographic sort
    if (!(flags & GSMART_COUNT_ONLY) && n_rows) {
      const uint32_t nc = nvar;
      std::vector<uint32_t> col_of_level(L);
      bool identity = true;
      for (uint32_t k = 0; k < L; k++) {
        col_of_level[k] = (uint32_t)plan->col_of[plan->levels[k].var];
        if (col_of_level[k] != k) identity = false;
      }
      uint32_t* rows = nullptr;
      TRY(identity ? alloc_result((void**)&rows, n_rows * nc * 4) : sc.get(&rows, n_rows * nc));
      prof.begin(K_ENUMERATE);
      CU(launch_enumerate(pt, L, col_of_level.data(), (uint32_t)n_rows, nc, rows, ctx->st));
      launches[K_ENUMERATE]++;
      prof.end();
      if (identity) {
        R->d_rows = rows;  // trie order == lexicographic order in variable-index order
      } else {
        TRY(alloc_result((void**)&R->d_rows, n_rows * nc * 4));
        size_t tb = sort_rows_tmp_bytes(n_rows, nc);
        void* tmp = nullptr;
        TRY(sc.get((char**)&tmp, tb));
        int key_bits = bits_for(N - 1);
        prof.begin(K_SORT_ROWS);
        CU(sort_rows(rows, R->d_rows, n_rows, nc, key_bits, tmp, tb, ctx->st, &launches[K_SORT_ROWS]));
        prof.end();
      }
      if (!(flags & GSMART_KEEP_ON_DEVICE)) {
        R->h_rows.resize(n_rows * nc);
        CU(cudaMemcpyAsync(R->h_rows.data(), R->d_rows, n_rows * nc * 4, cudaMemcpyDeviceToHost, ctx->st));
        R->host_valid = true;
      }
    } else {
      R->host_valid = (flags & GSMART_COUNT_ONLY) == 0;  // zero rows
      R->count_only = (flags & GSMART_COUNT_ONLY) != 0;
    }
    return GSMART_OK;
  }
};

}  // namespace

extern "C" gsmart_status gsmart_execute(gsmart_ctx* ctx, const gsmart_plan_t* plan, uint32_t flags,
                                        gsmart_result** out) {
  if (!ctx || !plan || !out) return GSMART_E_INVALID_ARG;
  *out = nullptr;
  if (ctx->poisoned) return GSMART_E_CUDA;
  if (!ctx->f[0].built || !ctx->f[1].built) FAIL(GSMART_E_STATE, "gsmart_build_lspm(CSR|CSC) must be called first");
  if (ctx->cfg.world > 1) FAIL(GSMART_E_UNSUPPORTED, "world > 1 execute is not available in this build");
  for (auto& e : plan->edges)
    if (e.pred > ctx->P) FAIL(GSMART_E_INVALID_ARG, "query predicate id > n_predicates");
  CU(cudaSetDevice(ctx->cfg.device));
  auto t0 = std::chrono::steady_clock::now();
  auto R = std::make_unique<gsmart_result>();
  R->ctx = ctx;
  R->n_cols = (uint32_t)plan->vars.size();
  R->var_of_col = plan->vars;
  R->count_only = (flags & GSMART_COUNT_ONLY) != 0;
  for (int i = 0; i < GSMART_NKERNELS; i++) R->stats.kernel_names[i] = kKernelNames[i];
  gsmart_status s;
  {
    Exec ex(ctx, plan, flags, R.get());
    s = ex.run();
    cudaError_t e = cudaStreamSynchronize(ctx->st);
    if (s == GSMART_OK && e != cudaSuccess) s = cuda_fail(ctx, e, "execute sync", __LINE__);
    ex.prof.flush();
    for (int i = 0; i < GSMART_NKERNELS; i++) R->stats.launches[i] = (uint64_t)ex.launches[i];
  }
  if (s == GSMART_OK || s == GSMART_E_RESULT_OVERFLOW) {
    unsigned long long c[C_NCTR];
    if (readback(ctx, ctx->d_ctr, C_NCTR, c) == GSMART_OK) {
      auto& st = R->stats;
      st.filter_rows = c[C_FILTER_ROWS];
      st.filter_entries = c[C_FILTER_SCANNED];
      st.seed_entries = c[C_SEED];
      st.expand_entries = c[C_EXPAND];
      st.closing_checks = c[C_CLOSING];
      st.edges_evaluated = c[C_FILTER_MATCHED] + c[C_SEED] + c[C_EXPAND];
      const uint64_t pb = (uint64_t)ctx->pred_bytes;
      // algorithmic bytes: what each step must move
      st.bytes[K_FILTER] = 8 * c[C_FILTER_ROWS] + pb * c[C_FILTER_SCANNED] + 4 * c[C_FILTER_MATCHED] +
                           8ull * st.launches[K_FILTER] / 3 * ((ctx->N + 31) / 32);
      st.bytes[K_SEED] = 4 * c[C_SEED];
      st.bytes[K_EXPAND_COUNT] = 4 * c[C_EXPAND];
      uint64_t children = 0;
      for (uint32_t k = 1; k < st.n_levels && k < GSMART_MAX_LEVELS; k++) children += st.level_nodes[k];
      st.bytes[K_EXPAND_EMIT] = 4 * c[C_EXPAND] + 8 * children;
    }
  }
  R->stats.ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (s != GSMART_OK) {
    if (s == GSMART_E_RESULT_OVERFLOW) {
      *out = R.release();  // n_rows reported
    } else {
      gsmart_result_free(R.release());
    }
    return s;
  }
  *out = R.release();
  return GSMART_OK;
}

// ------------------------------------------------------------------------ results
extern "C" gsmart_status gsmart_result_shape(const gsmart_result* r, uint64_t* n_rows, uint32_t* n_cols,
                                             const uint32_t** var_of_col) {
  if (!r) return GSMART_E_INVALID_ARG;
  if (n_rows) *n_rows = r->n_rows;
  if (n_cols) *n_cols = r->n_cols;
  if (var_of_col) *var_of_col = r->var_of_col.data();
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_result_rows(gsmart_result* r, const uint32_t** rows) {
  if (!r || !rows) return GSMART_E_INVALID_ARG;
  if (r->count_only) return GSMART_E_STATE;
  if (!r->host_valid) {
    if (!r->d_rows) return GSMART_E_STATE;
    r->h_rows.resize(r->n_rows * r->n_cols);
    if (cudaMemcpy(r->h_rows.data(), r->d_rows, r->n_rows * r->n_cols * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
      return GSMART_E_CUDA;
    r->host_valid = true;
  }
  *rows = r->h_rows.data();
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_result_rows_device(const gsmart_result* r, const uint32_t** rows_dev) {
  if (!r || !rows_dev) return GSMART_E_INVALID_ARG;
  if (r->count_only) return GSMART_E_STATE;
  *rows_dev = r->d_rows;
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_result_candidates(const gsmart_result* r, uint32_t vertex, const uint32_t** bits_dev,
                                                  uint32_t* n_words) {
  if (!r || !bits_dev || vertex >= r->cand_slot.size() || r->cand_slot[vertex] < 0 || !r->d_cand)
    return GSMART_E_INVALID_ARG;
  *bits_dev = r->d_cand + (uint64_t)r->cand_slot[vertex] * r->stride_words;
  if (n_words) *n_words = r->n_words;
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_result_level(const gsmart_result* r, uint32_t k, uint32_t* vertex, uint64_t* n,
                                             const uint32_t** parent_dev, const uint32_t** bind_dev) {
  if (!r || k >= r->levels.size()) return GSMART_E_INVALID_ARG;
  const auto& L = r->levels[k];
  if (vertex) *vertex = L.var;
  if (n) *n = L.n;
  if (parent_dev) *parent_dev = L.parent;
  if (bind_dev) *bind_dev = L.bind;
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_result_stats(const gsmart_result* r, gsmart_stats* out) {
  if (!r || !out) return GSMART_E_INVALID_ARG;
  *out = r->stats;
  return GSMART_OK;
}

extern "C" void gsmart_result_free(gsmart_result* r) {
  if (!r) return;
  if (r->ctx) {
    cudaSetDevice(r->ctx->cfg.device);
    for (void* p : r->owned) cudaFreeAsync(p, r->ctx->st);
    cudaStreamSynchronize(r->ctx->st);
  }
  delete r;
}

extern "C" gsmart_status gsmart_copy_to_host(gsmart_ctx* ctx, void* dst, const void* src_dev, size_t bytes) {
  if (!ctx || (bytes && (!dst || !src_dev))) return GSMART_E_INVALID_ARG;
  if (ctx->poisoned) return GSMART_E_CUDA;
  if (!bytes) return GSMART_OK;
  CU(cudaSetDevice(ctx->cfg.device));
  CU(cudaMemcpyAsync(dst, src_dev, bytes, cudaMemcpyDeviceToHost, ctx->st));
  CU(cudaStreamSynchronize(ctx->st));
  return GSMART_OK;
}
