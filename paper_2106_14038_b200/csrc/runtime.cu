// C-ABI implementation, part 1: context, device memory, triple loading, LSpM
// build orchestration (a1, §6.2), planning entry points and result
// accessors.  Host code only sequences kernels; every data-path step runs on
// the GPU.  The executor (a3-a9) is in execute.cu.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <set>

#include "runtime.h"

using namespace gsm;

#define GSM_STR2(x) #x
#define GSM_STR(x) GSM_STR2(x)

namespace gsm {

const char* kKernelNames[GSMART_NKERNELS] = {
    "build_pack", "build_sort", "build_unique", "build_rowptr", "seed", "group_filter", "bitmap",
    "compact", "scan", "expand_seg", "expand_count", "expand_emit", "prune", "enumerate", "sort_rows",
    "collective"};

thread_local std::string g_static_err;

// live contexts, so gsmart_plan_free can drop the plan's cache entries in each
static std::mutex g_live_mu;
static std::set<gsmart_ctx*> g_live;

gsmart_status cuda_fail(gsmart_ctx* ctx, cudaError_t e, const char* what, int line) {
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    ctx->err = std::string("device out of memory at ") + what;
    return GSMART_E_OOM;
  }
  ctx->poisoned = true;
  ctx->err = std::string("CUDA error '") + cudaGetErrorString(e) + "' at " + what + " (line " +
             std::to_string(line) + ")";
  return GSMART_E_CUDA;
}

gsmart_status readback(gsmart_ctx* ctx, cudaStream_t st, unsigned long long* h_pin, const unsigned long long* dev,
                       int n, unsigned long long* host) {
  CU(cudaMemcpyAsync(h_pin, dev, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  memcpy(host, h_pin, n * sizeof(unsigned long long));
  return GSMART_OK;
}

}  // namespace gsm

static gsmart_status readback(gsmart_ctx* ctx, const unsigned long long* dev, int n, unsigned long long* host) {
  return gsm::readback(ctx, ctx->st, ctx->h_pin, dev, n, host);
}

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
  if (const char* fv = getenv("GSMART_FILTER_VARIANT")) ctx->filter_variant = atoi(fv);
  if (const char* sv = getenv("GSMART_SPEC_TEST")) ctx->spec_test = atoi(sv) ? 1u : 0u;
  if (const char* tv = getenv("GSMART_NO_TMA")) ctx->use_tma = atoi(tv) == 0;
  if (const char* pv = getenv("GSMART_PUSH_MIN")) ctx->push_min = strtoull(pv, nullptr, 10);
  if (const char* lv = getenv("GSMART_L2_PERSIST")) ctx->l2_persist = atoi(lv) != 0;
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
  // The context's own stream-ordered pool, kept warm (freed blocks stay cached).
  // Own pool, and no reuse that inserts waits on another stream's frees: ranks
  // that share a device (threads of one process) must never have an allocation
  // on one rank's stream wait on a free queued behind another rank's barrier.
  {
    cudaMemPoolProps pp = {};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = cfg->device;
    if (cudaMemPoolCreate(&ctx->pool, &pp) != cudaSuccess) {
      g_static_err = "cudaMemPoolCreate failed";
      return GSMART_E_CUDA;
    }
    uint64_t thr = UINT64_MAX;
    int no = 0;
    cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &thr);
    cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolReuseAllowInternalDependencies, &no);
  }
  if (cudaMalloc(&ctx->d_ctr, 64 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMallocHost(&ctx->h_pin, 64 * sizeof(unsigned long long)) != cudaSuccess) {
    g_static_err = "context allocation failed";
    return GSMART_E_OOM;
  }
  ctx->rank = cfg->rank;
  ctx->world = cfg->world;
  ctx->exchange = cfg->exchange;
  if (cfg->world > gsm::MAX_WORLD || cfg->exchange > GSMART_XCHG_NCCL || (!cfg->alloc != !cfg->free)) {
    g_static_err = "world > 8, unknown exchange mode, or only one of alloc/free given";
    return GSMART_E_INVALID_ARG;
  }
  if (cfg->world > 1 && cfg->local_comm) {  // ranks = threads of this process
    if (cfg->local_comm->world != cfg->world) {
      g_static_err = "local_comm world differs from cfg.world";
      return GSMART_E_INVALID_ARG;
    }
    ctx->lcomm = cfg->local_comm;
  } else if (cfg->world > 1) {  // ranks = processes: socket rendezvous named by the unique id
    if (!cfg->nccl_unique_id) {
      g_static_err = "world > 1 across processes needs the 128-byte unique id (gsmart_get_nccl_id)";
      return GSMART_E_INVALID_ARG;
    }
    ctx->chan = std::make_unique<gsm::SockChan>();
    std::string err;
    if (!ctx->chan->open(cfg->nccl_unique_id, cfg->rank, cfg->world, &err)) {
      g_static_err = err;
      return GSMART_E_NCCL;
    }
  }
  // NCCL communicator: the NCCL exchange across processes, or (world == 1 with an
  // id) a one-rank communicator that runs the same collective calls
  if (!ctx->lcomm && cfg->nccl_unique_id && (cfg->world == 1 || cfg->exchange == GSMART_XCHG_NCCL)) {
    const NcclApi* api = nccl_api();
    if (!api) {
      g_static_err = "NCCL library (libnccl.so.2) not loadable";
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
  {
    std::lock_guard<std::mutex> lk(g_live_mu);
    g_live.insert(*out);
  }
  return GSMART_OK;
}

gsmart_status gsm::ctx_sync(gsmart_ctx* ctx) {
  CU(cudaStreamSynchronize(ctx->st));
  for (auto& sp : ctx->slots) CU(cudaStreamSynchronize(sp->st));
  return GSMART_OK;
}

void gsm::free_lspm(gsmart_ctx* ctx) {
  if (ctx->lm_keys) {  // a build that failed between the CSR and the label-major lists
    dfree(ctx, ctx->lm_keys);
    ctx->lm_keys = nullptr;
  }
  for (auto& f : ctx->f) {
    if (f.sym) {
      cudaStreamSynchronize(ctx->st);
      sym_free(ctx, &f.s_rp);
      sym_free(ctx, &f.s_col);
      sym_free(ctx, &f.s_pred);
      sym_free(ctx, &f.s_lmask);
    } else {
      dfree(ctx, f.rp);
      dfree(ctx, f.col);
      dfree(ctx, f.pred);
      dfree(ctx, f.lmask);
    }
    f = Lspm();
  }
  for (LabelMajor* L : {&ctx->lm, &ctx->lm_in}) {
    dfree(ctx, L->s);
    dfree(ctx, L->o);
    *L = LabelMajor();
  }
  ctx->lspm_gen++;
}

extern "C" void gsmart_destroy(gsmart_ctx* ctx) {
  if (!ctx) return;
  {
    std::lock_guard<std::mutex> lk(g_live_mu);
    g_live.erase(ctx);
  }
  cudaSetDevice(ctx->cfg.device);
  slots_free(ctx);
  free_lspm(ctx);
  dict_free(ctx);
  dfree(ctx, ctx->d_s);
  dfree(ctx, ctx->d_p);
  dfree(ctx, ctx->d_o);
  cudaStreamSynchronize(ctx->st);
  if (ctx->comm) {
    const NcclApi* api = nccl_api();
    if (api) api->CommDestroy(ctx->comm);
  }
  stage_ring_free(ctx);
  ctx->pinned.clear();
  ctx->workers.reset();
  cudaFree(ctx->d_ctr);
  cudaFreeHost(ctx->h_pin);
  cudaStreamSynchronize(ctx->st);
  if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
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
  if (n_predicates == 0 || n_predicates > 65534) FAIL(GSMART_E_INVALID_ARG, "n_predicates must be in [1, 65534]");
  if (n >= 0xffffffffull) FAIL(GSMART_E_INVALID_ARG, "n must be < 2^32 - 1");
  if (flags != GSMART_PTR_HOST && flags != GSMART_PTR_DEVICE) FAIL(GSMART_E_INVALID_ARG, "flags must be PTR_HOST or PTR_DEVICE");
  CU(cudaSetDevice(ctx->cfg.device));
  free_lspm(ctx);
  dict_free(ctx);
  dfree(ctx, ctx->d_s);
  dfree(ctx, ctx->d_p);
  dfree(ctx, ctx->d_o);
  ctx->d_s = ctx->d_p = ctx->d_o = nullptr;
  ctx->n_triples = 0;
  ctx->N = 0;
  TRY(dalloc(ctx, &ctx->d_s, n));
  TRY(dalloc(ctx, &ctx->d_p, n));
  TRY(dalloc(ctx, &ctx->d_o, n));
  if (n && flags == GSMART_PTR_HOST) {  // pinned: one copy each; pageable: staged through pinned chunks
    TRY(h2d_staged(ctx, ctx->d_s, s, n * 4, ctx->st));
    TRY(h2d_staged(ctx, ctx->d_p, p, n * 4, ctx->st));
    TRY(h2d_staged(ctx, ctx->d_o, o, n * 4, ctx->st));
  } else if (n) {
    CU(cudaMemcpyAsync(ctx->d_s, s, n * 4, cudaMemcpyDeviceToDevice, ctx->st));
    CU(cudaMemcpyAsync(ctx->d_p, p, n * 4, cudaMemcpyDeviceToDevice, ctx->st));
    CU(cudaMemcpyAsync(ctx->d_o, o, n * 4, cudaMemcpyDeviceToDevice, ctx->st));
  }
  if (n) {  // ids are validated on the device after the copy (host and device input alike)
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
  ctx->pred_bytes = n_predicates <= 254 ? 1 : 2;  // 0xff / 0xffff: sentinel label (partitioned LSpM)
  CU(cudaStreamSynchronize(ctx->st));  // caller may free / reuse its buffers after return
  return GSMART_OK;
}

// ------------------------------------------------------------------------ build (a1)
// Sorted, de-duplicated entry keys of the kept triples (§6.2.1 steps 1-4,
// P:L406-L413): mode 0 orders (a, pred, b) (an LSpM format: a = row, b = col),
// mode 1 orders (pred, a, b) (the label-major lists: a = s, b = o).  Keys that
// fit 63 bits are packed into one word (one radix sort over 2nb + pb + 1
// bits); wider keys (e.g. 100M entities x 10,000 labels: 27 + 14 + 27 bits)
// are two words, hi = the first two fields, lo = b, sorted by lo and then
// stably by hi.  flags[i] becomes the output position of sorted key i
// (exclusive scan of "kept and first of its run"); *M = kept entries.
struct SortedKeys {
  bool wide = false;
  int drop = 0;        // narrow: drop bit of the packed key; wide: drop bit of hi
  uint64_t* k = nullptr;  // narrow keys, or hi
  uint32_t* lo = nullptr;
  uint32_t* pos = nullptr;
  unsigned long long M = 0;
};

static gsmart_status sort_triple_keys(gsmart_ctx* ctx, Scratch& sc, const uint32_t* a, const uint32_t* b, int mode,
                                      const uint8_t* d_keep, SortedKeys* out, uint32_t rlo = 0,
                                      uint32_t rhi = 0xffffffffu) {
  const uint64_t n = ctx->n_triples;
  const int nb = bits_for(ctx->N - 1), pb = bits_for(ctx->P);
  unsigned long long* tot = ctx->d_ctr + 40;
  out->wide = 2 * nb + pb >= 64;
  TRY(sc.get(&out->pos, n + 1));
  if (!n) {
    CU(cudaMemsetAsync(tot, 0, 8, ctx->st));
    out->M = 0;
    return GSMART_OK;
  }
  void* rtmp = nullptr;
  const size_t rb = radix_tmp_bytes(n);
  TRY(sc.get((char**)&rtmp, rb));
  int second = 0;
  if (!out->wide) {
    uint64_t *k0 = nullptr, *k1 = nullptr;
    TRY(sc.get(&k0, n));
    TRY(sc.get(&k1, n));
    out->drop = 2 * nb + pb;
    if (mode == 0) CU(launch_pack_keys(a, ctx->d_p, b, n, d_keep, nb + pb, nb, out->drop, rlo, rhi, k0, ctx->st));
    else CU(launch_pack_pso(a, ctx->d_p, b, n, d_keep, nb, out->drop, rlo, rhi, k0, ctx->st));
    CU(radix_sort_keys_u64(k0, k1, n, 0, out->drop + 1, rtmp, rb, ctx->st, &second, nullptr, true));
    out->k = second ? k1 : k0;
    CU(launch_unique_flags(out->k, n, out->drop, out->pos, ctx->st));
  } else {
    uint64_t *h0 = nullptr, *h1 = nullptr;
    uint32_t *l0 = nullptr, *l1 = nullptr;
    TRY(sc.get(&h0, n));
    TRY(sc.get(&h1, n));
    TRY(sc.get(&l0, n));
    TRY(sc.get(&l1, n));
    out->drop = nb + pb;
    CU(launch_pack_keys2(a, ctx->d_p, b, n, d_keep, mode, mode == 0 ? pb : nb, out->drop, rlo, rhi, h0, l0, ctx->st));
    // LSD: the low word first (hi as payload), then the high word (lo as payload)
    CU(radix_sort_pairs_u32_u64(l0, l1, h0, h1, n, 0, nb, rtmp, rb, ctx->st, &second, nullptr, true));
    uint64_t *hc = second ? h1 : h0, *ho = second ? h0 : h1;
    uint32_t *lc = second ? l1 : l0, *lo_ = second ? l0 : l1;
    CU(radix_sort_pairs_u64_u32(hc, ho, lc, lo_, n, 0, out->drop + 1, rtmp, rb, ctx->st, &second, nullptr, true));
    out->k = second ? ho : hc;
    out->lo = second ? lo_ : lc;
    CU(launch_unique_flags2(out->k, out->lo, n, out->drop, out->pos, ctx->st));
  }
  void* stmp = nullptr;
  TRY(sc.get((char**)&stmp, scan_tmp_bytes(n)));
  CU(scan_exclusive_u32(out->pos, out->pos, n, tot, stmp, ctx->st, nullptr));
  TRY(readback(ctx, tot, 1, &out->M));
  return GSMART_OK;
}

// ---- world > 1: the partitioned LSpM.  Rank r stores the rows
// [v_r, v_r+1) of a format in its own chunks of four symmetric regions (row
// pointers, columns, labels, row label signatures); every rank maps every chunk,
// so the kernels read any row through one pointer (peer loads over NVLink).
// Entry space: rank r's entries start at G_r, a multiple of 2^21 entries (so the
// column/label chunks start on a mapping granule), with room for M_r + 64;
// the gap before G_r+1 is filled with sentinel entries (label 0xff.. > any
// label, column 0xffffffff >= N) that end the rank's last row: rows stay
// sorted by (label, col) and no label search ever reaches them.
constexpr uint64_t PART_ALIGN_ENTRIES = 1ull << 21;

static gsmart_status compute_partition(gsmart_ctx* ctx, const uint8_t* d_keep) {
  const int W = ctx->world;
  const uint32_t N = ctx->N;
  const uint32_t nbk = (N + PART_ALIGN_ROWS - 1) / PART_ALIGN_ROWS;
  Scratch sc(ctx);
  unsigned long long* hist = nullptr;
  TRY(sc.get(&hist, nbk));
  CU(cudaMemsetAsync(hist, 0, (size_t)nbk * 8, ctx->st));
  if (ctx->n_triples)
    CU(launch_bucket_degree(ctx->d_s, ctx->d_p, ctx->d_o, ctx->n_triples, d_keep, 19, hist, ctx->st));
  std::vector<unsigned long long> h(nbk);
  CU(cudaMemcpyAsync(h.data(), hist, (size_t)nbk * 8, cudaMemcpyDeviceToHost, ctx->st));
  CU(cudaStreamSynchronize(ctx->st));
  ctx->part.v.assign(W + 1, 0);
  if (gsmart_partition_split((const uint64_t*)h.data(), nbk, N, W, ctx->part.v.data()) != GSMART_OK)
    FAIL(GSMART_E_INVALID_ARG, "partition split failed");
  // every rank must have passed the same triples: the same split points
  std::vector<uint32_t> all((size_t)W * (W + 1));
  TRY(host_allgather(ctx, ctx->part.v.data(), (W + 1) * 4, all.data()));
  for (int q = 0; q < W; q++)
    if (memcmp(all.data() + (size_t)q * (W + 1), ctx->part.v.data(), (W + 1) * 4) != 0)
      FAIL(GSMART_E_INVALID_ARG, "world > 1: every rank must load the same triple set");
  return GSMART_OK;
}

// offset of a chunk of `bytes` for rows [lo, hi): at lo*elt when the range is
// non-empty, else parked past every real chunk (never read)
static uint64_t row_chunk_off(gsmart_ctx* ctx, uint32_t lo, uint32_t hi, uint64_t elt) {
  const uint64_t g = sym_granularity(ctx);
  if (hi > lo) return (uint64_t)lo * elt;
  const uint64_t end = ((uint64_t)ctx->N + 1) * elt;
  return (end + g - 1) / g * g + (uint64_t)ctx->rank * g;
}

// rows per label (summed over the ranks when world > 1); none when P > 8192
static gsmart_status label_rows_readback(gsmart_ctx* ctx, const unsigned long long* d, std::vector<unsigned long long>* out) {
  out->clear();
  if (ctx->P + 1 > 4096) return GSMART_OK;
  std::vector<unsigned long long> h(2 * ((size_t)ctx->P + 1));
  CU(cudaMemcpyAsync(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost, ctx->st));
  CU(cudaStreamSynchronize(ctx->st));
  if (ctx->world > 1) {
    std::vector<unsigned long long> all(h.size() * ctx->world);
    TRY(host_allgather(ctx, h.data(), h.size() * 8, all.data()));
    for (size_t i = 0; i < h.size(); i++) {
      h[i] = 0;
      for (int q = 0; q < ctx->world; q++) h[i] += all[(size_t)q * h.size() + i];
    }
  }
  *out = h;
  return GSMART_OK;
}

// functional labels of a format (no row holds two entries of the label; OR of
// the ranks' non-functional bits when world > 1)
static gsmart_status functional_readback(gsmart_ctx* ctx, const uint32_t* d, std::vector<uint8_t>* out) {
  const size_t words = ((size_t)ctx->P + 1 + 31) / 32;
  std::vector<uint32_t> h(words);
  CU(cudaMemcpyAsync(h.data(), d, words * 4, cudaMemcpyDeviceToHost, ctx->st));
  CU(cudaStreamSynchronize(ctx->st));
  if (ctx->world > 1) {
    std::vector<uint32_t> all(words * ctx->world);
    TRY(host_allgather(ctx, h.data(), words * 4, all.data()));
    for (size_t i = 0; i < words; i++)
      for (int q = 0; q < ctx->world; q++) h[i] |= all[(size_t)q * words + i];
  }
  out->assign((size_t)ctx->P + 1, 0);
  for (size_t l = 0; l <= ctx->P; l++) (*out)[l] = ((h[l >> 5] >> (l & 31)) & 1u) ? 0 : 1;
  return GSMART_OK;
}

static gsmart_status build_format_part(gsmart_ctx* ctx, int fmt, const uint8_t* d_keep) {
  Lspm& L = ctx->f[fmt];
  const uint64_t n = ctx->n_triples;
  const int W = ctx->world, me = ctx->rank, pbytes = ctx->pred_bytes;
  const uint32_t N = ctx->N;
  const int nb = bits_for(N - 1), pb = bits_for(ctx->P);
  const uint32_t rlo = ctx->part.v[me], rhi = ctx->part.v[me + 1], nloc = rhi - rlo;
  int last_rank = 0;  // the rank holding row N - 1 also stores row_ptr[N]
  for (int q = 0; q < W; q++)
    if (ctx->part.v[q] < ctx->part.v[q + 1]) last_rank = q;
  const bool last = me == last_rank;
  Scratch sc(ctx);
  const uint32_t* rowv = fmt == 0 ? ctx->d_s : ctx->d_o;
  const uint32_t* colv = fmt == 0 ? ctx->d_o : ctx->d_s;
  unsigned long long* tot = ctx->d_ctr + 40;
  SortedKeys sk;
  TRY(sort_triple_keys(ctx, sc, rowv, colv, 0, d_keep, &sk, rlo, rhi));
  std::vector<unsigned long long> Ms(W);
  TRY(host_allgather(ctx, &sk.M, 8, Ms.data()));
  std::vector<uint64_t> G(W + 1, 0);
  for (int q = 0; q < W; q++)
    G[q + 1] = G[q] + (Ms[q] + 64 + PART_ALIGN_ENTRIES - 1) / PART_ALIGN_ENTRIES * PART_ALIGN_ENTRIES;
  if (G[W] >= 0xffffffffull) FAIL(GSMART_E_UNSUPPORTED, "more than 2^32 padded entries in one LSpM format");
  const uint64_t span = G[me + 1] - G[me];
  TRY(sym_alloc(ctx, G[me] * 4, span * 4, &L.s_col));
  TRY(sym_alloc(ctx, G[me] * pbytes, span * pbytes, &L.s_pred));
  TRY(sym_alloc(ctx, row_chunk_off(ctx, rlo, rhi, 4), ((uint64_t)nloc + (last ? 1 : 0)) * 4, &L.s_rp));
  TRY(sym_alloc(ctx, row_chunk_off(ctx, rlo, rhi, 4), (uint64_t)nloc * 4, &L.s_lmask));
  uint32_t* col_l = (uint32_t*)L.s_col.local();
  void* pred_l = L.s_pred.local();
  // sentinel entries past this rank's last real one (see above)
  CU(cudaMemsetAsync(col_l + sk.M, 0xff, (span - sk.M) * 4, ctx->st));
  CU(cudaMemsetAsync((char*)pred_l + sk.M * pbytes, 0xff, (span - sk.M) * pbytes, ctx->st));
  uint32_t* cnt = nullptr;
  TRY(sc.get(&cnt, (uint64_t)nloc + 1));
  CU(cudaMemsetAsync(cnt, 0, ((uint64_t)nloc + 1) * 4, ctx->st));
  uint32_t* cnt_rows = cnt - rlo;  // indexed by global row
  if (n && !sk.wide)
    CU(launch_unpack(sk.k, n, sk.pos, sk.drop, nb + pb, nb, col_l, pred_l, pbytes, cnt_rows, ctx->st));
  else if (n)
    CU(launch_unpack2(sk.k, sk.lo, n, sk.pos, sk.drop, pb, 0, col_l, pred_l, pbytes, nullptr, cnt_rows, ctx->st));
  {
    void* stmp = nullptr;
    TRY(sc.get((char**)&stmp, scan_tmp_bytes((uint64_t)nloc + 1)));
    CU(scan_exclusive_u32(cnt, cnt, (uint64_t)nloc + 1, tot, stmp, ctx->st, nullptr));
  }
  if (nloc || last)
    CU(launch_add_copy((uint32_t*)L.s_rp.local(), cnt, (uint64_t)nloc + (last ? 1 : 0), (uint32_t)G[me], ctx->st));
  CU(cudaStreamSynchronize(ctx->st));
  TRY(host_barrier(ctx));  // every rank's row pointers are in place (the last row reads the next chunk)
  L.rp = (uint32_t*)L.s_rp.va;
  L.col = (uint32_t*)L.s_col.va;
  L.pred = (void*)L.s_pred.va;
  L.lmask = (uint32_t*)L.s_lmask.va;
  unsigned long long* lrows = nullptr;
  TRY(sc.get(&lrows, 2 * ((uint64_t)ctx->P + 1)));
  CU(cudaMemsetAsync(lrows, 0, ((size_t)ctx->P + 1) * 16, ctx->st));
  uint32_t* nonfunc = nullptr;
  TRY(sc.get(&nonfunc, ((uint64_t)ctx->P + 1 + 31) / 32));
  CU(cudaMemsetAsync(nonfunc, 0, ((size_t)ctx->P + 1 + 31) / 32 * 4, ctx->st));
  if (nloc)
    CU(launch_label_mask(L.rp + rlo, L.pred, pbytes, nloc, L.lmask + rlo, lrows, ctx->P + 1, ctx->st, nonfunc));
  TRY(label_rows_readback(ctx, lrows, &L.label_rows));
  TRY(functional_readback(ctx, nonfunc, &L.functional));
  CU(cudaMemsetAsync(ctx->d_ctr + 42, 0, 16, ctx->st));
  if (nloc) CU(launch_heavy_stats(L.rp + rlo, nloc, ctx->d_ctr + 42, ctx->st));
  unsigned long long hv[2];
  TRY(readback(ctx, ctx->d_ctr + 42, 2, hv));
  L.heavy_rows = hv[0];
  L.heavy_chunks = hv[1];
  L.nnz = 0;
  for (int q = 0; q < W; q++) L.nnz += Ms[q];
  L.sym = true;
  L.built = true;
  TRY(host_barrier(ctx));
  return GSMART_OK;
}

static gsmart_status finish_format(gsmart_ctx* ctx, int fmt, unsigned long long M);

static gsmart_status build_format(gsmart_ctx* ctx, int fmt, const uint8_t* d_keep, bool lm_from_csr = false) {
  if (ctx->world > 1) return build_format_part(ctx, fmt, d_keep);
  Lspm& L = ctx->f[fmt];
  const uint64_t n = ctx->n_triples;
  const uint32_t N = ctx->N;
  const int nb = bits_for(N - 1), pb = bits_for(ctx->P);
  Scratch sc(ctx);
  const uint32_t* rowv = fmt == 0 ? ctx->d_s : ctx->d_o;
  const uint32_t* colv = fmt == 0 ? ctx->d_o : ctx->d_s;
  unsigned long long* tot = ctx->d_ctr + 40;
  SortedKeys sk;
  TRY(sort_triple_keys(ctx, sc, rowv, colv, 0, d_keep, &sk));
  const unsigned long long M = sk.M;
  if (M >= 0xffffffffull) FAIL(GSMART_E_UNSUPPORTED, "more than 2^32-2 entries in one LSpM format");
  TRY(dalloc(ctx, &L.rp, (uint64_t)N + 1));
  TRY(dalloc(ctx, &L.col, M));
  TRY(dalloc(ctx, (uint8_t**)&L.pred, M * ctx->pred_bytes + 64));  // +64: 16-byte label loads may overrun
  CU(cudaMemsetAsync(L.rp, 0, ((uint64_t)N + 1) * 4, ctx->st));
  if (n && !sk.wide)
    CU(launch_unpack(sk.k, n, sk.pos, sk.drop, nb + pb, nb, L.col, L.pred, ctx->pred_bytes, L.rp, ctx->st));
  else if (n)
    CU(launch_unpack2(sk.k, sk.lo, n, sk.pos, sk.drop, pb, 0, L.col, L.pred, ctx->pred_bytes, nullptr, L.rp, ctx->st));
  if (fmt == 0 && lm_from_csr && n && !sk.wide && M) {  // hand the unique (s, p, o) keys to the label-major build
    TRY(dalloc(ctx, &ctx->lm_keys, M));
    CU(launch_compact_keys(sk.k, n, sk.pos, sk.drop, nb, pb, ctx->lm_keys, ctx->st));
    ctx->lm_keys_n = M;
  }
  return finish_format(ctx, fmt, M);
}

// row counts in L.rp -> row pointers; row label signatures, label statistics,
// functional labels, heavy-row statistics
static gsmart_status finish_format(gsmart_ctx* ctx, int fmt, unsigned long long M) {
  Lspm& L = ctx->f[fmt];
  const uint32_t N = ctx->N;
  Scratch sc(ctx);
  unsigned long long* tot = ctx->d_ctr + 40;
  {
    void* stmp = nullptr;
    TRY(sc.get((char**)&stmp, scan_tmp_bytes((uint64_t)N + 1)));
    CU(scan_exclusive_u32(L.rp, L.rp, (uint64_t)N + 1, tot, stmp, ctx->st, nullptr));
  }
  TRY(dalloc(ctx, &L.lmask, (uint64_t)N + 1));
  unsigned long long* lrows = nullptr;
  TRY(sc.get(&lrows, 2 * ((uint64_t)ctx->P + 1)));
  CU(cudaMemsetAsync(lrows, 0, ((size_t)ctx->P + 1) * 16, ctx->st));
  uint32_t* nonfunc = nullptr;
  TRY(sc.get(&nonfunc, ((uint64_t)ctx->P + 1 + 31) / 32));
  CU(cudaMemsetAsync(nonfunc, 0, ((size_t)ctx->P + 1 + 31) / 32 * 4, ctx->st));
  CU(launch_label_mask(L.rp, L.pred, ctx->pred_bytes, N, L.lmask, lrows, ctx->P + 1, ctx->st, nonfunc));
  TRY(label_rows_readback(ctx, lrows, &L.label_rows));
  TRY(functional_readback(ctx, nonfunc, &L.functional));
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

// label-major lists: the kept, de-duplicated triples sorted by (p, s, o).
// world > 1 (in_side = false): only this rank's subjects; in_side = true: this
// rank's objects, sorted by (p, o, s) and stored as (o, s) — the center of an
// IN edge comes first, like the subject of an OUT edge.
static gsmart_status build_label_major(gsmart_ctx* ctx, const uint8_t* d_keep, bool in_side = false,
                                       bool keep_keys = false) {
  LabelMajor& L = in_side ? ctx->lm_in : ctx->lm;
  const uint64_t n = ctx->n_triples;
  const int nb = bits_for(ctx->N - 1);
  Scratch sc(ctx);
  uint32_t* cnt = nullptr;
  TRY(sc.get(&cnt, (uint64_t)ctx->P + 2));
  CU(cudaMemsetAsync(cnt, 0, ((size_t)ctx->P + 2) * 4, ctx->st));
  if (!in_side && ctx->lm_keys) {
    // the CSR's keys are in (s, p, o) order, re-laid out as (p, s, o) keys: a stable
    // LSD pass on the label bits alone sorts them — one radix pass instead of a full sort
    const int pb = bits_for(ctx->P);
    const unsigned long long M = ctx->lm_keys_n;
    uint64_t* k1 = nullptr;
    void* rtmp = nullptr;
    TRY(dalloc(ctx, &k1, M));
    const size_t rb = radix_tmp_bytes(M);
    TRY(sc.get((char**)&rtmp, rb));
    int second = 0;
    CU(radix_sort_keys_u64(ctx->lm_keys, k1, M, 2 * nb, 2 * nb + pb, rtmp, rb, ctx->st, &second, nullptr, true));
    TRY(dalloc(ctx, &L.s, M + 4));  // +4: k_push_edge's 16-byte loads may overrun the last label
    TRY(dalloc(ctx, &L.o, M + 4));
    uint64_t* sorted = second ? k1 : ctx->lm_keys;
    uint64_t* other = second ? ctx->lm_keys : k1;
    // keep_keys: the entries re-laid out as (o, p, s) keys go into the other buffer —
    // in (p, s, o) order, the CSC is one stable sort on the object away
    CU(launch_unpack_spo_lm(sorted, M, nb, pb, L.s, L.o, cnt, ctx->st, keep_keys ? other : nullptr));
    std::vector<uint32_t> h(ctx->P + 2);
    CU(cudaMemcpyAsync(h.data(), cnt, h.size() * 4, cudaMemcpyDeviceToHost, ctx->st));
    CU(cudaStreamSynchronize(ctx->st));
    dfree(ctx, sorted);
    if (keep_keys) ctx->lm_keys = other;
    else {
      dfree(ctx, other);
      ctx->lm_keys = nullptr;
    }
    L.off.assign(ctx->P + 2, 0);
    for (uint32_t l = 0; l + 1 < ctx->P + 2; l++) L.off[l + 1] = L.off[l] + h[l];
    L.M = M;
    L.built = true;
    return GSMART_OK;
  }
  SortedKeys sk;
  const uint32_t rlo = ctx->world > 1 ? ctx->part.v[ctx->rank] : 0u;
  const uint32_t rhi = ctx->world > 1 ? ctx->part.v[ctx->rank + 1] : 0xffffffffu;
  TRY(sort_triple_keys(ctx, sc, in_side ? ctx->d_o : ctx->d_s, in_side ? ctx->d_s : ctx->d_o, 1, d_keep, &sk, rlo,
                       rhi));
  const unsigned long long M = sk.M;
  TRY(dalloc(ctx, &L.s, M + 4));  // +4: k_push_edge's 16-byte loads may overrun the last label
  TRY(dalloc(ctx, &L.o, M + 4));
  if (M && !sk.wide) CU(launch_unpack_pso(sk.k, n, sk.pos, sk.drop, nb, L.s, L.o, cnt, ctx->st));
  else if (M) CU(launch_unpack2(sk.k, sk.lo, n, sk.pos, sk.drop, nb, 1, L.s, nullptr, ctx->pred_bytes, L.o, cnt, ctx->st));
  std::vector<uint32_t> h(ctx->P + 2);
  CU(cudaMemcpyAsync(h.data(), cnt, h.size() * 4, cudaMemcpyDeviceToHost, ctx->st));
  CU(cudaStreamSynchronize(ctx->st));
  L.off.assign(ctx->P + 2, 0);
  for (uint32_t l = 0; l + 1 < ctx->P + 2; l++) L.off[l + 1] = L.off[l] + h[l];
  L.M = M;
  L.built = true;
  return GSMART_OK;
}

// CSC from the label-major entries ((o, p, s)-layout keys in (p, s, o) order): a
// stable LSD sort on the object field alone (zeros above it) gives (o, p, s)
// order — the CSC's entry order — in nb/8 passes instead of a full sort
static gsmart_status build_csc_from_lm(gsmart_ctx* ctx) {
  Lspm& L = ctx->f[1];
  const uint32_t N = ctx->N;
  const int nb = bits_for(N - 1), pb = bits_for(ctx->P);
  const unsigned long long M = ctx->lm_keys_n;
  Scratch sc(ctx);
  uint64_t* k1 = nullptr;
  void* rtmp = nullptr;
  TRY(sc.get(&k1, M));
  const size_t rb = radix_tmp_bytes(M);
  TRY(sc.get((char**)&rtmp, rb));
  int second = 0;
  CU(radix_sort_keys_u64(ctx->lm_keys, k1, M, nb + pb, 2 * nb + pb, rtmp, rb, ctx->st, &second, nullptr, true));
  TRY(dalloc(ctx, &L.rp, (uint64_t)N + 1));
  TRY(dalloc(ctx, &L.col, M));
  TRY(dalloc(ctx, (uint8_t**)&L.pred, M * ctx->pred_bytes + 64));
  CU(cudaMemsetAsync(L.rp, 0, ((uint64_t)N + 1) * 4, ctx->st));
  CU(launch_unpack_lm_csc(second ? k1 : ctx->lm_keys, M, nb, pb, L.col, L.pred, ctx->pred_bytes, L.rp, ctx->st));
  CU(cudaStreamSynchronize(ctx->st));
  dfree(ctx, ctx->lm_keys);
  ctx->lm_keys = nullptr;
  return finish_format(ctx, 1, M);
}

static gsmart_status keep_mask(gsmart_ctx* ctx, const uint32_t* ids, uint32_t n, bool all, std::vector<uint8_t>* out) {
  out->assign(ctx->P + 1, all ? 1 : 0);
  (*out)[0] = 0;
  for (uint32_t i = 0; i < n; i++) {
    if (ids[i] == 0 || ids[i] > ctx->P) FAIL(GSMART_E_INVALID_ARG, "keep id out of range");
    (*out)[ids[i]] = 1;
  }
  return GSMART_OK;
}

static gsmart_status build_lspm_masks(gsmart_ctx* ctx, const std::vector<uint8_t>& kcsr,
                                      const std::vector<uint8_t>& kcsc, uint32_t formats);

extern "C" gsmart_status gsmart_build_lspm_split(gsmart_ctx* ctx, const uint32_t* keep_csr, uint32_t n_csr,
                                                 const uint32_t* keep_csc, uint32_t n_csc) {
  if (!ctx) return GSMART_E_INVALID_ARG;
  if (ctx->poisoned) return GSMART_E_CUDA;
  if (ctx->N == 0) FAIL(GSMART_E_STATE, "gsmart_load_triples must be called first");
  if ((n_csr && !keep_csr) || (n_csc && !keep_csc)) FAIL(GSMART_E_INVALID_ARG, "null keep set");
  std::vector<uint8_t> kcsr, kcsc;
  TRY(keep_mask(ctx, keep_csr, n_csr, false, &kcsr));
  TRY(keep_mask(ctx, keep_csc, n_csc, false, &kcsc));
  return build_lspm_masks(ctx, kcsr, kcsc, GSMART_CSR | GSMART_CSC);
}

extern "C" gsmart_status gsmart_build_lspm(gsmart_ctx* ctx, const uint32_t* keep_preds, uint32_t n_keep,
                                           uint32_t formats) {
  if (!ctx) return GSMART_E_INVALID_ARG;
  if (ctx->poisoned) return GSMART_E_CUDA;
  if (ctx->N == 0) FAIL(GSMART_E_STATE, "gsmart_load_triples must be called first");
  if (formats == 0 || (formats & ~(GSMART_CSR | GSMART_CSC))) FAIL(GSMART_E_INVALID_ARG, "formats must be CSR|CSC");
  if (n_keep && !keep_preds) FAIL(GSMART_E_INVALID_ARG, "null keep_preds");
  std::vector<uint8_t> keep;
  TRY(keep_mask(ctx, keep_preds, n_keep, n_keep == 0, &keep));
  return build_lspm_masks(ctx, keep, keep, formats);
}

static gsmart_status build_lspm_masks(gsmart_ctx* ctx, const std::vector<uint8_t>& kcsr,
                                      const std::vector<uint8_t>& kcsc, uint32_t formats) {
  CU(cudaSetDevice(ctx->cfg.device));
  std::vector<uint8_t> keep(kcsr.size());
  for (size_t i = 0; i < keep.size(); i++) keep[i] = kcsr[i] | kcsc[i];  // label-major lists, partition
  free_lspm(ctx);
  ctx->keep[0] = kcsr;
  ctx->keep[1] = kcsc;
  // Warm the context's pool to the build's peak once: the pool keeps freed memory
  // (release threshold = max), so the build's many large temporaries are carved
  // from memory it already holds instead of mapping new physical memory per call
  // (which made repeated builds vary 2-10x)
  if (!ctx->cfg.alloc) {
    const uint64_t want = ctx->n_triples * 48ull + (uint64_t)ctx->N * 24ull + (64ull << 20);
    uint64_t have = 0;
    cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrReservedMemCurrent, &have);
    if (have < want) {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      if (want - have + (4ull << 30) < fr) {
        void* w = nullptr;
        if (cudaMallocFromPoolAsync(&w, want - have, ctx->pool, ctx->st) == cudaSuccess) cudaFreeAsync(w, ctx->st);
        cudaGetLastError();
      }
    }
  }
  Scratch sc(ctx);
  uint8_t *d_keep = nullptr, *d_kf[2] = {nullptr, nullptr};
  TRY(sc.get(&d_keep, keep.size()));
  CU(cudaMemcpyAsync(d_keep, keep.data(), keep.size(), cudaMemcpyHostToDevice, ctx->st));
  for (int f = 0; f < 2; f++) {
    TRY(sc.get(&d_kf[f], keep.size()));
    CU(cudaMemcpyAsync(d_kf[f], (f ? kcsc : kcsr).data(), keep.size(), cudaMemcpyHostToDevice, ctx->st));
  }
  static const bool trace = getenv("GSMART_TRACE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(ctx->st);
    const auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "[gsmart] build %-12s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  if (ctx->world > 1) TRY(compute_partition(ctx, d_keep));
  lap("partition");
  // world == 1 and the CSR holds every kept label: the label-major lists come from
  // the CSR's sorted keys (one pass on the label bits) instead of a sort of their own
  const bool lm_csr = ctx->world == 1 && formats == (GSMART_CSR | GSMART_CSC) && keep == kcsr &&
                      !getenv("GSMART_LM_SORT");
  if (lm_csr && kcsc == keep) {  // CSR -> label-major lists -> CSC, each from the previous one's keys
    TRY(build_format(ctx, 0, d_kf[0], true));
    lap("csr");
    const bool derive = ctx->lm_keys != nullptr;
    TRY(build_label_major(ctx, d_keep, false, derive));
    lap("label-major");
    if (derive) TRY(build_csc_from_lm(ctx));
    else TRY(build_format(ctx, 1, d_kf[1]));
    lap("csc");
  } else {
    for (int fmt = 0; fmt < 2; fmt++) {
      if (formats & (fmt == 0 ? GSMART_CSR : GSMART_CSC)) TRY(build_format(ctx, fmt, d_kf[fmt], lm_csr));
      lap(fmt == 0 ? "csr" : "csc");
    }
    if (formats == (GSMART_CSR | GSMART_CSC)) {
      TRY(build_label_major(ctx, d_keep));
      if (ctx->world > 1) TRY(build_label_major(ctx, d_keep, true));
      lap("label-major");
    }
  }
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
  out->label_mask = L.lmask;
  return GSMART_OK;
}

// ------------------------------------------------------------------------ plan
extern "C" gsmart_status gsmart_plan(gsmart_ctx* ctx, const gsmart_query* q, uint32_t traversal,
                                     gsmart_plan_t** out) {
  if (!out) return GSMART_E_INVALID_ARG;
  *out = nullptr;
  static std::atomic<uint64_t> next_uid{1};
  auto p = std::make_unique<gsmart_plan_t>();
  p->uid = next_uid++;
  std::string err;
  // trie order by expected fan-out when the ctx has a built LSpM with label statistics
  std::function<double(uint32_t, uint32_t)> fan;
  const bool stats = ctx && ctx->f[0].built && ctx->f[1].built &&
                     ctx->f[0].label_rows.size() == 2 * ((size_t)ctx->P + 1) &&
                     ctx->f[1].label_rows.size() == 2 * ((size_t)ctx->P + 1);
  if (stats)
    fan = [ctx](uint32_t label, uint32_t dir) {
      const auto& lr = ctx->f[dir == OUT ? 0 : 1].label_rows;
      if (label > ctx->P) return 0.0;
      const double rows = (double)lr[label], ent = (double)lr[ctx->P + 1 + label];
      return rows > 0 ? ent / rows : 0.0;
    };
  const bool csr_only = ctx && ctx->f[0].built && !ctx->f[1].built;
  gsmart_status s = build_plan(q, traversal, p.get(), &err, stats ? &fan : nullptr, csr_only);
  if (s != GSMART_OK) {
    if (ctx) ctx->err = err; else g_static_err = err;
    return s;
  }
  *out = p.release();
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_plan_keep_sets(const gsmart_plan_t* const* plans, uint32_t n, uint32_t flags,
                                               uint32_t* csr_out, uint32_t* n_csr, uint32_t* csc_out, uint32_t* n_csc,
                                               uint32_t cap) {
  if ((n && !plans) || !n_csr || !n_csc || (cap && (!csr_out || !csc_out))) return GSMART_E_INVALID_ARG;
  std::set<uint32_t> a, b;
  for (uint32_t i = 0; i < n; i++) {
    if (!plans[i]) return GSMART_E_INVALID_ARG;
    plan_access(*plans[i], (flags & GSMART_BACK_EDGES) != 0, &a, &b);
  }
  *n_csr = (uint32_t)a.size();
  *n_csc = (uint32_t)b.size();
  uint32_t i = 0;
  for (uint32_t l : a) if (i < cap) csr_out[i++] = l;
  i = 0;
  for (uint32_t l : b) if (i < cap) csc_out[i++] = l;
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

extern "C" void gsmart_plan_free(gsmart_plan_t* plan) {
  if (!plan) return;
  const uint64_t uid = plan->uid;
  {
    std::lock_guard<std::mutex> lk(g_live_mu);
    int dev0 = -1;
    for (gsmart_ctx* ctx : g_live) {
      ctx->push_cache.erase(uid * 2);
      ctx->push_cache.erase(uid * 2 + 1);
      ctx->p2_guess.erase(uid);
      ctx->plan_cost.erase(uid);
      bool any = false;
      for (auto& sp : ctx->slots) {
        for (auto& kv : sp->graphs) any = any || (kv.first >> 3) == uid;
        for (auto it = sp->seen.begin(); it != sp->seen.end();) {
          if ((*it >> 3) == uid) it = sp->seen.erase(it);
          else ++it;
        }
      }
      if (!any) continue;
      if (dev0 < 0) cudaGetDevice(&dev0);
      cudaSetDevice(ctx->cfg.device);
      for (auto& sp : ctx->slots)
        for (auto it = sp->graphs.begin(); it != sp->graphs.end();) {
          if ((it->first >> 3) == uid) {
            cudaGraphExecDestroy(it->second.exec);
            it = sp->graphs.erase(it);
          } else {
            ++it;
          }
        }
    }
    if (dev0 >= 0) cudaSetDevice(dev0);
  }
  delete plan;
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
    gsmart_ctx* ctx = r->ctx;
    CU(cudaSetDevice(ctx->cfg.device));
    TRY(rows_to_host(ctx, r, r->st ? r->st : ctx->st));
  }
  *rows = r->h_rows;
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

extern "C" gsmart_status gsmart_result_tree(const gsmart_result* r, uint32_t k, uint32_t* vertex, int32_t* parent_level,
                                            uint64_t* n, const uint32_t** parent_dev, const uint32_t** bind_dev,
                                            const uint8_t** alive_dev) {
  if (!r || k >= r->levels.size()) return GSMART_E_INVALID_ARG;
  const auto& L = r->levels[k];
  if (vertex) *vertex = L.var;
  if (parent_level) *parent_level = L.parent_level == -2 ? (int32_t)k - 1 : L.parent_level;
  if (n) *n = L.n;
  if (parent_dev) *parent_dev = L.parent;
  if (bind_dev) *bind_dev = L.bind;
  if (alive_dev) *alive_dev = L.alive;
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
    cudaStream_t st = r->st ? r->st : r->ctx->st;
    for (void* p : r->owned) dfree(r->ctx, st, p);
    if (r->h_rows) r->ctx->pinned.put(r->h_rows, r->h_cls);
  }
  delete r;
}

extern "C" gsmart_status gsmart_copy_to_host(gsmart_ctx* ctx, void* dst, const void* src_dev, size_t bytes) {
  if (!ctx || (bytes && (!dst || !src_dev))) return GSMART_E_INVALID_ARG;
  if (ctx->poisoned) return GSMART_E_CUDA;
  if (!bytes) return GSMART_OK;
  CU(cudaSetDevice(ctx->cfg.device));
  TRY(ctx_sync(ctx));  // results may be ordered on any slot stream (never a device-wide sync: ranks may share it)
  CU(cudaMemcpyAsync(dst, src_dev, bytes, cudaMemcpyDeviceToHost, ctx->st));
  CU(cudaStreamSynchronize(ctx->st));
  return GSMART_OK;
}
