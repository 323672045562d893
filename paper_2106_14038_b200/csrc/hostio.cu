// Host <-> device transfer paths of the C ABI (product code): the host side of
// gsmart_load_triples (H2D of the caller's triples) and of the result rows
// (D2H).  Pinned (page-locked) host memory is what lets a copy run at link
// rate, so:
//   - a caller's pageable triple arrays are staged through a ring of pinned
//     chunks: host threads fill chunk i+1 while the copy engine moves chunk i;
//     already pinned arrays (cudaHostAlloc / torch pin_memory) go straight;
//   - result rows land in pinned blocks from a per-context caching pool
//     (cudaMallocHost is expensive; blocks are reused across results).
#include <cstring>
#include <thread>

#include "runtime.h"

namespace gsm {

// ------------------------------------------------------------------ worker threads
HostWorkers::HostWorkers(int n) {
  for (int i = 0; i < n; i++) th.emplace_back([this, i] { loop(i); });
}

HostWorkers::~HostWorkers() {
  {
    std::lock_guard<std::mutex> lk(mu);
    stop = true;
    gen++;
  }
  cv.notify_all();
  for (auto& t : th) t.join();
}

void HostWorkers::loop(int idx) {
  uint64_t seen = 0;
  while (true) {
    std::function<void(int)> f;
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return gen != seen; });
      seen = gen;
      if (stop) return;
      f = job;
    }
    f(idx);
    {
      std::lock_guard<std::mutex> lk(mu);
      if (--pending == 0) done_cv.notify_all();
    }
  }
}

void HostWorkers::run(const std::function<void(int)>& f) {  // f(i) for i in [0, size()), blocking
  if (th.empty()) return;
  std::unique_lock<std::mutex> lk(mu);
  job = f;
  pending = (int)th.size();
  gen++;
  cv.notify_all();
  done_cv.wait(lk, [&] { return pending == 0; });
}

static void parallel_memcpy(gsmart_ctx* ctx, void* dst, const void* src, size_t bytes) {
  const int nt = ctx->workers ? (int)ctx->workers->size() : 0;
  if (bytes < (4u << 20) || nt < 2) {
    memcpy(dst, src, bytes);
    return;
  }
  const size_t per = (bytes / nt + 4095) & ~(size_t)4095;
  ctx->workers->run([&](int i) {
    const size_t a = std::min(bytes, (size_t)i * per), b = std::min(bytes, a + per);
    if (b > a) memcpy((char*)dst + a, (const char*)src + a, b - a);
  });
}

static gsmart_status ensure_workers(gsmart_ctx* ctx) {
  if (!ctx->workers) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    ctx->workers = std::make_unique<HostWorkers>((int)std::min(8u, hw));
  }
  return GSMART_OK;
}

bool host_is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// ------------------------------------------------------------------ H2D
gsmart_status h2d_staged(gsmart_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (!bytes) return GSMART_OK;
  if (host_is_pinned(src)) {
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return GSMART_OK;
  }
  TRY(ensure_workers(ctx));
  StageRing& R = ctx->ring;
  if (!R.buf[0]) {
    for (int i = 0; i < StageRing::K; i++) {
      CU(cudaMallocHost(&R.buf[i], StageRing::CHUNK));
      CU(cudaEventCreateWithFlags(&R.ev[i], cudaEventDisableTiming));
      R.used[i] = false;
    }
  }
  for (size_t off = 0, i = 0; off < bytes; off += StageRing::CHUNK, i++) {
    const int b = (int)(R.next++ % StageRing::K);
    const size_t n = std::min(StageRing::CHUNK, bytes - off);
    if (R.used[b]) CU(cudaEventSynchronize(R.ev[b]));  // the copy engine is done with this chunk
    parallel_memcpy(ctx, R.buf[b], (const char*)src + off, n);
    CU(cudaMemcpyAsync((char*)dst + off, R.buf[b], n, cudaMemcpyHostToDevice, st));
    CU(cudaEventRecord(R.ev[b], st));
    R.used[b] = true;
  }
  return GSMART_OK;
}

void stage_ring_free(gsmart_ctx* ctx) {
  StageRing& R = ctx->ring;
  for (int i = 0; i < StageRing::K; i++) {
    if (R.buf[i]) cudaFreeHost(R.buf[i]);
    if (R.ev[i]) cudaEventDestroy(R.ev[i]);
    R.buf[i] = nullptr;
    R.ev[i] = nullptr;
  }
}

// ------------------------------------------------------------------ pinned pool
static size_t size_class(size_t bytes) {
  size_t c = 1u << 16;
  while (c < bytes) c <<= 1;
  return c;
}

void* PinnedPool::get(size_t bytes, size_t* cls) {
  const size_t c = size_class(bytes);
  *cls = c;
  auto it = free_blocks.find(c);
  if (it != free_blocks.end()) {
    void* p = it->second;
    free_blocks.erase(it);
    cached -= c;
    return p;
  }
  void* p = nullptr;
  if (cudaMallocHost(&p, c) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void PinnedPool::put(void* p, size_t cls) {
  if (!p) return;
  if (cached + cls > CAP) {  // bounded cache: release instead
    cudaFreeHost(p);
    return;
  }
  free_blocks.emplace(cls, p);
  cached += cls;
}

void PinnedPool::clear() {
  for (auto& kv : free_blocks) cudaFreeHost(kv.second);
  free_blocks.clear();
  cached = 0;
}

// rows of a result into a pinned block of the ctx pool (one D2H at link rate)
gsmart_status rows_to_host(gsmart_ctx* ctx, gsmart_result* r, cudaStream_t st) {
  const size_t bytes = (size_t)r->n_rows * r->n_cols * 4;
  if (!bytes) {
    r->host_valid = true;
    return GSMART_OK;
  }
  size_t cls = 0;
  void* p = ctx->pinned.get(bytes, &cls);
  if (!p) FAIL(GSMART_E_OOM, "pinned host allocation failed");
  r->h_rows = (uint32_t*)p;
  r->h_cls = cls;
  CU(cudaMemcpyAsync(p, r->d_rows, bytes, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  r->host_valid = true;
  return GSMART_OK;
}

}  // namespace gsm
