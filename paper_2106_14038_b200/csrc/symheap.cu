// Symmetric device memory across the ranks of one NVLink domain (SURVEY
// §8(e)): every rank backs its own chunk of a region with
// physical memory (cuMemCreate) and maps EVERY rank's chunk into one virtual
// address range at the same offsets (cuMemMap), so a kernel dereferences a
// peer's data with an ordinary load or atomic over NVLink / NVSwitch — no
// copy, no NCCL call.  The partitioned LSpM (each rank stores only its vertex
// range of CSR/CSC rows) is laid out this way, so the unchanged kernels read
// any row through one pointer; the candidate bitmaps are replicated
// symmetric buffers that the filter updates on every rank with peer atomics.
//
// Handle exchange: ranks that are threads of one process share handles
// directly (gsmart_comm); ranks that are processes exchange POSIX file
// descriptors (SCM_RIGHTS) over an abstract Unix socket named from the
// 128-byte unique id, which also carries the small host all-gathers.
#include <cstdio>
#include <cstring>

#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <chrono>
#include <thread>

#include <cuda.h>

#include "runtime.h"

namespace gsm {

// ------------------------------------------------------------------ driver API (VMM) via the runtime
struct VmmApi {
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
  CUresult (*MemRelease)(CUmemGenericAllocationHandle);
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*MemAddressFree)(CUdeviceptr, size_t);
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*MemUnmap)(CUdeviceptr, size_t);
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
  CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long);
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
};

static const VmmApi* vmm() {
  static VmmApi api;
  static int state = 0;  // 0 unknown, 1 ok, -1 missing
  if (state) return state > 0 ? &api : nullptr;
  auto get = [](const char* name, void** fn) {
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess;
  };
  bool ok = get("cuMemCreate", (void**)&api.MemCreate) && get("cuMemRelease", (void**)&api.MemRelease) &&
            get("cuMemAddressReserve", (void**)&api.MemAddressReserve) &&
            get("cuMemAddressFree", (void**)&api.MemAddressFree) && get("cuMemMap", (void**)&api.MemMap) &&
            get("cuMemUnmap", (void**)&api.MemUnmap) && get("cuMemSetAccess", (void**)&api.MemSetAccess) &&
            get("cuMemGetAllocationGranularity", (void**)&api.MemGetAllocationGranularity) &&
            get("cuMemExportToShareableHandle", (void**)&api.MemExportToShareableHandle) &&
            get("cuMemImportFromShareableHandle", (void**)&api.MemImportFromShareableHandle);
  state = ok ? 1 : -1;
  return ok ? &api : nullptr;
}

// ------------------------------------------------------------------ host channel, multi-process
static bool send_all(int fd, const void* p, size_t n) {
  const char* c = (const char*)p;
  while (n) {
    ssize_t k = ::send(fd, c, n, MSG_NOSIGNAL);
    if (k <= 0) return false;
    c += k;
    n -= (size_t)k;
  }
  return true;
}

static bool recv_all(int fd, void* p, size_t n) {
  char* c = (char*)p;
  while (n) {
    ssize_t k = ::recv(fd, c, n, 0);
    if (k <= 0) return false;
    c += k;
    n -= (size_t)k;
  }
  return true;
}

static bool send_fds(int sock, const int* fds, int n) {
  char dummy = 'F';
  iovec iov{&dummy, 1};
  std::vector<char> ctl(CMSG_SPACE(sizeof(int) * n));
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctl.data();
  m.msg_controllen = ctl.size();
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(sizeof(int) * n);
  memcpy(CMSG_DATA(c), fds, sizeof(int) * n);
  return ::sendmsg(sock, &m, MSG_NOSIGNAL) == 1;
}

static bool recv_fds(int sock, int* fds, int n) {
  char dummy;
  iovec iov{&dummy, 1};
  std::vector<char> ctl(CMSG_SPACE(sizeof(int) * n));
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctl.data();
  m.msg_controllen = ctl.size();
  if (::recvmsg(sock, &m, 0) != 1) return false;
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  if (!c || c->cmsg_type != SCM_RIGHTS || c->cmsg_len != CMSG_LEN(sizeof(int) * n)) return false;
  memcpy(fds, CMSG_DATA(c), sizeof(int) * n);
  return true;
}

SockChan::~SockChan() {
  for (int fd : peers)
    if (fd >= 0) ::close(fd);
  if (listen_fd >= 0) ::close(listen_fd);
}

bool SockChan::open(const void* id128, int rank_, int world_, std::string* err) {
  rank = rank_;
  world = world_;
  uint64_t h = 1469598103934665603ull;  // FNV-1a of the unique id -> socket name
  for (int i = 0; i < 128; i++) h = (h ^ ((const unsigned char*)id128)[i]) * 1099511628211ull;
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  char name[64];
  snprintf(name, sizeof name, "gsmart-%016llx", (unsigned long long)h);
  memcpy(a.sun_path + 1, name, strlen(name));  // abstract namespace (leading NUL)
  const socklen_t alen = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + strlen(name));
  peers.assign(world, -1);
  if (rank == 0) {
    listen_fd = ::socket(AF_UNIX, SOCK_STREAM, 0);
    if (listen_fd < 0 || ::bind(listen_fd, (sockaddr*)&a, alen) != 0 || ::listen(listen_fd, world) != 0) {
      *err = "rank 0 could not listen on the rendezvous socket";
      return false;
    }
    for (int i = 1; i < world; i++) {
      int fd = ::accept(listen_fd, nullptr, nullptr);
      int32_t r = -1;
      if (fd < 0 || !recv_all(fd, &r, 4) || r <= 0 || r >= world || peers[r] >= 0) {
        *err = "rendezvous accept failed";
        return false;
      }
      peers[r] = fd;
    }
  } else {
    const auto t0 = std::chrono::steady_clock::now();
    while (true) {
      int fd = ::socket(AF_UNIX, SOCK_STREAM, 0);
      if (fd >= 0 && ::connect(fd, (sockaddr*)&a, alen) == 0) {
        int32_t r = rank;
        if (!send_all(fd, &r, 4)) {
          *err = "rendezvous send failed";
          return false;
        }
        peers[0] = fd;
        break;
      }
      if (fd >= 0) ::close(fd);
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
        *err = "rendezvous connect timed out";
        return false;
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(20));
    }
  }
  return true;
}

// all-gather of n bytes per rank (star through rank 0)
bool SockChan::allgather(const void* mine, size_t n, void* all) {
  char* out = (char*)all;
  memcpy(out + (size_t)rank * n, mine, n);
  if (rank == 0) {
    for (int q = 1; q < world; q++)
      if (!recv_all(peers[q], out + (size_t)q * n, n)) return false;
    for (int q = 1; q < world; q++)
      if (!send_all(peers[q], out, n * world)) return false;
    return true;
  }
  return send_all(peers[0], mine, n) && recv_all(peers[0], out, n * world);
}

// every rank's file descriptor, duplicated into this process (own slot: my_fd itself)
bool SockChan::allgather_fds(int my_fd, std::vector<int>* fds) {
  fds->assign(world, -1);
  (*fds)[rank] = my_fd;
  if (rank == 0) {
    for (int q = 1; q < world; q++)
      if (!recv_fds(peers[q], &(*fds)[q], 1)) return false;
    for (int q = 1; q < world; q++)
      for (int r = 0; r < world; r++)
        if (r != q && !send_fds(peers[q], &(*fds)[r], 1)) return false;
    return true;
  }
  if (!send_fds(peers[0], &my_fd, 1)) return false;
  for (int r = 0; r < world; r++)
    if (r != rank && !recv_fds(peers[0], &(*fds)[r], 1)) return false;
  return true;
}

// ------------------------------------------------------------------ host all-gather on either channel
gsmart_status host_allgather(gsmart_ctx* ctx, const void* mine, size_t n, void* all) {
  if (ctx->world == 1) {
    memcpy(all, mine, n);
    return GSMART_OK;
  }
  if (ctx->lcomm) {
    gsmart_comm* c = ctx->lcomm;
    c->blob[ctx->rank].assign((const char*)mine, (const char*)mine + n);
    c->barrier();
    for (int q = 0; q < ctx->world; q++) memcpy((char*)all + (size_t)q * n, c->blob[q].data(), n);
    c->barrier();
    return GSMART_OK;
  }
  if (!ctx->chan || !ctx->chan->allgather(mine, n, all)) FAIL(GSMART_E_NCCL, "host all-gather over the rendezvous socket failed");
  return GSMART_OK;
}

gsmart_status host_barrier(gsmart_ctx* ctx) {
  char x = 0;
  std::vector<char> all(ctx->world);
  return host_allgather(ctx, &x, 1, all.data());
}

// ------------------------------------------------------------------ symmetric regions
size_t sym_granularity(gsmart_ctx* ctx) {
  const VmmApi* api = vmm();
  if (!api) return 2u << 20;
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = ctx->cfg.device;
  size_t g = 0;
  if (api->MemGetAllocationGranularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS || !g)
    g = 2u << 20;
  return g;
}

#define DRV(x, what)                                                                 \
  do {                                                                               \
    CUresult r_ = (x);                                                               \
    if (r_ != CUDA_SUCCESS) {                                                        \
      ctx->err = std::string("CUDA driver error ") + std::to_string((int)r_) + " in " + what; \
      return r_ == CUDA_ERROR_OUT_OF_MEMORY ? GSMART_E_OOM : GSMART_E_CUDA;          \
    }                                                                                \
  } while (0)

// Collective: rank r backs [my_off, my_off + my_bytes) of the region (offsets and
// sizes multiples of the granularity, chunks disjoint); every rank maps every chunk.
gsmart_status sym_alloc(gsmart_ctx* ctx, uint64_t my_off, uint64_t my_bytes, SymRegion* out) {
  const VmmApi* api = vmm();
  if (!api) FAIL(GSMART_E_UNSUPPORTED, "CUDA virtual memory management API unavailable");
  const int W = ctx->world, me = ctx->rank;
  const size_t g = sym_granularity(ctx);
  my_bytes = std::max<uint64_t>(g, (my_bytes + g - 1) / g * g);
  if (my_off % g) FAIL(GSMART_E_INVALID_ARG, "symmetric chunk offset not granular");
  uint64_t mine[2] = {my_off, my_bytes};
  std::vector<uint64_t> all(2 * W);
  TRY(host_allgather(ctx, mine, 16, all.data()));
  SymRegion R;
  R.off.resize(W);
  R.bytes.resize(W);
  uint64_t total = 0;
  for (int q = 0; q < W; q++) {
    R.off[q] = all[2 * q];
    R.bytes[q] = all[2 * q + 1];
    total = std::max<uint64_t>(total, R.off[q] + R.bytes[q]);
  }
  R.total = (total + g - 1) / g * g;
  const bool multi_proc = W > 1 && !ctx->lcomm;
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = ctx->cfg.device;
  prop.requestedHandleTypes = multi_proc ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
  CUmemGenericAllocationHandle local;
  DRV(api->MemCreate(&local, my_bytes, &prop, 0), "cuMemCreate");
  R.handles.assign(W, 0);
  R.handles[me] = local;
  if (W > 1 && ctx->lcomm) {  // threads of one process: handles are process-wide
    uint64_t h = (uint64_t)local;
    std::vector<uint64_t> hs(W);
    TRY(host_allgather(ctx, &h, 8, hs.data()));
    for (int q = 0; q < W; q++) R.handles[q] = (CUmemGenericAllocationHandle)hs[q];
    R.own_only = true;
  } else if (multi_proc) {
    int fd = -1;
    DRV(api->MemExportToShareableHandle(&fd, local, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExport");
    std::vector<int> fds;
    if (!ctx->chan || !ctx->chan->allgather_fds(fd, &fds)) FAIL(GSMART_E_NCCL, "file-descriptor exchange failed");
    for (int q = 0; q < W; q++) {
      if (q == me) continue;
      CUmemGenericAllocationHandle h;
      DRV(api->MemImportFromShareableHandle(&h, (void*)(uintptr_t)fds[q], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
          "cuMemImport");
      ::close(fds[q]);
      R.handles[q] = h;
    }
    ::close(fd);
  }
  CUdeviceptr va = 0;
  DRV(api->MemAddressReserve(&va, R.total, g, 0, 0), "cuMemAddressReserve");
  R.va = va;
  for (int q = 0; q < W; q++) DRV(api->MemMap(va + R.off[q], R.bytes[q], 0, R.handles[q], 0), "cuMemMap");
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = ctx->cfg.device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (int q = 0; q < W; q++)  // per chunk: the reservation may have holes (parked empty chunks)
    DRV(api->MemSetAccess(va + R.off[q], R.bytes[q], &acc, 1), "cuMemSetAccess");
  R.rank = me;
  *out = R;
  return GSMART_OK;
}

void sym_free(gsmart_ctx* ctx, SymRegion* R) {
  const VmmApi* api = vmm();
  if (!api || !R->va) return;
  ctx_sync(ctx);  // this rank's work on the region is done (peers keep their own mappings)
  for (size_t q = 0; q < R->off.size(); q++) api->MemUnmap(R->va + R->off[q], R->bytes[q]);
  api->MemAddressFree(R->va, R->total);
  for (size_t q = 0; q < R->handles.size(); q++)
    if (!R->own_only || (int)q == R->rank) api->MemRelease(R->handles[q]);
  *R = SymRegion();
}

// ------------------------------------------------------------------ device barrier
// One CTA: lane q < world stores gen into rank q's flag word for this rank
// (release, system scope) then spins until every rank's flag word here holds
// >= gen (acquire).  Kernels before and after it on the stream are ordered by
// stream order; the fence makes this rank's earlier peer stores/atomics visible
// before its signal.
// Unlike the other query kernels it lets its dependents launch only AFTER the
// barrier: an early-launched successor grid would sit resident (at its
// griddepcontrol.wait) and could take the SMs other ranks' kernels need to
// reach this barrier — with ranks sharing a device, a deadlock.
__global__ void k_rank_barrier(unsigned long long* flags_local, SymDelta d, uint32_t rank, uint32_t world,
                               const unsigned long long* gen_base, uint32_t gen_off) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const unsigned long long gen = *(volatile const unsigned long long*)gen_base + gen_off;
  const uint32_t q = threadIdx.x;
  if (q < world) {
    __threadfence_system();
    unsigned long long* dst = flags_local + d.words[q] / 2 + rank;  // rank q's flag array, my slot
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(gen) : "memory");
    unsigned long long v = 0;
    const long long t0 = clock64();
    do {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags_local + q) : "memory");
      if (v < gen) {
        __nanosleep(256);
        // a peer that never arrives is a bug (mismatched collective sequence): fail
        // loudly (~30 s at 2 GHz) instead of hanging the device
        if (clock64() - t0 > 60000000000ll) {
          printf("gsmart: rank %u barrier gen %llu (base %llu + %u) timed out waiting for rank %u (flag %llu)\n", rank,
                 gen, *(volatile const unsigned long long*)gen_base, gen_off, q, v);
          __trap();
        }
      }
    } while (v < gen);
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" :::);
}

cudaError_t launch_rank_barrier(unsigned long long* flags_local, const SymDelta& d, uint32_t rank, uint32_t world,
                                const unsigned long long* gen_base, uint32_t gen_off, cudaStream_t st) {
  return pdl_launch(k_rank_barrier, 1, 32, st, flags_local, d, rank, world, gen_base, gen_off);
}

}  // namespace gsm

// Host-side self-check of the ranks-as-processes channel (no device needed):
// rendezvous on the unique id, all-gather one value per rank, and pass one file
// descriptor per rank (a pipe holding the rank's number) to every other rank.
extern "C" gsmart_status gsmart_rendezvous_check(const void* id128, int rank, int world, uint64_t value,
                                                 uint64_t* all_values) {
  if (!id128 || !all_values || world < 1 || world > gsm::MAX_WORLD || rank < 0 || rank >= world)
    return GSMART_E_INVALID_ARG;
  gsm::SockChan c;
  std::string err;
  if (world > 1 && !c.open(id128, rank, world, &err)) {
    gsm::g_static_err = err;
    return GSMART_E_NCCL;
  }
  if (world == 1) {
    all_values[0] = value;
    return GSMART_OK;
  }
  if (!c.allgather(&value, 8, all_values)) return GSMART_E_NCCL;
  int p[2];
  if (pipe(p) != 0) return GSMART_E_NCCL;
  const int32_t me = rank;
  if (write(p[1], &me, 4) != 4) return GSMART_E_NCCL;
  ::close(p[1]);
  std::vector<int> fds;
  if (!c.allgather_fds(p[0], &fds)) return GSMART_E_NCCL;
  bool ok = true;
  for (int q = 0; q < world; q++) {
    if (q == rank) continue;
    int32_t got = -1;
    ok = ok && read(fds[q], &got, 4) == 4 && got == q;
    ::close(fds[q]);
  }
  ::close(p[0]);
  char x = 0;
  std::vector<char> bar(world);
  if (!c.allgather(&x, 1, bar.data())) return GSMART_E_NCCL;  // keep every fd alive until all have read
  if (!ok) {
    gsm::g_static_err = "descriptor exchange delivered wrong descriptors";
    return GSMART_E_NCCL;
  }
  return GSMART_OK;
}
