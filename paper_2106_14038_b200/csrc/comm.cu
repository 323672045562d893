// Collectives of the row-partitioned execution:
// all-gather of candidate-bitmap slices after each grouped evaluation, and the
// final gather of solution rows to rank 0.  NCCL when the context was created
// with a unique id; otherwise an in-process communicator (gsmart_comm) that
// copies device buffers between the ranks' threads.
#include <cstring>

#include "runtime.h"

using namespace gsm;

namespace gsm {

static gsmart_status nccl_check(gsmart_ctx* ctx, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return GSMART_OK;
  const NcclApi* api = nccl_api();
  ctx->err = std::string("NCCL error in ") + what + ": " + (api ? api->GetErrorString(r) : "?");
  return GSMART_E_NCCL;
}

gsmart_status coll_allgather(gsmart_ctx* ctx, cudaStream_t st, void* buf, size_t bytes) {
  if (ctx->world == 1) return GSMART_OK;
  char* b = (char*)buf;
  if (ctx->comm) {
    const NcclApi* api = nccl_api();
    return nccl_check(ctx, api->AllGather(b + (size_t)ctx->rank * bytes, b, bytes, ncclUint8, ctx->comm, st),
                      "ncclAllGather");
  }
  gsmart_comm* c = ctx->lcomm;
  CU(cudaStreamSynchronize(st));  // own slice complete before peers read it
  c->ptr[ctx->rank] = buf;
  c->dev[ctx->rank] = ctx->cfg.device;
  c->barrier();
  for (int q = 0; q < ctx->world; q++) {
    if (q == ctx->rank) continue;
    CU(cudaMemcpyPeerAsync(b + (size_t)q * bytes, ctx->cfg.device, (const char*)c->ptr[q] + (size_t)q * bytes,
                           c->dev[q], bytes, st));
  }
  CU(cudaStreamSynchronize(st));
  c->barrier();  // no rank reuses its buffer before every peer copied from it
  return GSMART_OK;
}

gsmart_status coll_allgather_host(gsmart_ctx* ctx, cudaStream_t st, unsigned long long v,
                                  std::vector<unsigned long long>* out) {
  out->assign(ctx->world, 0);
  if (ctx->world == 1) {
    (*out)[0] = v;
    return GSMART_OK;
  }
  if (ctx->comm) {
    const NcclApi* api = nccl_api();
    unsigned long long* d = nullptr;
    TRY(dalloc(ctx, &d, ctx->world, st));
    CU(cudaMemcpyAsync(d + ctx->rank, &v, 8, cudaMemcpyHostToDevice, st));
    gsmart_status s = nccl_check(ctx, api->AllGather(d + ctx->rank, d, 8, ncclUint8, ctx->comm, st), "ncclAllGather");
    if (s == GSMART_OK) {
      CU(cudaMemcpyAsync(out->data(), d, 8 * ctx->world, cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
    }
    dfree(st, d);
    return s;
  }
  gsmart_comm* c = ctx->lcomm;
  c->val[ctx->rank] = v;
  c->barrier();
  for (int q = 0; q < ctx->world; q++) (*out)[q] = c->val[q];
  c->barrier();
  return GSMART_OK;
}

gsmart_status coll_gather_root(gsmart_ctx* ctx, cudaStream_t st, const void* send, void* recv,
                               const std::vector<unsigned long long>& bytes) {
  const int W = ctx->world, me = ctx->rank;
  std::vector<unsigned long long> off(W, 0);
  for (int q = 1; q < W; q++) off[q] = off[q - 1] + bytes[q - 1];
  if (ctx->comm) {
    const NcclApi* api = nccl_api();
    api->GroupStart();
    if (me == 0) {
      for (int q = 1; q < W; q++)
        if (bytes[q]) api->Recv((char*)recv + off[q], bytes[q], ncclUint8, q, ctx->comm, st);
    } else if (bytes[me]) {
      api->Send(send, bytes[me], ncclUint8, 0, ctx->comm, st);
    }
    gsmart_status s = nccl_check(ctx, api->GroupEnd(), "ncclGroupEnd");
    if (s != GSMART_OK) return s;
    if (me == 0 && bytes[0]) CU(cudaMemcpyAsync(recv, send, bytes[0], cudaMemcpyDeviceToDevice, st));
    CU(cudaStreamSynchronize(st));
    return GSMART_OK;
  }
  gsmart_comm* c = ctx->lcomm;
  CU(cudaStreamSynchronize(st));
  c->ptr[me] = send;
  c->dev[me] = ctx->cfg.device;
  c->barrier();
  if (me == 0) {
    for (int q = 0; q < W; q++)
      if (bytes[q])
        CU(cudaMemcpyPeerAsync((char*)recv + off[q], ctx->cfg.device, c->ptr[q], c->dev[q], bytes[q], st));
    CU(cudaStreamSynchronize(st));
  }
  c->barrier();
  return GSMART_OK;
}

}  // namespace gsm

extern "C" gsmart_status gsmart_comm_create_local(int world, gsmart_comm** out) {
  if (!out || world < 1 || world > 1024) return GSMART_E_INVALID_ARG;
  auto* c = new gsmart_comm();
  c->world = world;
  c->ptr.assign(world, nullptr);
  c->dev.assign(world, 0);
  c->val.assign(world, 0);
  *out = c;
  return GSMART_OK;
}

extern "C" void gsmart_comm_destroy(gsmart_comm* c) { delete c; }

extern "C" gsmart_status gsmart_partition_words(uint32_t n_entities, int world, int rank, uint32_t* word_lo,
                                                uint32_t* word_hi) {
  if (world < 1 || rank < 0 || rank >= world || !word_lo || !word_hi) return GSMART_E_INVALID_ARG;
  const uint32_t W = (uint32_t)(((uint64_t)n_entities + 31) / 32);
  const uint32_t slice = partition_slice(W, world);
  const uint64_t lo = (uint64_t)rank * slice;
  *word_lo = (uint32_t)std::min<uint64_t>(lo, W);
  *word_hi = (uint32_t)std::min<uint64_t>(lo + slice, W);
  return GSMART_OK;
}
