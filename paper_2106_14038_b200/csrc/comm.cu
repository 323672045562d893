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

// All-gather of the ranks' slices of a replicated bitmap (the baseline exchange):
// rank q owns words [v_q / 32, ceil(v_q+1 / 32)).  NCCL: one broadcast per rank
// in a group (an all-gather with per-rank sizes; a 1-rank communicator runs the
// same calls); in-process ranks: peer copies between the threads' buffers.
gsmart_status coll_allgatherv(gsmart_ctx* ctx, cudaStream_t st, uint32_t* bm) {
  const int W = ctx->world;
  auto lo = [&](int q) { return W == 1 ? 0u : part_word_lo(ctx, q); };
  auto hi = [&](int q) { return W == 1 ? (ctx->N + 31) / 32 : part_word_hi(ctx, q); };
  if (ctx->comm) {
    const NcclApi* api = nccl_api();
    if (!api->Broadcast) FAIL(GSMART_E_NCCL, "ncclBroadcast not available");
    api->GroupStart();
    for (int q = 0; q < W; q++)
      if (hi(q) > lo(q))
        api->Broadcast(bm + lo(q), bm + lo(q), (size_t)(hi(q) - lo(q)) * 4, ncclUint8, q, ctx->comm, st);
    return nccl_check(ctx, api->GroupEnd(), "ncclGroupEnd (all-gather)");
  }
  if (W == 1) return GSMART_OK;
  gsmart_comm* c = ctx->lcomm;
  CU(cudaStreamSynchronize(st));  // own slice complete before peers read it
  c->ptr[ctx->rank] = bm;
  c->dev[ctx->rank] = ctx->cfg.device;
  c->barrier();
  for (int q = 0; q < W; q++) {
    if (q == ctx->rank || hi(q) <= lo(q)) continue;
    CU(cudaMemcpyPeerAsync(bm + lo(q), ctx->cfg.device, (const uint32_t*)c->ptr[q] + lo(q), c->dev[q],
                           (size_t)(hi(q) - lo(q)) * 4, st));
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
  if (!ctx->lcomm && ctx->chan) return host_allgather(ctx, &v, 8, out->data());
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
    dfree(ctx, st, d);
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
  c->blob.assign(world, std::string());
  *out = c;
  return GSMART_OK;
}

extern "C" void gsmart_comm_destroy(gsmart_comm* c) { delete c; }

extern "C" gsmart_status gsmart_partition_split(const uint64_t* bucket, uint32_t n_buckets, uint32_t n_entities,
                                                int world, uint32_t* v) {
  if (!v || world < 1 || world > MAX_WORLD || (n_buckets && !bucket)) return GSMART_E_INVALID_ARG;
  if (n_buckets != (uint32_t)(((uint64_t)n_entities + PART_ALIGN_ROWS - 1) / PART_ALIGN_ROWS))
    return GSMART_E_INVALID_ARG;
  unsigned long long total = 0;
  for (uint32_t i = 0; i < n_buckets; i++) total += bucket[i];
  v[0] = 0;
  uint32_t b = 0;
  unsigned long long cum = 0;
  for (int r = 1; r < world; r++) {
    const unsigned long long target = (total * (unsigned long long)r + world - 1) / world;
    while (b < n_buckets && cum < target) cum += bucket[b++];
    v[r] = (uint32_t)std::min<uint64_t>((uint64_t)b * PART_ALIGN_ROWS, n_entities);
  }
  v[world] = n_entities;
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_partition_get(const gsmart_ctx* ctx, uint32_t* v) {
  if (!ctx || !v) return GSMART_E_INVALID_ARG;
  if (ctx->world == 1) {
    v[0] = 0;
    v[1] = ctx->N;
    return GSMART_OK;
  }
  if (ctx->part.v.empty()) return GSMART_E_STATE;
  for (int q = 0; q <= ctx->world; q++) v[q] = ctx->part.v[q];
  return GSMART_OK;
}
