// f4 — N-Triples read + dictionary encode on the device (§6.2.1 steps 1-2,
// P:L408-L409; grammar and id order: DESIGN.md R24).
//
// Pipeline (all on ctx->st, one host read for the sizes and one for the
// dictionary sizes):
//   1 newline scan: per 64 KB chunk count '\n' (uint4 loads, __vcmpeq4), scan
//     the counts, write the newline positions in order -> line bounds;
//   2 parse: one thread per line -> term (offset, length) x3 or skip / error
//     (first bad line = atomicMin);
//   3 compact the triple lines (scan of the valid flags) and hash every term
//     occurrence (FNV-1a 64 + murmur finaliser);
//   4 per kind (entities: 2 occurrences per triple, s then o; predicates: 1):
//     radix sort (hash, occurrence) pairs — stable, so each equal-hash run
//     starts at the term's first occurrence; run heads; equal hashes with
//     different bytes = collision (checked for every adjacent pair);
//     id = rank of the head's occurrence among all heads (scan of a mark
//     array indexed by occurrence) = first-appearance order;
//   5 scatter ids into s/p/o; the sorted unique hashes + ids are the lookup
//     table, (offset, length) by id the decode table.
#include <algorithm>
#include <string>
#include <vector>

#include "kernels.h"
#include "runtime.h"

namespace gsm {

namespace {

constexpr int IG_T = 256;                             // threads per CTA
constexpr int IG_PER = 256;                           // bytes per thread in the newline scan
constexpr uint64_t IG_CHUNK = (uint64_t)IG_T * IG_PER;  // 64 KB per CTA

__host__ __device__ inline uint64_t term_hash(const uint8_t* b, uint64_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < n; i++) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  h ^= n;
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  h *= 0xc4ceb9fe1a85ec53ull;
  h ^= h >> 33;
  return h;
}

__device__ __forceinline__ uint32_t nl_in_word(uint32_t w) { return __popc(__vcmpeq4(w, 0x0a0a0a0au)) >> 3; }

// '\n' bytes in [lo, hi) of this thread's IG_PER-byte slice (lo is 256-aligned)
__device__ uint32_t count_nl(const uint8_t* __restrict__ t, uint64_t lo, uint64_t hi) {
  uint32_t c = 0;
  if (hi - lo == IG_PER) {
    const uint4* v = reinterpret_cast<const uint4*>(t + lo);
#pragma unroll 4
    for (int k = 0; k < IG_PER / 16; k++) {
      const uint4 x = __ldg(v + k);
      c += nl_in_word(x.x) + nl_in_word(x.y) + nl_in_word(x.z) + nl_in_word(x.w);
    }
  } else {
    for (uint64_t j = lo; j < hi; j++) c += t[j] == '\n';
  }
  return c;
}

__global__ void __launch_bounds__(IG_T) k_ig_count(const uint8_t* __restrict__ t, uint64_t n, uint32_t* cnt) {
  __shared__ uint32_t ws[IG_T / 32];
  const uint64_t lo = blockIdx.x * IG_CHUNK + (uint64_t)threadIdx.x * IG_PER;
  uint32_t c = lo < n ? count_nl(t, lo, min(lo + IG_PER, n)) : 0;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < IG_T / 32; w++) s += ws[w];
    cnt[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(IG_T) k_ig_nlpos(const uint8_t* __restrict__ t, uint64_t n,
                                                   const uint32_t* __restrict__ base, uint64_t* __restrict__ pos) {
  __shared__ uint32_t sm[32];
  const uint64_t lo = blockIdx.x * IG_CHUNK + (uint64_t)threadIdx.x * IG_PER;
  const uint64_t hi = lo < n ? min(lo + IG_PER, n) : lo;
  const uint32_t c = lo < n ? count_nl(t, lo, hi) : 0;
  uint64_t w = (uint64_t)base[blockIdx.x] + block_exclusive_scan<uint32_t>(c, sm, nullptr);
  if (c == 0) return;
  for (uint64_t j = lo; j < hi; j++)
    if (t[j] == '\n') pos[w++] = j;
}

__device__ __forceinline__ bool sp_tab(uint8_t c) { return c == ' ' || c == '\t'; }
__device__ __forceinline__ bool sp_tab_cr(uint8_t c) { return c == ' ' || c == '\t' || c == '\r'; }

// one term at t[i] of a line ending at e: *end = one past it; false = malformed
__device__ bool ig_term(const uint8_t* __restrict__ t, uint64_t i, uint64_t e, uint64_t* end) {
  const uint8_t c = t[i];
  uint64_t j;
  if (c == '<') {
    for (j = i; j < e && t[j] != '>'; j++) {
    }
    if (j >= e) return false;
    *end = j + 1;
    return true;
  }
  if (c == '_') {
    for (j = i; j < e && !sp_tab(t[j]); j++) {
    }
    *end = j;
    return true;
  }
  if (c == '"') {
    j = i + 1;
    while (true) {
      if (j >= e) return false;
      if (t[j] == '\\') {
        j += 2;
        continue;
      }
      if (t[j] == '"') break;
      j++;
    }
    j++;
    if (j < e && t[j] == '@') {
      while (j < e && !sp_tab(t[j])) j++;
    } else if (j + 1 < e && t[j] == '^' && t[j + 1] == '^') {
      uint64_t k = j;
      while (k < e && t[k] != '>') k++;
      if (k >= e) return false;
      j = k + 1;
    }
    *end = j;
    return true;
  }
  return false;
}

struct LineTerms {
  uint64_t* off;  // [3 * L]: s, p, o of line i at 3i..3i+2
  uint32_t* len;
  uint32_t* valid;  // [L]: 1 = a triple line
};

// line i = [start, end): 0 / after the (i-1)th newline, up to the ith newline / n
__global__ void k_ig_parse(const uint8_t* __restrict__ t, uint64_t n, const uint64_t* __restrict__ nl, uint64_t n_nl,
                           LineTerms lt, unsigned long long* bad_line) {
  const uint64_t L = n_nl + 1;
  for (uint64_t li = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; li < L; li += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s0 = li ? nl[li - 1] + 1 : 0, e = li < n_nl ? nl[li] : n;
    lt.valid[li] = 0;
    uint64_t i = s0;
    while (i < e && sp_tab_cr(t[i])) i++;
    if (i == e || t[i] == '#') continue;
    bool ok = true;
    uint64_t b[3], en[3];
    for (int k = 0; k < 3 && ok; k++) {
      while (i < e && sp_tab(t[i])) i++;
      if (i >= e) {
        ok = false;
        break;
      }
      b[k] = i;
      ok = ig_term(t, i, e, &en[k]);
      i = en[k];
    }
    if (ok) ok = t[b[1]] == '<' && t[b[0]] != '"';
    if (ok) {  // the rest, stripped of ' ', '\t', '\r', must be exactly "."
      uint64_t a = i, z = e;
      while (a < z && sp_tab_cr(t[a])) a++;
      while (z > a && sp_tab_cr(t[z - 1])) z--;
      ok = z - a == 1 && t[a] == '.';
    }
    if (ok)
      for (int k = 0; k < 3; k++) ok = ok && en[k] - b[k] < 0xffffffffull;
    if (!ok) {
      atomicMin(bad_line, (unsigned long long)li);
      continue;
    }
    lt.valid[li] = 1;
    for (int k = 0; k < 3; k++) {
      lt.off[3 * li + k] = b[k];
      lt.len[3 * li + k] = (uint32_t)(en[k] - b[k]);
    }
  }
}

// compact the triple lines to triple order and hash each term occurrence
__global__ void k_ig_hash(const uint8_t* __restrict__ t, uint64_t L, LineTerms lt, const uint32_t* __restrict__ tpos,
                          uint64_t* __restrict__ toff, uint32_t* __restrict__ tlen, uint64_t* __restrict__ ek,
                          uint32_t* __restrict__ ev, uint64_t* __restrict__ pk, uint32_t* __restrict__ pv) {
  for (uint64_t li = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; li < L; li += (uint64_t)gridDim.x * blockDim.x) {
    if (!lt.valid[li]) continue;
    const uint64_t tr = tpos[li];
    uint64_t h[3];
    for (int k = 0; k < 3; k++) {
      const uint64_t o = lt.off[3 * li + k];
      const uint32_t n = lt.len[3 * li + k];
      toff[3 * tr + k] = o;
      tlen[3 * tr + k] = n;
      h[k] = term_hash(t + o, n);
    }
    ek[2 * tr] = h[0];
    ek[2 * tr + 1] = h[2];
    ev[2 * tr] = (uint32_t)(2 * tr);
    ev[2 * tr + 1] = (uint32_t)(2 * tr + 1);
    pk[tr] = h[1];
    pv[tr] = (uint32_t)tr;
  }
}

// term slot (into toff/tlen) of occurrence `occ` of a kind
__device__ __forceinline__ uint64_t occ_term(uint32_t occ, int kind) {
  return kind == 0 ? 3ull * (occ >> 1) + ((occ & 1) ? 2 : 0) : 3ull * occ + 1;
}

__device__ bool same_term(const uint8_t* __restrict__ t, uint64_t oa, uint32_t la, uint64_t ob, uint32_t lb) {
  if (la != lb) return false;
  for (uint32_t i = 0; i < la; i++)
    if (t[oa + i] != t[ob + i]) return false;
  return true;
}

// run heads of the sorted (hash, occ) pairs; mark[occ] = 1 at a head (every
// occ is written once); collision = equal hashes, different bytes
__global__ void k_ig_heads(const uint8_t* __restrict__ t, const uint64_t* __restrict__ k,
                           const uint32_t* __restrict__ v, uint64_t m, int kind, const uint64_t* __restrict__ toff,
                           const uint32_t* __restrict__ tlen, uint32_t* __restrict__ head,
                           uint32_t* __restrict__ mark, unsigned long long* collision) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const bool hd = i == 0 || k[i] != k[i - 1];
    head[i] = hd;
    mark[v[i]] = hd;
    if (!hd) {
      const uint64_t a = occ_term(v[i], kind), b = occ_term(v[i - 1], kind);
      if (!same_term(t, toff[a], tlen[a], toff[b], tlen[b])) atomicAdd(collision, 1ull);
    }
  }
}

// at each head: run r gets id = idx[occ] (rank among first occurrences); the
// lookup table (hash, id) by run and the decode table (offset, length) by id
__global__ void k_ig_tables(const uint64_t* __restrict__ k, const uint32_t* __restrict__ v, uint64_t m, int kind,
                            const uint32_t* __restrict__ head, const uint32_t* __restrict__ runx,
                            const uint32_t* __restrict__ idx, const uint64_t* __restrict__ toff,
                            const uint32_t* __restrict__ tlen, uint64_t* __restrict__ hash,
                            uint32_t* __restrict__ hid, uint64_t* __restrict__ doff, uint32_t* __restrict__ dlen) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    if (!head[i]) continue;
    const uint32_t r = runx[i], occ = v[i], id = idx[occ];
    const uint64_t ts = occ_term(occ, kind);
    hash[r] = k[i];
    hid[r] = id;
    doff[id] = toff[ts];
    dlen[id] = tlen[ts];
  }
}

// every occurrence takes its run's id: entities -> s (even occ) / o (odd);
// predicates -> p = id + 1
__global__ void k_ig_scatter(const uint32_t* __restrict__ v, uint64_t m, int kind, const uint32_t* __restrict__ head,
                             const uint32_t* __restrict__ runx, const uint32_t* __restrict__ hid,
                             uint32_t* __restrict__ s, uint32_t* __restrict__ p, uint32_t* __restrict__ o) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = hid[runx[i] + head[i] - 1], occ = v[i];
    if (kind == 0)
      ((occ & 1) ? o : s)[occ >> 1] = id;
    else
      p[occ] = id + 1;
  }
}

__global__ void k_ig_lookup(const uint8_t* __restrict__ t, const uint64_t* __restrict__ hash,
                            const uint32_t* __restrict__ hid, uint32_t u, const uint64_t* __restrict__ doff,
                            const uint32_t* __restrict__ dlen, const uint8_t* __restrict__ q, uint64_t qlen,
                            uint64_t h, unsigned long long* out) {
  uint32_t lo = 0, hi = u;
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (hash[mid] < h)
      lo = mid + 1;
    else
      hi = mid;
  }
  unsigned long long r = 0xffffffffull;
  if (lo < u && hash[lo] == h) {
    const uint32_t id = hid[lo];
    bool eq = dlen[id] == qlen;
    for (uint64_t i = 0; eq && i < qlen; i++) eq = t[doff[id] + i] == q[i];
    if (eq) r = id;
  }
  *out = r;
}

unsigned grid_of(uint64_t n, int sm_count) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count * 16));
}

}  // namespace

void dict_free(gsmart_ctx* ctx) {
  Dict& d = ctx->dict;
  dfree(ctx, d.text);
  for (int k = 0; k < 2; k++) {
    dfree(ctx, d.off[k]);
    dfree(ctx, d.len[k]);
    dfree(ctx, d.hash[k]);
    dfree(ctx, d.hid[k]);
  }
  d = Dict{};
}

// encode one kind: sorts (keys, occ) in place (ping-pong with k1/v1), fills
// the dictionary tables of the kind and scatters ids into s/p/o
static gsmart_status encode_kind(gsmart_ctx* ctx, Scratch& sc, int kind, uint64_t* k0, uint32_t* v0, uint64_t m,
                                 const uint64_t* toff, const uint32_t* tlen, unsigned long long* d_cnt,
                                 uint32_t* n_unique) {
  cudaStream_t st = ctx->st;
  Dict& d = ctx->dict;
  uint64_t* k1;
  uint32_t* v1;
  void* rtmp;
  const size_t rb = radix_tmp_bytes(m);
  TRY(sc.get(&k1, m));
  TRY(sc.get(&v1, m));
  TRY(sc.get((char**)&rtmp, rb));
  int second = 0, nl = 0;
  CU(radix_sort_pairs_u64_u32(k0, k1, v0, v1, m, 0, 64, rtmp, rb, st, &second, &nl, false));
  uint64_t* k = second ? k1 : k0;
  uint32_t* v = second ? v1 : v0;
  uint32_t *head, *mark, *runx, *idx;
  TRY(sc.get(&head, m));
  TRY(sc.get(&mark, m));
  TRY(sc.get(&runx, m));
  TRY(sc.get(&idx, m));
  void* stmp;
  TRY(sc.get((char**)&stmp, scan_tmp_bytes(m)));
  CU(cudaMemsetAsync(d_cnt, 0, 3 * 8, st));
  k_ig_heads<<<grid_of(m, ctx->sm_count), 256, 0, st>>>(d.text, k, v, m, kind, toff, tlen, head, mark, d_cnt + 2);
  CU(cudaGetLastError());
  CU(scan_exclusive_u32(head, runx, m, d_cnt, stmp, st, nullptr));
  CU(scan_exclusive_u32(mark, idx, m, d_cnt + 1, stmp, st, nullptr));
  unsigned long long h[3];
  TRY(readback(ctx, st, ctx->h_pin, d_cnt, 3, h));
  if (h[2]) FAIL(GSMART_E_UNSUPPORTED, "64-bit term hash collision between distinct terms");
  const uint64_t u = h[0];
  if (kind == 0 && u >= 0x80000000ull) FAIL(GSMART_E_UNSUPPORTED, "more than 2^31 - 1 distinct entities");
  if (kind == 1 && u > 65534) FAIL(GSMART_E_UNSUPPORTED, "more than 65534 distinct predicates");
  TRY(dalloc(ctx, &d.hash[kind], u));
  TRY(dalloc(ctx, &d.hid[kind], u));
  TRY(dalloc(ctx, &d.off[kind], u));
  TRY(dalloc(ctx, &d.len[kind], u));
  d.n[kind] = (uint32_t)u;
  k_ig_tables<<<grid_of(m, ctx->sm_count), 256, 0, st>>>(k, v, m, kind, head, runx, idx, toff, tlen, d.hash[kind],
                                                         d.hid[kind], d.off[kind], d.len[kind]);
  CU(cudaGetLastError());
  k_ig_scatter<<<grid_of(m, ctx->sm_count), 256, 0, st>>>(v, m, kind, head, runx, d.hid[kind], ctx->d_s, ctx->d_p,
                                                          ctx->d_o);
  CU(cudaGetLastError());
  *n_unique = (uint32_t)u;
  return GSMART_OK;
}

static gsmart_status ingest(gsmart_ctx* ctx, const char* text, uint64_t n, uint32_t flags, uint64_t* out_n,
                            uint32_t* out_ne, uint32_t* out_np) {
  cudaStream_t st = ctx->st;
  Dict& d = ctx->dict;
  TRY(dalloc(ctx, &d.text, n + 16));
  d.bytes = n;
  if (n && flags == GSMART_PTR_HOST)
    TRY(h2d_staged(ctx, d.text, text, n, st));
  else if (n)
    CU(cudaMemcpyAsync(d.text, text, n, cudaMemcpyDeviceToDevice, st));
  Scratch sc(ctx);
  unsigned long long* d_cnt;
  TRY(sc.get(&d_cnt, 8));
  // 1 newline positions
  const uint64_t chunks = std::max<uint64_t>(1, (n + IG_CHUNK - 1) / IG_CHUNK);
  if (chunks >= 0xffffffffull) FAIL(GSMART_E_UNSUPPORTED, "text too large");
  uint32_t* cnt;
  void* stmp;
  TRY(sc.get(&cnt, chunks));
  TRY(sc.get((char**)&stmp, scan_tmp_bytes(chunks)));
  k_ig_count<<<(unsigned)chunks, IG_T, 0, st>>>(d.text, n, cnt);
  CU(cudaGetLastError());
  CU(scan_exclusive_u32(cnt, cnt, chunks, d_cnt, stmp, st, nullptr));
  unsigned long long h[2];
  TRY(readback(ctx, st, ctx->h_pin, d_cnt, 1, h));
  const uint64_t n_nl = h[0], L = n_nl + 1;
  if (L >= 0xffffffffull) FAIL(GSMART_E_UNSUPPORTED, "more than 2^32 - 2 lines");
  uint64_t* nl;
  TRY(sc.get(&nl, n_nl));
  k_ig_nlpos<<<(unsigned)chunks, IG_T, 0, st>>>(d.text, n, cnt, nl);
  CU(cudaGetLastError());
  // 2 parse
  LineTerms lt;
  TRY(sc.get(&lt.off, 3 * L));
  TRY(sc.get(&lt.len, 3 * L));
  TRY(sc.get(&lt.valid, L));
  CU(cudaMemsetAsync(d_cnt + 1, 0xff, 8, st));
  k_ig_parse<<<grid_of(L, ctx->sm_count), 256, 0, st>>>(d.text, n, nl, n_nl, lt, d_cnt + 1);
  CU(cudaGetLastError());
  uint32_t* tpos;
  TRY(sc.get(&tpos, L));
  void* stmp2;
  TRY(sc.get((char**)&stmp2, scan_tmp_bytes(L)));
  CU(scan_exclusive_u32(lt.valid, tpos, L, d_cnt, stmp2, st, nullptr));
  TRY(readback(ctx, st, ctx->h_pin, d_cnt, 2, h));
  if (h[1] != ~0ull) FAIL(GSMART_E_INVALID_ARG, "line " + std::to_string(h[1]) + ": malformed N-Triples line");
  const uint64_t T = h[0];
  if (T >= 0x80000000ull) FAIL(GSMART_E_UNSUPPORTED, "more than 2^31 - 1 triples");
  if (T == 0) {
    dict_free(ctx);
    if (out_n) *out_n = 0;
    if (out_ne) *out_ne = 0;
    if (out_np) *out_np = 0;
    return GSMART_OK;
  }
  // 3 compact + hash
  uint64_t *toff, *ek, *pk;
  uint32_t *tlen, *ev, *pv;
  TRY(sc.get(&toff, 3 * T));
  TRY(sc.get(&tlen, 3 * T));
  TRY(sc.get(&ek, 2 * T));
  TRY(sc.get(&ev, 2 * T));
  TRY(sc.get(&pk, T));
  TRY(sc.get(&pv, T));
  k_ig_hash<<<grid_of(L, ctx->sm_count), 256, 0, st>>>(d.text, L, lt, tpos, toff, tlen, ek, ev, pk, pv);
  CU(cudaGetLastError());
  TRY(dalloc(ctx, &ctx->d_s, T));
  TRY(dalloc(ctx, &ctx->d_p, T));
  TRY(dalloc(ctx, &ctx->d_o, T));
  // 4-5 per kind
  uint32_t ne = 0, np = 0;
  TRY(encode_kind(ctx, sc, 0, ek, ev, 2 * T, toff, tlen, d_cnt, &ne));
  TRY(encode_kind(ctx, sc, 1, pk, pv, T, toff, tlen, d_cnt, &np));
  ctx->n_triples = T;
  ctx->N = ne;
  ctx->P = np;
  ctx->pred_bytes = np <= 254 ? 1 : 2;
  d.valid = true;
  if (out_n) *out_n = T;
  if (out_ne) *out_ne = ne;
  if (out_np) *out_np = np;
  return GSMART_OK;
}

}  // namespace gsm

using namespace gsm;

extern "C" gsmart_status gsmart_ingest_ntriples(gsmart_ctx* ctx, const char* text, uint64_t bytes, uint32_t flags,
                                                uint64_t* n_triples, uint32_t* n_entities, uint32_t* n_predicates) {
  if (!ctx) return GSMART_E_INVALID_ARG;
  if (ctx->poisoned) return GSMART_E_CUDA;
  if (bytes && !text) FAIL(GSMART_E_INVALID_ARG, "null text");
  if (flags != GSMART_PTR_HOST && flags != GSMART_PTR_DEVICE) FAIL(GSMART_E_INVALID_ARG, "flags must be PTR_HOST or PTR_DEVICE");
  if (ctx->world != 1) FAIL(GSMART_E_UNSUPPORTED, "ingest needs world == 1");
  CU(cudaSetDevice(ctx->cfg.device));
  free_lspm(ctx);
  dict_free(ctx);
  dfree(ctx, ctx->d_s);
  dfree(ctx, ctx->d_p);
  dfree(ctx, ctx->d_o);
  ctx->d_s = ctx->d_p = ctx->d_o = nullptr;
  ctx->n_triples = 0;
  ctx->N = 0;
  gsmart_status s = ingest(ctx, text, bytes, flags, n_triples, n_entities, n_predicates);
  if (s != GSMART_OK) {  // nothing loaded
    std::string err = ctx->err;
    cudaStreamSynchronize(ctx->st);
    dict_free(ctx);
    dfree(ctx, ctx->d_s);
    dfree(ctx, ctx->d_p);
    dfree(ctx, ctx->d_o);
    ctx->d_s = ctx->d_p = ctx->d_o = nullptr;
    ctx->n_triples = 0;
    ctx->N = 0;
    ctx->err = err;
    return s;
  }
  CU(cudaStreamSynchronize(ctx->st));
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_dict_lookup(gsmart_ctx* ctx, uint32_t kind, const char* term, uint64_t len,
                                            uint32_t* id) {
  if (!ctx) return GSMART_E_INVALID_ARG;
  if (ctx->poisoned) return GSMART_E_CUDA;
  if (kind > 1 || !id || (len && !term)) FAIL(GSMART_E_INVALID_ARG, "bad kind / null pointer");
  const Dict& d = ctx->dict;
  if (!d.valid) FAIL(GSMART_E_STATE, "no dictionary: the loaded data did not come from gsmart_ingest_ntriples");
  CU(cudaSetDevice(ctx->cfg.device));
  Scratch sc(ctx);
  uint8_t* q;
  unsigned long long* out;
  TRY(sc.get(&q, len + 1));
  TRY(sc.get(&out, 1));
  if (len) CU(cudaMemcpyAsync(q, term, len, cudaMemcpyHostToDevice, ctx->st));
  k_ig_lookup<<<1, 1, 0, ctx->st>>>(d.text, d.hash[kind], d.hid[kind], d.n[kind], d.off[kind], d.len[kind], q, len,
                                    term_hash((const uint8_t*)term, len), out);
  CU(cudaGetLastError());
  unsigned long long r;
  TRY(readback(ctx, ctx->st, ctx->h_pin, out, 1, &r));
  *id = r == 0xffffffffull ? 0xffffffffu : (uint32_t)r + (kind == 1 ? 1 : 0);
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_dict_term(gsmart_ctx* ctx, uint32_t kind, uint32_t id, char* buf, uint64_t cap,
                                          uint64_t* len) {
  if (!ctx) return GSMART_E_INVALID_ARG;
  if (ctx->poisoned) return GSMART_E_CUDA;
  if (kind > 1 || !len || (cap && !buf)) FAIL(GSMART_E_INVALID_ARG, "bad kind / null pointer");
  const Dict& d = ctx->dict;
  if (!d.valid) FAIL(GSMART_E_STATE, "no dictionary: the loaded data did not come from gsmart_ingest_ntriples");
  const uint32_t i = kind == 1 ? id - 1 : id;
  if ((kind == 1 && id == 0) || i >= d.n[kind]) FAIL(GSMART_E_INVALID_ARG, "id out of range");
  CU(cudaSetDevice(ctx->cfg.device));
  uint64_t off = 0;
  uint32_t l = 0;
  CU(cudaMemcpyAsync(&off, d.off[kind] + i, 8, cudaMemcpyDeviceToHost, ctx->st));
  CU(cudaMemcpyAsync(&l, d.len[kind] + i, 4, cudaMemcpyDeviceToHost, ctx->st));
  CU(cudaStreamSynchronize(ctx->st));
  *len = l;
  if (cap && l) {
    CU(cudaMemcpyAsync(buf, d.text + off, std::min<uint64_t>(cap, l), cudaMemcpyDeviceToHost, ctx->st));
    CU(cudaStreamSynchronize(ctx->st));
  }
  return GSMART_OK;
}

extern "C" gsmart_status gsmart_triples_get(const gsmart_ctx* ctx, const uint32_t** s, const uint32_t** p,
                                            const uint32_t** o, uint64_t* n) {
  if (!ctx) return GSMART_E_INVALID_ARG;
  if (s) *s = ctx->d_s;
  if (p) *p = ctx->d_p;
  if (o) *o = ctx->d_o;
  if (n) *n = ctx->n_triples;
  return GSMART_OK;
}
