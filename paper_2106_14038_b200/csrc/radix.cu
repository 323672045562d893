// Hand-written sm_100a LSD radix sort (onesweep form) — the sort of the LSpM
// build (a1: (row, pred, col) keys) and of large result rows
// (a9).  HBM-bound: every pass reads and writes each key (and payload) once.
//
// Per sort: one histogram launch counts the 8-bit digits of every pass at once
// (the key multiset does not change between passes) and one tiny launch scans
// them; then one launch per pass.  A pass kernel takes tiles of RS_TILE keys in
// ticket order (forward progress for the look-back), and per tile:
//   1. loads its keys warp-striped (coalesced) and ranks them in original order
//      with a warp multi-split (__match_any_sync per item, per-warp digit
//      counters in shared memory) — stable;
//   2. publishes its per-digit counts and finds, per digit, the count of that
//      digit in all earlier tiles by a decoupled look-back (one thread per
//      digit, epoch-stamped status words: no clearing between passes);
//   3. scatters keys (and payload) into shared memory in digit order, then
//      writes them out in that order: runs of one digit go to consecutive
//      global addresses.
// Passes whose digit is the same for every key are skipped (read from the
// histogram on the host before launching).
#include <algorithm>
#include <vector>

#include "kernels.h"

namespace gsm {

constexpr int RS_T = 512, RS_I = 8, RS_TILE = RS_T * RS_I, RS_W = RS_T / 32;
constexpr int RS_MAX_PASSES = 8;
constexpr uint64_t RS_VMASK = (1ull << 56) - 1;

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
  return (uint32_t)(k >> shift) & 0xffu;
}

// digit counts of every pass; hist[p * 256 + d] (64-bit)
template <typename K>
__global__ void __launch_bounds__(256) k_rs_hist(const K* __restrict__ keys, uint64_t n, int b0, int npass,
                                                 unsigned long long* __restrict__ hist, const int* skip) {
  __shared__ uint32_t sh[RS_MAX_PASSES][256];
  if (skip && *skip) return;
  for (int i = threadIdx.x; i < RS_MAX_PASSES * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const K k = keys[i];
#pragma unroll
    for (int p = 0; p < RS_MAX_PASSES; p++)
      if (p < npass) atomicAdd(&sh[p][digit_of(k, b0 + 8 * p)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) {
    const uint32_t c = (&sh[0][0])[i];
    if (c) atomicAdd(hist + i, (unsigned long long)c);
  }
}

// exclusive scan of each pass's 256 counts (one CTA per pass): base[p * 256 + d]
__global__ void __launch_bounds__(256) k_rs_scan(const unsigned long long* __restrict__ hist,
                                                 unsigned long long* __restrict__ base) {
  __shared__ unsigned long long sm[32];
  const int p = blockIdx.x;
  const unsigned long long v = hist[p * 256 + threadIdx.x];
  base[p * 256 + threadIdx.x] = block_exclusive_scan<unsigned long long>(v, sm, nullptr);
}

template <typename K, typename V, bool HAS_V>
__global__ void __launch_bounds__(RS_T) k_rs_pass(const K* __restrict__ kin, K* __restrict__ kout,
                                                  const V* __restrict__ vin, V* __restrict__ vout, uint64_t n,
                                                  int shift, const unsigned long long* __restrict__ dbase,
                                                  unsigned long long* __restrict__ status, uint32_t* counter,
                                                  uint32_t epoch, const int* skip) {
  if (skip && *skip) return;  // the caller found the data already in order
  __shared__ uint32_t s_wh[RS_W][256];     // per-warp digit counts -> exclusive warp offsets
  __shared__ uint32_t s_local[256];        // tile-local start of each digit
  __shared__ unsigned long long s_glob[256];  // global start of each digit for this tile
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long sm_scan[32];
  extern __shared__ __align__(16) unsigned char rs_dyn[];  // keys [RS_TILE], then payload [RS_TILE]
  K* s_keys = reinterpret_cast<K*>(rs_dyn);
  V* s_vals = reinterpret_cast<V*>(rs_dyn + sizeof(K) * RS_TILE);
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  for (int i = threadIdx.x; i < RS_W * 256; i += RS_T) (&s_wh[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t t0 = (uint64_t)tile * RS_TILE;
  if (t0 >= n) return;
  const uint64_t wbase = t0 + (uint64_t)w * 32 * RS_I;
  K key[RS_I];
  V val[RS_I];
  uint32_t rank[RS_I];
  uint32_t valid = 0;
#pragma unroll
  for (int j = 0; j < RS_I; j++) {
    const uint64_t i = wbase + j * 32 + lane;
    if (i < n) {
      key[j] = kin[i];
      if constexpr (HAS_V) val[j] = vin[i];
      valid |= 1u << j;
    }
  }
  // 1. warp multi-split ranking, items in original order (j outer, lane inner)
#pragma unroll
  for (int j = 0; j < RS_I; j++) {
    const bool ok = (valid >> j) & 1u;
    const uint32_t d = ok ? digit_of(key[j], shift) : 0x100u;
    const uint32_t peers = __match_any_sync(GSM_FULL, d);
    const uint32_t before = __popc(peers & lanemask_lt());
    uint32_t b = 0;
    if (ok) b = s_wh[w][d];
    rank[j] = b + before;
    __syncwarp();
    if (ok && before == 0) s_wh[w][d] = b + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // 2. per digit: exclusive offsets over warps, tile count, look-back over tiles
  unsigned long long tcount = 0;
  if (threadIdx.x < 256) {
    const uint32_t d = threadIdx.x;
    uint32_t off = 0;
#pragma unroll
    for (int ww = 0; ww < RS_W; ww++) {
      const uint32_t c = s_wh[ww][d];
      s_wh[ww][d] = off;
      off += c;
    }
    tcount = off;
    unsigned long long* st = status + (uint64_t)tile * 256 + d;
    const unsigned long long tagged_epoch = (unsigned long long)epoch << 56;
    if (tile == 0) {
      atomicExch(st, (2ull << 62) | tagged_epoch | tcount);
      s_glob[d] = dbase[d];
    } else {
      atomicExch(st, (1ull << 62) | tagged_epoch | tcount);
      unsigned long long excl = 0;
      for (int64_t t = (int64_t)tile - 1; t >= 0; t--) {
        unsigned long long v;
        do {
          v = *((volatile unsigned long long*)(status + (uint64_t)t * 256 + d));
        } while (((v >> 56) & 0x3full) != epoch || (v >> 62) == 0);
        excl += v & RS_VMASK;
        if ((v >> 62) == 2) break;
      }
      atomicExch(st, (2ull << 62) | tagged_epoch | (excl + tcount));
      s_glob[d] = dbase[d] + excl;
    }
  }
  // tile-local digit starts: exclusive scan of the tile counts over digits
  {
    const unsigned long long v = threadIdx.x < 256 ? tcount : 0ull;
    const unsigned long long ex = block_exclusive_scan<unsigned long long>(v, sm_scan, nullptr);
    if (threadIdx.x < 256) s_local[threadIdx.x] = (uint32_t)ex;
  }
  __syncthreads();
  // 3. scatter into shared memory in digit order, then out
#pragma unroll
  for (int j = 0; j < RS_I; j++) {
    if (!((valid >> j) & 1u)) continue;
    const uint32_t d = digit_of(key[j], shift);
    const uint32_t pos = s_local[d] + s_wh[w][d] + rank[j];
    s_keys[pos] = key[j];
    if constexpr (HAS_V) s_vals[pos] = val[j];
  }
  __syncthreads();
  const uint32_t m = (uint32_t)(n - t0 < (uint64_t)RS_TILE ? n - t0 : (uint64_t)RS_TILE);
  for (uint32_t i = threadIdx.x; i < m; i += RS_T) {
    const K k = s_keys[i];
    const uint32_t d = digit_of(k, shift);
    const unsigned long long g = s_glob[d] + (i - s_local[d]);
    kout[g] = k;
    if constexpr (HAS_V) vout[g] = s_vals[i];
  }
}

size_t radix_tmp_bytes(uint64_t n) {
  const uint64_t tiles = (n + RS_TILE - 1) / RS_TILE;
  return 2 * RS_MAX_PASSES * 256 * 8 + 64 * 4 + std::max<uint64_t>(tiles, 1) * 256 * 8 + 256;
}

template <typename K, typename V, bool HAS_V>
static cudaError_t radix_sort_t(K* k0, K* k1, V* v0, V* v1, uint64_t n, int b0, int b1, void* tmp, size_t tmp_bytes,
                                cudaStream_t st, int* in_second, int* launches, bool skip_trivial,
                                const int* skip = nullptr) {
  *in_second = 0;
  if (n <= 1 || b1 <= b0) return cudaSuccess;
  const size_t dyn = sizeof(K) * RS_TILE + (HAS_V ? sizeof(V) * RS_TILE : 0);
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_rs_pass<K, V, HAS_V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (tmp_bytes < radix_tmp_bytes(n)) return cudaErrorInvalidValue;
  const int npass_total = (b1 - b0 + 7) / 8;
  char* t = (char*)tmp;
  auto* hist = (unsigned long long*)t;
  auto* base = hist + RS_MAX_PASSES * 256;
  auto* counters = (uint32_t*)(base + RS_MAX_PASSES * 256);
  auto* status = (unsigned long long*)(counters + 64);
  const uint64_t tiles = (n + RS_TILE - 1) / RS_TILE;
  int nl = 0;
  // passes in groups of <= RS_MAX_PASSES (one histogram launch per group)
  int cur = 0;  // 0: data in (k0, v0); 1: in (k1, v1)
  for (int g0 = 0; g0 < npass_total; g0 += RS_MAX_PASSES) {
    const int np = std::min(RS_MAX_PASSES, npass_total - g0);
    const int gb = b0 + 8 * g0;
    cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)RS_MAX_PASSES * 256 * 8, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(counters, 0, 64 * 4, st);  // tile tickets of every pass
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(status, 0, tiles * 256 * 8, st);
    if (e != cudaSuccess) return e;
    const K* src = cur ? k1 : k0;
    const unsigned g = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 8);
    k_rs_hist<K><<<g, 256, 0, st>>>(src, n, gb, np, hist, skip);
    k_rs_scan<<<np, 256, 0, st>>>(hist, base);
    nl += 2;
    std::vector<unsigned long long> h(np * 256, 0);
    if (skip_trivial) {  // one host read of the histograms (build: a host-synchronous phase anyway)
      e = cudaMemcpyAsync(h.data(), hist, h.size() * 8, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return e;
    }
    for (int p = 0; p < np; p++) {
      bool trivial = false;
      for (int d = 0; d < 256; d++) trivial = trivial || h[p * 256 + d] == n;
      if (trivial) continue;  // one digit value for every key: the pass is the identity
      const K* ki = cur ? k1 : k0;
      K* ko = cur ? k0 : k1;
      const V* vi = cur ? v1 : v0;
      V* vo = cur ? v0 : v1;
      k_rs_pass<K, V, HAS_V><<<(unsigned)tiles, RS_T, dyn, st>>>(ki, ko, vi, vo, n, gb + 8 * p, base + p * 256, status,
                                                               counters + p, (uint32_t)(p + 1), skip);
      nl++;
      cur ^= 1;
    }
  }
  *in_second = cur;
  if (launches) *launches += nl;
  return cudaGetLastError();
}

cudaError_t radix_sort_keys_u64(uint64_t* k0, uint64_t* k1, uint64_t n, int b0, int b1, void* tmp, size_t tmp_bytes,
                                cudaStream_t st, int* in_second, int* launches, bool skip_trivial) {
  return radix_sort_t<uint64_t, uint32_t, false>(k0, k1, nullptr, nullptr, n, b0, b1, tmp, tmp_bytes, st, in_second,
                                                 launches, skip_trivial);
}

cudaError_t radix_sort_pairs_u64_u32(uint64_t* k0, uint64_t* k1, uint32_t* v0, uint32_t* v1, uint64_t n, int b0,
                                     int b1, void* tmp, size_t tmp_bytes, cudaStream_t st, int* in_second,
                                     int* launches, bool skip_trivial, const int* skip) {
  return radix_sort_t<uint64_t, uint32_t, true>(k0, k1, v0, v1, n, b0, b1, tmp, tmp_bytes, st, in_second, launches,
                                                skip_trivial, skip);
}

cudaError_t radix_sort_pairs_u32_u64(uint32_t* k0, uint32_t* k1, uint64_t* v0, uint64_t* v1, uint64_t n, int b0,
                                     int b1, void* tmp, size_t tmp_bytes, cudaStream_t st, int* in_second,
                                     int* launches, bool skip_trivial) {
  return radix_sort_t<uint32_t, uint64_t, true>(k0, k1, v0, v1, n, b0, b1, tmp, tmp_bytes, st, in_second, launches,
                                                skip_trivial);
}

}  // namespace gsm
