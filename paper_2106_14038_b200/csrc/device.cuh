// Device-side primitives of the gSmart hot path (sm_100a only).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define GSM_FULL 0xffffffffu

namespace gsm {

constexpr int MAXG = 16;          // max edges per direction in one group evaluation
constexpr int MAXL = 32;          // max trie levels (= variables)
constexpr int MAXC = 16;          // max closing edges per level
constexpr int MAXANC = 4;         // max materialised ancestor-binding columns per trie level
constexpr uint32_t SHORT_ROW = 32;     // rows <= this: one lane scans it (group filter)
constexpr uint32_t MED_SCAN = 64;      // longer rows: a lane probes up to this many entries of a label
constexpr uint32_t HEAVY_ROW = 16384;  // rows > this: split into chunks across CTAs
constexpr uint32_t HEAVY_CHUNK = 16384;
constexpr uint32_t EXP_CHUNK = 256;    // expansion work item = <= 256 segment entries

// counters (uint64) in the ctx stats array
enum Ctr { C_FILTER_ROWS = 0, C_FILTER_SCANNED, C_FILTER_MATCHED, C_SEED, C_EXPAND, C_CLOSING,
           C_HEAVY, C_FILTER_MASKED, C_FILTER_SKIPPED, C_PUSH, C_PUSH_MATCHED, C_NCTR };
static_assert(C_NCTR <= 16, "slot counter words [16, 32) hold the SkipIf change sequence");

// One LSpM format on the device: entries of row r are [rp[r], rp[r+1]) sorted by (pred, col).
template <typename PT>
struct Fmt {
  const uint32_t* __restrict__ rp;
  const uint32_t* __restrict__ col;
  const PT* __restrict__ pred;
  // label signature of every row: bit (l & 31) set iff the row holds an entry
  // with a label l' where (l' & 31) == (l & 31) — Eqs. 4/5's "row has label l"
  // for all labels at once (exact when P <= 32, a necessary condition beyond)
  const uint32_t* __restrict__ lmask;
};

__host__ __device__ __forceinline__ uint32_t label_bit(uint32_t l) { return 1u << (l & 31u); }

__device__ __forceinline__ uint32_t bit_of(const uint32_t* __restrict__ bm, uint32_t i) {
  return (__ldg(bm + (i >> 5)) >> (i & 31)) & 1u;
}

// [lo, hi) = entries of row r with label l (binary search on the sorted pred run).
template <typename PT>
__device__ __forceinline__ void label_range(const Fmt<PT>& f, uint32_t r, uint32_t l, uint32_t& lo,
                                            uint32_t& hi) {
  uint32_t a = __ldg(f.rp + r), e = __ldg(f.rp + r + 1), z = e;
  while (a < z) {
    uint32_t m = (a + z) >> 1;
    if ((uint32_t)__ldg(f.pred + m) < l) a = m + 1; else z = m;
  }
  lo = a; z = e;
  while (a < z) {
    uint32_t m = (a + z) >> 1;
    if ((uint32_t)__ldg(f.pred + m) <= l) a = m + 1; else z = m;
  }
  hi = a;
}

// First k in [lo, hi) with pred[k] >= key, by a warp: 33-way splits (one probe
// per lane + ballot) shrink the range 33x per round -> ~5 dependent loads for
// a 1e8-entry hub row instead of ~27.  All 32 lanes must call it.
template <typename PT>
__device__ __forceinline__ uint32_t warp_lower_bound(const PT* __restrict__ pred, uint32_t lo, uint32_t hi,
                                                     uint32_t key) {
  const uint32_t lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const uint64_t n = hi - lo;
    const uint32_t p = lo + (uint32_t)((n * (lane + 1)) / 33);
    const uint32_t below = __ballot_sync(GSM_FULL, (uint32_t)__ldg(pred + p) < key);
    const int cnt = __popc(below);
    const uint32_t nlo = cnt ? __shfl_sync(GSM_FULL, p, cnt - 1) + 1 : lo;
    const uint32_t nhi = cnt < 32 ? __shfl_sync(GSM_FULL, p, cnt & 31) : hi;
    lo = nlo;
    hi = nhi;
  }
  const uint32_t k = lo + lane;
  const uint32_t below = __ballot_sync(GSM_FULL, k < hi && (uint32_t)__ldg(pred + k) < key);
  return lo + __popc(below);
}

template <typename PT>
__device__ __forceinline__ void warp_label_range(const Fmt<PT>& f, uint32_t r, uint32_t l, uint32_t& lo,
                                                 uint32_t& hi) {
  const uint32_t b = __ldg(f.rp + r), e = __ldg(f.rp + r + 1);
  lo = warp_lower_bound(f.pred, b, e, l);
  hi = warp_lower_bound(f.pred, lo, e, l + 1);
}

// Is (r, l, target) an entry?  (membership of target in seg_l(r)).  A row's
// entries are sorted by (pred, col): one binary search on that pair (label and
// column loaded together per step, ~log2(len) dependent steps) instead of two
// label-bound searches followed by a column search.
template <typename PT>
__device__ __forceinline__ bool has_entry(const Fmt<PT>& f, uint32_t r, uint32_t l, uint32_t target) {
  uint32_t lo = __ldg(f.rp + r), hi = __ldg(f.rp + r + 1);
  while (lo < hi) {
    const uint32_t m = (lo + hi) >> 1;
    const uint32_t p = __ldg(f.pred + m), c = __ldg(f.col + m);
    if (p == l && c == target) return true;
    if (p < l || (p == l && c < target)) lo = m + 1; else hi = m;
  }
  return false;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Programmatic dependent launch (sm_90+): every query-path kernel is launched
// with programmatic stream serialization (pdl_launch), so the next kernel's CTAs
// are scheduled while this one drains.  Each kernel first waits for its
// predecessor grid to complete and flush (griddepcontrol.wait) - before ANY load
// or store, so no read-after-write or write-after-read hazard can cross it - then
// at once lets its own dependents launch (griddepcontrol.launch_dependents); they
// in turn wait for this grid's completion before touching memory.
#define GSM_PDL_ENTRY()                                        \
  do {                                                         \
    asm volatile("griddepcontrol.wait;" ::: "memory");         \
    asm volatile("griddepcontrol.launch_dependents;" :::);     \
  } while (0)

// ---- 1-D TMA bulk copies (cp.async.bulk, completion on a shared-memory
// mbarrier): global -> shared staging of contiguous tiles without register
// round trips.  src, dst and bytes must be 16-byte aligned / multiples.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, unsigned long long* m) {
  // generic-proxy accesses of dst before this point are ordered before the async write
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(m)),
      "r"(phase)
      : "memory");
}

// Block-wide exclusive scan of one value per thread (blockDim.x <= 1024, multiple of 32).
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* smem /* >= 32 */, T* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(GSM_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T w = lane < nw ? smem[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(GSM_FULL, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) smem[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  T warp_off = wid ? smem[wid - 1] : T(0);
  if (total) *total = smem[nw - 1];
  T r = warp_off + x - v;
  __syncthreads();
  return r;
}

template <typename T>
__device__ __forceinline__ T block_reduce_sum(T v, T* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(GSM_FULL, v, o);
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  T r = 0;
  if (wid == 0) {
    r = lane < nw ? smem[lane] : T(0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(GSM_FULL, r, o);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

}  // namespace gsm
