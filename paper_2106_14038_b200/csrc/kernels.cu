// sm_100a kernels of the gSmart hot path (§5-§8).
// Every kernel here is HBM/L2-bound integer/boolean work: no tensor cores
// (not a dense contraction — BASELINE.json north_star).
#include <cstdlib>
#include "kernels.h"

namespace gsm {

static inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 1u << 30) {
  uint64_t g = (n + block - 1) / block;
  if (g == 0) g = 1;
  return (unsigned)(g > cap ? cap : g);
}

// =====================================================================================
// Scans (reduce-then-scan; tile = 256 threads x 8 items)
// =====================================================================================
constexpr int SB = 256, SI = 8, ST = SB * SI;

__global__ void __launch_bounds__(SB) k_scan_reduce(const uint32_t* __restrict__ in, uint64_t n,
                                                   unsigned long long* __restrict__ partial) {
  __shared__ unsigned long long sm[32];
  uint64_t base = (uint64_t)blockIdx.x * ST + (uint64_t)threadIdx.x * SI;
  unsigned long long s = 0;
#pragma unroll
  for (int i = 0; i < SI; i++)
    if (base + i < n) s += in[base + i];
  s = block_reduce_sum<unsigned long long>(s, sm);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// single block: exclusive scan of np partials in place (carry loop), total -> *total
__global__ void __launch_bounds__(1024) k_scan_partials(unsigned long long* __restrict__ partial, uint64_t np,
                                                        unsigned long long* __restrict__ total) {
  __shared__ unsigned long long sm[32];
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t base = 0; base < np; base += blockDim.x) {
    uint64_t i = base + threadIdx.x;
    unsigned long long v = i < np ? partial[i] : 0ull, tot;
    unsigned long long ex = block_exclusive_scan<unsigned long long>(v, sm, &tot);
    if (i < np) partial[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(SB) k_scan_apply(const uint32_t* in, uint32_t* out, uint64_t n,
                                                  const unsigned long long* __restrict__ partial) {
  __shared__ unsigned long long sm[32];
  uint64_t base = (uint64_t)blockIdx.x * ST + (uint64_t)threadIdx.x * SI;
  uint32_t v[SI];
  unsigned long long s = 0;
#pragma unroll
  for (int i = 0; i < SI; i++) {
    v[i] = base + i < n ? in[base + i] : 0u;
    s += v[i];
  }
  unsigned long long ex = block_exclusive_scan<unsigned long long>(s, sm, nullptr) + partial[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SI; i++) {
    if (base + i < n) out[base + i] = (uint32_t)ex;
    ex += v[i];
  }
}

size_t scan_tmp_bytes(uint64_t n) {
  uint64_t np = (n + ST - 1) / ST;
  return (np + 1) * sizeof(unsigned long long) + 256;
}

cudaError_t scan_exclusive_u32(const uint32_t* in, uint32_t* out, uint64_t n, unsigned long long* total_dev,
                               void* tmp, cudaStream_t st, int* launches) {
  uint64_t np = (n + ST - 1) / ST;
  if (np == 0) np = 1;
  auto* partial = (unsigned long long*)tmp;
  k_scan_reduce<<<(unsigned)np, SB, 0, st>>>(in, n, partial);
  k_scan_partials<<<1, 1024, 0, st>>>(partial, np, total_dev);
  k_scan_apply<<<(unsigned)np, SB, 0, st>>>(in, out, n, partial);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

// =====================================================================================
// a1 — LSpM build (§6.2): key pack -> radix sort -> unique -> unpack + row counts
// key = row << sh_row | pred << sh_pred | col ; bit drop_bit set = filtered out
// =====================================================================================
// rows outside [rlo, rhi) (another rank's vertex range, world > 1) are dropped like
// filtered predicates
__global__ void k_pack_keys(const uint32_t* __restrict__ rowv, const uint32_t* __restrict__ p,
                            const uint32_t* __restrict__ colv, uint64_t n, const uint8_t* __restrict__ keep,
                            int sh_row, int sh_pred, int drop_bit, uint32_t rlo, uint32_t rhi,
                            uint64_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t r = __ldg(rowv + i), l = __ldg(p + i), c = __ldg(colv + i);
    uint64_t k = ((uint64_t)r << sh_row) | ((uint64_t)l << sh_pred) | (uint64_t)c;
    if (!__ldg(keep + l) || r < rlo || r >= rhi) k |= 1ull << drop_bit;
    keys[i] = k;
  }
}

cudaError_t launch_pack_keys(const uint32_t* rowv, const uint32_t* p, const uint32_t* colv, uint64_t n,
                             const uint8_t* keep, int sh_row, int sh_pred, int drop_bit, uint32_t rlo, uint32_t rhi,
                             uint64_t* keys, cudaStream_t st) {
  k_pack_keys<<<grid_for(n, 256, 148 * 32), 256, 0, st>>>(rowv, p, colv, n, keep, sh_row, sh_pred, drop_bit, rlo, rhi,
                                                          keys);
  return cudaGetLastError();
}

__global__ void k_pack_pso(const uint32_t* __restrict__ s, const uint32_t* __restrict__ p,
                           const uint32_t* __restrict__ o, uint64_t n, const uint8_t* __restrict__ keep, int nb,
                           int drop_bit, uint32_t rlo, uint32_t rhi, uint64_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t l = __ldg(p + i), a = __ldg(s + i);
    uint64_t k = ((uint64_t)l << (2 * nb)) | ((uint64_t)a << nb) | (uint64_t)__ldg(o + i);
    if (!__ldg(keep + l) || a < rlo || a >= rhi) k |= 1ull << drop_bit;
    keys[i] = k;
  }
}

cudaError_t launch_pack_pso(const uint32_t* s, const uint32_t* p, const uint32_t* o, uint64_t n, const uint8_t* keep,
                            int nb, int drop_bit, uint32_t rlo, uint32_t rhi, uint64_t* keys, cudaStream_t st) {
  k_pack_pso<<<grid_for(n, 256, 148 * 32), 256, 0, st>>>(s, p, o, n, keep, nb, drop_bit, rlo, rhi, keys);
  return cudaGetLastError();
}

// world > 1: out+in entries per 2^shift-vertex bucket (partition split points)
__global__ void k_bucket_degree(const uint32_t* __restrict__ s, const uint32_t* __restrict__ p,
                                const uint32_t* __restrict__ o, uint64_t n, const uint8_t* __restrict__ keep, int shift,
                                unsigned long long* __restrict__ hist) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (!__ldg(keep + __ldg(p + i))) continue;
    atomicAdd(hist + (__ldg(s + i) >> shift), 1ull);
    atomicAdd(hist + (__ldg(o + i) >> shift), 1ull);
  }
}

cudaError_t launch_bucket_degree(const uint32_t* s, const uint32_t* p, const uint32_t* o, uint64_t n,
                                 const uint8_t* keep, int shift, unsigned long long* hist, cudaStream_t st) {
  k_bucket_degree<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(s, p, o, n, keep, shift, hist);
  return cudaGetLastError();
}

// dst[i] = src[i] + add (row pointers of a rank's chunk -> global entry indices)
__global__ void k_add_copy(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, uint64_t n, uint32_t add) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i] + add;
}

cudaError_t launch_add_copy(uint32_t* dst, const uint32_t* src, uint64_t n, uint32_t add, cudaStream_t st) {
  if (!n) return cudaSuccess;
  k_add_copy<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(dst, src, n, add);
  return cudaGetLastError();
}

__global__ void k_unpack_pso(const uint64_t* __restrict__ keys, uint64_t n, const uint32_t* __restrict__ pos,
                             int drop_bit, int nb, uint32_t* __restrict__ ls, uint32_t* __restrict__ lo,
                             uint32_t* __restrict__ counts) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t m = (1ull << nb) - 1;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < n; base += stride) {
    const uint64_t i = base + threadIdx.x;
    bool valid = false;
    uint32_t l = 0xffffffffu;
    if (i < n) {
      const uint64_t k = keys[i];
      valid = !((k >> drop_bit) & 1ull) && (i == 0 || keys[i - 1] != k);
      if (valid) {
        const uint32_t q = pos[i];
        l = (uint32_t)(k >> (2 * nb));
        ls[q] = (uint32_t)((k >> nb) & m);
        lo[q] = (uint32_t)(k & m);
      }
    }
    const uint32_t peers = __match_any_sync(GSM_FULL, l);
    const uint32_t cnt = __popc(peers & __ballot_sync(GSM_FULL, valid));
    if (valid && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(counts + l, cnt);
  }
}

// the CSR's sorted keys (s, p, o) without duplicates / dropped labels, compacted
// (the label-major lists are then one stable pass on the label bits away)
// (compacted and re-laid out as (p, s, o) keys: p above bit 2 nb, so a stable
// pass on the label digit — whose window above the label holds zeros — sorts them)
__global__ void k_compact_keys(const uint64_t* __restrict__ keys, uint64_t n, const uint32_t* __restrict__ pos,
                               int drop_bit, int nb, int pb, uint64_t* __restrict__ out) {
  const uint64_t m = (1ull << nb) - 1, pm = (1ull << pb) - 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    if (!((k >> drop_bit) & 1ull) && (i == 0 || keys[i - 1] != k)) {
      const uint64_t srow = k >> (nb + pb), p = (k >> nb) & pm, o = k & m;
      out[pos[i]] = (p << (2 * nb)) | (srow << nb) | o;
    }
  }
}

cudaError_t launch_compact_keys(const uint64_t* keys, uint64_t n, const uint32_t* pos, int drop_bit, int nb, int pb,
                                uint64_t* out, cudaStream_t st) {
  k_compact_keys<<<grid_for(n, 256, 148 * 32), 256, 0, st>>>(keys, n, pos, drop_bit, nb, pb, out);
  return cudaGetLastError();
}

// label-major lists from (s, p, o) keys already stably sorted by p: ls/lo and
// entries per label (warp-aggregated counts)
// (csc_keys, optional: the same entries re-laid out as (o, p, s) keys — the
// object on top, so a stable pass on its digits sees zeros above it)
__global__ void k_unpack_spo_lm(const uint64_t* __restrict__ keys, uint64_t n, int nb, int pb,
                                uint32_t* __restrict__ ls, uint32_t* __restrict__ lo, uint32_t* __restrict__ counts,
                                uint64_t* __restrict__ csc_keys) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t m = (1ull << nb) - 1, pm = (1ull << pb) - 1;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < n; base += stride) {
    const uint64_t i = base + threadIdx.x;
    uint32_t l = 0xffffffffu;
    const bool valid = i < n;
    if (valid) {  // (p, s, o) layout
      const uint64_t k = keys[i];
      l = (uint32_t)((k >> (2 * nb)) & pm);
      const uint32_t sv = (uint32_t)((k >> nb) & m), ov = (uint32_t)(k & m);
      ls[i] = sv;
      lo[i] = ov;
      if (csc_keys) csc_keys[i] = ((uint64_t)ov << (nb + pb)) | ((uint64_t)l << nb) | sv;
    }
    const uint32_t peers = __match_any_sync(GSM_FULL, l);
    const uint32_t cnt = __popc(peers & __ballot_sync(GSM_FULL, valid));
    if (valid && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(counts + l, cnt);
  }
}

cudaError_t launch_unpack_spo_lm(const uint64_t* keys, uint64_t n, int nb, int pb, uint32_t* ls, uint32_t* lo,
                                 uint32_t* counts, cudaStream_t st, uint64_t* csc_keys) {
  k_unpack_spo_lm<<<grid_for(n, 256, 148 * 32), 256, 0, st>>>(keys, n, nb, pb, ls, lo, counts, csc_keys);
  return cudaGetLastError();
}

// CSC entries from (o, p, s)-layout keys in (o, p, s) order: row o, label p,
// column s; warp-aggregated row counts
template <typename PT>
__global__ void k_unpack_lm_csc(const uint64_t* __restrict__ keys, uint64_t n, int nb, int pb,
                                uint32_t* __restrict__ col, PT* __restrict__ pred, uint32_t* __restrict__ counts) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t m = (1ull << nb) - 1, pm = (1ull << pb) - 1;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < n; base += stride) {
    const uint64_t i = base + threadIdx.x;
    const bool valid = i < n;
    uint32_t row = 0xffffffffu;
    if (valid) {  // (o, p, s) layout
      const uint64_t k = keys[i];
      row = (uint32_t)(k >> (nb + pb));
      col[i] = (uint32_t)(k & m);
      pred[i] = (PT)((k >> nb) & pm);
    }
    const uint32_t peers = __match_any_sync(GSM_FULL, row);
    const uint32_t cnt = __popc(peers & __ballot_sync(GSM_FULL, valid));
    if (valid && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(counts + row, cnt);
  }
}

cudaError_t launch_unpack_lm_csc(const uint64_t* keys, uint64_t n, int nb, int pb, uint32_t* col, void* pred,
                                 int pred_bytes, uint32_t* counts, cudaStream_t st) {
  const unsigned g = grid_for(n, 256, 148 * 32);
  if (pred_bytes == 1) k_unpack_lm_csc<uint8_t><<<g, 256, 0, st>>>(keys, n, nb, pb, col, (uint8_t*)pred, counts);
  else k_unpack_lm_csc<uint16_t><<<g, 256, 0, st>>>(keys, n, nb, pb, col, (uint16_t*)pred, counts);
  return cudaGetLastError();
}

cudaError_t launch_unpack_pso(const uint64_t* keys, uint64_t n, const uint32_t* pos, int drop_bit, int nb,
                              uint32_t* ls, uint32_t* lo, uint32_t* counts, cudaStream_t st) {
  k_unpack_pso<<<grid_for(n, 256, 148 * 32), 256, 0, st>>>(keys, n, pos, drop_bit, nb, ls, lo, counts);
  return cudaGetLastError();
}

__global__ void k_unique_flags(const uint64_t* __restrict__ keys, uint64_t n, int drop_bit,
                               uint32_t* __restrict__ flags) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    bool keepk = !((k >> drop_bit) & 1ull) && (i == 0 || keys[i - 1] != k);
    flags[i] = keepk ? 1u : 0u;
  }
}

cudaError_t launch_unique_flags(const uint64_t* keys, uint64_t n, int drop_bit, uint32_t* flags, cudaStream_t st) {
  k_unique_flags<<<grid_for(n, 256, 148 * 32), 256, 0, st>>>(keys, n, drop_bit, flags);
  return cudaGetLastError();
}

template <typename PT>
__global__ void k_unpack(const uint64_t* __restrict__ keys, uint64_t n, const uint32_t* __restrict__ pos,
                         int drop_bit, int sh_row, int sh_pred, uint32_t* __restrict__ col, PT* __restrict__ pred,
                         uint32_t* __restrict__ counts) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t pmask = (1ull << (sh_row - sh_pred)) - 1, cmask = (1ull << sh_pred) - 1;
  // all lanes iterate the same number of times (warp-aggregated row counting)
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < n; base += stride) {
    uint64_t i = base + threadIdx.x;
    bool valid = false;
    uint32_t row = 0xffffffffu;
    if (i < n) {
      uint64_t k = keys[i];
      valid = !((k >> drop_bit) & 1ull) && (i == 0 || keys[i - 1] != k);
      if (valid) {
        uint32_t q = pos[i];
        row = (uint32_t)(k >> sh_row);
        col[q] = (uint32_t)(k & cmask);
        pred[q] = (PT)((k >> sh_pred) & pmask);
      }
    }
    uint32_t peers = __match_any_sync(GSM_FULL, row);
    uint32_t cnt = __popc(peers & __ballot_sync(GSM_FULL, valid));
    int leader = __ffs(peers) - 1;
    if (valid && (threadIdx.x & 31) == leader) atomicAdd(counts + row, cnt);
  }
}

cudaError_t launch_unpack(const uint64_t* keys, uint64_t n, const uint32_t* pos, int drop_bit, int sh_row,
                          int sh_pred, uint32_t* col, void* pred, int pred_bytes, uint32_t* counts,
                          cudaStream_t st) {
  unsigned g = grid_for(n, 256, 148 * 32);
  if (pred_bytes == 1)
    k_unpack<uint8_t><<<g, 256, 0, st>>>(keys, n, pos, drop_bit, sh_row, sh_pred, col, (uint8_t*)pred, counts);
  else
    k_unpack<uint16_t><<<g, 256, 0, st>>>(keys, n, pos, drop_bit, sh_row, sh_pred, col, (uint16_t*)pred, counts);
  return cudaGetLastError();
}

// ---- keys wider than 63 bits (e.g. 27 + 14 + 27 bits: 100M entities, 10,000
// labels): hi = row << pb | pred (drop flag at bit drop_hi), lo = col; sorted
// by lo then stably by hi (two LSD key groups, radix.cu)
// mode 0 (LSpM format): hi = a << sh | pred; mode 1 (label-major): hi = pred << sh | a; lo = b
__global__ void k_pack_keys2(const uint32_t* __restrict__ a, const uint32_t* __restrict__ p,
                             const uint32_t* __restrict__ b, uint64_t n, const uint8_t* __restrict__ keep, int mode,
                             int sh, int drop_hi, uint32_t rlo, uint32_t rhi, uint64_t* __restrict__ hi,
                             uint32_t* __restrict__ lo) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t l = __ldg(p + i);
    const uint32_t x32 = __ldg(a + i);
    const uint64_t x = x32;
    uint64_t h = mode == 0 ? ((x << sh) | (uint64_t)l) : (((uint64_t)l << sh) | x);
    if (!__ldg(keep + l) || x32 < rlo || x32 >= rhi) h |= 1ull << drop_hi;
    hi[i] = h;
    lo[i] = __ldg(b + i);
  }
}

cudaError_t launch_pack_keys2(const uint32_t* a, const uint32_t* p, const uint32_t* b, uint64_t n, const uint8_t* keep,
                              int mode, int sh, int drop_hi, uint32_t rlo, uint32_t rhi, uint64_t* hi, uint32_t* lo,
                              cudaStream_t st) {
  k_pack_keys2<<<grid_for(n, 256, 148 * 32), 256, 0, st>>>(a, p, b, n, keep, mode, sh, drop_hi, rlo, rhi, hi, lo);
  return cudaGetLastError();
}

__global__ void k_unique_flags2(const uint64_t* __restrict__ hi, const uint32_t* __restrict__ lo, uint64_t n,
                                int drop_hi, uint32_t* __restrict__ flags) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = hi[i];
    const uint32_t l = lo[i];
    flags[i] = (!((h >> drop_hi) & 1ull) && (i == 0 || hi[i - 1] != h || lo[i - 1] != l)) ? 1u : 0u;
  }
}

cudaError_t launch_unique_flags2(const uint64_t* hi, const uint32_t* lo, uint64_t n, int drop_hi, uint32_t* flags,
                                 cudaStream_t st) {
  k_unique_flags2<<<grid_for(n, 256, 148 * 32), 256, 0, st>>>(hi, lo, n, drop_hi, flags);
  return cudaGetLastError();
}

// unpack of the two-word keys: mode 0 = LSpM format (row = hi >> pb, pred = low
// pb bits of hi, col = lo; row counts), mode 1 = label-major (label = hi >> nb,
// s = low nb bits of hi, o = lo; label counts)
template <typename PT>
__global__ void k_unpack2(const uint64_t* __restrict__ hi, const uint32_t* __restrict__ lo, uint64_t n,
                          const uint32_t* __restrict__ pos, int drop_hi, int sh, int mode, uint32_t* __restrict__ a_out,
                          PT* __restrict__ pred, uint32_t* __restrict__ b_out, uint32_t* __restrict__ counts) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t lowmask = (1ull << sh) - 1;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < n; base += stride) {
    const uint64_t i = base + threadIdx.x;
    bool valid = false;
    uint32_t key = 0xffffffffu;
    if (i < n) {
      const uint64_t h = hi[i];
      const uint32_t l = lo[i];
      valid = !((h >> drop_hi) & 1ull) && (i == 0 || hi[i - 1] != h || lo[i - 1] != l);
      if (valid) {
        const uint32_t q = pos[i];
        const uint32_t top = (uint32_t)((h & ~(1ull << drop_hi)) >> sh), low = (uint32_t)(h & lowmask);
        if (mode == 0) {  // LSpM: col, pred; count rows
          a_out[q] = l;
          pred[q] = (PT)low;
        } else {          // label-major: s, o; count labels
          a_out[q] = low;
          b_out[q] = l;
        }
        key = top;
      }
    }
    const uint32_t peers = __match_any_sync(GSM_FULL, key);
    const uint32_t cnt = __popc(peers & __ballot_sync(GSM_FULL, valid));
    if (valid && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(counts + key, cnt);
  }
}

cudaError_t launch_unpack2(const uint64_t* hi, const uint32_t* lo, uint64_t n, const uint32_t* pos, int drop_hi, int sh,
                           int mode, uint32_t* a_out, void* pred, int pred_bytes, uint32_t* b_out, uint32_t* counts,
                           cudaStream_t st) {
  const unsigned g = grid_for(n, 256, 148 * 32);
  if (pred_bytes == 1)
    k_unpack2<uint8_t><<<g, 256, 0, st>>>(hi, lo, n, pos, drop_hi, sh, mode, a_out, (uint8_t*)pred, b_out, counts);
  else
    k_unpack2<uint16_t><<<g, 256, 0, st>>>(hi, lo, n, pos, drop_hi, sh, mode, a_out, (uint16_t*)pred, b_out, counts);
  return cudaGetLastError();
}

__global__ void k_heavy_stats(const uint32_t* __restrict__ rp, uint32_t n_rows, unsigned long long* out2) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
    uint32_t len = rp[r + 1] - rp[r];
    if (len > HEAVY_ROW) {
      atomicAdd(out2, 1ull);
      atomicAdd(out2 + 1, (unsigned long long)((len + HEAVY_CHUNK - 1) / HEAVY_CHUNK));
    }
  }
}

cudaError_t launch_heavy_stats(const uint32_t* rp, uint32_t n_rows, unsigned long long* out2, cudaStream_t st) {
  k_heavy_stats<<<grid_for(n_rows, 256, 148 * 16), 256, 0, st>>>(rp, n_rows, out2);
  return cudaGetLastError();
}

// One thread per row.  Entries are sorted by label, so a row's label set is
// walked label by label: short rows linearly, long rows by jumping to the
// first entry past the current label (binary search) — O(#labels · log len)
// even for hub rows.  Optionally samples, per label, the rows holding it and
// their entries (every 16th row; a per-CTA shared histogram flushed once;
// labels < LR_MAX): the fan-out statistics of the trie order.
constexpr uint32_t LR_MAX = 4096;

// Also (every row, exact): nonfunc bit l is set iff some row holds >= 2 entries
// with label l — a pattern with label l seen from this format's rows then has
// at most one child per parent (a "functional" level, expanded by k_expand_func).
template <typename PT>
__global__ void k_label_mask(const uint32_t* __restrict__ rp, const PT* __restrict__ pred, uint32_t n_rows,
                             uint32_t* __restrict__ lmask, unsigned long long* __restrict__ label_rows,
                             uint32_t n_labels, uint32_t* __restrict__ nonfunc) {
  extern __shared__ uint32_t s_lr[];
  const bool count = label_rows != nullptr;
  // non-functional bits gathered per CTA in shared memory (a global word per
  // label would be one L2 hot spot for every thread of the grid)
  uint32_t* s_nf = s_lr + (count ? 2 * n_labels : 0);
  const uint32_t nf_words = nonfunc ? (n_labels + 31) / 32 : 0;
  for (uint32_t i = threadIdx.x; i < nf_words; i += blockDim.x) s_nf[i] = 0;
  if (count) {  // [0, n_labels): rows holding the label, [n_labels, 2 n_labels): its entries
    for (uint32_t i = threadIdx.x; i < 2 * n_labels; i += blockDim.x) s_lr[i] = 0;
  }
  __syncthreads();
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
    uint32_t k = rp[r];
    const uint32_t e = rp[r + 1];
    uint32_t m = 0;
    while (k < e) {
      const uint32_t l = pred[k];
      const uint32_t k0 = k;
      m |= label_bit(l);
      if (e - k <= 16) {  // short remainder: step linearly past this label
        k++;
        while (k < e && (uint32_t)pred[k] == l) k++;
      } else {
        uint32_t lo = k + 1, hi = e;  // first entry with label > l
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if ((uint32_t)pred[mid] <= l) lo = mid + 1;
          else hi = mid;
        }
        k = lo;
      }
      if (nonfunc && k - k0 > 1 && l < n_labels && !((s_nf[l >> 5] >> (l & 31)) & 1u))
        atomicOr(s_nf + (l >> 5), 1u << (l & 31));
      if (count && (r & 15u) == 0 && l < n_labels) {  // a 1-in-16 row sample: the ratio is what matters
        atomicAdd(&s_lr[l], 1u);
        atomicAdd(&s_lr[n_labels + l], k - k0);
      }
    }
    lmask[r] = m;
  }
  __syncthreads();
  if (count)
    for (uint32_t i = threadIdx.x; i < 2 * n_labels; i += blockDim.x)
      if (s_lr[i]) atomicAdd(label_rows + i, (unsigned long long)s_lr[i]);
  for (uint32_t i = threadIdx.x; i < nf_words; i += blockDim.x)
    if (s_nf[i]) atomicOr(nonfunc + i, s_nf[i]);
}

cudaError_t launch_label_mask(const uint32_t* rp, const void* pred, int pred_bytes, uint32_t n_rows,
                              uint32_t* lmask, unsigned long long* label_rows, uint32_t n_labels, cudaStream_t st,
                              uint32_t* nonfunc) {
  const unsigned g = grid_for(n_rows, 256, 148 * 16);
  if (n_labels > LR_MAX) label_rows = nullptr;
  const size_t sm = (label_rows ? (size_t)n_labels * 8 : 0) + (nonfunc ? ((size_t)n_labels + 31) / 32 * 4 : 0);
  if (pred_bytes == 1)
    k_label_mask<uint8_t><<<g, 256, sm, st>>>(rp, (const uint8_t*)pred, n_rows, lmask, label_rows, n_labels, nonfunc);
  else
    k_label_mask<uint16_t><<<g, 256, sm, st>>>(rp, (const uint16_t*)pred, n_rows, lmask, label_rows, n_labels, nonfunc);
  return cudaGetLastError();
}

// =====================================================================================
// bitmaps
// =====================================================================================
// all-ones over bits [0, n_bits), zero beyond (padding words included)
__global__ void k_fill_ones(uint32_t* bm, uint32_t n_words, uint32_t n_bits) {
  GSM_PDL_ENTRY();
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < n_words; w += gridDim.x * blockDim.x) {
    uint64_t lo = (uint64_t)w * 32;
    uint32_t v;
    if (lo >= n_bits) v = 0u;
    else if (lo + 32 <= n_bits) v = 0xffffffffu;
    else v = (1u << (n_bits - lo)) - 1u;
    bm[w] = v;
  }
}

// every variable's candidate bitmap in one launch: slot s is all-ones over
// [0, n_bits) if bit s of ones_mask is set (no seed), else zero (seeded)
__global__ void k_init_cands(uint32_t* cand, uint32_t n_slots, uint32_t stride, uint32_t n_bits, uint32_t ones_mask,
                             InitExtra x) {
  GSM_PDL_ENTRY();
  // first kernel of an execute: publish the look-back epoch base the host wrote to
  // pinned memory (a replayed graph thus needs no extra launch to set it) and zero
  // the execute's counters and size words (no memset nodes)
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0 && x.d_epoch) *x.d_epoch = *x.h_epoch;
    if (threadIdx.x == 0 && x.d_bar) *x.d_bar = *x.h_bar;
    if (threadIdx.x == 0 && x.ovf) *x.ovf = 0;
    for (uint32_t i = threadIdx.x; i < x.n_zero; i += blockDim.x) x.zero[i] = 0;
    for (uint32_t i = threadIdx.x; i < x.n_zero2; i += blockDim.x) x.zero2[i] = 0;
    for (uint32_t i = threadIdx.x; i < x.n_zero32; i += blockDim.x) x.zero32[i] = 0;
  }
  const uint64_t total = (uint64_t)n_slots * stride;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(i / stride), w = (uint32_t)(i - (uint64_t)s * stride);
    uint32_t v = 0;
    if ((ones_mask >> s) & 1u) {
      const uint64_t lo = (uint64_t)w * 32;
      v = lo >= n_bits ? 0u : (lo + 32 <= n_bits ? 0xffffffffu : ((1u << (n_bits - lo)) - 1u));
    }
    cand[i] = v;
  }
}

cudaError_t launch_init_cands(uint32_t* cand, uint32_t n_slots, uint32_t stride_words, uint32_t n_bits,
                              uint32_t ones_mask, const InitExtra& x, cudaStream_t st) {
  pdl_launch(k_init_cands, grid_for((uint64_t)n_slots * stride_words, 256, 148 * 16), 256, st,
      cand, n_slots, stride_words, n_bits, ones_mask, x);
  return cudaGetLastError();
}

cudaError_t launch_fill_ones(uint32_t* bm, uint32_t n_words, uint32_t n_bits, cudaStream_t st) {
  pdl_launch(k_fill_ones, grid_for(n_words, 256, 148 * 16), 256, st, bm, n_words, n_bits);
  return cudaGetLastError();
}

__global__ void k_and_inplace(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, uint32_t n_words) {
  GSM_PDL_ENTRY();
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < n_words; w += gridDim.x * blockDim.x)
    dst[w] &= __ldg(src + w);
}

cudaError_t launch_and_inplace(uint32_t* dst, const uint32_t* src, uint32_t n_words, cudaStream_t st) {
  pdl_launch(k_and_inplace, grid_for(n_words, 256, 148 * 16), 256, st, dst, src, n_words);
  return cudaGetLastError();
}

__global__ void k_zero_if_flag(uint32_t* bm, uint64_t n_words, const int* flag) {
  GSM_PDL_ENTRY();
  if (*flag) return;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < n_words; w += (uint64_t)gridDim.x * blockDim.x)
    bm[w] = 0;
}

cudaError_t launch_zero_if_flag(uint32_t* bm, uint64_t n_words, const int* flag, cudaStream_t st) {
  pdl_launch(k_zero_if_flag, grid_for(n_words, 256, 148 * 16), 256, st, bm, n_words, flag);
  return cudaGetLastError();
}

// =====================================================================================
// a3 — constant seeding ("light" edges): bits |= {col : (c, l, col)}
// =====================================================================================
template <typename PT>
__global__ void k_seed_scatter(SeedBatch sb, unsigned long long* ctr) {
  GSM_PDL_ENTRY();
  // blockIdx.y = seed; every warp finds the label range itself (warp-cooperative
  // search, no CTA barrier)
  const uint32_t si = blockIdx.y;
  uint32_t dir = 0, c = 0, l = 0;
  uint32_t* bits = nullptr;
#pragma unroll
  for (uint32_t i = 0; i < MAX_SEEDS; i++)  // constant offsets into the parameter block
    if (i == si) {
      dir = sb.dir[i];
      c = sb.c[i];
      l = sb.label[i];
      bits = sb.bits[i];
    }
  const Fmt<PT> f = fmt_of<PT>(dir ? sb.f[1] : sb.f[0]);
  uint32_t lo, hi;
  warp_label_range(f, c, l, lo, hi);
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(ctr + C_SEED, (unsigned long long)(hi - lo));
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  __shared__ uint32_t s_words[8][32];  // per-warp window of 32 bitmap words
  // A warp takes SEED_R rounds of 128 consecutive (sorted) entries, rounds strided by
  // the grid (small ranges still spread over all warps), all loads issued before
  // any is used (SEED_R x 512 B in flight per warp); in a round lane i holds
  // entries 4i..4i+3.  If a round spans < 32 words, its bits are OR-ed into a shared
  // window and written with one atomicOr per non-zero word; else per-entry
  // warp-aggregated atomics.
  constexpr int SEED_R = 4;
  const uint64_t stride = (uint64_t)nwarps * 128;
  for (uint64_t base0 = lo + (uint64_t)warp * 128; base0 < hi; base0 += stride * SEED_R) {
    uint32_t id[SEED_R][4];
#pragma unroll
    for (int r = 0; r < SEED_R; r++)
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const uint64_t k = base0 + r * stride + lane * 4 + j;
        id[r][j] = k < hi ? __ldg(f.col + k) : 0u;
      }
#pragma unroll
    for (int r = 0; r < SEED_R; r++) {
      const uint64_t base64 = base0 + r * stride;
      if (base64 >= hi) break;
      const uint32_t base = (uint32_t)base64;
      bool v[4];
#pragma unroll
      for (int j = 0; j < 4; j++) v[j] = base + lane * 4 + j < hi;
      const uint32_t w_first = __shfl_sync(GSM_FULL, id[r][0], 0) >> 5;
      const uint32_t last_k = min(hi, base + 128) - 1 - base;
      uint32_t idl = id[r][0];
#pragma unroll
      for (int j = 1; j < 4; j++)
        if ((last_k & 3) == (uint32_t)j) idl = id[r][j];
      const uint32_t w_last = __shfl_sync(GSM_FULL, idl, last_k >> 2) >> 5;
      if (w_last - w_first < 32) {
        s_words[wib][lane] = 0;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; j++)
          if (v[j]) atomicOr(&s_words[wib][(id[r][j] >> 5) - w_first], 1u << (id[r][j] & 31));
        __syncwarp();
        const uint32_t x = s_words[wib][lane];
        if (x) atomicOr(bits + w_first + lane, x);
        __syncwarp();
      } else {
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint32_t word = v[j] ? (id[r][j] >> 5) : 0xffffffffu;
          const uint32_t peers = __match_any_sync(GSM_FULL, word);
          const uint32_t orv = __reduce_or_sync(peers, v[j] ? (1u << (id[r][j] & 31)) : 0u);
          if (v[j] && (int)lane == __ffs(peers) - 1) atomicOr(bits + word, orv);
        }
      }
    }
  }
}

cudaError_t launch_seed_scatter(const SeedBatch& sb, int pred_bytes, unsigned long long* ctr, int sm_count,
                                cudaStream_t st) {
  if (sb.n == 0) return cudaSuccess;
  const dim3 g((unsigned)sm_count * 4, sb.n);
  if (pred_bytes == 1) pdl_launch(k_seed_scatter<uint8_t>, g, 256, st, sb, ctr);
  else pdl_launch(k_seed_scatter<uint16_t>, g, 256, st, sb, ctr);
  return cudaGetLastError();
}

template <typename PT>
__global__ void k_guard(Fmt<PT> f, uint32_t s, uint32_t l, uint32_t o, int* flag) {
  GSM_PDL_ENTRY();
  if (!has_entry(f, s, l, o)) *flag = 0;
}

cudaError_t launch_guard(FmtAny f, int pred_bytes, uint32_t s, uint32_t label, uint32_t o, int* flag,
                         cudaStream_t st) {
  if (pred_bytes == 1) pdl_launch(k_guard<uint8_t>, 1, 1, st, fmt_of<uint8_t>(f), s, label, o, flag);
  else pdl_launch(k_guard<uint16_t>, 1, 1, st, fmt_of<uint16_t>(f), s, label, o, flag);
  return cudaGetLastError();
}

// =====================================================================================
// a4 — grouped incident-edge evaluation (§5, Eqs. 17/21): for every candidate row i
// of the center x and every group edge e = (l, dir, w):
//   y_e(i) = OR_{j in seg^dir_l(i)} cand_w(j)      (self-loop: j == i)
//   cand_x(i) <- cand_x(i) AND (AND_e y_e(i))
// One warp owns one 32-bit bitmap word (32 consecutive rows) in each direction:
//  - rows <= SHORT_ROW entries: each lane scans its own row (entries sorted by
//    (pred, col): stop once every edge is satisfied or labels pass the max);
//  - longer rows: the whole warp scans the row with coalesced 32-entry strides;
//  - rows > HEAVY_ROW: deferred to chunked CTAs (k_filter_heavy) + finalize.
// =====================================================================================
template <typename PT>
struct FilterArgsT {
  Fmt<PT> f[2];
  GEdge e[2][MAXG];
  uint32_t ne[2];
  uint32_t minl[2], maxl[2];
  uint32_t needm[2];  // OR of label_bit() over the direction's edges
  uint32_t* cand;
  uint32_t n_words;
  uint32_t* heavy_rows;
  uint32_t* heavy_chunks;
  uint32_t* heavy_sat;
  uint32_t* heavy_count;
  unsigned long long* ctr;
  int variant;
  uint32_t word_lo;
  LBArgs claim;
  SkipIf skip;
  uint32_t center_slot, seq;
  uint32_t world;
  SymDelta peers;
};

// world > 1 (peer exchange): a bit cleared / a change word raised on this rank is
// applied to every rank's copy of the symmetric buffer (NVLink atomics)
__device__ __forceinline__ uint32_t and_all_ranks(uint32_t* p, uint32_t mask, uint32_t world, const SymDelta& d) {
  const uint32_t old = atomicAnd(p, mask);
  for (uint32_t q = 0; q < world; q++)
    if (d.words[q]) atomicAnd(p + d.words[q], mask);
  return old;
}

__device__ __forceinline__ void max_all_ranks(uint32_t* p, uint32_t v, uint32_t world, const SymDelta& d) {
  atomicMax(p, v);
  for (uint32_t q = 0; q < world; q++)
    if (d.words[q]) atomicMax(p + d.words[q], v);
}

template <typename PT>
__device__ __forceinline__ uint32_t match_entry(const FilterArgsT<PT>& a, int d, uint32_t l, uint32_t c,
                                                uint32_t row, uint32_t sat, uint32_t& matched) {
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < MAXG; j++) {
    if (j >= (int)a.ne[d]) break;
    if (l == a.e[d][j].label && !((sat >> j) & 1u)) {
      matched++;
      const uint32_t mode = a.e[d][j].mode;
      bool ok = mode == GE_PROBE ? (bit_of(a.e[d][j].nbr, c) != 0) : (c == (mode == GE_SELF ? row : a.e[d][j].cval));
      if (ok) s |= 1u << j;
    }
  }
  return s;
}

// Short row (<= SHORT_ROW entries) with uint8 labels: the row's labels are read
// with <= 3 aligned 16-byte loads; each edge's label range [lo, hi) inside the
// row follows from SIMD byte compares (__vcmpltu4 / __vcmpeq4 + popc), then only
// the cols of that range are loaded and probed.  4 dependent load levels per row.
template <typename PT>
__device__ __forceinline__ uint32_t short_row_u8(const FilterArgsT<PT>& a, const int d, const uint32_t row,
                                                 const uint32_t b, const uint32_t e, const uint32_t need,
                                                 unsigned long long& n_scanned, uint32_t& n_matched) {
  const uint8_t* P = reinterpret_cast<const uint8_t*>(a.f[d].pred);
  const uint32_t a0 = b & ~15u;
  uint32_t w[12];
  const uint4 v0 = __ldg(reinterpret_cast<const uint4*>(P + a0));
  const uint4 v1 = a0 + 16 < e ? __ldg(reinterpret_cast<const uint4*>(P + a0 + 16)) : make_uint4(0, 0, 0, 0);
  const uint4 v2 = a0 + 32 < e ? __ldg(reinterpret_cast<const uint4*>(P + a0 + 32)) : make_uint4(0, 0, 0, 0);
  w[0] = v0.x; w[1] = v0.y; w[2] = v0.z; w[3] = v0.w;
  w[4] = v1.x; w[5] = v1.y; w[6] = v1.z; w[7] = v1.w;
  w[8] = v2.x; w[9] = v2.y; w[10] = v2.z; w[11] = v2.w;
  uint32_t vm[12];  // byte masks of positions inside [b, e)
#pragma unroll
  for (int i = 0; i < 12; i++) {
    const int p0 = (int)(a0 + 4 * i);
    const int lo = min(max((int)b - p0, 0), 4), hi = min(max((int)e - p0, 0), 4);
    const uint32_t mhi = hi >= 4 ? 0xffffffffu : ((1u << (8 * hi)) - 1u);
    const uint32_t mlo = lo >= 4 ? 0xffffffffu : ((1u << (8 * lo)) - 1u);
    vm[i] = mhi & ~mlo;
  }
  n_scanned += e - b;
  uint32_t sat = 0;
#pragma unroll
  for (int j = 0; j < MAXG; j++) {
    if (j >= (int)a.ne[d]) break;
    const uint32_t L = a.e[d][j].label * 0x01010101u;
    uint32_t lt = 0, eq = 0;
#pragma unroll
    for (int i = 0; i < 12; i++) {
      lt += __popc(__vcmpltu4(w[i], L) & vm[i]);
      eq += __popc(__vcmpeq4(w[i], L) & vm[i]);
    }
    uint32_t k = b + (lt >> 3);
    const uint32_t kend = k + (eq >> 3);
    const uint32_t mode = a.e[d][j].mode;
    for (; k < kend; k++) {
      const uint32_t c = __ldg(a.f[d].col + k);
      n_matched++;
      const bool ok = mode == GE_PROBE ? (bit_of(a.e[d][j].nbr, c) != 0) : (c == (mode == GE_SELF ? row : a.e[d][j].cval));
      if (ok) {
        sat |= 1u << j;
        break;
      }
    }
  }
  (void)need;
  return sat;
}

// Evaluate the group's edges of one direction set for 32 candidate rows, one per
// lane (lanes with has == false idle).  Returns per-lane "all edges satisfied".
// Label pre-test (Eqs. 4/5 over the row label signatures): a row lacking one of
// the group's labels fails without touching row_ptr, labels or columns.
template <typename PT>
__device__ __forceinline__ bool label_pretest(const FilterArgsT<PT>& a, const uint32_t row, uint32_t& n_masked) {
  uint32_t m[2] = {~0u, ~0u};
#pragma unroll
  for (int d = 0; d < 2; d++)
    if (a.ne[d] && a.f[d].lmask) {
      m[d] = __ldg(a.f[d].lmask + row);
      n_masked++;
    }
  bool ok = true;
#pragma unroll
  for (int d = 0; d < 2; d++) ok = ok && (m[d] & a.needm[d]) == a.needm[d];
  return ok;
}

// PRE: the caller already ran label_pretest (has == passed)
template <typename PT, bool SIMD, bool PRE = false>
__device__ __forceinline__ bool eval_rows(const FilterArgsT<PT>& a, const uint32_t row, const bool has,
                                          const uint32_t lane, unsigned long long& n_rows,
                                          unsigned long long& n_scanned, uint32_t& n_matched,
                                          uint32_t& n_masked) {
  bool ok = has;
  if constexpr (!PRE) {
    if (ok) ok = label_pretest(a, row, n_masked);
  }
#pragma unroll
  for (int d = 0; d < 2; d++) {
    if (a.ne[d] == 0) continue;
    const uint32_t need = (a.ne[d] >= 32) ? 0xffffffffu : ((1u << a.ne[d]) - 1u);
    uint32_t b = 0, e = 0, sat = 0;
    bool medium = false;
    if (ok) {
      b = __ldg(a.f[d].rp + row);
      e = __ldg(a.f[d].rp + row + 1);
      n_rows++;
      const uint32_t len = e - b;
      if (len > HEAVY_ROW) {
        // defer: provisional keep; chunks OR their satisfied edges into heavy_sat[slot]
        const uint32_t slot = atomicAdd(a.heavy_count, 1u);
        const uint32_t nch = (len + HEAVY_CHUNK - 1) / HEAVY_CHUNK;
        const uint32_t c0 = atomicAdd(a.heavy_count + 1, nch);
        a.heavy_rows[slot] = row | ((uint32_t)d << 31);
        for (uint32_t c = 0; c < nch; c++) {
          a.heavy_chunks[2 * (c0 + c)] = slot;
          a.heavy_chunks[2 * (c0 + c) + 1] = c;
        }
        sat = need;
      } else if (len > SHORT_ROW) {
        // medium row, lane-private: per group label, a binary search for its first
        // entry, then its range probed 4 entries per step until a probe hits; all
        // 32 lanes search in parallel (latency overlapped across rows).  A label
        // range longer than MED_SCAN without a hit goes to the warp-cooperative
        // scan below (rare: long runs of non-candidate neighbours).
        for (int j = 0; j < MAXG; j++) {
          if (j >= (int)a.ne[d]) break;
          if ((sat >> j) & 1u) continue;
          const uint32_t lab = a.e[d][j].label;
          uint32_t lo = b, hi = e;
          while (lo < hi) {
            const uint32_t m = (lo + hi) >> 1;
            if ((uint32_t)__ldg(a.f[d].pred + m) < lab) lo = m + 1; else hi = m;
          }
          const uint32_t kcap = min(e, lo + MED_SCAN);
          const uint32_t mode = a.e[d][j].mode;
          bool hit = false, done = false;  // done: the label's range ended inside the window
          for (uint32_t k = lo; k < kcap && !hit && !done; k += 4) {
            uint32_t l4[4], c4[4];
#pragma unroll
            for (int t = 0; t < 4; t++) l4[t] = k + t < kcap ? (uint32_t)__ldg(a.f[d].pred + k + t) : lab;
#pragma unroll
            for (int t = 0; t < 4; t++) c4[t] = (k + t < kcap && l4[t] == lab) ? __ldg(a.f[d].col + k + t) : 0u;
#pragma unroll
            for (int t = 0; t < 4; t++) {
              if (hit || done || k + t >= kcap) break;
              if (l4[t] != lab) { done = true; break; }
              n_scanned++;
              n_matched++;
              hit = mode == GE_PROBE ? (bit_of(a.e[d][j].nbr, c4[t]) != 0)
                                     : (c4[t] == (mode == GE_SELF ? row : a.e[d][j].cval));
            }
          }
          if (hit) sat |= 1u << j;
          else if (!done && kcap < e && (uint32_t)__ldg(a.f[d].pred + kcap) == lab) medium = true;  // range goes on
          else break;  // this label has no satisfying entry: the row fails
        }
      } else if constexpr (SIMD) {
        sat = short_row_u8(a, d, row, b, e, need, n_scanned, n_matched);
      } else {
        // 4 entries per step: their pred loads, then col loads, then bitmap probes
        // are issued together (3 dependent load levels per 4 entries, not 12)
        for (uint32_t k = b; k < e && sat != need; k += 4) {
          uint32_t l[4], c[4];
#pragma unroll
          for (int j = 0; j < 4; j++) l[j] = k + j < e ? (uint32_t)__ldg(a.f[d].pred + k + j) : 0xffffffffu;
#pragma unroll
          for (int j = 0; j < 4; j++)
            c[j] = (l[j] >= a.minl[d] && l[j] <= a.maxl[d]) ? __ldg(a.f[d].col + k + j) : 0u;
          bool past = false;
#pragma unroll
          for (int j = 0; j < 4; j++) {
            if (l[j] == 0xffffffffu) break;
            n_scanned++;
            if (l[j] > a.maxl[d]) { past = true; break; }
            if (l[j] >= a.minl[d]) sat |= match_entry(a, d, l[j], c[j], row, sat, n_matched);
          }
          if (past) break;
        }
      }
    }
    // warp-cooperative scan of medium rows, one row at a time
    uint32_t mm = __ballot_sync(GSM_FULL, medium);
    while (mm) {
      const int src = __ffs(mm) - 1;
      mm &= mm - 1;
      const uint32_t rb0 = __shfl_sync(GSM_FULL, b, src), re0 = __shfl_sync(GSM_FULL, e, src);
      const uint32_t rrow = __shfl_sync(GSM_FULL, row, src);
      // only the entries whose labels lie in [minl, maxl] (rows are sorted by label)
      const uint32_t rb = warp_lower_bound(a.f[d].pred, rb0, re0, a.minl[d]);
      const uint32_t re = warp_lower_bound(a.f[d].pred, rb, re0, a.maxl[d] + 1);
      uint32_t wsat = 0;
      for (uint32_t base = rb; base < re; base += 32) {
        const uint32_t k = base + lane;
        uint32_t s = 0;
        if (k < re) {
          const uint32_t l = __ldg(a.f[d].pred + k);
          n_scanned++;
          if (l >= a.minl[d] && l <= a.maxl[d]) s = match_entry(a, d, l, __ldg(a.f[d].col + k), rrow, wsat, n_matched);
        }
        wsat |= __reduce_or_sync(GSM_FULL, s);
        if (wsat == need) break;
      }
      if ((int)lane == src) sat = wsat;
    }
    ok = ok && (sat == need);
  }
  return ok;
}

// clear the candidate bits of failed rows (one atomicAnd per distinct word per
// warp, on every rank's copy when world > 1); `changed` notes whether a bit
// actually went from 1 to 0
template <typename PT>
__device__ __forceinline__ void clear_failed(const FilterArgsT<PT>& a, const uint32_t row, const bool fail,
                                             const uint32_t lane, bool& changed) {
  const uint32_t word = fail ? (row >> 5) : 0xffffffffu;
  const uint32_t peers = __match_any_sync(GSM_FULL, word);
  const uint32_t bits = __reduce_or_sync(peers, fail ? (1u << (row & 31)) : 0u);
  if (fail && (int)lane == __ffs(peers) - 1)
    changed |= (and_all_ranks(a.cand + word, ~bits, a.world, a.peers) & bits) != 0;
}

// end of a filter launch: publish "the center's bitmap changed at this sequence"
template <typename PT>
__device__ __forceinline__ void note_change(const FilterArgsT<PT>& a, const bool changed) {
  if (__any_sync(GSM_FULL, changed) && (threadIdx.x & 31) == 0 && a.skip.chg)
    max_all_ranks(a.skip.chg + a.center_slot, a.seq, a.world, a.peers);
}

template <typename PT, bool SIMD>
__global__ void __launch_bounds__(256) k_group_filter(FilterArgsT<PT> a) {
  GSM_PDL_ENTRY();
  if (a.skip.skip()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(a.ctr + C_FILTER_SKIPPED, 1ull);
    return;
  }
  bool changed = false;
  constexpr uint32_t QCAP = 64;
  __shared__ uint32_t s_q[8][QCAP];  // per-warp queue of candidate rows (< 64)
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t* q = s_q[wib];
  unsigned long long n_rows = 0, n_scanned = 0;
  uint32_t n_matched = 0, n_masked = 0;
  // A warp streams chunks of 32 bitmap words (1024 rows; one coalesced load,
  // next chunk prefetched), queues the candidate rows (set bits, ascending) and
  // evaluates them 32 at a time, one row per lane: sparse candidate sets keep
  // every lane busy and all rows of a batch have their loads in flight together.
  const uint32_t n_chunks = (a.n_words + 31) >> 5;
  uint32_t qn = 0;  // warp-uniform queue length
  const bool dyn = (a.variant & 2) != 0;
  const uint32_t c_begin = a.word_lo >> 5;  // partitioned: this rank's first chunk
  uint32_t ch = c_begin + warp;
  if (dyn) {
    uint32_t c0 = 0;
    if (lane == 0) c0 = atomicAdd(a.claim.counter(), 1u);
    ch = c_begin + __shfl_sync(GSM_FULL, c0, 0);
  }
  uint32_t nxt = 0;
  if (ch < n_chunks) {
    const uint32_t wl = (ch << 5) + lane;
    nxt = wl < a.n_words ? __ldcg(a.cand + wl) : 0u;
  }
  while (ch < n_chunks) {
    const uint32_t mine = nxt;
    uint32_t cn = ch + nwarps;
    if (dyn) {
      uint32_t c0 = 0;
      if (lane == 0) c0 = atomicAdd(a.claim.counter(), 1u);
      cn = c_begin + __shfl_sync(GSM_FULL, c0, 0);
    }
    if (cn < n_chunks) {
      const uint32_t wn = (cn << 5) + lane;
      nxt = wn < a.n_words ? __ldcg(a.cand + wn) : 0u;
    }
    const uint32_t chc = ch;
    ch = cn;
    uint32_t nz = __ballot_sync(GSM_FULL, mine != 0);
    while (nz) {  // enqueue word by word (queue holds < 64 rows), evaluate 32 at a time
      const int j = __ffs(nz) - 1;
      nz &= nz - 1;
      const uint32_t wj = __shfl_sync(GSM_FULL, mine, j);
      if ((wj >> lane) & 1u) q[qn + __popc(wj & lanemask_lt())] = (((chc << 5) + j) << 5) + lane;
      qn += __popc(wj);
      __syncwarp();
      if (qn >= 32) {
        const uint32_t row = q[lane];
        const uint32_t extra = lane + 32 < qn ? q[lane + 32] : 0u;
        __syncwarp();
        if (lane + 32 < qn) q[lane] = extra;
        qn -= 32;
        __syncwarp();
        const bool ok = eval_rows<PT, SIMD>(a, row, true, lane, n_rows, n_scanned, n_matched, n_masked);
        clear_failed(a, row, !ok, lane, changed);
      }
    }
  }
  if (qn) {
    const bool has = lane < qn;
    const uint32_t row = has ? q[lane] : 0u;
    const bool ok = eval_rows<PT, SIMD>(a, row, has, lane, n_rows, n_scanned, n_matched, n_masked);
    clear_failed(a, row, has && !ok, lane, changed);
  }
  // one atomic per warp per counter
  note_change(a, changed);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    n_rows += __shfl_down_sync(GSM_FULL, n_rows, o);
    n_scanned += __shfl_down_sync(GSM_FULL, n_scanned, o);
    n_matched += __shfl_down_sync(GSM_FULL, n_matched, o);
    n_masked += __shfl_down_sync(GSM_FULL, n_masked, o);
  }
  if (lane == 0) {
    if (n_masked) atomicAdd(a.ctr + C_FILTER_MASKED, (unsigned long long)n_masked);
    if (n_rows) atomicAdd(a.ctr + C_FILTER_ROWS, n_rows);
    if (n_scanned) atomicAdd(a.ctr + C_FILTER_SCANNED, n_scanned);
    if (n_matched) atomicAdd(a.ctr + C_FILTER_MATCHED, (unsigned long long)n_matched);
  }
}

// Candidate rows given as a compacted id list (k_bitmap_compact_lb): every warp
// takes batches of 32 consecutive ids, one row per lane, so dense and sparse
// candidate sets alike spread over all warps of the GPU (no per-chunk serial
// batches), then failed rows are cleared in the center's bitmap.
template <typename PT, bool SIMD>
__global__ void __launch_bounds__(256, SIMD ? 4 : 6) k_group_filter_rows(FilterArgsT<PT> a, const uint32_t* __restrict__ rows,
                                                          const unsigned long long* __restrict__ d_nrows) {
  GSM_PDL_ENTRY();
  if (a.skip.skip()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(a.ctr + C_FILTER_SKIPPED, 1ull);
    return;
  }
  bool changed = false;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint64_t n = *d_nrows;
  unsigned long long n_rows = 0, n_scanned = 0;
  uint32_t n_matched = 0, n_masked = 0;
  // A warp takes RB batches of 32 rows at once when there are enough rows to
  // keep every warp busy: the RB row ids, then their label signatures, are
  // loaded together (RB-fold memory-level parallelism for the pre-test, which
  // decides most rows of the big groups), then the surviving rows are evaluated
  // batch by batch.
  constexpr int RB = 4;
  const uint32_t rb = n >= (uint64_t)nwarps * 32 * RB ? RB : 1;
  for (uint64_t base = (uint64_t)warp * 32 * rb; base < n; base += (uint64_t)nwarps * 32 * rb) {
    uint32_t row[RB], pass = 0, hasm = 0;
#pragma unroll
    for (int j = 0; j < RB; j++) {
      const uint64_t i = base + (uint64_t)j * 32 + lane;
      const bool has = (uint32_t)j < rb && i < n;
      row[j] = has ? __ldg(rows + i) : 0u;
      hasm |= (uint32_t)has << j;
    }
#pragma unroll
    for (int j = 0; j < RB; j++)
      if ((hasm >> j) & 1u) pass |= (uint32_t)label_pretest(a, row[j], n_masked) << j;
#pragma unroll 1
    for (uint32_t j = 0; j < rb; j++) {
      uint32_t r = row[0];
#pragma unroll
      for (int t = 1; t < RB; t++)
        if (j == (uint32_t)t) r = row[t];
      const bool has = (hasm >> j) & 1u;
      const bool ok = eval_rows<PT, SIMD, true>(a, r, (pass >> j) & 1u, lane, n_rows, n_scanned, n_matched, n_masked);
      clear_failed(a, r, has && !ok, lane, changed);
    }
  }
  note_change(a, changed);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    n_rows += __shfl_down_sync(GSM_FULL, n_rows, o);
    n_scanned += __shfl_down_sync(GSM_FULL, n_scanned, o);
    n_matched += __shfl_down_sync(GSM_FULL, n_matched, o);
    n_masked += __shfl_down_sync(GSM_FULL, n_masked, o);
  }
  if (lane == 0) {
    if (n_masked) atomicAdd(a.ctr + C_FILTER_MASKED, (unsigned long long)n_masked);
    if (n_rows) atomicAdd(a.ctr + C_FILTER_ROWS, n_rows);
    if (n_scanned) atomicAdd(a.ctr + C_FILTER_SCANNED, n_scanned);
    if (n_matched) atomicAdd(a.ctr + C_FILTER_MATCHED, (unsigned long long)n_matched);
  }
}

// heavy-row chunks: CTA per chunk, OR of satisfied edge bits into heavy_sat[slot].
// A chunk is skipped once the row's edges are all satisfied (by other chunks); a
// chunk scans only the entries inside the direction's label window (two warp
// searches), 4 independent entries per thread per step, and stops as soon as
// every edge is satisfied.
template <typename PT>
__global__ void __launch_bounds__(256) k_filter_heavy(FilterArgsT<PT> a) {
  GSM_PDL_ENTRY();
  __shared__ uint32_t s_sat, s_lo, s_hi, s_skip;
  const uint32_t nch = a.heavy_count[1];
  for (uint32_t it = blockIdx.x; it < nch; it += gridDim.x) {
    const uint32_t slot = a.heavy_chunks[2 * it], c = a.heavy_chunks[2 * it + 1];
    const uint32_t rec = a.heavy_rows[slot];
    const uint32_t row = rec & 0x7fffffffu;
    const int d = (int)(rec >> 31);
    const uint32_t need = (a.ne[d] >= 32) ? 0xffffffffu : ((1u << a.ne[d]) - 1u);
    const uint32_t b0 = a.f[d].rp[row], e0 = a.f[d].rp[row + 1];
    const uint32_t b = b0 + c * HEAVY_CHUNK, e = min(e0, b + HEAVY_CHUNK);
    __syncthreads();  // the previous chunk is done with the shared words
    if (threadIdx.x < 32) {
      const uint32_t lo = warp_lower_bound(a.f[d].pred, b, e, a.minl[d]);
      const uint32_t hi = warp_lower_bound(a.f[d].pred, lo, e, a.maxl[d] + 1);
      if (threadIdx.x == 0) {
        s_lo = lo;
        s_hi = hi;
        s_sat = 0;
        // the row is already satisfied by other chunks: nothing to learn here
        s_skip = *(volatile const uint32_t*)(a.heavy_sat + slot) == need;
      }
    }
    __syncthreads();
    if (s_skip) continue;
    const uint32_t lo = s_lo, hi = s_hi;
    uint32_t sat = 0, matched = 0;
    for (uint32_t k0 = lo; k0 < hi; k0 += 4 * blockDim.x) {
      uint32_t l4[4], c4[4];
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const uint32_t k = k0 + t * blockDim.x + threadIdx.x;
        l4[t] = k < hi ? (uint32_t)__ldg(a.f[d].pred + k) : 0u;
        c4[t] = k < hi ? __ldg(a.f[d].col + k) : 0u;
      }
#pragma unroll
      for (int t = 0; t < 4; t++)
        if (l4[t]) sat |= match_entry(a, d, l4[t], c4[t], row, sat, matched);
      // every 4 steps: stop when the CTA has satisfied every edge of the row
      if (((k0 - lo) / (4 * blockDim.x)) % 4 == 3) {
        if (sat) atomicOr(&s_sat, sat);
        __syncthreads();
        const bool all = s_sat == need;
        __syncthreads();
        if (all) break;
      }
    }
    sat = __reduce_or_sync(GSM_FULL, sat);
    if ((threadIdx.x & 31) == 0 && sat) atomicOr(&s_sat, sat);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_sat) atomicOr(a.heavy_sat + slot, s_sat);
      atomicAdd(a.ctr + C_HEAVY, (unsigned long long)(hi - lo));
      atomicAdd(a.ctr + C_FILTER_SCANNED, (unsigned long long)(hi - lo));
    }
  }
}

// single CTA: clear the bits of heavy rows that missed an edge, then reset the
// heavy-row state for the next launch (no host memsets between launches)
template <typename PT>
__global__ void k_filter_finalize(FilterArgsT<PT> a) {
  GSM_PDL_ENTRY();
  const uint32_t nr = a.heavy_count[0];
  for (uint32_t i = threadIdx.x; i < nr; i += blockDim.x) {
    const uint32_t rec = a.heavy_rows[i];
    const uint32_t row = rec & 0x7fffffffu;
    const int d = (int)(rec >> 31);
    const uint32_t need = (a.ne[d] >= 32) ? 0xffffffffu : ((1u << a.ne[d]) - 1u);
    if (a.heavy_sat[i] != need) {
      const uint32_t b = 1u << (row & 31);
      if ((and_all_ranks(a.cand + (row >> 5), ~b, a.world, a.peers) & b) && a.skip.chg)
        max_all_ranks(a.skip.chg + a.center_slot, a.seq, a.world, a.peers);
    }
    a.heavy_sat[i] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a.heavy_count[0] = 0;
    a.heavy_count[1] = 0;
  }
}

template <typename PT>
static FilterArgsT<PT> to_t(const FilterArgs& a) {
  FilterArgsT<PT> t;
  for (int d = 0; d < 2; d++) {
    t.f[d] = fmt_of<PT>(a.f[d]);
    t.ne[d] = a.ne[d];
    t.minl[d] = 0xffffffffu; t.maxl[d] = 0;
    t.needm[d] = 0;
    for (int j = 0; j < MAXG; j++) {
      t.e[d][j] = a.e[d][j];
      if (j < (int)a.ne[d]) {
        t.needm[d] |= label_bit(a.e[d][j].label);
        t.minl[d] = min(t.minl[d], a.e[d][j].label);
        t.maxl[d] = max(t.maxl[d], a.e[d][j].label);
      }
    }
  }
  t.cand = a.cand; t.n_words = a.n_words;
  t.heavy_rows = a.heavy_rows; t.heavy_chunks = a.heavy_chunks; t.heavy_sat = a.heavy_sat;
  t.heavy_count = a.heavy_count; t.ctr = a.ctr; t.variant = a.variant; t.word_lo = a.word_lo; t.claim = a.claim;
  t.skip = a.skip; t.center_slot = a.center_slot; t.seq = a.seq;
  t.world = a.world < 1 ? 1u : a.world; t.peers = a.peers;
  return t;
}

template <typename PT>
static cudaError_t group_filter_t(const FilterArgs& a, int sm_count, cudaStream_t st, int* launches) {
  FilterArgsT<PT> t = to_t<PT>(a);
  const bool simd = sizeof(PT) == 1 && (a.variant & 1);  // byte-SIMD short rows (opt-in)
  if (a.rows) {  // candidate rows already compacted: perfectly balanced batches of 32 rows
    // one resident wave: 6 CTAs/SM at <= 40 registers (4 for the SIMD variant)
    if (simd) pdl_launch(k_group_filter_rows<PT, true>, (unsigned)sm_count * 4, 256, st, t, a.rows, a.d_nrows);
    else pdl_launch(k_group_filter_rows<PT, false>, (unsigned)sm_count * 6, 256, st, t, a.rows, a.d_nrows);
  } else {
    // 8 warps per CTA; one 32-word chunk per warp, persistent (one wave)
    uint64_t want = (((uint64_t)a.n_words + 31) / 32 + 7) / 8;
    unsigned g = (unsigned)std::min<uint64_t>(std::max<uint64_t>(want, 1), (uint64_t)sm_count * 6);
    if (simd) pdl_launch(k_group_filter<PT, true>, g, 256, st, t);
    else pdl_launch(k_group_filter<PT, false>, g, 256, st, t);
  }
  if (launches) *launches += 1;
  if (a.heavy) {  // only when a scanned format has rows > HEAVY_ROW entries
    pdl_launch(k_filter_heavy<PT>, (unsigned)sm_count * 2, 256, st, t);
    if (launches) *launches += 1;
  }
  if (a.heavy) {  // clears failed heavy rows, resets the heavy counters
    pdl_launch(k_filter_finalize<PT>, 1, 1024, st, t);
    if (launches) *launches += 1;
  }
  return cudaGetLastError();
}

// ---- push form (label-major streaming).  Each thread takes 8 consecutive
// entries per step (two 16-byte loads of s and two of o; the label's range is
// widened to 4-aligned bounds and masked) and already holds the next step's
// loads while it probes the current ones (software pipeline: ~128 B of stream
// in flight per thread).  The probes of an entry (center bit, previous marks,
// neighbour bit) are issued together.  Marks are OR-ed per distinct word
// across the warp (entries are sorted by (s, o): OUT edges aggregate well).
constexpr int PU_G = 2;  // 4-entry groups per thread per step
__device__ __forceinline__ void push_load(const PushArgs& a, uint64_t b4, uint64_t n4, uint64_t g0, uint4 (&vs)[PU_G],
                                          uint4 (&vo)[PU_G]) {
#pragma unroll
  for (int h = 0; h < PU_G; h++) {
    const uint64_t g = g0 + h;
    vs[h] = g < n4 ? __ldcs(reinterpret_cast<const uint4*>(a.s + b4) + g) : make_uint4(0, 0, 0, 0);
    vo[h] = g < n4 ? __ldcs(reinterpret_cast<const uint4*>(a.o + b4) + g) : make_uint4(0, 0, 0, 0);
  }
}

template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_push_edge(PushArgs a) {
  GSM_PDL_ENTRY();
  if (a.skip.skip()) return;
  if (a.in_cnt && *(volatile const unsigned long long*)a.in_cnt == 0) return;  // no row left to mark
  const uint64_t b4 = a.beg & ~3ull;
  const uint64_t n4 = (a.end - b4 + 3) >> 2;  // 4-entry groups
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x * PU_G;
  uint32_t matched = 0;
  uint64_t base = (uint64_t)blockIdx.x * blockDim.x * PU_G;
  uint4 vs[PU_G], vo[PU_G];
  push_load(a, b4, n4, base + (uint64_t)threadIdx.x * PU_G, vs, vo);
  for (; base < n4; base += step) {  // warp-uniform trip count
    const uint64_t g0 = base + (uint64_t)threadIdx.x * PU_G;
    uint32_t ss[4 * PU_G], oo[4 * PU_G];
#pragma unroll
    for (int h = 0; h < PU_G; h++) {
      ss[4 * h] = vs[h].x; ss[4 * h + 1] = vs[h].y; ss[4 * h + 2] = vs[h].z; ss[4 * h + 3] = vs[h].w;
      oo[4 * h] = vo[h].x; oo[4 * h + 1] = vo[h].y; oo[4 * h + 2] = vo[h].z; oo[4 * h + 3] = vo[h].w;
    }
    if (base + step < n4) push_load(a, b4, n4, g0 + step, vs, vo);  // next step, in flight during the probes
    uint32_t x[4 * PU_G], pc[4 * PU_G], pp[4 * PU_G], pn[4 * PU_G];
    uint32_t inr = 0;
#pragma unroll
    for (int j = 0; j < 4 * PU_G; j++) {
      const uint64_t k = b4 + 4 * g0 + j;
      x[j] = a.out ? ss[j] : oo[j];
      const uint32_t w = a.out ? oo[j] : ss[j];
      const bool in = k >= a.beg && k < a.end;
      inr |= (uint32_t)in << j;
      pc[j] = in ? __ldg(a.cand + (x[j] >> 5)) : 0u;
      pp[j] = (in && a.sat_in) ? __ldg(a.sat_in + (x[j] >> 5)) : ~0u;
      pn[j] = (in && a.mode == GE_PROBE) ? __ldg(a.nbr + (w >> 5)) : 0u;
      oo[j] = w;  // reuse: the neighbour end
    }
    // a thread's entries are consecutive: marks of one word are OR-ed locally and
    // flushed with one atomicOr when the word changes (OUT edges: a row's entries
    // and neighbouring rows share words; IN edges: one atomic per marked entry)
    uint32_t cur_w = 0xffffffffu, cur_b = 0;
#pragma unroll
    for (int j = 0; j < 4 * PU_G; j++) {
      const uint32_t w = oo[j];
      const bool m = a.mode == GE_PROBE ? ((pn[j] >> (w & 31)) & 1u) != 0 : (w == (a.mode == GE_SELF ? x[j] : a.cval));
      const bool ok = ((inr >> j) & 1u) && ((pc[j] & pp[j]) >> (x[j] & 31) & 1u) && m;
      if (ok) {
        const uint32_t word = x[j] >> 5;
        if (word != cur_w) {
          if (cur_b) atomicOr(a.sat_out + cur_w, cur_b);
          cur_w = word;
          cur_b = 0;
        }
        cur_b |= 1u << (x[j] & 31);
        matched++;
      }
    }
    if (cur_b) atomicOr(a.sat_out + cur_w, cur_b);
  }
  matched = __reduce_add_sync(GSM_FULL, matched);
  if ((threadIdx.x & 31) == 0 && matched) {
    atomicAdd(a.ctr + C_PUSH_MATCHED, (unsigned long long)matched);
    atomicAdd(a.out_cnt, (unsigned long long)matched);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(a.ctr + C_PUSH, (unsigned long long)(a.end - a.beg));
}

cudaError_t launch_push_edge(const PushArgs& a, int sm_count, cudaStream_t st) {
  const uint64_t n4 = a.end > a.beg ? (a.end - (a.beg & ~3ull) + 3) / 4 : 0;
  const uint64_t per_cta = 256ull * PU_G;
  const char* ev = getenv("GSMART_PUSH_MINB");  // A/B: resident CTAs per SM (register budget)
  const int mb = ev ? atoi(ev) : 3;
  const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n4 + per_cta - 1) / per_cta, (uint64_t)sm_count * mb));
  if (mb == 4) return pdl_launch(k_push_edge<4>, g, 256, st, a);
  if (mb == 6) return pdl_launch(k_push_edge<6>, g, 256, st, a);
  return pdl_launch(k_push_edge<3>, g, 256, st, a);
}

// cand[0, n_words) &= sat — this rank's word range; world > 1: the new words are
// stored into every rank's copy (only this rank writes these words)
__global__ void __launch_bounds__(256) k_and_tracked(uint32_t* __restrict__ cand, const uint32_t* __restrict__ sat,
                                                    uint32_t n_words, SkipIf skip, uint32_t center_slot,
                                                    uint32_t seq, PeerSet ps) {
  GSM_PDL_ENTRY();
  if (skip.skip()) return;
  bool changed = false;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < n_words; w += gridDim.x * blockDim.x) {
    const uint32_t c = cand[w], v = c & __ldcs(sat + w);
    if (v != c) {
      cand[w] = v;
      for (uint32_t q = 0; q < ps.world; q++)
        if (ps.peers.words[q]) cand[w + ps.peers.words[q]] = v;
      changed = true;
    }
  }
  if (__any_sync(GSM_FULL, changed) && (threadIdx.x & 31) == 0 && skip.chg)
    max_all_ranks(skip.chg + center_slot, seq, ps.world, ps.peers);
}

cudaError_t launch_and_tracked(uint32_t* cand, const uint32_t* sat, uint32_t n_words, SkipIf skip,
                               uint32_t center_slot, uint32_t seq, const PeerSet& ps, cudaStream_t st, int sm_count) {
  const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_words + 255) / 256, (uint64_t)sm_count * 8));
  PeerSet p = ps;
  if (p.world < 1) p.world = 1;
  return pdl_launch(k_and_tracked, g, 256, st, cand, sat, n_words, skip, center_slot, seq, p);
}

cudaError_t launch_group_filter(const FilterArgs& a, int pred_bytes, int sm_count, cudaStream_t st,
                                int* launches) {
  return pred_bytes == 1 ? group_filter_t<uint8_t>(a, sm_count, st, launches)
                         : group_filter_t<uint16_t>(a, sm_count, st, launches);
}

// =====================================================================================
// a9 — row enumeration (one row per surviving leaf) and lexicographic sort
// =====================================================================================
struct ColMap {
  uint32_t c[MAXL];
};

// One row per leaf, 256 rows per CTA step: each thread walks its leaf's parent
// chain into a shared-memory tile (row-major, n_cols words per row), then the
// CTA writes the tile's contiguous n_cols * 256 words with coalesced stores
// (a direct store per column would touch n_cols * 32 scattered words per warp).
constexpr int EN_T = 256;
// Fused last level (lf.bind != null): every node of the last trie level is a
// solution (a8 removes none), so its compaction is a copy — the kernel reads the
// uncompacted level, remaps parents through the previous level's new indices,
// writes the compacted level into the result and the rows in the same pass.
__device__ __forceinline__ void walk_row(const OutTab* __restrict__ ot, uint32_t L, const ColMap& cm,
                                         const LastLevel& lf, uint32_t m, uint32_t* r, bool store_level) {
  uint32_t idx = m;
  int k = (int)L - 1;
  if (lf.bind) {
    const uint32_t b = __ldcs(lf.bind + m), p = __ldg(lf.newidx_prev + __ldcs(lf.parent + m));
    if (store_level) {
      __stcs(ot->bind[k] + m, b);
      __stcs(ot->parent[k] + m, p);
    }
    r[cm.c[k]] = b;
    idx = p;
    k--;
  }
  for (; k >= 0; k--) {
    r[cm.c[k]] = __ldg(ot->bind[k] + idx);
    if (k > 0) idx = __ldg(ot->parent[k] + idx);
  }
}

// lexicographic a > b over n columns
__device__ __forceinline__ bool row_gt(const uint32_t* a, const uint32_t* b, uint32_t n) {
  for (uint32_t c = 0; c < n; c++)
    if (a[c] != b[c]) return a[c] > b[c];
  return false;
}

__global__ void __launch_bounds__(EN_T) k_enumerate(const OutTab* __restrict__ ot, uint32_t L, ColMap cm,
                                                   const unsigned long long* __restrict__ d_n_last, uint32_t n_cols,
                                                   LastLevel lf) {
  GSM_PDL_ENTRY();
  if (!ot->go) return;
  extern __shared__ uint32_t s_rows[];
  const uint32_t n_last = (uint32_t)*d_n_last;
  uint32_t* __restrict__ rows = ot->rows;
  uint32_t* __restrict__ rank = ot->rank;
  if (lf.bind && blockIdx.x == 0 && threadIdx.x == 0) *lf.d_n_out = n_last;
  bool descent = false;
  for (uint64_t base = (uint64_t)blockIdx.x * EN_T; base < n_last; base += (uint64_t)gridDim.x * EN_T) {
    const uint64_t m = base + threadIdx.x;
    if (m < n_last) {
      walk_row(ot, L, cm, lf, (uint32_t)m, s_rows + threadIdx.x * n_cols, true);
      if (rank && m < SORT_SMALL_MAXN) rank[m] = 0;  // the rank sort adds into it
    }
    __syncthreads();
    if (lf.sorted && m < n_last) {  // the sort check rides along: each row against its predecessor
      if (threadIdx.x > 0) {
        descent = descent || row_gt(s_rows + (threadIdx.x - 1) * n_cols, s_rows + threadIdx.x * n_cols, n_cols);
      } else if (base > 0) {  // the previous tile's last row, recomputed
        uint32_t prev[MAXL];
        walk_row(ot, L, cm, lf, (uint32_t)(base - 1), prev, false);
        descent = descent || row_gt(prev, s_rows, n_cols);
      }
    }
    const uint64_t nr = min((uint64_t)EN_T, (uint64_t)n_last - base);
    const uint32_t words = (uint32_t)(nr * n_cols);
    uint32_t* out = rows + base * n_cols;
    for (uint32_t i = threadIdx.x; i < words; i += EN_T) __stcs(out + i, s_rows[i]);
    __syncthreads();
  }
  if (lf.sorted && __any_sync(GSM_FULL, descent) && (threadIdx.x & 31) == 0) *lf.sorted = 0;
}

cudaError_t launch_enumerate(const OutTab* ot, uint32_t n_levels, const uint32_t* col_of_level,
                             const unsigned long long* d_n_last, uint32_t n_cols, int sm_count, cudaStream_t st,
                             LastLevel lf) {
  ColMap cm;
  for (uint32_t k = 0; k < MAXL; k++) cm.c[k] = k < n_levels ? col_of_level[k] : 0;
  const size_t smem = (size_t)EN_T * n_cols * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_enumerate, cudaFuncAttributeMaxDynamicSharedMemorySize, EN_T * MAXL * 4);
    attr = true;
  }
  pdl_launch_smem(k_enumerate, (unsigned)sm_count * 8, EN_T, smem, st, ot, n_levels, cm, d_n_last, n_cols, lf);
  return cudaGetLastError();
}

// Are the rows already lexicographically sorted?  (A trie order that puts
// functional patterns first yields sorted rows whenever those columns are
// determined by the earlier ones.)  *sorted starts at 1; any descent clears it
// and the sort runs; otherwise every sort kernel exits at entry and the rows
// are copied.
__global__ void k_rows_sorted(const uint32_t* __restrict__ rows, uint64_t n, uint32_t n_cols, int* sorted) {
  GSM_PDL_ENTRY();
  bool bad = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* a = rows + i * n_cols;
    for (uint32_t c = 0; c < n_cols; c++) {
      const uint32_t x = a[c], y = a[n_cols + c];
      if (x != y) {
        bad = bad || x > y;
        break;
      }
    }
  }
  if (__any_sync(GSM_FULL, bad) && (threadIdx.x & 31) == 0) *sorted = 0;
}

// in-place sort: the rows move to the sort's scratch only when they are not sorted
__global__ void k_copy_unless_sorted(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, uint64_t m,
                                     const int* sorted) {
  GSM_PDL_ENTRY();
  if (*sorted) return;
  const uint64_t m4 = (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15 ? 0 : m / 4;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m4; i += (uint64_t)gridDim.x * blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = __ldcs(reinterpret_cast<const uint4*>(src) + i);
  for (uint64_t i = 4 * m4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_iota(uint32_t* v, uint64_t n, const int* skip) {
  GSM_PDL_ENTRY();
  if (skip && *skip) return;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = (uint32_t)i;
}

// key of up to 64 bits: columns [c0, c1) concatenated, most significant first
__global__ void k_gather_key(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ perm, uint64_t n,
                             uint32_t n_cols, uint32_t c0, uint32_t c1, int key_bits,
                             unsigned long long* __restrict__ keys, const int* skip) {
  GSM_PDL_ENTRY();
  if (skip && *skip) return;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* r = rows + (uint64_t)perm[i] * n_cols;
    unsigned long long k = 0;
    for (uint32_t c = c0; c < c1; c++) k = (k << key_bits) | r[c];
    keys[i] = k;
  }
}

__global__ void k_gather_rows(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ perm, uint64_t n,
                              uint32_t n_cols, uint32_t* __restrict__ out, const int* skip, int ident_copy) {
  GSM_PDL_ENTRY();
  const bool ident = skip && *skip;  // already sorted: a straight copy (in place: nothing to do)
  if (ident && !ident_copy) return;
  if (ident) {
    const uint64_t m = n * n_cols;
    const uint64_t m4 = (reinterpret_cast<uintptr_t>(rows) | reinterpret_cast<uintptr_t>(out)) & 15 ? 0 : m / 4;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m4; i += (uint64_t)gridDim.x * blockDim.x)
      reinterpret_cast<uint4*>(out)[i] = __ldcs(reinterpret_cast<const uint4*>(rows) + i);
    for (uint64_t i = 4 * m4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
      out[i] = rows[i];
    return;
  }
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * n_cols;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t r = i / n_cols, c = i - r * n_cols;
    out[i] = rows[(uint64_t)perm[r] * n_cols + c];
  }
}

// Small results: rank sort.  rank(i) = #{j : row_j < row_i} is a permutation
// (rows are distinct); the j range is split over gridDim.y CTAs whose partial
// counts are added atomically (ot->rank was zeroed by the enumeration), then rows
// are scattered to their ranks.  n is read from device memory, so the fixed grid
// below is valid for any n <= SORT_SMALL_MAXN (CTAs past n exit at once).
constexpr uint32_t SR_T = 256, SR_SMEM_W = 8192, SR_SPLIT = 32;
static_assert((SORT_SMALL_MAXN / SR_SPLIT + 1) * SORT_SMALL_MAXC <= SR_SMEM_W, "rank-sort split fits smem");

__global__ void __launch_bounds__(SR_T) k_rank_rows(const OutTab* __restrict__ ot,
                                                   const unsigned long long* __restrict__ d_n, uint32_t nc) {
  GSM_PDL_ENTRY();
  __shared__ uint32_t s_rows[SR_SMEM_W];
  if (!ot->go) return;
  const uint32_t n = (uint32_t)*d_n;
  if (blockIdx.x * SR_T >= n) return;
  const uint32_t* __restrict__ rows = ot->rows;
  const uint32_t per = (n + gridDim.y - 1) / gridDim.y;
  const uint32_t j0 = min(n, blockIdx.y * per), j1 = min(n, j0 + per);
  for (uint32_t k = threadIdx.x; k < (j1 - j0) * nc; k += SR_T) s_rows[k] = rows[(uint64_t)j0 * nc + k];
  __syncthreads();
  const uint32_t i = blockIdx.x * SR_T + threadIdx.x;
  if (i >= n || j1 == j0) return;
  uint32_t me[SORT_SMALL_MAXC];
#pragma unroll
  for (uint32_t c = 0; c < SORT_SMALL_MAXC; c++) me[c] = c < nc ? rows[(uint64_t)i * nc + c] : 0u;
  uint32_t cnt = 0;
  for (uint32_t j = 0; j < j1 - j0; j++) {
    const uint32_t* r = s_rows + j * nc;
    int cmp = 0;  // sign of row_j - row_i
#pragma unroll
    for (uint32_t c = 0; c < SORT_SMALL_MAXC; c++) {
      if (c >= nc || cmp) break;
      const uint32_t x = r[c];
      cmp = x < me[c] ? -1 : (x > me[c] ? 1 : 0);
    }
    cnt += cmp < 0;
  }
  if (cnt) atomicAdd(ot->rank + i, cnt);
}

__global__ void k_scatter_rows(const OutTab* __restrict__ ot, const unsigned long long* __restrict__ d_n,
                               uint32_t nc) {
  GSM_PDL_ENTRY();
  if (!ot->go) return;
  const uint32_t n = (uint32_t)*d_n;
  const uint32_t* __restrict__ rows = ot->rows;
  const uint32_t* __restrict__ rank = ot->rank;
  uint32_t* __restrict__ out = ot->sorted;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < (uint64_t)n * nc;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(k / nc), c = (uint32_t)(k - (uint64_t)i * nc);
    out[(uint64_t)rank[i] * nc + c] = rows[k];
  }
}

cudaError_t sort_rows_small(const OutTab* ot, const unsigned long long* d_n, uint32_t n_cols, cudaStream_t st,
                            int* launches) {
  pdl_launch(k_rank_rows, dim3(SORT_SMALL_MAXN / SR_T, SR_SPLIT), SR_T, st, ot, d_n, n_cols);
  pdl_launch(k_scatter_rows, 148 * 8, 256, st, ot, d_n, n_cols);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

// columns [0, n_key) in chunks of <= 64 key bits, least significant chunk first
static int sort_chunk_cols(int key_bits) { return std::max(1, 64 / std::max(key_bits, 1)); }

size_t sort_rows_tmp_bytes(uint64_t n, uint32_t n_cols) {
  const size_t s4 = ((n * 4 + 255) / 256) * 256, s8 = ((n * 8 + 255) / 256) * 256;
  (void)n_cols;
  return 2 * s4 + 2 * s8 + radix_tmp_bytes(n) + 256;
}

// Lexicographic sort of distinct rows.  Only columns [0, n_key) need sorting: the
// input order already sorts rows that agree on them (the caller derives n_key from
// the trie order).  LSD over <= 64-bit keys of packed columns (hand-written radix
// sort, radix.cu, permutation as payload), least significant chunk first; stable.
cudaError_t sort_rows(const uint32_t* rows, uint32_t* rows_out, uint64_t n, uint32_t n_cols, uint32_t n_key,
                      int key_bits, void* tmp, size_t tmp_bytes, cudaStream_t st, int* launches, int* sorted_flag,
                      bool inplace, bool prechecked) {
  const size_t s4 = ((n * 4 + 255) / 256) * 256, s8 = ((n * 8 + 255) / 256) * 256;
  uint32_t* perm = (uint32_t*)tmp;
  uint32_t* perm2 = (uint32_t*)((char*)tmp + s4);
  unsigned long long* keys = (unsigned long long*)((char*)tmp + 2 * s4);
  unsigned long long* keys2 = (unsigned long long*)((char*)tmp + 2 * s4 + s8);
  void* rtmp = (char*)tmp + 2 * s4 + 2 * s8;
  const size_t rbytes = tmp_bytes - 2 * s4 - 2 * s8;
  unsigned g = grid_for(n, 256, 148 * 32);
  int nl = 1;
  if (inplace && !sorted_flag) return cudaErrorInvalidValue;
  if (sorted_flag && prechecked) {  // the enumeration already set the flag
    if (inplace) {
      pdl_launch(k_copy_unless_sorted, grid_for(n * n_cols / 4 + 1, 256, 148 * 32), 256, st, (const uint32_t*)rows_out,
                 const_cast<uint32_t*>(rows), n * n_cols, (const int*)sorted_flag);
      nl++;
    }
  } else if (sorted_flag) {  // rows often arrive sorted (functional patterns first in the trie): check once
    cudaError_t e = cudaMemsetAsync(sorted_flag, 0, 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(sorted_flag, 1, 1, st);  // little-endian int 1
    if (e != cudaSuccess) return e;
    pdl_launch(k_rows_sorted, g, 256, st, inplace ? rows_out : rows, n, n_cols, sorted_flag);
    nl++;
    if (inplace) {  // rows_out holds the input: move it to `rows` (scratch) only if a sort follows
      pdl_launch(k_copy_unless_sorted, grid_for(n * n_cols / 4 + 1, 256, 148 * 32), 256, st, (const uint32_t*)rows_out,
                 const_cast<uint32_t*>(rows), n * n_cols, (const int*)sorted_flag);
      nl++;
    }
  }
  pdl_launch(k_iota, g, 256, st, perm, n, (const int*)sorted_flag);
  const int per = sort_chunk_cols(key_bits);
  for (int c1 = (int)std::min(n_key, n_cols); c1 > 0; c1 -= per) {
    const int c0 = std::max(0, c1 - per);
    pdl_launch(k_gather_key, g, 256, st, rows, perm, n, n_cols, (uint32_t)c0, (uint32_t)c1, key_bits, keys,
               (const int*)sorted_flag);
    int second = 0;
    cudaError_t e = radix_sort_pairs_u64_u32((uint64_t*)keys, (uint64_t*)keys2, perm, perm2, n, 0,
                                             (c1 - c0) * key_bits, rtmp, rbytes, st, &second, &nl, false, sorted_flag);
    if (e != cudaSuccess) return e;
    if (second) std::swap(perm, perm2);
    nl += 1;
  }
  pdl_launch(k_gather_rows, grid_for(n * n_cols, 256, 148 * 32), 256, st, rows, perm, n, n_cols, rows_out,
             (const int*)sorted_flag, inplace ? 0 : 1);
  if (launches) *launches += nl + 1;
  return cudaGetLastError();
}

}  // namespace gsm
