// a5-a8 without host round trips: single-pass decoupled look-back kernels whose
// sizes live in device memory (§7.1 tree-based binding storage,
// §7.2.2 pre-pruning, §8.1 steps 3-4 tree pruning; DESIGN.md §1 steps 5-6).
//
// Level k of the trie is built by two launches:
//   k_seg_scan : per parent n, the child segment (beg, len) = seg^dir_label of the
//                parent-level binding (or the candidate list of a free level),
//                exclusive-scanned into off[] (off[F] = T = total entries);
//   k_expand_lb: tiles of 1024 virtual entries t in [0, T): parent by search in
//                off[], child = col[beg + t - off[n]], keep = cand bit (pre-prune)
//                AND every closing edge; order-preserving emit at the tile's
//                look-back prefix, so parent[] stays non-decreasing.
// Overflow of a capacity is flagged in device memory and handled by the host
// after the single sync (grow + re-run the expansion).
#include "kernels.h"
#include "lookback.cuh"

namespace gsm {

__device__ __forceinline__ uint32_t ub_global(const uint32_t* __restrict__ a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;  // first i with a[i] > x
  while (lo < hi) {
    uint32_t m = (lo + hi) >> 1;
    if (__ldg(a + m) <= x) lo = m + 1; else hi = m;
  }
  return lo;
}

__device__ __forceinline__ uint32_t ancestor(const LevelTab& t, uint32_t k, uint32_t n, uint32_t j) {
  while (k > j) {
    n = __ldg(t.parent[k] + n);
    k--;
  }
  return __ldg(t.bind[j] + n);
}

// ------------------------------------------------------------------ bitmap -> ids
constexpr int BC_T = 256, BC_W = 8, BC_TILE = BC_T * BC_W;  // words per tile

__global__ void __launch_bounds__(BC_T) k_bitmap_compact_lb(const uint32_t* __restrict__ bm, uint32_t n_words,
                                                           uint32_t* __restrict__ ids, uint64_t cap,
                                                           unsigned long long* d_count, int* overflow,
                                                           LBArgs lb, uint32_t id_base) {
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_red[32];
  __shared__ unsigned long long s_pref;
  const uint32_t ntiles = (n_words + BC_TILE - 1) / BC_TILE;
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // warp wib of a tile owns words [tile*2048 + wib*256, +256) in 8 coalesced rounds of
  // 32 words; ids are emitted warp-cooperatively (lane b writes bit b of each word)
  while (true) {
    const uint32_t tile = lb_claim(lb.counter(), &s_tile);
    if (tile >= ntiles) break;
    const uint64_t wbase = (uint64_t)tile * BC_TILE + wib * (BC_W * 32);
    uint32_t w[BC_W], off[BC_W];
    uint32_t run = 0;  // words of earlier rounds in this warp
#pragma unroll
    for (int r = 0; r < BC_W; r++) {
      const uint64_t wi = wbase + r * 32 + lane;
      w[r] = wi < n_words ? __ldcg(bm + wi) : 0u;
    }
#pragma unroll
    for (int r = 0; r < BC_W; r++) {
      const uint32_t c = __popc(w[r]);
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(GSM_FULL, incl, o);
        if ((int)lane >= o) incl += y;
      }
      off[r] = run + incl - c;
      run += __shfl_sync(GSM_FULL, incl, 31);
    }
    // block: exclusive scan of the 8 warp totals
    unsigned long long tot;
    const unsigned long long wex =
        block_exclusive_scan<unsigned long long>(lane == 0 ? (unsigned long long)run : 0ull, s_red, &tot);
    const uint64_t pref = lb_prefix(lb.status, lb.epoch(), tile, tot, &s_pref);
    const uint64_t base_pos = pref + __shfl_sync(GSM_FULL, wex, 0);
#pragma unroll
    for (int r = 0; r < BC_W; r++) {
      uint32_t nz = __ballot_sync(GSM_FULL, w[r] != 0);
      while (nz) {
        const int j = __ffs(nz) - 1;
        nz &= nz - 1;
        const uint32_t wj = __shfl_sync(GSM_FULL, w[r], j), oj = __shfl_sync(GSM_FULL, off[r], j);
        if ((wj >> lane) & 1u) {
          const uint64_t pos = base_pos + oj + __popc(wj & lanemask_lt());
          if (pos < cap) ids[pos] = (uint32_t)((wbase + r * 32 + j) * 32 + lane) + id_base;
          else atomicOr(overflow, 1);
        }
      }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) *d_count = pref + tot;
  }
}

cudaError_t launch_bitmap_compact_lb(const uint32_t* bm, uint32_t n_words, uint32_t* ids, uint64_t cap,
                                     unsigned long long* d_count, int* overflow, LBArgs lb, int sm_count,
                                     cudaStream_t st, uint32_t id_base) {
  uint32_t ntiles = (n_words + BC_TILE - 1) / BC_TILE;
  unsigned g = std::max(1u, std::min(ntiles, (uint32_t)sm_count * 8));
  k_bitmap_compact_lb<<<g, BC_T, 0, st>>>(bm, n_words, ids, cap, d_count, overflow, lb, id_base);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ level k: segments + scan
constexpr int SS_T = 256, SS_I = 4, SS_TILE = SS_T * SS_I;
constexpr int EX_T = 256, EX_I = 4, EX_TILE = EX_T * EX_I;  // expansion tile (entries)

template <typename PT>
__global__ void __launch_bounds__(SS_T) k_seg_scan(ExpArgs2 a) {
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_red[32];
  __shared__ unsigned long long s_pref;
  const uint64_t F = *a.d_nparent;
  if (F > a.cap_par) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(a.overflow, 1);
    return;
  }
  const uint32_t ntiles = (uint32_t)((F + SS_TILE - 1) / SS_TILE);
  Fmt<PT> f = fmt_of<PT>(a.f[a.dir & 1]);
  const uint32_t list_len = a.tree ? 0u : (uint32_t)*a.d_list_len;
  while (true) {
    const uint32_t tile = lb_claim(a.lb.counter(), &s_tile);
    if (tile >= ntiles) break;
    const uint64_t base = (uint64_t)tile * SS_TILE + threadIdx.x * SS_I;
    uint32_t len[SS_I];
    unsigned long long sum = 0;
#pragma unroll
    for (int j = 0; j < SS_I; j++) {
      len[j] = 0;
      const uint64_t n = base + j;
      if (n < F) {
        uint32_t beg = 0, l = list_len;
        if (a.tree) {
          uint32_t b = ancestor(a.tab, a.k - 1, (uint32_t)n, a.parent_level), lo, hi;
          label_range(f, b, a.label, lo, hi);
          beg = lo;
          l = hi - lo;
        }
        a.seg_beg[n] = beg;
        len[j] = l;
        sum += l;
      }
    }
    unsigned long long tot;
    unsigned long long ex = block_exclusive_scan<unsigned long long>(sum, s_red, &tot);
    const uint64_t pref = lb_prefix(a.lb.status, a.lb.epoch(), tile, tot, &s_pref);
    uint64_t run = pref + ex;
#pragma unroll
    for (int j = 0; j < SS_I; j++) {
      const uint64_t n = base + j;
      if (n < F) {
        a.off[n] = (uint32_t)run;
        // the parent holding each expansion-tile boundary t records itself, so
        // k_expand_lb finds a tile's parent range without a global search
        for (uint64_t t = (run + EX_TILE - 1) / EX_TILE * EX_TILE; t < run + len[j]; t += EX_TILE)
          if (t / EX_TILE < a.lb.cap_tiles) a.tile_start[t / EX_TILE] = (uint32_t)n;
        run += len[j];
      }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      const uint64_t T = pref + tot;
      a.off[F] = (uint32_t)T;
      *a.d_T = T;
      const uint64_t nt = (T + EX_TILE - 1) / EX_TILE;
      if (nt < a.lb.cap_tiles) a.tile_start[nt] = (uint32_t)F;  // sentinel
    }
  }
}

// ------------------------------------------------------------------ level k: expansion
constexpr uint32_t OFFCAP = 2048, TGTP = 1024, TGTC = 4;

template <typename PT>
__global__ void __launch_bounds__(EX_T, 4) k_expand_lb(ExpArgs2 a) {
  __shared__ uint32_t s_off[OFFCAP];
  __shared__ uint32_t s_tgt[TGTP * TGTC];
  __shared__ uint32_t s_tile, s_nlo, s_nhi;
  __shared__ unsigned long long s_red[32];
  __shared__ unsigned long long s_pref;
  const uint64_t F = *a.d_nparent;
  if (F > a.cap_par) return;  // flagged by k_seg_scan
  const uint64_t T = *a.d_T;
  if (T >= 0xffffffffull) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(a.overflow, 2);
    return;
  }
  const uint32_t ntiles = (uint32_t)((T + EX_TILE - 1) / EX_TILE);
  if (ntiles > a.lb.cap_tiles) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(a.overflow, 2);
    return;
  }
  const Fmt<PT> fsrc = fmt_of<PT>(a.f[a.dir & 1]);
  const Fmt<PT> f0 = fmt_of<PT>(a.f[0]), f1 = fmt_of<PT>(a.f[1]);
  const uint32_t F1 = (uint32_t)F + 1;
  unsigned long long n_exam = 0, n_close = 0;
  while (true) {
    const uint32_t tile = lb_claim(a.lb.counter(), &s_tile);
    if (tile >= ntiles) break;
    const uint32_t base = tile * EX_TILE;
    const uint32_t last = (uint32_t)min((uint64_t)base + EX_TILE, T) - 1;
    if (threadIdx.x == 0) {
      s_nlo = __ldg(a.tile_start + tile);
      s_nhi = min(__ldg(a.tile_start + tile + 1), (uint32_t)F - 1);
    }
    __syncthreads();
    const uint32_t nlo = s_nlo, nr = s_nhi - s_nlo + 1;
    const bool soff = nr + 1 <= OFFCAP;
    if (soff)
      for (uint32_t i = threadIdx.x; i <= nr; i += EX_T) s_off[i] = __ldg(a.off + nlo + i);
    const bool stgt = a.ncl > 0 && a.ncl <= TGTC && nr <= TGTP;
    if (stgt)
      for (uint32_t i = threadIdx.x; i < nr * a.ncl; i += EX_T) {
        const uint32_t p = i / a.ncl, c = i - p * a.ncl;
        s_tgt[p * TGTC + c] = a.cl[c].self ? 0u : ancestor(a.tab, a.k - 1, nlo + p, a.cl[c].other_level);
      }
    __syncthreads();
    uint32_t node[EX_I], child[EX_I], keepm = 0;
    const uint32_t t0 = base + threadIdx.x * EX_I;
#pragma unroll
    for (int j = 0; j < EX_I; j++) {
      const uint32_t t = t0 + j;
      node[j] = 0;
      child[j] = 0;
      if (t > last) continue;
      uint32_t n, o;
      if (soff) {
        uint32_t lo = 0, hi = nr + 1;
        while (lo < hi) {
          uint32_t m = (lo + hi) >> 1;
          if (s_off[m] <= t) lo = m + 1; else hi = m;
        }
        n = nlo + lo - 1;
        o = s_off[lo - 1];
      } else {
        n = ub_global(a.off, F1, t) - 1;
        o = __ldg(a.off + n);
      }
      const uint32_t pos = t - o;
      const uint32_t c = a.tree ? __ldg(fsrc.col + __ldg(a.seg_beg + n) + pos) : __ldg(a.list + pos);
      bool keep = bit_of(a.cand, c) != 0;
      n_exam++;
      for (uint32_t q = 0; q < a.ncl && keep; q++) {
        const ClosingDev cl = a.cl[q];
        uint32_t tgt = c;
        if (!cl.self) tgt = stgt ? s_tgt[(n - nlo) * TGTC + q] : ancestor(a.tab, a.k - 1, n, cl.other_level);
        // (c, l, tgt) in the child's row of format dir  <=>  (tgt, l, c) in tgt's row of the
        // other format: binary-search the shorter row (a hub on one side costs log of the other)
        const Fmt<PT>& fc = cl.dir ? f1 : f0;
        const Fmt<PT>& fo = cl.dir ? f0 : f1;
        const uint32_t lc = __ldg(fc.rp + c + 1) - __ldg(fc.rp + c);
        const uint32_t lt = __ldg(fo.rp + tgt + 1) - __ldg(fo.rp + tgt);
        keep = lc <= lt ? has_entry(fc, c, cl.label, tgt) : has_entry(fo, tgt, cl.label, c);
        n_close++;
      }
      node[j] = n;
      child[j] = c;
      if (keep) keepm |= 1u << j;
    }
    unsigned long long tot;
    unsigned long long ex = block_exclusive_scan<unsigned long long>((unsigned long long)__popc(keepm), s_red, &tot);
    const uint64_t pref = lb_prefix(a.lb.status, a.lb.epoch(), tile, tot, &s_pref);
    uint64_t pos = pref + ex;
#pragma unroll
    for (int j = 0; j < EX_I; j++) {
      if (!((keepm >> j) & 1u)) continue;
      if (pos < a.cap_out) {
        a.out_parent[pos] = node[j];
        a.out_bind[pos] = child[j];
        if (a.out_alive) a.out_alive[pos] = 0;
      } else {
        atomicOr(a.overflow, 1);
      }
      pos++;
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) *a.d_nout = pref + tot;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    n_exam += __shfl_down_sync(GSM_FULL, n_exam, o);
    n_close += __shfl_down_sync(GSM_FULL, n_close, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (n_exam) atomicAdd(a.ctr + C_EXPAND, n_exam);
    if (n_close) atomicAdd(a.ctr + C_CLOSING, n_close);
  }
}

cudaError_t launch_seg_scan(const ExpArgs2& a, int pred_bytes, int sm_count, cudaStream_t st) {
  unsigned g = (unsigned)sm_count * 8;
  if (pred_bytes == 1) k_seg_scan<uint8_t><<<g, SS_T, 0, st>>>(a);
  else k_seg_scan<uint16_t><<<g, SS_T, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_expand_lb(const ExpArgs2& a, int pred_bytes, int sm_count, cudaStream_t st) {
  unsigned g = (unsigned)sm_count * 6;
  if (pred_bytes == 1) k_expand_lb<uint8_t><<<g, EX_T, 0, st>>>(a);
  else k_expand_lb<uint16_t><<<g, EX_T, 0, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a8 prune + compaction
__global__ void k_prune_mark_d(const uint32_t* __restrict__ parent, const uint8_t* __restrict__ alive,
                               const unsigned long long* d_n, uint8_t* __restrict__ alive_prev) {
  const uint64_t n = *d_n;
  for (uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < n; m += (uint64_t)gridDim.x * blockDim.x)
    if (!alive || alive[m]) alive_prev[__ldg(parent + m)] = 1;
}

cudaError_t launch_prune_mark_d(const uint32_t* parent, const uint8_t* alive, const unsigned long long* d_n,
                                uint8_t* alive_prev, int sm_count, cudaStream_t st) {
  k_prune_mark_d<<<(unsigned)sm_count * 8, 256, 0, st>>>(parent, alive, d_n, alive_prev);
  return cudaGetLastError();
}

constexpr int CA_T = 256, CA_I = 4, CA_TILE = CA_T * CA_I;

__global__ void __launch_bounds__(CA_T) k_compact_alive_lb(const uint32_t* __restrict__ parent,
                                                          const uint32_t* __restrict__ bind,
                                                          const uint8_t* __restrict__ alive,
                                                          const unsigned long long* d_n,
                                                          const uint32_t* __restrict__ newidx_prev,
                                                          uint32_t* __restrict__ out_parent,
                                                          uint32_t* __restrict__ out_bind,
                                                          uint32_t* __restrict__ newidx,
                                                          unsigned long long* d_count, LBArgs lb) {
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_red[32];
  __shared__ unsigned long long s_pref;
  const uint64_t n = *d_n;
  const uint32_t ntiles = (uint32_t)((n + CA_TILE - 1) / CA_TILE);
  while (true) {
    const uint32_t tile = lb_claim(lb.counter(), &s_tile);
    if (tile >= ntiles) break;
    const uint64_t base = (uint64_t)tile * CA_TILE + threadIdx.x * CA_I;
    uint32_t fl = 0;
#pragma unroll
    for (int j = 0; j < CA_I; j++)
      if (base + j < n && (!alive || alive[base + j])) fl |= 1u << j;
    unsigned long long tot;
    unsigned long long ex = block_exclusive_scan<unsigned long long>((unsigned long long)__popc(fl), s_red, &tot);
    const uint64_t pref = lb_prefix(lb.status, lb.epoch(), tile, tot, &s_pref);
    uint64_t q = pref + ex;
#pragma unroll
    for (int j = 0; j < CA_I; j++) {
      if (!((fl >> j) & 1u)) continue;
      const uint64_t m = base + j;
      out_bind[q] = bind[m];
      if (out_parent) out_parent[q] = newidx_prev ? newidx_prev[parent[m]] : parent[m];
      if (newidx) newidx[m] = (uint32_t)q;
      q++;
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) *d_count = pref + tot;
  }
}

cudaError_t launch_compact_alive_lb(const uint32_t* parent, const uint32_t* bind, const uint8_t* alive,
                                    const unsigned long long* d_n, const uint32_t* newidx_prev, uint32_t* out_parent,
                                    uint32_t* out_bind, uint32_t* newidx, unsigned long long* d_count, LBArgs lb,
                                    int sm_count, cudaStream_t st) {
  k_compact_alive_lb<<<(unsigned)sm_count * 8, CA_T, 0, st>>>(parent, bind, alive, d_n, newidx_prev, out_parent,
                                                              out_bind, newidx, d_count, lb);
  return cudaGetLastError();
}

}  // namespace gsm
