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
#include <cstdlib>

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
  while (k != j) {  // j is an ancestor level of k
    n = __ldg(t.parent[k] + n);
    k = t.up[k];
  }
  return __ldg(t.bind[j] + n);
}

// binding of level j for node n of level k-1 (the expansion's parent level):
// its own binding, a materialised ancestor column, or (fallback) a walk
__device__ __forceinline__ uint32_t anc_binding(const ExpArgs2& a, int idx, uint32_t n, uint32_t j) {
  if (idx == ANC_BIND) return __ldg(a.tab.bind[a.k - 1] + n);
  if (idx >= 0) return __ldg(a.par_anc[idx] + n);
  return ancestor(a.tab, a.k - 1, n, j);
}

// ------------------------------------------------------------------ bitmap -> ids
// One launch, no inter-CTA chain.  The range is cut into <= ~4 chunks per SM of
// whole 2048-word sub-tiles; a CTA takes a ticket (chunks in ticket order, so it
// only ever waits on CTAs that are already running), and
//   1. streams its chunk once (each lane 32 contiguous bytes per 256-word slice)
//      into per-slice popcounts kept in shared memory, publishes the chunk total;
//   2. sums the totals of all earlier chunks - every one is published directly,
//      so this is one parallel read, not a walk back to an inclusive prefix;
//   3. emits its ids sub-tile by sub-tile: a warp's offset comes from the slice
//      counts (no block barrier), empty slices are skipped, and the re-read of a
//      non-empty slice hits L2.
// (A decoupled look-back over thousands of small tiles spent most of its time
// walking back to the last inclusive prefix.)
// BC_W words per lane per slice (8: 32-byte lane loads).  BC_W = 1 for small
// bitmaps (more, shorter CTAs) was measured slower at LUBM-100 (0.29 vs 0.255
// ms of compaction per batch), so one width serves every size.
constexpr int BC_T = 256, BC_W_DEFAULT = 8;
constexpr uint32_t BC_MAX_SLICES = 2048;  // slices per chunk (their counts live in smem)
constexpr uint32_t BC_MAX_CHUNKS = 8192;

template <int BC_W>
static uint32_t bc_chunk_words(uint32_t n_words, int sm_count) {
  constexpr uint32_t BC_SLICE = BC_W * 32, BC_SUB = BC_SLICE * (BC_T / 32);
  const uint64_t want = (uint64_t)sm_count * 4;
  const uint64_t per = std::max<uint64_t>(((uint64_t)n_words + want - 1) / want,
                                          ((uint64_t)n_words + BC_MAX_CHUNKS - 1) / BC_MAX_CHUNKS);
  const uint64_t c = std::max<uint64_t>(BC_SUB, (per + BC_SUB - 1) / BC_SUB * BC_SUB);
  return (uint32_t)std::min<uint64_t>(c, (uint64_t)BC_MAX_SLICES * BC_SLICE);
}

template <int BC_W>
__global__ void __launch_bounds__(BC_T) k_bitmap_compact(const uint32_t* __restrict__ bm, uint32_t n_words,
                                                        uint32_t chunk, uint32_t* __restrict__ ids, uint64_t cap,
                                                        unsigned long long* d_count, int* overflow, LBArgs lb,
                                                        uint32_t id_base, SkipIf skip) {
  GSM_PDL_ENTRY();
  if (skip.skip()) return;
  constexpr uint32_t BC_SLICE = BC_W * 32, BC_SUB = BC_SLICE * (BC_T / 32);
  __shared__ unsigned long long s_red[32];
  __shared__ unsigned long long s_p;
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_cnt[BC_MAX_SLICES];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t nch = (n_words + chunk - 1) / chunk;
  const uint32_t epoch = lb.epoch();
  const uint32_t tk = lb_claim(lb.counter(), &s_tile);
  if (tk >= nch) return;
  const uint64_t w0 = (uint64_t)tk * chunk, w1 = std::min<uint64_t>(n_words, w0 + chunk);
  const uint32_t nsl = (uint32_t)((w1 - w0 + BC_SLICE - 1) / BC_SLICE);
  // 1. slice counts
  const bool vec = (reinterpret_cast<uintptr_t>(bm) & 15) == 0;
  uint32_t wtot = 0;
#pragma unroll 4
  for (uint32_t si = wib; si < nsl; si += BC_T / 32) {
    const uint64_t lw = w0 + (uint64_t)si * BC_SLICE + lane * BC_W;  // this lane's BC_W words
    uint32_t c = 0;
    if (BC_W == 1) {
      c = lw < w1 ? __popc(__ldcg(bm + lw)) : 0u;
    } else if (vec && lw + 8 <= w1) {
      const uint4 x = __ldcg(reinterpret_cast<const uint4*>(bm + lw));
      const uint4 y = __ldcg(reinterpret_cast<const uint4*>(bm + lw + 4));
      c = __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w) + __popc(y.x) + __popc(y.y) + __popc(y.z) +
          __popc(y.w);
    } else {
      for (uint64_t i = lw; i < std::min<uint64_t>(lw + BC_W, w1); i++) c += __popc(__ldcg(bm + i));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(GSM_FULL, c, o);
    if (lane == 0) s_cnt[si] = c;
    wtot += c;
  }
  const unsigned long long tot =
      block_reduce_sum<unsigned long long>(lane == 0 ? (unsigned long long)wtot : 0ull, s_red);
  if (threadIdx.x == 0) atomicExch(lb.status + tk, lb_pack(epoch, 1, tot));
  // 2. prefix = sum of the earlier chunks' totals (each published on its own)
  unsigned long long p = 0;
  for (uint32_t i = threadIdx.x; i < tk; i += BC_T) {
    unsigned long long v;
    do {
      v = *((volatile unsigned long long*)(lb.status + i));
    } while ((uint32_t)(v >> 48) != epoch);
    p += v & LB_VMASK;
  }
  p = block_reduce_sum<unsigned long long>(p, s_red);
  if (threadIdx.x == 0) s_p = p;
  __syncthreads();
  // 3. emission
  uint64_t run_base = s_p;  // ids before the current sub-tile (identical in all warps)
  for (uint64_t t = w0; t < w1; t += BC_SUB) {
    const uint32_t s0 = (uint32_t)((t - w0) / BC_SLICE);
    const uint32_t c = (lane < BC_T / 32 && s0 + lane < nsl) ? s_cnt[s0 + lane] : 0u;
    uint32_t tot8 = c, before = lane < wib ? c : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tot8 += __shfl_xor_sync(GSM_FULL, tot8, o);
      before += __shfl_xor_sync(GSM_FULL, before, o);
    }
    const uint32_t mine = __shfl_sync(GSM_FULL, c, wib);
    if (run_base + tot8 > cap) {  // capacity: flag once, the host grows and re-runs
      if (threadIdx.x == 0 && tot8) atomicOr(overflow, 1);
    } else if (mine) {
      const uint64_t wbase = t + (uint64_t)wib * BC_SLICE;
      uint32_t w[BC_W], incl[BC_W], rbase[BC_W];
#pragma unroll
      for (int r = 0; r < BC_W; r++) {
        const uint64_t wi = wbase + r * 32 + lane;
        w[r] = wi < w1 ? __ldcs(bm + wi) : 0u;
      }
      uint32_t run = 0;
#pragma unroll
      for (int r = 0; r < BC_W; r++) {
        incl[r] = __popc(w[r]);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(GSM_FULL, incl[r], o);
          if ((int)lane >= o) incl[r] += y;
        }
        rbase[r] = run;
        run += __shfl_sync(GSM_FULL, incl[r], 31);
      }
      const uint64_t base_pos = run_base + before;
#pragma unroll
      for (int r = 0; r < BC_W; r++) {
        const uint32_t total = __shfl_sync(GSM_FULL, incl[r], 31);
        uint32_t nz = __ballot_sync(GSM_FULL, w[r] != 0);
        const uint32_t id0 = (uint32_t)((wbase + r * 32) * 32) + id_base;
        uint32_t* out = ids + base_pos + rbase[r];
        if ((total + 31) / 32 * 3 <= (uint32_t)__popc(nz)) {
          // sparse words: id j of the round goes to lane j % 32 (coalesced stores);
          // its word = #lanes with incl <= j, its bit = the (j - excl)-th set bit
          for (uint32_t j0 = 0; j0 < total; j0 += 32) {
            const uint32_t j = j0 + lane;
            uint32_t q = 0;
#pragma unroll
            for (int s = 16; s > 0; s >>= 1)
              if (__shfl_sync(GSM_FULL, incl[r], q + s - 1) <= j) q += s;
            uint32_t wq = __shfl_sync(GSM_FULL, w[r], q);
            uint32_t k = j - (__shfl_sync(GSM_FULL, incl[r], q) - __popc(wq));
            uint32_t bit = 0;
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) {
              const uint32_t lowc = __popc(wq & ((1u << s) - 1u));
              if (k >= lowc) {
                k -= lowc;
                wq >>= s;
                bit += s;
              }
            }
            if (j < total) out[j] = id0 + q * 32 + bit;
          }
        } else {
          // dense words: the warp walks the non-zero words, lane b emits bit b
          const uint32_t excl = incl[r] - __popc(w[r]);
          while (nz) {
            const int j = __ffs(nz) - 1;
            nz &= nz - 1;
            const uint32_t wj = __shfl_sync(GSM_FULL, w[r], j), oj = __shfl_sync(GSM_FULL, excl, j);
            if ((wj >> lane) & 1u) out[oj + __popc(wj & lanemask_lt())] = id0 + j * 32 + lane;
          }
        }
      }
    }
    run_base += tot8;
  }
  if (tk == nch - 1 && threadIdx.x == 0) *d_count = run_base;
}

cudaError_t launch_bitmap_compact_lb(const uint32_t* bm, uint32_t n_words, uint32_t* ids, uint64_t cap,
                                     unsigned long long* d_count, int* overflow, LBArgs lb, int sm_count,
                                     cudaStream_t st, uint32_t id_base, SkipIf skip) {
  if (n_words == 0) return cudaMemsetAsync(d_count, 0, 8, st);
  const char* ev = getenv("GSMART_BC_W");  // A/B: words per lane per slice (8 default, 1)
  if (ev && atoi(ev) == 1) {
    const uint32_t chunk = bc_chunk_words<1>(n_words, sm_count);
    const uint32_t nch = (n_words + chunk - 1) / chunk;
    if (nch > BC_MAX_CHUNKS || nch > lb.cap_tiles) return cudaErrorInvalidValue;
    pdl_launch(k_bitmap_compact<1>, nch, BC_T, st, bm, n_words, chunk, ids, cap, d_count, overflow, lb, id_base,
               skip);
    return cudaGetLastError();
  }
  const uint32_t chunk = bc_chunk_words<BC_W_DEFAULT>(n_words, sm_count);
  const uint32_t nch = (n_words + chunk - 1) / chunk;
  if (nch > BC_MAX_CHUNKS || nch > lb.cap_tiles) return cudaErrorInvalidValue;
  pdl_launch(k_bitmap_compact<BC_W_DEFAULT>, nch, BC_T, st, bm, n_words, chunk, ids, cap, d_count, overflow, lb,
             id_base, skip);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ level k: segments + scan
constexpr int SS_T = 256;
constexpr int EX_TILE = 1024;  // expansion tile (entries); EX_T threads x EX_I entries each

template <typename PT, int SS_I>
__global__ void __launch_bounds__(SS_T) k_seg_scan(ExpArgs2 a) {
  GSM_PDL_ENTRY();
  constexpr int SS_TILE = SS_T * SS_I;
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
    // the SS_I parents of a thread go through each step together (ancestor,
    // row bounds, lock-step label searches), so their loads overlap
    uint32_t act = 0, lo[SS_I], hi[SS_I], e[SS_I];
#pragma unroll
    for (int j = 0; j < SS_I; j++) {
      lo[j] = hi[j] = e[j] = 0;
      if (base + j < F) act |= 1u << j;
    }
    if (a.tree) {
      uint32_t b[SS_I];
#pragma unroll
      for (int j = 0; j < SS_I; j++)
        b[j] = ((act >> j) & 1u) ? anc_binding(a, a.par_idx, (uint32_t)(base + j), a.parent_level) : 0u;
      // consecutive nodes of a thread with the same parent-side binding (a run
      // under one ancestor) share its segment: only the first of a run searches
      uint32_t srch = act;
#pragma unroll
      for (int j = 1; j < SS_I; j++)
        if (((act >> j) & 1u) && b[j] == b[j - 1]) srch &= ~(1u << j);
#pragma unroll
      for (int j = 0; j < SS_I; j++)
        if ((srch >> j) & 1u) {
          lo[j] = __ldg(f.rp + b[j]);
          e[j] = hi[j] = __ldg(f.rp + b[j] + 1);
        }
      // first entry with label >= l, then first with label > l
#pragma unroll
      for (int pass = 0; pass < 2; pass++) {
        const uint32_t key = a.label + (uint32_t)pass;
        uint32_t live = srch;
        while (live) {
#pragma unroll
          for (int j = 0; j < SS_I; j++) {
            if (!((live >> j) & 1u)) continue;
            if (lo[j] >= hi[j]) {
              live &= ~(1u << j);
              continue;
            }
            const uint32_t m = (lo[j] + hi[j]) >> 1;
            if ((uint32_t)__ldg(f.pred + m) < key) lo[j] = m + 1; else hi[j] = m;
          }
        }
        if (pass == 0) {
#pragma unroll
          for (int j = 0; j < SS_I; j++) {
            b[j] = lo[j];  // segment begin
            hi[j] = e[j];
          }
        } else {
#pragma unroll
          for (int j = 0; j < SS_I; j++) {
            hi[j] = lo[j];  // segment end
            lo[j] = b[j];
          }
        }
      }
#pragma unroll
      for (int j = 1; j < SS_I; j++)
        if (((act >> j) & 1u) && !((srch >> j) & 1u)) {
          lo[j] = lo[j - 1];
          hi[j] = hi[j - 1];
        }
    }
#pragma unroll
    for (int j = 0; j < SS_I; j++) {
      len[j] = 0;
      const uint64_t n = base + j;
      if ((act >> j) & 1u) {
        const uint32_t beg = a.tree ? lo[j] : 0u, l = a.tree ? hi[j] - lo[j] : list_len;
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

template <typename PT, int EX_T>
__global__ void __launch_bounds__(EX_T, 1024 / EX_T) k_expand_lb(ExpArgs2 a) {
  GSM_PDL_ENTRY();
  constexpr int EX_I = EX_TILE / EX_T;
  __shared__ __align__(16) uint32_t s_offbuf[OFFCAP + 8];
  __shared__ __align__(8) unsigned long long s_mbar;
  __shared__ uint32_t s_tgt[TGTP * TGTC];
  __shared__ uint32_t s_tile, s_nlo, s_nhi;
  uint32_t tma_phase = 0;
  if (a.use_tma && threadIdx.x == 0) mbar_init(&s_mbar, 1);
  __syncthreads();
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
  const bool csr_only = a.closing_csr != 0 || a.f[1].rp == nullptr;
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
    // the tile's parent offsets off[nlo .. nlo + nr] into shared memory: one TMA
    // bulk copy of the 16-byte-aligned span (issued by one thread, overlapping
    // the closing-target staging below), else plain loads
    uint32_t shift = 0;
    if (soff && a.use_tma) {
      const uint32_t a0 = nlo & ~3u;
      shift = nlo - a0;
      const uint32_t words = (shift + nr + 1 + 3) & ~3u;
      if (threadIdx.x == 0) tma_load_1d(s_offbuf, a.off + a0, words * 4, &s_mbar);
    } else if (soff) {
      for (uint32_t i = threadIdx.x; i <= nr; i += EX_T) s_offbuf[i] = __ldg(a.off + nlo + i);
    }
    const bool stgt = a.ncl > 0 && a.ncl <= TGTC && nr <= TGTP;
    if (stgt)
      for (uint32_t i = threadIdx.x; i < nr * a.ncl; i += EX_T) {
        const uint32_t p = i / a.ncl, c = i - p * a.ncl;
        s_tgt[p * TGTC + c] = a.cl[c].self ? 0u : anc_binding(a, a.cl_idx[c], nlo + p, a.cl[c].other_level);
      }
    if (soff && a.use_tma) {
      mbar_wait(&s_mbar, tma_phase);
      tma_phase ^= 1u;
    }
    __syncthreads();
    const uint32_t* s_off = s_offbuf + shift;
    // The EX_I entries of a thread go through each stage together, so their
    // independent loads (segment begin, column, candidate probe, row bounds,
    // closing-edge search steps) are in flight at the same time.
    uint32_t node[EX_I], child[EX_I], epos[EX_I], keepm = 0;
    const uint32_t t0 = base + threadIdx.x * EX_I;
#pragma unroll
    for (int j = 0; j < EX_I; j++) {  // parent of each entry (shared-memory search)
      const uint32_t t = t0 + j;
      node[j] = 0;
      epos[j] = 0;
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
      node[j] = n;
      epos[j] = t - o;
      keepm |= 1u << j;
    }
    const uint32_t actm = keepm;
    uint32_t sb[EX_I];
#pragma unroll
    for (int j = 0; j < EX_I; j++) sb[j] = (a.tree && ((actm >> j) & 1u)) ? __ldg(a.seg_beg + node[j]) : 0u;
#pragma unroll
    for (int j = 0; j < EX_I; j++)
      child[j] = ((actm >> j) & 1u) ? (a.tree ? __ldg(fsrc.col + sb[j] + epos[j]) : __ldg(a.list + epos[j])) : 0u;
#pragma unroll
    for (int j = 0; j < EX_I; j++)
      if (((actm >> j) & 1u) && !bit_of(a.cand, child[j])) keepm &= ~(1u << j);
    if (a.om_tab) {  // f2: the child must occur under the same root binding at its first occurrence
#pragma unroll
      for (int j = 0; j < EX_I; j++) {
        if (!((keepm >> j) & 1u)) continue;
        const uint32_t r = ancestor(a.tab, a.k - 1, node[j], 0);
        const unsigned long long key = ((unsigned long long)r << 32) | child[j];
        uint64_t h = f_hash(key) & a.om_mask;
        while (true) {
          const unsigned long long v = __ldg(a.om_tab + h);
          if (v == key) break;
          if (v == ~0ull) {
            keepm &= ~(1u << j);
            break;
          }
          h = (h + 1) & a.om_mask;
        }
      }
    }
    n_exam += __popc(actm);
    for (uint32_t q = 0; q < a.ncl && keepm; q++) {
      const ClosingDev cl = a.cl[q];
      // (c, l, tgt) in the child's row of format dir  <=>  (tgt, l, c) in tgt's row of the
      // other format: search the shorter row (a hub on one side costs log of the other)
      const Fmt<PT>& fc = cl.dir ? f1 : f0;
      const Fmt<PT>& fo = cl.dir ? f0 : f1;
      uint32_t row[EX_I], key[EX_I], lo[EX_I], hi[EX_I];
      bool useo[EX_I];
#pragma unroll
      for (int j = 0; j < EX_I; j++) {
        uint32_t tgt = child[j];
        if (!cl.self && ((keepm >> j) & 1u))
          tgt = stgt ? s_tgt[(node[j] - nlo) * TGTC + q] : anc_binding(a, a.cl_idx[q], node[j], cl.other_level);
        row[j] = tgt;  // temporarily the target
      }
#pragma unroll
      for (int j = 0; j < EX_I; j++) {
        const uint32_t c = child[j], tgt = row[j];
        const bool on = (keepm >> j) & 1u;
        // CSR-only LSpM (direction-driven plans): the pattern's subject row is the
        // only one stored — the child's when it is the subject, else the target's
        const bool use_c = on && (!csr_only || cl.dir == 0), use_g = on && (!csr_only || cl.dir == 1);
        const uint32_t c0 = use_c ? __ldg(fc.rp + c) : 0u, c1 = use_c ? __ldg(fc.rp + c + 1) : 0u;
        const uint32_t g0 = use_g ? __ldg(fo.rp + tgt) : 0u, g1 = use_g ? __ldg(fo.rp + tgt + 1) : 0u;
        useo[j] = csr_only ? cl.dir == 1 : (g1 - g0) < (c1 - c0);
        row[j] = useo[j] ? tgt : c;
        key[j] = useo[j] ? c : tgt;
        lo[j] = useo[j] ? g0 : c0;
        hi[j] = useo[j] ? g1 : c1;
      }
      // lock-step binary searches on (pred, col) for the EX_I entries
      uint32_t live = keepm, found = 0;
      while (live) {
#pragma unroll
        for (int j = 0; j < EX_I; j++) {
          if (!((live >> j) & 1u)) continue;
          if (lo[j] >= hi[j]) {
            live &= ~(1u << j);
            continue;
          }
          const uint32_t m = (lo[j] + hi[j]) >> 1;
          const PT* pr = useo[j] ? fo.pred : fc.pred;
          const uint32_t* co = useo[j] ? fo.col : fc.col;
          const uint32_t p = __ldg(pr + m), cc = __ldg(co + m);
          if (p == cl.label && cc == key[j]) {
            found |= 1u << j;
            live &= ~(1u << j);
          } else if (p < cl.label || (p == cl.label && cc < key[j])) {
            lo[j] = m + 1;
          } else {
            hi[j] = m;
          }
        }
      }
      n_close += __popc(keepm);
      keepm &= found;
    }
    unsigned long long tot;
    unsigned long long ex = block_exclusive_scan<unsigned long long>((unsigned long long)__popc(keepm), s_red, &tot);
    const uint64_t pref = lb_prefix(a.lb.status, a.lb.epoch(), tile, tot, &s_pref);
    uint64_t pos = pref + ex;
    if (pref + tot > a.cap_out) {  // capacity: flag once per tile, the host grows and re-runs
      if (threadIdx.x == 0 && tot) atomicOr(a.overflow, 1);
      keepm = 0;
    }
#pragma unroll
    for (int j = 0; j < EX_I; j++) {
      if (!((keepm >> j) & 1u)) continue;
      a.out_parent[pos] = node[j];
      a.out_bind[pos] = child[j];
      if (a.out_alive) a.out_alive[pos] = 0;
      for (uint32_t i = 0; i < a.n_anc_out; i++)  // ancestor columns the deeper levels read
        a.out_anc[i][pos] = a.anc_src[i] == ANC_BIND ? __ldg(a.tab.bind[a.k - 1] + node[j])
                                                     : __ldg(a.par_anc[a.anc_src[i]] + node[j]);
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

// ------------------------------------------------------------------ level k: functional tree edge
// The tree edge's label holds at most one entry per row of the parent's format
// (Lspm::functional, exact from the build): every parent has 0 or 1 child, so
// the segment scan and the load-balanced emit collapse into one pass — per
// parent (one per thread): its binding, the label's first entry in its row,
// the child, candidate probe, closing checks; a block scan + look-back keeps
// the emit order (parent[] non-decreasing).
template <typename PT>
__device__ __forceinline__ bool closing_ok1(const ExpArgs2& a, const Fmt<PT>& f0, const Fmt<PT>& f1, bool csr_only,
                                           uint32_t child, uint32_t node) {
  for (uint32_t q = 0; q < a.ncl; q++) {
    const ClosingDev cl = a.cl[q];
    // (c, l, tgt) in the child's row of format dir <=> (tgt, l, c) in tgt's row of the other
    const Fmt<PT>& fc = cl.dir ? f1 : f0;
    const Fmt<PT>& fo = cl.dir ? f0 : f1;
    const uint32_t tgt = cl.self ? child : anc_binding(a, a.cl_idx[q], node, cl.other_level);
    const bool use_c = !csr_only || cl.dir == 0, use_g = !csr_only || cl.dir == 1;
    const uint32_t c0 = use_c ? __ldg(fc.rp + child) : 0u, c1 = use_c ? __ldg(fc.rp + child + 1) : 0u;
    const uint32_t g0 = use_g ? __ldg(fo.rp + tgt) : 0u, g1 = use_g ? __ldg(fo.rp + tgt + 1) : 0u;
    const bool useo = csr_only ? cl.dir == 1 : (g1 - g0) < (c1 - c0);
    const uint32_t key = useo ? child : tgt;
    uint32_t lo = useo ? g0 : c0, hi = useo ? g1 : c1;
    const PT* pr = useo ? fo.pred : fc.pred;
    const uint32_t* co = useo ? fo.col : fc.col;
    bool found = false;
    while (lo < hi) {
      const uint32_t m = (lo + hi) >> 1;
      const uint32_t p = __ldg(pr + m), cc = __ldg(co + m);
      if (p == cl.label && cc == key) {
        found = true;
        break;
      }
      if (p < cl.label || (p == cl.label && cc < key)) lo = m + 1; else hi = m;
    }
    if (!found) return false;
  }
  return true;
}

constexpr int FX_T = 256;

template <typename PT>
__global__ void __launch_bounds__(FX_T) k_expand_func(ExpArgs2 a) {
  GSM_PDL_ENTRY();
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_red[32];
  __shared__ unsigned long long s_pref;
  const uint64_t F = *a.d_nparent;
  if (F > a.cap_par) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(a.overflow, 1);
    return;
  }
  const uint32_t ntiles = (uint32_t)((F + FX_T - 1) / FX_T);
  const Fmt<PT> fsrc = fmt_of<PT>(a.f[a.dir & 1]);
  const Fmt<PT> f0 = fmt_of<PT>(a.f[0]), f1 = fmt_of<PT>(a.f[1]);
  const bool csr_only = a.closing_csr != 0 || a.f[1].rp == nullptr;
  unsigned long long n_exam = 0;
  while (true) {
    const uint32_t tile = lb_claim(a.lb.counter(), &s_tile);
    if (tile >= ntiles) break;
    const uint64_t n = (uint64_t)tile * FX_T + threadIdx.x;
    uint32_t child = 0;
    bool keep = false;
    if (n < F) {
      const uint32_t b = anc_binding(a, a.par_idx, (uint32_t)n, a.parent_level);
      const uint32_t e = __ldg(fsrc.rp + b + 1);
      uint32_t lo = __ldg(fsrc.rp + b), hi = e;
      while (lo < hi) {  // first entry with label >= l
        const uint32_t m = (lo + hi) >> 1;
        if ((uint32_t)__ldg(fsrc.pred + m) < a.label) lo = m + 1; else hi = m;
      }
      if (lo < e && (uint32_t)__ldg(fsrc.pred + lo) == a.label) {
        child = __ldg(fsrc.col + lo);
        n_exam++;
        keep = bit_of(a.cand, child) && closing_ok1<PT>(a, f0, f1, csr_only, child, (uint32_t)n);
      }
    }
    unsigned long long tot;
    const unsigned long long ex = block_exclusive_scan<unsigned long long>(keep ? 1ull : 0ull, s_red, &tot);
    const uint64_t pref = lb_prefix(a.lb.status, a.lb.epoch(), tile, tot, &s_pref);
    if (pref + tot > a.cap_out) {  // capacity: flag, the host grows and re-runs
      if (threadIdx.x == 0 && tot) atomicOr(a.overflow, 1);
      keep = false;
    }
    if (keep) {
      const uint64_t pos = pref + ex;
      a.out_parent[pos] = (uint32_t)n;
      a.out_bind[pos] = child;
      if (a.out_alive) a.out_alive[pos] = 0;
      for (uint32_t i = 0; i < a.n_anc_out; i++)
        a.out_anc[i][pos] = a.anc_src[i] == ANC_BIND ? __ldg(a.tab.bind[a.k - 1] + n) : __ldg(a.par_anc[a.anc_src[i]] + n);
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) *a.d_nout = pref + tot;
  }
  if (ntiles == 0 && blockIdx.x == 0 && threadIdx.x == 0) *a.d_nout = 0;
  n_exam = __reduce_add_sync(GSM_FULL, (uint32_t)n_exam);
  if ((threadIdx.x & 31) == 0 && n_exam) atomicAdd(a.ctr + C_EXPAND, n_exam);
}

cudaError_t launch_expand_func(const ExpArgs2& a, int pred_bytes, int sm_count, cudaStream_t st) {
  const unsigned g = (unsigned)sm_count * 8;
  if (pred_bytes == 1) pdl_launch(k_expand_func<uint8_t>, g, FX_T, st, a);
  else pdl_launch(k_expand_func<uint16_t>, g, FX_T, st, a);
  return cudaGetLastError();
}

cudaError_t launch_seg_scan(const ExpArgs2& a, int pred_bytes, int sm_count, cudaStream_t st) {
  unsigned g = (unsigned)sm_count * 8;
  // parents per thread: small parent levels want more, shorter tiles (WatDiv-100M
  // batch 4.88 ms at 1 vs 5.07 at 4), levels of tens of millions more work per
  // thread (LUBM-10k batch 7.56 at 4 vs 8.04 at 1); the parent level's capacity
  // (host-known, graph-stable) picks.  GSMART_SS_I forces a value (A/B).
  const char* ev = getenv("GSMART_SS_I");
  const int ssi = ev ? atoi(ev) : (a.cap_par >= (1ull << 23) ? 4 : 1);
  if (ssi == 8) {
    if (pred_bytes == 1) pdl_launch(k_seg_scan<uint8_t, 8>, g, SS_T, st, a);
    else pdl_launch(k_seg_scan<uint16_t, 8>, g, SS_T, st, a);
  } else if (ssi == 1) {
    if (pred_bytes == 1) pdl_launch(k_seg_scan<uint8_t, 1>, g, SS_T, st, a);
    else pdl_launch(k_seg_scan<uint16_t, 1>, g, SS_T, st, a);
  } else if (ssi == 2) {
    if (pred_bytes == 1) pdl_launch(k_seg_scan<uint8_t, 2>, g, SS_T, st, a);
    else pdl_launch(k_seg_scan<uint16_t, 2>, g, SS_T, st, a);
  } else {
    if (pred_bytes == 1) pdl_launch(k_seg_scan<uint8_t, 4>, g, SS_T, st, a);
    else pdl_launch(k_seg_scan<uint16_t, 4>, g, SS_T, st, a);
  }
  return cudaGetLastError();
}

cudaError_t launch_expand_lb(const ExpArgs2& a, int pred_bytes, int sm_count, cudaStream_t st) {
  unsigned g = (unsigned)sm_count * 6;
  const char* ev = getenv("GSMART_EX_T");  // A/B: threads per 1024-entry tile
  const int ext = ev ? atoi(ev) : 256;
  if (ext == 512) {
    g = (unsigned)sm_count * 3;
    if (pred_bytes == 1) pdl_launch(k_expand_lb<uint8_t, 512>, g, 512, st, a);
    else pdl_launch(k_expand_lb<uint16_t, 512>, g, 512, st, a);
  } else if (ext == 1024) {
    g = (unsigned)sm_count * 2;
    if (pred_bytes == 1) pdl_launch(k_expand_lb<uint8_t, 1024>, g, 1024, st, a);
    else pdl_launch(k_expand_lb<uint16_t, 1024>, g, 1024, st, a);
  } else {
    if (pred_bytes == 1) pdl_launch(k_expand_lb<uint8_t, 256>, g, 256, st, a);
    else pdl_launch(k_expand_lb<uint16_t, 256>, g, 256, st, a);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a8 prune + compaction
__global__ void k_phase2_guard(OutTab* ot, const unsigned long long* d_sz, const int* ovf, uint32_t L) {
  GSM_PDL_ENTRY();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int go = *(volatile const int*)ovf == 0;
  for (uint32_t k = 0; k < L; k++) go = go && d_sz[k] <= ot->cap[k];
  if (ot->small_sort && L) go = go && d_sz[L - 1] <= SORT_SMALL_MAXN;
  ot->go = go;
}

cudaError_t launch_phase2_guard(OutTab* ot, const unsigned long long* d_sz, const int* ovf, uint32_t L,
                                cudaStream_t st) {
  return pdl_launch(k_phase2_guard, 1, 32, st, ot, d_sz, ovf, L);
}

__global__ void k_prune_mark_d(const OutTab* __restrict__ ot, const uint32_t* __restrict__ parent,
                               const uint8_t* __restrict__ alive, const unsigned long long* d_n,
                               uint8_t* __restrict__ alive_prev) {
  GSM_PDL_ENTRY();
  if (!ot->go) return;
  const uint64_t n = *d_n;
  for (uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < n; m += (uint64_t)gridDim.x * blockDim.x)
    if (!alive || alive[m]) alive_prev[__ldg(parent + m)] = 1;
}

cudaError_t launch_prune_mark_d(const OutTab* ot, const uint32_t* parent, const uint8_t* alive,
                                const unsigned long long* d_n, uint8_t* alive_prev, int sm_count, cudaStream_t st) {
  pdl_launch(k_prune_mark_d, (unsigned)sm_count * 8, 256, st, ot, parent, alive, d_n, alive_prev);
  return cudaGetLastError();
}

constexpr int CA_T = 256;

template <int CA_I>
__global__ void __launch_bounds__(CA_T) k_compact_alive_lb(const uint32_t* __restrict__ parent,
                                                          const uint32_t* __restrict__ bind,
                                                          const uint8_t* __restrict__ alive,
                                                          const unsigned long long* d_n,
                                                          const uint32_t* __restrict__ newidx_prev,
                                                          const OutTab* __restrict__ ot, uint32_t k,
                                                          uint32_t* __restrict__ newidx,
                                                          unsigned long long* d_count, LBArgs lb) {
  GSM_PDL_ENTRY();
  constexpr int CA_TILE = CA_T * CA_I;
  if (!ot->go) return;
  uint32_t* __restrict__ out_parent = k ? ot->parent[k] : nullptr;
  uint32_t* __restrict__ out_bind = ot->bind[k];
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
                                    const unsigned long long* d_n, const uint32_t* newidx_prev, const OutTab* ot,
                                    uint32_t k, uint32_t* newidx, unsigned long long* d_count, LBArgs lb,
                                    int sm_count, cudaStream_t st) {
  const char* ev = getenv("GSMART_CA_I");  // A/B: nodes per thread
  const int cai = ev ? atoi(ev) : 4;  // 4: measured best (batch 4.67 vs 4.91 ms at 8)
  auto kern = cai == 2 ? k_compact_alive_lb<2> : cai == 4 ? k_compact_alive_lb<4> : k_compact_alive_lb<8>;
  pdl_launch(kern, (unsigned)sm_count * 8, CA_T, st, parent, bind, alive, d_n, newidx_prev, ot, k, newidx, d_count,
             lb);
  return cudaGetLastError();
}

}  // namespace gsm
