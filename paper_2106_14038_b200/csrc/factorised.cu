// f2: factorised binding trees (§7.1 tree-based binding storage,
// P:L512-L518; §8.1 local tree-pruning).
//
// The trie of a9 stores every combination of the bindings of a star's leaves
// (a cross product).  The factorised form keeps one level per *occurrence* of
// a variable in the plan's DFS tree: its nodes hang off the nodes of its tree
// parent's occurrence, so sibling branches are stored side by side instead of
// multiplied out.  A pattern closing onto an earlier, non-parent vertex gives
// that vertex's variable a second occurrence (the paper's per-path trees,
// Ex. 7.1), and the common variables Ω are intersected per root binding (§8.1).
//
// Kernels (all grid-stride or look-back, host-known sizes):
//   k_f_fill        alive = 1 (or 0 past the live range)
//   k_f_mark        hc[parent[m]] = 1 for alive children  (a8 bottom-up, per branch)
//   k_f_and         alive &= hc                            (conjunction over branches)
//   k_f_down        alive &= alive[parent], root binding of every node
//   k_f_keys        (root binding, binding) key per alive node of an Ω occurrence
//   k_f_probe       an Ω node survives iff its key is in every other occurrence's sorted keys
//   k_f_ranges      child range [beg, end) of every parent node in one child occurrence
//   k_f_count_scan  subtree counts (product over branches of the children's sums), exclusive scan
//   k_f_enum        combination index -> nodes (mixed radix, per-branch search), Ω equality, row
#include "kernels.h"
#include "lookback.cuh"

namespace gsm {

__global__ void k_f_fill(uint8_t* __restrict__ a, uint64_t n, uint8_t v) {
  GSM_PDL_ENTRY();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

__global__ void k_f_mark(const uint32_t* __restrict__ parent, const uint8_t* __restrict__ alive, uint64_t n,
                         uint8_t* __restrict__ hc) {
  GSM_PDL_ENTRY();
  for (uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < n; m += (uint64_t)gridDim.x * blockDim.x)
    if (alive[m]) hc[__ldg(parent + m)] = 1;  // race-benign byte stores
}

__global__ void k_f_and(uint8_t* __restrict__ alive, const uint8_t* __restrict__ hc, uint64_t n) {
  GSM_PDL_ENTRY();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (!hc[i]) alive[i] = 0;
}

__global__ void k_f_down(uint8_t* __restrict__ alive, const uint32_t* __restrict__ parent,
                         const uint8_t* __restrict__ alive_par, const uint32_t* __restrict__ root_par,
                         uint32_t* __restrict__ root, uint64_t n) {
  GSM_PDL_ENTRY();
  for (uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < n; m += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = __ldg(parent + m);
    if (!alive_par[p]) alive[m] = 0;
    if (root) root[m] = __ldg(root_par + p);
  }
}

__global__ void k_f_keys(const uint32_t* __restrict__ root, const uint32_t* __restrict__ bind,
                         const uint8_t* __restrict__ alive, uint64_t n, unsigned long long* __restrict__ keys) {
  GSM_PDL_ENTRY();
  for (uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < n; m += (uint64_t)gridDim.x * blockDim.x)
    keys[m] = alive[m] ? ((unsigned long long)__ldg(root + m) << 32) | __ldg(bind + m) : ~0ull;
}

__global__ void k_f_probe(FProbeArgs a) {
  GSM_PDL_ENTRY();
  for (uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < a.n; m += (uint64_t)gridDim.x * blockDim.x) {
    if (!a.alive[m]) continue;
    const unsigned long long key = ((unsigned long long)__ldg(a.root + m) << 32) | __ldg(a.bind + m);
    bool ok = true;
    for (uint32_t j = 0; j < a.n_other && ok; j++) {
      const unsigned long long* __restrict__ K = a.keys[j];
      uint64_t lo = 0, hi = a.n_keys[j];
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (__ldg(K + mid) < key) lo = mid + 1; else hi = mid;
      }
      ok = lo < a.n_keys[j] && __ldg(K + lo) == key;
    }
    if (!ok) a.alive[m] = 0;
  }
}

// children of one parent node are contiguous (parent[] non-decreasing, emit order)
__global__ void k_f_ranges(const uint32_t* __restrict__ parent, uint64_t n, uint32_t* __restrict__ beg,
                           uint32_t* __restrict__ end) {
  GSM_PDL_ENTRY();
  for (uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < n; m += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = __ldg(parent + m);
    if (m == 0 || __ldg(parent + m - 1) != p) beg[p] = (uint32_t)m;
    if (m + 1 == n || __ldg(parent + m + 1) != p) end[p] = (uint32_t)(m + 1);
  }
}

constexpr int FC_T = 256, FC_I = 4, FC_TILE = FC_T * FC_I;
constexpr unsigned long long FCOUNT_MAX = LB_VMASK;  // look-back values are 46-bit

// cnt(m) = alive[m] ? prod over child occurrences c of (P_c[end_c[m]] - P_c[beg_c[m]]) : 0
// (a leaf occurrence: alive[m]); out[m] = exclusive prefix, out[n] = total.
__global__ void __launch_bounds__(FC_T) k_f_count_scan(FCountArgs a) {
  GSM_PDL_ENTRY();
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_red[32];
  __shared__ unsigned long long s_pref;
  const uint32_t ntiles = (uint32_t)((a.n + FC_TILE - 1) / FC_TILE);
  while (true) {
    const uint32_t tile = lb_claim(a.lb.counter(), &s_tile);
    if (tile >= ntiles) break;
    const uint64_t base = (uint64_t)tile * FC_TILE + threadIdx.x * FC_I;
    unsigned long long c[FC_I], sum = 0;
#pragma unroll
    for (int j = 0; j < FC_I; j++) {
      const uint64_t m = base + j;
      c[j] = 0;
      if (m < a.n && a.alive[m]) {
        unsigned long long v = 1;
        for (uint32_t q = 0; q < a.nch && v; q++) {
          const uint32_t b = __ldg(a.beg[q] + m), e = __ldg(a.end[q] + m);
          const unsigned long long s = b < e ? __ldg(a.P[q] + e) - __ldg(a.P[q] + b) : 0ull;
          if (s && v > FCOUNT_MAX / s) {
            atomicOr(a.overflow, 4);
            v = FCOUNT_MAX;
          } else {
            v *= s;
          }
        }
        c[j] = v;
      }
      sum += c[j];
    }
    if (sum > FCOUNT_MAX) {
      atomicOr(a.overflow, 4);
      sum = FCOUNT_MAX;
    }
    unsigned long long tot;
    unsigned long long ex = block_exclusive_scan<unsigned long long>(sum, s_red, &tot);
    if (tot > FCOUNT_MAX) tot = FCOUNT_MAX;
    const uint64_t pref = lb_prefix(a.lb.status, a.lb.epoch(), tile, tot, &s_pref);
    unsigned long long run = pref + ex;
#pragma unroll
    for (int j = 0; j < FC_I; j++) {
      const uint64_t m = base + j;
      if (m < a.n) a.out[m] = run;
      run += c[j];
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) a.out[a.n] = pref + tot;
  }
}

// largest i in [lo, hi) with P[i] <= x, given P[lo] <= x < P[hi]: the node whose
// combinations hold x (a node with a zero count never qualifies: its P equals
// the next node's, and the last one is excluded by x < P[hi])
__device__ __forceinline__ uint32_t f_pick(const unsigned long long* __restrict__ P, uint32_t lo, uint32_t hi,
                                           unsigned long long x) {
  uint32_t a = lo + 1, b = hi;  // search (lo, hi) for the first P[i] > x
  while (a < b) {
    const uint32_t m = (a + b) >> 1;
    if (__ldg(P + m) <= x) a = m + 1; else b = m;
  }
  return a - 1;
}

__global__ void __launch_bounds__(256) k_f_enum(const FEnumArgs a) {
  GSM_PDL_ENTRY();
  uint32_t node[MAXOCC];
  unsigned long long rem[MAXOCC], dig[MAXOCC];
  const uint32_t lane = threadIdx.x & 31;
  for (unsigned long long g0 = blockIdx.x * (unsigned long long)blockDim.x + (threadIdx.x & ~31u); g0 < a.total;
       g0 += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long g = g0 + lane;
    bool ok = g < a.total;
    if (ok) {
      node[0] = f_pick(a.o[0].P, 0, a.n_root, g);
      rem[0] = g - __ldg(a.o[0].P + node[0]);
      for (uint32_t o = 1; o < a.n_occ; o++) {
        const FOcc& oc = a.o[o];
        const uint32_t np = node[oc.par];
        if (oc.first) {
          // the parent's combination index splits over its child occurrences with the
          // first one most significant, so rows come out ordered by the occurrences
          // (= the trie's visitation order) and often need no sort: digits are taken
          // from the last child occurrence backwards
          for (int q = (int)a.n_occ - 1; q >= (int)o; q--) {
            if (a.o[q].par != oc.par) continue;
            const uint32_t bq = __ldg(a.o[q].beg + np), eq = __ldg(a.o[q].end + np);
            const unsigned long long Sq = __ldg(a.o[q].P + eq) - __ldg(a.o[q].P + bq);
            dig[q] = rem[oc.par] % Sq;
            rem[oc.par] /= Sq;
          }
        }
        const uint32_t b = __ldg(oc.beg + np), e = __ldg(oc.end + np);
        const unsigned long long base = __ldg(oc.P + b), S = __ldg(oc.P + e) - base;
        const unsigned long long i = dig[o];
        // a leaf occurrence whose children all live (counts 0/1 summing to e - b): direct index
        const uint32_t m = (oc.leaf && S == (unsigned long long)(e - b)) ? b + (uint32_t)i : f_pick(oc.P, b, e, base + i);
        node[o] = m;
        rem[o] = base + i - __ldg(oc.P + m);
      }
      for (uint32_t o = 1; o < a.n_occ && ok; o++)
        if (a.o[o].same >= 0)
          ok = __ldg(a.o[o].bind + node[o]) == __ldg(a.o[a.o[o].same].bind + node[a.o[o].same]);
    }
    unsigned long long idx = g;
    if (a.filtered) {  // Ω equality drops combinations: warp-aggregated append
      const uint32_t bal = __ballot_sync(GSM_FULL, ok);
      unsigned long long wbase = 0;
      if (lane == 0 && bal) wbase = atomicAdd(a.d_count, (unsigned long long)__popc(bal));
      wbase = __shfl_sync(GSM_FULL, wbase, 0);
      idx = wbase + __popc(bal & ((1u << lane) - 1u));
    }
    if (!ok || a.count_only) continue;
    if (idx >= a.cap_rows) {
      atomicOr(a.overflow, 8);
      continue;
    }
    uint32_t* row = a.rows + idx * a.nc;
    for (uint32_t o = 0; o < a.n_occ; o++)
      if (a.o[o].col >= 0) row[a.o[o].col] = __ldg(a.o[o].bind + node[o]);
  }
}

__global__ void k_f_hash_build(const LevelTab tab, uint32_t lev, const unsigned long long* d_n, uint64_t cap,
                               unsigned long long* __restrict__ keys, uint64_t mask) {
  GSM_PDL_ENTRY();
  const uint64_t n = *d_n;
  if (n > cap) return;  // the level overflowed its capacity: the host grows it and re-runs the expansion
  for (uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < n; m += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)m, k = lev;
    while (k != 0) {  // root node of m
      x = __ldg(tab.parent[k] + x);
      k = tab.up[k];
    }
    const unsigned long long key = ((unsigned long long)__ldg(tab.bind[0] + x) << 32) | __ldg(tab.bind[lev] + m);
    uint64_t h = f_hash(key) & mask;
    while (true) {
      const unsigned long long prev = atomicCAS(keys + h, ~0ull, key);
      if (prev == ~0ull || prev == key) break;
      h = (h + 1) & mask;
    }
  }
}

static unsigned grid_for(uint64_t n, int sm_count) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count * 8));
}

cudaError_t launch_f_fill(uint8_t* a, uint64_t n, uint8_t v, int sm, cudaStream_t st) {
  if (!n) return cudaSuccess;
  return pdl_launch(k_f_fill, grid_for(n, sm), 256, st, a, n, v);
}
cudaError_t launch_f_mark(const uint32_t* parent, const uint8_t* alive, uint64_t n, uint8_t* hc, int sm,
                          cudaStream_t st) {
  if (!n) return cudaSuccess;
  return pdl_launch(k_f_mark, grid_for(n, sm), 256, st, parent, alive, n, hc);
}
cudaError_t launch_f_and(uint8_t* alive, const uint8_t* hc, uint64_t n, int sm, cudaStream_t st) {
  if (!n) return cudaSuccess;
  return pdl_launch(k_f_and, grid_for(n, sm), 256, st, alive, hc, n);
}
cudaError_t launch_f_down(uint8_t* alive, const uint32_t* parent, const uint8_t* alive_par, const uint32_t* root_par,
                          uint32_t* root, uint64_t n, int sm, cudaStream_t st) {
  if (!n) return cudaSuccess;
  return pdl_launch(k_f_down, grid_for(n, sm), 256, st, alive, parent, alive_par, root_par, root, n);
}
cudaError_t launch_f_keys(const uint32_t* root, const uint32_t* bind, const uint8_t* alive, uint64_t n,
                          unsigned long long* keys, int sm, cudaStream_t st) {
  if (!n) return cudaSuccess;
  return pdl_launch(k_f_keys, grid_for(n, sm), 256, st, root, bind, alive, n, keys);
}
cudaError_t launch_f_probe(const FProbeArgs& a, int sm, cudaStream_t st) {
  if (!a.n) return cudaSuccess;
  return pdl_launch(k_f_probe, grid_for(a.n, sm), 256, st, a);
}
cudaError_t launch_f_ranges(const uint32_t* parent, uint64_t n, uint32_t* beg, uint32_t* end, int sm,
                            cudaStream_t st) {
  if (!n) return cudaSuccess;
  return pdl_launch(k_f_ranges, grid_for(n, sm), 256, st, parent, n, beg, end);
}
cudaError_t launch_f_count_scan(const FCountArgs& a, int sm, cudaStream_t st) {
  if (!a.n) return cudaMemsetAsync(a.out, 0, 8, st);
  const uint64_t tiles = (a.n + FC_TILE - 1) / FC_TILE;
  if (tiles > a.lb.cap_tiles) return cudaErrorInvalidValue;
  return pdl_launch(k_f_count_scan, (unsigned)std::min<uint64_t>(tiles, (uint64_t)sm * 8), FC_T, st, a);
}
cudaError_t launch_f_hash_build(const LevelTab& tab, uint32_t lev, const unsigned long long* d_n, uint64_t cap,
                                unsigned long long* tab_keys, uint64_t mask, int sm, cudaStream_t st) {
  return pdl_launch(k_f_hash_build, (unsigned)sm * 8, 256, st, tab, lev, d_n, cap, tab_keys, mask);
}
cudaError_t launch_f_enum(const FEnumArgs& a, int sm, cudaStream_t st) {
  if (!a.total) return cudaSuccess;
  const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((a.total + 255) / 256, (uint64_t)sm * 16));
  return pdl_launch(k_f_enum, g, 256, st, a);
}

}  // namespace gsm
