// Host-callable launchers of the sm_100a kernels (product code).
#pragma once
#include <cstddef>
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

#include "device.cuh"

namespace gsm {

// Launch with programmatic stream serialization (see GSM_PDL_ENTRY): the kernel
// must begin with GSM_PDL_ENTRY().  Inside a stream capture this becomes a
// programmatic graph edge.
template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
// the same with dynamic shared memory
template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch_smem(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                   Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ----------------------------------------------------------------- scans
// Exclusive scan of n uint32 values (in may alias out).  Writes the 64-bit
// total to *total_dev.  tmp: >= scan_tmp_bytes(n) bytes of device memory.
size_t scan_tmp_bytes(uint64_t n);
cudaError_t scan_exclusive_u32(const uint32_t* in, uint32_t* out, uint64_t n,
                               unsigned long long* total_dev, void* tmp, cudaStream_t st,
                               int* launches);

// ----------------------------------------------------------------- a1 LSpM build
// rows outside [rlo, rhi) are dropped (world > 1: another rank's range)
cudaError_t launch_pack_keys(const uint32_t* rowv, const uint32_t* p, const uint32_t* colv, uint64_t n,
                             const uint8_t* keep, int sh_row, int sh_pred, int drop_bit, uint32_t rlo, uint32_t rhi,
                             uint64_t* keys, cudaStream_t st);
cudaError_t launch_bucket_degree(const uint32_t* s, const uint32_t* p, const uint32_t* o, uint64_t n,
                                 const uint8_t* keep, int shift, unsigned long long* hist, cudaStream_t st);
cudaError_t launch_add_copy(uint32_t* dst, const uint32_t* src, uint64_t n, uint32_t add, cudaStream_t st);
// hand-written onesweep LSD radix sort (radix.cu): sorts by key bits [b0, b1);
// (k0, v0) hold the input, (k1, v1) are same-sized ping-pong buffers; on
// return *in_second says which pair holds the sorted output.  Stable.
// skip_trivial: read the digit histograms on the host (one sync) and skip
// passes whose digit is the same for every key.
size_t radix_tmp_bytes(uint64_t n);
cudaError_t radix_sort_keys_u64(uint64_t* k0, uint64_t* k1, uint64_t n, int b0, int b1, void* tmp, size_t tmp_bytes,
                                cudaStream_t st, int* in_second, int* launches, bool skip_trivial);
cudaError_t radix_sort_pairs_u64_u32(uint64_t* k0, uint64_t* k1, uint32_t* v0, uint32_t* v1, uint64_t n, int b0,
                                     int b1, void* tmp, size_t tmp_bytes, cudaStream_t st, int* in_second,
                                     int* launches, bool skip_trivial, const int* skip = nullptr);
cudaError_t radix_sort_pairs_u32_u64(uint32_t* k0, uint32_t* k1, uint64_t* v0, uint64_t* v1, uint64_t n, int b0,
                                     int b1, void* tmp, size_t tmp_bytes, cudaStream_t st, int* in_second,
                                     int* launches, bool skip_trivial);
cudaError_t launch_unique_flags(const uint64_t* keys, uint64_t n, int drop_bit, uint32_t* flags,
                                cudaStream_t st);
// keys wider than 63 bits (+ drop flag at drop_hi), lo = b:
// mode 0 (LSpM format): hi = a << sh | pred; mode 1 (label-major): hi = pred << sh | a
cudaError_t launch_pack_keys2(const uint32_t* a, const uint32_t* p, const uint32_t* b, uint64_t n, const uint8_t* keep,
                              int mode, int sh, int drop_hi, uint32_t rlo, uint32_t rhi, uint64_t* hi, uint32_t* lo,
                              cudaStream_t st);
cudaError_t launch_unique_flags2(const uint64_t* hi, const uint32_t* lo, uint64_t n, int drop_hi, uint32_t* flags,
                                 cudaStream_t st);
// mode 0: a_out = col, pred, counts per row (sh = pb); mode 1: a_out = s, b_out = o,
// counts per label (sh = nb)
cudaError_t launch_unpack2(const uint64_t* hi, const uint32_t* lo, uint64_t n, const uint32_t* pos, int drop_hi, int sh,
                           int mode, uint32_t* a_out, void* pred, int pred_bytes, uint32_t* b_out, uint32_t* counts,
                           cudaStream_t st);
cudaError_t launch_unpack(const uint64_t* keys, uint64_t n, const uint32_t* pos, int drop_bit, int sh_row,
                          int sh_pred, uint32_t* col, void* pred, int pred_bytes, uint32_t* counts,
                          cudaStream_t st);
cudaError_t launch_heavy_stats(const uint32_t* rp, uint32_t n_rows, unsigned long long* out2,
                               cudaStream_t st);
// label-major entry lists (the per-predicate form of SURVEY §8 a1): keys
// (p << 2nb | s << nb | o), sorted and de-duplicated like the CSR keys, unpacked
// into s/o arrays grouped by label; counts[p] += entries of label p
cudaError_t launch_pack_pso(const uint32_t* s, const uint32_t* p, const uint32_t* o, uint64_t n, const uint8_t* keep,
                            int nb, int drop_bit, uint32_t rlo, uint32_t rhi, uint64_t* keys, cudaStream_t st);
cudaError_t launch_compact_keys(const uint64_t* keys, uint64_t n, const uint32_t* pos, int drop_bit, int nb, int pb,
                                uint64_t* out, cudaStream_t st);
cudaError_t launch_unpack_spo_lm(const uint64_t* keys, uint64_t n, int nb, int pb, uint32_t* ls, uint32_t* lo,
                                 uint32_t* counts, cudaStream_t st, uint64_t* csc_keys = nullptr);
cudaError_t launch_unpack_lm_csc(const uint64_t* keys, uint64_t n, int nb, int pb, uint32_t* col, void* pred,
                                 int pred_bytes, uint32_t* counts, cudaStream_t st);
cudaError_t launch_unpack_pso(const uint64_t* keys, uint64_t n, const uint32_t* pos, int drop_bit, int nb,
                              uint32_t* ls, uint32_t* lo, uint32_t* counts, cudaStream_t st);
// per-row label signature (Fmt::lmask) from row_ptr + pred
// label_rows (optional, n_labels <= 4096; 2 n_labels words): over every 16th row,
// [l] += rows holding label l, [n_labels + l] += its entries (fan-out statistics)
cudaError_t launch_label_mask(const uint32_t* rp, const void* pred, int pred_bytes, uint32_t n_rows,
                              uint32_t* lmask, unsigned long long* label_rows, uint32_t n_labels, cudaStream_t st,
                              uint32_t* nonfunc = nullptr);

// ----------------------------------------------------------------- bitmaps
cudaError_t launch_fill_ones(uint32_t* bm, uint32_t n_words, uint32_t n_bits, cudaStream_t st);
cudaError_t launch_and_inplace(uint32_t* dst, const uint32_t* src, uint32_t n_words, cudaStream_t st);
cudaError_t launch_zero_if_flag(uint32_t* bm, uint64_t n_words, const int* flag, cudaStream_t st);

// ----------------------------------------------------------------- a3 seeds
struct FmtAny {
  const uint32_t* rp;
  const uint32_t* col;
  const void* pred;
  const uint32_t* lmask;
};
template <typename PT>
__host__ __device__ __forceinline__ Fmt<PT> fmt_of(const FmtAny& a) {
  Fmt<PT> f;
  f.rp = a.rp;
  f.col = a.col;
  f.pred = (const PT*)a.pred;
  f.lmask = a.lmask;
  return f;
}

// Change tracking of the candidate bitmaps within one execute: chg[v] = sequence
// number of the last group evaluation that cleared a bit of variable slot v
// (0 = unchanged since the seeds).  A re-evaluation of a group (DESIGN.md
// R-refine) whose neighbour bitmaps are all unchanged since its previous
// evaluation cannot clear anything: its compaction and filter launches exit at
// entry (decided on the device, so the per-plan CUDA graph stays valid).
struct SkipIf {
  uint32_t* chg = nullptr;   // [32] per variable slot (slot counters, zeroed by k_init_cands)
  uint32_t nbr_mask = 0;     // variable slots the group probes
  uint32_t prev = 0;         // sequence of the group's previous evaluation; 0 = never skip
#ifdef __CUDACC__
  __device__ __forceinline__ bool skip() const {
    if (prev == 0) return false;
    uint32_t m = nbr_mask;
    while (m) {
      const int v = __ffs(m) - 1;
      m &= m - 1;
      if (*(volatile const uint32_t*)(chg + v) > prev) return false;
    }
    return true;
  }
#endif
};

// decoupled look-back state of one launch (lookback.cuh).  The epoch is
// device-resident (base of the current launch sequence + this launch's offset)
// so a captured CUDA graph replays with fresh epochs: status words of an
// earlier replay never look valid, and each epoch owns a zeroed tile counter.
struct LBArgs {
  unsigned long long* status;  // epoch-stamped tile status words [cap_tiles]
  uint32_t* counters;          // [LB_EPOCHS] zero until their epoch is used
  const uint32_t* d_epoch;     // base epoch of the launch sequence (device)
  uint32_t off;                // this launch's epoch offset from the base
  uint32_t cap_tiles;
#ifdef __CUDACC__
  __device__ __forceinline__ uint32_t epoch() const { return *(volatile const uint32_t*)d_epoch + off; }
  __device__ __forceinline__ uint32_t* counter() const { return counters + epoch(); }
#endif
};
// world > 1: distance in 32-bit words from this rank's copy of a symmetric
// buffer to rank q's copy (peer address = local + words[q]); world ranks used
constexpr int MAX_WORLD = 8;
struct SymDelta {
  long long words[MAX_WORLD];
};
cudaError_t launch_rank_barrier(unsigned long long* flags_local, const SymDelta& d, uint32_t rank, uint32_t world,
                                const unsigned long long* gen_base, uint32_t gen_off, cudaStream_t st);

// a3: the first seed of every seeded variable in one launch (blockIdx.y = seed)
constexpr uint32_t MAX_SEEDS = 16;
struct SeedBatch {
  FmtAny f[2];
  uint32_t n;
  uint32_t dir[MAX_SEEDS], c[MAX_SEEDS], label[MAX_SEEDS];
  uint32_t* bits[MAX_SEEDS];
};
cudaError_t launch_seed_scatter(const SeedBatch& sb, int pred_bytes, unsigned long long* ctr, int sm_count,
                                cudaStream_t st);
cudaError_t launch_guard(FmtAny f, int pred_bytes, uint32_t s, uint32_t label, uint32_t o, int* flag,
                         cudaStream_t st);

// ----------------------------------------------------------------- a4 grouped incident-edge filter
enum GEdgeMode : uint32_t { GE_PROBE = 0, GE_SELF = 1, GE_CONST = 2 };
struct GEdge {
  const uint32_t* nbr;  // GE_PROBE: neighbour candidate bitmap
  uint32_t label;
  uint32_t mode;        // GE_PROBE: cand_w(col); GE_SELF: col == row (self-loop); GE_CONST: col == cval (seed)
  uint32_t cval;
  uint32_t pad;
};
struct FilterArgs {
  FmtAny f[2];              // CSR (OUT edges), CSC (IN edges)
  GEdge e[2][MAXG];
  uint32_t ne[2];
  uint32_t* cand;           // candidate bitmap of the center, updated in place
  uint32_t n_words;
  uint32_t* heavy_rows;     // records: row | dir << 31
  uint32_t* heavy_chunks;   // records: heavy-row slot, chunk index (2 x uint32)
  uint32_t* heavy_sat;      // per heavy-row slot: OR of satisfied-edge bits
  uint32_t* heavy_count;    // [0] rows, [1] chunks (zero between launches; finalize resets)
  unsigned long long* ctr;
  int heavy;                // launch the heavy-row kernels
  int variant;              // bit0: SIMD label ranges (uint8 labels); bit1: dynamic chunk claiming
  uint32_t word_lo;         // first bitmap word of this rank's range (multiple of 32); n_words = end
  LBArgs claim;             // its counter() is this launch's zeroed chunk counter (dynamic claiming)
  const uint32_t* rows;     // non-null: the center's candidate rows, compacted (row-list path)
  const unsigned long long* d_nrows;  // their count (device)
  SkipIf skip;              // re-evaluation guard
  uint32_t center_slot;     // chg[center_slot] = seq when this launch clears a bit
  uint32_t seq;
  uint32_t world;           // world > 1 (peer exchange): cleared bits and change words go to every rank's copy
  SymDelta peers;           // (cand and chg live in one symmetric region: one delta per rank)
};
// a4, push form of one incident edge (x, l, w, dir): stream the label-major
// entries of l, mark sat_out(x) for every entry whose center row x is a
// candidate (and in sat_in, the previous push edge of the group, if any) and
// whose other end matches (cand_w probe / constant / self-loop)
struct PushArgs {
  const uint32_t* s;
  const uint32_t* o;
  uint64_t beg, end;        // entries of label l: [beg, end)
  uint32_t out;             // 1: center = subject (OUT edge), 0: center = object (IN edge)
  const uint32_t* cand;     // center bitmap
  const uint32_t* sat_in;   // nullptr for the group's first push edge
  uint32_t* sat_out;        // zeroed before the launch
  const unsigned long long* in_cnt;  // marks of the previous push edge (nullptr: first); 0 -> nothing to do
  unsigned long long* out_cnt;       // this edge's marks (zeroed before the launch)
  const uint32_t* nbr;      // GE_PROBE
  uint32_t mode, cval;
  SkipIf skip;
  unsigned long long* ctr;
};
// world > 1 peers for k_and_tracked (the group's push marks AND-ed into cand on every rank)
struct PeerSet {
  uint32_t world;
  SymDelta peers;
};
cudaError_t launch_push_edge(const PushArgs& a, int sm_count, cudaStream_t st);
// cand[0, n_words) &= sat (the group's push edges), change-tracked and skippable like the filter
cudaError_t launch_and_tracked(uint32_t* cand, const uint32_t* sat, uint32_t n_words, SkipIf skip,
                               uint32_t center_slot, uint32_t seq, const PeerSet& ps, cudaStream_t st, int sm_count);

// extra work of the first kernel of an execute (all optional)
struct InitExtra {
  const volatile uint32_t* h_epoch = nullptr;  // pinned host word: the look-back epoch base
  uint32_t* d_epoch = nullptr;
  unsigned long long* zero = nullptr;
  uint32_t n_zero = 0;
  unsigned long long* zero2 = nullptr;
  uint32_t n_zero2 = 0;
  uint32_t* zero32 = nullptr;                      // world > 1: change words in the symmetric region
  uint32_t n_zero32 = 0;
  const volatile unsigned long long* h_bar = nullptr;  // pinned: rank-barrier generation base
  unsigned long long* d_bar = nullptr;
  int* ovf = nullptr;
};
cudaError_t launch_init_cands(uint32_t* cand, uint32_t n_slots, uint32_t stride_words, uint32_t n_bits,
                              uint32_t ones_mask, const InitExtra& x, cudaStream_t st);
cudaError_t launch_group_filter(const FilterArgs& a, int pred_bytes, int sm_count, cudaStream_t st,
                                int* launches);

// ----------------------------------------------------------------- trie tables
struct LevelTab {
  const uint32_t* parent[MAXL];
  const uint32_t* bind[MAXL];
  uint8_t up[MAXL];  // the level parent[k] indexes (trie: k - 1; factorised: the parent occurrence)
};
struct ClosingDev {
  uint32_t label, other_level, dir, self;
};

// ----------------------------------------------------------------- sync-free expansion (expand.cu)
struct ExpArgs2 {
  LevelTab tab;
  uint32_t k;                              // level being built (>= 1)
  const unsigned long long* d_nparent;     // F_{k-1} (device)
  uint64_t cap_par;                        // capacity of parent-side arrays (seg_beg, off)
  int tree;
  uint32_t parent_level, label, dir;
  FmtAny f[2];
  const uint32_t* list;                    // free level: candidate id list
  const unsigned long long* d_list_len;
  const uint32_t* cand;
  ClosingDev cl[MAXC];
  uint32_t ncl;
  uint32_t* seg_beg;                       // [cap_par]
  uint32_t* off;                           // [cap_par + 1]
  uint32_t* tile_start;                    // [lb.cap_tiles]: parent holding each expansion-tile boundary
  unsigned long long* d_T;                 // total entries of level k
  uint32_t* out_parent;
  uint32_t* out_bind;
  uint8_t* out_alive;                      // zeroed for emitted nodes (prune flags), may be null
  uint64_t cap_out;
  unsigned long long* d_nout;              // F_k (device)
  int* overflow;                           // |= 1 capacity (retry), |= 2 fatal (> 2^32 entries)
  unsigned long long* ctr;
  LBArgs lb;
  // materialised ancestor bindings (no parent-pointer walks): a node of level
  // k-1 carries the bindings of the older levels deeper levels still need, in
  // columns par_anc[i]; ANC_BIND = the parent's own binding, ANC_WALK = walk
  int par_idx;                             // the tree edge's parent-level binding
  int cl_idx[MAXC];                        // each closing edge's other-level binding
  const uint32_t* par_anc[MAXANC];
  uint32_t n_anc_out;                      // columns level k carries for its children
  int anc_src[MAXANC];                     // column i of level k: ANC_BIND or an index into par_anc
  uint32_t* out_anc[MAXANC];
  int use_tma;                             // stage tile offsets with cp.async.bulk (off[] has >= 8 words of tail)
  int closing_csr;                         // closing checks read the subject's CSR row (CSR-only or split keep-sets)
  // f2 Ω pre-pruning of a second occurrence: a child c of a node under root
  // binding r is kept only if (r, c) is a node of the variable's first
  // occurrence (open-addressing set of keys r << 32 | c; empty = ~0)
  const unsigned long long* om_tab;
  uint64_t om_mask;
};
// f2: insert the (root binding, binding) key of every node of a level into an
// open-addressing set (capacity om_mask + 1, a power of two, cleared to ~0)
cudaError_t launch_f_hash_build(const LevelTab& tab, uint32_t lev, const unsigned long long* d_n, uint64_t cap,
                                unsigned long long* tab_keys, uint64_t mask, int sm, cudaStream_t st);
__host__ __device__ __forceinline__ uint64_t f_hash(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}
constexpr int ANC_BIND = -1, ANC_WALK = -2;
// ids of set bits of bm[0, n_words) plus id_base
// kernels one launch_bitmap_compact_lb issues (none for an empty range)
inline int compact_launches(uint32_t n_words) { return n_words ? 1 : 0; }
cudaError_t launch_bitmap_compact_lb(const uint32_t* bm, uint32_t n_words, uint32_t* ids, uint64_t cap,
                                     unsigned long long* d_count, int* overflow, LBArgs lb, int sm_count,
                                     cudaStream_t st, uint32_t id_base = 0, SkipIf skip = SkipIf());
cudaError_t launch_seg_scan(const ExpArgs2& a, int pred_bytes, int sm_count, cudaStream_t st);
cudaError_t launch_expand_lb(const ExpArgs2& a, int pred_bytes, int sm_count, cudaStream_t st);
// one launch for a level whose tree-edge label is functional in the parent's format
cudaError_t launch_expand_func(const ExpArgs2& a, int pred_bytes, int sm_count, cudaStream_t st);
struct OutTab;
cudaError_t launch_prune_mark_d(const OutTab* ot, const uint32_t* parent, const uint8_t* alive, const unsigned long long* d_n,
                                uint8_t* alive_prev, int sm_count, cudaStream_t st);
// Where phase 2 writes one execute's output.  Phase-2 kernels read these pointers
// from a device copy of a table the host fills per execute, so a captured phase-2
// graph writes into each result's own memory on every replay.
struct OutTab {
  uint32_t* parent[MAXL];  // compacted level k (parent index into level k-1), k >= 1
  uint32_t* bind[MAXL];    // compacted level k bindings
  uint32_t* rows;          // enumeration output [n_rows x n_cols]
  uint32_t* sorted;        // rank-sort output (rows sorted lexicographically)
  uint32_t* rank;          // rank-sort scratch [SORT_SMALL_MAXN], zeroed by the enumeration
  unsigned long long cap[MAXL];  // nodes of level k the host sized the outputs for
  int go;                  // written by k_phase2_guard: every phase-2 kernel exits at entry when 0
  int small_sort;          // outputs laid out for the rank sort (needs <= SORT_SMALL_MAXN rows)
};
// Phase-2 guard (speculative launch): go = no expansion overflow
// and every level fits the capacity the outputs were sized for.
cudaError_t launch_phase2_guard(OutTab* ot, const unsigned long long* d_sz, const int* ovf, uint32_t L,
                                cudaStream_t st);
constexpr uint32_t SORT_SMALL_MAXN = 8192, SORT_SMALL_MAXC = 16;

cudaError_t launch_compact_alive_lb(const uint32_t* parent, const uint32_t* bind, const uint8_t* alive,
                                    const unsigned long long* d_n, const uint32_t* newidx_prev, const OutTab* ot,
                                    uint32_t k, uint32_t* newidx, unsigned long long* d_count, LBArgs lb,
                                    int sm_count, cudaStream_t st);

// ----------------------------------------------------------------- a8 prune, a9 rows
// one row per leaf; n_last read from device memory (grid-stride)
// the uncompacted last level (its compaction fused into the enumeration): raw
// bindings/parents, the previous level's new indices, where to write its count
struct LastLevel {
  const uint32_t* bind = nullptr;
  const uint32_t* parent = nullptr;
  const uint32_t* newidx_prev = nullptr;
  unsigned long long* d_n_out = nullptr;
  int* sorted = nullptr;  // set to 1 beforehand: cleared if a row is smaller than its predecessor
};
// d_n_last: rows (= nodes of the last level; with lf.bind its uncompacted count)
cudaError_t launch_enumerate(const OutTab* ot, uint32_t n_levels, const uint32_t* col_of_level,
                             const unsigned long long* d_n_last, uint32_t n_cols, int sm_count, cudaStream_t st,
                             LastLevel lf = LastLevel());
// rank sort of ot->rows into ot->sorted for n (device) <= SORT_SMALL_MAXN, n_cols <= SORT_SMALL_MAXC
inline bool sort_small_ok(uint64_t n, uint32_t n_cols) { return n <= SORT_SMALL_MAXN && n_cols <= SORT_SMALL_MAXC; }
cudaError_t sort_rows_small(const OutTab* ot, const unsigned long long* d_n, uint32_t n_cols, cudaStream_t st,
                            int* launches);
size_t sort_rows_tmp_bytes(uint64_t n, uint32_t n_cols);
// rows: [n x n_cols] uint32, distinct, sorted lexicographically into rows_out
// (packed-key LSD radix passes).
// The input must already be ordered on columns [n_key, n_cols) among rows that
// agree on [0, n_key) (n_key = n_cols: no assumption).
// sorted_flag (device int, optional): the rows are first checked for order; if
// already sorted, every sort kernel exits at entry and the rows are copied.
// inplace: the input is in rows_out (rows = scratch of the same size, used only
// when the rows turn out unsorted); needs sorted_flag.
cudaError_t sort_rows(const uint32_t* rows, uint32_t* rows_out, uint64_t n, uint32_t n_cols, uint32_t n_key,
                      int key_bits, void* tmp, size_t tmp_bytes, cudaStream_t st, int* launches,
                      int* sorted_flag = nullptr, bool inplace = false, bool prechecked = false);


// ----------------------------------------------------------------- f2 factorised trees (factorised.cu)
constexpr int MAXOCC = 32;  // occurrences of variables in the factorised tree (= GSMART_MAX_LEVELS)
struct FProbeArgs {         // Ω pruning of one occurrence against the other occurrences of its variable
  const uint32_t* root;     // root binding of each node
  const uint32_t* bind;
  uint8_t* alive;
  uint64_t n;
  uint32_t n_other;
  const unsigned long long* keys[MAXOCC];  // sorted (root, binding) keys of the other occurrences
  uint64_t n_keys[MAXOCC];
};
struct FCountArgs {         // subtree counts of one occurrence from its child occurrences
  const uint8_t* alive;
  uint64_t n;
  uint32_t nch;
  const unsigned long long* P[MAXOCC];  // child occurrence q: exclusive scan of its counts
  const uint32_t* beg[MAXOCC];          // child range of each node of this occurrence
  const uint32_t* end[MAXOCC];
  unsigned long long* out;              // [n + 1]
  LBArgs lb;
  int* overflow;                        // |= 4: a count exceeds 2^46
};
struct FOcc {               // one occurrence, as the enumeration reads it
  const uint32_t* bind;
  const unsigned long long* P;  // exclusive scan of the counts of its nodes
  const uint32_t* beg;          // [n of the parent occurrence]: this occurrence's children of a parent node
  const uint32_t* end;
  int par;                      // parent occurrence (-1 for the root)
  int col;                      // output column, -1 for a second occurrence (Ω)
  int same;                     // Ω: the first occurrence of the same variable, else -1
  int leaf;                     // no child occurrences: every node counts 0 or 1
  int first;                    // the first child occurrence of its parent (splits the parent's index)
};
struct FEnumArgs {
  FOcc o[MAXOCC];
  uint32_t n_occ, n_root, nc;
  unsigned long long total;     // combinations of the pruned trees
  uint32_t* rows;               // [cap_rows x nc]
  uint64_t cap_rows;
  unsigned long long* d_count;  // rows kept (filtered)
  int* overflow;                // |= 8: more rows than cap_rows
  int count_only, filtered;
};
cudaError_t launch_f_fill(uint8_t* a, uint64_t n, uint8_t v, int sm, cudaStream_t st);
cudaError_t launch_f_mark(const uint32_t* parent, const uint8_t* alive, uint64_t n, uint8_t* hc, int sm,
                          cudaStream_t st);
cudaError_t launch_f_and(uint8_t* alive, const uint8_t* hc, uint64_t n, int sm, cudaStream_t st);
cudaError_t launch_f_down(uint8_t* alive, const uint32_t* parent, const uint8_t* alive_par, const uint32_t* root_par,
                          uint32_t* root, uint64_t n, int sm, cudaStream_t st);
cudaError_t launch_f_keys(const uint32_t* root, const uint32_t* bind, const uint8_t* alive, uint64_t n,
                          unsigned long long* keys, int sm, cudaStream_t st);
cudaError_t launch_f_probe(const FProbeArgs& a, int sm, cudaStream_t st);
cudaError_t launch_f_ranges(const uint32_t* parent, uint64_t n, uint32_t* beg, uint32_t* end, int sm,
                            cudaStream_t st);
cudaError_t launch_f_count_scan(const FCountArgs& a, int sm, cudaStream_t st);
cudaError_t launch_f_enum(const FEnumArgs& a, int sm, cudaStream_t st);

}  // namespace gsm
