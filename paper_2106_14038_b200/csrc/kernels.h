// Host-callable launchers of the sm_100a kernels (product code).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "device.cuh"

namespace gsm {

// ----------------------------------------------------------------- scans
// Exclusive scan of n uint32 values (in may alias out).  Writes the 64-bit
// total to *total_dev.  tmp: >= scan_tmp_bytes(n) bytes of device memory.
size_t scan_tmp_bytes(uint64_t n);
cudaError_t scan_exclusive_u32(const uint32_t* in, uint32_t* out, uint64_t n,
                               unsigned long long* total_dev, void* tmp, cudaStream_t st,
                               int* launches);

// ----------------------------------------------------------------- a1 LSpM build
cudaError_t launch_pack_keys(const uint32_t* rowv, const uint32_t* p, const uint32_t* colv, uint64_t n,
                             const uint8_t* keep, int sh_row, int sh_pred, int drop_bit,
                             uint64_t* keys, cudaStream_t st);
size_t sort_keys_tmp_bytes(uint64_t n, int end_bit);
cudaError_t sort_keys_u64(void* tmp, size_t tmp_bytes, const uint64_t* in, uint64_t* out, uint64_t n,
                          int end_bit, cudaStream_t st);
cudaError_t launch_unique_flags(const uint64_t* keys, uint64_t n, int drop_bit, uint32_t* flags,
                                cudaStream_t st);
cudaError_t launch_unpack(const uint64_t* keys, uint64_t n, const uint32_t* pos, int drop_bit, int sh_row,
                          int sh_pred, uint32_t* col, void* pred, int pred_bytes, uint32_t* counts,
                          cudaStream_t st);
cudaError_t launch_heavy_stats(const uint32_t* rp, uint32_t n_rows, unsigned long long* out2,
                               cudaStream_t st);

// ----------------------------------------------------------------- bitmaps
cudaError_t launch_fill_ones(uint32_t* bm, uint32_t n_words, uint32_t n_bits, cudaStream_t st);
cudaError_t launch_and_inplace(uint32_t* dst, const uint32_t* src, uint32_t n_words, cudaStream_t st);
cudaError_t launch_zero_if_flag(uint32_t* bm, uint64_t n_words, const int* flag, cudaStream_t st);

// ----------------------------------------------------------------- a3 seeds
struct FmtAny {
  const uint32_t* rp;
  const uint32_t* col;
  const void* pred;
};
cudaError_t launch_seed_scatter(FmtAny f, int pred_bytes, uint32_t c, uint32_t label, uint32_t* bits,
                                unsigned long long* ctr, int sm_count, cudaStream_t st);
cudaError_t launch_guard(FmtAny f, int pred_bytes, uint32_t s, uint32_t label, uint32_t o, int* flag,
                         cudaStream_t st);

// ----------------------------------------------------------------- a4 grouped incident-edge filter
struct GEdge {
  const uint32_t* nbr;  // neighbour candidate bitmap (unused for self-loops)
  uint32_t label;
  uint32_t self;        // 1: self-loop pattern (entry must have col == row)
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
  uint32_t* heavy_count;    // [0] rows, [1] chunks
  unsigned long long* ctr;
};
cudaError_t launch_group_filter(const FilterArgs& a, int pred_bytes, int sm_count, cudaStream_t st,
                                int* launches);

// ----------------------------------------------------------------- a5 compaction
// bitmap -> ascending id list in two calls sharing tmp: count (total to
// *count_dev) then emit (ids sized from the count).
size_t compact_tmp_bytes(uint32_t n_words);
cudaError_t compact_count(const uint32_t* bm, uint32_t n_words, unsigned long long* count_dev, void* tmp,
                          cudaStream_t st, int* launches);
cudaError_t compact_emit(const uint32_t* bm, uint32_t n_words, uint32_t* ids, void* tmp, cudaStream_t st,
                         int* launches);

// ----------------------------------------------------------------- a6/a7 expansion
struct LevelTab {
  const uint32_t* parent[MAXL];
  const uint32_t* bind[MAXL];
};
struct ClosingDev {
  uint32_t label, other_level, dir, self;
};
struct ExpandArgs {
  LevelTab tab;
  uint32_t k;               // level being built (>= 1); parents are level k-1
  uint32_t n_parents;       // F_{k-1}
  int tree;                 // 1: children = seg_label(dir)(binding at parent_level); 0: children = list
  uint32_t parent_level, label, dir;
  FmtAny f[2];
  const uint32_t* list;     // free level: candidate id list
  uint32_t list_len;
  const uint32_t* cand;     // candidate bitmap of the level's variable
  ClosingDev cl[MAXC];
  uint32_t ncl;
  // work arrays
  uint32_t* seg_beg;        // [n_parents]
  uint32_t* seg_len;        // [n_parents]
  uint32_t* item_off;       // [n_parents] (in: counts, out: exclusive offsets)
  uint32_t* item_node;      // [n_items]
  uint32_t n_items;
  uint32_t* item_cnt;       // [n_items] (count pass; then exclusive offsets)
  uint32_t* out_parent;
  uint32_t* out_bind;
  unsigned long long* ctr;
};
cudaError_t launch_expand_seg(const ExpandArgs& a, int pred_bytes, cudaStream_t st);
cudaError_t launch_items_fill(const ExpandArgs& a, cudaStream_t st);
cudaError_t launch_expand_pass(const ExpandArgs& a, int pred_bytes, bool emit, int sm_count, cudaStream_t st);

// ----------------------------------------------------------------- a8 prune, a9 rows
cudaError_t launch_prune_mark(const uint32_t* parent, const uint8_t* alive, uint32_t n, uint8_t* alive_prev,
                              cudaStream_t st);
cudaError_t launch_u8_to_u32(const uint8_t* in, uint32_t* out, uint32_t n, cudaStream_t st);
cudaError_t launch_compact_level(const uint32_t* parent, const uint32_t* bind, const uint8_t* alive,
                                 const uint32_t* newpos, const uint32_t* newidx_prev, uint32_t n,
                                 uint32_t* out_parent, uint32_t* out_bind, cudaStream_t st);
cudaError_t launch_enumerate(const LevelTab& tab, uint32_t n_levels, const uint32_t* col_of_level,
                             uint32_t n_last, uint32_t n_cols, uint32_t* rows, cudaStream_t st);
size_t sort_rows_tmp_bytes(uint64_t n, uint32_t n_cols);
// rows: [n x n_cols] uint32, sorted lexicographically into rows_out
cudaError_t sort_rows(const uint32_t* rows, uint32_t* rows_out, uint64_t n, uint32_t n_cols, int key_bits,
                      void* tmp, size_t tmp_bytes, cudaStream_t st, int* launches);

}  // namespace gsm
