// C-ABI implementation, part 2: the executor (a3-a9; §4 main
// computation + §8 post-processing, re-designed level-synchronous).
//
// An execute runs on one Slot (stream + workspace).  Host work is split into
// phases so that a batch of plans (gsmart_execute_batch) keeps every slot's
// stream busy while the host waits on only two events per plan:
//   start()        seeds -> grouped incident-edge evaluation -> trie expansion,
//                  all asynchronous; sizes are copied to pinned memory + event;
//   after_expand() reads sizes; on a workspace overflow grows it and re-launches
//                  the expansion (rare), else launches phase 2;
//   phase2()       pruning -> level compaction -> rows -> sort (async);
//   finalize()     after the stream drained: alive counts, counters, stats.
#include <chrono>
#include <cstring>
#include <thread>

#include "runtime.h"

using namespace gsm;

namespace gsm {

static gsmart_status slot_init(gsmart_ctx* ctx, Slot& s, bool primary) {
  if (primary) {
    s.st = ctx->st;
  } else {
    CU(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
    s.own_stream = true;
  }
  CU(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
  TRY(dalloc(ctx, &s.lb_status, LB_CAP_TILES, s.st));
  TRY(dalloc(ctx, &s.lb_counters, LB_EPOCHS, s.st));
  TRY(dalloc(ctx, &s.tile_start, LB_CAP_TILES, s.st));
  TRY(dalloc(ctx, &s.d_sz, 128, s.st));
  s.d_ovf = reinterpret_cast<int*>(s.d_sz + 127);  // overflow flags travel with the sizes
  TRY(dalloc(ctx, &s.d_ctr, 64, s.st));
  TRY(dalloc(ctx, &s.heavy_cnt, 4, s.st));
  TRY(dalloc(ctx, &s.d_epoch, 1, s.st));
  TRY(dalloc(ctx, &s.d_bar, 1, s.st));
  CU(cudaMemsetAsync(s.lb_status, 0, (size_t)LB_CAP_TILES * 8, s.st));
  CU(cudaMemsetAsync(s.lb_counters, 0, (size_t)LB_EPOCHS * 4, s.st));
  CU(cudaMemsetAsync(s.heavy_cnt, 0, 16, s.st));
  CU(cudaMallocHost(&s.h_pin, 256 * sizeof(unsigned long long)));
  CU(cudaMallocHost(&s.h_tab, sizeof(OutTab)));
  TRY(dalloc(ctx, &s.d_tab, 1, s.st));
  s.epoch_next = 1;
  return GSMART_OK;
}

static void slot_free(gsmart_ctx* ctx, Slot& s) {
  cudaStream_t st = s.st;
  for (auto& b : s.lv) {
    dfree(ctx, st, b.bind); dfree(ctx, st, b.parent); dfree(ctx, st, b.seg_beg); dfree(ctx, st, b.off); dfree(ctx, st, b.newidx);
    dfree(ctx, st, b.alive);
    for (int i = 0; i < MAXANC; i++) dfree(ctx, st, b.anc[i]);
  }
  for (int k = 0; k < GSMART_MAX_LEVELS; k++) dfree(ctx, st, s.list[k]);
  dfree(ctx, st, s.lb_status); dfree(ctx, st, s.lb_counters); dfree(ctx, st, s.tile_start); dfree(ctx, st, s.d_sz); dfree(ctx, st, s.d_ctr);
  dfree(ctx, st, s.heavy_rows); dfree(ctx, st, s.heavy_chunks); dfree(ctx, st, s.heavy_sat); dfree(ctx, st, s.heavy_cnt);
  dfree(ctx, st, s.frows); dfree(ctx, st, s.sat); dfree(ctx, st, s.d_epoch); dfree(ctx, st, s.p2); dfree(ctx, st, s.d_tab);
  dfree(ctx, st, s.d_bar);
  dfree(ctx, st, s.om);
  if (s.sym.va) {
    cudaStreamSynchronize(st);
    sym_free(ctx, &s.sym);
  } else {
    dfree(ctx, st, s.cand);
  }
  if (s.gath.va) sym_free(ctx, &s.gath);
  for (auto& kv : s.graphs) cudaGraphExecDestroy(kv.second.exec);
  s.graphs.clear();
  cudaStreamSynchronize(st);
  if (s.h_pin) cudaFreeHost(s.h_pin);
  if (s.h_tab) cudaFreeHost(s.h_tab);
  if (s.ev) cudaEventDestroy(s.ev);
  if (s.own_stream) cudaStreamDestroy(s.st);
  (void)ctx;
}

void slots_free(gsmart_ctx* ctx) {
  for (auto& s : ctx->slots) slot_free(ctx, *s);
  ctx->slots.clear();
}

static gsmart_status ensure_slots(gsmart_ctx* ctx, uint32_t n) {
  while (ctx->slots.size() < n) {
    auto s = std::make_unique<Slot>();
    TRY(slot_init(ctx, *s, ctx->slots.empty()));
    ctx->slots.push_back(std::move(s));
  }
  return GSMART_OK;
}

// heavy-row buffers sized from the LSpM's heavy-row statistics
static gsmart_status slot_heavy(gsmart_ctx* ctx, Slot& s) {
  if (s.heavy_gen == ctx->lspm_gen) return GSMART_OK;
  dfree(ctx, s.st, s.heavy_rows); dfree(ctx, s.st, s.heavy_chunks); dfree(ctx, s.st, s.heavy_sat);
  const uint64_t rows = std::max<uint64_t>(ctx->f[0].heavy_rows + ctx->f[1].heavy_rows, 1);
  const uint64_t chunks = std::max<uint64_t>(ctx->f[0].heavy_chunks + ctx->f[1].heavy_chunks, 1);
  TRY(dalloc(ctx, &s.heavy_rows, rows, s.st));
  TRY(dalloc(ctx, &s.heavy_sat, rows, s.st));
  TRY(dalloc(ctx, &s.heavy_chunks, 2 * chunks, s.st));
  CU(cudaMemsetAsync(s.heavy_sat, 0, rows * 4, s.st));
  CU(cudaMemsetAsync(s.heavy_cnt, 0, 8, s.st));
  s.heavy_gen = ctx->lspm_gen;
  s.ws_gen++;
  return GSMART_OK;
}

// Look-back epochs.  An execute is one launch sequence: its look-back launches
// take epochs base + 0, 1, 2, ... where base lives in device memory (set by a
// one-thread kernel), so a captured phase-1 graph replays with fresh epochs.
constexpr uint32_t SEQ_MAX = 8192;  // epochs one execute may use

static gsmart_status begin_seq(gsmart_ctx* ctx, Slot& s) {
  if (s.epoch_next + SEQ_MAX >= LB_EPOCHS) {  // wrap: every status word / counter back to "unused"
    CU(cudaMemsetAsync(s.lb_status, 0, (size_t)LB_CAP_TILES * 8, s.st));
    CU(cudaMemsetAsync(s.lb_counters, 0, (size_t)LB_EPOCHS * 4, s.st));
    s.epoch_next = 1;
  }
  s.seq_base = s.epoch_next;
  s.seq_off = 0;
  s.bar_base = s.bar_next;
  s.bar_off = 0;
  // the sequence's first kernel (k_init_cands) copies them to s.d_epoch / s.d_bar;
  // the slot is idle here (every execute drains its stream before the next one begins)
  reinterpret_cast<volatile uint32_t*>(s.h_pin + H_EPOCH)[0] = s.seq_base;
  reinterpret_cast<volatile unsigned long long*>(s.h_pin)[H_BAR] = s.bar_base;
  return GSMART_OK;
}

// barrier generations only grow (ranks compare flags with >=), look-back epochs wrap
static void end_seq(Slot& s) {
  s.epoch_next = s.seq_base + std::min(s.seq_off, SEQ_MAX);
  s.bar_next = s.bar_base + s.bar_off + 1;
}

// the next look-back launch of the current sequence
static LBArgs next_lb(Slot& s) {
  LBArgs a;
  a.status = s.lb_status;
  a.counters = s.lb_counters;
  a.d_epoch = s.d_epoch;
  a.off = s.seq_off < SEQ_MAX ? s.seq_off++ : SEQ_MAX - 1;
  a.cap_tiles = LB_CAP_TILES;
  return a;
}

static gsmart_status slot_level(gsmart_ctx* ctx, Slot& s, uint32_t k, uint64_t need, uint32_t n_anc = 0) {
  auto& b = s.lv[k];
  if (b.bind && b.cap >= need) {
    for (uint32_t i = 0; i < n_anc; i++)  // ancestor columns this plan needs at level k
      if (!b.anc[i]) {
        TRY(dalloc(ctx, &b.anc[i], b.cap, s.st));
        s.ws_gen++;
      }
    return GSMART_OK;
  }
  uint32_t keep_anc = n_anc;
  for (uint32_t i = 0; i < (uint32_t)MAXANC; i++)
    if (b.anc[i]) keep_anc = std::max(keep_anc, i + 1);
  uint64_t cap = std::max<uint64_t>(need, std::max<uint64_t>(2 * b.cap, 1u << 16));
  cap = (cap + 1023) / 1024 * 1024;
  dfree(ctx, s.st, b.bind); dfree(ctx, s.st, b.parent); dfree(ctx, s.st, b.seg_beg); dfree(ctx, s.st, b.off); dfree(ctx, s.st, b.newidx);
  dfree(ctx, s.st, b.alive);
  for (uint32_t i = 0; i < (uint32_t)MAXANC; i++) dfree(ctx, s.st, b.anc[i]);
  b = Slot::LvBuf();
  for (uint32_t i = 0; i < keep_anc; i++) TRY(dalloc(ctx, &b.anc[i], cap, s.st));
  TRY(dalloc(ctx, &b.bind, cap, s.st));
  TRY(dalloc(ctx, &b.parent, cap, s.st));
  TRY(dalloc(ctx, &b.seg_beg, cap, s.st));
  TRY(dalloc(ctx, &b.off, cap + 8, s.st));  // + 8: 16-byte TMA spans may round past the end
  TRY(dalloc(ctx, &b.newidx, cap, s.st));
  TRY(dalloc(ctx, &b.alive, cap, s.st));
  b.cap = cap;
  s.ws_gen++;
  return GSMART_OK;
}

// grow a plain workspace buffer (moves it: cached graphs of this slot go stale)
template <typename T>
static gsmart_status slot_buf(gsmart_ctx* ctx, Slot& s, T** p, uint64_t* cap, uint64_t need) {
  if (*p && *cap >= need) return GSMART_OK;
  dfree(ctx, s.st, *p);
  *p = nullptr;
  TRY(dalloc(ctx, p, need, s.st));
  *cap = need;
  s.ws_gen++;
  return GSMART_OK;
}

}  // namespace gsm

namespace {

struct Prof {
  cudaStream_t st;
  gsmart_stats* stats;
  bool on;
  struct Rec { int kid; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  int cur = -1;
  cudaEvent_t cur_a = nullptr;
  Prof(cudaStream_t s, gsmart_stats* r, bool enable) : st(s), stats(r), on(enable) {}
  void begin(int kid) {
    if (!on) return;
    cur = kid;
    cudaEventCreate(&cur_a);
    cudaEventRecord(cur_a, st);
  }
  void end() {
    if (!on || cur < 0) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, st);
    recs.push_back({cur, cur_a, b});
    cur = -1;
  }
  void flush() {  // after the stream drained
    for (auto& r : recs) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) stats->ms_kernel[r.kid] += ms;
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    recs.clear();
  }
  ~Prof() { flush(); }
};

struct Exec {
  enum State { S_NEW, S_EXPANDING, S_PHASE2, S_DONE };
  gsmart_ctx* ctx;
  Slot& sl;
  const gsmart_plan_t* plan;
  uint32_t flags;
  gsmart_result* R;
  Prof prof;
  Scratch sc;
  State state = S_NEW;
  uint32_t W = 0, Wpad = 0, L = 0;
  std::vector<int32_t> slot;  // vertex -> cand slot
  FmtAny fa[2];
  int launches[GSMART_NKERNELS] = {0};
  uint64_t filter_main = 0;  // main group-filter launches (one bitmap pass each)
  uint32_t filter_seq = 0;             // group evaluations issued so far (SkipIf sequence)
  std::vector<std::vector<GroupEdge>> gedges;  // per group: its edges, then its back edges (Eq. 16)
  // per trie level k: the older levels (< k) whose bindings deeper levels read
  // (tree-edge parents, closing-edge targets), carried as columns by level k's
  // nodes — at most MAXANC, the rest are found by walking parent pointers
  std::vector<std::vector<uint32_t>> anc_cols;
  void plan_ancestors() {
    anc_cols.assign(L, {});
    std::vector<std::vector<uint32_t>> need(L);
    for (uint32_t k = 1; k < L; k++) {
      const Level& Lv = plan->levels[k];
      if (Lv.tree_edge >= 0) need[k].push_back(Lv.parent_level);
      for (auto& c : Lv.closing)
        if (c.other_level != k) need[k].push_back(c.other_level);
    }
    for (uint32_t k = 1; k < L; k++) {
      std::vector<uint32_t> cols;
      for (uint32_t kk = k + 1; kk < L; kk++)
        for (uint32_t j : need[kk])
          if (j < k && std::find(cols.begin(), cols.end(), j) == cols.end()) cols.push_back(j);
      std::sort(cols.begin(), cols.end());
      // a column of level k must be derivable from level k-1: its own binding or its column
      std::vector<uint32_t> ok;
      for (uint32_t j : cols)
        if ((j == k - 1 || std::find(anc_cols[k - 1].begin(), anc_cols[k - 1].end(), j) != anc_cols[k - 1].end()) &&
            ok.size() < (size_t)MAXANC)
          ok.push_back(j);
      anc_cols[k] = ok;
    }
  }
  // where expanding level k (parent level k-1) finds the binding of level j
  int anc_index(uint32_t k, uint32_t j) const {
    if (j == k - 1) return ANC_BIND;
    const auto& c = anc_cols[k - 1];
    auto it = std::find(c.begin(), c.end(), j);
    return it == c.end() ? ANC_WALK : (int)(it - c.begin());
  }
  std::vector<std::vector<uint8_t>> push_dec;  // per group, per edge of gedges: push form (label-major)
  uint64_t push_and = 0;               // k_and_tracked launches (bitmap bytes)
  uint64_t n_exchanges = 0;            // candidate-bitmap exchanges (world > 1: one per group evaluation)
  std::vector<uint32_t> group_seq;     // per group: sequence of its last evaluation
  int attempts = 0;
  bool seq_open = false;        // a look-back launch sequence was started (end it in finalize)
  bool graph_replayed = false;  // phase 1 came from the plan's cached CUDA graph
  bool ctr_pinned = false;      // counters already copied to sl.h_pin[192..) on the stream
  uint32_t wlo = 0, whi = 0;  // this rank's bitmap words (1-D vertex-range partition)
  bool identity = false;                 // trie order == column order: rows come out sorted
  std::vector<uint64_t> F;
  std::chrono::steady_clock::time_point t0;
  int smc;  // SMs this execute sizes its grids for (a share of the device when a batch runs concurrently)

  // ---- f2: factorised binding trees (GSMART_FACTORISED; §7.1, §8.1).
  // One level per occurrence of a variable: the trie level's variable hangs off
  // its tree parent's occurrence (not off the previous trie level), and each
  // closing pattern onto a non-parent earlier level adds a second occurrence of
  // the variable under that level (the paper's per-path trees: a variable on
  // two paths, Ω).  Self-loops and patterns parallel to the tree edge stay
  // closing checks of the occurrence (target = the parent binding).
  struct Occ {
    uint32_t var = 0;
    int par = -1;       // parent occurrence (-1: root)
    bool tree = true;   // false: a free level (children = the candidate list), under the root
    uint32_t label = 0, dir = 0;  // tree edge; dir seen from the parent (OUT: the parent is the subject)
    std::vector<ClosingDev> cl;
    std::vector<int> cl_idx;
    int col = -1;       // output column (first occurrence), -1 for a second occurrence
    int same = -1;      // second occurrence: the first occurrence of its variable
  };
  bool fact = false;
  std::vector<Occ> occ;
  std::vector<uint8_t> fused_lv;  // per level: expanded by the fused functional kernel
  uint32_t n_omega = 0;
  std::vector<uint64_t> om_off, om_mask;  // per occurrence: its key set in sl.om (second occurrences only)
  // key sets of the first occurrences, one per second occurrence, sized for the
  // first occurrence's level capacity (load factor <= 1/2)
  gsmart_status ensure_om() {
    om_off.assign(L, 0);
    om_mask.assign(L, 0);
    uint64_t total = 0;
    for (uint32_t o = 0; o < L; o++) {
      if (occ[o].same < 0) continue;
      uint64_t c = 1024;
      while (c < 2 * sl.lv[occ[o].same].cap) c <<= 1;
      om_off[o] = total;
      om_mask[o] = c - 1;
      total += c;
    }
    if (total) TRY(slot_buf(ctx, sl, &sl.om, &sl.om_cap, total));
    return GSMART_OK;
  }
  gsmart_status build_occurrences() {
    const uint32_t LT = (uint32_t)plan->levels.size();
    std::vector<int> of_var(plan->n_vertices, -1);
    std::vector<int> center_of(plan->edges.size(), -1);  // the group that evaluated each pattern
    for (auto& g : plan->groups)
      for (auto& e : g.edges) center_of[e.edge] = (int)g.center;
    occ.clear();
    n_omega = 0;
    // (center, other variable) -> the patterns between them that close onto a non-parent level
    std::map<std::pair<uint32_t, uint32_t>, std::vector<uint32_t>> cross;
    auto is_anc = [&](int from, int a) {  // occurrence a on the path from `from` up to the root
      for (int x = from; x >= 0; x = occ[x].par)
        if (x == a) return true;
      return false;
    };
    for (uint32_t k = 0; k < LT; k++) {
      const Level& Lv = plan->levels[k];
      Occ o;
      o.var = Lv.var;
      o.col = plan->col_of[Lv.var];
      o.tree = k > 0 && Lv.tree_edge >= 0;
      const uint32_t plev = o.tree ? Lv.parent_level : 0;
      if (k > 0) {
        o.par = of_var[plan->levels[plev].var];
        o.label = Lv.label;
        o.dir = Lv.dir;
      }
      for (auto& c : Lv.closing) {
        if (c.other_level == k) {
          if (k > 0) {  // the root level's self-loops are exact in its candidate set
            o.cl.push_back({c.label, k, c.dir == OUT ? 0u : 1u, 1u});
            o.cl_idx.push_back(ANC_WALK);
          }
        } else if (k > 0 && c.other_level == plev) {
          o.cl.push_back({c.label, plev, c.dir == OUT ? 0u : 1u, 0u});
          o.cl_idx.push_back(ANC_BIND);
        } else if (k > 0 && is_anc(o.par, of_var[plan->levels[c.other_level].var])) {
          // onto an older level on this node's own root path: checked during expansion
          // (a walk up the parent occurrences), no second occurrence needed
          o.cl.push_back({c.label, (uint32_t)of_var[plan->levels[c.other_level].var], c.dir == OUT ? 0u : 1u, 0u});
          o.cl_idx.push_back(ANC_WALK);
        } else {
          // the path of the pattern's center continues to the other endpoint (P:L516,
          // Ex. 7.1 "v2 -> v0 -> v1"): a second occurrence of that variable under the center
          const uint32_t other = plan->levels[c.other_level].var;
          const int ctr = center_of[c.edge] >= 0 ? center_of[c.edge] : (int)other;
          const uint32_t dupv = (uint32_t)ctr == Lv.var ? other : Lv.var;
          cross[{(uint32_t)ctr, dupv}].push_back(c.edge);
        }
      }
      of_var[Lv.var] = (int)occ.size();
      occ.push_back(o);
    }
    for (auto& kv : cross) {
      const uint32_t ctr = kv.first.first, v = kv.first.second;
      Occ d;
      d.var = v;
      d.par = of_var[ctr];
      const gsmart_qedge& e0 = plan->edges[kv.second[0]];
      d.label = e0.pred;
      d.dir = e0.src == ctr ? (uint32_t)OUT : (uint32_t)IN;  // seen from the center
      for (size_t i = 1; i < kv.second.size(); i++) {
        const gsmart_qedge& e = plan->edges[kv.second[i]];
        d.cl.push_back({e.pred, (uint32_t)d.par, e.src == v ? 0u : 1u, 0u});  // seen from the new child
        d.cl_idx.push_back(ANC_BIND);
      }
      d.same = of_var[v];
      occ.push_back(d);
      n_omega++;
    }
    if (occ.size() > (size_t)MAXOCC || occ.size() > (size_t)GSMART_MAX_LEVELS)
      FAIL(GSMART_E_UNSUPPORTED, "GSMART_FACTORISED: more than 32 occurrences");
    // a second occurrence reads its center's row in the pattern's direction, which
    // the trie never does: that format must hold the label (keep-sets, CSR-only)
    for (size_t o = 1; o < occ.size(); o++) {
      if (!occ[o].tree) continue;
      const int fmt = occ[o].dir == OUT ? 0 : 1;
      const auto& kp = ctx->keep[fmt];
      if (!ctx->f[fmt].built || (occ[o].label < kp.size() && !kp[occ[o].label]))
        FAIL(GSMART_E_STATE, std::string("GSMART_FACTORISED: the ") + (fmt ? "CSC" : "CSR") +
                                 " LSpM does not hold predicate " + std::to_string(occ[o].label) +
                                 " that an occurrence expands over (build it with that label)");
    }
    return GSMART_OK;
  }

  Exec(gsmart_ctx* c, Slot& s, const gsmart_plan_t* p, uint32_t fl, gsmart_result* r)
      : ctx(c), sl(s), plan(p), flags(fl), R(r), prof(s.st, &r->stats, (fl & GSMART_PROFILE) != 0), sc(c, s.st),
        smc(c->sm_count) {
    t0 = std::chrono::steady_clock::now();
  }

  // candidate bitmaps live in the slot (stable addresses for graph replay);
  // GSMART_KEEP_CANDIDATES copies them into the result at the end
  uint32_t* cand(uint32_t vertex) { return sl.cand + (uint64_t)slot[vertex] * Wpad; }

  // world > 1 with the peer exchange: bitmaps and change words are symmetric,
  // filters update every rank's copy, a device barrier ends each group
  bool peer_mode() const { return ctx->world > 1 && ctx->exchange == GSMART_XCHG_PEER; }
  SymDelta peer_delta() const {
    SymDelta d{};
    if (peer_mode()) d = sl.sym.delta(ctx->world);
    return d;
  }
  uint32_t peer_world() const { return peer_mode() ? (uint32_t)ctx->world : 1u; }
  uint32_t* chg_words() {
    return peer_mode() ? sl.cand + sl.sym_cand_words : reinterpret_cast<uint32_t*>(sl.d_ctr + 16);
  }
  // Ranks that are threads of one process share one CUDA context, and streams of
  // one context share a few hardware queues (CUDA_DEVICE_MAX_CONNECTIONS): a
  // spinning barrier kernel at the head of a queue would block another rank's
  // kernels queued behind it.  Those ranks synchronise on the host instead (and
  // run without graphs); ranks that are processes (one context each, the
  // deployment layout) use the device barrier.
  bool host_barriers() const { return ctx->world > 1 && ctx->lcomm != nullptr; }
  gsmart_status rank_barrier() {
    if (host_barriers()) {
      prof.begin(K_COLLECTIVE);
      CU(cudaStreamSynchronize(sl.st));
      TRY(host_barrier(ctx));
      prof.end();
      ++sl.bar_off;
      launches[K_COLLECTIVE]++;
      return GSMART_OK;
    }
    unsigned long long* flags = reinterpret_cast<unsigned long long*>(sl.cand + sl.sym_cand_words + 32);
    prof.begin(K_COLLECTIVE);
    CU(launch_rank_barrier(flags, peer_delta(), (uint32_t)ctx->rank, (uint32_t)ctx->world, sl.d_bar, ++sl.bar_off,
                           sl.st));
    prof.end();
    launches[K_COLLECTIVE]++;
    return GSMART_OK;
  }
  // label-major list of an edge's center side (world > 1: OUT -> this rank's
  // subjects, IN -> this rank's objects stored as (o, s))
  const LabelMajor& lm_for(const GroupEdge& e) const {
    return (ctx->world > 1 && e.dir == IN) ? ctx->lm_in : ctx->lm;
  }

  gsmart_status alloc_result(void** p, uint64_t bytes) {
    TRY(dalloc(ctx, (char**)p, bytes, sl.st));
    R->owned.push_back(*p);
    return GSMART_OK;
  }

  // ---- a3: seeds (light edges) and guards.  The first seed of a variable is
  // scattered into its bitmap; further seeds become constant-target filter edges.
  // A constant id >= N is an entity absent from the data (R12): its segments are
  // empty, so a seed from it empties its variable's candidate set (no scatter)
  // and a guard on it is false.
  gsmart_status seeds_and_guards() {
    const uint32_t N = ctx->N;
    std::vector<std::vector<const Seed*>> by_var(plan->n_vertices);
    for (auto& sd : plan->seeds) by_var[sd.var].push_back(&sd);
    uint32_t ones = 0;
    for (uint32_t v : plan->vars)
      if (by_var[v].empty()) ones |= 1u << slot[v];
    if (!plan->vars.empty()) {
      InitExtra x;
      x.h_epoch = reinterpret_cast<const volatile uint32_t*>(sl.h_pin + H_EPOCH);
      x.d_epoch = sl.d_epoch;
      x.zero = sl.d_ctr;  // counters
      x.n_zero = 32;  // counters [0, C_NCTR) and the SkipIf change words at [16, 32)
      x.zero2 = sl.d_sz;  // expansion sizes
      x.n_zero2 = 128;
      x.ovf = sl.d_ovf;
      x.h_bar = reinterpret_cast<const volatile unsigned long long*>(sl.h_pin + H_BAR);
      x.d_bar = sl.d_bar;
      if (peer_mode()) {
        x.zero32 = chg_words();
        x.n_zero32 = 32;
      }
      prof.begin(K_BITMAP);
      CU(launch_init_cands(sl.cand, (uint32_t)plan->vars.size(), Wpad, N, ones, x, sl.st));
      launches[K_BITMAP]++;
      prof.end();
    }
    int* flag = (int*)(sl.d_ctr + 48);
    if (!plan->guards.empty()) {
      bool absent = false;
      for (auto& g : plan->guards) absent = absent || g.s >= N || g.o >= N;
      CU(cudaMemsetAsync(flag, absent ? 0 : 0xff, 4, sl.st));  // nonzero = guards hold
      prof.begin(K_SEED);
      for (auto& g : plan->guards) {
        if (absent) break;
        CU(launch_guard(fa[0], ctx->pred_bytes, g.s, g.label, g.o, flag, sl.st));
        launches[K_SEED]++;
      }
      prof.end();
    }
    SeedBatch sb;
    memset(&sb, 0, sizeof sb);
    sb.f[0] = fa[0];
    sb.f[1] = fa[1];
    for (uint32_t v : plan->vars) {
      const auto& ss = by_var[v];
      if (ss.empty() || ss[0]->cid >= N) continue;  // absent constant: the zeroed bitmap is the seed
      if (sb.n == MAX_SEEDS) FAIL(GSMART_E_UNSUPPORTED, "more than 16 seeded variables");
      sb.dir[sb.n] = ss[0]->dir == OUT ? 0 : 1;
      sb.c[sb.n] = ss[0]->cid;
      sb.label[sb.n] = ss[0]->label;
      sb.bits[sb.n] = cand(v);
      sb.n++;
    }
    if (sb.n) {
      prof.begin(K_SEED);
      CU(launch_seed_scatter(sb, ctx->pred_bytes, sl.d_ctr, smc, sl.st));
      launches[K_SEED]++;
      prof.end();
    }
    for (uint32_t v : plan->vars) {
      const auto& ss = by_var[v];
      if (ss.size() > 1) {
        // (c -l-> v): v's CSC row must hold (l, c); (v -l-> c): v's CSR row must hold (l, c)
        Group g;
        g.center = v;
        for (size_t i = 1; i < ss.size(); i++)  // an absent constant (>= N) matches no column
          g.edges.push_back({ss[i]->edge, ss[i]->label, ss[i]->dir == OUT ? (uint32_t)IN : (uint32_t)OUT,
                             0x80000000u | std::min(ss[i]->cid, N)});
        TRY(eval_group(g, SIZE_MAX));  // constant-target filter edges: evaluated once
      }
    }
    if (!plan->guards.empty() && !plan->vars.empty()) {
      prof.begin(K_BITMAP);
      CU(launch_zero_if_flag(sl.cand, (uint64_t)Wpad * plan->vars.size(), flag, sl.st));
      launches[K_BITMAP]++;
      prof.end();
    }
    return GSMART_OK;
  }

  // ---- a4: grouped incident-edge evaluation of one group (§5 Eqs. 17/21).
  // nbr with bit 31 set = constant target (extra seed).
  gsmart_status eval_group(const Group& g, size_t gi) {
    std::vector<const GroupEdge*> by[2], push;
    const std::vector<uint8_t>* dec = gi < push_dec.size() ? &push_dec[gi] : nullptr;
    const std::vector<GroupEdge>& GE = gi < gedges.size() ? gedges[gi] : g.edges;
    for (size_t ei = 0; ei < GE.size(); ei++) {
      const GroupEdge& e = GE[ei];
      if (dec && (*dec)[ei]) push.push_back(&e);
      else by[e.dir == OUT ? 0 : 1].push_back(&e);
    }
    // cheapest (and most selective) label first: later edges only mark rows that
    // passed the earlier ones, and stop at once when none did
    auto lm_size = [&](const GroupEdge* e) {
      const LabelMajor& L = lm_for(*e);
      return L.off[e->label + 1] - L.off[e->label];
    };
    std::stable_sort(push.begin(), push.end(),
                     [&](const GroupEdge* x, const GroupEdge* y) { return lm_size(x) < lm_size(y); });
    // change tracking (SkipIf): a re-evaluation is skipped on the device when no
    // neighbour bitmap changed since this group's previous evaluation (world == 1)
    const uint32_t seq = ++filter_seq;
    SkipIf sk;
    sk.chg = chg_words();
    const uint32_t prev = gi < group_seq.size() ? group_seq[gi] : 0u;
    if (prev && (ctx->world == 1 || peer_mode())) {
      sk.prev = prev;
      for (auto& e : GE)
        if (!(e.nbr & 0x80000000u) && e.nbr != g.center) sk.nbr_mask |= 1u << slot[e.nbr];
    }
    if (gi < group_seq.size()) group_seq[gi] = seq;
    if (!push.empty()) {
      // push form (label-major streaming) of the chosen edges: each marks the rows
      // that also passed the previous one, the last mark set is AND-ed into cand_x
      const uint32_t* prev_sat = nullptr;
      prof.begin(K_FILTER);
      for (size_t i = 0; i < push.size(); i++) {
        const GroupEdge* e = push[i];
        const LabelMajor& lm = lm_for(*e);
        const bool center_first = e->dir == OUT || ctx->world > 1;  // lm_in stores (o, s)
        uint32_t* out = sl.sat + (i & 1) * (uint64_t)Wpad;
        unsigned long long* cnt = sl.d_ctr + 32 + (i & 1);
        CU(cudaMemsetAsync(out, 0, (size_t)W * 4, sl.st));
        CU(cudaMemsetAsync(cnt, 0, 8, sl.st));
        PushArgs pa;
        memset(&pa, 0, sizeof pa);
        pa.s = lm.s;
        pa.o = lm.o;
        pa.beg = lm.off[e->label];
        pa.end = lm.off[e->label + 1];
        pa.out = center_first ? 1u : 0u;
        pa.cand = cand(g.center);
        pa.sat_in = prev_sat;
        pa.sat_out = out;
        pa.in_cnt = prev_sat ? sl.d_ctr + 32 + ((i + 1) & 1) : nullptr;
        pa.out_cnt = cnt;
        if (e->nbr & 0x80000000u) {
          pa.mode = GE_CONST;
          pa.cval = e->nbr & 0x7fffffffu;
        } else if (e->nbr == g.center) {
          pa.mode = GE_SELF;
        } else {
          pa.mode = GE_PROBE;
          pa.nbr = cand(e->nbr);
        }
        pa.skip = sk;
        pa.ctr = sl.d_ctr;
        CU(launch_push_edge(pa, smc, sl.st));
        launches[K_FILTER]++;
        prev_sat = out;
      }
      PeerSet ps;
      ps.world = peer_world();
      ps.peers = peer_delta();
      CU(launch_and_tracked(cand(g.center) + wlo, prev_sat + wlo, whi - wlo, sk, (uint32_t)slot[g.center], seq, ps,
                            sl.st, smc));
      launches[K_FILTER]++;
      push_and++;
      prof.end();
    }
    if (!by[0].empty() || !by[1].empty()) TRY(eval_pull(g, by, sk, seq));
    return exchange_center(g);
  }

  // pull form of a group's remaining edges (row filter over the center's candidate rows)
  gsmart_status eval_pull(const Group& g, std::vector<const GroupEdge*> (&by)[2], const SkipIf& sk, uint32_t seq) {
    size_t done[2] = {0, 0};
    // row-list path: compact the center's candidate rows of this rank once per group
    const bool rowlist = (ctx->filter_variant & 4) != 0;
    unsigned long long* d_nrows = sl.d_ctr + 56;
    if (rowlist) {  // sl.frows sized in ensure_workspace()
      prof.begin(K_COMPACT);
      CU(cudaMemsetAsync(d_nrows, 0, 8, sl.st));
      CU(launch_bitmap_compact_lb(cand(g.center) + wlo, whi > wlo ? whi - wlo : 0, sl.frows, sl.frows_cap, d_nrows,
                                  sl.d_ovf, next_lb(sl), smc, sl.st, wlo * 32, sk));
      launches[K_COMPACT] += compact_launches(whi > wlo ? whi - wlo : 0);
      prof.end();
    }
    while (done[0] < by[0].size() || done[1] < by[1].size()) {
      FilterArgs a;
      memset(&a, 0, sizeof a);
      a.f[0] = fa[0];
      a.f[1] = fa[1];
      for (int d = 0; d < 2; d++) {
        while (done[d] < by[d].size() && a.ne[d] < (uint32_t)MAXG) {
          const GroupEdge* e = by[d][done[d]++];
          GEdge& ge = a.e[d][a.ne[d]++];
          ge.label = e->label;
          if (e->nbr & 0x80000000u) {
            ge.mode = GE_CONST;
            ge.cval = e->nbr & 0x7fffffffu;
          } else if (e->nbr == g.center) {
            ge.mode = GE_SELF;
          } else {
            ge.mode = GE_PROBE;
            ge.nbr = cand(e->nbr);
          }
        }
        if (a.ne[d] && ctx->f[d].heavy_rows) a.heavy = 1;
      }
      a.cand = cand(g.center);
      a.word_lo = wlo & ~31u;
      a.n_words = whi > wlo ? whi : 0;  // this rank's rows only (world > 1)
      a.heavy_rows = sl.heavy_rows;
      a.heavy_chunks = sl.heavy_chunks;
      a.heavy_sat = sl.heavy_sat;
      a.heavy_count = sl.heavy_cnt;
      a.ctr = sl.d_ctr;
      a.variant = ctx->filter_variant;
      a.claim = next_lb(sl);  // its counter() is fresh and zeroed: no reset launch
      a.skip = sk;
      a.center_slot = (uint32_t)slot[g.center];
      a.seq = seq;
      a.world = peer_world();
      a.peers = peer_delta();
      if (rowlist) {
        a.rows = sl.frows;
        a.d_nrows = d_nrows;
      }
      prof.begin(K_FILTER);
      CU(launch_group_filter(a, ctx->pred_bytes, smc, sl.st, &launches[K_FILTER]));
      prof.end();
      filter_main++;
    }
    return GSMART_OK;
  }

  // world > 1: every rank needs the whole candidate bitmap of the center.  Peer
  // exchange: the filter already cleared the bits on every rank's copy; a device
  // barrier orders them before anyone reads.  NCCL / in-process copies (the
  // baseline): an all-gather of the ranks' slices (variable sizes).
  gsmart_status exchange_center(const Group& g) {
    if (ctx->world == 1 && !ctx->comm) return GSMART_OK;
    n_exchanges++;
    if (peer_mode()) return rank_barrier();
    prof.begin(K_COLLECTIVE);
    TRY(coll_allgatherv(ctx, sl.st, cand(g.center)));
    prof.end();
    launches[K_COLLECTIVE]++;
    return GSMART_OK;
  }

  // ---- a5/a6/a7: one expansion attempt over all levels (async), sizes -> pinned
  // fresh: sizes and overflow flags were zeroed by this execute's k_init_cands
  gsmart_status launch_expansion(bool fresh) {
    if (fact) return launch_expansion_f(fresh);
    unsigned long long* dsz = sl.d_sz;
    if (!fresh) CU(cudaMemsetAsync(dsz, 0, 128 * 8, sl.st));
    if (L > 1) CU(cudaMemsetAsync(sl.lv[0].alive, 0, sl.lv[0].cap, sl.st));
    prof.begin(K_COMPACT);
    // level 0 = this rank's root candidates (its word range; all of them when world == 1)
    CU(launch_bitmap_compact_lb(cand(plan->levels[0].var) + wlo, whi - wlo, sl.lv[0].bind, sl.lv[0].cap, dsz + 0,
                                sl.d_ovf, next_lb(sl), smc, sl.st, wlo * 32));
    launches[K_COMPACT] += compact_launches(whi - wlo);
    prof.end();
    for (uint32_t k = 1; k < L; k++) {
      const Level& Lv = plan->levels[k];
      ExpArgs2 a;
      memset(&a, 0, sizeof a);
      for (uint32_t j = 0; j < k; j++) {
        a.tab.parent[j] = sl.lv[j].parent;
        a.tab.bind[j] = sl.lv[j].bind;
        a.tab.up[j] = (uint8_t)(j ? j - 1 : 0);
      }
      a.k = k;
      a.d_nparent = dsz + (k - 1);
      a.cap_par = sl.lv[k - 1].cap;
      a.tree = Lv.tree_edge >= 0 ? 1 : 0;
      a.parent_level = Lv.parent_level;
      a.label = Lv.label;
      a.dir = Lv.dir == OUT ? 0 : 1;
      a.f[0] = fa[0];
      a.f[1] = fa[1];
      a.cand = cand(Lv.var);
      for (auto& c : Lv.closing) {
        a.cl_idx[a.ncl] = c.other_level == k ? ANC_WALK : anc_index(k, c.other_level);
        ClosingDev& d = a.cl[a.ncl++];
        d.label = c.label;
        d.other_level = c.other_level;
        d.dir = c.dir == OUT ? 0 : 1;
        d.self = c.other_level == k ? 1u : 0u;
      }
      a.par_idx = a.tree ? anc_index(k, Lv.parent_level) : ANC_WALK;
      // closing checks in the subject's CSR row when the formats hold different labels
      a.closing_csr = (!ctx->f[1].built || ctx->keep[0] != ctx->keep[1]) ? 1 : 0;
      a.use_tma = ctx->use_tma ? 1 : 0;
      for (size_t i = 0; i < anc_cols[k - 1].size(); i++) a.par_anc[i] = sl.lv[k - 1].anc[i];
      a.n_anc_out = (uint32_t)anc_cols[k].size();
      for (uint32_t i = 0; i < a.n_anc_out; i++) {
        a.anc_src[i] = anc_index(k, anc_cols[k][i]);
        a.out_anc[i] = sl.lv[k].anc[i];
      }
      if (!a.tree) {
        prof.begin(K_COMPACT);
        CU(launch_bitmap_compact_lb(cand(Lv.var), W, sl.list[k], sl.list_cap[k], dsz + 64 + k, sl.d_ovf,
                                    next_lb(sl), smc, sl.st));
        launches[K_COMPACT] += compact_launches(W);
        prof.end();
        a.list = sl.list[k];
        a.d_list_len = dsz + 64 + k;
      }
      a.seg_beg = sl.lv[k - 1].seg_beg;
      a.off = sl.lv[k - 1].off;
      a.tile_start = sl.tile_start;
      a.d_T = dsz + 32 + k;
      a.out_parent = sl.lv[k].parent;
      a.out_bind = sl.lv[k].bind;
      a.out_alive = k + 1 < L ? sl.lv[k].alive : nullptr;
      a.cap_out = sl.lv[k].cap;
      a.d_nout = dsz + k;
      a.overflow = sl.d_ovf;
      a.ctr = sl.d_ctr;
      a.lb = next_lb(sl);
      if (a.tree && functional_edge(a.dir & 1, Lv.label)) {  // <= 1 child per parent: one fused pass
        fused_lv[k] = 1;
        prof.begin(K_EXPAND_EMIT);
        CU(launch_expand_func(a, ctx->pred_bytes, smc, sl.st));
        launches[K_EXPAND_EMIT]++;
        prof.end();
        continue;
      }
      prof.begin(K_EXPAND_SEG);
      CU(launch_seg_scan(a, ctx->pred_bytes, smc, sl.st));
      launches[K_EXPAND_SEG]++;
      prof.end();
      a.lb = next_lb(sl);
      prof.begin(K_EXPAND_EMIT);
      CU(launch_expand_lb(a, ctx->pred_bytes, smc, sl.st));
      launches[K_EXPAND_EMIT]++;
      prof.end();
    }
    CU(cudaMemcpyAsync(sl.h_pin, dsz, 128 * 8, cudaMemcpyDeviceToHost, sl.st));
    return GSMART_OK;
  }

  // Rows leave the trie in visitation (pi-lexicographic) order.  They are also in
  // column order when every level k that an earlier level d precedes in pi but
  // follows in column order is determined by levels before d: the chain of
  // functional tree edges above k reaches a level < d (two rows that first differ
  // at d then agree on every column before d's).  Then no sort runs.
  bool sorted_by_construction() const {
    const uint32_t LT = (uint32_t)plan->levels.size();
    std::vector<uint32_t> root(LT);  // anc_func: the top of k's chain of functional tree edges
    for (uint32_t k = 0; k < LT; k++) {
      const Level& Lv = plan->levels[k];
      root[k] = (k > 0 && Lv.tree_edge >= 0 && functional_edge(Lv.dir == OUT ? 0u : 1u, Lv.label))
                    ? root[Lv.parent_level]
                    : k;
    }
    for (uint32_t d = 0; d < LT; d++)
      for (uint32_t k = d + 1; k < LT; k++)
        if (plan->col_of[plan->levels[k].var] < plan->col_of[plan->levels[d].var] && root[k] >= d) return false;
    return true;
  }

  // a tree edge over `label` read from format `fmt`'s rows reaches at most one child
  // per parent (exact build statistic); GSMART_NO_FUNC=1 disables the fused pass (A/B)
  bool functional_edge(uint32_t fmt, uint32_t label) const {
    const char* ev = getenv("GSMART_NO_FUNC");
    const auto& fu = ctx->f[fmt].functional;
    return !(ev && atoi(ev) != 0) && label < fu.size() && fu[label];
  }

  // f2: level 0 as in the trie, then every occurrence from its parent occurrence
  // (k_seg_scan + k_expand_lb unchanged: the parent level index p is passed as
  // k - 1, so ANC_BIND reads the parent occurrence's bindings)
  gsmart_status launch_expansion_f(bool fresh) {
    unsigned long long* dsz = sl.d_sz;
    if (!fresh) {
      CU(cudaMemsetAsync(dsz, 0, 128 * 8, sl.st));
      TRY(ensure_om());  // a level grew: key sets follow (not inside a capture: re-runs launch directly)
    }
    prof.begin(K_COMPACT);
    CU(launch_bitmap_compact_lb(cand(occ[0].var), W, sl.lv[0].bind, sl.lv[0].cap, dsz + 0, sl.d_ovf, next_lb(sl),
                                smc, sl.st));
    launches[K_COMPACT] += compact_launches(W);
    prof.end();
    for (uint32_t o = 1; o < L; o++) {
      const Occ& oc = occ[o];
      const uint32_t p = (uint32_t)oc.par;
      ExpArgs2 a;
      memset(&a, 0, sizeof a);
      for (uint32_t j = 0; j < o; j++) {
        a.tab.parent[j] = sl.lv[j].parent;
        a.tab.bind[j] = sl.lv[j].bind;
        a.tab.up[j] = (uint8_t)(j ? occ[j].par : 0);
      }
      a.k = p + 1;
      a.d_nparent = dsz + p;
      a.cap_par = sl.lv[p].cap;
      a.tree = oc.tree ? 1 : 0;
      a.parent_level = p;
      a.label = oc.label;
      a.dir = oc.dir == OUT ? 0 : 1;
      a.f[0] = fa[0];
      a.f[1] = fa[1];
      a.cand = cand(oc.var);
      for (size_t i = 0; i < oc.cl.size(); i++) {
        a.cl[a.ncl] = oc.cl[i];
        a.cl_idx[a.ncl++] = oc.cl_idx[i];
      }
      a.par_idx = ANC_BIND;
      a.closing_csr = (!ctx->f[1].built || ctx->keep[0] != ctx->keep[1]) ? 1 : 0;
      a.use_tma = ctx->use_tma ? 1 : 0;
      if (oc.same >= 0) {  // Ω pre-pruning (§7.2.2 applied to §8.1's common variable)
        unsigned long long* t = sl.om + om_off[o];
        CU(cudaMemsetAsync(t, 0xff, (om_mask[o] + 1) * 8, sl.st));
        prof.begin(K_PRUNE);
        CU(launch_f_hash_build(a.tab, (uint32_t)oc.same, dsz + oc.same, sl.lv[oc.same].cap, t, om_mask[o],
                               smc, sl.st));
        launches[K_PRUNE]++;
        prof.end();
        a.om_tab = t;
        a.om_mask = om_mask[o];
      }
      if (!a.tree) {
        prof.begin(K_COMPACT);
        CU(launch_bitmap_compact_lb(cand(oc.var), W, sl.list[o], sl.list_cap[o], dsz + 64 + o, sl.d_ovf,
                                    next_lb(sl), smc, sl.st));
        launches[K_COMPACT] += compact_launches(W);
        prof.end();
        a.list = sl.list[o];
        a.d_list_len = dsz + 64 + o;
      }
      a.seg_beg = sl.lv[p].seg_beg;
      a.off = sl.lv[p].off;
      a.tile_start = sl.tile_start;
      a.d_T = dsz + 32 + o;
      a.out_parent = sl.lv[o].parent;
      a.out_bind = sl.lv[o].bind;
      a.cap_out = sl.lv[o].cap;
      a.d_nout = dsz + o;
      a.overflow = sl.d_ovf;
      a.ctr = sl.d_ctr;
      a.lb = next_lb(sl);
      if (a.tree && !a.om_tab && functional_edge(a.dir & 1, oc.label)) {  // <= 1 child per parent
        fused_lv[o] = 1;
        prof.begin(K_EXPAND_EMIT);
        CU(launch_expand_func(a, ctx->pred_bytes, smc, sl.st));
        launches[K_EXPAND_EMIT]++;
        prof.end();
        continue;
      }
      prof.begin(K_EXPAND_SEG);
      CU(launch_seg_scan(a, ctx->pred_bytes, smc, sl.st));
      launches[K_EXPAND_SEG]++;
      prof.end();
      a.lb = next_lb(sl);
      prof.begin(K_EXPAND_EMIT);
      CU(launch_expand_lb(a, ctx->pred_bytes, smc, sl.st));
      launches[K_EXPAND_EMIT]++;
      prof.end();
    }
    CU(cudaMemcpyAsync(sl.h_pin, dsz, 128 * 8, cudaMemcpyDeviceToHost, sl.st));
    return GSMART_OK;
  }

  // f2 phase 2 (host-synchronous; no speculation or graph): a8 on the factorised
  // trees (a node lives iff every branch below it keeps a child, and its parent
  // lives), §8.1 Ω pruning per root binding, subtree counts, then a9 rows
  // enumerated from the trees and sorted.
  gsmart_status phase2_f() {
    state = S_PHASE2;
    TRY(keep_candidates());
    const int sm = smc;
    const uint32_t nc = (uint32_t)plan->vars.size();
    std::vector<std::vector<uint32_t>> kids(L);
    for (uint32_t o = 1; o < L; o++) kids[occ[o].par].push_back(o);
    uint64_t maxF = 1;
    for (uint32_t o = 0; o < L; o++) maxF = std::max<uint64_t>(maxF, F[o]);
    uint8_t* hc = nullptr;
    TRY(sc.get(&hc, maxF));
    auto rootb = [&](uint32_t o) { return o == 0 ? sl.lv[0].bind : sl.lv[o].newidx; };
    prof.begin(K_PRUNE);
    for (uint32_t o = 0; o < L; o++) {
      CU(launch_f_fill(sl.lv[o].alive, F[o], 1, sm, sl.st));
      launches[K_PRUNE]++;
    }
    auto bottom_up = [&]() -> gsmart_status {
      for (uint32_t o = L - 1; o >= 1; o--) {
        const uint32_t p = (uint32_t)occ[o].par;
        if (!F[p]) continue;
        CU(cudaMemsetAsync(hc, 0, F[p], sl.st));
        CU(launch_f_mark(sl.lv[o].parent, sl.lv[o].alive, F[o], hc, sm, sl.st));
        CU(launch_f_and(sl.lv[p].alive, hc, F[p], sm, sl.st));
        launches[K_PRUNE] += 2;
      }
      return GSMART_OK;
    };
    auto top_down = [&](bool roots) -> gsmart_status {
      for (uint32_t o = 1; o < L; o++) {
        const uint32_t p = (uint32_t)occ[o].par;
        CU(launch_f_down(sl.lv[o].alive, sl.lv[o].parent, sl.lv[p].alive, roots ? rootb(p) : nullptr,
                         roots ? rootb(o) : nullptr, F[o], sm, sl.st));
        launches[K_PRUNE]++;
      }
      return GSMART_OK;
    };
    TRY(bottom_up());
    TRY(top_down(n_omega > 0));
    if (n_omega) {  // §8.1 steps 1-3: per root binding, a variable's bindings must occur at all its occurrences
      std::map<uint32_t, std::vector<uint32_t>> by_var;
      for (uint32_t o = 0; o < L; o++) by_var[occ[o].var].push_back(o);
      // one bit above every live key: dead nodes' keys (all ones) sort strictly last
      const int kb = std::min(64, 33 + bits_for(ctx->N ? ctx->N - 1 : 0));
      for (auto& kv : by_var) {
        const auto& G = kv.second;
        if (G.size() < 2) continue;
        std::vector<unsigned long long*> sorted(G.size());
        for (size_t i = 0; i < G.size(); i++) {
          const uint32_t X = G[i];
          unsigned long long *k0 = nullptr, *k1 = nullptr;
          void* tmp = nullptr;
          const uint64_t n = std::max<uint64_t>(F[X], 1);
          TRY(sc.get(&k0, n));
          TRY(sc.get(&k1, n));
          const size_t tb = radix_tmp_bytes(n);
          TRY(sc.get((char**)&tmp, tb));
          CU(launch_f_keys(rootb(X), sl.lv[X].bind, sl.lv[X].alive, F[X], k0, sm, sl.st));
          int second = 0;
          CU(radix_sort_keys_u64(reinterpret_cast<uint64_t*>(k0), reinterpret_cast<uint64_t*>(k1), F[X], 0, kb, tmp,
                                 tb, sl.st, &second, &launches[K_PRUNE], false));
          sorted[i] = second ? k1 : k0;
          launches[K_PRUNE]++;
        }
        for (size_t i = 0; i < G.size(); i++) {
          FProbeArgs pa;
          memset(&pa, 0, sizeof pa);
          pa.root = rootb(G[i]);
          pa.bind = sl.lv[G[i]].bind;
          pa.alive = sl.lv[G[i]].alive;
          pa.n = F[G[i]];
          for (size_t j = 0; j < G.size(); j++)
            if (j != i) {
              pa.keys[pa.n_other] = sorted[j];
              pa.n_keys[pa.n_other++] = F[G[j]];
            }
          CU(launch_f_probe(pa, sm, sl.st));
          launches[K_PRUNE]++;
        }
      }
      TRY(bottom_up());  // step 4: parents left without a child in some branch
      TRY(top_down(false));
    }
    // subtree counts, leaves first: cnt(m) = prod over branches of the children's counts
    std::vector<unsigned long long*> P(L, nullptr);
    std::vector<uint32_t*> cb(L, nullptr), ce(L, nullptr);
    unsigned long long* n_alive = nullptr;
    TRY(sc.get(&n_alive, 1));
    for (uint32_t o = 0; o < L; o++) TRY(sc.get(&P[o], F[o] + 1));
    for (uint32_t o = 1; o < L; o++) {
      const uint64_t np = std::max<uint64_t>(F[occ[o].par], 1);
      TRY(sc.get(&cb[o], np));
      TRY(sc.get(&ce[o], np));
      CU(cudaMemsetAsync(cb[o], 0, np * 4, sl.st));
      CU(cudaMemsetAsync(ce[o], 0, np * 4, sl.st));
      CU(launch_f_ranges(sl.lv[o].parent, F[o], cb[o], ce[o], sm, sl.st));
      launches[K_PRUNE]++;
    }
    for (uint32_t o = L; o-- > 0;) {
      FCountArgs ca;
      memset(&ca, 0, sizeof ca);
      ca.alive = sl.lv[o].alive;
      ca.n = F[o];
      for (uint32_t c : kids[o]) {
        ca.P[ca.nch] = P[c];
        ca.beg[ca.nch] = cb[c];
        ca.end[ca.nch++] = ce[c];
      }
      ca.out = P[o];
      ca.lb = next_lb(sl);
      ca.overflow = sl.d_ovf;
      CU(launch_f_count_scan(ca, sm, sl.st));
      launches[K_PRUNE]++;
    }
    prof.end();
    unsigned long long total = 0;
    int ovf = 0;
    CU(cudaMemcpyAsync(&total, P[0] + F[0], 8, cudaMemcpyDeviceToHost, sl.st));
    CU(cudaMemcpyAsync(&ovf, sl.d_ovf, 4, cudaMemcpyDeviceToHost, sl.st));
    CU(cudaStreamSynchronize(sl.st));
    if (ovf & 4) FAIL(GSMART_E_RESULT_OVERFLOW, "factorised: more than 2^46 combinations");
    R->stats.factorised = 1;
    R->stats.n_omega = n_omega;
    R->stats.combinations = total;
    // the trees themselves (gsmart_result_tree): bindings, parent links, alive flags
    R->levels.clear();
    {
      uint64_t bytes = 0;
      auto al = [](uint64_t b) { return (b + 255) / 256 * 256; };
      for (uint32_t o = 0; o < L; o++) bytes += al(F[o] * 4) * 2 + al(F[o]);
      char* arena = nullptr;
      TRY(alloc_result((void**)&arena, std::max<uint64_t>(bytes, 256)));
      for (uint32_t o = 0; o < L; o++) {
        gsmart_result::Lv lv{occ[o].var, F[o], nullptr, nullptr};
        lv.parent_level = occ[o].par;
        lv.bind = (uint32_t*)arena;
        arena += al(F[o] * 4);
        if (o) {
          lv.parent = (uint32_t*)arena;
          CU(cudaMemcpyAsync(lv.parent, sl.lv[o].parent, F[o] * 4, cudaMemcpyDeviceToDevice, sl.st));
        }
        arena += al(F[o] * 4);
        lv.alive = (uint8_t*)arena;
        arena += al(F[o]);
        CU(cudaMemcpyAsync(lv.bind, sl.lv[o].bind, F[o] * 4, cudaMemcpyDeviceToDevice, sl.st));
        CU(cudaMemcpyAsync(lv.alive, sl.lv[o].alive, F[o], cudaMemcpyDeviceToDevice, sl.st));
        R->levels.push_back(lv);
      }
    }
    const bool filtered = n_omega > 0;
    const bool want_rows = !(flags & GSMART_COUNT_ONLY);
    R->count_only = !want_rows;
    FEnumArgs ea;
    memset(&ea, 0, sizeof ea);
    for (uint32_t o = 0; o < L; o++) {
      FOcc& fo = ea.o[o];
      fo.bind = sl.lv[o].bind;
      fo.P = P[o];
      fo.beg = cb[o];
      fo.end = ce[o];
      fo.par = occ[o].par;
      fo.col = occ[o].col;
      fo.same = occ[o].same;
      fo.leaf = kids[o].empty() ? 1 : 0;
      fo.first = (o > 0 && kids[occ[o].par].front() == o) ? 1 : 0;
    }
    ea.n_occ = L;
    ea.n_root = (uint32_t)F[0];
    ea.nc = nc;
    ea.total = total;
    ea.overflow = sl.d_ovf;
    ea.filtered = filtered ? 1 : 0;
    unsigned long long* d_cnt = sl.d_ctr + 60;
    ea.d_count = d_cnt;
    uint64_t n_rows = total;
    if (filtered && total) {  // Ω equality: count the consistent combinations first
      ea.count_only = 1;
      CU(cudaMemsetAsync(d_cnt, 0, 8, sl.st));
      prof.begin(K_ENUMERATE);
      CU(launch_f_enum(ea, sm, sl.st));
      prof.end();
      launches[K_ENUMERATE]++;
      CU(cudaMemcpyAsync(&n_rows, d_cnt, 8, cudaMemcpyDeviceToHost, sl.st));
      CU(cudaStreamSynchronize(sl.st));
    }
    R->n_rows = n_rows;
    if (n_rows > ctx->cap()) FAIL(GSMART_E_RESULT_OVERFLOW, "factorised: rows exceed max_result_rows");
    CU(cudaMemcpyAsync(sl.h_pin + 192, sl.d_ctr, C_NCTR * 8, cudaMemcpyDeviceToHost, sl.st));
    ctr_pinned = true;
    if (!want_rows || !n_rows) {
      R->host_valid = !n_rows && want_rows;
      return GSMART_OK;
    }
    uint32_t* raw = nullptr;
    TRY(sc.get(&raw, n_rows * nc));
    TRY(alloc_result((void**)&R->d_rows, n_rows * nc * 4));
    ea.count_only = 0;
    ea.rows = R->d_rows;  // enumerated into the result, sorted in place (raw = scratch if unsorted)
    ea.cap_rows = n_rows;
    if (filtered) CU(cudaMemsetAsync(d_cnt, 0, 8, sl.st));
    prof.begin(K_ENUMERATE);
    CU(launch_f_enum(ea, sm, sl.st));
    launches[K_ENUMERATE]++;
    prof.end();
    const size_t tb = sort_rows_tmp_bytes(n_rows, nc);
    void* tmp = nullptr;
    TRY(sc.get((char**)&tmp, std::max<size_t>(tb, 256)));
    prof.begin(K_SORT_ROWS);
    CU(sort_rows(raw, R->d_rows, n_rows, nc, nc, bits_for(ctx->N ? ctx->N - 1 : 0), tmp, tb, sl.st,
                 &launches[K_SORT_ROWS], reinterpret_cast<int*>(sl.d_ctr + 50), true));
    prof.end();
    return GSMART_OK;
  }

  gsmart_status relaunch_expansion() {
    TRY(launch_expansion(false));
    CU(cudaEventRecord(sl.ev, sl.st));
    state = S_EXPANDING;
    return GSMART_OK;
  }

  // Push or pull per group edge (cached per plan and LSpM generation).  Pull
  // (k_group_filter_rows) costs ~40-60 DRAM bytes per candidate row of the
  // center (scattered row_ptr / label / column sectors); push (k_push_edge)
  // streams 8 bytes per entry of the edge's label.  The center's candidate count
  // is bounded by its seed segments (row lengths read once here) or N.
  // A small label is cheap to stream (64K entries = 512 KB), while pulling an
  // unconstrained center touches every row's signature: push below PUSH_RATIO x bound.
  // (ctx->push_min, default 2^16 entries)
  static constexpr uint64_t PUSH_RATIO = 6;
  gsmart_status decide_push() {
    push_dec.clear();
    const int v = ctx->filter_variant;
    if (!ctx->lm.built || (ctx->world > 1 && !ctx->lm_in.built) || (v & 16) || plan->groups.empty())
      return GSMART_OK;
    const uint64_t pkey = plan->uid * 2 + ((flags & GSMART_BACK_EDGES) ? 1 : 0);  // decisions per edge set
    auto it = ctx->push_cache.find(pkey);
    if (it != ctx->push_cache.end() && it->second.first == ctx->lspm_gen) {
      push_dec = it->second.second;
      return GSMART_OK;
    }
    const uint32_t N = ctx->N;
    std::vector<uint64_t> est(plan->n_vertices, N);
    std::vector<uint32_t> rp2(2 * plan->seeds.size(), 0);
    for (size_t i = 0; i < plan->seeds.size(); i++) {
      const Seed& sd = plan->seeds[i];
      if (sd.cid >= N) continue;
      CU(cudaMemcpyAsync(&rp2[2 * i], ctx->f[sd.dir == OUT ? 0 : 1].rp + sd.cid, 8, cudaMemcpyDeviceToHost, sl.st));
    }
    if (!plan->seeds.empty()) CU(cudaStreamSynchronize(sl.st));
    for (size_t i = 0; i < plan->seeds.size(); i++) {
      const Seed& sd = plan->seeds[i];
      if (sd.cid < N) est[sd.var] = std::min<uint64_t>(est[sd.var], rp2[2 * i + 1] - rp2[2 * i]);
    }
    push_dec.resize(plan->groups.size());
    for (size_t gi = 0; gi < plan->groups.size(); gi++) {
      const Group& g = plan->groups[gi];
      const std::vector<GroupEdge>& GE = gedges[gi];
      push_dec[gi].assign(GE.size(), 0);
      // in ascending label size (the launch order); a pushed edge bounds the
      // center's candidates by its label's entry count for the next decision
      std::vector<size_t> ord(GE.size());
      for (size_t ei = 0; ei < ord.size(); ei++) ord[ei] = ei;
      auto M_of = [&](size_t ei) {
        const uint32_t l = GE[ei].label;
        const LabelMajor& Lm = lm_for(GE[ei]);
        return l + 1 < Lm.off.size() ? Lm.off[l + 1] - Lm.off[l] : 0ull;
      };
      std::stable_sort(ord.begin(), ord.end(), [&](size_t x, size_t y) { return M_of(x) < M_of(y); });
      uint64_t bound = est[g.center];
      for (size_t ei : ord) {
        const uint64_t M = M_of(ei);
        const bool p = (v & 8) || (M >= ctx->push_min && M <= PUSH_RATIO * bound);
        push_dec[gi][ei] = p;
        if (p) bound = std::min(bound, M);
      }
    }
    ctx->push_cache[pkey] = {ctx->lspm_gen, push_dec};
    return GSMART_OK;
  }

  // every workspace buffer phase 1 touches, sized before any launch (a graph
  // replay must see the same addresses; growth bumps sl.ws_gen)
  gsmart_status ensure_workspace() {
    const uint64_t nvar = plan->vars.size();
    TRY(slot_heavy(ctx, sl));
    if (peer_mode()) {
      // symmetric: [bitmaps (Wpad words per variable)][32 change words][barrier flags, u64 per rank]
      const uint64_t need = std::max<uint64_t>((uint64_t)Wpad * nvar, 32);
      if (!sl.sym.va || sl.sym_cand_words < need) {  // collective: every rank runs the same plans
        CU(cudaStreamSynchronize(sl.st));
        const uint64_t words = need + 32 + 2 * MAX_WORLD;
        const uint64_t g = sym_granularity(ctx);
        const uint64_t bytes = (words * 4 + g - 1) / g * g;
        SymRegion R2;
        TRY(sym_alloc(ctx, (uint64_t)ctx->rank * bytes, bytes, &R2));
        CU(cudaMemsetAsync(R2.local(), 0, bytes, sl.st));
        CU(cudaStreamSynchronize(sl.st));
        if (sl.sym.va) sym_free(ctx, &sl.sym);
        TRY(host_barrier(ctx));  // every rank's flags are zero before any barrier kernel runs
        sl.sym = R2;
        sl.cand = (uint32_t*)R2.local();
        sl.sym_cand_words = need;
        sl.bar_next = 1;
        sl.ws_gen++;
      }
    } else {
      TRY(slot_buf(ctx, sl, &sl.cand, &sl.cand_words, std::max<uint64_t>((uint64_t)Wpad * nvar, 1)));
    }
    if (ctx->filter_variant & 4) TRY(slot_buf(ctx, sl, &sl.frows, &sl.frows_cap, (uint64_t)W * 32));
    if (ctx->lm.built) TRY(slot_buf(ctx, sl, &sl.sat, &sl.sat_cap, 2ull * Wpad));
    if (ctx->l2_persist) {  // A/B: keep the candidate bitmaps (random probes) resident in a persisting L2 window
      static bool limit_set = false;
      int dev = ctx->cfg.device, max_persist = 0, max_window = 0;
      cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
      cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
      if (!limit_set && max_persist > 0) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)max_persist);
        limit_set = true;
      }
      cudaStreamAttrValue v = {};
      v.accessPolicyWindow.base_ptr = sl.cand;
      v.accessPolicyWindow.num_bytes = std::min<size_t>((size_t)Wpad * nvar * 4, (size_t)std::max(max_window, 0));
      v.accessPolicyWindow.hitRatio = 1.0f;
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(sl.st, cudaStreamAttributeAccessPolicyWindow, &v);
      cudaGetLastError();
    }
    for (uint32_t k = 0; k < L; k++) TRY(slot_level(ctx, sl, k, 1, (uint32_t)anc_cols[k].size()));
    if (fact) TRY(ensure_om());
    for (uint32_t k = 1; k < L; k++)
      if (fact ? !occ[k].tree : plan->levels[k].tree_edge < 0)
        TRY(slot_buf(ctx, sl, &sl.list[k], &sl.list_cap[k], (uint64_t)W * 32));
    return GSMART_OK;
  }

  // phase 1 = seeds + grouped evaluation + expansion: pure device work on
  // stable workspace addresses, launched directly or replayed from a graph
  gsmart_status phase1_kernels() {  // counters/sizes are zeroed by k_init_cands
    group_seq.assign(plan->groups.size(), 0);
    filter_seq = 0;
    TRY(seeds_and_guards());
    // peers clear bits in this rank's bitmaps from the first group on: not before
    // this rank initialised and seeded them
    if (peer_mode()) TRY(rank_barrier());
    for (size_t i = 0; i < plan->groups.size(); i++) TRY(eval_group(plan->groups[i], i));
    if ((flags & GSMART_REFINE) && !(flags & GSMART_NO_REFINE) && plan->groups.size() > 1)
      for (size_t i = plan->groups.size() - 1; i-- > 0;) TRY(eval_group(plan->groups[i], i));
    return launch_expansion(true);
  }

  // Run `body` (stream work on stable workspace addresses only) directly, or
  // replay it from this slot's graph cache under `key` (captured on first use).
  // Look-back epochs inside are offsets from the execute's base, so a replay is
  // valid only if the body starts at the same offset as when it was captured.
  template <typename Body>
  gsmart_status run_cached(uint64_t key, uint32_t key_flags, Body&& body) {
    const bool graphable = !(flags & (GSMART_PROFILE | GSMART_NO_GRAPH)) && !ctx->comm &&
                           (ctx->world == 1 || (peer_mode() && !host_barriers()));
    if (!graphable) return body();
    auto it = sl.graphs.find(key);
    if (it != sl.graphs.end() && it->second.ws_gen == sl.ws_gen && it->second.lspm_gen == ctx->lspm_gen &&
        it->second.flags == key_flags) {
      if (it->second.off0 != sl.seq_off || it->second.bar0 != sl.bar_off) return body();  // e.g. after a re-run
      CU(cudaGraphLaunch(it->second.exec, sl.st));
      sl.seq_off += it->second.n_lb;
      sl.bar_off += it->second.n_bar;
      graph_replayed = true;
      for (int i = 0; i < GSMART_NKERNELS; i++) launches[i] += it->second.launches[i];
      filter_main += it->second.filter_main;
      push_and += it->second.push_and;
      n_exchanges += it->second.n_exchanges;
      return GSMART_OK;
    }
    if (it != sl.graphs.end()) {
      cudaGraphExecDestroy(it->second.exec);
      sl.graphs.erase(it);
    }
    // capture on the second use: a plan executed once (a cold query) pays no
    // capture/instantiation; a repeated plan replays from then on
    if (sl.seen.insert(key).second) return body();
    const uint32_t off0 = sl.seq_off, bar0 = sl.bar_off;
    const std::vector<int> l0(launches, launches + GSMART_NKERNELS);
    const uint64_t fm0 = filter_main, pa0 = push_and, nx0 = n_exchanges;
    CU(cudaStreamBeginCapture(sl.st, cudaStreamCaptureModeThreadLocal));
    gsmart_status s = body();
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(sl.st, &graph);
    if (s != GSMART_OK) {
      if (graph) cudaGraphDestroy(graph);
      return s;
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamEndCapture", __LINE__);
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphInstantiate", __LINE__);
    Slot::GraphEntry ge;
    ge.exec = exec;
    ge.ws_gen = sl.ws_gen;
    ge.lspm_gen = ctx->lspm_gen;
    ge.flags = key_flags;
    ge.off0 = off0;
    ge.n_lb = sl.seq_off - off0;
    ge.bar0 = bar0;
    ge.n_bar = sl.bar_off - bar0;
    ge.launches.resize(GSMART_NKERNELS);
    for (int i = 0; i < GSMART_NKERNELS; i++) ge.launches[i] = launches[i] - l0[i];
    ge.filter_main = filter_main - fm0;
    ge.push_and = push_and - pa0;
    ge.n_exchanges = n_exchanges - nx0;
    if (sl.graphs.size() >= 512) {  // bounded cache
      for (auto& kv : sl.graphs) cudaGraphExecDestroy(kv.second.exec);
      sl.graphs.clear();
    }
    sl.graphs[key] = ge;
    CU(cudaGraphLaunch(exec, sl.st));
    return GSMART_OK;
  }

  // phase 1 = seeds + grouped evaluation + expansion (graph key: uid, tag 0)
  gsmart_status run_phase1() {
    return run_cached(plan->uid << 3, flags & (GSMART_NO_REFINE | GSMART_REFINE | GSMART_BACK_EDGES | GSMART_FACTORISED),
                      [&] { return phase1_kernels(); });
  }

  gsmart_status start() {
    const uint32_t N = ctx->N;
    const uint32_t nvar = (uint32_t)plan->vars.size();
    W = (N + 31) / 32;
    Wpad = (W + 31) / 32 * 32;
    wlo = 0;
    whi = W;
    if (ctx->world > 1) {  // this rank's vertex range (partition split points are multiples of 2^19)
      wlo = part_word_lo(ctx, ctx->rank);
      whi = part_word_hi(ctx, ctx->rank);
    }
    L = (uint32_t)plan->levels.size();
    identity = true;
    for (uint32_t k = 0; k < L; k++)
      if ((uint32_t)plan->col_of[plan->levels[k].var] != k) identity = false;
    if (!identity && !(flags & GSMART_FACTORISED)) identity = sorted_by_construction();
    R->n_words = W;
    R->stride_words = Wpad;
    slot.assign(plan->n_vertices, -1);
    for (uint32_t i = 0; i < nvar; i++) slot[plan->vars[i]] = (int32_t)i;
    R->cand_slot = slot;
    for (int d = 0; d < 2; d++) {
      fa[d].rp = ctx->f[d].rp;
      fa[d].col = ctx->f[d].col;
      fa[d].pred = ctx->f[d].pred;
      fa[d].lmask = ctx->f[d].lmask;
    }
    for (uint32_t k = 1; k < L; k++)
      if (plan->levels[k].closing.size() > (size_t)MAXC)
        FAIL(GSMART_E_UNSUPPORTED, "more than 16 closing edges on one level");
    gedges.resize(plan->groups.size());
    for (size_t gi = 0; gi < plan->groups.size(); gi++) {
      gedges[gi] = plan->groups[gi].edges;
      if (flags & GSMART_BACK_EDGES)
        gedges[gi].insert(gedges[gi].end(), plan->groups[gi].back.begin(), plan->groups[gi].back.end());
    }
    fact = (flags & GSMART_FACTORISED) != 0;
    if (fact) {
      if (ctx->world > 1 || ctx->comm) FAIL(GSMART_E_UNSUPPORTED, "GSMART_FACTORISED needs world == 1");
      TRY(build_occurrences());
      L = (uint32_t)occ.size();
      identity = false;
      anc_cols.assign(L, {});
    } else {
      plan_ancestors();
    }
    // levels the fused functional kernel expands (the same decision the launch
    // paths take; kept for the byte accounting, which also runs after graph replays)
    fused_lv.assign(L, 0);
    for (uint32_t k = 1; k < L; k++) {
      if (fact) fused_lv[k] = occ[k].tree && occ[k].same < 0 && functional_edge(occ[k].dir == OUT ? 0u : 1u, occ[k].label);
      else fused_lv[k] = plan->levels[k].tree_edge >= 0 &&
                         functional_edge(plan->levels[k].dir == OUT ? 0u : 1u, plan->levels[k].label);
    }
    TRY(decide_push());
    TRY(ensure_workspace());
    TRY(begin_seq(ctx, sl));
    seq_open = true;
    F.assign(L, 0);
    R->stats.n_levels = L;

    if (nvar > 0) {  // the common path: all device work of phase 1, then one event
      TRY(run_phase1());
      if (can_speculate()) {  // phase 2 goes behind phase 1 once every plan's phase 1 is queued
        spec_pending = true;
        state = S_EXPANDING;
        return GSMART_OK;
      }
      CU(cudaEventRecord(sl.ev, sl.st));
      state = S_EXPANDING;
      return GSMART_OK;
    }
    // only guards (or nothing): one empty row iff all hold
    CU(cudaMemsetAsync(sl.d_ctr, 0, C_NCTR * 8, sl.st));
    TRY(seeds_and_guards());
    int flag = 1;
    if (!plan->guards.empty()) {
      CU(cudaMemcpyAsync(&flag, sl.d_ctr + 48, 4, cudaMemcpyDeviceToHost, sl.st));
      CU(cudaStreamSynchronize(sl.st));
    }
    R->n_rows = flag ? 1 : 0;
    R->host_valid = true;
    state = S_DONE;
    return GSMART_OK;
  }

  // Speculative phase 2: a plan re-executed on the same LSpM with the same flags
  // produces the same level sizes, so phase 2 is sized from the previous run and
  // queued right behind phase 1 — no host round trip between the phases.  A
  // device guard (k_phase2_guard) turns every phase-2 kernel into a no-op if a
  // level would not fit; after the drain the host compares the real sizes with
  // the guess and, on a mismatch, redoes phase 2 the ordinary way.
  bool spec = false, spec_pending = false;
  bool can_speculate() const {
    if ((ctx->world > 1 && !peer_mode()) || (flags & GSMART_NO_SPECULATE) || fact) return false;
    auto it = ctx->p2_guess.find(plan->uid);
    if (it == ctx->p2_guess.end() || it->second.gen != ctx->lspm_gen || it->second.flags != flags ||
        it->second.F.size() != L)
      return false;
    for (uint32_t k = 0; k < L; k++)
      if (it->second.F[k] > sl.lv[k].cap) return false;
    return true;
  }
  size_t spec_owned0 = 0;  // R->owned entries before the speculative phase 2
  gsmart_status speculate() {
    spec_pending = false;
    F = ctx->p2_guess.find(plan->uid)->second.F;
    if (ctx->spec_test && F[L - 1]) F[L - 1] += (ctx->spec_test++ & 1) ? 1 : -1;  // test hook: force a wrong guess
    for (uint32_t k = 0; k < L && k < GSMART_MAX_LEVELS; k++) R->stats.level_nodes[k] = F[k];
    spec_owned0 = R->owned.size();
    TRY(phase2());
    spec = true;
    R->stats.spec_phase2 = 1;
    return GSMART_OK;
  }
  // after the drain of a speculative run: did phase 1 produce the guessed sizes?
  bool spec_holds() const {
    const unsigned long long* hv = sl.h_pin;
    if (hv[127] & 0xffffffffu) return false;
    for (uint32_t k = 0; k < L; k++)
      if (hv[k] != F[k]) return false;
    return true;
  }
  gsmart_status redo_phase2() {  // mis-speculation: the ordinary path from the real sizes
    spec = false;
    R->stats.spec_redo = 1;
    // the speculative outputs (arena, candidate copy) are dead: free them before
    // the redo allocates its own (the stream is drained)
    for (size_t i = spec_owned0; i < R->owned.size(); i++) dfree(ctx, sl.st, R->owned[i]);
    R->owned.resize(spec_owned0);
    R->d_cand = nullptr;
    R->levels.clear();
    R->d_rows = nullptr;
    R->n_rows = 0;
    ctr_pinned = false;
    return after_expand();
  }

  // called once sl.ev completed
  gsmart_status after_expand() {
    const unsigned long long* hv = sl.h_pin;
    const int ovf = (int)(hv[127] & 0xffffffffu);
    if (ovf & 2) FAIL(GSMART_E_RESULT_OVERFLOW, "expansion entries of one level exceed 2^32");
    const uint64_t cap = ctx->cap();
    for (uint32_t k = 0; k < L; k++) {
      F[k] = hv[k];
      if (F[k] > cap) {
        R->n_rows = F[k];
        FAIL(GSMART_E_RESULT_OVERFLOW, "trie level " + std::to_string(k) + " exceeds max_result_rows");
      }
      if (F[k] > sl.lv[k].cap) {  // later levels are invalid: grow and re-run the expansion
        TRY(slot_level(ctx, sl, k, F[k], (uint32_t)anc_cols[k].size()));
        if (++attempts > 2 * (int)L + 2) FAIL(GSMART_E_CUDA, "expansion capacity did not converge");
        return relaunch_expansion();
      }
    }
    for (uint32_t k = 0; k < L; k++) R->stats.level_nodes[k] = F[k];
    return phase2();
  }

  // GSMART_KEEP_CANDIDATES: the result gets its own copy of the slot's bitmaps
  gsmart_status keep_candidates() {
    if (!(flags & GSMART_KEEP_CANDIDATES) || plan->vars.empty()) return GSMART_OK;
    const uint64_t bytes = (uint64_t)Wpad * plan->vars.size() * 4;
    TRY(alloc_result((void**)&R->d_cand, bytes));
    CU(cudaMemcpyAsync(R->d_cand, sl.cand, bytes, cudaMemcpyDeviceToDevice, sl.st));
    return GSMART_OK;
  }

  // ---- a8 prune + compaction, a9 rows + sort (async).  The device work reads its
  // output pointers from the slot's OutTab (filled here per execute, copied to the
  // device inside the work), so it replays from a per-plan graph like phase 1.
  gsmart_status phase2() {
    if (fact) return phase2_f();
    state = S_PHASE2;
    static_assert(C_NCTR <= 64, "counter readback slots");
    TRY(keep_candidates());
    const uint64_t n_rows = F[L - 1];
    unsigned long long* dsz = sl.d_sz;
    R->levels.clear();
    R->n_rows = n_rows;
    if (!n_rows) {
      CU(cudaMemcpyAsync(sl.h_pin + 192, sl.d_ctr, C_NCTR * 8, cudaMemcpyDeviceToHost, sl.st));
      ctr_pinned = true;
      for (uint32_t k = 0; k < L; k++) R->levels.push_back({plan->levels[k].var, 0, nullptr, nullptr});
      R->host_valid = (flags & GSMART_COUNT_ONLY) == 0;
      R->count_only = (flags & GSMART_COUNT_ONLY) != 0;
      return GSMART_OK;
    }
    // one allocation owns the result's levels and rows (each part 256-B aligned)
    const uint32_t nc = (uint32_t)plan->vars.size();
    const bool want_rows = !(flags & GSMART_COUNT_ONLY);
    enum { M_COUNT = 0, M_IDENTITY, M_SORT_SMALL, M_SORT_BIG };
    const int mode = !want_rows ? M_COUNT
                     : identity ? M_IDENTITY
                                : (sort_small_ok(n_rows, nc) ? M_SORT_SMALL : M_SORT_BIG);
    auto al = [](uint64_t b) { return (b + 255) / 256 * 256; };
    // one variable in trie order: the rows are the compacted level-0 bindings
    // themselves (no enumeration, no second copy)
    const bool alias_rows = mode == M_IDENTITY && L == 1 && nc == 1;
    uint64_t arena_bytes = 0;
    for (uint32_t k = 0; k < L; k++) arena_bytes += al(F[k] * 4) * (k > 0 ? 2 : 1);
    if (want_rows && !alias_rows) arena_bytes += al(n_rows * nc * 4);
    char* arena = nullptr;
    TRY(alloc_result((void**)&arena, arena_bytes));
    auto take = [&](uint64_t b) {
      char* p = arena;
      arena += al(b);
      return p;
    };
    OutTab& ot = *sl.h_tab;
    memset(&ot, 0, sizeof ot);
    for (uint32_t k = 0; k < L; k++) {
      gsmart_result::Lv lv{plan->levels[k].var, 0, nullptr, nullptr};
      lv.bind = ot.bind[k] = (uint32_t*)take(F[k] * 4);
      if (k > 0) lv.parent = ot.parent[k] = (uint32_t*)take(F[k] * 4);
      R->levels.push_back(lv);
    }
    size_t tb = 0;
    if (want_rows) {
      R->d_rows = alias_rows ? ot.bind[0] : (uint32_t*)take(n_rows * nc * 4);
      ot.rows = ot.sorted = R->d_rows;
      if (mode != M_IDENTITY) {  // small: enumerate into slot scratch, rank-sort into the result;
                                 // big: enumerate into the result, sort in place (scratch only if unsorted)
        tb = mode == M_SORT_SMALL ? SORT_SMALL_MAXN * 4 : sort_rows_tmp_bytes(n_rows, nc);
        const uint64_t need = al(n_rows * nc * 4) + al(tb);
        if (need > sl.p2_cap) {
          dfree(ctx, sl.st, sl.p2);
          sl.p2 = nullptr;
          sl.p2_cap = 0;
          TRY(dalloc(ctx, &sl.p2, need + need / 4, sl.st));
          sl.p2_cap = need + need / 4;
        }
        if (mode == M_SORT_SMALL) {
          ot.rows = (uint32_t*)sl.p2;
          ot.rank = (uint32_t*)(sl.p2 + al(n_rows * nc * 4));
        }
      }
    } else {
      R->count_only = true;
    }
    std::vector<uint32_t> col_of_level(L);
    for (uint32_t k = 0; k < L; k++) col_of_level[k] = (uint32_t)plan->col_of[plan->levels[k].var];
    for (uint32_t k = 0; k < L && k < (uint32_t)MAXL; k++) ot.cap[k] = F[k];
    ot.small_sort = mode == M_SORT_SMALL;
    auto body = [&]() -> gsmart_status {
      CU(cudaMemcpyAsync(sl.d_tab, sl.h_tab, sizeof(OutTab), cudaMemcpyHostToDevice, sl.st));
      CU(launch_phase2_guard(sl.d_tab, dsz, sl.d_ovf, L, sl.st));
      // phase 1 wrote every counter: read them back with the rest of the stream
      CU(cudaMemcpyAsync(sl.h_pin + 192, sl.d_ctr, C_NCTR * 8, cudaMemcpyDeviceToHost, sl.st));
      prof.begin(K_PRUNE);
      for (uint32_t k = L - 1; k >= 1; k--) {
        CU(launch_prune_mark_d(sl.d_tab, sl.lv[k].parent, k == L - 1 ? nullptr : sl.lv[k].alive, dsz + k, sl.lv[k - 1].alive,
                               smc, sl.st));
        launches[K_PRUNE]++;
      }
      // rows wanted and >= 2 levels: the last level's compaction (a copy) happens
      // inside the enumeration
      const bool fuse_last = L >= 2 && mode != M_COUNT && !alias_rows;
      for (uint32_t k = 0; k < (fuse_last ? L - 1 : L); k++) {
        CU(launch_compact_alive_lb(k > 0 ? sl.lv[k].parent : nullptr, sl.lv[k].bind,
                                   k + 1 < L ? sl.lv[k].alive : nullptr, dsz + k,
                                   k > 0 ? sl.lv[k - 1].newidx : nullptr, sl.d_tab, k,
                                   k + 1 < L ? sl.lv[k].newidx : nullptr, dsz + 96 + k, next_lb(sl), smc,
                                   sl.st));
        launches[K_PRUNE]++;
      }
      prof.end();
      if (mode != M_COUNT && !alias_rows) {
        LastLevel lf;
        if (fuse_last) {
          lf.bind = sl.lv[L - 1].bind;
          lf.parent = sl.lv[L - 1].parent;
          lf.newidx_prev = sl.lv[L - 2].newidx;
          lf.d_n_out = dsz + 96 + (L - 1);
        }
        if (mode == M_SORT_BIG) {  // the sortedness check rides along with the enumeration
          int* fl = reinterpret_cast<int*>(sl.d_ctr + 50);
          CU(cudaMemsetAsync(fl, 0, 4, sl.st));
          CU(cudaMemsetAsync(fl, 1, 1, sl.st));
          lf.sorted = fl;
        }
        prof.begin(K_ENUMERATE);
        CU(launch_enumerate(sl.d_tab, L, col_of_level.data(), fuse_last ? dsz + (L - 1) : dsz + 96 + (L - 1), nc,
                            smc, sl.st, lf));
        launches[K_ENUMERATE]++;
        prof.end();
      }
      CU(cudaMemcpyAsync(sl.h_pin + 128, dsz + 96, 32 * 8, cudaMemcpyDeviceToHost, sl.st));
      if (mode == M_SORT_SMALL) {
        prof.begin(K_SORT_ROWS);
        CU(sort_rows_small(sl.d_tab, dsz + 96 + (L - 1), nc, sl.st, &launches[K_SORT_ROWS]));
        prof.end();
      }
      return GSMART_OK;
    };
    TRY(run_cached((plan->uid << 3) | (uint64_t)(1 + mode), flags & GSMART_COUNT_ONLY, body));
    ctr_pinned = true;
    if (mode == M_SORT_BIG) {
      // rows arrive in trie (pi-lexicographic) order: the longest tail of columns whose
      // levels already increase needs no sort pass
      std::vector<uint32_t> col_level(nc);
      for (uint32_t k = 0; k < L; k++) col_level[col_of_level[k]] = k;
      uint32_t n_key = nc - 1;  // columns [n_key, nc) have increasing levels
      while (n_key > 0 && col_level[n_key - 1] < col_level[n_key]) n_key--;
      void* tmp = sl.p2 + al(n_rows * nc * 4);
      prof.begin(K_SORT_ROWS);
      CU(sort_rows((const uint32_t*)sl.p2, R->d_rows, n_rows, nc, n_key, bits_for(ctx->N - 1), tmp, tb, sl.st,
                   &launches[K_SORT_ROWS], reinterpret_cast<int*>(sl.d_ctr + 50), true, true));
      prof.end();
    }
    return GSMART_OK;
  }

  // after the slot stream drained
  // world > 1: every rank holds the rows of its own root bindings; rank 0
  // gathers them (rank order = ascending root ranges) and sorts unless the trie
  // order is already the column order.  All ranks report the global count.
  gsmart_status gather_rows() {
    std::vector<unsigned long long> cnt;
    TRY(coll_allgather_host(ctx, sl.st, R->n_rows, &cnt));
    uint64_t total = 0;
    for (auto c : cnt) total += c;
    const uint32_t nc = R->n_cols;
    if (!(flags & GSMART_COUNT_ONLY) && total && nc) {
      std::vector<unsigned long long> bytes(ctx->world);
      for (int q = 0; q < ctx->world; q++) bytes[q] = cnt[q] * nc * 4;
      uint32_t* all = nullptr;
      if (ctx->rank == 0) TRY(alloc_result((void**)&all, total * nc * 4));
      prof.begin(K_COLLECTIVE);
      if (peer_mode()) TRY(gather_peer(R->d_rows, all, bytes));
      else TRY(coll_gather_root(ctx, sl.st, R->d_rows, all, bytes));
      prof.end();
      launches[K_COLLECTIVE]++;
      if (ctx->rank == 0 && !identity) {
        uint32_t* sorted = nullptr;
        TRY(alloc_result((void**)&sorted, total * nc * 4));
        const size_t tb = sort_rows_tmp_bytes(total, nc);
        void* tmp = nullptr;
        TRY(sc.get((char**)&tmp, tb));
        CU(sort_rows(all, sorted, total, nc, nc, bits_for(ctx->N - 1), tmp, tb, sl.st, &launches[K_SORT_ROWS]));
        all = sorted;
      }
      R->d_rows = ctx->rank == 0 ? all : nullptr;  // rows live on rank 0
      CU(cudaStreamSynchronize(sl.st));
    }
    R->n_rows = total;
    return GSMART_OK;
  }

  // peer exchange: every rank puts its rows into its chunk of a symmetric gather
  // buffer; rank 0 copies the chunks (NVLink reads) in rank order
  gsmart_status gather_peer(const uint32_t* mine, uint32_t* all, const std::vector<unsigned long long>& bytes) {
    unsigned long long need = 0;
    for (auto b : bytes) need = std::max(need, b);
    if (need > sl.gath_cap) {  // collective: every rank sees the same byte counts
      const uint64_t g = sym_granularity(ctx);
      const uint64_t cap = std::max<uint64_t>((need + need / 4 + g - 1) / g * g, g);
      if (sl.gath.va) sym_free(ctx, &sl.gath);
      sl.gath_cap = 0;
      TRY(sym_alloc(ctx, (uint64_t)ctx->rank * cap, cap, &sl.gath));
      sl.gath_cap = cap;
    }
    const int me = ctx->rank;
    if (bytes[me]) CU(cudaMemcpyAsync(sl.gath.local(), mine, bytes[me], cudaMemcpyDeviceToDevice, sl.st));
    CU(cudaStreamSynchronize(sl.st));
    TRY(host_barrier(ctx));
    if (me == 0) {
      uint64_t off = 0;
      for (int q = 0; q < ctx->world; q++) {
        if (bytes[q])
          CU(cudaMemcpyAsync((char*)all + off, (const char*)(sl.gath.va + sl.gath.off[q]), bytes[q],
                             cudaMemcpyDeviceToDevice, sl.st));
        off += bytes[q];
      }
      CU(cudaStreamSynchronize(sl.st));
    }
    return host_barrier(ctx);  // no rank rewrites its chunk before rank 0 has read it
  }

  gsmart_status finalize() {
    prof.flush();
    static const bool trace = getenv("GSMART_TRACE") != nullptr;
    if (trace && ctx->world > 1)
      fprintf(stderr, "[gsmart] rank %d plan %llu: barrier gens %llu..%llu, lb epochs %u..%u\n", ctx->rank,
              (unsigned long long)plan->uid, (unsigned long long)sl.bar_base + 1,
              (unsigned long long)(sl.bar_base + sl.bar_off), sl.seq_base, sl.seq_base + sl.seq_off);
    if (seq_open) {
      end_seq(sl);
      seq_open = false;
    }
    if (state == S_PHASE2 && R->n_rows && !fact) {
      for (uint32_t k = 0; k < L && k < (uint32_t)R->levels.size(); k++) {
        R->levels[k].n = sl.h_pin[128 + k];
        R->stats.level_alive[k] = sl.h_pin[128 + k];
      }
    }
    if (ctx->world > 1 && state == S_PHASE2) {
      TRY(gather_rows());
      R->host_valid = R->n_rows == 0 && !(flags & GSMART_COUNT_ONLY);  // rank 0's gathered rows are copied on demand
    }
    unsigned long long c[C_NCTR];
    if (ctr_pinned) memcpy(c, sl.h_pin + 192, C_NCTR * 8);
    else CU(cudaMemcpy(c, sl.d_ctr, C_NCTR * 8, cudaMemcpyDeviceToHost));
    auto& st = R->stats;
    st.filter_rows = c[C_FILTER_ROWS];
    st.filter_entries = c[C_FILTER_SCANNED];
    st.seed_entries = c[C_SEED];
    st.expand_entries = c[C_EXPAND];
    st.closing_checks = c[C_CLOSING];
    if (ctx->world > 1) {  // each exchange brings every other rank's slice of the center's bitmap
      uint64_t other = 0;
      for (int q = 0; q < ctx->world; q++)
        if (q != ctx->rank) other += part_word_hi(ctx, q) - part_word_lo(ctx, q);
      st.allgather_bytes = 4 * other * n_exchanges;
    }
    st.edges_evaluated = c[C_FILTER_MATCHED] + c[C_SEED] + c[C_EXPAND] + c[C_PUSH];
    const uint64_t pb = (uint64_t)ctx->pred_bytes;
    // algorithmic bytes: what each step must move
    uint64_t parents = 0, children = 0;
    // launches skipped on the device (SkipIf) move no bitmap bytes
    const uint64_t skipped = std::min<uint64_t>(c[C_FILTER_SKIPPED], filter_main);
    st.bytes[K_FILTER] = 4 * c[C_FILTER_MASKED] + 8 * c[C_FILTER_ROWS] + pb * c[C_FILTER_SCANNED] + 4 * c[C_FILTER_MATCHED] +
                         8ull * (filter_main - skipped) * W +
                         8 * c[C_PUSH] + 12ull * push_and * W;  // push: (s, o) per entry; AND: cand r/w + sat
    st.bytes[K_SEED] = 4 * c[C_SEED];
    // per expanded level: its parents (the previous trie level, or the parent
    // occurrence) — a fused functional level does the segment work in the emit kernel
    uint64_t parents_fused = 0;
    for (uint32_t k = 1; k < st.n_levels && k < GSMART_MAX_LEVELS; k++) {
      const uint32_t pk = fact ? (uint32_t)occ[k].par : k - 1;
      const uint64_t np = st.level_nodes[pk];
      if (k < fused_lv.size() && fused_lv[k]) parents_fused += np;
      else parents += np;
      children += st.level_nodes[k];
    }
    st.bytes[K_EXPAND_SEG] = 12 * parents;
    st.bytes[K_EXPAND_EMIT] = 4 * c[C_EXPAND] + 9 * children + 8 * parents + 12 * parents_fused;
    // a5: every compaction reads this rank's bitmap range once and writes 4 B per id
    // (row lists of the groups + level 0); initialisation writes the bitmaps once
    const uint64_t range_bytes = 4ull * (whi - wlo);
    const uint64_t compact_run = (uint64_t)launches[K_COMPACT] - std::min<uint64_t>(skipped, launches[K_COMPACT]);
    st.bytes[K_COMPACT] = range_bytes * compact_run + 4 * (c[C_FILTER_ROWS] + st.level_nodes[0]);
    st.bytes[K_BITMAP] = 4ull * Wpad * plan->vars.size();
    // a8: mark reads parent (4) + alive (1) per child; compaction reads bind/parent/alive
    // (9) and writes newidx (4) per node, plus 8 B per surviving node
    // a9: 4 B per output cell + 8 B per surviving trie node read while walking parents
    uint64_t prune = 0, alive = 0;
    for (uint32_t k = 0; k < st.n_levels && k < GSMART_MAX_LEVELS; k++) {
      prune += (k ? 5 : 0) * st.level_nodes[k] + 13 * st.level_nodes[k] + 8 * st.level_alive[k];
      alive += st.level_alive[k];
    }
    st.bytes[K_PRUNE] = state == S_PHASE2 ? prune : 0;
    st.bytes[K_ENUMERATE] = launches[K_ENUMERATE] ? 4ull * R->n_rows * R->n_cols + 8 * alive : 0;
    for (int i = 0; i < GSMART_NKERNELS; i++) st.launches[i] = (uint64_t)launches[i];
    for (int i = 0; i < GSMART_NKERNELS; i++) st.kernel_names[i] = kKernelNames[i];
    if (!(flags & (GSMART_KEEP_ON_DEVICE | GSMART_COUNT_ONLY)) && R->d_rows && R->n_rows) {
      if (ctx->world == 1 || ctx->rank == 0) TRY(rows_to_host(ctx, R, sl.st));
    } else if (!R->n_rows && !(flags & GSMART_COUNT_ONLY)) {
      R->host_valid = true;
    }
    st.ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    state = S_DONE;
    return GSMART_OK;
  }
};

gsmart_status check_plan(gsmart_ctx* ctx, const gsmart_plan_t* plan, uint32_t flags) {
  if (!plan) FAIL(GSMART_E_INVALID_ARG, "null plan");
  for (auto& e : plan->edges)
    if (e.pred > ctx->P) FAIL(GSMART_E_INVALID_ARG, "query predicate id > n_predicates");
  // every label the plan reads must be held by that format (keep-sets)
  std::set<uint32_t> acc[2];
  plan_access(*plan, (flags & GSMART_BACK_EDGES) != 0, &acc[0], &acc[1]);
  for (int f = 0; f < 2; f++)
    if (ctx->f[f].built)
      for (uint32_t l : acc[f])
        if (l < ctx->keep[f].size() && !ctx->keep[f][l])
          FAIL(GSMART_E_STATE, std::string("the plan reads predicate ") + std::to_string(l) + " in the " +
                                   (f ? "CSC" : "CSR") + " LSpM, which the build did not keep");
  if (!ctx->f[1].built) {  // CSR-only LSpM: a direction-driven plan reading subject rows only
    bool ok = plan->traversal == GSMART_DIRECTION;
    for (auto& L : plan->levels) ok = ok && (L.tree_edge < 0 || L.dir == OUT);
    if (!ok) FAIL(GSMART_E_STATE, "this plan needs the CSC LSpM (build CSR|CSC, or plan direction-driven after a CSR-only build)");
  }
  return GSMART_OK;
}

gsmart_status run_batch(gsmart_ctx* ctx, const gsmart_plan_t* const* plans, uint32_t n, uint32_t flags,
                        gsmart_result** out) {
  for (uint32_t i = 0; i < n; i++) TRY(check_plan(ctx, plans[i], flags));
  // world > 1: collectives of one plan complete before the next plan starts (same
  // order on every rank), so a batch runs one plan at a time on slot 0
  const uint32_t ns = ctx->world > 1 ? 1u : std::min<uint32_t>(std::max<uint32_t>(n, 1), MAX_SLOTS);
  TRY(ensure_slots(ctx, ns));
  // fork: every slot stream starts after the work already queued on ctx->st
  cudaEvent_t fork;
  CU(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  CU(cudaEventRecord(fork, ctx->st));
  for (uint32_t s = 1; s < ns; s++) CU(cudaStreamWaitEvent(ctx->slots[s]->st, fork, 0));
  cudaEventDestroy(fork);
  gsmart_status status = GSMART_OK;
  for (uint32_t base = 0; base < n && status == GSMART_OK; base += ns) {
    const uint32_t m = std::min(ns, n - base);
    std::vector<std::unique_ptr<gsmart_result>> res(m);
    std::vector<std::unique_ptr<Exec>> ex(m);
    for (uint32_t i = 0; i < m; i++) {
      res[i] = std::make_unique<gsmart_result>();
      gsmart_result* R = res[i].get();
      const gsmart_plan_t* p = plans[base + i];
      R->ctx = ctx;
      R->st = ctx->slots[i]->st;
      R->n_cols = (uint32_t)p->vars.size();
      R->var_of_col = p->vars;
      R->count_only = (flags & GSMART_COUNT_ONLY) != 0;
      for (int k = 0; k < GSMART_NKERNELS; k++) R->stats.kernel_names[k] = kKernelNames[k];
      ex[i] = std::make_unique<Exec>(ctx, *ctx->slots[i], p, flags, R);
    }
    if (m > 1) {
      // concurrent plans: the costliest one (by the previous run's work) sizes its
      // grids for the whole device, the others for half of it, so their latency-
      // bound kernels co-reside instead of each filling every SM with waiting CTAs
      // (WatDiv-100M batch 4.41 vs 4.66 ms with every plan at half; LUBM-10k needs
      // its dominant L1 at full width).  GSMART_SM_SHARE=f sets the others' share.
      const char* ev = getenv("GSMART_SM_SHARE");
      const double f = ev ? atof(ev) : 0.5;
      unsigned long long top = 0;
      uint32_t top_i = m;
      for (uint32_t i = 0; i < m; i++) {
        auto it = ctx->plan_cost.find(plans[base + i]->uid);
        if (it != ctx->plan_cost.end() && it->second >= top) {
          top = it->second;
          top_i = i;
        }
      }
      if (top_i < m && f > 0 && f < 1)
        for (uint32_t i = 0; i < m; i++)
          if (i != top_i) ex[i]->smc = std::max(16, (int)(ctx->sm_count * f));
    }
    std::vector<gsmart_status> st(m, GSMART_OK);
    static const bool trace = getenv("GSMART_TRACE") != nullptr;
    const auto tb = std::chrono::steady_clock::now();
    auto us = [&] { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tb).count(); };
    // start the plans that were the most work last time first (the batch ends
    // with its longest plan; slots keep their plan, so cached graphs stay valid)
    std::vector<uint32_t> order(m);
    for (uint32_t i = 0; i < m; i++) order[i] = i;
    auto cost = [&](uint32_t i) {
      auto it = ctx->plan_cost.find(plans[base + i]->uid);
      return it == ctx->plan_cost.end() ? 0ull : it->second;
    };
    std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) { return cost(x) > cost(y); });
    for (uint32_t i : order) st[i] = ex[i]->start();
    for (uint32_t i : order)  // speculative phase 2s, queued while the phase 1s run
      if (st[i] == GSMART_OK && ex[i]->spec_pending) st[i] = ex[i]->speculate();
    if (trace) fprintf(stderr, "[gsmart] %u plans: phase-1 launched at %.1f us\n", m, us());
    // serve the plans in completion order (a slow plan never holds back the
    // host work of the others): expansion readback -> re-launch on overflow or
    // phase 2; then, per drained stream, finalize
    auto expanding = [&](uint32_t i) { return st[i] == GSMART_OK && ex[i]->state == Exec::S_EXPANDING; };
    std::vector<uint8_t> done(m, 0);
    for (uint32_t left = m; left;) {
      bool progressed = false;
      for (uint32_t i = 0; i < m; i++) {
        if (done[i]) continue;
        if (expanding(i)) {
          const cudaError_t e = cudaEventQuery(ex[i]->sl.ev);
          if (e == cudaErrorNotReady) continue;
          progressed = true;
          if (e != cudaSuccess) {
            st[i] = cuda_fail(ctx, e, "expansion event", __LINE__);
          } else {
            if (trace) fprintf(stderr, "[gsmart]   plan %u expansion done at %.1f us\n", i, us());
            st[i] = ex[i]->after_expand();
            if (trace) fprintf(stderr, "[gsmart]   plan %u phase-2 launched at %.1f us\n", i, us());
          }
          continue;  // relaunched (still expanding) or phase 2 queued: drain later
        }
        const cudaError_t e = cudaStreamQuery(ex[i]->sl.st);
        if (e == cudaErrorNotReady) continue;
        progressed = true;
        if (trace) fprintf(stderr, "[gsmart]   plan %u drained at %.1f us\n", i, us());
        if (e != cudaSuccess && st[i] == GSMART_OK) st[i] = cuda_fail(ctx, e, "execute sync", __LINE__);
        if (st[i] == GSMART_OK && ex[i]->spec) {
          ex[i]->spec = false;
          if (!ex[i]->spec_holds()) {
            if (trace) fprintf(stderr, "[gsmart]   plan %u mis-speculated at %.1f us\n", i, us());
            st[i] = ex[i]->redo_phase2();
            if (st[i] == GSMART_OK) continue;  // expanding again or phase 2 queued: drain later
          }
        }
        const bool reached_p2 = ex[i]->state == Exec::S_PHASE2;
        if (st[i] == GSMART_OK) st[i] = ex[i]->finalize();
        else ex[i]->prof.flush();
        if (st[i] == GSMART_OK && reached_p2 && (ctx->world == 1 || ctx->exchange == GSMART_XCHG_PEER)) {
          auto& g = ctx->p2_guess[plans[base + i]->uid];
          g.gen = ctx->lspm_gen;
          g.flags = flags;
          g.F = ex[i]->F;
        }
        if (st[i] == GSMART_OK) {
          const gsmart_stats& s = res[i]->stats;
          unsigned long long c = s.edges_evaluated + s.filter_rows;
          for (uint32_t k = 0; k < s.n_levels && k < GSMART_MAX_LEVELS; k++) c += s.level_nodes[k];
          ctx->plan_cost[plans[base + i]->uid] = c;
        }
        if (trace) fprintf(stderr, "[gsmart]   plan %u finalized at %.1f us\n", i, us());
        done[i] = 1;
        left--;
      }
      if (!progressed) std::this_thread::yield();
    }
    for (uint32_t i = 0; i < m; i++) {
      if (ex[i]->seq_open) end_seq(ex[i]->sl);  // epochs of a failed run are never reused
      ex[i].reset();  // frees stream-ordered scratch
      if (st[i] == GSMART_OK || (st[i] == GSMART_E_RESULT_OVERFLOW && n == 1)) {
        out[base + i] = res[i].release();
      } else {
        gsmart_result_free(res[i].release());
      }
      if (st[i] != GSMART_OK && status == GSMART_OK) status = st[i];
    }
  }
  // join: later work on ctx->st sees the batch (already drained above)
  return status;
}

}  // namespace

extern "C" gsmart_status gsmart_execute(gsmart_ctx* ctx, const gsmart_plan_t* plan, uint32_t flags,
                                        gsmart_result** out) {
  if (!ctx || !plan || !out) return GSMART_E_INVALID_ARG;
  *out = nullptr;
  if (ctx->poisoned) return GSMART_E_CUDA;
  if (!ctx->f[0].built) FAIL(GSMART_E_STATE, "gsmart_build_lspm must be called first");
  CU(cudaSetDevice(ctx->cfg.device));
  return run_batch(ctx, &plan, 1, flags, out);
}

extern "C" gsmart_status gsmart_execute_batch(gsmart_ctx* ctx, const gsmart_plan_t* const* plans, uint32_t n,
                                              uint32_t flags, gsmart_result** out) {
  if (!ctx || (n && (!plans || !out))) return GSMART_E_INVALID_ARG;
  for (uint32_t i = 0; i < n; i++) out[i] = nullptr;
  if (ctx->poisoned) return GSMART_E_CUDA;
  if (!ctx->f[0].built) FAIL(GSMART_E_STATE, "gsmart_build_lspm must be called first");
  CU(cudaSetDevice(ctx->cfg.device));
  gsmart_status s = run_batch(ctx, plans, n, flags, out);
  if (s != GSMART_OK)
    for (uint32_t i = 0; i < n; i++) {
      gsmart_result_free(out[i]);
      out[i] = nullptr;
    }
  return s;
}
