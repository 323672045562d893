/* gsmart.h — C ABI of the B200-native gSmart hot path.
 *
 * Method: gSmart, "An Efficient SPARQL Query Engine Using Sparse Matrix
 * Algebra" (arXiv 2106.14038; /root/reference/PAPER.md, cited as P:L<line>).
 * The library answers SPARQL basic graph patterns (BGPs) over an RDF
 * triple set with the paper's matrix-algebra method: LSpM storage (§6.2),
 * degree-driven planning (§6.1.2), grouped incident-edge evaluation (§5) as
 * label-filtered boolean SpMVs over candidate bitmaps, tree-based binding
 * storage (§7.1) with pre-pruning (§7.2.2) and bottom-up tree pruning
 * (§8.1 steps 3-4), and returns the solution rows.  All steps of
 * gsmart_build_lspm and gsmart_execute run as CUDA kernels for sm_100a; there
 * is no CPU fallback (a missing GPU is GSMART_E_CUDA).
 *
 * Call order (P:L263-L289 phase order):
 *   gsmart_create -> gsmart_load_triples -> gsmart_build_lspm
 *   -> gsmart_plan(query graph) -> gsmart_execute -> gsmart_result_*
 *
 * Conventions
 *  - Every call returns gsmart_status; nothing throws or aborts across the ABI.
 *    After an error, gsmart_last_error(ctx) gives a message.  A failed CUDA
 *    call poisons the context (all later calls return GSMART_E_CUDA).
 *  - Ids: entities are 0-based < n_entities, predicates 1-based
 *    <= n_predicates.  Triples are a set: duplicates are removed
 *    (reading R5 of DESIGN.md).
 *  - Ownership: input pointers are borrowed for the duration of the call only.
 *    ctx / plan / result objects are library-owned and released with their
 *    *_destroy / *_free call.  Pointers returned by gsmart_result_* stay valid
 *    until gsmart_result_free.  A plan is immutable and reusable.  A ctx is not
 *    thread-safe: one ctx per GPU per process.
 *  - Query semantics ("the conjunction of these triple patterns"):
 *    solutions are all mappings of the query's variables to entity ids such
 *    that every pattern is a triple of the set (homomorphism, reading R6).
 *    Rows list the bindings of the variable vertices in ascending vertex
 *    index, sorted lexicographically ascending; rows are distinct.
 *  - An empty result is GSMART_OK with 0 rows.  A constant id >= n_entities
 *    or absent from the data yields an empty result, not an error.  A query
 *    with no variables yields one empty row if all its patterns hold, else 0.
 */
#ifndef GSMART_H
#define GSMART_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSMART_ABI_VERSION 3

typedef enum {
  GSMART_OK = 0,
  GSMART_E_INVALID_ARG = -1,     /* bad pointer, size, id, or query shape */
  GSMART_E_STATE = -2,           /* call-order violation (e.g. execute before build) */
  GSMART_E_OOM = -3,             /* device allocation failed */
  GSMART_E_CUDA = -4,            /* CUDA error / no device; ctx is poisoned */
  GSMART_E_NCCL = -5,            /* collective failure (world > 1) */
  GSMART_E_UNSUPPORTED = -6,     /* variable predicate, direction-driven plan with constants, too many levels */
  GSMART_E_RESULT_OVERFLOW = -7  /* rows (or a trie level) > max_result_rows; n_rows still reported */
} gsmart_status;

/* pointer kinds for gsmart_load_triples */
#define GSMART_PTR_HOST 1u
#define GSMART_PTR_DEVICE 2u
/* LSpM formats (P:L411 LSpM_CSR, P:L432 LSpM_CSC) */
#define GSMART_CSR 1u
#define GSMART_CSC 2u
/* traversal */
#define GSMART_DEGREE 0u     /* degree-driven, §6.1.2 (supported) */
#define GSMART_DIRECTION 1u  /* direction-driven, §6.1.1 (GSMART_E_UNSUPPORTED in this version) */
/* execute flags */
#define GSMART_COUNT_ONLY 1u      /* stop after pruning: n_rows only, no row enumeration */
#define GSMART_KEEP_ON_DEVICE 2u  /* do not copy rows to host (use gsmart_result_rows_device) */
#define GSMART_NO_REFINE 4u       /* no backward group re-evaluation (the default since ABI 3; wins over GSMART_REFINE) */
#define GSMART_PROFILE 8u         /* per-kernel CUDA-event timing into gsmart_stats (no graph replay) */
#define GSMART_KEEP_CANDIDATES 16u /* keep the candidate bitmaps for gsmart_result_candidates */
#define GSMART_NO_GRAPH 32u       /* launch kernels one by one instead of replaying the plan's CUDA graph */
#define GSMART_NO_SPECULATE 64u   /* always wait for the level sizes before pruning/rows (no speculative phase 2) */
#define GSMART_BACK_EDGES 128u    /* every evaluation of a group also tests the center's already-evaluated patterns
                                     against the earlier centers' bitmaps (Eq. 16 over Eq. 14 binding vectors,
                                     DESIGN.md R-back): tighter candidate sets, more work per group */
#define GSMART_REFINE 512u        /* after the groups in plan order (each evaluated once), re-evaluate them in
                                     reverse plan order (DESIGN.md R-refine): tighter candidate sets before the
                                     expansion, same rows; measured slower on WatDiv-100M (3.80 vs 3.47 ms) */
#define GSMART_FACTORISED 256u    /* f2: factorised binding trees (§7.1, per-path trees that
                                     share their DFS prefix) instead of the prefix trie: one level per occurrence of
                                     a variable, hanging off its tree parent's level; a pattern that closes onto a
                                     non-parent vertex adds a second occurrence of the variable and Ω pruning
                                     (§8.1) intersects its bindings per root binding; the rows are
                                     enumerated from the pruned trees (combination index -> one node per
                                     occurrence, Ω occurrences equal) and sorted.  COUNT_ONLY without Ω variables
                                     reads the count off the trees (no enumeration).  Same rows as the trie.
                                     world > 1: GSMART_E_UNSUPPORTED.  See gsmart_result_tree. */

typedef struct gsmart_ctx gsmart_ctx;
typedef struct gsmart_plan_s gsmart_plan_t;
typedef struct gsmart_result gsmart_result;
typedef struct gsmart_comm gsmart_comm;

/* how ranks exchange candidate bitmaps when world > 1 */
#define GSMART_XCHG_PEER 0u  /* default: symmetric device memory, the filter clears bits on every rank (peer atomics) */
#define GSMART_XCHG_NCCL 1u  /* baseline: NCCL all-gather (grouped broadcasts) of each rank's slice after a group */

typedef struct {
  int device;                 /* CUDA device ordinal */
  int rank, world;            /* world >= 1 (<= 8); world > 1 = 1-D vertex-range partition of the LSpM */
  const void* nccl_unique_id; /* 128 bytes from gsmart_get_nccl_id on rank 0, broadcast to every rank (processes:
                                 rendezvous of the ranks, and the NCCL communicator when exchange == NCCL;
                                 world == 1: optional, creates a 1-rank NCCL communicator) */
  void* stream;               /* cudaStream_t to run on, or NULL: the library creates one */
  uint64_t max_result_rows;   /* capacity for rows and for each trie level; 0 = 2^31 - 1 */
  gsmart_comm* local_comm;    /* world > 1 inside one process (one thread per rank); else NULL */
  uint32_t exchange;          /* GSMART_XCHG_PEER (default) or GSMART_XCHG_NCCL */
  /* optional device allocator (e.g. a framework's caching allocator): every
   * device buffer the library owns, except the world > 1 symmetric regions
   * (which need the virtual-memory API), comes from alloc(bytes, stream, user)
   * and returns through free(ptr, stream, user), ordered on `stream`.  NULL:
   * the stream-ordered allocator on a memory pool of the context's own. */
  void* (*alloc)(size_t bytes, void* stream, void* user);
  void (*free)(void* ptr, void* stream, void* user);
  void* alloc_user;
} gsmart_config;

/* In-process communicator for `world` ranks driven by `world` host threads of
 * one process (ranks may share a GPU).  Pass it as cfg.local_comm to every
 * rank's gsmart_create; destroy after every rank's context.  Collective calls
 * (execute with world > 1) must be made by all ranks in the same order. */
gsmart_status gsmart_comm_create_local(int world, gsmart_comm** out);
void gsmart_comm_destroy(gsmart_comm* comm);

/* Split points of the 1-D vertex-range partition (host helper, no device; the
 * build uses it on the GPU-computed histogram).  bucket[i] = out+in entries of
 * vertices [i * 2^19, (i+1) * 2^19) (n_buckets = ceil(n_entities / 2^19)).
 * Writes v[0..world]: v[0] = 0, v[world] = n_entities, every inner split a
 * multiple of 2^19 (2 MiB of row pointers = one symmetric mapping granule),
 * non-decreasing, rank r owning [v[r], v[r+1]); split r is the first bucket
 * boundary where the running total reaches r/world of the entries. */
gsmart_status gsmart_partition_split(const uint64_t* bucket, uint32_t n_buckets, uint32_t n_entities, int world,
                                     uint32_t* v);
/* The split points of a built world > 1 context (v[0..world]). */
gsmart_status gsmart_partition_get(const gsmart_ctx* ctx, uint32_t* v);

/* Host-side self-check of the channel that ranks running as separate
 * processes use (no device needed): rendezvous on the 128-byte id, all-gather
 * `value` into all_values[world], and hand one file descriptor per rank to
 * every other rank (the path the symmetric chunks' POSIX handles take).
 * Collective over the `world` processes. */
gsmart_status gsmart_rendezvous_check(const void* id128, int rank, int world, uint64_t value, uint64_t* all_values);

/* ABI version and a build string (static storage). */
int gsmart_abi_version(void);
const char* gsmart_build_info(void);

/* NCCL bootstrap: rank 0 fills 128 bytes to broadcast (e.g. via torch.distributed). */
gsmart_status gsmart_get_nccl_id(void* out128);

/* Context on cfg->device.  Fails with GSMART_E_CUDA if no usable sm_100 device. */
gsmart_status gsmart_create(const gsmart_config* cfg, gsmart_ctx** out);
void gsmart_destroy(gsmart_ctx* ctx);
/* Message of the last error on ctx (static storage if ctx is NULL). */
const char* gsmart_last_error(const gsmart_ctx* ctx);

/* Copy n triples (s[i], p[i], o[i]) into device memory owned by ctx
 * (§6.2.1 steps 1-2 input: encoded ids).  flags: GSMART_PTR_HOST or
 * GSMART_PTR_DEVICE for where s/p/o live.  Ids are validated on the device
 * after the copy (s,o < n_entities, 1 <= p <= n_predicates) ->
 * GSMART_E_INVALID_ARG with no triples loaded (build then gives E_STATE).  Replaces any
 * previously loaded triples and invalidates the LSpM.  n may be 0.
 * n_entities < 2^31, n_predicates <= 65534 (labels are stored as uint8 when
 * n_predicates <= 254, else uint16; the all-ones value is a sentinel).
 * world > 1: every rank passes the SAME full triple set (collective); each
 * rank keeps only its vertex range when the LSpM is built. */
gsmart_status gsmart_load_triples(gsmart_ctx* ctx, const uint32_t* s, const uint32_t* p,
                                  const uint32_t* o, uint64_t n, uint32_t n_entities,
                                  uint32_t n_predicates, uint32_t flags);

/* Build the LSpM (§6.2) on the GPU: keep only triples whose
 * predicate is in keep_preds (host array of n_keep ids; n_keep = 0 keeps all —
 * P:L408 "Read necessary RDF triples where predicates appear in the
 * queries"), de-duplicate, and store CSR (rows = subjects) and/or CSC (rows =
 * objects) as row_ptr[N+1] (uint32), col[M] (uint32) and pred[M] (uint8 when
 * n_predicates <= 254, else uint16), entries sorted by (row, pred, col), so
 * every (row, predicate) pair is one contiguous range.  Empty rows have
 * row_ptr[i] == row_ptr[i+1] (the paper's Mr/Pr row elimination).
 * formats: GSMART_CSR | GSMART_CSC (execute needs both).  Requires kept
 * M < 2^32.  GSMART_E_STATE if no triples were loaded. */
gsmart_status gsmart_build_lspm(gsmart_ctx* ctx, const uint32_t* keep_preds, uint32_t n_keep,
                                uint32_t formats);

/* Query-dependent LSpM with direction-split keep-sets (§6.2; Ex. 6.4
 * the CSR keeps the predicates evaluated along their direction,
 * the CSC those evaluated against it).  keep_csr[n_csr] / keep_csc[n_csc]:
 * predicate ids (host arrays; an empty set stores no triples in that format).
 * Builds both formats and the label-major lists (their union).  Executing a
 * plan that reads a label a format does not hold fails with GSMART_E_STATE
 * (gsmart_plan_keep_sets gives the sets a batch of plans needs). */
gsmart_status gsmart_build_lspm_split(gsmart_ctx* ctx, const uint32_t* keep_csr, uint32_t n_csr,
                                      const uint32_t* keep_csc, uint32_t n_csc);
/* The predicate ids each format must hold to execute the n plans with the
 * execute flags `flags` (GSMART_BACK_EDGES adds the back edges): writes at
 * most cap ids to each of csr_out / csc_out (ascending) and the full counts to
 * *n_csr / *n_csc.  Closing edges are charged to the CSR (the subject's row). */
gsmart_status gsmart_plan_keep_sets(const gsmart_plan_t* const* plans, uint32_t n, uint32_t flags, uint32_t* csr_out,
                                    uint32_t* n_csr, uint32_t* csc_out, uint32_t* n_csc, uint32_t cap);

/* Device view of one built LSpM format (for inspection / parity tests).
 * Pointers are device pointers owned by ctx, valid until the next load/build. */
typedef struct {
  uint32_t n_rows;          /* = n_entities */
  uint64_t nnz;             /* M after keep + de-duplication */
  uint32_t pred_bytes;      /* 1 or 2 */
  const uint32_t* row_ptr;  /* [n_rows + 1] */
  const uint32_t* col;      /* [nnz] */
  const void* pred;         /* [nnz] uint8 or uint16 */
  /* [n_rows] row label signatures: bit (l & 31) set iff the row holds an entry
   * whose label l' has (l' & 31) == (l & 31).  Eqs. 4/5 evaluated
   * for every label at once; exact presence when n_predicates <= 32, else a
   * necessary condition.  The group filter tests it before reading a row. */
  const uint32_t* label_mask;
} gsmart_lspm_view;
gsmart_status gsmart_lspm_get(const gsmart_ctx* ctx, uint32_t format, gsmart_lspm_view* out);

/* Query graph (vertices = variables / constants, edges = patterns). */
typedef struct { uint32_t is_const, const_id; } gsmart_qvertex; /* vertex index = array position */
typedef struct { uint32_t src, pred, dst; } gsmart_qedge;       /* pattern src --pred--> dst */
typedef struct {
  uint32_t n_vertices; const gsmart_qvertex* v;
  uint32_t n_edges; const gsmart_qedge* e;
} gsmart_query;

/* Plan (host only, microseconds; ctx may be NULL; with a ctx whose LSpM is
 * built and n_predicates < 4096, a group's new neighbours enter the trie in
 * ascending expected fan-out — entries per row of the label — so functional
 * patterns precede the fan-out ones; results are identical).  Degree-driven traversal
 * (§6.1.2): constant-incident patterns become seeds (light
 * queries); roots by max unevaluated edges, then max
 * unevaluated out-edges, then lowest index; groups = all unevaluated incident
 * edges of each popped vertex.  Also derives the trie order (variables in
 * first-visit order), tree and closing edges.  Errors:
 * GSMART_E_INVALID_ARG (vertex index out of range, pred == 0, a variable in
 * no pattern, > 32 variables, > 32 edges), GSMART_E_UNSUPPORTED
 * (traversal == GSMART_DIRECTION). */
gsmart_status gsmart_plan(gsmart_ctx* ctx, const gsmart_query* q, uint32_t traversal,
                          gsmart_plan_t** out);
/* JSON description (roots, seeds, groups, levels, pi, tree/closing edges,
 * paths).  Writes at most cap bytes (NUL-terminated when cap > 0) and sets
 * *need to the full length + 1. */
gsmart_status gsmart_plan_describe(const gsmart_plan_t* plan, char* buf, size_t cap, size_t* need);
/* Frees the plan and drops every per-plan cache entry (push/pull decisions,
 * speculative sizes, captured CUDA graphs) of every live context.  Must not run
 * concurrently with an execute of any context. */
void gsmart_plan_free(gsmart_plan_t* plan);

/* Execute plan on the built LSpM: seeds -> grouped incident-edge evaluation
 * (in plan order; with GSMART_REFINE also backward) -> trie
 * expansion with pre-pruning and closing-edge checks -> bottom-up prune ->
 * row enumeration + lexicographic sort.  Collective when world > 1.
 * Synchronises the ctx stream before returning. */
gsmart_status gsmart_execute(gsmart_ctx* ctx, const gsmart_plan_t* plan, uint32_t flags,
                             gsmart_result** out);

/* Execute n independent plans as one batch: up to 16 run concurrently, each on
 * its own CUDA stream with its own workspace, so small (latency-bound) queries
 * overlap on the GPU.  out[i] receives plan i's result, identical to what
 * gsmart_execute(plans[i]) returns.  The batch starts after work already
 * queued on the ctx stream and has completed when the call returns.  On
 * error every out[i] is NULL and the first failing status is returned.
 * Results of a ctx must be freed before gsmart_destroy. */
gsmart_status gsmart_execute_batch(gsmart_ctx* ctx, const gsmart_plan_t* const* plans, uint32_t n,
                                   uint32_t flags, gsmart_result** out);

/* n_rows, n_cols (= number of variables) and var_of_col[n_cols] (query vertex
 * index of each column; host memory owned by the result). */
gsmart_status gsmart_result_shape(const gsmart_result* r, uint64_t* n_rows, uint32_t* n_cols,
                                  const uint32_t** var_of_col);
/* Host rows, row-major uint32[n_rows * n_cols], sorted, distinct (rank 0 when
 * world > 1).  Copied from the device on first call if KEEP_ON_DEVICE. */
gsmart_status gsmart_result_rows(gsmart_result* r, const uint32_t** rows);
/* Device rows (same layout) — valid unless GSMART_COUNT_ONLY. */
gsmart_status gsmart_result_rows_device(const gsmart_result* r, const uint32_t** rows_dev);
/* Candidate bitmap of query vertex `vertex` after the filter schedule:
 * device pointer to ceil(n_entities/32) uint32 words, bit (i & 31) of word
 * (i >> 5) set iff entity i is a candidate.  Only when the execute was given
 * GSMART_KEEP_CANDIDATES (else GSMART_E_INVALID_ARG). */
gsmart_status gsmart_result_candidates(const gsmart_result* r, uint32_t vertex,
                                       const uint32_t** bits_dev, uint32_t* n_words);
/* Trie level k (0 = root level) after pruning: variable vertex, node count and
 * device pointers parent[n] (index into level k-1; undefined for k = 0) and
 * bind[n] (entity id).  Children of a node are contiguous, parent[] is
 * non-decreasing. */
gsmart_status gsmart_result_level(const gsmart_result* r, uint32_t k, uint32_t* vertex,
                                  uint64_t* n, const uint32_t** parent_dev,
                                  const uint32_t** bind_dev);

/* Level k of the result's tree form.  Trie (default): as gsmart_result_level,
 * *parent_level = k - 1 (-1 for k = 0), *alive_dev = NULL (every node alive).
 * GSMART_FACTORISED: occurrence k of the factorised binding trees (§7.1,
 * P:L516) — *parent_level = the occurrence its nodes hang off (-1 for the
 * root occurrence), parent[i] indexes that occurrence's nodes, children of a
 * node are contiguous; alive_dev[i] (uint8) = 1 iff node i survived pre-,
 * bottom-up and Ω pruning; *vertex = the variable (a second occurrence repeats
 * it).  The solutions are, per alive root node, every choice of one alive
 * node per occurrence consistent with the parent links and with equal
 * bindings at every occurrence of a variable.  Device memory owned by the
 * result. */
gsmart_status gsmart_result_tree(const gsmart_result* r, uint32_t k, uint32_t* vertex, int32_t* parent_level,
                                 uint64_t* n, const uint32_t** parent_dev, const uint32_t** bind_dev,
                                 const uint8_t** alive_dev);

#define GSMART_MAX_LEVELS 32
#define GSMART_NKERNELS 16
typedef struct {
  double ms_total;              /* host wall time of gsmart_execute */
  double ms_kernel[GSMART_NKERNELS]; /* per kernel class (GSMART_PROFILE), see kernel_names */
  uint64_t launches[GSMART_NKERNELS];
  uint64_t bytes[GSMART_NKERNELS];   /* algorithmic bytes per kernel class */
  uint64_t edges_evaluated;     /* LSpM entries read whose label matched (seed + filter + push + expansion) */
  uint64_t filter_rows;         /* rows (candidate bits) processed by the group filter */
  uint64_t filter_entries;      /* LSpM entries scanned by the group filter */
  uint64_t seed_entries;        /* segment entries scattered by seeds */
  uint64_t expand_entries;      /* segment entries examined by the expansion */
  uint64_t closing_checks;      /* closing-edge membership tests */
  uint32_t n_levels;
  uint64_t level_nodes[GSMART_MAX_LEVELS];   /* F_k before pruning */
  uint64_t level_alive[GSMART_MAX_LEVELS];   /* F_k after pruning */
  uint64_t allgather_bytes;     /* world > 1 */
  uint32_t spec_phase2;         /* 1: phase 2 (prune, rows) was queued speculatively behind phase 1 */
  uint32_t spec_redo;           /* 1: the speculation guessed wrong sizes; phase 2 was redone */
  uint32_t factorised;          /* 1: GSMART_FACTORISED (levels = occurrences, see gsmart_result_tree) */
  uint32_t n_omega;             /* factorised: second occurrences (Ω) */
  uint64_t combinations;        /* factorised: combinations of the pruned trees (= n_rows when n_omega == 0) */
  const char* kernel_names[GSMART_NKERNELS];
} gsmart_stats;
gsmart_status gsmart_result_stats(const gsmart_result* r, gsmart_stats* out);
void gsmart_result_free(gsmart_result* r);

/* Utility for bindings without a CUDA runtime of their own: synchronous copy
 * of `bytes` from device memory `src_dev` (on ctx's device) into host `dst`. */
gsmart_status gsmart_copy_to_host(gsmart_ctx* ctx, void* dst, const void* src_dev, size_t bytes);

/* ------------------------------------------------------------------ f4: ingest
 * N-Triples read + dictionary encode on the device (§6.2.1 steps 1-2,
 * "Read ... RDF triples", "Encode RDF strings into numeric ids
 * ... the index of subject and object is 0-based, the index of predicate is
 * 1-based").
 *
 * Input subset (R24): lines split at '\n'; a line that is empty or
 * whitespace (' ', '\t', '\r') or whose first non-blank byte is '#' is
 * skipped; otherwise it holds S P O '.' with terms separated by spaces/tabs
 * (none needed after an IRI): S = <IRI> | _:blank, P = <IRI>,
 * O = <IRI> | _:blank | "literal" (backslash escapes) [@lang | ^^<IRI>].
 * Only ' ', '\t', '\r' may follow the '.'.  A term is its exact bytes.
 * Ids follow first appearance in file order, subject before object; entities
 * from 0, predicates from 1 (R24).
 *
 * text: `bytes` bytes (flags GSMART_PTR_HOST or GSMART_PTR_DEVICE), not
 * NUL-terminated; the context copies it (the dictionary's term bytes) and
 * the caller may free it on return.  Loads the encoded triples exactly like
 * gsmart_load_triples (replaces earlier data, invalidates the LSpM) and
 * returns n_triples, n_entities, n_predicates (any out pointer may be NULL).
 * A document without triples returns GSMART_OK with all three 0 and nothing
 * loaded.  Errors: GSMART_E_INVALID_ARG "line L: ..." for the first malformed
 * line L (0-based, counting every '\n'-separated line), nothing loaded;
 * GSMART_E_UNSUPPORTED for > 2^31 - 1 triples, >= 2^31 entities, > 65534
 * predicates, or a 64-bit term-hash collision between two distinct terms
 * (detected exactly by byte comparison; the ids are never silently merged).
 * world must be 1. */
gsmart_status gsmart_ingest_ntriples(gsmart_ctx* ctx, const char* text, uint64_t bytes, uint32_t flags,
                                     uint64_t* n_triples, uint32_t* n_entities, uint32_t* n_predicates);

#define GSMART_DICT_ENTITY 0u
#define GSMART_DICT_PREDICATE 1u
/* Id of a term (exact bytes, `len` of them, host memory) in the dictionary of
 * the last gsmart_ingest_ntriples: *id = entity id (kind ENTITY) or predicate
 * id >= 1 (kind PREDICATE), or 0xFFFFFFFF when the term does not occur (an
 * absent entity used as a query constant gives empty results, R12).
 * GSMART_E_STATE when the loaded data did not come from an ingest. */
gsmart_status gsmart_dict_lookup(gsmart_ctx* ctx, uint32_t kind, const char* term, uint64_t len, uint32_t* id);
/* Bytes of term `id` (inverse of gsmart_dict_lookup) copied to host buf (at
 * most cap bytes); *len = the full term length.  GSMART_E_INVALID_ARG for an
 * id outside [0, n_entities) / [1, n_predicates]; GSMART_E_STATE as above. */
gsmart_status gsmart_dict_term(gsmart_ctx* ctx, uint32_t kind, uint32_t id, char* buf, uint64_t cap, uint64_t* len);
/* Device pointers to the loaded (s, p, o) arrays (n entries each, uint32,
 * context-owned, valid until the next load/ingest or gsmart_destroy). */
gsmart_status gsmart_triples_get(const gsmart_ctx* ctx, const uint32_t** s, const uint32_t** p, const uint32_t** o,
                                 uint64_t* n);

#ifdef __cplusplus
}
#endif
#endif /* GSMART_H */
