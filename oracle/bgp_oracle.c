/* ORACLE — test infrastructure only (see oracle/__init__.py).  Not product code.
 *
 * Plain backtracking evaluator of a SPARQL basic graph pattern (BGP) over an
 * RDF triple set: the definition gSmart computes (§2.2, "A
 * set of triple patterns is called basic graph pattern"; "its
 * semantics is the conjunction of these triple patterns").  No blocking, no
 * matrix form, nothing shared with the CUDA path:
 *   1. de-duplicate the triples (set semantics, R5) into sorted SPO and OPS
 *      copies;
 *   2. fix a static variable order (most constrained first — affects speed
 *      only, never the answer);
 *   3. backtrack: a variable's candidates are the entries of one pattern to an
 *      already-bound vertex / constant (equal_range on SPO or OPS), else the
 *      distinct subjects/objects of one of its patterns; every pattern between
 *      the variable and bound vertices (self-loops included) is then checked
 *      by binary search;
 *   4. rows (bindings of the variables in ascending vertex index) are sorted
 *      lexicographically and made distinct.
 * Homomorphism semantics (R6): distinct variables may bind the same entity.
 * Optional OpenMP over the first variable's candidates; the output is sorted,
 * hence independent of the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct { uint32_t a, p, b; } trip_t;

static int cmp_trip(const void* x, const void* y) {
  const trip_t* u = (const trip_t*)x; const trip_t* v = (const trip_t*)y;
  if (u->a != v->a) return u->a < v->a ? -1 : 1;
  if (u->p != v->p) return u->p < v->p ? -1 : 1;
  if (u->b != v->b) return u->b < v->b ? -1 : 1;
  return 0;
}

/* first index with (a,p) >= (x,l) */
static uint64_t lower_ap(const trip_t* t, uint64_t n, uint32_t x, uint32_t l, uint32_t b) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = (lo + hi) / 2;
    int less = t[mid].a < x || (t[mid].a == x && (t[mid].p < l || (t[mid].p == l && t[mid].b < b)));
    if (less) lo = mid + 1; else hi = mid;
  }
  return lo;
}

static int member(const trip_t* spo, uint64_t n, uint32_t s, uint32_t p, uint32_t o) {
  uint64_t i = lower_ap(spo, n, s, p, o);
  return i < n && spo[i].a == s && spo[i].p == p && spo[i].b == o;
}

typedef struct {
  const trip_t *spo, *ops; uint64_t n;
  uint32_t nv;                /* number of query vertices */
  const uint32_t *is_const, *const_id;
  uint32_t ne; const uint32_t *es, *ep, *ed;
  uint32_t nvar;              /* number of variables */
  uint32_t *order;            /* order[d] = vertex index bound at depth d */
  uint32_t *col_of;           /* vertex -> output column (variables) */
  int32_t *gen_edge;          /* per depth: generating edge or -1 */
  uint32_t **free_cands; uint64_t *free_n; /* per depth (gen_edge<0) */
} prob_t;

typedef struct { uint32_t* rows; uint64_t n, cap; uint32_t w; } buf_t;

static void push_row(buf_t* b, const uint32_t* row) {
  if (b->n == b->cap) {
    b->cap = b->cap ? b->cap * 2 : 1024;
    b->rows = (uint32_t*)realloc(b->rows, (size_t)b->cap * b->w * sizeof(uint32_t) + 4);
  }
  if (b->w) memcpy(b->rows + (size_t)b->n * b->w, row, b->w * sizeof(uint32_t));
  b->n++;
}

static int check_edges(const prob_t* P, const uint32_t* val, const uint8_t* bound, uint32_t v) {
  for (uint32_t k = 0; k < P->ne; k++) {
    uint32_t a = P->es[k], b = P->ed[k];
    if (a != v && b != v) continue;
    if (!bound[a] || !bound[b]) continue;
    if (!member(P->spo, P->n, val[a], P->ep[k], val[b])) return 0;
  }
  return 1;
}

static void rec(const prob_t* P, uint32_t d, uint32_t* val, uint8_t* bound, buf_t* out, uint32_t* row) {
  if (d == P->nvar) {
    for (uint32_t i = 0; i < P->nv; i++)
      if (!P->is_const[i]) row[P->col_of[i]] = val[i];
    push_row(out, row);
    return;
  }
  uint32_t v = P->order[d];
  int32_t g = P->gen_edge[d];
  if (g < 0) {
    for (uint64_t i = 0; i < P->free_n[d]; i++) {
      val[v] = P->free_cands[d][i]; bound[v] = 1;
      if (check_edges(P, val, bound, v)) rec(P, d + 1, val, bound, out, row);
      bound[v] = 0;
    }
    return;
  }
  /* generating pattern: among v's patterns to bound vertices, the one with
     the fewest entries (speed only; every pattern is checked anyway) */
  const trip_t* t = NULL; uint32_t key = 0, l = 0; uint64_t i = 0, iend = 0, best = UINT64_MAX;
  for (uint32_t k = 0; k < P->ne; k++) {
    uint32_t a = P->es[k], b = P->ed[k];
    if (a == b || (a != v && b != v)) continue;
    uint32_t other = a == v ? b : a;
    if (!bound[other]) continue;
    const trip_t* tk = (b == v) ? P->spo : P->ops;   /* (bound a)-l->v : objects; v-l->(bound b) : subjects */
    uint32_t kk = val[other];
    uint64_t lo = lower_ap(tk, P->n, kk, P->ep[k], 0);
    uint64_t hi = lower_ap(tk, P->n, kk, P->ep[k] + 1, 0);
    if (P->ep[k] == UINT32_MAX) hi = lower_ap(tk, P->n, kk + 1, 0, 0);
    if (hi - lo < best) { best = hi - lo; t = tk; key = kk; l = P->ep[k]; i = lo; iend = hi; }
  }
  (void)g; (void)key; (void)l;
  for (; i < iend; i++) {
    val[v] = t[i].b; bound[v] = 1;
    if (check_edges(P, val, bound, v)) rec(P, d + 1, val, bound, out, row);
    bound[v] = 0;
  }
}

static int cmp_rows_w;
static int cmp_rows(const void* x, const void* y) {
  const uint32_t* u = (const uint32_t*)x; const uint32_t* v = (const uint32_t*)y;
  for (int i = 0; i < cmp_rows_w; i++)
    if (u[i] != v[i]) return u[i] < v[i] ? -1 : 1;
  return 0;
}

typedef struct { trip_t *spo, *ops; uint64_t m; } oracle_index_t;

/* Index build: de-duplicated, sorted SPO and OPS copies (step 1). */
void* oracle_index_create(const uint32_t* s, const uint32_t* p, const uint32_t* o, uint64_t n) {
  oracle_index_t* ix = (oracle_index_t*)malloc(sizeof(oracle_index_t));
  trip_t* spo = (trip_t*)malloc((n ? n : 1) * sizeof(trip_t));
  trip_t* ops = (trip_t*)malloc((n ? n : 1) * sizeof(trip_t));
  for (uint64_t i = 0; i < n; i++) { spo[i].a = s[i]; spo[i].p = p[i]; spo[i].b = o[i]; }
  qsort(spo, n, sizeof(trip_t), cmp_trip);
  uint64_t m = 0;
  for (uint64_t i = 0; i < n; i++)
    if (m == 0 || cmp_trip(&spo[m - 1], &spo[i]) != 0) spo[m++] = spo[i];
  for (uint64_t i = 0; i < m; i++) { ops[i].a = spo[i].b; ops[i].p = spo[i].p; ops[i].b = spo[i].a; }
  qsort(ops, m, sizeof(trip_t), cmp_trip);
  ix->spo = spo; ix->ops = ops; ix->m = m;
  return ix;
}

void oracle_index_free(void* h) {
  oracle_index_t* ix = (oracle_index_t*)h;
  if (!ix) return;
  free(ix->spo); free(ix->ops); free(ix);
}

/* Query (steps 2-4).  Returns 0 on success.  *rows_out: malloc'd row-major
 * uint32[n_rows * n_vars] (free with oracle_free).  n_threads <= 0: OpenMP default. */
int oracle_index_query(void* h, uint32_t nv, const uint32_t* is_const, const uint32_t* const_id,
                       uint32_t ne, const uint32_t* es, const uint32_t* ep, const uint32_t* ed,
                       int n_threads, uint32_t** rows_out, uint64_t* n_rows_out, uint32_t* n_cols_out) {
  oracle_index_t* ix = (oracle_index_t*)h;
  trip_t* spo = ix->spo; trip_t* ops = ix->ops; uint64_t m = ix->m;
  *rows_out = NULL; *n_rows_out = 0;
  prob_t P; memset(&P, 0, sizeof P);
  P.spo = spo; P.ops = ops; P.n = m; P.nv = nv; P.is_const = is_const; P.const_id = const_id;
  P.ne = ne; P.es = es; P.ep = ep; P.ed = ed;
  P.col_of = (uint32_t*)calloc(nv + 1, sizeof(uint32_t));
  uint32_t nvar = 0;
  for (uint32_t i = 0; i < nv; i++) if (!is_const[i]) P.col_of[i] = nvar++;
  P.nvar = nvar;
  *n_cols_out = nvar;
  P.order = (uint32_t*)calloc(nvar + 1, sizeof(uint32_t));
  P.gen_edge = (int32_t*)calloc(nvar + 1, sizeof(int32_t));
  P.free_cands = (uint32_t**)calloc(nvar + 1, sizeof(uint32_t*));
  P.free_n = (uint64_t*)calloc(nvar + 1, sizeof(uint64_t));

  /* const-const patterns: boolean guards */
  int guard = 1;
  for (uint32_t k = 0; k < ne; k++)
    if (is_const[es[k]] && is_const[ed[k]] && !member(spo, m, const_id[es[k]], ep[k], const_id[ed[k]])) guard = 0;

  /* static order: greedily the variable with most patterns to bound/constant
     vertices, then most patterns, then lowest index */
  uint8_t* placed = (uint8_t*)calloc(nv + 1, 1);
  for (uint32_t i = 0; i < nv; i++) if (is_const[i]) placed[i] = 1;
  for (uint32_t d = 0; d < nvar; d++) {
    int64_t best = -1, bc = -1, bdeg = -1;
    for (uint32_t v = 0; v < nv; v++) {
      if (placed[v]) continue;
      int64_t c = 0, deg = 0;
      for (uint32_t k = 0; k < ne; k++) {
        if (es[k] != v && ed[k] != v) continue;
        deg++;
        uint32_t other = es[k] == v ? ed[k] : es[k];
        if (other != v && placed[other]) c++;
      }
      if (c > bc || (c == bc && deg > bdeg)) { best = v; bc = c; bdeg = deg; }
    }
    uint32_t v = (uint32_t)best;
    P.order[d] = v;
    P.gen_edge[d] = -1;
    for (uint32_t k = 0; k < ne; k++) {
      uint32_t other = es[k] == v ? ed[k] : (ed[k] == v ? es[k] : v);
      if (other != v && placed[other]) { P.gen_edge[d] = (int32_t)k; break; }
    }
    if (P.gen_edge[d] < 0) {
      /* distinct subjects/objects of v's first pattern (any self-loop works too) */
      int32_t k0 = -1;
      for (uint32_t k = 0; k < ne; k++) if (es[k] == v || ed[k] == v) { k0 = (int32_t)k; break; }
      uint64_t cnt = 0;
      uint32_t* c = (uint32_t*)malloc((m ? m : 1) * sizeof(uint32_t));
      if (k0 >= 0) {
        int as_subject = es[k0] == v;
        const trip_t* t = as_subject ? spo : ops;  /* t[i].a = role value */
        for (uint64_t i = 0; i < m; i++)
          if (t[i].p == ep[k0] && (cnt == 0 || c[cnt - 1] != t[i].a)) c[cnt++] = t[i].a;
      }
      P.free_cands[d] = c; P.free_n[d] = cnt;
    }
    placed[v] = 1;
  }

  uint32_t* val = (uint32_t*)calloc(nv + 1, sizeof(uint32_t));
  uint8_t* bound0 = (uint8_t*)calloc(nv + 1, 1);
  for (uint32_t i = 0; i < nv; i++) if (is_const[i]) { val[i] = const_id[i]; bound0[i] = 1; }

  buf_t all; memset(&all, 0, sizeof all); all.w = nvar;
  if (guard) {
    if (nvar == 0) {
      uint32_t dummy = 0; push_row(&all, &dummy);
    } else {
      /* candidates of depth 0 */
      uint32_t v0 = P.order[0];
      uint64_t n0; uint32_t* c0 = NULL; int own = 0;
      if (P.gen_edge[0] < 0) { c0 = P.free_cands[0]; n0 = P.free_n[0]; }
      else {
        int32_t g = P.gen_edge[0];
        uint32_t a = es[g], l = ep[g], b = ed[g];
        const trip_t* t = (b == v0) ? spo : ops; uint32_t key = (b == v0) ? val[a] : val[b];
        uint64_t i = lower_ap(t, m, key, l, 0), j = i;
        while (j < m && t[j].a == key && t[j].p == l) j++;
        n0 = j - i; c0 = (uint32_t*)malloc((n0 ? n0 : 1) * sizeof(uint32_t)); own = 1;
        for (uint64_t k = 0; k < n0; k++) c0[k] = t[i + k].b;
      }
      int nth = 1;
#ifdef _OPENMP
      nth = n_threads > 0 ? n_threads : omp_get_max_threads();
#endif
      buf_t* bufs = (buf_t*)calloc(nth, sizeof(buf_t));
      for (int t = 0; t < nth; t++) bufs[t].w = nvar;
#ifdef _OPENMP
#pragma omp parallel num_threads(nth)
#endif
      {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        uint32_t* lval = (uint32_t*)malloc((nv + 1) * sizeof(uint32_t));
        uint8_t* lb = (uint8_t*)malloc(nv + 1);
        uint32_t* row = (uint32_t*)malloc((nvar + 1) * sizeof(uint32_t));
        memcpy(lval, val, (nv + 1) * sizeof(uint32_t)); memcpy(lb, bound0, nv + 1);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 64)
#endif
        for (int64_t i = 0; i < (int64_t)n0; i++) {
          lval[v0] = c0[i]; lb[v0] = 1;
          if (check_edges(&P, lval, lb, v0)) rec(&P, 1, lval, lb, &bufs[tid], row);
          lb[v0] = 0;
        }
        free(lval); free(lb); free(row);
      }
      for (int t = 0; t < nth; t++) {
        for (uint64_t r = 0; r < bufs[t].n; r++) push_row(&all, bufs[t].rows + (size_t)r * nvar);
        free(bufs[t].rows);
      }
      free(bufs);
      if (own) free(c0);
    }
  }
  if (nvar > 0 && all.n > 1) {
    cmp_rows_w = (int)nvar;
    qsort(all.rows, all.n, nvar * sizeof(uint32_t), cmp_rows);
    uint64_t u = 0;
    for (uint64_t r = 0; r < all.n; r++)
      if (u == 0 || memcmp(all.rows + (size_t)(u - 1) * nvar, all.rows + (size_t)r * nvar, nvar * 4) != 0) {
        if (u != r) memmove(all.rows + (size_t)u * nvar, all.rows + (size_t)r * nvar, nvar * 4);
        u++;
      }
    all.n = u;
  }
  *rows_out = all.rows ? all.rows : (uint32_t*)malloc(4);
  *n_rows_out = all.n;
  for (uint32_t d = 0; d < nvar; d++) free(P.free_cands[d]);
  free(P.free_cands); free(P.free_n); free(P.order); free(P.gen_edge); free(P.col_of);
  free(placed); free(val); free(bound0);
  return 0;
}


/* Convenience: index + query + free. */
int oracle_bgp(const uint32_t* s, const uint32_t* p, const uint32_t* o, uint64_t n,
               uint32_t nv, const uint32_t* is_const, const uint32_t* const_id,
               uint32_t ne, const uint32_t* es, const uint32_t* ep, const uint32_t* ed,
               int n_threads, uint32_t** rows_out, uint64_t* n_rows_out, uint32_t* n_cols_out) {
  void* ix = oracle_index_create(s, p, o, n);
  int rc = oracle_index_query(ix, nv, is_const, const_id, ne, es, ep, ed, n_threads,
                              rows_out, n_rows_out, n_cols_out);
  oracle_index_free(ix);
  return rc;
}

void oracle_free(void* p) { free(p); }
