// Host query planner: degree-driven traversal (§6.1.2)
// plus the trie order / tree edges / closing edges the level-synchronous
// executor needs.  Host microseconds; no device work.
#include <algorithm>
#include <functional>
#include <cstdio>
#include <set>
#include <sstream>

#include "internal.h"

namespace gsm {

gsmart_status build_plan(const gsmart_query* q, uint32_t traversal, gsmart_plan_t* P, std::string* err,
                         const std::function<double(uint32_t, uint32_t)>* fanout, bool csr_only) {
  if (!q || (q->n_vertices && !q->v) || (q->n_edges && !q->e)) { *err = "null query arrays"; return GSMART_E_INVALID_ARG; }
  if (traversal != GSMART_DEGREE && traversal != GSMART_DIRECTION) { *err = "unknown traversal"; return GSMART_E_INVALID_ARG; }
  P->traversal = traversal;
  const uint32_t n = q->n_vertices, ne = q->n_edges;
  if (ne > 32) { *err = "more than 32 patterns"; return GSMART_E_INVALID_ARG; }
  P->n_vertices = n;
  P->vertices.assign(q->v, q->v + n);
  P->edges.assign(q->e, q->e + ne);
  for (uint32_t k = 0; k < ne; k++) {
    const auto& e = q->e[k];
    if (e.src >= n || e.dst >= n) { *err = "pattern vertex index out of range"; return GSMART_E_INVALID_ARG; }
    if (e.pred == 0 || e.pred > 65535) { *err = "predicate id must be in [1, 65535]"; return GSMART_E_INVALID_ARG; }
  }
  std::vector<bool> is_c(n), used(n, false);
  P->col_of.assign(n, -1);
  for (uint32_t i = 0; i < n; i++) {
    is_c[i] = q->v[i].is_const != 0;
    if (!is_c[i]) { P->col_of[i] = (int32_t)P->vars.size(); P->vars.push_back(i); }
  }
  if (P->vars.size() > GSMART_MAX_LEVELS) { *err = "more than 32 variables"; return GSMART_E_INVALID_ARG; }
  for (uint32_t k = 0; k < ne; k++) { used[q->e[k].src] = used[q->e[k].dst] = true; }
  for (uint32_t v : P->vars)
    if (!used[v]) { *err = "variable vertex occurs in no pattern"; return GSMART_E_INVALID_ARG; }

  // Step 1 (constants variant): W = constants, F = constant-incident edges.
  std::vector<bool> W(n, false), F(ne, false), const_adj(n, false);
  for (uint32_t i = 0; i < n; i++) W[i] = is_c[i];
  for (uint32_t k = 0; k < ne; k++) {
    const auto& e = q->e[k];
    bool cs = is_c[e.src], cd = is_c[e.dst];
    if (cs && cd) { F[k] = true; P->guards.push_back({k, q->v[e.src].const_id, e.pred, q->v[e.dst].const_id}); }
    else if (cs) { F[k] = true; P->seeds.push_back({k, e.dst, e.pred, q->v[e.src].const_id, OUT}); const_adj[e.dst] = true; }
    else if (cd) { F[k] = true; P->seeds.push_back({k, e.src, e.pred, q->v[e.dst].const_id, IN}); const_adj[e.src] = true; }
  }
  auto unev = [&](uint32_t v) {
    uint32_t c = 0;
    for (uint32_t k = 0; k < ne; k++) if (!F[k] && (q->e[k].src == v || q->e[k].dst == v)) c++;
    return c;
  };
  auto unev_out = [&](uint32_t v) {
    uint32_t c = 0;
    for (uint32_t k = 0; k < ne; k++) if (!F[k] && q->e[k].src == v) c++;
    return c;
  };
  auto n_unev = [&]() { uint32_t c = 0; for (uint32_t k = 0; k < ne; k++) c += !F[k]; return c; };

  std::vector<uint32_t> depth(n, 0);
  std::vector<int32_t> first_parent(n, -1);
  if (traversal == GSMART_DIRECTION) {
    // Direction-driven traversal (§6.1.1): a query with constants is
    // planned degree-driven, so it is refused here.
    if (!P->seeds.empty() || !P->guards.empty()) {
      *err = "direction-driven plans take variable-only queries (P:L381)";
      return GSMART_E_UNSUPPORTED;
    }
    auto unev_in = [&](uint32_t v) {
      uint32_t c = 0;
      for (uint32_t k = 0; k < ne; k++) if (!F[k] && q->e[k].dst == v) c++;
      return c;
    };
    while (n_unev() > 0) {
      // Step 2: an unvisited vertex without unevaluated incoming edges, max unevaluated
      // outgoing edges (cyclic variant P:L377: else max unevaluated outgoing), lowest index
      int32_t best = -1;
      uint32_t bo = 0;
      for (int pass = 0; pass < 3 && best < 0; pass++)
        for (uint32_t v = 0; v < n; v++) {
          if ((pass < 2 && W[v]) || unev_out(v) == 0) continue;
          if (pass == 0 && unev_in(v) != 0) continue;
          const uint32_t o = unev_out(v);
          if (best < 0 || o > bo) { best = (int32_t)v; bo = o; }
        }
      const uint32_t root = (uint32_t)best;
      P->roots.push_back(root);
      W[root] = true; depth[root] = 0; first_parent[root] = -1;
      std::vector<uint32_t> S{root};
      while (!S.empty()) {                    // Steps 3-4: all unevaluated OUTGOING edges
        const uint32_t v = S.back(); S.pop_back();
        Group g; g.center = v; g.level = depth[v];
        for (uint32_t k = 0; k < ne; k++)
          if (!F[k] && q->e[k].src == v) g.edges.push_back({k, q->e[k].pred, OUT, q->e[k].dst});
        for (auto& ge : g.edges) F[ge.edge] = true;
        std::vector<uint32_t> fresh;
        for (auto& ge : g.edges)
          if (!W[ge.nbr]) { W[ge.nbr] = true; depth[ge.nbr] = depth[v] + 1; first_parent[ge.nbr] = (int32_t)v; fresh.push_back(ge.nbr); }
        std::sort(fresh.begin(), fresh.end(), [&](uint32_t a, uint32_t b) {
          const uint32_t oa = unev_out(a), ob = unev_out(b);
          return oa != ob ? oa < ob : a < b;
        });
        for (uint32_t w : fresh) S.push_back(w);
        if (!g.edges.empty()) P->groups.push_back(std::move(g));
      }
    }
  }
  while (traversal == GSMART_DEGREE && n_unev() > 0) {
    // Step 2: root = max unevaluated edges (among constant neighbours first,
    // P:L398), then max unevaluated out-edges, then lowest index (R16).
    int32_t best = -1; bool best_pref = false; uint32_t bu = 0, bo = 0;
    for (uint32_t v = 0; v < n; v++) {
      if (W[v]) continue;
      uint32_t u = unev(v);
      if (u == 0) continue;
      uint32_t o = unev_out(v);
      bool pref = const_adj[v];
      bool better = best < 0 || (pref && !best_pref) ||
                    (pref == best_pref && (u > bu || (u == bu && o > bo)));
      if (better) { best = (int32_t)v; best_pref = pref; bu = u; bo = o; }
    }
    uint32_t root = (uint32_t)best;
    P->roots.push_back(root);
    W[root] = true; depth[root] = 0; first_parent[root] = -1;
    std::vector<uint32_t> S{root};
    while (!S.empty()) {                       // Step 3
      uint32_t v = S.back(); S.pop_back();
      Group g; g.center = v; g.level = depth[v];
      for (uint32_t k = 0; k < ne; k++) {      // Step 4: all unevaluated incident edges
        const auto& e = q->e[k];
        if (F[k]) {
          // evaluated at an earlier center (variables at both ends): a back edge
          if (e.src != e.dst && !is_c[e.src] && !is_c[e.dst]) {
            if (e.src == v) g.back.push_back({k, e.pred, OUT, e.dst});
            else if (e.dst == v) g.back.push_back({k, e.pred, IN, e.src});
          }
          continue;
        }
        if (e.src == v) g.edges.push_back({k, e.pred, OUT, e.dst});
        else if (e.dst == v) g.edges.push_back({k, e.pred, IN, e.src});
      }
      for (auto& ge : g.edges) F[ge.edge] = true;
      std::vector<uint32_t> fresh;
      for (auto& ge : g.edges) {
        uint32_t w = ge.nbr;
        if (!W[w]) { W[w] = true; depth[w] = depth[v] + 1; first_parent[w] = (int32_t)v; fresh.push_back(w); }
      }
      // push ascending (unevaluated, unevaluated-out, index): the largest pops first (R16)
      std::sort(fresh.begin(), fresh.end(), [&](uint32_t a, uint32_t b) {
        uint32_t ua = unev(a), ub = unev(b);
        if (ua != ub) return ua < ub;
        uint32_t oa = unev_out(a), ob = unev_out(b);
        if (oa != ob) return oa < ob;
        return a < b;
      });
      for (uint32_t w : fresh) S.push_back(w);
      if (!g.edges.empty()) P->groups.push_back(std::move(g));
    }
  }

  // Trie order pi: roots and first-discovered neighbours in group order; each
  // later pattern between two visited variables is a closing edge of the one
  // visited later (self-loops: of the variable itself).
  std::vector<int32_t> pos(n, -1);
  auto add_level = [&](uint32_t v, int32_t tree_edge, uint32_t parent, uint32_t label, uint32_t dir) {
    Level L; L.var = v; L.tree_edge = tree_edge;
    L.parent_level = tree_edge >= 0 ? (uint32_t)pos[parent] : 0;
    L.label = label; L.dir = dir;
    pos[v] = (int32_t)P->levels.size();
    P->levels.push_back(L);
  };
  std::set<uint32_t> root_set(P->roots.begin(), P->roots.end());
  for (auto& g : P->groups) {
    uint32_t v = g.center;
    int32_t joined = -1;  // the edge through which a later root joins the trie
    if (pos[v] < 0) {
      // a root; a later one (direction-driven) joins through its first edge to a
      // visited vertex, as that vertex's child over the reversed direction
      // (not over a CSR-only LSpM: the join reads the visited vertex's CSC row; the
      // root is then a free level and the edge a closing edge, checked in CSR rows)
      for (auto& ge : g.edges)
        if (!csr_only && ge.nbr != v && pos[ge.nbr] >= 0) { joined = (int32_t)ge.edge; break; }
      if (joined >= 0) {
        const auto& e = q->e[joined];
        const uint32_t w = e.src == v ? e.dst : e.src;
        add_level(v, joined, w, e.pred, e.src == v ? (uint32_t)IN : (uint32_t)OUT);
      } else {
        add_level(v, -1, 0, 0, 0);
      }
    }
    // With LSpM statistics (gsmart_plan given a built ctx) a group's new
    // neighbours enter the trie in ascending expected fan-out (entries per row
    // of the label, from the center's side): functional patterns (one child
    // per parent) come before the fan-out ones, so the big levels are built
    // once, at the end, instead of being copied level after level.  The result
    // is the same for every order (the rows are sorted at the end).
    std::vector<const GroupEdge*> order;
    for (auto& ge : g.edges) order.push_back(&ge);
    if (fanout)
      std::stable_sort(order.begin(), order.end(), [&](const GroupEdge* a, const GroupEdge* b) {
        return (*fanout)(a->label, a->dir) < (*fanout)(b->label, b->dir);
      });
    for (const GroupEdge* gp : order) {
      const GroupEdge& ge = *gp;
      if ((int32_t)ge.edge == joined) continue;
      uint32_t w = ge.nbr;
      if (w == v) {
        P->levels[pos[v]].closing.push_back({ge.edge, ge.label, (uint32_t)pos[v], OUT});
      } else if (pos[w] < 0) {
        add_level(w, (int32_t)ge.edge, v, ge.label, ge.dir);
      } else {
        uint32_t later = pos[w] > pos[v] ? w : v, other = later == w ? v : w;
        const auto& e = q->e[ge.edge];
        P->levels[pos[later]].closing.push_back({ge.edge, ge.label, (uint32_t)pos[other],
                                                 e.src == later ? (uint32_t)OUT : (uint32_t)IN});
      }
    }
  }
  for (uint32_t v : P->vars)
    if (pos[v] < 0) add_level(v, -1, 0, 0, 0);   // only light edges: a free level

  // Paths (Ex. 7.1): DFS branches over group edges from each root.
  std::vector<int32_t> gidx(n, -1);
  for (size_t i = 0; i < P->groups.size(); i++) gidx[P->groups[i].center] = (int32_t)i;
  for (uint32_t r : P->roots) {
    std::vector<std::vector<uint32_t>> out;
    std::vector<uint32_t> acc{r};
    std::function<void(uint32_t)> walk = [&](uint32_t v) {
      std::vector<uint32_t> kids;
      if (gidx[v] >= 0)
        for (auto& ge : P->groups[gidx[v]].edges) if (ge.nbr != v) kids.push_back(ge.nbr);
      if (kids.empty()) { out.push_back(acc); return; }
      for (uint32_t w : kids) {
        acc.push_back(w);
        if (first_parent[w] == (int32_t)v && gidx[w] >= 0) walk(w);
        else out.push_back(acc);
        acc.pop_back();
      }
    };
    walk(r);
    P->paths.push_back(out);
  }
  (void)root_set;
  return GSMART_OK;
}

// Labels each LSpM format must hold to execute plan p (query-
// dependent LSpM, P:L408 / Ex. 6.4): seeds read the constant's row (CSR for
// (c -l-> v), CSC for (v -l-> c)); a variable's later seeds and the group edges
// read the center's row (OUT: CSR, IN: CSC); tree edges the parent's row;
// closing edges the subject's CSR row (the executor's choice when the formats
// keep different labels).
void plan_access(const gsmart_plan_t& p, bool back_edges, std::set<uint32_t>* csr, std::set<uint32_t>* csc) {
  std::vector<bool> seeded(p.n_vertices, false);
  for (const auto& g : p.guards) csr->insert(g.label);
  std::vector<const Seed*> order;
  for (const auto& sd : p.seeds) order.push_back(&sd);
  std::sort(order.begin(), order.end(), [](const Seed* a, const Seed* b) { return a->edge < b->edge; });
  for (const Seed* sd : order) {
    const bool first = !seeded[sd->var];
    seeded[sd->var] = true;
    if (sd->dir == OUT) (first ? csr : csc)->insert(sd->label);  // c -l-> v
    else (first ? csc : csr)->insert(sd->label);                 // v -l-> c
  }
  for (const auto& g : p.groups) {
    for (const auto& e : g.edges) (e.dir == OUT ? csr : csc)->insert(e.label);
    if (back_edges)
      for (const auto& e : g.back) (e.dir == OUT ? csr : csc)->insert(e.label);
  }
  for (const auto& L : p.levels) {
    if (L.tree_edge >= 0) (L.dir == OUT ? csr : csc)->insert(L.label);
    for (const auto& c : L.closing) csr->insert(c.label);
  }
}

static void jarr(std::ostringstream& o, const std::vector<uint32_t>& v) {
  o << "[";
  for (size_t i = 0; i < v.size(); i++) o << (i ? "," : "") << v[i];
  o << "]";
}

std::string describe_plan(const gsmart_plan_t& p) {
  std::ostringstream o;
  o << "{\"traversal\":\"" << (p.traversal == GSMART_DIRECTION ? "direction" : "degree") << "\",\"roots\":";
  jarr(o, p.roots);
  o << ",\"seeds\":[";
  for (size_t i = 0; i < p.seeds.size(); i++) {
    auto& s = p.seeds[i];
    o << (i ? "," : "") << "{\"edge\":" << s.edge << ",\"var\":" << s.var << ",\"label\":" << s.label
      << ",\"const\":" << s.cid << ",\"dir\":\"" << (s.dir == OUT ? "out" : "in") << "\"}";
  }
  o << "],\"guards\":[";
  for (size_t i = 0; i < p.guards.size(); i++) o << (i ? "," : "") << p.guards[i].edge;
  o << "],\"groups\":[";
  for (size_t i = 0; i < p.groups.size(); i++) {
    auto& g = p.groups[i];
    o << (i ? "," : "") << "{\"center\":" << g.center << ",\"level\":" << g.level << ",\"edges\":[";
    for (size_t j = 0; j < g.edges.size(); j++) {
      auto& e = g.edges[j];
      o << (j ? "," : "") << "{\"edge\":" << e.edge << ",\"label\":" << e.label << ",\"dir\":\""
        << (e.dir == OUT ? "out" : "in") << "\",\"nbr\":" << e.nbr << "}";
    }
    o << "],\"back\":[";
    for (size_t j = 0; j < g.back.size(); j++) {
      auto& e = g.back[j];
      o << (j ? "," : "") << "{\"edge\":" << e.edge << ",\"label\":" << e.label << ",\"dir\":\""
        << (e.dir == OUT ? "out" : "in") << "\",\"nbr\":" << e.nbr << "}";
    }
    o << "]}";
  }
  o << "],\"pi\":[";
  for (size_t i = 0; i < p.levels.size(); i++) o << (i ? "," : "") << p.levels[i].var;
  o << "],\"levels\":[";
  for (size_t i = 0; i < p.levels.size(); i++) {
    auto& L = p.levels[i];
    o << (i ? "," : "") << "{\"var\":" << L.var << ",\"tree_edge\":" << L.tree_edge;
    if (L.tree_edge >= 0)
      o << ",\"parent_level\":" << L.parent_level << ",\"label\":" << L.label << ",\"dir\":\""
        << (L.dir == OUT ? "out" : "in") << "\"";
    o << ",\"closing\":[";
    for (size_t j = 0; j < L.closing.size(); j++) {
      auto& c = L.closing[j];
      o << (j ? "," : "") << "{\"edge\":" << c.edge << ",\"label\":" << c.label << ",\"other_level\":"
        << c.other_level << ",\"dir\":\"" << (c.dir == OUT ? "out" : "in") << "\"}";
    }
    o << "]}";
  }
  o << "],\"paths\":[";
  for (size_t i = 0; i < p.paths.size(); i++) {
    o << (i ? "," : "") << "[";
    for (size_t j = 0; j < p.paths[i].size(); j++) { o << (j ? "," : ""); jarr(o, p.paths[i][j]); }
    o << "]";
  }
  o << "],\"vars\":";
  jarr(o, p.vars);
  o << "}";
  return o.str();
}

}  // namespace gsm
