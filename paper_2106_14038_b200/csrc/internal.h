// Internal declarations shared by the library's translation units.
// (Product code; nothing here is shared with oracle/.)
#pragma once
#include <cstdint>
#include <functional>
#include <set>
#include <string>
#include <vector>

#include "gsmart.h"

namespace gsm {

enum Dir : uint32_t { OUT = 0, IN = 1 };  // OUT: center/var is the subject (CSR row); IN: object (CSC row)

// ---------------------------------------------------------------- plan (host)
struct GroupEdge {
  uint32_t edge;   // query edge index
  uint32_t label;  // predicate id
  uint32_t dir;    // OUT / IN, seen from the group's center
  uint32_t nbr;    // neighbour vertex (== center for a self-loop)
};
struct Group {
  uint32_t center;
  uint32_t level;  // DFS depth of the center from its root (edge level)
  std::vector<GroupEdge> edges;
  // the center's variable-variable patterns already evaluated at earlier
  // centers: Eq. 16 restricts the center's rows by their binding
  // vectors, so every evaluation of the group also tests them
  std::vector<GroupEdge> back;
};
struct Seed {      // light edge: constant c, variable v
  uint32_t edge, var, label, cid;
  uint32_t dir;    // OUT: c -l-> v, read CSR row c ; IN: v -l-> c, read CSC row c
};
struct Guard { uint32_t edge, s, label, o; };  // constant-constant pattern
struct Closing {
  uint32_t edge, label;
  uint32_t other_level;  // trie level of the other endpoint (== own level for a self-loop)
  uint32_t dir;          // OUT: this var is the subject -> check CSR row of the child
};
struct Level {           // trie level = one variable in visitation order pi
  uint32_t var;
  int32_t tree_edge;     // -1: no tree edge (first root or a new component: children = candidate list)
  uint32_t parent_level, label, dir;  // dir seen from the parent: OUT = parent is the subject (CSR row of parent)
  std::vector<Closing> closing;
};

}  // namespace gsm

struct gsmart_plan_s {
  uint64_t uid = 0;                    // process-unique id (keys cached CUDA graphs)
  uint32_t traversal = GSMART_DEGREE;  // GSMART_DEGREE or GSMART_DIRECTION
  uint32_t n_vertices = 0;
  std::vector<gsmart_qvertex> vertices;
  std::vector<gsmart_qedge> edges;
  std::vector<uint32_t> vars;          // variable vertices ascending (= output columns)
  std::vector<int32_t> col_of;         // vertex -> column or -1
  std::vector<gsm::Seed> seeds;
  std::vector<gsm::Guard> guards;
  std::vector<uint32_t> roots;
  std::vector<gsm::Group> groups;
  std::vector<gsm::Level> levels;      // trie levels in visitation order
  std::vector<std::vector<std::vector<uint32_t>>> paths;  // per root: DFS branches
};

namespace gsm {
// fanout (optional): expected children per parent of a pattern (label, dir seen
// from the center) — orders a group's new neighbours in the trie
// csr_only: plan for a CSR-only LSpM (direction-driven: later roots are free levels)
gsmart_status build_plan(const gsmart_query* q, uint32_t traversal, gsmart_plan_t* out, std::string* err,
                         const std::function<double(uint32_t, uint32_t)>* fanout = nullptr, bool csr_only = false);
std::string describe_plan(const gsmart_plan_t& p);
// labels the CSR / CSC LSpM must hold to execute p (query-dependent LSpM)
void plan_access(const gsmart_plan_t& p, bool back_edges, std::set<uint32_t>* csr, std::set<uint32_t>* csc);
}  // namespace gsm
