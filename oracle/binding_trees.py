"""ORACLE (test infrastructure only) — the paper's tree-based binding storage
(§7.1), pre-pruning (§7.2.2 / Alg. 1-2), local and
global tree-pruning (§8.1-8.2) and the join that reads the
solution rows off the pruned trees, written from /root/reference/PAPER.md in
the paper's order and notation, as sets of tuples.  SURVEY.md §8(f) row f2.

A binding tree of path P = (u_0 = Root_r, u_1, ..., u_k) for one binding b of
Root_r stores the bindings of the path's vertices level by level; a
root-to-leaf branch of it is a tuple (b, x_1, ..., x_k).  Here a tree is the
set of those tuples (a node = a tuple prefix), so "remove the sub-tree of a
node" = drop every tuple through that prefix, and §8.1 step 4 (remove parents
left without children) holds by construction.

Readings (R-f2a..R-f2d):
  R-f2a  a path hop (u_{i-1}, u_i) holds iff every query edge of u_{i-1}'s
         group (Alg. 2 l.4 "Evaluate w_l, W_{l+1}") between the two vertices
         holds for the pair (multi-edges: all of them); a vertex's own
         constraints — its constant edges (seeds) and self-loops (R7)
         — hold for every binding stored at any of its occurrences;
  R-f2b  pre-pruning (Alg. 1 l.4, Alg. 2 l.5-11) = a binding of w_l survives
         only if every path continuing through it has a result: repeated until
         nothing changes, over every pair of paths sharing a prefix; a root
         binding with an empty tree is dropped with all its trees;
  R-f2c  Ω = the variables other than the root on >= 2 paths of the
         root, processed once each in ascending vertex index; constant edges
         are already applied per occurrence (R-f2a), which covers the
         "adjacent to constants" clause;
  R-f2d  Φ (§8.2) = variables on paths of >= 2 roots: a binding survives only
         if it occurs under every root whose paths hold the variable; then the
         local pruning again.  The rows are the natural join of the trees of
         one root binding (shared variables equal), crossed over the roots /
         vertices without paths and joined on Φ.
"""

from .reference import IN, OUT, plan_degree, triple_set


def plan_paths(plan):
    """Per root: the DFS branches over the plan's groups ("once each
    branch of Root_r has been traversed (before backtracking), the branch is
    recorded as a path"; Ex. 7.1).  A neighbour continues a path only if this
    center reached it first and it is a center itself (reading R-paths);
    duplicate branches (multi-edges) are listed once."""
    gmap = {v: grp for v, grp in plan["groups"]}
    first = {}
    for v, grp in plan["groups"]:
        for _, _, w in grp:
            if w != v and w not in first and w not in plan["roots"]:
                first[w] = v
    paths = {}
    for r in plan["roots"]:
        out = []

        def walk(v, acc):
            kids = []
            for _, _, w in gmap.get(v, []):
                if w != v and w not in kids:
                    kids.append(w)
            if not kids:
                out.append(tuple(acc))
                return
            for w in kids:
                if first.get(w) == v and w in gmap:
                    walk(w, acc + [w])
                else:
                    out.append(tuple(acc + [w]))
        walk(r, [r])
        paths[r] = out
    return paths


def _constraints(q, plan, T):
    """(local(v, x), hop(u, w, xu, xw)) per R-f2a."""
    E = q.edges
    vert = q.vertices
    gedges = {}
    for v, grp in plan["groups"]:
        for k, _, w in grp:
            if w != v:
                gedges.setdefault((v, w), []).append(k)

    def holds(k, xa, xb):  # pattern k with its ends bound to xa (src) and xb (dst)
        return (xa, E[k][1], xb) in T

    def local(v, x):
        for k, (a, l, b) in enumerate(E):
            if a == v and b == v and (x, l, x) not in T:
                return False
            if a == v and b != v and vert[b] is not None and (x, l, vert[b]) not in T:
                return False
            if b == v and a != v and vert[a] is not None and (vert[a], l, x) not in T:
                return False
        return True

    def hop(u, w, xu, xw):
        for k in gedges.get((u, w), []):
            a, _, b = E[k]
            if not holds(k, xu if a == u else xw, xw if b == w else xu):
                return False
        return True
    return local, hop


def _prefix_prune(paths, trees):
    """R-f2b: drop tuples whose shared prefix with another path has no
    continuation there; repeat to a fixpoint.  Returns False when a tree of
    the root binding is empty (Alg. 2 l.9-10 up to the root: the binding is
    invalid)."""
    changed = True
    while changed:
        changed = False
        for i, P in enumerate(paths):
            for j, Q in enumerate(paths):
                if i == j:
                    continue
                c = 0
                while c < min(len(P), len(Q)) and P[c] == Q[c]:
                    c += 1
                heads = {t[:c] for t in trees[j]}
                keep = {t for t in trees[i] if t[:c] in heads}
                if keep != trees[i]:
                    trees[i] = keep
                    changed = True
    return all(trees)


def binding_trees(s, p, o, n_entities, q, plan=None, omega=True):
    """Main computation phase (§7.2, Alg. 1-2) then local tree-pruning (§8.1)
    and, for several roots, global tree-pruning (§8.2).

    Returns {"paths": {root: [path tuples]}, "trees": {root: {b: [set of tuples
    per path]}}, "omega": {root: [vars]}, "phi": [vars], "free": {var: set},
    "guards": bool}.  `free` = variables on no path (their only patterns are
    constant edges): the set of their bindings (a tree of one level).
    omega=False skips §8.1 (the trees as the main computation leaves them)."""
    N = int(n_entities)
    T = triple_set(s, p, o)
    plan = plan or plan_degree(q)
    paths = {r: ps for r, ps in plan_paths(plan).items()}
    local, hop = _constraints(q, plan, T)
    guards = all((q.vertices[a], l, q.vertices[b]) in T for a, l, b in q.edges
                 if q.is_const(a) and q.is_const(b))
    trees = {}
    for r, ps in paths.items():
        trees[r] = {}
        for b in range(N):                        # Alg. 1 l.2: each row / column
            if not guards or not local(r, b):
                continue
            per = []
            for P in ps:
                X = {(b,)}
                for i in range(1, len(P)):        # Alg. 2: level by level along the path
                    X = {t + (x,) for t in X for x in range(N)
                         if local(P[i], x) and hop(P[i - 1], P[i], t[-1], x)}
                per.append(X)
            if _prefix_prune(ps, per):            # Alg. 1 l.4, Alg. 2 l.9-11
                trees[r][b] = per
    omega_vars = {}
    for r, ps in paths.items():
        cnt = {}
        for P in ps:
            for v in set(P[1:]):
                cnt[v] = cnt.get(v, 0) + 1
        omega_vars[r] = sorted(v for v, c in cnt.items() if c >= 2)
    if omega:
        for r in paths:
            _local_prune(paths[r], trees[r], omega_vars[r])
    # §8.2: common variables of different roots
    on_root = {}
    for r, ps in paths.items():
        for P in ps:
            for v in P:
                on_root.setdefault(v, set()).add(r)
    phi = sorted(v for v, rs in on_root.items() if len(rs) >= 2)
    if omega and phi:
        for v in phi:
            S = None
            for r in on_root[v]:
                vals = {t[P.index(v)] for b, per in trees[r].items()
                        for P, X in zip(paths[r], per) if v in P for t in X}
                S = vals if S is None else S & vals
            for r in on_root[v]:
                for b in list(trees[r]):
                    per = trees[r][b]
                    for i, P in enumerate(paths[r]):
                        if v in P:
                            per[i] = {t for t in per[i] if t[P.index(v)] in S}
                    if not all(per):
                        del trees[r][b]
        for r in paths:
            _local_prune(paths[r], trees[r], omega_vars[r])
    on_path = {v for ps in paths.values() for P in ps for v in P}
    free = {v: {x for x in range(N) if guards and local(v, x)} for v in q.variables if v not in on_path}
    return {"paths": paths, "trees": trees, "omega": omega_vars, "phi": phi, "free": free, "guards": guards}


def _local_prune(ps, rtrees, omega_vars):
    """§8.1 steps 1-4 for one root, every root binding: for v in Ω, the target
    nodes are the v-bindings missing from another tree of the same root
    binding; their sub-trees go (step 3) and childless parents with them
    (step 4).  A root binding left with an empty tree is dropped."""
    for v in omega_vars:                          # step 1
        for b in list(rtrees):
            per = rtrees[b]
            S = None
            for P, X in zip(ps, per):             # step 2: bindings of v in every tree
                if v in P:
                    vals = {t[P.index(v)] for t in X}
                    S = vals if S is None else S & vals
            for i, P in enumerate(ps):            # steps 3-4
                if v in P:
                    per[i] = {t for t in per[i] if t[P.index(v)] in S}
            if not all(per):
                del rtrees[b]


def _join(parts):
    """Natural join of relations given as (vertex tuple, set of value tuples)."""
    cols, rows = (), [()]
    for vs, X in parts:
        new_cols = cols + tuple(v for v in vs if v not in cols)
        out = []
        for r in rows:
            cur = dict(zip(cols, r))
            for t in X:
                ok = True
                ext = dict(cur)
                for v, x in zip(vs, t):
                    if ext.get(v, x) != x:
                        ok = False
                        break
                    ext[v] = x
                if ok:
                    out.append(tuple(ext[c] for c in new_cols))
        cols, rows = new_cols, out
    return cols, rows


def factorised_rows(bt, q):
    """Solution rows read off the pruned binding trees: per root binding the
    natural join of its trees; the roots' relations and the free variables
    joined (cross product when nothing is shared).  Rows in variable-index
    order, sorted, distinct (R10/R11)."""
    if not bt["guards"]:
        return []
    parts = []
    for r, per_b in bt["trees"].items():
        rel = set()
        for b, per in per_b.items():
            cols, rows = _join(list(zip(bt["paths"][r], per)))
            rel.update((cols, x) for x in rows)
        # one relation per root over the union of its path vertices
        vs = tuple(sorted({v for P in bt["paths"][r] for v in P}))
        X = set()
        for cols, x in rel:
            d = dict(zip(cols, x))
            X.add(tuple(d[v] for v in vs))
        parts.append((vs, X))
    for v, S in bt["free"].items():
        parts.append(((v,), {(x,) for x in S}))
    cols, rows = _join(parts)
    vs = q.variables
    out = {tuple(dict(zip(cols, r))[v] for v in vs) for r in rows}
    return sorted(out)


def tree_sizes(bt):
    """Per root binding and path: the number of tree nodes (distinct non-empty
    tuple prefixes, root node included) — the memory the paper's form holds."""
    out = {}
    for r, per_b in bt["trees"].items():
        for b, per in per_b.items():
            out[(r, b)] = [len({t[:i] for t in X for i in range(1, len(t) + 1)}) for X in per]
    return out


__all__ = ["plan_paths", "binding_trees", "factorised_rows", "tree_sizes"]
