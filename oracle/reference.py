"""ORACLE (test infrastructure only) — plain Python/numpy reference of the
gSmart hot path, written from /root/reference/PAPER.md.  See oracle/__init__.py.

Citations: "P:L<n>" = PAPER.md line n.  Readings of garbled / silent passages
are numbered R<k> and listed in DESIGN.md ("Readings of the paper").
"""
from itertools import product

import numpy as np

# --------------------------------------------------------------------------
# Triple set ("a set of RDF triples"; R5: duplicates collapse)
# --------------------------------------------------------------------------


def triple_set(s, p, o, keep=None):
    """Set of (s, p, o) int tuples; `keep` = iterable of predicate ids to retain
    ("Read necessary RDF triples where predicates appear in the queries")."""
    ks = None if keep is None or len(keep) == 0 else set(int(x) for x in keep)
    return {(int(a), int(b), int(c)) for a, b, c in zip(s, p, o) if ks is None or int(b) in ks}


# --------------------------------------------------------------------------
# §2.2 BGP semantics — the definition the whole method computes (F1)
# --------------------------------------------------------------------------


def brute_force(s, p, o, n_entities, q):
    """All solution rows of BGP query q, by the plain definition
    (P:L185 BGP = set of triple patterns; "its semantics is the
    conjunction of these triple patterns").  Enumerates [0,N)^k — tiny inputs
    only.  Rows: bindings of q.variables (ascending vertex index), sorted
    lexicographically, distinct (R10/R11).  Homomorphism semantics (R6)."""
    T = triple_set(s, p, o)
    vs = q.variables
    rows = []
    for asg in product(range(n_entities), repeat=len(vs)):
        mu = dict(zip(vs, asg))

        def val(i):
            return mu[i] if q.vertices[i] is None else q.vertices[i]
        if all((val(a), l, val(b)) in T for a, l, b in q.edges):
            rows.append(tuple(asg))
    return sorted(rows)


def tree_dp_count(s, p, o, n_entities, q):
    """Exact |answer set| for queries whose variable graph (pairs of distinct
    variables joined by >= 1 pattern) is a forest; closed form:
    count = prod over components of sum_x f_root(x), where
    f_v = allowed_v * prod_children (R_{v,c} @ f_c); R_{v,c} = intersection of
    the relations of all patterns between v and c; allowed_v folds in patterns
    to constants and self-loops.  Raises ValueError if the graph has a cycle."""
    import scipy.sparse as sp
    N = int(n_entities)
    T = triple_set(s, p, o)
    by_label = {}
    for a, b, c in T:
        by_label.setdefault(b, []).append((a, c))

    def mat(label):
        pr = by_label.get(label, [])
        if not pr:
            return sp.csr_matrix((N, N), dtype=np.int64)
        r = np.array([x for x, _ in pr]); c = np.array([y for _, y in pr])
        return sp.csr_matrix((np.ones(len(pr), np.int64), (r, c)), shape=(N, N))

    vs = q.variables
    allowed = {v: np.ones(N, dtype=np.int64) for v in vs}
    rel = {}
    for a, l, b in q.edges:
        ca, cb = q.vertices[a], q.vertices[b]
        if ca is not None and cb is not None:
            if (ca, l, cb) not in T:
                return 0
        elif ca is not None:          # const -> var
            m = np.zeros(N, np.int64)
            for x, y in by_label.get(l, []):
                if x == ca:
                    m[y] = 1
            allowed[b] *= m
        elif cb is not None:          # var -> const
            m = np.zeros(N, np.int64)
            for x, y in by_label.get(l, []):
                if y == cb:
                    m[x] = 1
            allowed[a] *= m
        elif a == b:                  # self-loop
            m = np.zeros(N, np.int64)
            for x, y in by_label.get(l, []):
                if x == y:
                    m[x] = 1
            allowed[a] *= m
        else:
            key = (min(a, b), max(a, b))
            M = mat(l) if a == key[0] else mat(l).T.tocsr()
            rel[key] = M if key not in rel else rel[key].multiply(M).tocsr()
    adj = {v: [] for v in vs}
    for (a, b) in rel:
        adj[a].append(b); adj[b].append(a)
    seen, total = set(), 1
    for r in vs:
        if r in seen:
            continue
        # DFS order, detect cycles
        order, parent, stack = [], {r: None}, [r]
        seen.add(r)
        while stack:
            v = stack.pop(); order.append(v)
            for w in adj[v]:
                if w == parent[v]:
                    continue
                if w in seen:
                    raise ValueError("cyclic variable graph")
                seen.add(w); parent[w] = v; stack.append(w)
        f = {}
        for v in reversed(order):
            fv = allowed[v].copy()
            for w in adj[v]:
                if parent.get(w) == v:
                    key = (min(v, w), max(v, w))
                    R = rel[key] if v == key[0] else rel[key].T.tocsr()
                    fv = fv * (R @ f[w])
            f[v] = fv
        total *= int(f[r].sum())
    return total


# --------------------------------------------------------------------------
# §2.1 matrix-algebra operators on dense label matrices (Eqs. 2-11)
# A is an N x N int array, A[i, j] = predicate id or 0.
# --------------------------------------------------------------------------


def row_selection(S, A):
    """Eq. 2: S x A with S diagonal 0/1 keeps rows i with S(i,i)=1."""
    return np.asarray(S) @ np.asarray(A)


def column_selection(A, S):
    """Eq. 3: A x S keeps columns j with S(j,j)=1."""
    return np.asarray(A) @ np.asarray(S)


def row_predicate_test(A, p):
    """Eq. 4: y(i) = OR_j A(i,j) ^ p, where ^ between a predicate
    and a cell is label equality (R1)."""
    A = np.asarray(A)
    return np.array([int(any(A[i, j] == p for j in range(A.shape[1]))) for i in range(A.shape[0])])


def column_predicate_test(A, p):
    """Eq. 5, read as y(j) = OR_i [A(i,j) = p] (R3: the printed
    A(j,i) is a cell of A^T)."""
    A = np.asarray(A)
    return np.array([int(any(A[i, j] == p for i in range(A.shape[0]))) for j in range(A.shape[1])])


def predicate_positions(A, p):
    """Eq. 8: M = S_p (x) A, M(i,j) = 1 iff A(i,j) = p (R1)."""
    A = np.asarray(A)
    return (A == p).astype(int)


def vector_and(x, y):
    """Eq. 10: bitwise AND of two binary vectors."""
    return (np.asarray(x) & np.asarray(y)).astype(int)


def vector_or(x, y):
    """Eq. 11: bitwise OR of two binary vectors."""
    return (np.asarray(x) | np.asarray(y)).astype(int)


def binding_vector(M):
    """Eq. 14: v_y = OR_i M^T(:, i) = OR over rows of M (column bindings)."""
    M = np.asarray(M)
    out = np.zeros(M.shape[1], dtype=int)
    for i in range(M.shape[0]):
        out = vector_or(out, M[i, :])
    return out


def binding_matrix_rows(A, v, p):
    """Eqs. 15/18-19: M = p x I (x) (diag(v) x A):
    entries of label p in the rows selected by the binding vector v."""
    A = np.asarray(A)
    S = np.diag(np.asarray(v, dtype=int))
    return predicate_positions(row_selection(S, A), p)


def binding_matrix_cols(A, v, p):
    """Eqs. 22-23: M = p x I (x) (A x diag(v)): entries of
    label p in the columns selected by v (M(k, i) = 1 iff A(k, i) = p, v(i))."""
    A = np.asarray(A)
    S = np.diag(np.asarray(v, dtype=int))
    return predicate_positions(column_selection(A, S), p)


def neighbour_bindings(A, v_x, p, x_is_subject):
    """Binding vector of the other end w of an evaluated edge (x, p, w) or
    (w, p, x), given x's binding vector v_x: Eq. 14 over the binding matrix of
    Eqs. 15/19 (x the subject: v_w = OR of the rows of M_xw) or of Eqs. 22-23
    (x the object: M_wx has x in the columns, v_w = OR of the rows of
    M_wx^T)."""
    if x_is_subject:
        return binding_vector(binding_matrix_rows(A, v_x, p))
    return binding_vector(binding_matrix_cols(A, v_x, p).T)


def grouped_eval_out_out(A, p_xy, p_xz):
    """Eq. 17: v_x = (A (x) u_pxy) AND (A (x) u_pxz)."""
    return vector_and(row_predicate_test(A, p_xy), row_predicate_test(A, p_xz))


def grouped_eval_in_out(A, p_yx, p_xz):
    """Eq. 21: v_x = (A^T (x) u_pyx) AND (A (x) u_pxz)."""
    return vector_and(column_predicate_test(A, p_yx), row_predicate_test(A, p_xz))


def label_matrix(s, p, o, n):
    """Dense A of P:L61 (cell = predicate id; R4: at most one label per cell
    is assumed by the dense form — callers use it only on such inputs)."""
    A = np.zeros((n, n), dtype=int)
    for a, b, c in zip(s, p, o):
        A[a, c] = b
    return A


# --------------------------------------------------------------------------
# §6.2 LSpM arrays
# --------------------------------------------------------------------------


def lspm_paper_form(s, p, o, n_entities, keep=None):
    """LSpM_CSR of §6.2.1 exactly as Example 6.3 prints it:
    keep predicates, drop empty rows, Mr[N+1] (Mr[i+1]-Mr[i] = 1 iff row i is
    non-empty), Pr over non-empty rows, Val/Col with entries of a row in
    column order (then label)."""
    T = sorted(triple_set(s, p, o, keep), key=lambda t: (t[0], t[2], t[1]))
    N = int(n_entities)
    nonempty = sorted({t[0] for t in T})
    Mr = [0] * (N + 1)
    for i in range(N):
        Mr[i + 1] = Mr[i] + (1 if i in set(nonempty) else 0)
    Pr, Val, Col = [0], [], []
    for r in nonempty:
        ent = [t for t in T if t[0] == r]
        Val += [t[1] for t in ent]
        Col += [t[2] for t in ent]
        Pr.append(len(Val))
    return {"Mr": Mr, "Pr": Pr, "Val": Val, "Col": Col, "rows": len(nonempty), "nnz": len(Val)}


def lspm_csc_paper_form(s, p, o, n_entities, keep=None):
    """LSpM_CSC of §6.2.2: the CSC analogue (columns = objects)."""
    d = lspm_paper_form(o, p, s, n_entities, keep)
    return {"Mc": d["Mr"], "Pc": d["Pr"], "Val": d["Val"], "Row": d["Col"],
            "cols": d["rows"], "nnz": d["nnz"]}


def lspm_arrays(s, p, o, n_entities, keep=None, fmt="csr"):
    """The product's LSpM layout by its plain definition (DESIGN.md "Data
    layout"): entries of the kept, de-duplicated triple set sorted by
    (row, pred, col) with row = subject (CSR) or object (CSC):
      row_ptr[N+1], col[M], pred[M], and per label l the ascending list of
      rows having >= 1 l-entry (label_off[P+2], label_rows[R]) — the paper's
      "eliminate empty rows" per predicate."""
    T = triple_set(s, p, o, keep)
    if fmt == "csr":
        E = sorted((a, b, c) for a, b, c in T)
    else:
        E = sorted((c, b, a) for a, b, c in T)
    N = int(n_entities)
    rows = np.array([e[0] for e in E], dtype=np.int64)
    row_ptr = np.searchsorted(rows, np.arange(N + 1), side="left").astype(np.uint64)
    col = np.array([e[2] for e in E], dtype=np.uint32)
    pred = np.array([e[1] for e in E], dtype=np.uint32)
    P = int(max([e[1] for e in E], default=0))
    pairs = sorted({(e[1], e[0]) for e in E})
    return {"row_ptr": row_ptr, "col": col, "pred": pred, "label_pairs": pairs, "max_pred": P}


# --------------------------------------------------------------------------
# §6.1.2 degree-driven traversal + trie order (§7.1)
# --------------------------------------------------------------------------

OUT, IN = 0, 1


def plan_degree(q):
    """Degree-driven traversal, constants variant P:L395-L398.

    Returns dict:
      seeds   : edge indices incident to a constant (pre-evaluated)
      roots   : Root_r in order
      groups  : list of (center, [(edge, dir, neighbour)]) in evaluation order;
                dir OUT = the center is the edge's subject (CSR row), IN = object
      back    : per group, the center's variable-variable patterns evaluated
                at earlier centers, same (edge, dir, neighbour) form
      level   : per group, DFS depth of its center (edge level, R-level)
      pi      : variable visitation order (trie levels; DESIGN "trie")
      tree    : {var: (edge, parent_var, dir-from-parent)} for non-root vars
      closing : {var: [(edge, other_var, dir-from-var)]} checked at var's level
      paths   : per root, the DFS branches (Ex. 7.1)
    Tie-breaks beyond the paper's keys: lowest vertex index (R16); push order
    ascending (unevaluated edges, unevaluated out-edges, index) (R16)."""
    n = q.n_vertices
    E = q.edges
    is_c = [q.is_const(i) for i in range(n)]
    W = {i for i in range(n) if is_c[i]}
    F = {k for k, (a, _, b) in enumerate(E) if is_c[a] or is_c[b]}
    seeds = sorted(F)
    const_adj = {b if is_c[a] else a for k, (a, _, b) in enumerate(E)
                 if is_c[a] != is_c[b]}

    def unev(v):
        return sum(1 for k, (a, _, b) in enumerate(E) if k not in F and (a == v or b == v))

    def unev_out(v):
        return sum(1 for k, (a, _, b) in enumerate(E) if k not in F and a == v)

    groups, roots, glevel, back = [], [], [], []
    depth = {}
    first_parent = {}
    while len(F) < len(E):
        # step 2: root selection
        cands = [v for v in range(n) if v not in W and unev(v) > 0]
        pref = [v for v in cands if v in const_adj]
        pool = pref if pref else cands
        root = max(pool, key=lambda v: (unev(v), unev_out(v), -v))
        roots.append(root)
        W.add(root)
        depth[root] = 0
        first_parent[root] = None
        S = [root]
        while S:                                         # step 3
            v = S.pop()
            # patterns of v already evaluated at an earlier center (variables at
            # both ends): Eq. 16 restricts v's rows by their binding vectors
            bk = [(k, OUT if a == v else IN, b if a == v else a) for k, (a, _, b) in enumerate(E)
                  if k in F and (a == v or b == v) and a != b and not is_c[a] and not is_c[b]]
            grp = []
            for k, (a, l, b) in enumerate(E):           # step 4
                if k in F or (a != v and b != v):
                    continue
                if a == v:
                    grp.append((k, OUT, b))
                else:
                    grp.append((k, IN, a))
            for k, _, _ in grp:
                F.add(k)
            new = []
            for _, _, w in grp:
                if w not in W:
                    W.add(w)
                    depth[w] = depth[v] + 1
                    first_parent[w] = v
                    new.append(w)
            new.sort(key=lambda w: (unev(w), unev_out(w), w))
            S.extend(new)
            if grp:
                groups.append((v, grp))
                glevel.append(depth[v])
                back.append(bk)
    # trie order pi, tree edges, closing edges
    pi, tree, closing = [], {}, {}
    pos = {}

    def add(v):
        pos[v] = len(pi)
        pi.append(v)
        closing.setdefault(v, [])
    gi = 0
    root_set = set(roots)
    for v, grp in groups:
        if v in root_set and v not in pos:
            add(v)
        for k, d, w in grp:
            if w == v:
                closing[v].append((k, v, d))
            elif w not in pos:
                add(w)
                tree[w] = (k, v, d)
            else:
                later, other = (w, v) if pos[w] > pos[v] else (v, w)
                # direction from `later`'s point of view
                a, _, b = E[k]
                closing[later].append((k, other, OUT if a == later else IN))
        gi += 1
    for v in q.variables:
        if v not in pos:
            add(v)
    # paths (Ex. 7.1): DFS branches over group edges
    gmap = {v: grp for v, grp in groups}
    paths = {}
    for r in roots:
        out = []

        def walk(v, acc):
            kids = [w for _, _, w in gmap.get(v, []) if w != v]
            if not kids:
                out.append(acc)
                return
            for w in kids:
                if first_parent.get(w) == v and w in gmap:
                    walk(w, acc + [w])
                else:
                    out.append(acc + [w])
        walk(r, [r])
        paths[r] = out
    return {"seeds": seeds, "roots": roots, "groups": groups, "back": back, "level": glevel,
            "pi": pi, "tree": tree, "closing": closing, "paths": paths}


def plan_direction(q):
    """Direction-driven traversal, P:L365-L379 (§6.1.1), with the cyclic
    variant of step 2: roots are unvisited vertices without
    unevaluated incoming edges (max unevaluated outgoing edges first; cyclic:
    else the unvisited vertex with the most unevaluated outgoing edges); a
    popped vertex evaluates all its unevaluated OUTGOING edges (one group, all
    `OUT`, rows of the CSR LSpM only); newly visited targets are pushed in
    ascending (unevaluated outgoing edges, index) order so the largest pops
    first.  Ties beyond the paper's keys: lowest vertex index (R16).  A query
    with constants is planned degree-driven, so it is refused here
    (ValueError).  Returns the plan_degree dict shape; no back edges (the
    groups read CSR rows only), trie order / tree / closing edges derived the
    same way as for degree-driven plans, a later root joining through its
    first edge to a visited vertex."""
    n = q.n_vertices
    E = q.edges
    if any(q.is_const(i) for i in range(n)):
        raise ValueError("direction-driven plans take variable-only queries (P:L381)")
    F, W = set(), set()

    def unev_in(v):
        return sum(1 for k, (a, _, b) in enumerate(E) if k not in F and b == v)

    def unev_out(v):
        return sum(1 for k, (a, _, b) in enumerate(E) if k not in F and a == v)

    groups, roots, glevel, depth = [], [], [], {}
    while len(F) < len(E):
        cands = [v for v in range(n) if v not in W and unev_in(v) == 0 and unev_out(v) > 0]
        if not cands:  # cyclic: P:L377
            cands = [v for v in range(n) if v not in W and unev_out(v) > 0]
        if not cands:  # every remaining edge starts at a visited vertex (cannot happen: popped ones are drained)
            cands = [v for v in range(n) if unev_out(v) > 0]
        root = max(cands, key=lambda v: (unev_out(v), -v))
        roots.append(root)
        W.add(root)
        depth[root] = 0
        S = [root]
        while S:
            v = S.pop()
            grp = [(k, OUT, b) for k, (a, _, b) in enumerate(E) if k not in F and a == v]
            for k, _, _ in grp:
                F.add(k)
            new = []
            for _, _, w in grp:
                if w not in W:
                    W.add(w)
                    depth[w] = depth[v] + 1
                    new.append(w)
            new.sort(key=lambda w: (unev_out(w), w))
            S.extend(new)
            if grp:
                groups.append((v, grp))
                glevel.append(depth[v])
    pi, tree, closing, pos = [], {}, {}, {}

    def add(v):
        pos[v] = len(pi)
        pi.append(v)
        closing.setdefault(v, [])
    for v, grp in groups:
        if v not in pos:
            add(v)
            # a later root joins the trie through its first edge to a visited vertex
            for k, d, w in grp:
                if w != v and w in pos:
                    tree[v] = (k, w, IN)
                    break
        for k, d, w in grp:
            if w == v:
                closing[v].append((k, v, d))
            elif w not in pos:
                add(w)
                tree[w] = (k, v, d)
            elif tree.get(v, (None,))[0] == k:
                continue  # the edge that joined v to the trie
            else:
                later, other = (w, v) if pos[w] > pos[v] else (v, w)
                a, _, b = E[k]
                closing[later].append((k, other, OUT if a == later else IN))
    for v in q.variables:
        if v not in pos:
            add(v)
    return {"seeds": [], "roots": roots, "groups": groups, "back": [[] for _ in groups], "level": glevel,
            "pi": pi, "tree": tree, "closing": closing, "paths": {}}


def keep_sets(q, plan=None, back_edges=False):
    """Query-dependent LSpM (§6.2, "Read necessary RDF triples where
    predicates appear in the queries"; Ex. 6.4 P:L436-L448: the CSR keeps the
    predicates evaluated along their direction, the CSC those evaluated
    against it): the labels each format must hold for the schedule and the
    trie of `plan`, as (csr, csc) sorted lists:
      seed (c -l-> v): c's CSR row; (v -l-> c): c's CSC row; guard: CSR;
      a variable's 2nd+ seed, tested in v's row: (c -l-> v) CSC, (v -l-> c) CSR;
      group edge (and back edge): OUT -> CSR, IN -> CSC;
      trie tree edge: parent's row, OUT -> CSR, IN -> CSC;
      closing edge: the subject's CSR row."""
    plan = plan or plan_degree(q)
    csr, csc = set(), set()
    is_c = [q.is_const(i) for i in range(q.n_vertices)]
    seeded = {}
    for k in plan["seeds"]:
        a, l, b = q.edges[k]
        if is_c[a] and is_c[b]:
            csr.add(l)
        elif is_c[a]:
            (csc if b in seeded else csr).add(l)
            seeded.setdefault(b, k)
        else:
            (csr if a in seeded else csc).add(l)
            seeded.setdefault(a, k)
    back = plan.get("back") if back_edges else None
    for gi, (x, grp) in enumerate(plan["groups"]):
        for k, d, w in list(grp) + (list(back[gi]) if back else []):
            (csr if d == OUT else csc).add(q.edges[k][1])
    for v, (k, parent, d) in plan["tree"].items():
        (csr if d == OUT else csc).add(q.edges[k][1])
    for v, cl in plan["closing"].items():
        for k, _, _ in cl:
            csr.add(q.edges[k][1])
    return sorted(csr), sorted(csc)


# --------------------------------------------------------------------------
# Filter schedule: seeds (light edges), then every group center
# in plan order is "revised" against all its incident patterns (§5 Eqs. 17/21
# for the group's unevaluated edges; Eqs. 14-16 for the already evaluated
# ones, whose binding vectors restrict the center's rows), then the centers
# again in reverse order (R-refine).  Bitmaps as bool arrays.
# --------------------------------------------------------------------------


def filter_schedule(s, p, o, n_entities, q, plan=None, refine=False, back_edges=False):
    """Candidate sets per variable after the schedule DESIGN.md states:
      1. cand_v = [0, N) for every variable (Eq. 4/5 with no constraint yet);
      2. each seed edge in edge-index order (light edges):
         (c -l-> v): cand_v &= {o : (c,l,o) in T}; (v -l-> c): cand_v &=
         {s : (s,l,c) in T} (a constant absent from the data, id >= N
         included, has no entries: the set is empty, R12); const-const
         pattern: a guard (R13); a false guard makes the conjunction
         unsatisfiable, so every candidate set is emptied;
      3. revise(x) for each group center x in plan order, where
         revise(x): cand_x &= AND_e y_e over the group's patterns — its
         unevaluated edges (§5), and with back_edges (GSMART_BACK_EDGES) also
         its back edges, so that for a degree-driven plan it is EVERY pattern
         incident to x whose other end is a variable (or x itself):
           e = (x, l, w): y_e(i) = OR_j [(i,l,j) in T] ^ cand_w(j)   (Eq. 17)
           e = (w, l, x): y_e(i) = OR_j [(j,l,i) in T] ^ cand_w(j)   (Eq. 21)
           e = (x, l, x): y_e(i) = [(i,l,i) in T]                    (R7)
         For the group's unevaluated edges this is §5 (Eqs. 17/21 with the
         neighbours' binding vectors as the diag(.) selections of Eqs.
         15-16); for back edges (evaluated at an earlier center c) it is
         Eq. 16's restriction of x's rows to c's Eq. 14 binding vector;
      4. if refine (GSMART_REFINE, reading R-refine; off by default: the paper
         evaluates each group once): revise(x) for the centers in
         reverse plan order, the last one skipped (nothing it reads changed
         after it).
    Returns ({var: np.bool_ array of length N}, guards_hold)."""
    N = int(n_entities)
    T = triple_set(s, p, o)
    plan = plan or plan_degree(q)
    cand = {v: np.ones(N, dtype=bool) for v in q.variables}
    ok = True
    out_nb, in_nb = {}, {}
    for a, l, c in T:
        out_nb.setdefault((a, l), []).append(c)
        in_nb.setdefault((c, l), []).append(a)
    for k in plan["seeds"]:
        a, l, b = q.edges[k]
        ca, cb = q.vertices[a], q.vertices[b]
        if ca is not None and cb is not None:
            ok = ok and ((ca, l, cb) in T)
            continue
        m = np.zeros(N, dtype=bool)
        if ca is not None:
            for j in out_nb.get((ca, l), []):
                m[j] = True
            cand[b] &= m
        else:
            for j in in_nb.get((cb, l), []):
                m[j] = True
            cand[a] &= m
    if not ok:
        for v in cand:
            cand[v][:] = False

    def revise(x, ks):
        y_all = np.ones(N, dtype=bool)
        for k in ks:
            a, l, b = q.edges[k]
            y = np.zeros(N, dtype=bool)
            for i in range(N):
                if not cand[x][i]:
                    continue
                if a == b:
                    y[i] = (i, l, i) in T
                elif a == x:
                    y[i] = any(cand[b][j] for j in out_nb.get((i, l), []))
                else:
                    y[i] = any(cand[a][j] for j in in_nb.get((i, l), []))
            y_all &= y
        cand[x] &= y_all

    # a group's patterns: its unevaluated edges, plus (back_edges: GSMART_BACK_EDGES)
    # its back edges — with them a degree-driven group is every variable pattern
    # incident to the center (R-back); direction-driven plans have none
    back = (plan.get("back") if back_edges else None) or [[] for _ in plan["groups"]]
    evals = [(x, [k for k, _, _ in grp] + [k for k, _, _ in bk]) for (x, grp), bk in zip(plan["groups"], back)]
    for x, ks in evals:
        revise(x, ks)
    if refine:
        for x, ks in list(reversed(evals))[1:]:
            revise(x, ks)
    return cand, ok


# --------------------------------------------------------------------------
# Sampled parity at any size: all solutions whose binding of one variable lies
# in a sample of values, computed on the triples within `hops` of the sample.
# --------------------------------------------------------------------------


def query_hops(q, var):
    """Largest undirected distance (in pattern edges) from variable `var` to any
    vertex of q, walking through variables only: every triple of a solution
    has an endpoint bound to a variable within hops-1 of var's binding, so the
    triples within `hops` of it contain the solution.  A walk does not pass
    through a constant (its entity may be a hub joined to unrelated data), so a
    variable reachable from `var` only through a constant makes the local
    method inapplicable: ValueError (never a silently incomplete subset)."""
    adj = {i: set() for i in range(q.n_vertices)}
    for a, _, b in q.edges:
        adj[a].add(b)
        adj[b].add(a)
    dist, frontier = {var: 0}, [var]
    while frontier:
        nxt = []
        for v in frontier:
            if q.vertices[v] is not None:
                continue  # a constant ends the walk (its own patterns were reached from a variable)
            for w in adj[v]:
                if w not in dist:
                    dist[w] = dist[v] + 1
                    nxt.append(w)
        frontier = nxt
    missing = [v for v in q.variables if v not in dist]
    if missing:
        raise ValueError(f"variables {missing} are joined to {var} only through constants")
    return max(dist.values())


def local_triples(s, p, o, seeds, hops):
    """Triples with an endpoint reachable from `seeds` in < hops steps (undirected)."""
    s = np.asarray(s)
    p = np.asarray(p)
    o = np.asarray(o)
    front = np.unique(np.asarray(seeds, dtype=s.dtype))
    keep = np.zeros(len(s), dtype=bool)
    for _ in range(hops):
        m = np.isin(s, front) | np.isin(o, front)
        new = m & ~keep
        keep |= m
        front = np.unique(np.concatenate([s[new], o[new]]))
    return s[keep], p[keep], o[keep]


def solutions_for_bindings(s, p, o, q, var, values):
    """The exact solution rows of q whose binding of variable `var` is in
    `values` (BGP definition restricted to those bindings), via the C oracle on
    the local triple subset around `values`."""
    from .coracle import oracle_bgp
    ls, lp, lo = local_triples(s, p, o, values, query_hops(q, var))
    rows = oracle_bgp(ls, lp, lo, q)
    col = q.variables.index(var)
    return rows[np.isin(rows[:, col], np.asarray(values))] if len(rows) else rows
