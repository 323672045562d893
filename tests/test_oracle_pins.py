"""Pins of the oracle against things other than itself (task ③): the paper's
worked examples, closed forms, brute force on tiny inputs, invariants.
CPU only (-m "not gpu")."""
import numpy as np
import pytest

from oracle import reference as R
from oracle.coracle import oracle_bgp
from synth import fixtures, tiny, lubm
from synth.query import Query


def _rows(a):
    return [tuple(int(x) for x in r) for r in np.asarray(a).tolist()]


# ---------------------------------------------------------------- Fig. 1/2
def test_fig12_answer_brute_force(golden_fig):
    s, p, o = fixtures.fig1_triples()
    q = fixtures.fig2_query()
    assert R.brute_force(s, p, o, 8, q) == [tuple(r) for r in golden_fig["solution_rows"]]


def test_fig12_answer_c_oracle(golden_fig):
    s, p, o = fixtures.fig1_triples()
    q = fixtures.fig2_query()
    assert _rows(oracle_bgp(s, p, o, q)) == [tuple(r) for r in golden_fig["solution_rows"]]
    # thread-count independence
    assert _rows(oracle_bgp(s, p, o, q, n_threads=1)) == _rows(oracle_bgp(s, p, o, q, n_threads=4))


# ---------------------------------------------------------------- §2.1 operators
# A of Eq. 1 with letters a..i -> labels 1..9
A1 = np.arange(1, 10).reshape(3, 3)
a, b, c, d, e, f, g, h, i = range(1, 10)


def test_eq2_row_selection():
    S = np.diag([1, 0, 1])
    np.testing.assert_array_equal(R.row_selection(S, A1), [[a, b, c], [0, 0, 0], [g, h, i]])


def test_eq3_column_selection():
    S = np.diag([0, 0, 1])
    np.testing.assert_array_equal(R.column_selection(A1, S), [[0, 0, c], [0, 0, f], [0, 0, i]])


def test_eq6_eq7_predicate_tests():
    np.testing.assert_array_equal(R.row_predicate_test(A1, b), [1, 0, 0])      # Eq. 6
    np.testing.assert_array_equal(R.column_predicate_test(A1, b), [0, 1, 0])   # Eq. 7


def test_eq9_predicate_positions():
    np.testing.assert_array_equal(R.predicate_positions(A1, c), [[0, 0, 1], [0, 0, 0], [0, 0, 0]])


def test_eq10_eq11_vector_ops():
    np.testing.assert_array_equal(R.vector_and([1, 0, 1], [0, 0, 1]), [0, 0, 1])
    np.testing.assert_array_equal(R.vector_or([1, 0, 1], [0, 0, 1]), [1, 0, 1])


def test_eq14_neighbour_bindings_fig1(golden_fig):
    """Eq. 14 over the binding matrices of Eqs. 15/19 (center = subject) and
    22-23 (center = object): the binding vectors of v2's neighbours given
    v2 = {1, 5}, hand-derived from the Fig. 1a triples (golden)."""
    s, p, o = fixtures.fig1_triples()
    A = R.label_matrix(s, p, o, 8)
    F, D = fixtures.PREDICATE_IDS["follows"], fixtures.PREDICATE_IDS["director"]
    v2 = np.zeros(8, dtype=int)
    v2[golden_fig["level0_candidates"]] = 1
    g = golden_fig["eq14_neighbour_bindings_of_v2_1_5"]
    assert R.neighbour_bindings(A, v2, F, x_is_subject=True).nonzero()[0].tolist() == g["v1_out_follows"]
    assert R.neighbour_bindings(A, v2, D, x_is_subject=False).nonzero()[0].tolist() == g["v0_in_director"]
    assert R.neighbour_bindings(A, v2, F, x_is_subject=False).nonzero()[0].tolist() == g["v3_in_follows"]
    # Eq. 14 alone: OR over the rows of a binding matrix = the set of its columns
    M = R.binding_matrix_rows(A, v2, F)
    assert R.binding_vector(M).nonzero()[0].tolist() == sorted({j for i, j in zip(*M.nonzero())})


def test_eq17_out_out_fig1(golden_fig):
    """Eq. 17: rows holding both labels (Fig. 1a: actor and director)."""
    s, p, o = fixtures.fig1_triples()
    A = R.label_matrix(s, p, o, 8)
    P = fixtures.PREDICATE_IDS
    v = R.grouped_eval_out_out(A, P["actor"], P["director"])
    assert v.nonzero()[0].tolist() == golden_fig["eq17_actor_and_director_rows"]
    # label order is irrelevant, a label no row holds empties it
    assert R.grouped_eval_out_out(A, P["director"], P["actor"]).tolist() == v.tolist()
    assert not R.grouped_eval_out_out(A, P["actor"], 9).any()


def test_level0_bitmaps_fig1(golden_fig):
    """Eqs. 4/5 on Fig. 1 give the per-edge row/column sets; their AND (Eq. 21
    with two in-edges + one out-edge) is Ex. 7.2's surviving level-0 set."""
    s, p, o = fixtures.fig1_triples()
    A = R.label_matrix(s, p, o, 8)   # Fig. 1 has at most one label per cell
    F, D = fixtures.PREDICATE_IDS["follows"], fixtures.PREDICATE_IDS["director"]
    out_f = R.row_predicate_test(A, F)
    in_d = R.column_predicate_test(A, D)
    in_f = R.column_predicate_test(A, F)
    pe = golden_fig["level0_per_edge"]
    assert out_f.nonzero()[0].tolist() == pe["out_follows"]
    assert in_d.nonzero()[0].tolist() == pe["in_director"]
    assert in_f.nonzero()[0].tolist() == pe["in_follows"]
    v2 = R.vector_and(R.vector_and(out_f, in_d), in_f)
    assert v2.nonzero()[0].tolist() == golden_fig["level0_candidates"]
    # Eq. 17 / Eq. 21 helpers agree with the composition
    assert R.grouped_eval_in_out(A, D, F).nonzero()[0].tolist() == [1, 4, 5]


@pytest.mark.parametrize("back", [False, True])
def test_filter_schedule_fig1_steps(golden_fig, back):
    """Every step of the filter schedule on Fig. 1/2 (golden, hand-derived):
    group 0 -> {1,5} (Ex. 7.2), group 1 -> v0 = {2}, backward -> v2 = {1};
    with and without the back edges (group 1 then also tests v0 director v2
    against {1,5}: Product0 still qualifies)."""
    s, p, o = fixtures.fig1_triples()
    q = fixtures.fig2_query()
    plan = R.plan_degree(q)
    g = golden_fig["schedule_fig1"]
    one = dict(plan, groups=plan["groups"][:1], back=plan["back"][:1])
    c1, ok = R.filter_schedule(s, p, o, 8, q, plan=one, refine=False, back_edges=back)
    assert ok
    assert c1[2].nonzero()[0].tolist() == g["after_group0_v2"] == golden_fig["level0_candidates"]
    c2, _ = R.filter_schedule(s, p, o, 8, q, refine=False, back_edges=back)
    assert c2[0].nonzero()[0].tolist() == g["after_group1_v0"]
    assert c2[2].nonzero()[0].tolist() == g["after_group0_v2"]
    c3, _ = R.filter_schedule(s, p, o, 8, q, refine=True, back_edges=back)
    assert c3[2].nonzero()[0].tolist() == g["after_refine_v2"]
    assert c3[0].nonzero()[0].tolist() == g["after_group1_v0"]
    for v in g["never_centers"]:
        assert c3[v].all()


def _tree_no_multi(q):
    """True if the variable graph (patterns between two distinct variables) is
    a spanning tree of the variables with at most one pattern per pair."""
    pairs = [(min(a, b), max(a, b)) for a, _, b in q.edges
             if a != b and not q.is_const(a) and not q.is_const(b)]
    if len(set(pairs)) != len(pairs):
        return False
    parent = {v: v for v in q.variables}

    def find(x):
        while parent[x] != x:
            x = parent[x]
        return x
    for a, b in pairs:
        ra, rb = find(a), find(b)
        if ra == rb:
            return False
        parent[ra] = rb
    return len({find(v) for v in q.variables}) == 1


@pytest.mark.parametrize("back", [False, True])
def test_filter_schedule_root_exact_acyclic(back):
    """Exactness, not just soundness: for a connected query whose variable graph
    is a tree (constants and self-loops allowed), the forward pass followed by
    the backward re-evaluation is a bottom-up semijoin reduction, so the root's
    candidate set equals the projection of the brute-force answer on the root.
    A dropped term, a wrong direction or a wrong neighbour fails it."""
    checked = 0
    for seed in range(1500):
        (s, p, o), n, P, q = tiny.random_case(seed)
        if not _tree_no_multi(q):
            continue
        plan = R.plan_degree(q)
        if len(plan["roots"]) != 1:
            continue
        rows = R.brute_force(s, p, o, n, q)
        cand, ok = R.filter_schedule(s, p, o, n, q, plan=plan, refine=True, back_edges=back)
        r = plan["roots"][0]
        proj = sorted({row[q.variables.index(r)] for row in rows})
        assert cand[r].nonzero()[0].tolist() == proj, (seed, q)
        checked += 1
    assert checked > 300


# ---------------------------------------------------------------- §6.1 planner
def test_ex62_degree_plan(golden_fig):
    q = fixtures.fig2_query()
    pl = R.plan_degree(q)
    assert pl["roots"] == [golden_fig["root"]]
    assert len(pl["groups"]) == 2
    c0, g0 = pl["groups"][0]
    assert c0 == golden_fig["group0_center"]
    assert sorted(q.edges[k] for k, _, _ in g0) == sorted(tuple(x) for x in golden_fig["group0_edges"])
    c1, g1 = pl["groups"][1]
    assert [q.edges[k] for k, _, _ in g1] == [tuple(x) for x in golden_fig["group1_edges"]]
    assert c1 == 0  # evaluated at v0, direction-consistent (R18)
    assert g1[0][1] == R.OUT
    assert max(pl["level"]) + 1 == golden_fig["edge_levels_L0"]
    assert sorted(pl["paths"][2]) == sorted(golden_fig["paths"])


def test_ex61_direction_plan(golden_fig):
    """Ex. 6.1: the direction-driven traversal of Fig. 2b."""
    q = fixtures.fig2_query()
    pl = R.plan_direction(q)
    assert pl["roots"] == golden_fig["ex61_roots"]
    got = [[c, [list(q.edges[k]) for k, _, _ in g]] for c, g in pl["groups"]]
    assert got == golden_fig["ex61_direction_groups"]
    assert all(d == R.OUT for _, g in pl["groups"] for _, d, _ in g)  # rows of the CSR LSpM only


def test_direction_plan_invariants():
    """Every pattern evaluated exactly once, at its source (OUT); roots have no
    unevaluated incoming edge unless the rest is cyclic; constants refused."""
    checked = 0
    for seed in range(400):
        (_, _, _), n, P, q = tiny.random_case(seed, n_consts=0)
        pl = R.plan_direction(q)
        ks = [k for _, g in pl["groups"] for k, _, _ in g]
        assert sorted(ks) == list(range(len(q.edges)))
        for v, g in pl["groups"]:
            for k, d, w in g:
                assert q.edges[k][0] == v and q.edges[k][2] == w and d == R.OUT
        assert sorted(pl["pi"]) == q.variables
        checked += 1
    assert checked == 400
    with pytest.raises(ValueError):
        R.plan_direction(Query((None, 3), ((0, 1, 1),)))


def test_filter_schedule_direction_sound_and_exact():
    """The schedule under direction-driven plans: sound (⊇ projections) and,
    for acyclic connected queries whose variable graph is a tree, the first
    root's set is exact when every pattern points away from it (an
    out-tree: the backward pass is a bottom-up semijoin)."""
    exact = 0
    for seed in range(600):
        (s, p, o), n, P, q = tiny.random_case(seed, n_consts=0)
        rows = R.brute_force(s, p, o, n, q)
        plan = R.plan_direction(q)
        cand, ok = R.filter_schedule(s, p, o, n, q, plan=plan, refine=True)
        for ci, v in enumerate(q.variables):
            assert all(cand[v][r[ci]] for r in rows), (seed, v)
        if _tree_no_multi(q) and len(plan["roots"]) == 1 and not any(a == b for a, _, b in q.edges):
            r0 = plan["roots"][0]
            proj = sorted({row[q.variables.index(r0)] for row in rows})
            assert cand[r0].nonzero()[0].tolist() == proj, (seed, q)
            exact += 1
    assert exact > 50


def test_planner_constants_seed_and_root():
    # ?x worksFor <D> . ?x name ?y  : the constant edge is a seed, root = x
    q = Query((None, None, 7), ((0, 6, 2), (0, 2, 1)))
    pl = R.plan_degree(q)
    assert pl["seeds"] == [0]
    assert pl["roots"] == [0]
    assert pl["pi"] == [0, 1]


def test_planner_covers_every_edge_once():
    for seed in range(300):
        (_, _, _), n, P, q = tiny.random_case(seed)
        pl = R.plan_degree(q)
        ks = list(pl["seeds"]) + [k for _, g in pl["groups"] for k, _, _ in g]
        assert sorted(ks) == list(range(len(q.edges)))
        assert sorted(pl["pi"]) == q.variables
        for v, grp in pl["groups"]:
            for k, d, w in grp:
                a, _, b = q.edges[k]
                assert (a == v and b == w and d == R.OUT) or (b == v and a == w and d == R.IN)


# ---------------------------------------------------------------- §6.2 LSpM
def test_ex63_lspm_csr(golden_fig):
    s, p, o = fixtures.fig1_triples()
    keep = [fixtures.PREDICATE_IDS[x] for x in ("follows", "actor", "director")]
    d = R.lspm_paper_form(s, p, o, 8, keep)
    assert d["Mr"] == golden_fig["ex63_Mr"]
    assert d["nnz"] == golden_fig["ex63_nnz"]
    assert d["rows"] == golden_fig["ex63_reduced_rows"]
    assert d["Pr"][:4] == golden_fig["ex63_Pr_prefix"]
    assert d["Val"][:6] == golden_fig["ex63_Val_prefix"]
    assert d["Col"][:6] == golden_fig["ex63_Col_prefix"]


def test_ex64_counts(golden_fig):
    s, p, o = fixtures.fig1_triples()
    P = fixtures.PREDICATE_IDS
    g = golden_fig
    csr = R.lspm_paper_form(s, p, o, 8, [P[x] for x in g["ex64_csr"]["keep"]])
    assert (csr["rows"], csr["nnz"]) == (g["ex64_csr"]["rows"], g["ex64_csr"]["nnz"])
    csc = R.lspm_csc_paper_form(s, p, o, 8, [P[x] for x in g["ex64_csc"]["keep"]])
    assert (csc["cols"], csc["nnz"]) == (g["ex64_csc"]["cols"], g["ex64_csc"]["nnz"])


def test_lspm_arrays_definition():
    """row_ptr/col/pred reproduce the de-duplicated triple set, rows sorted by
    (pred, col) within each row."""
    s, p, o = tiny.random_graph(3, 50, 4, 400)
    for fmt in ("csr", "csc"):
        d = R.lspm_arrays(s, p, o, 50, fmt=fmt)
        rp, col, pred = d["row_ptr"], d["col"], d["pred"]
        got = set()
        for r in range(50):
            ent = list(zip(pred[rp[r]:rp[r + 1]].tolist(), col[rp[r]:rp[r + 1]].tolist()))
            assert ent == sorted(set(ent))
            got |= {(r, l, c) for l, c in ent}
        T = R.triple_set(s, p, o)
        exp = T if fmt == "csr" else {(c, l, a) for a, l, c in T}
        assert got == exp


# ---------------------------------------------------------------- brute force pins
@pytest.mark.parametrize("chunk", range(4))
def test_c_oracle_equals_brute_force_random(chunk):
    for seed in range(chunk * 300, (chunk + 1) * 300):
        (s, p, o), n, P, q = tiny.random_case(seed)
        assert _rows(oracle_bgp(s, p, o, q)) == R.brute_force(s, p, o, n, q), seed


def test_tree_dp_equals_brute_force_random():
    checked = 0
    for seed in range(600):
        (s, p, o), n, P, q = tiny.random_case(seed, extra_edges=0)
        try:
            cnt = R.tree_dp_count(s, p, o, n, q)
        except ValueError:
            continue
        assert cnt == len(R.brute_force(s, p, o, n, q)), seed
        checked += 1
    assert checked > 300


def test_filter_schedule_sound_random():
    """Every candidate set contains the projection of the answer (soundness of
    Eqs. 17/21 pruning), on tree and cyclic queries; the back edges only
    shrink the sets."""
    for seed in range(300):
        (s, p, o), n, P, q = tiny.random_case(seed)
        rows = R.brute_force(s, p, o, n, q)
        for refine in (False, True):
            c0, _ = R.filter_schedule(s, p, o, n, q, refine=refine)
            cb, _ = R.filter_schedule(s, p, o, n, q, refine=refine, back_edges=True)
            for v in q.variables:
                assert not (cb[v] & ~c0[v]).any(), (seed, v)
        for refine, back in ((False, False), (True, False), (True, True)):
            cand, ok = R.filter_schedule(s, p, o, n, q, refine=refine, back_edges=back)
            for ci, v in enumerate(q.variables):
                proj = {r[ci] for r in rows}
                assert all(cand[v][x] for x in proj), (seed, v)


# ---------------------------------------------------------------- closed forms
def test_single_pattern_closed_form():
    """Eqs. 12-13: the answer of ?x l ?y is exactly {(s,o) : (s,l,o) in T}."""
    d = lubm.generate(1)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    q = Query((None, None), ((0, lubm.TAKES_COURSE, 1),))
    got = _rows(oracle_bgp(s, p, o, q))
    exp = sorted({(int(a), int(c)) for a, b, c in zip(s, p, o) if b == lubm.TAKES_COURSE})
    assert got == exp


def test_star_and_acyclic_counts_lubm1():
    """Acyclic LUBM queries: C oracle row count == tree-DP closed form (F5);
    L2 == number of generated courses (generator-analytic count)."""
    d = lubm.generate(1)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    qs = {q.name: q for q in lubm.queries(d)}
    for name in ("L2", "L4", "L5", "L6", "Q14"):
        q = qs[name]
        assert len(oracle_bgp(s, p, o, q)) == R.tree_dp_count(s, p, o, d.n_entities, q), name
    assert len(oracle_bgp(s, p, o, qs["L2"])) == d.n_courses


def test_lubm_generator_counters_pin_counts():
    """The LUBM generator's counters (used as expected counts at full size,
    where enumeration by the oracle is too slow) equal the oracle's counts."""
    d = lubm.generate(2)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    for q in lubm.queries(d):
        if q.name in d.counts:
            assert len(oracle_bgp(s, p, o, q)) == d.counts[q.name], q.name


def test_sampled_bindings_equal_full_oracle():
    """solutions_for_bindings (local triple subset around sampled bindings) is
    exactly the full answer restricted to those bindings."""
    d = lubm.generate(3)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    for q in lubm.queries(d):
        full = oracle_bgp(s, p, o, q)
        vals = np.unique(np.concatenate([full[:30, 0] if len(full) else np.zeros(0, np.uint32),
                                         np.array([5, 17, 1234], np.uint32)]))
        got = R.solutions_for_bindings(s, p, o, q, q.variables[0], vals)
        exp = full[np.isin(full[:, 0], vals)] if len(full) else full
        assert np.array_equal(got, exp), q.name


def test_zero_edge_and_const_only_queries():
    s, p, o = fixtures.fig1_triples()
    assert R.brute_force(s, p, o, 8, Query((), ())) == [()]
    assert oracle_bgp(s, p, o, Query((), ())).shape == (1, 0)
    # const-const guard true / false
    assert oracle_bgp(s, p, o, Query((0, 1), ((0, 1, 1),))).shape == (1, 0)
    assert oracle_bgp(s, p, o, Query((0, 1), ((0, 2, 1),))).shape == (0, 0)
