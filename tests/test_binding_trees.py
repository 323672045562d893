"""Pins of the f2 oracle (oracle/binding_trees.py: §7.1 binding trees, §7.2.2
pre-pruning, §8.1/8.2 tree pruning) against the paper's worked example and
brute force.  CPU only (-m "not gpu")."""
import pytest

from oracle import binding_trees as B
from oracle import reference as R
from synth import fixtures, tiny


def _fig():
    s, p, o = fixtures.fig1_triples()
    return s, p, o, fixtures.FIG1_N_ENTITIES, fixtures.fig2_query()


def _as_lists(per):
    return [sorted(list(t) for t in X) for X in per]


def test_fig7_trees_before_local_pruning(golden_fig):
    """Ex. 7.2 / Fig. 7: only root binding 1 survives the main computation, with
    one binding tree per path of Ex. 7.1."""
    s, p, o, N, q = _fig()
    bt = B.binding_trees(s, p, o, N, q, omega=False)
    g = golden_fig["fig7_trees_root1"]
    assert [list(P) for P in bt["paths"][2]] == g["paths"]
    assert sorted(bt["trees"][2]) == golden_fig["ex72_surviving_root_bindings"]
    assert _as_lists(bt["trees"][2][1]) == g["trees"]


def test_fig8_local_tree_pruning(golden_fig):
    """Ex. 8.1 / Fig. 8: Ω = {v1}; binding 5 of v1 is missing from the first
    tree, so its node goes from the third tree."""
    s, p, o, N, q = _fig()
    bt = B.binding_trees(s, p, o, N, q)
    assert bt["omega"][2] == golden_fig["ex81_omega"]
    assert _as_lists(bt["trees"][2][1]) == golden_fig["fig8_trees_root1"]["trees"]
    assert B.factorised_rows(bt, q) == [tuple(r) for r in golden_fig["solution_rows"]]


def test_fig7_tree_sizes():
    """Node counts of the Fig. 7 trees (root node included): 4, 2, 3."""
    s, p, o, N, q = _fig()
    bt = B.binding_trees(s, p, o, N, q, omega=False)
    assert B.tree_sizes(bt)[(2, 1)] == [4, 2, 3]


def test_paths_match_planner():
    """plan_paths reproduces plan_degree's Ex. 7.1 paths on Fig. 2."""
    pl = R.plan_degree(fixtures.fig2_query())
    assert sorted(B.plan_paths(pl)[2]) == sorted(tuple(P) for P in pl["paths"][2])


@pytest.mark.parametrize("chunk", range(4))
def test_rows_equal_brute_force(chunk):
    """The join of the pruned trees is exactly the BGP answer,
    with Ω pruning on and off, on random tiny cases (cycles, self-loops,
    multi-edges, constants, absent constants)."""
    for seed in range(chunk * 100, chunk * 100 + 100):
        (s, p, o), n, P, q = tiny.random_case(9000 + seed, max_entities=5)
        exp = R.brute_force(s, p, o, n, q)
        for omega in (True, False):
            bt = B.binding_trees(s, p, o, n, q, omega=omega)
            assert B.factorised_rows(bt, q) == exp, (seed, omega, q)


def test_direction_plans_rows_equal_brute_force():
    """Multi-root direction plans (§8.2 global pruning over Φ)."""
    n_multi = 0
    for seed in range(300):
        (s, p, o), n, P, q = tiny.random_case(7000 + seed, max_entities=5, n_consts=0)
        pl = R.plan_direction(q)
        bt = B.binding_trees(s, p, o, n, q, plan=pl)
        n_multi += len(pl["roots"]) > 1 and bool(bt["phi"])
        assert B.factorised_rows(bt, q) == R.brute_force(s, p, o, n, q), (seed, q)
    assert n_multi > 10


def _projections(rows, q, P):
    cols = [q.variables.index(v) for v in P]
    return {tuple(r[c] for c in cols) for r in rows}


def test_acyclic_trees_are_final_results():
    """for an acyclic one-root query without several constants the
    main computation's trees "satisfy all the constraints and are the final
    results": every tuple of every path tree (no Ω step) is the projection of a
    solution, and every solution's projection is in the tree.  Exactness of
    pre-pruning (R-f2b)."""
    n_cases = 0
    for seed in range(600):
        (s, p, o), n, P, q = tiny.random_case(5000 + seed, max_entities=5, n_consts=0, extra_edges=0,
                                              allow_self_loops=False)
        pl = R.plan_degree(q)
        if len(pl["roots"]) != 1 or len(q.edges) != len({(min(a, b), max(a, b)) for a, _, b in q.edges}):
            continue
        rows = R.brute_force(s, p, o, n, q)
        bt = B.binding_trees(s, p, o, n, q, omega=False)
        r = pl["roots"][0]
        got = {P: set() for P in bt["paths"][r]}
        for b, per in bt["trees"][r].items():
            for Pth, X in zip(bt["paths"][r], per):
                got[Pth] |= X
        for Pth in bt["paths"][r]:
            assert got[Pth] == _projections(rows, q, Pth), (seed, q, Pth)
        n_cases += 1
    assert n_cases > 100


def test_pruning_is_sound():
    """Local/global pruning never removes a tuple that is part of a solution:
    each solution's projection on a path is in that path's tree."""
    for seed in range(300):
        (s, p, o), n, P, q = tiny.random_case(3000 + seed, max_entities=5)
        rows = R.brute_force(s, p, o, n, q)
        bt = B.binding_trees(s, p, o, n, q)
        for r, ps in bt["paths"].items():
            for Pth in ps:
                have = set()
                for b, per in bt["trees"][r].items():
                    have |= per[ps.index(Pth)]
                assert _projections(rows, q, Pth) <= have, (seed, q, Pth)


def test_omega_pruning_removes_something():
    """Guard against a no-op Ω step: on cyclic cases it must shrink some tree
    (Ex. 8.1 is one such case; random ones too)."""
    shrunk = 0
    for seed in range(300):
        (s, p, o), n, P, q = tiny.random_case(1000 + seed, max_entities=5, extra_edges=2)
        a = B.binding_trees(s, p, o, n, q, omega=False)
        b = B.binding_trees(s, p, o, n, q)
        sa = sum(len(X) for per_b in a["trees"].values() for per in per_b.values() for X in per)
        sb = sum(len(X) for per_b in b["trees"].values() for per in per_b.values() for X in per)
        assert sb <= sa
        shrunk += sb < sa
    assert shrunk > 5
