"""GPU parity of f2 (GSMART_FACTORISED: factorised binding trees, §7.1 /
§8.1) through the C ABI: the rows equal the oracle's, and the trees
themselves equal the oracle's binding trees (oracle/binding_trees.py) on the
worked example (Fig. 7/8) and on acyclic queries."""
import numpy as np
import pytest

from oracle import binding_trees as B
from oracle import reference as R
from oracle.coracle import oracle_bgp, OracleIndex
from synth import fixtures, tiny, lubm, watdiv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from conftest import build_product
    build_product()
    import paper_2106_14038_b200.gsmart as g
    return g


@pytest.fixture(scope="module")
def eng(G):
    e = G.Engine(0)
    yield e
    e.close()


def _rows(a):
    return [tuple(int(x) for x in r) for r in np.asarray(a).tolist()]


def _run(G, eng, q, flags):
    """rows, stats and the factorised trees as {vertex chain: set of alive tuples}."""
    pl = G.gsmart_plan(eng.ctx, q)
    r = G.gsmart_execute(eng.ctx, pl, flags)
    try:
        rows = None if flags & G.GSMART_COUNT_ONLY else G.gsmart_result_rows(r)
        n = G.gsmart_result_shape(r)[0]
        st = G.gsmart_result_stats(r)
        occ = []
        k = 0
        while True:
            try:
                v, par, cnt, pp, bp, ap = G.gsmart_result_tree(r, k)
            except G.GsmartError:
                break
            bind = G.gsmart_copy_to_host(eng.ctx, bp, cnt * 4) if cnt else np.zeros(0, np.uint32)
            parent = G.gsmart_copy_to_host(eng.ctx, pp, cnt * 4) if (cnt and k) else np.zeros(cnt, np.uint32)
            alive = G.gsmart_copy_to_host(eng.ctx, ap, cnt, dtype=np.uint8) if (cnt and ap) else np.ones(cnt, np.uint8)
            occ.append((v, par, bind, parent, alive))
            k += 1
    finally:
        G.gsmart_result_free(r)
        G.gsmart_plan_free(pl)
    return rows, n, st, occ


def _chains(occ):
    """Root-to-leaf chains of the occurrence tree with their alive tuples."""
    chain, tup = [], []
    kids = {i: [] for i in range(len(occ))}
    for i, (v, par, bind, parent, alive) in enumerate(occ):
        if par >= 0:
            kids[par].append(i)
        if par < 0:
            chain.append((v,))
            tup.append([(int(b),) if a else None for b, a in zip(bind, alive)])
        else:
            chain.append(chain[par] + (v,))
            tup.append([tup[par][int(pa)] + (int(b),) if (a and tup[par][int(pa)] is not None) else None
                        for b, pa, a in zip(bind, parent, alive)])
    out = {}
    for i in range(len(occ)):
        if not kids[i]:
            out.setdefault(chain[i], set()).update(t for t in tup[i] if t is not None)
    return out


def _oracle_chains(bt, root):
    out = {}
    for b, per in bt["trees"][root].items():
        for P, X in zip(bt["paths"][root], per):
            out.setdefault(tuple(P), set()).update(X)
    return out


def test_fig78_trees(G, eng, golden_fig):
    """Fig. 7/8: root binding 1 survives (Ex. 7.2: 5 dies at level 1 even
    without the backward refinement), Ω = {v1}, and the pruned trees are
    Fig. 8's."""
    s, p, o = fixtures.fig1_triples()
    eng.load(s, p, o, 8, 4)
    q = fixtures.fig2_query()
    g = golden_fig["fig8_trees_root1"]
    for flags in (G.GSMART_NO_REFINE, G.GSMART_REFINE):
        rows, n, st, occ = _run(G, eng, q, G.GSMART_FACTORISED | flags)
        assert _rows(rows) == [tuple(r) for r in golden_fig["solution_rows"]]
        assert st["factorised"] == 1 and st["n_omega"] == 1
        got = _chains(occ)
        exp = {tuple(P): {tuple(t) for t in X} for P, X in zip(g["paths"], g["trees"])}
        assert got == exp
        assert st["combinations"] == 2


def test_fig12_count_only(G, eng):
    s, p, o = fixtures.fig1_triples()
    eng.load(s, p, o, 8, 4)
    assert eng.query(fixtures.fig2_query(), flags=G.GSMART_FACTORISED | G.GSMART_COUNT_ONLY) == 2


@pytest.mark.parametrize("chunk", range(5))
def test_random_tiny_rows(G, eng, chunk):
    """Rows (and COUNT_ONLY counts) == brute force on random tiny cases:
    cycles, self-loops, multi-edges, constants, absent constants, cross products."""
    for seed in range(chunk * 200, chunk * 200 + 200):
        (s, p, o), n, P, q = tiny.random_case(seed)
        exp = R.brute_force(s, p, o, n, q)
        eng.load(s, p, o, n, P)
        got = eng.query(q, flags=G.GSMART_FACTORISED)
        assert _rows(got) == exp, (seed, q)
        assert eng.query(q, flags=G.GSMART_FACTORISED | G.GSMART_COUNT_ONLY) == len(exp), (seed, q)


def test_acyclic_trees_equal_oracle(G, eng):
    """Acyclic one-root queries (no Ω): the alive tuples of every root-to-leaf
    chain are exactly the oracle's binding trees of that path."""
    n_cases = 0
    for seed in range(400):
        (s, p, o), n, P, q = tiny.random_case(20000 + seed, max_entities=6, n_consts=0, extra_edges=0,
                                              allow_self_loops=False)
        pl = R.plan_degree(q)
        if len(pl["roots"]) != 1 or len(q.edges) != len({(min(a, b), max(a, b)) for a, _, b in q.edges}):
            continue
        eng.load(s, p, o, n, P)
        rows, cnt, st, occ = _run(G, eng, q, G.GSMART_FACTORISED)
        bt = B.binding_trees(s, p, o, n, q, omega=False)
        exp = _oracle_chains(bt, pl["roots"][0])
        got = _chains(occ)
        assert {k: v for k, v in got.items() if v} == {k: v for k, v in exp.items() if v}, (seed, q)
        assert st["n_omega"] == 0 and st["combinations"] == cnt
        n_cases += 1
    assert n_cases > 50


def test_omega_trees_sound(G, eng):
    """Cyclic queries: every solution's projection on a chain is in the GPU's
    pruned tree of that chain (Ω pruning never drops a solution)."""
    for seed in range(300):
        (s, p, o), n, P, q = tiny.random_case(30000 + seed, max_entities=6, extra_edges=2)
        eng.load(s, p, o, n, P)
        rows, cnt, st, occ = _run(G, eng, q, G.GSMART_FACTORISED)
        exp = R.brute_force(s, p, o, n, q)
        assert _rows(rows) == exp
        for chain, X in _chains(occ).items():
            cols = [q.variables.index(v) for v in chain]
            assert {tuple(r[c] for c in cols) for r in exp} <= X, (seed, q, chain)


def _check_dataset(G, eng, s, p, o, N, P, qs):
    eng.load(s, p, o, N, P)
    sn, pn, on = (np.asarray(x) for x in (s, p, o))
    for q in qs:
        exp = oracle_bgp(sn, pn, on, q)
        got = eng.query(q, flags=G.GSMART_FACTORISED)
        assert np.array_equal(got, exp), q.name
        trie = eng.query(q)
        assert np.array_equal(got, trie), q.name
        assert eng.query(q, flags=G.GSMART_FACTORISED | G.GSMART_COUNT_ONLY) == len(exp), q.name


@pytest.mark.parametrize("U", [2, 10])
def test_lubm_rows(G, eng, U):
    """U = 10: levels outgrow the first workspace (grow + re-run the expansion,
    Ω key sets re-sized with them)."""
    d = lubm.generate(U)
    _check_dataset(G, eng, d.s.numpy(), d.p.numpy(), d.o.numpy(), d.n_entities, d.n_predicates, lubm.queries(d))


def test_watdiv_rows(G, eng):
    d = watdiv.generate(0.01)
    _check_dataset(G, eng, d.s.numpy(), d.p.numpy(), d.o.numpy(), d.n_entities, d.n_predicates, watdiv.queries(d))


@pytest.mark.parametrize("seed,N,P,M,skew", [(11, 2000, 3, 150000, 1.3), (13, 500, 2, 120000, 1.6)])
def test_skewed_graphs_rows(G, eng, seed, N, P, M, skew):
    """Hub rows (> 16384 entries) and many tiles per occurrence; data-driven
    queries (stars, chains, cycles) as in the trie parity test."""
    from test_gpu_parity import _data_queries
    s, p, o = tiny.random_graph(seed, N, P, M, skew=skew)
    eng.load(s, p, o, N, P)
    ix = OracleIndex(s, p, o)
    rng = np.random.default_rng(seed)
    for q in _data_queries(rng, s, p, o, 25):
        exp = ix.query(q)
        if len(exp) > 3_000_000:
            continue
        got = eng.query(q, flags=G.GSMART_FACTORISED)
        assert got.shape == exp.shape and np.array_equal(got, exp), q


def test_direction_plans_rows(G, eng):
    """Direction-driven plans (multi-root, §8.2's Φ variables as occurrences)."""
    n = 0
    for seed in range(300):
        (s, p, o), nn, P, q = tiny.random_case(40000 + seed, n_consts=0)
        exp = R.brute_force(s, p, o, nn, q)
        eng.load(s, p, o, nn, P)
        with eng.plan(q, traversal=G.GSMART_DIRECTION) as pl:
            got = pl.run(flags=G.GSMART_FACTORISED)
        assert _rows(got) == exp, (seed, q)
        n += 1
    assert n == 300


def test_split_keep_sets_refused_or_exact(G, eng):
    """With query-dependent keep-sets a second occurrence may need a label its
    format does not hold: the execute is refused (E_STATE), never wrong."""
    s, p, o = fixtures.fig1_triples()
    q = fixtures.fig2_query()
    exp = R.brute_force(s, p, o, 8, q)
    eng.load(s, p, o, 8, 4)
    with eng.plan(q) as pl:
        csr, csc = G.gsmart_plan_keep_sets([pl.h])
    G.gsmart_build_lspm_split(eng.ctx, csr, csc)
    with eng.plan(q) as pl:
        assert _rows(pl.run()) == exp  # the trie reads only what the keep-sets hold
        try:
            got = pl.run(flags=G.GSMART_FACTORISED)
        except G.GsmartError as e:
            assert "E_STATE" in str(e), e
        else:
            assert _rows(got) == exp
