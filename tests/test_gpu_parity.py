"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by
element on the same seeded inputs.  Integer/boolean path => bit-exact."""
import numpy as np
import pytest

from oracle import reference as R
from oracle.coracle import oracle_bgp, OracleIndex
from synth import fixtures, tiny, lubm
from synth.query import Query

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


def _bits_to_set(words, n):
    b = np.unpackbits(words.view(np.uint8), bitorder="little")[:n]
    return set(np.nonzero(b)[0].tolist())


def _cands(G, eng, q, flags):
    """rows + candidate sets per variable from one execute."""
    pl = G.gsmart_plan(eng.ctx, q)
    r = G.gsmart_execute(eng.ctx, pl, flags | G.GSMART_KEEP_CANDIDATES)
    try:
        rows = G.gsmart_result_rows(r)
        cs = {}
        for v in q.variables:
            ptr, nw = G.gsmart_result_candidates(r, v)
            cs[v] = G.gsmart_copy_to_host(eng.ctx, ptr, nw * 4)
        st = G.gsmart_result_stats(r)
    finally:
        G.gsmart_result_free(r)
        G.gsmart_plan_free(pl)
    return rows, cs, st


# ------------------------------------------------------------------ worked example
def test_fig12_rows_and_level0(G, eng, golden_fig):
    s, p, o = fixtures.fig1_triples()
    eng.load(s, p, o, 8, 4)
    q = fixtures.fig2_query()
    rows, cs, _ = _cands(G, eng, q, G.GSMART_NO_REFINE)
    assert _rows(rows) == [tuple(r) for r in golden_fig["solution_rows"]]
    root = golden_fig["root"]
    assert sorted(_bits_to_set(cs[root], 8)) == golden_fig["level0_candidates"]  # Ex. 7.2
    rows2, cs2, st = _cands(G, eng, q, G.GSMART_REFINE)
    assert _rows(rows2) == [tuple(r) for r in golden_fig["solution_rows"]]
    assert sorted(_bits_to_set(cs2[root], 8)) == [1]
    assert st["level_alive"][-1] == 2


# ------------------------------------------------------------------ a1 LSpM arrays
@pytest.mark.parametrize("seed,N,P,M,keep", [(1, 50, 4, 400, None), (2, 3000, 300, 40000, None),
                                             (3, 1000, 7, 20000, [2, 5]), (4, 1, 1, 5, None),
                                             (5, 100, 3, 0, None)])
def test_lspm_arrays_match_definition(G, eng, seed, N, P, M, keep):
    s, p, o = tiny.random_graph(seed, N, P, M, skew=1.1 if M > 1000 else 0.0)
    # duplicates on purpose
    s = np.concatenate([s, s[: M // 3]]); p = np.concatenate([p, p[: M // 3]]); o = np.concatenate([o, o[: M // 3]])
    eng.load(s, p, o, N, P, keep=keep)
    for fmt, name in ((G.GSMART_CSR, "csr"), (G.GSMART_CSC, "csc")):
        v = G.gsmart_lspm_get(eng.ctx, fmt)
        ref = R.lspm_arrays(s, p, o, N, keep=keep, fmt=name)
        assert v["nnz"] == len(ref["col"])
        rp = G.gsmart_copy_to_host(eng.ctx, v["row_ptr"], (N + 1) * 4)
        col = G.gsmart_copy_to_host(eng.ctx, v["col"], v["nnz"] * 4)
        dt = np.uint8 if v["pred_bytes"] == 1 else np.uint16
        pred = G.gsmart_copy_to_host(eng.ctx, v["pred"], v["nnz"] * v["pred_bytes"], dtype=dt)
        np.testing.assert_array_equal(rp.astype(np.uint64), ref["row_ptr"])
        np.testing.assert_array_equal(col, ref["col"])
        np.testing.assert_array_equal(pred.astype(np.uint32), ref["pred"])
        # row label signatures: bit (l & 31) of every label present in the row
        lm = G.gsmart_copy_to_host(eng.ctx, v["label_mask"], N * 4)
        exp = np.zeros(N, dtype=np.uint64)
        rows = np.repeat(np.arange(N), np.diff(ref["row_ptr"].astype(np.int64)))
        np.bitwise_or.at(exp, rows, np.left_shift(1, ref["pred"].astype(np.uint64) & 31))
        np.testing.assert_array_equal(lm.astype(np.uint64), exp)


def test_lspm_wide_keys_match_definition(G):
    """(row, pred, col) keys wider than 63 bits (2^26 + 5 entities = 27 bits,
    10,000 labels = 14 bits: 68 bits, configs[4]'s shape) take the two-word
    sort path (low word first, then the high word, both with the
    hand-written radix sort): CSR/CSC arrays and the label-major lists equal
    the definition; ids span the whole range (top bits exercised), with
    duplicates and a keep-set."""
    N, P, M = (1 << 26) + 5, 10_000, 300_000
    rng = np.random.default_rng(68)
    s = rng.integers(0, N, M).astype(np.uint32)
    o = rng.integers(0, N, M).astype(np.uint32)
    s[:1000] = N - 1 - rng.integers(0, 3, 1000)   # rows at the top of the id range
    p = rng.integers(1, P + 1, M).astype(np.uint32)
    s = np.concatenate([s, s[:5000]]); p = np.concatenate([p, p[:5000]]); o = np.concatenate([o, o[:5000]])
    e = G.Engine(0)
    try:
        for keep in (None, list(range(1, P + 1, 3))):
            e.load(s, p, o, N, P, keep=keep)
            for fmt, name in ((G.GSMART_CSR, "csr"), (G.GSMART_CSC, "csc")):
                v = G.gsmart_lspm_get(e.ctx, fmt)
                ref = R.lspm_arrays(s, p, o, N, keep=keep, fmt=name)
                assert v["nnz"] == len(ref["col"])
                rp = G.gsmart_copy_to_host(e.ctx, v["row_ptr"], (N + 1) * 4)
                col = G.gsmart_copy_to_host(e.ctx, v["col"], v["nnz"] * 4)
                pred = G.gsmart_copy_to_host(e.ctx, v["pred"], v["nnz"] * 2, dtype=np.uint16)
                np.testing.assert_array_equal(rp.astype(np.uint64), ref["row_ptr"])
                np.testing.assert_array_equal(col, ref["col"])
                np.testing.assert_array_equal(pred.astype(np.uint32), ref["pred"])
        # queries through the wide-key LSpM and label-major lists (push form forced too)
        e.load(s, p, o, N, P)
        ix = OracleIndex(s, p, o)
        hub = int(np.bincount(p).argmax())
        qs = [Query((None, None), ((0, hub, 1),)),
              Query((None, None, None), ((0, int(p[0]), 1), (0, int(p[1]), 2))),
              Query((None, None, int(o[7])), ((0, int(p[7]), 2), (0, int(p[8]), 1)))]
        for q in qs:
            assert np.array_equal(e.query(q), ix.query(q)), q
    finally:
        e.close()


def test_powerlaw_wide_keys_vs_oracle(G):
    """configs[4]'s id widths at reduced triple count: 100M entities, 10,000
    labels (68-bit keys), 3M power-law triples; random-walk queries == C oracle."""
    from synth import powerlaw
    d = powerlaw.generate(3_000_000, 100_000_000, 10_000)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    e = G.Engine(0)
    try:
        G.gsmart_load_triples(e.ctx, d.s.cuda(), d.p.cuda(), d.o.cuda(), d.n_entities, d.n_predicates)
        G.gsmart_build_lspm(e.ctx)
        ix = OracleIndex(s, p, o)
        qs = powerlaw.queries(d, 15, seed=5)
        for q, got in zip(qs, e.query_batch(qs)):
            x = ix.query(q)
            assert got.shape == x.shape and np.array_equal(got, x), q
    finally:
        e.close()


# ------------------------------------------------------------------ random tiny cases
@pytest.mark.parametrize("chunk", range(5))
def test_random_tiny_rows_and_candidates(G, eng, chunk):
    for seed in range(chunk * 200, (chunk + 1) * 200):
        (s, p, o), n, P, q = tiny.random_case(seed)
        eng.load(s, p, o, n, P)
        exp = R.brute_force(s, p, o, n, q)
        for flags, refine, back in ((G.GSMART_REFINE, True, False), (0, False, False),
                                    (G.GSMART_REFINE | G.GSMART_BACK_EDGES, True, True)):
            rows, cs, _ = _cands(G, eng, q, flags)
            assert _rows(rows) == exp, (seed, q)
            ref, _ = R.filter_schedule(s, p, o, n, q, refine=refine, back_edges=back)
            for v in q.variables:
                got = _bits_to_set(cs[v], n)
                assert got == set(np.nonzero(ref[v])[0].tolist()), (seed, v, q, flags)


# ------------------------------------------------------------------ query-dependent LSpM (f3)
def test_split_keep_sets(G, golden_fig):
    """Direction-split keep-sets (§6.2, Ex. 6.4): built with the sets a batch of
    plans needs, the CSR/CSC hold only their labels (Fig. 1: 6 and 9 entries,
    R20), rows == oracle on the full triple set; a plan reading a label a
    format dropped is refused (E_STATE)."""
    from synth import lubm
    e = G.Engine(0)
    try:
        s, p, o = fixtures.fig1_triples()
        q = fixtures.fig2_query()
        G.gsmart_load_triples(e.ctx, s, p, o, 8, 4)
        h = G.gsmart_plan(None, q)
        csr, csc = G.gsmart_plan_keep_sets([h])
        G.gsmart_plan_free(h)
        G.gsmart_build_lspm_split(e.ctx, csr, csc)
        assert G.gsmart_lspm_get(e.ctx, G.GSMART_CSR)["nnz"] == golden_fig["ex64_csr"]["nnz"]
        assert G.gsmart_lspm_get(e.ctx, G.GSMART_CSC)["nnz"] == golden_fig["ex64_csc"]["nnz"]
        assert _rows(e.query(q)) == [tuple(r) for r in golden_fig["solution_rows"]]
        d = lubm.generate(5)
        s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
        qs = lubm.queries(d)
        G.gsmart_load_triples(e.ctx, s, p, o, d.n_entities, d.n_predicates)
        plans = [G.gsmart_plan(None, q) for q in qs]
        csr, csc = G.gsmart_plan_keep_sets(plans)
        G.gsmart_build_lspm_split(e.ctx, csr, csc)
        ix = OracleIndex(s, p, o)
        for q, r in zip(qs, G.gsmart_execute_batch(e.ctx, plans, 0)):
            assert np.array_equal(G.gsmart_result_rows(r), ix.query(q)), q.name
            G.gsmart_result_free(r)
        for pl in plans:
            G.gsmart_plan_free(pl)
        missing = sorted(set(range(1, d.n_predicates + 1)) - set(csr))
        bad = Query((None, None), ((0, missing[0], 1),))
        with pytest.raises(G.GsmartError) as ei:
            e.query(bad)
        assert ei.value.name == "E_STATE"
    finally:
        e.close()


# ------------------------------------------------------------------ direction-driven plans (§6.1.1, f1)
def test_direction_plans_rows_and_candidates(G, eng, golden_fig):
    """GSMART_DIRECTION (CSR-side groups, multi-root plans joined in one trie):
    rows == brute force and every candidate bitmap == filter_schedule under
    the oracle's plan_direction, refine on and off; Fig. 2 (two roots, Ex. 6.1)."""
    s, p, o = fixtures.fig1_triples()
    eng.load(s, p, o, 8, 4)
    q = fixtures.fig2_query()
    assert _rows(eng.query(q, traversal=G.GSMART_DIRECTION)) == [tuple(r) for r in golden_fig["solution_rows"]]
    for seed in range(600):
        (s, p, o), n, P, q = tiny.random_case(seed, n_consts=0)
        eng.load(s, p, o, n, P)
        exp = R.brute_force(s, p, o, n, q)
        plan = R.plan_direction(q)
        for flags, refine in ((G.GSMART_REFINE, True), (0, False)):
            pl = G.gsmart_plan(eng.ctx, q, G.GSMART_DIRECTION)
            r = G.gsmart_execute(eng.ctx, pl, flags | G.GSMART_KEEP_CANDIDATES)
            try:
                assert _rows(G.gsmart_result_rows(r)) == exp, (seed, q)
                ref, _ = R.filter_schedule(s, p, o, n, q, plan=plan, refine=refine)
                for v in q.variables:
                    ptr, nw = G.gsmart_result_candidates(r, v)
                    got = _bits_to_set(G.gsmart_copy_to_host(eng.ctx, ptr, nw * 4), n)
                    assert got == set(np.nonzero(ref[v])[0].tolist()), (seed, v, q)
            finally:
                G.gsmart_result_free(r)
                G.gsmart_plan_free(pl)


def test_direction_plans_csr_only(G):
    """The CSR-only LSpM (the direction-driven storage): direction
    plans read subject rows only — a later root is a free level joined by a
    closing edge checked in a CSR row; rows == brute force / C oracle.  A
    degree-driven plan needs CSC: E_STATE."""
    e = G.Engine(0)
    try:
        for seed in range(300):
            (s, p, o), n, P, q = tiny.random_case(seed, n_consts=0)
            G.gsmart_load_triples(e.ctx, s, p, o, n, P)
            G.gsmart_build_lspm(e.ctx, formats=G.GSMART_CSR)
            assert _rows(e.query(q, traversal=G.GSMART_DIRECTION)) == R.brute_force(s, p, o, n, q), (seed, q)
        with pytest.raises(G.GsmartError) as ei:
            e.query(q)
        assert ei.value.name == "E_STATE"
        from synth import watdiv
        d = watdiv.generate(0.02)
        s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
        G.gsmart_load_triples(e.ctx, s, p, o, d.n_entities, d.n_predicates)
        G.gsmart_build_lspm(e.ctx, formats=G.GSMART_CSR)
        ix = OracleIndex(s, p, o)
        for q in [q for q in watdiv.queries(d) if all(v is None for v in q.vertices)]:
            got = e.query(q, traversal=G.GSMART_DIRECTION)
            x = ix.query(q)
            assert got.shape == x.shape and np.array_equal(got, x), q.name
    finally:
        e.close()


def test_direction_plans_watdiv_vs_oracle(G, eng):
    """The variable-only WatDiv templates (C1, C3) and random-walk power-law
    queries planned direction-driven == C oracle (same rows as degree-driven)."""
    from synth import watdiv, powerlaw
    d = watdiv.generate(0.02)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    eng.load(s, p, o, d.n_entities, d.n_predicates)
    ix = OracleIndex(s, p, o)
    qs = [q for q in watdiv.queries(d) if all(v is None for v in q.vertices)]
    assert len(qs) >= 2
    for q, got in zip(qs, eng.query_batch(qs, traversal=G.GSMART_DIRECTION)):
        e = ix.query(q)
        assert got.shape == e.shape and np.array_equal(got, e), q.name
    d = powerlaw.generate(400_000, 20_000, 200)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    eng.load(s, p, o, d.n_entities, d.n_predicates)
    ix = OracleIndex(s, p, o)
    qs = [q for q in powerlaw.queries(d, 15, seed=9) if all(v is None for v in q.vertices)]
    for q, got in zip(qs, eng.query_batch(qs, traversal=G.GSMART_DIRECTION)):
        e = ix.query(q)
        assert got.shape == e.shape and np.array_equal(got, e), q


# ------------------------------------------------------------------ larger, skewed graphs
def _data_queries(rng, s, p, o, n_q):
    """random connected queries whose constants come from the data (non-empty-ish)."""
    out = []
    for _ in range(n_q):
        q = tiny.random_query(rng, int(max(s.max(), o.max())) + 1, int(p.max()),
                              n_vars=int(rng.integers(2, 5)), n_consts=int(rng.integers(0, 2)),
                              extra_edges=int(rng.integers(0, 2)))
        # replace constants by a random subject/object that exists
        verts = list(q.vertices)
        for i, c in enumerate(verts):
            if c is not None:
                verts[i] = int(s[rng.integers(0, len(s))]) if rng.random() < 0.5 else int(o[rng.integers(0, len(o))])
        out.append(Query(tuple(verts), q.edges))
    return out


@pytest.mark.parametrize("seed,N,P,M,skew", [(11, 2000, 3, 150000, 1.3), (12, 20000, 6, 200000, 0.0),
                                             (13, 500, 2, 120000, 1.6)])
def test_skewed_graphs_vs_oracle(G, eng, seed, N, P, M, skew):
    """Hub rows beyond the warp-cooperative threshold and beyond HEAVY_ROW
    (16384 entries) exercise all three group-filter paths and chunked expansion."""
    s, p, o = tiny.random_graph(seed, N, P, M, skew=skew)
    eng.load(s, p, o, N, P)
    ix = OracleIndex(s, p, o)
    rng = np.random.default_rng(seed)
    for q in _data_queries(rng, s, p, o, 25):
        exp = ix.query(q)
        if len(exp) > 3_000_000:
            continue
        with eng.plan(q) as pl:
            got = pl.run()
        assert got.shape == exp.shape and np.array_equal(got, exp), q


# ------------------------------------------------------------------ LUBM-shaped
def _relabel(q, perm):
    """The same query with vertex i renamed perm[i] (changes the output column order)."""
    inv = {old: new for new, old in enumerate(perm)}
    verts = [q.vertices[perm[i]] for i in range(q.n_vertices)]
    edges = [(inv[s], pr, inv[o]) for s, pr, o in q.edges]
    return Query(verts, edges, name=q.name + "_perm")


@pytest.mark.parametrize("U", [10])
def test_permuted_column_order_sorts(G, eng, U):
    """Relabelled variables make the trie order differ from the column order, so
    rows go through the sort: the one-CTA path for small results and the packed-key
    LSD path (with the already-ordered tail columns skipped) for large ones."""
    d = lubm.generate(U)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    eng.load(s, p, o, d.n_entities, d.n_predicates)
    ix = OracleIndex(s, p, o)
    sizes = []
    for q in lubm.queries(d):
        for perm in (list(range(q.n_vertices))[::-1], list(range(1, q.n_vertices)) + [0]):
            qp = _relabel(q, perm)
            exp = ix.query(qp)
            got = eng.query(qp)
            assert got.shape == exp.shape and np.array_equal(got, exp), (qp.name, perm)
            sizes.append(len(exp))
    assert max(sizes) > 4096 and any(0 < n <= 4096 for n in sizes)  # both sort paths ran


@pytest.mark.parametrize("U", [1, 10, 100])
def test_lubm_queries_vs_oracle(G, eng, U):
    d = lubm.generate(U)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    eng.load(s, p, o, d.n_entities, d.n_predicates)
    ix = OracleIndex(s, p, o)
    for q in lubm.queries(d):
        exp = ix.query(q)
        got = eng.query(q)
        assert got.shape == exp.shape and np.array_equal(got, exp), q.name
    # generator-analytic count (L2 = number of courses) and tree-DP closed form
    L2 = [q for q in lubm.queries(d) if q.name == "L2"][0]
    assert eng.query(L2, flags=G.GSMART_COUNT_ONLY) == d.n_courses


@pytest.mark.parametrize("scale", [0.01, 0.04])
def test_watdiv_queries_vs_oracle(G, eng, scale):
    """configs[2] shape (WatDiv-style L/S/F/C templates, 85 predicates) at
    parity-test scale; batch execution."""
    from synth import watdiv
    d = watdiv.generate(scale)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    eng.load(s, p, o, d.n_entities, d.n_predicates)
    ix = OracleIndex(s, p, o)
    qs = watdiv.queries(d)
    exp = [ix.query(q) for q in qs]
    for q, e, got in zip(qs, exp, eng.query_batch(qs)):
        assert got.shape == e.shape and np.array_equal(got, e), q.name


@pytest.mark.parametrize("n_pred", [200, 1000])
def test_powerlaw_queries_vs_oracle(G, eng, n_pred):
    """configs[4] shape (Zipf predicates, hub objects > HEAVY_ROW entries,
    random-walk stars/chains/triangles); n_pred > 255 exercises uint16 labels."""
    from synth import powerlaw
    d = powerlaw.generate(400_000, 20_000, n_pred)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    eng.load(s, p, o, d.n_entities, d.n_predicates)
    assert G.gsmart_lspm_get(eng.ctx, G.GSMART_CSR)["pred_bytes"] == (1 if n_pred <= 255 else 2)
    ix = OracleIndex(s, p, o)
    for q in powerlaw.queries(d, 15, seed=n_pred):
        e = ix.query(q)
        got = eng.query(q)
        assert got.shape == e.shape and np.array_equal(got, e), q


@pytest.mark.parametrize("U", [1000, 10000])
def test_lubm_full_size_sampled_parity(G, U):
    """BASELINE configs[3] at full size (LUBM-10k, ~1.3e9 triples, one B200) and
    LUBM-1000, in bench.py's launch configuration (device-resident input,
    gsmart_execute_batch): exact counts pinned by the generator's counters
    (L2, L3, L4, L5, L6, Q14), and for every query the rows of sampled root
    bindings equal the oracle's solutions for those bindings (computed on the
    local triple subset around them)."""
    import torch
    from oracle import reference as R
    d = lubm.generate(U, seed=lubm.SEED_LUBM10K, device="cuda")
    qs = lubm.queries(d)
    e = G.Engine(0)
    try:
        G.gsmart_load_triples(e.ctx, d.s, d.p, d.o, d.n_entities, d.n_predicates)
        G.gsmart_build_lspm(e.ctx)
        counts = e.query_batch(qs, flags=G.GSMART_COUNT_ONLY)
        for q, c in zip(qs, counts):
            if q.name in d.counts:
                assert c == d.counts[q.name], (q.name, c, d.counts[q.name])
        s, p, o = d.s.cpu().numpy(), d.p.cpu().numpy(), d.o.cpu().numpy()
        del d
        torch.cuda.empty_cache()
        rng = np.random.default_rng(U)
        for q, c in zip(qs, counts):
            if c > 50_000_000:
                continue
            rows = e.query(q)
            assert len(rows) == c
            var = q.variables[0]
            picked = rows[rng.integers(0, len(rows), 20), 0] if len(rows) else np.zeros(0, np.uint32)
            vals = np.unique(np.concatenate([picked, rng.integers(0, len(s), 5).astype(np.uint32) % 1000003]))
            exp = R.solutions_for_bindings(s, p, o, q, var, vals)
            got = rows[np.isin(rows[:, 0], vals)]
            assert got.shape == exp.shape and np.array_equal(got, exp), q.name
    finally:
        e.close()


def _row_hash(rows):
    """Order-independent 128-bit digest of a row set: the sum and
    the xor of splitmix64 over each row's packed columns."""
    M = (1 << 64) - 1
    s = x = 0
    for r in np.asarray(rows, dtype=np.uint64).tolist():
        h = 0
        for v in r:
            z = (h ^ v) + 0x9E3779B97F4A7C15 & M
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9 & M
            z = (z ^ (z >> 27)) * 0x94D049BB133111EB & M
            h = z ^ (z >> 31)
        s = (s + h) & M
        x ^= h
    return s, x


def test_lubm1000_l1_l7_full_oracle(G):
    """LUBM-1000 (~1.3e8 triples): the data-intensive triangles L1 and L7 against
    the C oracle's complete answer — every row, plus the order-independent
    128-bit digest — in bench.py's launch configuration (device input, batch)."""
    import torch
    d = lubm.generate(1000, seed=lubm.SEED_LUBM10K, device="cuda")
    qs = [q for q in lubm.queries(d) if q.name in ("L1", "L7")]
    e = G.Engine(0)
    try:
        G.gsmart_load_triples(e.ctx, d.s, d.p, d.o, d.n_entities, d.n_predicates)
        G.gsmart_build_lspm(e.ctx)
        got = e.query_batch(qs)
        s, p, o = d.s.cpu().numpy(), d.p.cpu().numpy(), d.o.cpu().numpy()
        del d
        torch.cuda.empty_cache()
        ix = OracleIndex(s, p, o)
        for q, g in zip(qs, got):
            exp = ix.query(q)
            assert len(exp) > 1000, q.name
            assert g.shape == exp.shape and np.array_equal(g, exp), q.name
            assert _row_hash(g) == _row_hash(exp)
    finally:
        e.close()


def test_watdiv100m_full_size_parity(G):
    """configs[2] at full size (scale 2.1, ~1.08e8 triples) in bench.py's launch
    configuration (device-resident generated input, the 11 queries as one
    gsmart_execute_batch): every row of every query == the C oracle."""
    import torch
    from synth import watdiv
    d = watdiv.generate(watdiv.SCALE_100M, device="cuda")
    qs = watdiv.queries(d)
    e = G.Engine(0)
    try:
        G.gsmart_load_triples(e.ctx, d.s, d.p, d.o, d.n_entities, d.n_predicates)
        G.gsmart_build_lspm(e.ctx)
        got = e.query_batch(qs)
        fact = e.query_batch(qs, flags=G.GSMART_FACTORISED)  # f2: rows read off the factorised trees
        s, p, o = d.s.cpu().numpy(), d.p.cpu().numpy(), d.o.cpu().numpy()
        del d
        torch.cuda.empty_cache()
        ix = OracleIndex(s, p, o)
        for q, g, gf in zip(qs, got, fact):
            exp = ix.query(q)
            assert g.shape == exp.shape and np.array_equal(g, exp), q.name
            assert gf.shape == exp.shape and np.array_equal(gf, exp), q.name
    finally:
        e.close()


def test_graph_replay_matches(G, eng):
    """Plans executed repeatedly replay their captured phase-1 CUDA graph (fresh
    look-back epochs each time); interleaved plans, batches and NO_GRAPH give
    identical rows, equal to the oracle."""
    d = lubm.generate(5)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    eng.load(s, p, o, d.n_entities, d.n_predicates)
    ix = OracleIndex(s, p, o)
    qs = lubm.queries(d)
    exp = [ix.query(q) for q in qs]
    plans = [G.gsmart_plan(eng.ctx, q) for q in qs]
    try:
        for rep in range(3):
            for flags in (0, G.GSMART_NO_GRAPH):
                for q, pl, e in zip(qs, plans, exp):
                    r = G.gsmart_execute(eng.ctx, pl, flags)
                    got = G.gsmart_result_rows(r)
                    G.gsmart_result_free(r)
                    assert np.array_equal(got, e), (q.name, rep, flags)
            for q, r, e in zip(qs, G.gsmart_execute_batch(eng.ctx, plans, 0), exp):
                assert np.array_equal(G.gsmart_result_rows(r), e), (q.name, rep, "batch")
                G.gsmart_result_free(r)
    finally:
        for pl in plans:
            G.gsmart_plan_free(pl)


def test_execute_batch_matches_single(G, eng):
    """gsmart_execute_batch (concurrent slots, > 16 plans => several waves) gives
    exactly the per-query results of the oracle."""
    d = lubm.generate(4)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    eng.load(s, p, o, d.n_entities, d.n_predicates)
    ix = OracleIndex(s, p, o)
    qs = lubm.queries(d) * 3
    for q, got in zip(qs, eng.query_batch(qs)):
        assert np.array_equal(got, ix.query(q)), q.name
    counts = eng.query_batch(qs[:8], flags=G.GSMART_COUNT_ONLY)
    assert counts == [len(ix.query(q)) for q in qs[:8]]


def test_lubm_device_input_and_keep_set(G, eng):
    import torch
    d = lubm.generate(3)
    qs = lubm.queries(d)
    keep = sorted({e[1] for q in qs for e in q.edges})
    eng.load(d.s.cuda(), d.p.cuda(), d.o.cuda(), d.n_entities, d.n_predicates, keep=keep)
    ix = OracleIndex(d.s.numpy(), d.p.numpy(), d.o.numpy())
    for q in qs:
        assert np.array_equal(eng.query(q), ix.query(q)), q.name
    torch.cuda.synchronize()


# ------------------------------------------------------------------ edge cases
def test_edge_cases(G, eng):
    s, p, o = fixtures.fig1_triples()
    eng.load(s, p, o, 8, 4)
    # constant outside [0, N): empty, not an error
    assert eng.query(Query((None, 99), ((0, 1, 1),))).shape == (0, 1)
    # no variables: guard true / false
    assert eng.query(Query((0, 1), ((0, 1, 1),))).shape == (1, 0)
    assert eng.query(Query((0, 1), ((0, 2, 1),))).shape == (0, 0)
    # self-loop with no data: empty
    assert eng.query(Query((None,), ((0, 1, 0),))).shape == (0, 1)
    # disconnected variables (cross product)
    q = Query((None, None, 2, 7), ((2, 2, 0), (3, 3, 1)))
    assert _rows(eng.query(q)) == R.brute_force(s, p, o, 8, q)
    # COUNT_ONLY / KEEP_ON_DEVICE
    q = fixtures.fig2_query()
    assert eng.query(q, flags=G.GSMART_COUNT_ONLY) == 2
    with eng.plan(q) as pl:
        r = G.gsmart_execute(eng.ctx, pl.h, G.GSMART_KEEP_ON_DEVICE)
        ptr = G.gsmart_result_rows_device(r)
        host = G.gsmart_copy_to_host(eng.ctx, ptr, 2 * 4 * 4).reshape(2, 4)
        assert _rows(host) == [(2, 0, 1, 0), (2, 0, 1, 5)]
        assert _rows(G.gsmart_result_rows(r)) == [(2, 0, 1, 0), (2, 0, 1, 5)]
        G.gsmart_result_free(r)


def test_absent_constants_candidates(G, eng):
    """A constant absent from the data (id >= N, up to 2^32 - 1) has no
    entries: as a seed it empties only its own variable's candidate set (the
    schedule then propagates), as a guard it is false (R12, R13).  Rows and
    every candidate bitmap equal filter_schedule."""
    s, p, o = fixtures.fig1_triples()
    eng.load(s, p, o, 8, 4)
    for q in (Query((None, None, 99), ((0, 1, 1), (1, 1, 2))),
              Query((None, None, 0xFFFFFFF0, 0x80000005), ((0, 1, 1), (2, 1, 1), (3, 2, 1))),
              Query((None, None, 8), ((0, 2, 1), (1, 1, 2), (1, 1, 0))),
              Query((None, None, 8, 3), ((0, 3, 1), (2, 1, 3))),
              Query((None, None, 1, 3), ((0, 3, 1), (2, 1, 3)))):
        rows, cs, _ = _cands(G, eng, q, G.GSMART_REFINE)
        assert _rows(rows) == R.brute_force(s, p, o, 8, q), q
        ref, _ = R.filter_schedule(s, p, o, 8, q, refine=True)
        for v in q.variables:
            assert _bits_to_set(cs[v], 8) == set(np.nonzero(ref[v])[0].tolist()), (q, v)


def test_label_signature_collisions(G, eng):
    """Row label signatures fold labels mod 32 (P > 32): labels 1, 33 and 65 share
    a bit, so rows holding only label 1 pass the pre-test for a label-33 edge and
    must still be rejected by the scan.  Rows vs brute force and the oracle."""
    rng = np.random.default_rng(5)
    n, P = 40, 70
    s = rng.integers(0, n, 600).astype(np.uint32)
    o = rng.integers(0, n, 600).astype(np.uint32)
    p = rng.choice(np.array([1, 33, 65, 2, 34], dtype=np.uint32), 600, p=[0.5, 0.05, 0.05, 0.3, 0.1])
    eng.load(s, p, o, n, P)
    for q in (Query((None, None), ((0, 33, 1),)),
              Query((None, None, None), ((0, 33, 1), (0, 2, 2))),
              Query((None, None, None), ((0, 65, 1), (2, 34, 0), (1, 1, 2))),
              Query((None, None), ((0, 33, 1), (1, 65, 0)))):
        got = _rows(eng.query(q))
        assert got == R.brute_force(s, p, o, n, q), q
        assert got == _rows(oracle_bgp(s, p, o, q)), q


def test_result_overflow_and_empty_load(G):
    e = G.Engine(0, max_result_rows=1)
    s, p, o = fixtures.fig1_triples()
    e.load(s, p, o, 8, 4)
    with pytest.raises(G.GsmartError) as ei:
        e.query(fixtures.fig2_query())
    assert ei.value.name == "E_RESULT_OVERFLOW"
    e.close()
    e = G.Engine(0)
    e.load([], [], [], 10, 3)
    assert e.query(Query((None, None), ((0, 1, 1),))).shape == (0, 2)
    e.close()


def test_call_order_and_bad_ids(G):
    e = G.Engine.__new__(G.Engine)
    e.ctx = G.gsmart_create(0)
    with pytest.raises(G.GsmartError) as ei:
        G.gsmart_build_lspm(e.ctx)
    assert ei.value.name == "E_STATE"
    with pytest.raises(G.GsmartError) as ei:
        G.gsmart_load_triples(e.ctx, [0], [5], [1], 4, 3)   # predicate > n_predicates
    assert ei.value.name == "E_INVALID_ARG"
    e.close()


def test_pruned_trie_invariants(G, eng):
    """a8: after bottom-up pruning every internal node has >= 1 child, parent[]
    is non-decreasing, and the last level holds exactly the rows."""
    d = lubm.generate(2)
    eng.load(d.s.numpy(), d.p.numpy(), d.o.numpy(), d.n_entities, d.n_predicates)
    for q in lubm.queries(d):
        with eng.plan(q) as pl:
            r = G.gsmart_execute(eng.ctx, pl.h, 0)
            n_rows = G.gsmart_result_shape(r)[0]
            st = G.gsmart_result_stats(r)
            L = st["n_levels"]
            prev_n = None
            for k in range(L):
                v, n, par, bnd = G.gsmart_result_level(r, k)
                assert n == st["level_alive"][k]
                if k > 0 and n:
                    parent = G.gsmart_copy_to_host(eng.ctx, par, n * 4)
                    assert np.all(np.diff(parent.astype(np.int64)) >= 0)
                    assert set(parent.tolist()) == set(range(prev_n)), q.name  # every node has a child
                prev_n = n
            assert prev_n == n_rows or L == 0
            G.gsmart_result_free(r)


# ------------------------------------------------------------------ push form of a4
@pytest.fixture(scope="module")
def eng_push(G):
    """An engine whose grouped evaluation streams the label-major lists for every
    edge (GSMART_FILTER_VARIANT bit 8: push form forced, no size threshold)."""
    import os
    old = os.environ.get("GSMART_FILTER_VARIANT")
    os.environ["GSMART_FILTER_VARIANT"] = "14"
    try:
        e = G.Engine(0)
    finally:
        if old is None:
            del os.environ["GSMART_FILTER_VARIANT"]
        else:
            os.environ["GSMART_FILTER_VARIANT"] = old
    yield e
    e.close()


def test_push_form_tiny_rows_and_candidates(G, eng_push):
    """Push (label-major streaming) and pull evaluate the same Eq. 17/21
    conjunction: rows == brute force and every candidate bitmap ==
    filter_schedule, refine on and off (skips included)."""
    for seed in range(400):
        (s, p, o), n, P, q = tiny.random_case(seed)
        eng_push.load(s, p, o, n, P)
        exp = R.brute_force(s, p, o, n, q)
        for flags, refine, back in ((G.GSMART_REFINE, True, False), (0, False, False),
                                    (G.GSMART_REFINE | G.GSMART_BACK_EDGES, True, True)):
            rows, cs, _ = _cands(G, eng_push, q, flags)
            assert _rows(rows) == exp, (seed, q)
            ref, _ = R.filter_schedule(s, p, o, n, q, refine=refine, back_edges=back)
            for v in q.variables:
                assert _bits_to_set(cs[v], n) == set(np.nonzero(ref[v])[0].tolist()), (seed, v, q)


@pytest.mark.parametrize("src", ["lubm10", "watdiv", "skewed", "powerlaw"])
def test_push_form_vs_oracle(G, eng_push, src):
    if src == "lubm10":
        d = lubm.generate(10)
        s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
        qs, N, P = lubm.queries(d), d.n_entities, d.n_predicates
    elif src == "watdiv":
        from synth import watdiv
        d = watdiv.generate(0.01)
        s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
        qs, N, P = watdiv.queries(d), d.n_entities, d.n_predicates
    elif src == "powerlaw":
        from synth import powerlaw
        d = powerlaw.generate(400_000, 20_000, 200)
        s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
        qs, N, P = powerlaw.queries(d, 10, seed=3), d.n_entities, d.n_predicates
    else:
        s, p, o = tiny.random_graph(11, 2000, 3, 150000, skew=1.3)
        N, P = 2000, 3
        qs = _data_queries(np.random.default_rng(11), s, p, o, 12)
    eng_push.load(s, p, o, N, P)
    ix = OracleIndex(s, p, o)
    for q, got in zip(qs, eng_push.query_batch(qs)):
        e = ix.query(q)
        assert got.shape == e.shape and np.array_equal(got, e), q


# ------------------------------------------------------------------ speculative phase 2
def _run_plans(G, ctx, plans, batch):
    """rows + stats of each plan, through one batch or one execute per plan"""
    res = G.gsmart_execute_batch(ctx, plans, 0) if batch else [G.gsmart_execute(ctx, pl, 0) for pl in plans]
    out = []
    for r in res:
        out.append((G.gsmart_result_rows(r), G.gsmart_result_stats(r)))
        G.gsmart_result_free(r)
    return out


def test_speculative_phase2_repeats(G, eng):
    """Re-executions of the SAME plan handles queue phase 2 sized from the
    previous run (one host wait): the first run never speculates, every later
    run does (stats.spec_phase2), guesses right (no redo) and gives the oracle's
    rows — single executes and batches alike."""
    d = lubm.generate(3)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    eng.load(s, p, o, d.n_entities, d.n_predicates)
    ix = OracleIndex(s, p, o)
    qs = lubm.queries(d)
    exp = [ix.query(q) for q in qs]
    plans = [G.gsmart_plan(eng.ctx, q) for q in qs]
    try:
        for rep in range(4):
            for q, e, (got, st) in zip(qs, exp, _run_plans(G, eng.ctx, plans, batch=rep % 2 == 1)):
                assert got.shape == e.shape and np.array_equal(got, e), (q.name, rep)
                assert st["spec_phase2"] == (1 if rep > 0 else 0), (q.name, rep, st["spec_phase2"])
                assert st["spec_redo"] == 0, q.name
    finally:
        for pl in plans:
            G.gsmart_plan_free(pl)


def test_speculative_phase2_wrong_guess(G):
    """GSMART_SPEC_TEST makes every speculation guess a wrong row count,
    alternately one fewer (the device guard k_phase2_guard voids phase 2) and
    one more (the host size check rejects it).  Plans are re-executed on the
    same handles, so speculation really happens; the redo must give the
    oracle's rows and the stats must record the speculation and the redo."""
    import os
    os.environ["GSMART_SPEC_TEST"] = "1"
    try:
        e = G.Engine(0)
    finally:
        del os.environ["GSMART_SPEC_TEST"]
    try:
        d = lubm.generate(2)
        s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
        e.load(s, p, o, d.n_entities, d.n_predicates)
        ix = OracleIndex(s, p, o)
        qs = lubm.queries(d)
        exp = [ix.query(q) for q in qs]
        plans = [G.gsmart_plan(e.ctx, q) for q in qs]
        redos = 0
        try:
            for rep in range(4):
                for q, x, (got, st) in zip(qs, exp, _run_plans(G, e.ctx, plans, batch=rep % 2 == 0)):
                    assert got.shape == x.shape and np.array_equal(got, x), (q.name, rep)
                    if rep > 0 and len(x) > 0:
                        assert st["spec_phase2"] == 1 and st["spec_redo"] == 1, (q.name, rep, st)
                        redos += 1
        finally:
            for pl in plans:
                G.gsmart_plan_free(pl)
        assert redos >= 3 * 6
    finally:
        e.close()


def test_plan_free_drops_caches(G, eng):
    """gsmart_plan_free drops the plan's cached graphs/decisions: many short-lived
    plans keep working and results stay exact (cache growth)."""
    s, p, o = fixtures.fig1_triples()
    eng.load(s, p, o, 8, 4)
    q = fixtures.fig2_query()
    for _ in range(50):
        pl = G.gsmart_plan(eng.ctx, q)
        for _ in range(2):
            r = G.gsmart_execute(eng.ctx, pl, 0)
            assert _rows(G.gsmart_result_rows(r)) == [(2, 0, 1, 0), (2, 0, 1, 5)]
            G.gsmart_result_free(r)
        G.gsmart_plan_free(pl)
