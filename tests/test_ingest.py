"""f4: N-Triples read + dictionary encode (§6.2.1
steps 1-2).  CPU part: the oracle (`oracle/ntriples.py`) pinned
against the Fig. 1a example, hand-written term lists and error lines, and
closed forms; the C-ABI exports.  GPU part: `gsmart_ingest_ntriples` against
the oracle, byte for byte (ids, term bytes, the first bad line)."""
import json
import os

import numpy as np
import pytest

from oracle import ntriples as NT
from synth import fixtures
from synth import ntriples as SN

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _fig1_doc():
    with open(os.path.join(GOLDEN, "fig1.nt"), "rb") as f:
        return f.read()


def _short(t):
    return t.decode()[len("<http://example.org/"):-1]


# ---------------------------------------------------------------- oracle pins
def test_fig1_first_appearance(golden_fig):
    trip = NT.parse(_fig1_doc())
    assert len(trip) == 12
    s, p, o, ents, preds = NT.encode(trip)
    g = golden_fig["ntriples_first_appearance"]
    assert {_short(t): i for i, t in enumerate(ents)} == g["entities"]
    assert {_short(t): i + 1 for i, t in enumerate(preds)} == g["predicates"]
    # re-labelled with the paper's Ex. 6.3 map (R21) the triples are Fig. 1a's
    em, pm = golden_fig["entity_ids"], golden_fig["predicate_ids"]
    got = sorted((em[_short(ents[a])], pm[_short(preds[b - 1])], em[_short(ents[c])]) for a, b, c in zip(s, p, o))
    fs, fp, fo = fixtures.fig1_triples()
    assert got == sorted(zip(map(int, fs), map(int, fp), map(int, fo)))


HAND_DOC = (b"# header comment\n"
            b"\n"
            b"  <http://a/x>\t<http://a/p> \"say \\\"hi\\\" . <x>\"@en-GB .\r\n"
            b"_:b1 <http://a/p><http://a/y> .\n"
            b"<http://a/x><http://a/q>\"1\"^^<http://www.w3.org/2001/XMLSchema#int>\t.  \n"
            b" \t\r\n"
            b"<http://a/y> <http://a/q> _:b1 .\n"
            b"<http://a/x> <http://a/p> \"a\\\\\" .")


def test_hand_doc_terms():
    assert NT.parse(HAND_DOC) == [
        (b"<http://a/x>", b"<http://a/p>", b"\"say \\\"hi\\\" . <x>\"@en-GB"),
        (b"_:b1", b"<http://a/p>", b"<http://a/y>"),
        (b"<http://a/x>", b"<http://a/q>", b"\"1\"^^<http://www.w3.org/2001/XMLSchema#int>"),
        (b"<http://a/y>", b"<http://a/q>", b"_:b1"),
        (b"<http://a/x>", b"<http://a/p>", b"\"a\\\\\""),
    ]
    s, p, o, ents, preds = NT.encode(NT.parse(HAND_DOC))
    # by hand: x 0, "say.." 1, _:b1 2, y 3, "1"^^int 4, "a\\" 5; p 1, q 2
    assert (s, p, o) == ([0, 2, 0, 3, 0], [1, 1, 2, 2, 1], [1, 3, 4, 2, 5])
    assert len(ents) == 6 and preds == [b"<http://a/p>", b"<http://a/q>"]


@pytest.mark.parametrize("line", [
    b"<a> <b> <c>",                 # no final dot
    b"<a> <b> <c> <d> .",           # four terms
    b"<a> \"p\" <c> .",             # literal predicate
    b"\"s\" <b> <c> .",             # literal subject
    b"<a> <b> \"c .",               # unterminated literal
    b"<a> <b> \"c\\\" .",           # escaped closing quote
    b"<a <b> <c> .",                # IRI "<a <b>", then "<c>", then '.' is no term
    b"<a> <b> .",                   # two terms
    b"<a> <b> \"x\"^^<dt .",        # unterminated datatype
    b"<a> <b> c .",                 # bare word
    b"<a> <b> <c> . x",             # trailing garbage
    b"<a>\r<b> <c> .",              # CR is not a separator between terms
])
def test_error_lines(line):
    doc = b"<ok> <ok> <ok> .\n# c\n" + line + b"\n<ok> <ok> <ok> .\n"
    with pytest.raises(NT.NTriplesError, match="line 2"):
        NT.parse(doc)


def test_empty_and_comment_only():
    assert NT.parse(b"") == []
    assert NT.parse(b"\n\n# x\n \t\r\n") == []
    assert NT.encode([]) == ([], [], [], [], [])


def test_render_ids_closed_form():
    """Fixed-width documents: terms carry their numeric id, so the encoder's
    ids must equal the first-appearance rank computed with np.unique."""
    rng = np.random.default_rng(5)
    n = 3000
    s = rng.integers(0, 500, n)
    o = rng.integers(0, 500, n)
    p = rng.integers(1, 9, n)
    doc = SN.render_ids(s, p, o)
    assert len(doc) == n * SN.LINE_W
    trip = NT.parse(doc)
    es, ep, eo, ents, preds = NT.encode(trip)
    inter = np.stack([s, o], 1).reshape(-1)
    u, first = np.unique(inter, return_index=True)
    rank = np.empty(u.max() + 1, np.int64)
    rank[u[np.argsort(first)]] = np.arange(u.size)
    np.testing.assert_array_equal(es, rank[s])
    np.testing.assert_array_equal(eo, rank[o])
    pu, pf = np.unique(p, return_index=True)
    prank = np.empty(pu.max() + 1, np.int64)
    prank[pu[np.argsort(pf)]] = np.arange(1, pu.size + 1)
    np.testing.assert_array_equal(ep, prank[p])
    assert [int(t[-10:-1]) for t in ents] == list(u[np.argsort(first)])


@pytest.mark.parametrize("seed", range(8))
def test_tricky_roundtrip(seed):
    doc = SN.tricky_doc(seed, 80)
    trip = NT.parse(doc)
    s, p, o, ents, preds = NT.encode(trip)
    for (a, b, c), i, j, k in zip(trip, s, p, o):
        assert (ents[i], preds[j - 1], ents[k]) == (a, b, c)
    # ids in first-appearance order: the running maximum grows by one
    seen = -1
    for v in np.stack([s, o], 1).reshape(-1):
        assert v <= seen + 1
        seen = max(seen, v)
    assert seen + 1 == len(ents) == len(set(ents))
    # canonical re-rendering parses to the same triples
    canon = b"".join(a + b" " + b + b" " + c + b" .\n" for a, b, c in trip)
    assert NT.parse(canon) == trip


@pytest.mark.parametrize("seed", range(6))
def test_corrupt_line_number(seed):
    doc, ln = SN.corrupt(SN.tricky_doc(100 + seed, 40), seed)
    with pytest.raises(NT.NTriplesError, match=f"line {ln}:"):
        NT.parse(doc)


# ---------------------------------------------------------------- GPU parity
def _ingest(G, doc, device):
    import torch
    eng = G.Engine(0)
    if device:
        buf = torch.frombuffer(bytearray(doc), dtype=torch.uint8).cuda() if doc else torch.empty(0, dtype=torch.uint8,
                                                                                                   device="cuda")
    else:
        buf = doc
    n, N, P = G.gsmart_ingest_ntriples(eng.ctx, buf)
    return eng, n, N, P


def _check(G, eng, doc, n, N, P):
    trip = NT.parse(doc)
    s, p, o, ents, preds = NT.encode(trip)
    assert (n, N, P) == (len(trip), len(ents), len(preds))
    if n == 0:
        return
    gs, gp, go = G.gsmart_triples_get(eng.ctx)
    np.testing.assert_array_equal(gs, s)
    np.testing.assert_array_equal(gp, p)
    np.testing.assert_array_equal(go, o)
    for i in range(N):
        assert G.gsmart_dict_term(eng.ctx, G.GSMART_DICT_ENTITY, i) == ents[i]
        assert G.gsmart_dict_lookup(eng.ctx, G.GSMART_DICT_ENTITY, ents[i]) == i
    for i in range(P):
        assert G.gsmart_dict_term(eng.ctx, G.GSMART_DICT_PREDICATE, i + 1) == preds[i]
        assert G.gsmart_dict_lookup(eng.ctx, G.GSMART_DICT_PREDICATE, preds[i]) == i + 1
    assert G.gsmart_dict_lookup(eng.ctx, G.GSMART_DICT_ENTITY, b"<http://absent/>") == 0xFFFFFFFF
    assert G.gsmart_dict_lookup(eng.ctx, G.GSMART_DICT_PREDICATE, ents[0] + b"x") == 0xFFFFFFFF


@pytest.mark.gpu
@pytest.mark.parametrize("device", [False, True])
def test_gpu_ingest_fig1(device, golden_fig):
    """Fig. 1a as text -> ids -> the Fig. 2 query: the answer, mapped through
    the dictionary to the paper's names, is the golden solution (Ex. 7.2)."""
    import paper_2106_14038_b200 as G
    from synth.query import Query
    doc = _fig1_doc()
    eng, n, N, P = _ingest(G, doc, device)
    try:
        _check(G, eng, doc, n, N, P)
        G.gsmart_build_lspm(eng.ctx)
        em, pm = golden_fig["entity_ids"], golden_fig["predicate_ids"]
        pname = {v: k for k, v in pm.items()}
        q = fixtures.fig2_query()
        pid = {l: G.gsmart_dict_lookup(eng.ctx, G.GSMART_DICT_PREDICATE,
                                       f"<http://example.org/{pname[l]}>".encode()) for _, l, _ in q.edges}
        q2 = Query(q.vertices, [(a, pid[l], b) for a, l, b in q.edges], "fig2")
        rows = eng.query(q2)
        back = sorted(tuple(em[_short(G.gsmart_dict_term(eng.ctx, G.GSMART_DICT_ENTITY, int(x)))] for x in r)
                      for r in rows)
        assert back == [tuple(r) for r in golden_fig["solution_rows"]]
    finally:
        eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_gpu_ingest_tricky(seed):
    import paper_2106_14038_b200 as G
    doc = SN.tricky_doc(seed, 40 + 37 * seed)
    eng, n, N, P = _ingest(G, doc, seed % 2 == 1)
    try:
        _check(G, eng, doc, n, N, P)
    finally:
        eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_gpu_ingest_error_line(seed):
    import paper_2106_14038_b200 as G
    doc, ln = SN.corrupt(SN.tricky_doc(100 + seed, 40), seed)
    eng = G.Engine(0)
    try:
        with pytest.raises(G.GsmartError, match=f"line {ln}:"):
            G.gsmart_ingest_ntriples(eng.ctx, doc)
    finally:
        eng.close()


@pytest.mark.gpu
def test_gpu_ingest_empty_and_comments():
    import paper_2106_14038_b200 as G
    for doc in (b"", b"\n\n# only a comment\n \t\r\n"):
        eng, n, N, P = _ingest(G, doc, False)
        try:
            assert (n, N, P) == (0, 0, 0)
        finally:
            eng.close()


@pytest.mark.gpu
def test_gpu_ingest_large_render():
    """Several chunks of the newline scan and many radix tiles: 400k
    fixed-width lines plus a tricky tail (ragged last chunk, no final
    newline), ids against the oracle."""
    import paper_2106_14038_b200 as G
    rng = np.random.default_rng(11)
    n = 400_000
    s = rng.zipf(1.6, n) % 90_000
    o = rng.integers(0, 120_000, n)
    p = rng.integers(1, 300, n)
    doc = SN.render_ids(s, p, o) + SN.tricky_doc(3, 50)
    eng, gn, N, P = _ingest(G, doc, True)
    try:
        trip = NT.parse(doc)
        es, ep, eo, ents, preds = NT.encode(trip)
        assert (gn, N, P) == (len(trip), len(ents), len(preds))
        gs, gp, go = G.gsmart_triples_get(eng.ctx)
        np.testing.assert_array_equal(gs, es)
        np.testing.assert_array_equal(gp, ep)
        np.testing.assert_array_equal(go, eo)
        for i in rng.integers(0, N, 200):
            assert G.gsmart_dict_term(eng.ctx, G.GSMART_DICT_ENTITY, int(i)) == ents[i]
    finally:
        eng.close()


@pytest.mark.gpu
def test_gpu_ingest_then_query_matches_oracle():
    """End to end: text -> ingest -> build -> query with constants looked up
    in the dictionary; rows equal the C oracle's over the oracle's encoding."""
    import paper_2106_14038_b200 as G
    from oracle.coracle import oracle_bgp
    from synth.query import Query, var, const
    rng = np.random.default_rng(2)
    n = 20_000
    s = rng.integers(0, 3000, n)
    o = rng.integers(0, 3000, n)
    p = rng.integers(1, 6, n)
    doc = SN.render_ids(s, p, o)
    trip = NT.parse(doc)
    es, ep, eo, ents, preds = NT.encode(trip)
    eng, gn, N, P = _ingest(G, doc, False)
    try:
        G.gsmart_build_lspm(eng.ctx)
        c = G.gsmart_dict_lookup(eng.ctx, G.GSMART_DICT_ENTITY, ents[7])
        p1 = G.gsmart_dict_lookup(eng.ctx, G.GSMART_DICT_PREDICATE, preds[0])
        p2 = G.gsmart_dict_lookup(eng.ctx, G.GSMART_DICT_PREDICATE, preds[1])
        assert (c, p1, p2) == (7, 1, 2)
        q = Query([var(), var(), var(), const(7)], [(0, 1, 1), (1, 2, 2), (0, 1, 3)], "e2e")
        got = eng.query(q)
        want = oracle_bgp(np.asarray(es, np.uint32), np.asarray(ep, np.uint32), np.asarray(eo, np.uint32), q)
        np.testing.assert_array_equal(got, want)
    finally:
        eng.close()


# ---------------------------------------------------------------- ABI (CPU)
def test_ingest_symbols_exported():
    import paper_2106_14038_b200 as G
    lib = G.lib()
    for sym in ("gsmart_ingest_ntriples", "gsmart_dict_lookup", "gsmart_dict_term", "gsmart_triples_get"):
        assert hasattr(lib, sym), sym
