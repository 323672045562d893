"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports
every symbol include/gsmart.h declares, plans queries (host-only planner),
and fails loudly (GSMART_E_CUDA) instead of falling back when no device."""
import ctypes
import os
import re

import pytest

from oracle import reference as R
from synth import fixtures, tiny, lubm
from synth.query import Query

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def G():
    from conftest import build_product
    build_product()
    import paper_2106_14038_b200.gsmart as g
    return g


def _declared_functions():
    txt = open(os.path.join(ROOT, "include", "gsmart.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gsmart_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported(G):
    lib = ctypes.CDLL(G.LIB_PATH)
    decl = _declared_functions()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(G.EXPORTED)


def test_abi_version_and_build_info(G):
    assert G.gsmart_abi_version() == 3
    assert "sm_100a" in G.gsmart_build_info()


def test_no_gpu_fails_loudly(G):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(G.GsmartError) as ei:
        G.gsmart_create(0)
    assert ei.value.name == "E_CUDA"


def _pydesc(q, direction=False):
    """oracle planner -> the describe() JSON shape, for comparison."""
    pl = R.plan_direction(q) if direction else R.plan_degree(q)
    D = {0: "out", 1: "in"}
    return {
        "roots": pl["roots"],
        "seeds": pl["seeds"],
        "groups": [{"center": c, "edges": [(k, D[d], w) for k, d, w in g], "back": [(k, D[d], w) for k, d, w in b]}
                   for (c, g), b in zip(pl["groups"], pl["back"])],
        "level": pl["level"],
        "pi": pl["pi"],
        "tree": {v: (k, p, D[d]) for v, (k, p, d) in pl["tree"].items()},
        "closing": {v: sorted((k, o, D[d]) for k, o, d in cl) for v, cl in pl["closing"].items()},
        "paths": [sorted(map(tuple, pl["paths"][r])) for r in pl["roots"]] if not direction else None,
    }


def _cdesc(G, q, direction=False):
    h = G.gsmart_plan(None, q, traversal=G.GSMART_DIRECTION if direction else G.GSMART_DEGREE)
    try:
        d = G.gsmart_plan_describe(h)
    finally:
        G.gsmart_plan_free(h)
    pi = d["pi"]
    tree, closing = {}, {}
    for L in d["levels"]:
        v = L["var"]
        if L["tree_edge"] >= 0:
            tree[v] = (L["tree_edge"], pi[L["parent_level"]], L["dir"])
        closing[v] = sorted((c["edge"], pi[c["other_level"]], c["dir"]) for c in L["closing"])
    return {
        "roots": d["roots"],
        "seeds": [s["edge"] for s in d["seeds"]] + [],
        "groups": [{"center": g["center"], "edges": [(e["edge"], e["dir"], e["nbr"]) for e in g["edges"]],
                    "back": [(e["edge"], e["dir"], e["nbr"]) for e in g["back"]]} for g in d["groups"]],
        "level": [g["level"] for g in d["groups"]],
        "pi": pi,
        "tree": tree,
        "closing": closing,
        "paths": [sorted(map(tuple, p)) for p in d["paths"]],
    }, d


def test_plan_fig2_matches_paper(G, golden_fig):
    c, d = _cdesc(G, fixtures.fig2_query())
    assert c["roots"] == [golden_fig["root"]]                     # Ex. 6.2
    assert len(c["groups"]) == 2
    assert max(c["level"]) + 1 == golden_fig["edge_levels_L0"]    # Ex. 6.5
    assert sorted(c["paths"][0]) == sorted(tuple(p) for p in golden_fig["paths"])  # Ex. 7.1


def test_plan_parity_with_oracle_planner(G):
    """The product's C++ planner and the oracle's independent Python planner
    agree on every field for random queries (cycles, constants, self-loops,
    multi-edges, disconnected parts) and the LUBM templates."""
    qs = [tiny.random_case(s)[3] for s in range(400)]
    qs += lubm.queries(lubm.generate(1))
    qs.append(fixtures.fig2_query())
    for q in qs:
        c, _ = _cdesc(G, q)
        p = _pydesc(q)
        guards = [k for k, (a, _, b) in enumerate(q.edges) if q.is_const(a) and q.is_const(b)]
        assert sorted(c["seeds"] + guards) == p["seeds"], q
        for key in ("roots", "groups", "level", "pi", "tree", "closing", "paths"):
            assert c[key] == p[key], (key, q, c[key], p[key])


def test_direction_plan_parity_with_oracle_planner(G, golden_fig):
    """GSMART_DIRECTION (§6.1.1): the C++ planner == the oracle's plan_direction
    on every field for random variable-only queries (cycles, self-loops,
    multi-edges, disconnected parts) and Fig. 2 (Ex. 6.1: roots v0, v3)."""
    qs = [tiny.random_case(s, n_consts=0)[3] for s in range(400)] + [fixtures.fig2_query()]
    for q in qs:
        c, d = _cdesc(G, q, direction=True)
        p = _pydesc(q, direction=True)
        assert d["traversal"] == "direction"
        for key in ("roots", "groups", "level", "pi", "tree", "closing"):
            assert c[key] == p[key], (key, q, c[key], p[key])
    c, _ = _cdesc(G, fixtures.fig2_query(), direction=True)
    assert c["roots"] == golden_fig["ex61_roots"]


def test_keep_sets_ex64_and_oracle(G, golden_fig):
    """Query-dependent LSpM (§6.2, f3): the labels each format must keep for a
    plan == the oracle's keep_sets; for Fig. 2 they are Ex. 6.4's
    direction-split keep-sets (CSR {follows, actor}, CSC {director, follows})."""
    P = fixtures.PREDICATE_IDS
    h = G.gsmart_plan(None, fixtures.fig2_query())
    try:
        csr, csc = G.gsmart_plan_keep_sets([h])
    finally:
        G.gsmart_plan_free(h)
    assert csr == sorted(P[x] for x in golden_fig["ex64_csr"]["keep"])
    assert csc == sorted(P[x] for x in golden_fig["ex64_csc"]["keep"])
    for seed in range(300):
        q = tiny.random_case(seed)[3]
        for back in (False, True):
            h = G.gsmart_plan(None, q)
            try:
                got = G.gsmart_plan_keep_sets([h], G.GSMART_BACK_EDGES if back else 0)
            finally:
                G.gsmart_plan_free(h)
            assert tuple(got) == R.keep_sets(q, back_edges=back), (seed, q, back)


def test_plan_errors(G):
    with pytest.raises(G.GsmartError) as e:
        G.gsmart_plan(None, Query((None,), ((0, 1, 1),)))       # vertex out of range
    assert e.value.name == "E_INVALID_ARG"
    with pytest.raises(G.GsmartError) as e:
        G.gsmart_plan(None, Query((None, None), ((0, 0, 0),)))  # pred 0, var 1 unused
    assert e.value.name == "E_INVALID_ARG"
    with pytest.raises(G.GsmartError) as e:  # direction-driven + constants: planned degree-driven
        G.gsmart_plan(None, Query((None, 3), ((0, 1, 1),)), traversal=G.GSMART_DIRECTION)
    assert e.value.name == "E_UNSUPPORTED"
