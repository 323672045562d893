"""Seeded tiny random (triple set, query) pairs for brute-force pinning and
edge-case parity (SURVEY.md §8(c) "Random properties": N in [2,6], P in
[1,3], <= 14 triples, 2-4 variables, tree queries plus closing edges).

Cases cover cycles, constants (incl. constants absent from the data),
self-loops, multi-edges between a vertex pair, duplicate triples and
duplicate patterns.  Pure input generation: no method arithmetic.
"""
import numpy as np

from .query import Query


def random_triples(rng, n_entities, n_predicates, n_triples):
    s = rng.integers(0, n_entities, n_triples)
    p = rng.integers(1, n_predicates + 1, n_triples)
    o = rng.integers(0, n_entities, n_triples)
    return s.tolist(), p.tolist(), o.tolist()


def random_query(rng, n_entities, n_predicates, n_vars=None, n_consts=None,
                 extra_edges=None, connected=True, allow_self_loops=True):
    nv = int(rng.integers(1, 5)) if n_vars is None else n_vars
    nc = int(rng.integers(0, 3)) if n_consts is None else n_consts
    verts = [None] * nv
    for _ in range(nc):
        # occasionally a constant outside the data (empty-result path)
        cid = int(rng.integers(0, n_entities + (1 if rng.random() < 0.1 else 0)))
        verts.append(cid)
    nvert = len(verts)
    order = rng.permutation(nvert).tolist()
    edges = []

    def pred():
        return int(rng.integers(1, n_predicates + 1))

    # spanning tree over all vertices (random direction) => connected
    for k in range(1, nvert):
        a = order[k]
        b = order[int(rng.integers(0, k))] if connected or rng.random() < 0.7 else None
        if b is None:
            continue
        if rng.random() < 0.5:
            a, b = b, a
        edges.append((a, pred(), b))
    ne = int(rng.integers(0, 3)) if extra_edges is None else extra_edges
    for _ in range(ne):
        a = int(rng.integers(0, nvert))
        b = int(rng.integers(0, nvert))
        if a == b and not allow_self_loops:
            continue
        edges.append((a, pred(), b))
    # every variable must occur in some edge (ABI precondition)
    used = {x for e in edges for x in (e[0], e[2])}
    for i in range(nvert):
        if i not in used:
            j = int(rng.integers(0, nvert))
            if j == i and not allow_self_loops:
                j = (i + 1) % nvert
            edges.append((i, pred(), j) if rng.random() < 0.5 else (j, pred(), i))
            used.update((i, j))
    # const-const only queries are legal but keep at least one variable
    return Query(tuple(verts), tuple(edges))


def random_case(seed, max_entities=6, max_predicates=3, max_triples=14, **qkw):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, max_entities + 1))
    P = int(rng.integers(1, max_predicates + 1))
    m = int(rng.integers(0, max_triples + 1))
    s, p, o = random_triples(rng, n, P, m)
    q = random_query(rng, n, P, **qkw)
    return (s, p, o), n, P, q


def random_graph(seed, n_entities, n_predicates, n_triples, skew=0.0):
    """Larger random graph (parity at sizes spanning several tiles).  skew > 0
    draws subjects/objects from a power law to create hub rows."""
    rng = np.random.default_rng(seed)
    if skew > 0:
        w = 1.0 / np.arange(1, n_entities + 1) ** skew
        w /= w.sum()
        perm = rng.permutation(n_entities)
        s = perm[rng.choice(n_entities, n_triples, p=w)]
        o = perm[rng.choice(n_entities, n_triples, p=w)]
    else:
        s = rng.integers(0, n_entities, n_triples)
        o = rng.integers(0, n_entities, n_triples)
    p = rng.integers(1, n_predicates + 1, n_triples)
    return (s.astype(np.uint32), p.astype(np.uint32), o.astype(np.uint32))
