"""Power-law (YAGO/DBpedia-shaped) synthetic RDF generator (BASELINE.json
configs[4]): ~500M triples, ~100M entities, 10,000 predicates with Zipf
frequencies, heavy-tailed subject out-degrees and object popularity with hub
objects (in-degree ~1e7 at full size) — the skew that stresses load balance
and tree pruning.  Integer-only counter-based draws: identical
on any device.  Queries are sampled by random walks over the generated
triples (stars, chains, triangles, 0-2 constants) so results are non-empty.
"""
from dataclasses import dataclass

import numpy as np
import torch

from .query import Query
from .rng import draw

SEED_POWERLAW = 0x504C415700


@dataclass
class PowerlawData:
    s: torch.Tensor
    p: torch.Tensor
    o: torch.Tensor
    n_entities: int
    n_predicates: int


def _loguniform(seed, stream, idx, m):
    """rank in [0, m): log-uniform (Zipf(1)-like) via a random right shift."""
    nb = int(m).bit_length()
    sh = draw(seed, stream + 1, idx) % (nb + 1)
    return (draw(seed, stream, idx) % m) >> sh


def generate(n_triples=500_000_000, n_entities=100_000_000, n_predicates=10_000, seed=SEED_POWERLAW,
             device="cpu", chunk=50_000_000) -> PowerlawData:
    dev = torch.device(device)
    S, P, O = [], [], []
    for b in range(0, n_triples, chunk):
        i = torch.arange(b, min(b + chunk, n_triples), device=dev, dtype=torch.int64)
        # subject: mix of log-uniform (heavy out-degree tail) and uniform
        su = draw(seed, 1, i) % n_entities
        sz = _loguniform(seed, 2, i, n_entities)
        s = torch.where(draw(seed, 3, i) % 4 == 0, sz, su)
        # object: log-uniform popularity (hubs at low ranks), scattered by a bijective
        # affine map so hubs do not all sit next to each other in id space
        o = (_loguniform(seed, 4, i, n_entities) * 2654435761 + 12345) % n_entities
        p = 1 + _loguniform(seed, 5, i, n_predicates)
        S.append(s.to(torch.int32))
        P.append(p.to(torch.int32))
        O.append(o.to(torch.int32))
    return PowerlawData(s=torch.cat(S), p=torch.cat(P), o=torch.cat(O), n_entities=int(n_entities),
                        n_predicates=int(n_predicates))


def queries(d: PowerlawData, n_queries=20, seed=7):
    """Random-walk sampled BGPs over the data (host numpy): stars (3-5 edges
    out of one subject), chains (3-4 hops), triangles when the walk closes,
    with 0-2 vertices replaced by their constant."""
    rng = np.random.default_rng(seed)
    s = d.s.cpu().numpy()
    # subject-grouped copies for the walks: a stable sort by subject (on the
    # data's device — the full 500M-triple set sorts in seconds on a GPU)
    order = torch.sort(d.s, stable=True).indices
    ss = d.s[order]
    pp = d.p[order].cpu().numpy()
    oo = d.o[order].cpu().numpy()
    starts = torch.searchsorted(ss, torch.arange(d.n_entities + 1, device=ss.device, dtype=ss.dtype)).cpu().numpy()
    del order, ss

    def out_edges(x):
        a, b = starts[x], starts[x + 1]
        return pp[a:b], oo[a:b]

    qs = []
    tries = 0
    while len(qs) < n_queries and tries < 50 * n_queries:
        tries += 1
        kind = ["star", "chain", "tri"][len(qs) % 3]
        x = int(s[rng.integers(0, len(s))])
        if kind == "star":
            lp, lo = out_edges(x)
            if len(lp) < 3:
                continue
            pick = rng.choice(len(lp), size=min(len(lp), int(rng.integers(3, 6))), replace=False)
            labels = sorted({int(lp[i]) for i in pick})
            verts = [None] * (1 + len(labels))
            edges = [(0, l, 1 + j) for j, l in enumerate(labels)]
        elif kind == "chain":
            verts, edges, cur = [None], [], x
            for h in range(int(rng.integers(3, 5))):
                lp, lo = out_edges(cur)
                if len(lp) == 0:
                    break
                j = int(rng.integers(0, len(lp)))
                verts.append(None)
                edges.append((h, int(lp[j]), h + 1))
                cur = int(lo[j])
            if len(edges) < 2:
                continue
        else:  # triangle x -> y -> z, closing z -> x or x -> z if present
            lp, lo = out_edges(x)
            if len(lp) == 0:
                continue
            j = int(rng.integers(0, len(lp)))
            y = int(lo[j])
            lp2, lo2 = out_edges(y)
            if len(lp2) == 0:
                continue
            k = int(rng.integers(0, len(lp2)))
            z = int(lo2[k])
            lp3, lo3 = out_edges(x)
            close = [int(lp3[t]) for t in range(len(lp3)) if int(lo3[t]) == z]
            verts = [None, None, None]
            edges = [(0, int(lp[j]), 1), (1, int(lp2[k]), 2)]
            if close:
                edges.append((0, close[0], 2))
            else:
                continue
        # 0-2 constants: replace vertices by the values of the walk where known
        nconst = int(rng.integers(0, 3))
        if nconst and kind == "star":
            lp, lo = out_edges(x)
            for (a, l, b) in edges[:nconst]:
                hits = lo[lp == l]
                if len(hits):
                    verts[b] = int(hits[0])
        qs.append(Query(tuple(verts), tuple(edges), name=f"{kind}{len(qs)}"))
    return qs
