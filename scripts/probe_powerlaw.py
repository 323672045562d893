"""Probe BASELINE.json configs[4] at full size on one GPU: the power-law
YAGO/DBpedia-shaped set (500M triples, 100M entities, 10,000 labels -> 68-bit
(row, pred, col) keys: the two-word radix-sort path), LSpM build time, and the
random-walk queries (count, latency).  With --oracle, the C oracle's counts
for the queries it finishes within a per-query budget."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--triples", type=int, default=500_000_000)
ap.add_argument("--queries", type=int, default=12)
ap.add_argument("--oracle", action="store_true")
args = ap.parse_args()

import paper_2106_14038_b200 as G  # noqa: E402
from synth import powerlaw  # noqa: E402

t0 = time.perf_counter()
d = powerlaw.generate(args.triples, device="cuda")
torch.cuda.synchronize()
print(f"gen triples={d.s.numel()} N={d.n_entities} P={d.n_predicates} {time.perf_counter() - t0:.1f}s", flush=True)
qs = powerlaw.queries(d, args.queries, seed=1)
print(f"queries sampled {time.perf_counter() - t0:.1f}s", flush=True)
eng = G.Engine(0, max_result_rows=1 << 30)
G.gsmart_load_triples(eng.ctx, d.s, d.p, d.o, d.n_entities, d.n_predicates)
for i in range(2):
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    G.gsmart_build_lspm(eng.ctx)
    torch.cuda.synchronize()
    print(f"build {1000 * (time.perf_counter() - t1):.1f} ms", flush=True)
v = G.gsmart_lspm_get(eng.ctx, G.GSMART_CSR)
print(f"CSR nnz={v['nnz']} pred_bytes={v['pred_bytes']}", flush=True)
counts = {}
for q in qs:
    try:
        with eng.plan(q) as pl:
            for rep in range(2):
                torch.cuda.synchronize()
                t1 = time.perf_counter()
                r = G.gsmart_execute(eng.ctx, pl.h, G.GSMART_COUNT_ONLY)
                dt = 1000 * (time.perf_counter() - t1)
                n = G.gsmart_result_shape(r)[0]
                st = G.gsmart_result_stats(r)
                G.gsmart_result_free(r)
        counts[q.name] = n
        print(f"{q.name:8s} edges={q.edges} rows={n} ms={dt:.2f} levels={st['level_nodes']}", flush=True)
    except G.GsmartError as e:
        print(f"{q.name:8s} edges={q.edges} {e.name}", flush=True)
eng.close()
if args.oracle:
    from oracle.coracle import OracleIndex
    s, p, o = d.s.cpu().numpy(), d.p.cpu().numpy(), d.o.cpu().numpy()
    del d
    t1 = time.perf_counter()
    ix = OracleIndex(s, p, o)
    print(f"oracle index {time.perf_counter() - t1:.1f}s", flush=True)
    for q in qs:
        if q.name not in counts or counts[q.name] > 5_000_000:
            continue
        t1 = time.perf_counter()
        n = len(ix.query(q, n_threads=len(os.sched_getaffinity(0))))
        print(f"oracle {q.name:8s} rows={n} gpu={counts[q.name]} match={n == counts[q.name]} "
              f"{time.perf_counter() - t1:.1f}s", flush=True)
