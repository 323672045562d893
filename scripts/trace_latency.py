"""Host-side timeline of single executes (GSMART_TRACE=1) on LUBM-100."""
import os, sys, time
os.environ["GSMART_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_14038_b200 as G
from synth import lubm
d = lubm.generate(100, device="cuda")
qs = lubm.queries(d)
e = G.Engine(0)
G.gsmart_load_triples(e.ctx, d.s, d.p, d.o, d.n_entities, d.n_predicates)
G.gsmart_build_lspm(e.ctx)
plans = [G.gsmart_plan(e.ctx, q) for q in qs]
for rep in range(4):
    for q, pl in zip(qs, plans):
        if rep == 3:
            print(f"--- {q.name}", file=sys.stderr, flush=True)
        t0 = time.perf_counter()
        r = G.gsmart_execute(e.ctx, pl, G.GSMART_KEEP_ON_DEVICE)
        t1 = time.perf_counter()
        G.gsmart_result_free(r)
        if rep == 3:
            print(f"    python wall {1e6*(t1-t0):.1f} us", file=sys.stderr, flush=True)
# the bench step: all queries in one gsmart_execute_batch
for rep in range(4):
    if rep == 3:
        print("--- batch", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    rs = G.gsmart_execute_batch(e.ctx, plans, G.GSMART_KEEP_ON_DEVICE)
    t1 = time.perf_counter()
    for r in rs:
        G.gsmart_result_free(r)
    if rep == 3:
        print(f"    python wall {1e6*(t1-t0):.1f} us", file=sys.stderr, flush=True)
