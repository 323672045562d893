"""Run the LUBM query batch sequentially on a resident LSpM (for ncu launch lists
of the query kernels only, and for host-vs-GPU time breakdowns)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--universities", type=int, default=100)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--queries", default="")
args = ap.parse_args()

import paper_2106_14038_b200 as G  # noqa: E402
from synth import lubm  # noqa: E402

dev = torch.device("cuda", 0)
d = lubm.generate(args.universities, seed=lubm.SEED_LUBM100 if args.universities == 100 else lubm.SEED_LUBM10K,
                  device=dev)
qs = lubm.queries(d)
if args.queries:
    qs = [q for q in qs if q.name in args.queries.split(",")]
eng = G.Engine(0)
G.gsmart_load_triples(eng.ctx, d.s, d.p, d.o, d.n_entities, d.n_predicates)
G.gsmart_build_lspm(eng.ctx)
plans = [G.gsmart_plan(eng.ctx, q) for q in qs]
for rep in range(args.reps):
    for q, pl in zip(qs, plans):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = G.gsmart_execute(eng.ctx, pl, G.GSMART_KEEP_ON_DEVICE)
        dt = 1000 * (time.perf_counter() - t0)
        st = G.gsmart_result_stats(r)
        n = G.gsmart_result_shape(r)[0]
        G.gsmart_result_free(r)
        if rep == args.reps - 1:
            print(f"{q.name:4s} rows={n:9d} wall_ms={dt:7.3f} launches={sum(st['launches'].values()):3d} "
                  f"levels={st['level_nodes']} filter_rows={st['filter_rows']} scanned={st['filter_entries']} "
                  f"expand={st['expand_entries']}", flush=True)
            print("     ", {k: v for k, v in st['launches'].items() if v}, flush=True)
# per-kernel-class CUDA-event times of each query (GSMART_PROFILE: events on the launch stream)
for q, pl in zip(qs, plans):
    r = G.gsmart_execute(eng.ctx, pl, G.GSMART_PROFILE | G.GSMART_KEEP_ON_DEVICE)
    st = G.gsmart_result_stats(r)
    G.gsmart_result_free(r)
    ms = {k: round(v, 4) for k, v in st["ms_kernel"].items() if v > 0}
    print(f"{q.name:4s} kernel_ms total={sum(ms.values()):.4f}", ms, flush=True)
