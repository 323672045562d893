"""Per-query A/B of execute flags on one resident workload: median latency
(host wall time around gsmart_execute, warm, rows kept on the device) of each
query under each flag set, plus the result sizes.

    python scripts/ab_queries.py --workload watdiv100m --variants "0;256;1;257"
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="watdiv100m")
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--variants", default="0;256")
args = ap.parse_args()

import bench  # noqa: E402
import paper_2106_14038_b200 as G  # noqa: E402

dev = torch.device("cuda", 0)
s, p, o, N, P, qs = bench.workload(args.workload, device=dev)
eng = G.Engine(0)
G.gsmart_load_triples(eng.ctx, s, p, o, N, P)
G.gsmart_build_lspm(eng.ctx)
del s, p, o
plans = [G.gsmart_plan(eng.ctx, q) for q in qs]
variants = [int(v) for v in args.variants.split(";")]
print("query " + " ".join(f"{'flags=' + str(v):>22s}" for v in variants))
tot = {v: 0.0 for v in variants}
for q, pl in zip(qs, plans):
    cells = []
    for v in variants:
        ts, n, st = [], 0, None
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = G.gsmart_execute(eng.ctx, pl, v | G.GSMART_KEEP_ON_DEVICE)
            ts.append((time.perf_counter() - t0) * 1e3)
            n = G.gsmart_result_shape(r)[0]
            st = G.gsmart_result_stats(r)
            G.gsmart_result_free(r)
        med = statistics.median(ts[2:] if len(ts) > 3 else ts)
        tot[v] += med
        nodes = sum(st["level_nodes"])
        cells.append(f"{med:8.3f} ms n={n:<9d} nodes={nodes:<9d}")
    print(f"{q.name:5s} " + " | ".join(cells), flush=True)
print("sum   " + " | ".join(f"{tot[v]:8.3f} ms" for v in variants))
