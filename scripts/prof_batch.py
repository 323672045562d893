"""Profiling driver: load + build one workload, warm up, then run ONE query
batch (or each query alone with --sequential) between cudaProfilerStart/Stop,
so `ncu --profile-from-start off` captures exactly the launches of one step.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python scripts/prof_batch.py --workload watdiv100m
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="watdiv100m")
ap.add_argument("--sequential", action="store_true")
ap.add_argument("--queries", default="")
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--build", action="store_true", help="profile the LSpM build instead of the batch")
args = ap.parse_args()

import bench  # noqa: E402
import paper_2106_14038_b200 as G  # noqa: E402

dev = torch.device("cuda", 0)
s, p, o, N, P, qs = bench.workload(args.workload, device=dev)
if args.queries:
    qs = [q for q in qs if q.name in args.queries.split(",")]
eng = G.Engine(0)
G.gsmart_load_triples(eng.ctx, s, p, o, N, P)
G.gsmart_build_lspm(eng.ctx)
if args.build:
    G.gsmart_build_lspm(eng.ctx)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    G.gsmart_build_lspm(eng.ctx)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    sys.exit(0)
del s, p, o
plans = [G.gsmart_plan(eng.ctx, q) for q in qs]
flags = args.flags | G.GSMART_KEEP_ON_DEVICE


def once():
    if args.sequential:
        for pl in plans:
            G.gsmart_result_free(G.gsmart_execute(eng.ctx, pl, flags))
    else:
        for r in G.gsmart_execute_batch(eng.ctx, plans, flags):
            G.gsmart_result_free(r)


for _ in range(3):
    once()
torch.cuda.synchronize()
torch.cuda.profiler.start()
once()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled", [q.name for q in qs])
