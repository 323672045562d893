"""LSpM build timing on one workload (GSMART_TRACE=1 prints per-phase laps):
    python scripts/probe_build.py --workload lubm10k --reps 3
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="lubm10k")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()

import bench  # noqa: E402
import paper_2106_14038_b200 as G  # noqa: E402

dev = torch.device("cuda", 0)
s, p, o, N, P, qs = bench.workload(args.workload, device=dev)
eng = G.Engine(0)
G.gsmart_load_triples(eng.ctx, s, p, o, N, P)
for i in range(args.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G.gsmart_build_lspm(eng.ctx)
    torch.cuda.synchronize()
    print(f"build {i}: {1000 * (time.perf_counter() - t0):.1f} ms", flush=True)
