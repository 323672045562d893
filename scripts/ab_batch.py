"""A/B of execution variants on one resident workload: batch ms/step (CUDA
events, L2 flushed between steps) for each setting of the library's A/B
switches (read at gsmart_create): default, GSMART_NO_TMA=1 (plain loads
instead of cp.async.bulk staging), GSMART_L2_PERSIST=1 (persisting L2 window
over the candidate bitmaps), GSMART_FILTER_VARIANT=...

    python scripts/ab_batch.py --workload watdiv100m --steps 20
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="watdiv100m")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--variants", default="default;GSMART_NO_TMA=1;GSMART_L2_PERSIST=1")
args = ap.parse_args()

import bench  # noqa: E402
import paper_2106_14038_b200 as G  # noqa: E402

dev = torch.device("cuda", 0)
s, p, o, N, P, qs = bench.workload(args.workload, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for var in args.variants.split(";"):
    env = {} if var == "default" else dict(kv.split("=") for kv in var.split(","))
    xflags = int(env.pop("flags", "0"))  # execute flags, e.g. flags=128 (GSMART_BACK_EDGES)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)  # kept for the whole variant (some switches are read per launch)
    eng = G.Engine(0)
    G.gsmart_load_triples(eng.ctx, s, p, o, N, P)
    G.gsmart_build_lspm(eng.ctx)
    plans = [G.gsmart_plan(eng.ctx, q) for q in qs]
    st = torch.cuda.current_stream(dev)

    def step():
        for r in G.gsmart_execute_batch(eng.ctx, plans, G.GSMART_KEEP_ON_DEVICE | xflags):
            G.gsmart_result_free(r)

    for _ in range(args.warmup):
        step()
    ts = []
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        step()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    lat = {}
    for q, pl in zip(qs, plans):
        xs = []
        for _ in range(5):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            G.gsmart_result_free(G.gsmart_execute(eng.ctx, pl, G.GSMART_KEEP_ON_DEVICE | xflags))
            e1.record(st)
            e1.synchronize()
            xs.append(e0.elapsed_time(e1))
        lat[q.name] = round(statistics.median(xs), 3)
    print(f"{var:40s} batch ms/step mean {statistics.mean(ts):.3f} median {statistics.median(ts):.3f}  "
          f"per-query {lat}", flush=True)
    for pl in plans:
        G.gsmart_plan_free(pl)
    eng.close()
    for k, v in old.items():
        if v is None:
            del os.environ[k]
        else:
            os.environ[k] = v
