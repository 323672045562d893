"""Probe the WatDiv-shaped configs[2] workload at a given scale on the GPU box:
generation time, LSpM build time, per-query rows / latency / launches, and
the C oracle's index build + per-query time on the host cores (bounded)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=float, default=2.1)
ap.add_argument("--oracle", action="store_true")
ap.add_argument("--parity", action="store_true")
args = ap.parse_args()

import paper_2106_14038_b200 as G  # noqa: E402
from synth import watdiv  # noqa: E402

t0 = time.perf_counter()
d = watdiv.generate(args.scale, device="cuda")
torch.cuda.synchronize()
print(f"gen scale={args.scale} triples={d.s.numel()} N={d.n_entities} {time.perf_counter() - t0:.2f}s", flush=True)
qs = watdiv.queries(d)
eng = G.Engine(0)
G.gsmart_load_triples(eng.ctx, d.s, d.p, d.o, d.n_entities, d.n_predicates)
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G.gsmart_build_lspm(eng.ctx)
    torch.cuda.synchronize()
    print(f"build {1000 * (time.perf_counter() - t0):.2f} ms", flush=True)
plans = [G.gsmart_plan(eng.ctx, q) for q in qs]
for rep in range(3):
    for q, pl in zip(qs, plans):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = G.gsmart_execute(eng.ctx, pl, G.GSMART_KEEP_ON_DEVICE)
        dt = 1000 * (time.perf_counter() - t0)
        st = G.gsmart_result_stats(r)
        n = G.gsmart_result_shape(r)[0]
        G.gsmart_result_free(r)
        if rep == 2:
            print(f"{q.name:3s} rows={n:10d} ms={dt:8.3f} launches={sum(st['launches'].values()):3d} "
                  f"levels={st['level_nodes']} edges_read={st['edges_evaluated']}", flush=True)
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for r in G.gsmart_execute_batch(eng.ctx, plans, G.GSMART_KEEP_ON_DEVICE):
        G.gsmart_result_free(r)
    torch.cuda.synchronize()
    print(f"batch {1000 * (time.perf_counter() - t0):.3f} ms", flush=True)
for q, pl in zip(qs, plans):
    r = G.gsmart_execute(eng.ctx, pl, G.GSMART_PROFILE | G.GSMART_KEEP_ON_DEVICE)
    st = G.gsmart_result_stats(r)
    G.gsmart_result_free(r)
    ms = {k: round(v, 4) for k, v in st["ms_kernel"].items() if v > 0}
    print(f"{q.name:3s} kernel_ms total={sum(ms.values()):.4f}", ms, flush=True)
if args.oracle or args.parity:
    from oracle.coracle import OracleIndex
    s, p, o = d.s.cpu().numpy(), d.p.cpu().numpy(), d.o.cpu().numpy()
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    ix = OracleIndex(s, p, o)
    print(f"oracle index {time.perf_counter() - t0:.2f}s cores={cores}", flush=True)
    for q, pl in zip(qs, plans):
        t0 = time.perf_counter()
        exp = ix.query(q, n_threads=cores)
        dt = time.perf_counter() - t0
        line = f"oracle {q.name:3s} rows={len(exp):10d} {dt:8.3f}s"
        if args.parity:
            r = G.gsmart_execute(eng.ctx, pl, 0)
            got = G.gsmart_result_rows(r)
            G.gsmart_result_free(r)
            line += f" parity={got.shape == exp.shape and np.array_equal(got, exp)}"
            r = G.gsmart_execute(eng.ctx, pl, G.GSMART_FACTORISED)  # f2: rows read off the factorised trees
            got = G.gsmart_result_rows(r)
            fst = G.gsmart_result_stats(r)
            G.gsmart_result_free(r)
            line += (f" factorised_parity={got.shape == exp.shape and np.array_equal(got, exp)}"
                     f" (omega={fst['n_omega']} nodes={sum(fst['level_nodes'])})")
        print(line, flush=True)
eng.close()
