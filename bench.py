#!/usr/bin/env python
"""Benchmark of the B200 gSmart hot path (BASELINE.json metric: query latency
ms & edges evaluated/sec per LUBM/WatDiv query; HBM GB/s fraction at 1-8 GPUs).

Workload (default, every N): BASELINE.json configs[2] — WatDiv-shaped
synthetic, scale 2.1 (~108M triples, 85 predicates), the 11-template L/S/F/C
query batch.  configs[2] names "1 and 8 B200", so the same command measures
N=1 and, under torchrun, N>1 (strong scaling: one batch over the 1-D
vertex-range partition).  `--workload lubm100|lubm10k|powerlaw` selects the
other configs (extra lines).

A "step" = one pass of the query batch through gsmart_execute_batch (a2..a9:
seeds, grouped incident-edge evaluation, compaction, trie expansion,
pre-pruning, bottom-up pruning, row enumeration + sort) over the LSpM
resident in HBM.  The LSpM build (a1) is timed separately ("build") and is
inside the end-to-end leg ("e2e": host triples -> load -> build -> plan ->
batch -> rows on host, per-stage breakdown).

`value` counts label-edges per second in the Graph500 TEPS convention: the
numerator is a property of the workload, not of an implementation,
E(q) = sum over the patterns of q of |{t in T : pred(t) = label}| (the
nonzeros of p*I (x) A, Eqs. 12-13, that the query's patterns select) — so
both arms divide the same E by their own time and the driver's ratio is a
time ratio.  SURVEY §8(d)'s implementation-side count (LSpM entries the GPU
path actually read whose label matched) and its rate are reported beside it
(`edges_read`), as are the batch latency and per-query latencies (ms).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload W]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "label-edges evaluated/s (TEPS convention), query batch"
UNIT = "edges/s"

WORKLOADS = {
    "watdiv100m": "WatDiv-100M (configs[2]): scale 2.1, 11 L/S/F/C templates as one batch",
    "lubm100": "LUBM-100 (configs[1]): L1-L7 + Q14 batch",
    "lubm10k": "LUBM-10k (configs[3]): L1-L7 + Q14 batch",
    "powerlaw": "power-law YAGO/DBpedia-shaped (configs[4]): 500M triples, 10k predicates, random-walk queries",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="watdiv100m", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--mode", default="partitioned", choices=["replicas", "partitioned"],
                    help="N>1: partitioned = one batch over the 1-D vertex-range partition of the LSpM "
                         "(strong scaling, default); replicas = every GPU serves its own copy of the batch")
    return ap.parse_args()


def config_of(args):
    """The workload description both arms print (identical dicts: same_config)."""
    return {"workload": WORKLOADS[args.workload], "name": args.workload,
            "l2": "flushed between timed steps (256 MiB write)"}


def workload(name, device="cpu"):
    """(s, p, o int32 tensors, n_entities, n_predicates, queries) — counter-based
    generators: identical triples on any device."""
    if name == "watdiv100m":
        from synth import watdiv
        d = watdiv.generate(watdiv.SCALE_100M, device=device)
        return d.s, d.p, d.o, d.n_entities, d.n_predicates, watdiv.queries(d)
    if name in ("lubm100", "lubm10k"):
        from synth import lubm
        U, seed = (100, lubm.SEED_LUBM100) if name == "lubm100" else (10000, lubm.SEED_LUBM10K)
        d = lubm.generate(U, seed=seed, device=device)
        return d.s, d.p, d.o, d.n_entities, d.n_predicates, lubm.queries(d)
    from synth import powerlaw
    d = powerlaw.generate(device=device)
    return d.s, d.p, d.o, d.n_entities, d.n_predicates, powerlaw.queries(d, 12, seed=1)


def label_counts(s, p, o):
    """De-duplicated triple count per predicate (input statistics; torch, any device)."""
    import torch
    out = {}
    key = (s.long() << 32) | o.long()
    for l in torch.unique(p).tolist():
        out[int(l)] = int(torch.unique(key[p == l]).numel())
    return out


def edges_per_query(queries, counts):
    """E(q) per query (module doc): the workload's label-edge count."""
    return [int(sum(counts.get(l, 0) for _, l, _ in q.edges)) for q in queries]


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(x[0]) for x in self.samples if x[0].replace(".", "").isdigit()]
        mx = [float(x[1]) for x in self.samples if x[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for x in self.samples for i in range(4) if x[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel_class, name):
    """DRAM bytes per launch of a kernel class from the committed `ncu --set
    full` capture of the same workload (profiles/ncu_traffic_<name>.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_traffic_{name}.json")) as f:
            e = json.load(f).get(kernel_class)
        return None if e is None else e.get("dram_bytes_per_launch")
    except Exception:
        return None


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec as N ranks."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle (plain CPU BGP engine, oracle/bgp_oracle.c), as it stands, on
    the host cores; index build excluded (the paper separates loading).  Each
    step is a bounded sample: the whole batch when (K + W) batches fit ~150 s,
    else a round-robin slice of the queries sized to fit."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle.coracle import OracleIndex
    s, p, o, N, P, qs = workload(args.workload)
    E = edges_per_query(qs, label_counts(s, p, o))
    s, p, o = s.numpy(), p.numpy(), o.numpy()
    ix = OracleIndex(s, p, o)
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    for q in qs:
        ix.query(q, n_threads=cores)
    t_batch = time.perf_counter() - t0
    per_step = max(1, min(len(qs), int(len(qs) * 150.0 / max(1e-9, t_batch * (args.steps + args.warmup)))))
    cursor = 0

    def one_step():
        nonlocal cursor
        e = 0
        for _ in range(per_step):
            i = cursor % len(qs)
            ix.query(qs[i], n_threads=cores)
            e += E[i]
            cursor += 1
        return e

    for _ in range(args.warmup):
        one_step()
    tot_e, tot_t = 0, 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        tot_e += one_step()
        tot_t += time.perf_counter() - t0
    value = tot_e / tot_t
    sample = (f"{per_step} of {len(qs)} queries per step, round-robin" if per_step < len(qs)
              else f"the full {len(qs)}-query batch per step") + " (oracle index build excluded)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic", "config": config_of(args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- our arm
def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus > 1 and world == 1 and "RANK" not in os.environ:
        return relaunch_under_torchrun(args)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    n_dev = max(1, torch.cuda.device_count())
    oversub = world > n_dev  # more ranks than devices (e.g. checking the N>1 path on one GPU): share devices
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo" if oversub else "nccl", init_method="env://")
    local = local % n_dev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2106_14038_b200 as G

    # inputs: generated in HBM (counter-based: identical triples on any device);
    # host copies for the e2e leg and the CPU baseline
    s_d, p_d, o_d, N, P, qs = workload(args.workload, device=dev)
    E = edges_per_query(qs, label_counts(s_d, p_d, o_d))
    # the e2e leg's inputs live in pinned host memory (the contract's H2D "from pinned host memory")
    s_h, p_h, o_h = s_d.cpu().pin_memory(), p_d.cpu().pin_memory(), o_d.cpu().pin_memory()
    torch.cuda.empty_cache()
    stream = torch.cuda.current_stream(dev)
    partitioned = world > 1 and args.mode == "partitioned"
    if partitioned:  # NCCL unique id from rank 0 over torch.distributed
        obj = [G.gsmart_get_nccl_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        eng = G.Engine(local, rank=rank, world=world, nccl_id=obj[0], stream=stream.cuda_stream)
    else:
        eng = G.Engine(local, stream=stream.cuda_stream)
    copies = 1 if partitioned else world  # batches processed per step across all ranks
    # ---- a1 build, timed separately (resident triples)
    G.gsmart_load_triples(eng.ctx, s_d, p_d, o_d, N, P)
    bt = []
    for i in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        G.gsmart_build_lspm(eng.ctx)
        e1.record(stream)
        torch.cuda.synchronize()
        if i:
            bt.append(e0.elapsed_time(e1))
    build_ms = statistics.median(bt)
    del s_d, p_d, o_d
    torch.cuda.empty_cache()
    plans = [G.gsmart_plan(eng.ctx, q) for q in qs]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step(flags=0, stats=None):
        # the query batch runs concurrently (gsmart_execute_batch: one stream + workspace per query)
        for r in G.gsmart_execute_batch(eng.ctx, plans, flags | G.GSMART_KEEP_ON_DEVICE):
            if stats is not None:
                stats.append(G.gsmart_result_stats(r))
            G.gsmart_result_free(r)

    for _ in range(args.warmup):
        step()
    # ---- timed region: K steps, each bracketed by events; L2 flushed between steps
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    times = []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    ms = statistics.mean(times)
    if world > 1:  # max over ranks
        t = torch.tensor([ms], device="cpu" if oversub else dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.barrier()
        ms = float(t.item())
    value = copies * sum(E) / (ms / 1000)

    # ---- launches and device counters of one batch (same flags as the timed steps)
    batch_stats = []
    step(stats=batch_stats)
    launches_per_step = sum(sum(st["launches"].values()) for st in batch_stats)
    edges_read = sum(st["edges_evaluated"] for st in batch_stats)
    xchg_bytes = sum(st["allgather_bytes"] for st in batch_stats)  # bitmap words this rank received per step

    # ---- profiled pass: the same queries one at a time (GSMART_PROFILE: per-kernel-class
    # CUDA events on the launching stream; sequential so no other stream shares the GPU)
    prof_stats = []
    n_prof = min(args.steps, 5)
    for _ in range(n_prof):
        flush.fill_(1)
        for pl in plans:
            r = G.gsmart_execute(eng.ctx, pl, G.GSMART_PROFILE | G.GSMART_KEEP_ON_DEVICE)
            prof_stats.append(G.gsmart_result_stats(r))
            G.gsmart_result_free(r)
    torch.cuda.synchronize()
    ksum, kbytes, klaunch = {}, {}, {}
    for st in prof_stats:
        for k, v in st["ms_kernel"].items():
            ksum[k] = ksum.get(k, 0.0) + v
        for k, v in st["bytes"].items():
            kbytes[k] = kbytes.get(k, 0) + v
        for k, v in st["launches"].items():
            klaunch[k] = klaunch.get(k, 0) + v
    measured = {k: v for k, v in ksum.items() if kbytes.get(k, 0) > 0 and v > 0}
    dom = max(measured, key=lambda k: ksum[k]) if measured else None
    peak, peak_src = peaks()
    roofline = None
    if dom:
        n_launch = max(1, klaunch[dom])
        achieved = kbytes[dom] / (ksum[dom] / 1000) / 1e9
        roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": ncu_traffic(dom, args.workload),
                    "algorithmic_bytes_per_launch": kbytes[dom] / n_launch,
                    "ms_share_of_step": ksum[dom] / max(1e-9, sum(ksum.values())),
                    "peak_source": peak_src,
                    "timing": "CUDA events on the launch stream around each launch of the class "
                              "(GSMART_PROFILE pass, queries one at a time)"}
    per_class = {k: {"ms_per_batch": ksum[k] / n_prof, "launches_per_batch": klaunch[k] / n_prof,
                     "algorithmic_GBps": (kbytes[k] / (ksum[k] / 1000) / 1e9) if ksum[k] > 0 else None}
                 for k in ksum if ksum[k] > 0}

    # ---- per-query latency: warm (same plan: graph replay + speculative phase 2) and
    # cold (a fresh plan per execute: push/pull decision, graph capture, no speculation)
    per_query = {}
    for i, q in enumerate(qs):
        warm, cold = [], []
        for _ in range(7):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = G.gsmart_execute(eng.ctx, plans[i], G.GSMART_KEEP_ON_DEVICE)
            warm.append(1000 * (time.perf_counter() - t0))
            G.gsmart_result_free(r)
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pl = G.gsmart_plan(eng.ctx, q)
            r = G.gsmart_execute(eng.ctx, pl, G.GSMART_KEEP_ON_DEVICE)
            cold.append(1000 * (time.perf_counter() - t0))
            G.gsmart_result_free(r)
            G.gsmart_plan_free(pl)
        st = batch_stats[i]
        per_query[q.name] = {"latency_ms": statistics.median(warm), "cold_latency_ms": statistics.median(cold),
                             "rows": int(st["level_alive"][-1]) if st["n_levels"] else 0, "edges": E[i],
                             "edges_read": st["edges_evaluated"]}

    # ---- e2e through the public API: host triples (pinned-staged by the library) ->
    # load -> build -> plan -> batch -> rows on host, per-stage wall time
    stages = {"load_h2d": [], "build": [], "plan": [], "execute": [], "rows_d2h": []}
    e2e_times = []
    d2h = 0
    for it in range(args.e2e_steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        G.gsmart_load_triples(eng.ctx, s_h, p_h, o_h, N, P)
        t1 = time.perf_counter()
        G.gsmart_build_lspm(eng.ctx)
        t2 = time.perf_counter()
        ps = [G.gsmart_plan(eng.ctx, q) for q in qs]
        t3 = time.perf_counter()
        res = G.gsmart_execute_batch(eng.ctx, ps, G.GSMART_KEEP_ON_DEVICE)
        t4 = time.perf_counter()
        nbytes = 0
        for r in res:
            if rank == 0 or not partitioned:
                rows = G.gsmart_result_rows(r, copy=False)  # D2H into the result's pinned block
                nbytes += rows.nbytes
                if rows.size:
                    _ = int(rows[-1, -1])  # touch the host copy
            G.gsmart_result_free(r)
        for pl in ps:
            G.gsmart_plan_free(pl)
        t5 = time.perf_counter()
        if it:
            e2e_times.append(t5 - t0)
            for k, a, b in (("load_h2d", t0, t1), ("build", t1, t2), ("plan", t2, t3), ("execute", t3, t4),
                            ("rows_d2h", t4, t5)):
                stages[k].append(1000 * (b - a))
        d2h = nbytes
    e2e_s = statistics.median(e2e_times)  # median of the e2e steps (robust to a slow outlier step)
    e2e_value = copies * sum(E) / e2e_s

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle.coracle import OracleIndex
        ix = OracleIndex(s_h.numpy(), p_h.numpy(), o_h.numpy())
        cores = len(os.sched_getaffinity(0))
        t0 = time.perf_counter()
        e_done, n_q = 0, 0
        while time.perf_counter() - t0 < 15.0 and n_q < 50 * len(qs):
            i = n_q % len(qs)
            ix.query(qs[i], n_threads=cores)
            e_done += E[i]
            n_q += 1
        cpu_s = time.perf_counter() - t0
        cpu = {"value": e_done / cpu_s, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{n_q} queries of the batch, round-robin (~15 s of CPU work), index build excluded",
               "ms_per_batch": 1000 * cpu_s * len(qs) / n_q}

    cfg = config_of(args)  # identical in both arms (same_config); sizes and layout beside it
    info = {}
    info.update({"triples": int(len(s_h)), "entities": int(N), "predicates": int(P),
                "queries": [q.name for q in qs], "edges_per_step": int(sum(E)),
                "parallelism": ("partitioned" if partitioned else "replicas") if world > 1 else "single",
                "devices": n_dev, "oversubscribed": oversub})
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if partitioned else "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic", "config": cfg, "workload_info": info,
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(3 * 4 * len(s_h)),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": 1000 * e2e_s,
                    "stages_ms": {k: statistics.median(v) for k, v in stages.items()}, "aggregate": "median over e2e steps"},
            "gpu_launches": int(launches_per_step * args.steps),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "edges_read": {"per_step": int(edges_read), "per_s": edges_read / (ms / 1000),
                           "definition": "SURVEY §8(d): LSpM entries read whose label matched (seed + filter + "
                                         "push + expansion device counters)"},
            "batch_latency_ms": ms,
            # SURVEY §8(d) NVLink term: per group, every rank receives the other ranks'
            # bitmap slices ((P-1)/P * N/8 bytes); against the measured 770 GB/s peer
            # copy per direction (B200_PROFILING.md).  0 at N = 1.
            "nvlink": {"bytes_per_step_per_rank": int(xchg_bytes),
                       "achieved_GBps": xchg_bytes / (ms / 1000) / 1e9, "peak_GBps": 770.0,
                       "frac": xchg_bytes / (ms / 1000) / 1e9 / 770.0,
                       "peak_source": "B200_PROFILING.md measured peer copy per direction"},
            "build": {"ms": build_ms, "triples_per_s": len(s_h) / (build_ms / 1000)},
            "kernel_classes": per_class,
            "queries": per_query}
    if rank == 0:
        print(json.dumps(line), flush=True)
    for pl in plans:
        G.gsmart_plan_free(pl)
    eng.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
