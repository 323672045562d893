#!/usr/bin/env python
"""Benchmark of the B200 gSmart hot path (BASELINE.json metric: query latency
ms & edges evaluated/sec per LUBM/WatDiv query; HBM GB/s fraction).

Workload (N=1): BASELINE.json configs[1] — LUBM-shaped synthetic, 100
universities (~12.3M triples), the LUBM L1-L7 + Q14-style query batch.

A "step" = one pass of the query batch through gsmart_plan/gsmart_execute
(a2..a9: seeds, grouped incident-edge evaluation, compaction, trie
expansion, pre-pruning, bottom-up pruning, row enumeration + sort) over the
LSpM resident in HBM.  The LSpM build (a1) is timed separately ("build") and
is inside the end-to-end leg ("e2e": host triples -> load -> build -> batch
-> rows on host).

Edges evaluated (the metric's numerator) is a property of the workload, not
of an implementation: E(q) = sum over the patterns of q of the number of
triples carrying that pattern's predicate (the nonzeros the matrix form
p*I (x) A of Eqs. 12-13 touches).  Both arms divide the same E by their time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
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

METRIC = "edges evaluated/s (LUBM query batch)"
UNIT = "edges/s"
WORKLOAD = "LUBM-100 (configs[1]): L1-L7 + Q14 batch, 1 B200"


def workload_name(U):
    if U == 100:
        return WORKLOAD
    tag = "configs[3]" if U == 10000 else "LUBM-shaped"
    return f"LUBM-{U} ({tag}): L1-L7 + Q14 batch, 1 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--universities", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--mode", default="replicas", choices=["replicas", "partitioned"],
                    help="N>1: replicas = every GPU serves its own copy of the batch (weak scaling); "
                         "partitioned = one batch over a 1-D vertex-range partition with NCCL all-gathers")
    return ap.parse_args()


def workload(U, device="cpu"):
    from synth import lubm
    seed = lubm.SEED_LUBM100 if U == 100 else lubm.SEED_LUBM10K
    d = lubm.generate(U, seed=seed, device=device)
    return d, lubm.queries(d)


def edges_evaluated(p_np, queries, dedup_counts):
    """E(q) per query (see module doc)."""
    return [int(sum(dedup_counts.get(l, 0) for _, l, _ in q.edges)) for q in queries]


def label_counts_torch(s, p, o):
    """De-duplicated triple count per predicate (input statistics; torch, any device)."""
    import torch
    out = {}
    key = (s.long() << 32) | o.long()
    for l in torch.unique(p).tolist():
        out[int(l)] = int(torch.unique(key[p == l]).numel())
    return out


def label_counts(s, p, o):
    """De-duplicated triple count per predicate (input statistics, host numpy)."""
    order = np.lexsort((o, p, s))
    ss, pp, oo = s[order], p[order], o[order]
    first = np.ones(len(ss), dtype=bool)
    first[1:] = (ss[1:] != ss[:-1]) | (pp[1:] != pp[:-1]) | (oo[1:] != oo[:-1])
    lab, cnt = np.unique(pp[first], return_counts=True)
    return {int(a): int(b) for a, b in zip(lab, cnt)}


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
                                          "--format=csv,noheader,nounits", "-lms", "100"],
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


def ncu_traffic(kernel_class, U=100):
    """DRAM bytes per launch of a kernel class from the committed ncu capture of
    the same workload (profiles/ncu_traffic.json is LUBM-100; other sizes use
    profiles/ncu_traffic_u<U>.json when one was captured, else null)."""
    name = "ncu_traffic.json" if U == 100 else f"ncu_traffic_u{U}.json"
    path = os.path.join(ROOT, "profiles", name)
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(kernel_class)
        return None if e is None else e.get("dram_bytes_per_launch")
    except Exception:
        return None


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle.coracle import OracleIndex
    d, qs = workload(args.universities)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    E = edges_evaluated(p, qs, label_counts(s, p, o))
    ix = OracleIndex(s, p, o)
    cores = len(os.sched_getaffinity(0))
    for _ in range(args.warmup):
        for q in qs:
            ix.query(q, n_threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        for q in qs:
            ix.query(q, n_threads=cores)
        times.append(time.perf_counter() - t0)
    ms = 1000 * statistics.mean(times)
    value = sum(E) / (ms / 1000)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": workload_name(args.universities), "queries": [q.name for q in qs], "triples": int(len(s)),
                       "edges_per_step": int(sum(E))},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": "full LUBM-100 query batch per step (oracle index build excluded)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2106_14038_b200 as G

    # inputs: generated on the host (numpy, for the e2e leg) and resident in HBM
    # counter-based generator: identical triples on any device; generate in HBM
    d, qs = workload(args.universities, device=dev)
    s_d, p_d, o_d = d.s, d.p, d.o
    E = edges_evaluated(None, qs, label_counts_torch(s_d, p_d, o_d))
    s_h, p_h, o_h = s_d.cpu().numpy(), p_d.cpu().numpy(), o_d.cpu().numpy()
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
    G.gsmart_load_triples(eng.ctx, s_d, p_d, o_d, d.n_entities, d.n_predicates)
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
    plans = [G.gsmart_plan(eng.ctx, q) for q in qs]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step(flags=0, stats=None):
        # the query batch runs concurrently (gsmart_execute_batch: one stream + workspace per query)
        for r in G.gsmart_execute_batch(eng.ctx, plans, flags | G.GSMART_KEEP_ON_DEVICE):
            if stats is not None:
                stats.append(G.gsmart_result_stats(r))
            G.gsmart_result_free(r)

    def latency(q_idx, reps=7):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            r = G.gsmart_execute(eng.ctx, plans[q_idx], G.GSMART_KEEP_ON_DEVICE)
            ts.append(1000 * (time.perf_counter() - t0))
            G.gsmart_result_free(r)
        return statistics.median(ts)

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
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.barrier()
        ms = float(t.item())
    value = copies * sum(E) / (ms / 1000)

    # ---- profiled pass: the same queries one at a time (GSMART_PROFILE: per-kernel-class
    # CUDA events on the launching stream; sequential so no other stream shares the GPU)
    prof_stats = []
    for _ in range(args.steps):
        flush.fill_(1)
        for pl in plans:
            r = G.gsmart_execute(eng.ctx, pl, G.GSMART_PROFILE | G.GSMART_KEEP_ON_DEVICE)
            prof_stats.append(G.gsmart_result_stats(r))
            G.gsmart_result_free(r)
    torch.cuda.synchronize()
    ksum, kbytes, klaunch = {}, {}, {}
    # SURVEY §8(d)'s implementation-side count: LSpM entries the GPU path read
    # whose label matched (seed + filter + expansion device counters), per batch
    edges_read = sum(st["edges_evaluated"] for st in prof_stats) / max(1, args.steps)
    for st in prof_stats:
        for k, v in st["ms_kernel"].items():
            ksum[k] = ksum.get(k, 0.0) + v
        for k, v in st["bytes"].items():
            kbytes[k] = kbytes.get(k, 0) + v
        for k, v in st["launches"].items():
            klaunch[k] = klaunch.get(k, 0) + v
    measured_kernels = {k: v for k, v in ksum.items() if kbytes.get(k, 0) > 0 and v > 0}
    dom = max(measured_kernels, key=lambda k: ksum[k]) if measured_kernels else None
    peak, peak_src = peaks()
    roofline = None
    if dom:
        n_launch = max(1, klaunch[dom])
        achieved = kbytes[dom] / (ksum[dom] / 1000) / 1e9
        traffic = ncu_traffic(dom, args.universities)
        roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "algorithmic_bytes_per_launch": kbytes[dom] / n_launch,
                    "ms_share_of_step": ksum[dom] / max(1e-9, sum(ksum.values())),
                    "peak_source": peak_src}
    launches_per_step = sum(sum(st["launches"].values()) for st in prof_stats) / max(1, len(prof_stats) // len(qs))
    per_query = {}
    for i, q in enumerate(qs):
        per_query[q.name] = {"latency_ms": latency(i),  # alone, host wall time of gsmart_execute
                             "rows": None, "edges": E[i]}

    # ---- e2e: host triples -> load -> build -> batch -> rows on host
    e2e_times = []
    d2h = 0
    for it in range(args.e2e_steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        G.gsmart_load_triples(eng.ctx, s_h, p_h, o_h, d.n_entities, d.n_predicates)
        G.gsmart_build_lspm(eng.ctx)
        nbytes = 0
        for q in qs:
            rows = eng.query(q)
            if rows is not None:  # partitioned: rows on rank 0
                nbytes += rows.nbytes
                if it == 0:
                    per_query[q.name]["rows"] = int(rows.shape[0])
        torch.cuda.synchronize()
        if it:
            e2e_times.append(time.perf_counter() - t0)
        d2h = nbytes
    e2e_s = statistics.mean(e2e_times)
    e2e_value = copies * sum(E) / e2e_s

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.universities <= 200:
        from oracle.coracle import OracleIndex
        ix = OracleIndex(s_h, p_h, o_h)
        cores = len(os.sched_getaffinity(0))
        t0 = time.perf_counter()
        reps = 0
        while time.perf_counter() - t0 < 10.0 and reps < 50:
            for q in qs:
                ix.query(q, n_threads=cores)
            reps += 1
        cpu_s = (time.perf_counter() - t0) / reps
        cpu = {"value": sum(E) / cpu_s, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"LUBM-100 query batch x{reps} (~10 s), index build excluded",
               "ms_per_batch": 1000 * cpu_s}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if partitioned else "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": workload_name(args.universities), "universities": args.universities, "triples": int(len(s_h)),
                       "entities": d.n_entities, "queries": [q.name for q in qs],
                       "edges_per_step": int(sum(E)), "edges_read_per_step": int(edges_read),
                       "l2": "flushed between timed steps (256 MiB write)",
                       "parallelism": ("partitioned" if partitioned else "replicas") if world > 1 else "single"},
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(3 * 4 * len(s_h)),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": 1000 * e2e_s},
            "gpu_launches": int(launches_per_step * args.steps),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "build": {"ms": build_ms, "triples_per_s": len(s_h) / (build_ms / 1000)},
            "kernel_ms_per_step": {k: v / args.steps for k, v in ksum.items() if v > 0},
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
