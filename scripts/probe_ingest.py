"""f4 measurement: device N-Triples ingest (parse + dictionary encode) of a
fixed-width synthetic document rendered from a seeded power-law triple set
(synth/ntriples.render_ids), timed with CUDA events from a device-resident
text (kernel path) and from pageable host bytes (e2e, H2D inside the timed
region).  Ids are checked against the first-appearance closed form (terms
carry their source ids, so the expected ids are the first-appearance ranks,
computed here with torch on the device), term bytes on a sample.

    python scripts/probe_ingest.py --triples 20000000
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--triples", type=int, default=20_000_000)
ap.add_argument("--entities", type=int, default=4_000_000)
ap.add_argument("--predicates", type=int, default=1000)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()

import paper_2106_14038_b200 as G  # noqa: E402
from synth import powerlaw, ntriples as SN  # noqa: E402

t0 = time.perf_counter()
d = powerlaw.generate(args.triples, n_entities=args.entities, n_predicates=args.predicates, device="cuda")
s, p, o = (x.cpu().numpy() for x in (d.s, d.p, d.o))
doc = SN.render_ids(s, p, o)
print(f"rendered {len(doc) / 1e9:.2f} GB, {args.triples} triples in {time.perf_counter() - t0:.1f}s", flush=True)

dev = torch.device("cuda", 0)
text_d = torch.frombuffer(bytearray(doc), dtype=torch.uint8).to(dev)
eng = G.Engine(0)
st = torch.cuda.current_stream(dev)


def timed(buf):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    r = G.gsmart_ingest_ntriples(eng.ctx, buf)
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1), r


timed(text_d)
dev_ms = []
for _ in range(args.reps):
    ms, (n, N, P) = timed(text_d)
    dev_ms.append(ms)
host_ms = []
for _ in range(max(2, args.reps // 2)):
    ms, _ = timed(doc)
    host_ms.append(ms)

# closed form: first-appearance ranks of the source ids
gs, gp, go = (torch.from_numpy(a.astype(np.int64)).to(dev) for a in G.gsmart_triples_get(eng.ctx))
src_s, src_p, src_o = (torch.from_numpy(a.astype(np.int64)).to(dev) for a in (s, p, o))


def first_rank(x):
    u, inv = torch.unique(x, return_inverse=True)
    first = torch.full((u.numel(),), x.numel(), dtype=torch.int64, device=dev)
    first.scatter_reduce_(0, inv, torch.arange(x.numel(), device=dev), reduce="amin")
    order = torch.argsort(first)
    rank = torch.empty_like(order)
    rank[order] = torch.arange(order.numel(), device=dev)
    return rank[inv]


ent = first_rank(torch.stack([src_s, src_o], 1).reshape(-1)).view(-1, 2)
ok = bool(torch.equal(gs, ent[:, 0]) and torch.equal(go, ent[:, 1]) and torch.equal(gp, first_rank(src_p) + 1))
rng = np.random.default_rng(0)
for i in rng.integers(0, args.triples, 50):
    t = G.gsmart_dict_term(eng.ctx, G.GSMART_DICT_ENTITY, int(gs[i]))
    ok = ok and int(t[-10:-1]) == int(s[i])
gb = len(doc) / 1e9
md, mh = statistics.median(dev_ms), statistics.median(host_ms)
print(f"ingest triples={n} entities={N} predicates={P} ids_match={ok}", flush=True)
print(f"device text: median {md:.1f} ms  {gb / (md / 1e3):.1f} GB/s  {n / (md / 1e3) / 1e6:.1f} M triples/s  "
      f"runs={['%.1f' % x for x in dev_ms]}", flush=True)
print(f"host text (e2e, H2D inside): median {mh:.1f} ms  {gb / (mh / 1e3):.1f} GB/s  "
      f"{n / (mh / 1e3) / 1e6:.1f} M triples/s", flush=True)
G.gsmart_build_lspm(eng.ctx)
eng.close()
