import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GSMART_TRACE"] = "1"
import numpy as np
import paper_2106_14038_b200.gsmart as G
from synth import lubm
d = lubm.generate(100)
s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
qs = lubm.queries(d)
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
comm = G.gsmart_comm_create_local(world)
errs = []
def worker(rank):
    try:
        eng = G.Engine(0, rank=rank, world=world, local_comm=comm)
        eng.load(s, p, o, d.n_entities, d.n_predicates)
        print("rank", rank, "part", G.gsmart_partition_get(eng.ctx, world), flush=True)
        for q in qs:
            with eng.plan(q) as pl:
                r = G.gsmart_execute(eng.ctx, pl.h, 0)
                n = G.gsmart_result_shape(r)[0]
                G.gsmart_result_free(r)
            print(f"rank {rank} {q.name} rows {n}", flush=True)
        eng.close()
    except Exception as e:
        errs.append((rank, repr(e)))
ts = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
[t.start() for t in ts]; [t.join() for t in ts]
print("errs", errs)
