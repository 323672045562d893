"""world > 1: 1-D vertex-range partition of the candidate
bitmaps, all-gather after each grouped evaluation, rank-local tries, rows
gathered to rank 0.

CPU (gloo, world_size 2): the host-side logic — the partition helper and the
NCCL-id bootstrap over torch.distributed.  GPU: world = 2, 3 ranks as threads
on one device through the in-process communicator, rows equal to the oracle.
"""
import os
import threading

import numpy as np
import pytest


def _G():
    from conftest import build_product
    build_product()
    import paper_2106_14038_b200.gsmart as g
    return g


@pytest.mark.parametrize("n", [1, 31, 32, 33, 1000, 4263473, 328_600_000])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_words_tiles_the_bitmap(n, world):
    G = _G()
    W = (n + 31) // 32
    ranges = [G.gsmart_partition_words(n, world, r) for r in range(world)]
    covered = []
    for lo, hi in ranges:
        assert (lo % 32 == 0 or lo == hi == W) and lo <= hi <= W
        covered += list(range(lo, hi)) if W < 10000 else [lo, hi]
    if W < 10000:
        assert covered == list(range(W))
    else:
        assert ranges[0][0] == 0 and ranges[-1][1] == W
        assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    G = _G()
    obj = [G.gsmart_get_nccl_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    nid = obj[0]
    n = 4263473
    lo, hi = G.gsmart_partition_words(n, world, rank)
    got = [None] * world
    dist.all_gather_object(got, (lo, hi, nid))
    ok = len(nid) == 128 and all(g[2] == nid for g in got)
    ok = ok and got[0][0] == 0 and got[-1][1] == (n + 31) // 32
    ok = ok and all(got[i][1] == got[i + 1][0] for i in range(world - 1))
    dist.destroy_process_group()
    q.put((rank, ok))


def test_gloo_bootstrap_world2():
    """NCCL unique id from rank 0 reaches every rank over torch.distributed
    (gloo); the ranks' word ranges tile the bitmap."""
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_virtual_ranks_match_oracle(world):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    G = _G()
    from synth import lubm, fixtures
    from oracle.coracle import OracleIndex
    d = lubm.generate(3)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    ix = OracleIndex(s, p, o)
    qs = lubm.queries(d) + [fixtures.fig2_query()]
    comm = G.gsmart_comm_create_local(world)
    out = {}
    errs = []

    def worker(rank):
        try:
            eng = G.Engine(0, rank=rank, world=world, local_comm=comm)
            eng.load(s, p, o, d.n_entities, d.n_predicates)
            res = []
            for q in qs[:-1]:
                with eng.plan(q) as pl:
                    r = G.gsmart_execute(eng.ctx, pl.h, 0)
                    n = G.gsmart_result_shape(r)[0]
                    rows = G.gsmart_result_rows(r) if rank == 0 else None
                    st = G.gsmart_result_stats(r)
                    G.gsmart_result_free(r)
                res.append((n, rows, st["allgather_bytes"]))
            out[rank] = res
            eng.close()
        except Exception as e:  # noqa: BLE001
            errs.append((rank, repr(e)))

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    G.gsmart_comm_destroy(comm)
    assert not errs, errs
    for i, q in enumerate(qs[:-1]):
        exp = ix.query(q)
        n0, rows0, _ = out[0][i]
        assert rows0.shape == exp.shape and np.array_equal(rows0, exp), q.name
        for r in range(world):
            assert out[r][i][0] == len(exp)  # every rank reports the global count
