"""world > 1: the LSpM is 1-D vertex-range
partitioned (rank r stores only the CSR/CSC rows of its nnz-balanced range,
in symmetric device memory every rank maps), candidate bitmaps are exchanged
by the filter's own peer atomics (or, baseline, an all-gather), tries stay
rank-local, rows are gathered to rank 0.

CPU (no device): the partition split helper, and — world_size 2 over gloo —
the NCCL/unique-id bootstrap plus the ranks-as-processes channel (socket
rendezvous, host all-gather, file-descriptor exchange).  GPU: ranks as threads
on one device (in-process communicator) at world 2, 3 and 8; ranks as two
processes on one device (socket rendezvous + VMM handle exchange); a 1-rank
NCCL communicator running the baseline exchange calls.
"""
import os
import threading

import numpy as np
import pytest

ALIGN = 1 << 19


def _G():
    from conftest import build_product
    build_product()
    import paper_2106_14038_b200.gsmart as g
    return g


def _split_ref(bucket, n, world):
    """the documented rule, restated: split r = first bucket boundary where the
    running total reaches ceil(r * total / world)"""
    tot = int(np.sum(bucket))
    cum = np.concatenate([[0], np.cumsum(bucket)])
    v = [0]
    for r in range(1, world):
        target = -(-tot * r // world)
        b = int(np.searchsorted(cum, target, side="left"))
        v.append(min(b * ALIGN, n))
    return v + [n]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("kind", ["uniform", "hub", "empty", "tail"])
def test_partition_split(world, kind):
    G = _G()
    rng = np.random.default_rng(world * 7 + len(kind))
    for n in (1, ALIGN - 1, ALIGN + 5, 20 * ALIGN + 3, 328_600_000):
        nb = (n + ALIGN - 1) // ALIGN
        if kind == "uniform":
            b = rng.integers(1000, 2000, nb)
        elif kind == "hub":
            b = rng.integers(0, 10, nb)
            b[rng.integers(0, nb)] = 10 ** 9
        elif kind == "empty":
            b = np.zeros(nb, dtype=np.int64)
        else:
            b = np.zeros(nb, dtype=np.int64)
            b[-1] = 5
        v = G.gsmart_partition_split(b, n, world)
        assert v == _split_ref(b, n, world), (n, kind)
        assert v[0] == 0 and v[-1] == n and all(v[i] <= v[i + 1] for i in range(world))
        assert all(x % ALIGN == 0 or x == n for x in v[:-1])
        if kind == "uniform" and nb >= 4 * world:  # balance within one bucket of the ideal share
            loads = [int(b[v[r] // ALIGN:(v[r + 1] + ALIGN - 1) // ALIGN].sum()) for r in range(world)]
            assert max(loads) <= b.sum() / world + b.max() + 1
    with pytest.raises(G.GsmartError):
        G.gsmart_partition_split([1, 2], ALIGN * 5, 2)  # wrong bucket count


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    G = _G()
    obj = [G.gsmart_get_nccl_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    nid = obj[0]
    ok = len(nid) == 128
    # the ranks-as-processes channel: rendezvous on the id, host all-gather, fd passing
    vals = G.gsmart_rendezvous_check(nid, rank, world, 1000 + rank)
    ok = ok and vals == [1000 + r for r in range(world)]
    # every rank derives the same split points from the same histogram
    b = np.arange(1, 41, dtype=np.uint64)
    v = G.gsmart_partition_split(b, 40 * ALIGN, world)
    got = [None] * world
    dist.all_gather_object(got, (v, nid))
    ok = ok and all(g[0] == v and g[1] == nid for g in got)
    dist.destroy_process_group()
    q.put((rank, ok))


def test_gloo_bootstrap_world2():
    """world_size 2 on CPU (gloo): the unique id from rank 0 reaches every rank
    over torch.distributed; the socket rendezvous named by it all-gathers host
    values and hands each rank the other's file descriptor (the path of the
    symmetric chunks' handles); split points agree."""
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
    res = dict(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


# ---------------------------------------------------------------------- GPU
def _lubm_case(U):
    from synth import lubm, fixtures
    from oracle.coracle import OracleIndex
    d = lubm.generate(U)
    s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
    return d, s, p, o, OracleIndex(s, p, o), lubm.queries(d) + [fixtures.fig2_query()]


def _threads(G, world, s, p, o, N, P, qs, exchange, flags=0, batch=False):
    comm = G.gsmart_comm_create_local(world)
    out, errs = {}, []

    def worker(rank):
        try:
            eng = G.Engine(0, rank=rank, world=world, local_comm=comm, exchange=exchange)
            eng.load(s, p, o, N, P)
            v = G.gsmart_partition_get(eng.ctx, world)
            nnz = [G.gsmart_lspm_get(eng.ctx, f)["nnz"] for f in (G.GSMART_CSR, G.GSMART_CSC)]
            res = []
            plans = [G.gsmart_plan(eng.ctx, q) for q in qs]
            for rep in range(2):  # the second pass replays graphs and speculates
                rs = G.gsmart_execute_batch(eng.ctx, plans, flags) if batch else \
                    [G.gsmart_execute(eng.ctx, pl, flags) for pl in plans]
                cur = []
                for r in rs:
                    n = G.gsmart_result_shape(r)[0]
                    rows = G.gsmart_result_rows(r) if rank == 0 else None
                    st = G.gsmart_result_stats(r)
                    G.gsmart_result_free(r)
                    cur.append((n, rows, st))
                res.append(cur)
            for pl in plans:
                G.gsmart_plan_free(pl)
            out[rank] = (v, nnz, res)
            eng.close()
        except Exception as e:  # noqa: BLE001
            errs.append((rank, repr(e)))

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=900)
    G.gsmart_comm_destroy(comm)
    assert not errs, errs
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("world,exchange", [(2, 0), (3, 0), (8, 0), (2, 1)])
def test_virtual_ranks_match_oracle(world, exchange):
    """Ranks as threads on one device: the partitioned LSpM (each rank stores
    only its rows; split points nnz-balanced, 2^19-aligned), the peer exchange
    (exchange 0: filters clear bits on every rank's copy, device barriers) or
    the baseline all-gather (exchange 1); rank 0's rows == C oracle, every rank
    reports the global count, twice (graph replay + speculation)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    G = _G()
    d, s, p, o, ix, qs = _lubm_case(100)   # 4.26M entities: several 2^19-vertex buckets per rank
    out = _threads(G, world, s, p, o, d.n_entities, d.n_predicates, qs, exchange)
    v0 = out[0][0]
    assert v0[0] == 0 and v0[-1] == d.n_entities and all(v0[i] <= v0[i + 1] for i in range(world))
    assert sum(v0[i] < v0[i + 1] for i in range(world)) >= 2  # really partitioned (a rank may own none)
    for r in range(world):
        assert out[r][0] == v0
        assert out[r][1] == out[0][1]
    for rep in range(2):
        for i, q in enumerate(qs):
            exp = ix.query(q)
            n0, rows0, st0 = out[0][2][rep][i]
            assert rows0.shape == exp.shape and np.array_equal(rows0, exp), (q.name, rep)
            for r in range(world):
                assert out[r][2][rep][i][0] == len(exp), (q.name, r)


@pytest.mark.gpu
def test_virtual_ranks_equal_single_gpu_bitmaps():
    """Byte identity of world 1 and world 4: the candidate bitmaps each rank
    ends with (replicated) equal the single-GPU bitmaps for every variable."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    G = _G()
    d, s, p, o, ix, qs = _lubm_case(100)
    e1 = G.Engine(0)
    e1.load(s, p, o, d.n_entities, d.n_predicates)
    ref = {}
    for q in qs:
        with e1.plan(q) as pl:
            r = G.gsmart_execute(e1.ctx, pl.h, G.GSMART_KEEP_CANDIDATES)
            for v in q.variables:
                ptr, nw = G.gsmart_result_candidates(r, v)
                ref[(q.name, v)] = G.gsmart_copy_to_host(e1.ctx, ptr, nw * 4)
            G.gsmart_result_free(r)
    e1.close()
    world = 4
    comm = G.gsmart_comm_create_local(world)
    got, errs = {}, []

    def worker(rank):
        try:
            eng = G.Engine(0, rank=rank, world=world, local_comm=comm)
            eng.load(s, p, o, d.n_entities, d.n_predicates)
            for q in qs:
                with eng.plan(q) as pl:
                    r = G.gsmart_execute(eng.ctx, pl.h, G.GSMART_KEEP_CANDIDATES)
                    for v in q.variables:
                        ptr, nw = G.gsmart_result_candidates(r, v)
                        got[(rank, q.name, v)] = G.gsmart_copy_to_host(eng.ctx, ptr, nw * 4)
                    G.gsmart_result_free(r)
            eng.close()
        except Exception as e:  # noqa: BLE001
            errs.append((rank, repr(e)))

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=900)
    G.gsmart_comm_destroy(comm)
    assert not errs, errs
    for (name, v), bits in ref.items():
        for rank in range(world):
            assert np.array_equal(got[(rank, name, v)], bits), (rank, name, v)


def _proc_worker(rank, world, nid, q):
    try:
        G = _G()
        from synth import lubm
        from oracle.coracle import OracleIndex
        d = lubm.generate(100)
        s, p, o = d.s.numpy(), d.p.numpy(), d.o.numpy()
        eng = G.Engine(0, rank=rank, world=world, nccl_id=nid)
        eng.load(s, p, o, d.n_entities, d.n_predicates)
        qs = lubm.queries(d)
        ok = True
        ix = OracleIndex(s, p, o) if rank == 0 else None
        for qq in qs:
            with eng.plan(qq) as pl:
                r = G.gsmart_execute(eng.ctx, pl.h, 0)
                n = G.gsmart_result_shape(r)[0]
                if rank == 0:
                    exp = ix.query(qq)
                    ok = ok and np.array_equal(G.gsmart_result_rows(r), exp)
                G.gsmart_result_free(r)
        eng.close()
        q.put((rank, ok, ""))
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, repr(e)))


@pytest.mark.gpu
def test_two_processes_one_device():
    """Ranks as PROCESSES (the bench's torchrun layout) on one device: socket
    rendezvous, symmetric chunks exchanged as POSIX file descriptors and mapped
    by cuMemMap, peer-atomic exchange with cross-process device barriers;
    rank 0's rows == C oracle."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import multiprocessing as mp
    G = _G()
    nid = G.gsmart_get_nccl_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_proc_worker, args=(r, 2, nid, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in ps:
        r, ok, err = q.get(timeout=900)
        res[r] = (ok, err)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: (True, ""), 1: (True, "")}, res


@pytest.mark.gpu
def test_nccl_world1_communicator():
    """A 1-rank NCCL communicator (created from a unique id) runs the baseline
    exchange's NCCL calls (grouped broadcasts) after every group evaluation;
    rows stay equal to the oracle."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    G = _G()
    d, s, p, o, ix, qs = _lubm_case(3)
    eng = G.Engine(0, nccl_id=G.gsmart_get_nccl_id())
    eng.load(s, p, o, d.n_entities, d.n_predicates)
    for q in qs:
        rows, st = eng.query(q, with_stats=True)
        assert np.array_equal(rows, ix.query(q)), q.name
        with eng.plan(q) as pl:
            n_groups = len(G.gsmart_plan_describe(pl.h)["groups"])
        assert st["launches"]["collective"] >= n_groups, q.name  # one exchange per group evaluation
    eng.close()
