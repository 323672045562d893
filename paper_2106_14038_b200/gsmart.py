"""Thin ctypes binding of include/gsmart.h (argument marshalling only).

Function names match the C ABI one to one.  Every step of the hot path runs
inside libgsmart.so's sm_100a kernels; this module never computes anything
itself and has no fallback: if libgsmart.so is missing, importing it raises.
"""
import ctypes
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgsmart.so")

GSMART_OK = 0
STATUS = {0: "OK", -1: "E_INVALID_ARG", -2: "E_STATE", -3: "E_OOM", -4: "E_CUDA", -5: "E_NCCL",
          -6: "E_UNSUPPORTED", -7: "E_RESULT_OVERFLOW"}
GSMART_PTR_HOST, GSMART_PTR_DEVICE = 1, 2
GSMART_CSR, GSMART_CSC = 1, 2
GSMART_DEGREE, GSMART_DIRECTION = 0, 1
GSMART_COUNT_ONLY, GSMART_KEEP_ON_DEVICE, GSMART_NO_REFINE, GSMART_PROFILE = 1, 2, 4, 8
GSMART_KEEP_CANDIDATES, GSMART_NO_GRAPH = 16, 32
GSMART_NO_SPECULATE = 64
GSMART_BACK_EDGES = 128
GSMART_FACTORISED = 256
GSMART_REFINE = 512
NKERNELS, MAX_LEVELS = 16, 32


class GsmartError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)
GSMART_XCHG_PEER, GSMART_XCHG_NCCL = 0, 1
GSMART_DICT_ENTITY, GSMART_DICT_PREDICATE = 0, 1


class gsmart_config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("rank", ctypes.c_int), ("world", ctypes.c_int),
                ("nccl_unique_id", ctypes.c_void_p), ("stream", ctypes.c_void_p),
                ("max_result_rows", ctypes.c_uint64), ("local_comm", ctypes.c_void_p),
                ("exchange", ctypes.c_uint32), ("alloc", ALLOC_FN), ("free", FREE_FN),
                ("alloc_user", ctypes.c_void_p)]


class gsmart_lspm_view(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_uint32), ("nnz", ctypes.c_uint64), ("pred_bytes", ctypes.c_uint32),
                ("row_ptr", ctypes.c_void_p), ("col", ctypes.c_void_p), ("pred", ctypes.c_void_p),
                ("label_mask", ctypes.c_void_p)]


class gsmart_qvertex(ctypes.Structure):
    _fields_ = [("is_const", ctypes.c_uint32), ("const_id", ctypes.c_uint32)]


class gsmart_qedge(ctypes.Structure):
    _fields_ = [("src", ctypes.c_uint32), ("pred", ctypes.c_uint32), ("dst", ctypes.c_uint32)]


class gsmart_query(ctypes.Structure):
    _fields_ = [("n_vertices", ctypes.c_uint32), ("v", ctypes.POINTER(gsmart_qvertex)),
                ("n_edges", ctypes.c_uint32), ("e", ctypes.POINTER(gsmart_qedge))]


class gsmart_stats(ctypes.Structure):
    _fields_ = [("ms_total", ctypes.c_double), ("ms_kernel", ctypes.c_double * NKERNELS),
                ("launches", ctypes.c_uint64 * NKERNELS), ("bytes", ctypes.c_uint64 * NKERNELS),
                ("edges_evaluated", ctypes.c_uint64), ("filter_rows", ctypes.c_uint64),
                ("filter_entries", ctypes.c_uint64), ("seed_entries", ctypes.c_uint64),
                ("expand_entries", ctypes.c_uint64), ("closing_checks", ctypes.c_uint64),
                ("n_levels", ctypes.c_uint32), ("level_nodes", ctypes.c_uint64 * MAX_LEVELS),
                ("level_alive", ctypes.c_uint64 * MAX_LEVELS), ("allgather_bytes", ctypes.c_uint64),
                ("spec_phase2", ctypes.c_uint32), ("spec_redo", ctypes.c_uint32),
                ("factorised", ctypes.c_uint32), ("n_omega", ctypes.c_uint32), ("combinations", ctypes.c_uint64),
                ("kernel_names", ctypes.c_char_p * NKERNELS)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run paper_2106_14038_b200.build.build() "
                          "(nvcc sm_100a); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    vp, u32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
    st = ctypes.c_int
    sig = {
        "gsmart_abi_version": (ctypes.c_int, []),
        "gsmart_build_info": (ctypes.c_char_p, []),
        "gsmart_get_nccl_id": (st, [vp]),
        "gsmart_create": (st, [ctypes.POINTER(gsmart_config), ctypes.POINTER(vp)]),
        "gsmart_destroy": (None, [vp]),
        "gsmart_last_error": (ctypes.c_char_p, [vp]),
        "gsmart_load_triples": (st, [vp, vp, vp, vp, u64, u32, u32, u32]),
        "gsmart_build_lspm": (st, [vp, vp, u32, u32]),
        "gsmart_build_lspm_split": (st, [vp, vp, u32, vp, u32]),
        "gsmart_plan_keep_sets": (st, [ctypes.POINTER(vp), u32, u32, vp, ctypes.POINTER(u32), vp,
                                       ctypes.POINTER(u32), u32]),
        "gsmart_lspm_get": (st, [vp, u32, ctypes.POINTER(gsmart_lspm_view)]),
        "gsmart_plan": (st, [vp, ctypes.POINTER(gsmart_query), u32, ctypes.POINTER(vp)]),
        "gsmart_plan_describe": (st, [vp, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
        "gsmart_plan_free": (None, [vp]),
        "gsmart_execute": (st, [vp, vp, u32, ctypes.POINTER(vp)]),
        "gsmart_execute_batch": (st, [vp, ctypes.POINTER(vp), u32, u32, ctypes.POINTER(vp)]),
        "gsmart_result_shape": (st, [vp, ctypes.POINTER(u64), ctypes.POINTER(u32),
                                     ctypes.POINTER(ctypes.POINTER(u32))]),
        "gsmart_result_rows": (st, [vp, ctypes.POINTER(ctypes.POINTER(u32))]),
        "gsmart_result_rows_device": (st, [vp, ctypes.POINTER(vp)]),
        "gsmart_result_candidates": (st, [vp, u32, ctypes.POINTER(vp), ctypes.POINTER(u32)]),
        "gsmart_result_level": (st, [vp, u32, ctypes.POINTER(u32), ctypes.POINTER(u64), ctypes.POINTER(vp),
                                     ctypes.POINTER(vp)]),
        "gsmart_result_tree": (st, [vp, u32, ctypes.POINTER(u32), ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(u64),
                                    ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp)]),
        "gsmart_result_stats": (st, [vp, ctypes.POINTER(gsmart_stats)]),
        "gsmart_result_free": (None, [vp]),
        "gsmart_copy_to_host": (st, [vp, vp, vp, ctypes.c_size_t]),
        "gsmart_comm_create_local": (st, [ctypes.c_int, ctypes.POINTER(vp)]),
        "gsmart_comm_destroy": (None, [vp]),
        "gsmart_partition_split": (st, [ctypes.POINTER(u64), u32, u32, ctypes.c_int, ctypes.POINTER(u32)]),
        "gsmart_partition_get": (st, [vp, ctypes.POINTER(u32)]),
        "gsmart_rendezvous_check": (st, [vp, ctypes.c_int, ctypes.c_int, u64, ctypes.POINTER(u64)]),
        "gsmart_ingest_ntriples": (st, [vp, vp, u64, u32, ctypes.POINTER(u64), ctypes.POINTER(u32),
                                        ctypes.POINTER(u32)]),
        "gsmart_dict_lookup": (st, [vp, u32, ctypes.c_char_p, u64, ctypes.POINTER(u32)]),
        "gsmart_dict_term": (st, [vp, u32, u32, vp, u64, ctypes.POINTER(u64)]),
        "gsmart_triples_get": (st, [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                    ctypes.POINTER(u64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()
EXPORTED = ["gsmart_abi_version", "gsmart_build_info", "gsmart_get_nccl_id", "gsmart_create", "gsmart_destroy",
            "gsmart_last_error", "gsmart_load_triples", "gsmart_build_lspm", "gsmart_build_lspm_split",
            "gsmart_plan_keep_sets", "gsmart_lspm_get", "gsmart_plan",
            "gsmart_plan_describe", "gsmart_plan_free", "gsmart_execute", "gsmart_execute_batch",
            "gsmart_result_shape",
            "gsmart_result_rows", "gsmart_result_rows_device", "gsmart_result_candidates",
            "gsmart_result_level", "gsmart_result_tree", "gsmart_result_stats", "gsmart_result_free", "gsmart_copy_to_host",
            "gsmart_comm_create_local", "gsmart_comm_destroy", "gsmart_partition_split", "gsmart_partition_get",
            "gsmart_rendezvous_check", "gsmart_ingest_ntriples", "gsmart_dict_lookup", "gsmart_dict_term",
            "gsmart_triples_get"]


def lib():
    return _lib


def _check(status, ctx=None):
    if status != GSMART_OK:
        msg = _lib.gsmart_last_error(ctx)
        raise GsmartError(status, msg.decode() if msg else "")


# ------------------------------------------------------------------------ ABI mirrors
def gsmart_abi_version():
    return _lib.gsmart_abi_version()


def gsmart_build_info():
    return _lib.gsmart_build_info().decode()


def gsmart_get_nccl_id():
    buf = ctypes.create_string_buffer(128)
    _check(_lib.gsmart_get_nccl_id(buf))
    return buf.raw


def gsmart_create(device=0, rank=0, world=1, nccl_id=None, stream=None, max_result_rows=0, local_comm=None,
                  exchange=GSMART_XCHG_PEER, alloc=None, free=None):
    """alloc/free: optional ALLOC_FN / FREE_FN callbacks (keep them alive while the ctx lives)."""
    cfg = gsmart_config()
    cfg.exchange = exchange
    if alloc is not None:
        cfg.alloc, cfg.free = alloc, free
    cfg.local_comm = local_comm.value if isinstance(local_comm, ctypes.c_void_p) else local_comm
    cfg.device, cfg.rank, cfg.world = device, rank, world
    idbuf = None
    if nccl_id is not None:
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        cfg.nccl_unique_id = ctypes.cast(idbuf, ctypes.c_void_p)
    cfg.stream = stream
    cfg.max_result_rows = max_result_rows
    h = ctypes.c_void_p()
    _check(_lib.gsmart_create(ctypes.byref(cfg), ctypes.byref(h)))
    return h


def gsmart_comm_create_local(world):
    h = ctypes.c_void_p()
    _check(_lib.gsmart_comm_create_local(world, ctypes.byref(h)))
    return h


def gsmart_comm_destroy(comm):
    _lib.gsmart_comm_destroy(comm)


PART_ALIGN_ROWS = 1 << 19


def gsmart_partition_split(bucket_counts, n_entities, world):
    """Split points v[0..world] of the nnz-balanced vertex-range partition."""
    b = np.ascontiguousarray(np.asarray(bucket_counts, dtype=np.uint64))
    v = (ctypes.c_uint32 * (world + 1))()
    _check(_lib.gsmart_partition_split(b.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)) if len(b) else None,
                                       len(b), int(n_entities), world, v))
    return [v[i] for i in range(world + 1)]


def gsmart_rendezvous_check(id128, rank, world, value):
    buf = ctypes.create_string_buffer(bytes(id128), 128)
    out = (ctypes.c_uint64 * world)()
    _check(_lib.gsmart_rendezvous_check(buf, rank, world, value, out))
    return [out[i] for i in range(world)]


def gsmart_partition_get(ctx, world):
    v = (ctypes.c_uint32 * (world + 1))()
    _check(_lib.gsmart_partition_get(ctx, v), ctx)
    return [v[i] for i in range(world + 1)]


def gsmart_destroy(ctx):
    _lib.gsmart_destroy(ctx)


def gsmart_last_error(ctx=None):
    m = _lib.gsmart_last_error(ctx)
    return m.decode() if m else ""


def _ptr_kind(a):
    """(pointer, keepalive, kind) for a numpy array / CPU tensor / CUDA tensor of uint32/int32."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.dtype not in (torch.int32,) and str(a.dtype) != "torch.uint32":
                raise TypeError("triple tensors must be int32/uint32")
            a = a.contiguous()  # int32 and uint32 share the bit pattern: ids are checked on the device
            return a.data_ptr(), a, (GSMART_PTR_DEVICE if a.is_cuda else GSMART_PTR_HOST)
    except ImportError:
        pass
    arr = np.ascontiguousarray(np.asarray(a))
    if arr.dtype == np.int32:
        return arr.ctypes.data, arr, GSMART_PTR_HOST  # viewed as uint32; negative ids fail the device check
    if arr.size and arr.dtype != np.uint32:
        if arr.dtype.kind not in "iu":
            raise TypeError("triple arrays must hold integers")
        if arr.min() < 0 or arr.max() >= 2 ** 32:
            raise ValueError("triple ids must lie in [0, 2^32)")  # never wrap silently
    arr = np.ascontiguousarray(arr.astype(np.uint32, copy=False))
    return arr.ctypes.data, arr, GSMART_PTR_HOST


def gsmart_load_triples(ctx, s, p, o, n_entities, n_predicates):
    ps, ks, kind_s = _ptr_kind(s)
    pp, kp, kind_p = _ptr_kind(p)
    po, ko, kind_o = _ptr_kind(o)
    if not (kind_s == kind_p == kind_o):
        raise ValueError("s, p, o must all be host or all be device")
    n = len(ks)
    _check(_lib.gsmart_load_triples(ctx, ps, pp, po, n, int(n_entities), int(n_predicates), kind_s), ctx)


def gsmart_build_lspm(ctx, keep=None, formats=GSMART_CSR | GSMART_CSC):
    keep = np.ascontiguousarray(np.asarray([] if keep is None else keep, dtype=np.uint32))
    ptr = keep.ctypes.data if len(keep) else None
    _check(_lib.gsmart_build_lspm(ctx, ptr, len(keep), formats), ctx)


def gsmart_build_lspm_split(ctx, keep_csr, keep_csc):
    """Query-dependent LSpM: the CSR keeps keep_csr, the CSC keep_csc (predicate ids)."""
    a = np.ascontiguousarray(np.asarray(list(keep_csr), dtype=np.uint32))
    b = np.ascontiguousarray(np.asarray(list(keep_csc), dtype=np.uint32))
    _check(_lib.gsmart_build_lspm_split(ctx, a.ctypes.data if len(a) else None, len(a),
                                        b.ctypes.data if len(b) else None, len(b)), ctx)


def gsmart_plan_keep_sets(plans, flags=0):
    """(csr, csc): the predicate ids each format must keep to execute the plans."""
    n = len(plans)
    arr = (ctypes.c_void_p * max(n, 1))(*[p.value if isinstance(p, ctypes.c_void_p) else p for p in plans])
    cap = 70000
    a = (ctypes.c_uint32 * cap)()
    b = (ctypes.c_uint32 * cap)()
    na, nb = ctypes.c_uint32(), ctypes.c_uint32()
    _check(_lib.gsmart_plan_keep_sets(arr, n, flags, a, ctypes.byref(na), b, ctypes.byref(nb), cap))
    return [a[i] for i in range(na.value)], [b[i] for i in range(nb.value)]


def gsmart_lspm_get(ctx, fmt):
    v = gsmart_lspm_view()
    _check(_lib.gsmart_lspm_get(ctx, fmt, ctypes.byref(v)), ctx)
    return {"n_rows": v.n_rows, "nnz": v.nnz, "pred_bytes": v.pred_bytes, "row_ptr": v.row_ptr,
            "col": v.col, "pred": v.pred, "label_mask": v.label_mask}


def _query_struct(q):
    """q: object with .vertices (None = variable, int = constant id) and .edges [(src, pred, dst)]."""
    verts = list(q.vertices)
    edges = list(q.edges)
    V = (gsmart_qvertex * max(len(verts), 1))()
    for i, c in enumerate(verts):
        V[i].is_const = 0 if c is None else 1
        V[i].const_id = 0 if c is None else min(int(c), 0xFFFFFFFF)
    E = (gsmart_qedge * max(len(edges), 1))()
    for i, (a, l, b) in enumerate(edges):
        E[i].src, E[i].pred, E[i].dst = int(a), int(l), int(b)
    qs = gsmart_query(len(verts), V, len(edges), E)
    return qs, (V, E)


def gsmart_plan(ctx, query, traversal=GSMART_DEGREE):
    qs, keep = _query_struct(query)
    h = ctypes.c_void_p()
    _check(_lib.gsmart_plan(ctx, ctypes.byref(qs), traversal, ctypes.byref(h)), ctx)
    return h


def gsmart_plan_describe(plan):
    need = ctypes.c_size_t(0)
    _check(_lib.gsmart_plan_describe(plan, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(_lib.gsmart_plan_describe(plan, buf, need.value, ctypes.byref(need)))
    return json.loads(buf.value.decode())


def gsmart_plan_free(plan):
    _lib.gsmart_plan_free(plan)


def gsmart_execute(ctx, plan, flags=0):
    h = ctypes.c_void_p()
    st = _lib.gsmart_execute(ctx, plan, flags, ctypes.byref(h))
    if st != GSMART_OK:
        err = GsmartError(st, gsmart_last_error(ctx))
        if h.value:
            n = ctypes.c_uint64()
            _lib.gsmart_result_shape(h, ctypes.byref(n), None, None)
            err.n_rows = n.value
            _lib.gsmart_result_free(h)
        raise err
    return h


def gsmart_execute_batch(ctx, plans, flags=0):
    """Run independent plans concurrently; returns one result handle per plan."""
    n = len(plans)
    arr = (ctypes.c_void_p * max(n, 1))(*[p.value if isinstance(p, ctypes.c_void_p) else p for p in plans])
    out = (ctypes.c_void_p * max(n, 1))()
    _check(_lib.gsmart_execute_batch(ctx, arr, n, flags, out), ctx)
    return [ctypes.c_void_p(out[i]) for i in range(n)]


def gsmart_result_shape(r):
    n = ctypes.c_uint64()
    c = ctypes.c_uint32()
    voc = ctypes.POINTER(ctypes.c_uint32)()
    _check(_lib.gsmart_result_shape(r, ctypes.byref(n), ctypes.byref(c), ctypes.byref(voc)))
    return n.value, c.value, [voc[i] for i in range(c.value)]


def gsmart_result_rows(r, copy=True):
    """Host rows [n_rows, n_cols] uint32.  copy=False returns a view of the
    result's pinned host block, valid until gsmart_result_free(r)."""
    n, c, _ = gsmart_result_shape(r)
    ptr = ctypes.POINTER(ctypes.c_uint32)()
    _check(_lib.gsmart_result_rows(r, ctypes.byref(ptr)))
    if n == 0 or c == 0:
        return np.zeros((n, c), dtype=np.uint32)
    a = np.ctypeslib.as_array(ptr, shape=(n * c,)).reshape(n, c)
    return a.copy() if copy else a


def gsmart_result_rows_device(r):
    p = ctypes.c_void_p()
    _check(_lib.gsmart_result_rows_device(r, ctypes.byref(p)))
    return p.value


def gsmart_result_candidates(r, vertex):
    p = ctypes.c_void_p()
    nw = ctypes.c_uint32()
    _check(_lib.gsmart_result_candidates(r, vertex, ctypes.byref(p), ctypes.byref(nw)))
    return p.value, nw.value


def gsmart_result_level(r, k):
    v = ctypes.c_uint32()
    n = ctypes.c_uint64()
    par = ctypes.c_void_p()
    bnd = ctypes.c_void_p()
    _check(_lib.gsmart_result_level(r, k, ctypes.byref(v), ctypes.byref(n), ctypes.byref(par), ctypes.byref(bnd)))
    return v.value, n.value, par.value, bnd.value


def gsmart_result_tree(r, k):
    """(vertex, parent_level, n, parent_dev, bind_dev, alive_dev) of level k of
    the result's tree form (occurrence k with GSMART_FACTORISED)."""
    v = ctypes.c_uint32()
    pl = ctypes.c_int32()
    n = ctypes.c_uint64()
    par, bnd, alv = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    _check(_lib.gsmart_result_tree(r, k, ctypes.byref(v), ctypes.byref(pl), ctypes.byref(n), ctypes.byref(par),
                                   ctypes.byref(bnd), ctypes.byref(alv)))
    return v.value, pl.value, n.value, par.value, bnd.value, alv.value


def gsmart_result_stats(r):
    s = gsmart_stats()
    _check(_lib.gsmart_result_stats(r, ctypes.byref(s)))
    names = [(s.kernel_names[i] or b"").decode() for i in range(NKERNELS)]
    return {
        "ms_total": s.ms_total,
        "ms_kernel": {names[i]: s.ms_kernel[i] for i in range(NKERNELS)},
        "launches": {names[i]: int(s.launches[i]) for i in range(NKERNELS)},
        "bytes": {names[i]: int(s.bytes[i]) for i in range(NKERNELS)},
        "edges_evaluated": int(s.edges_evaluated), "filter_rows": int(s.filter_rows),
        "filter_entries": int(s.filter_entries), "seed_entries": int(s.seed_entries),
        "expand_entries": int(s.expand_entries), "closing_checks": int(s.closing_checks),
        "n_levels": int(s.n_levels),
        "level_nodes": [int(s.level_nodes[i]) for i in range(s.n_levels)],
        "level_alive": [int(s.level_alive[i]) for i in range(s.n_levels)],
        "allgather_bytes": int(s.allgather_bytes),
        "spec_phase2": int(s.spec_phase2), "spec_redo": int(s.spec_redo),
        "factorised": int(s.factorised), "n_omega": int(s.n_omega), "combinations": int(s.combinations),
    }


def gsmart_result_free(r):
    _lib.gsmart_result_free(r)


def gsmart_copy_to_host(ctx, dev_ptr, nbytes, dtype=np.uint32):
    out = np.empty(nbytes // np.dtype(dtype).itemsize, dtype=dtype)
    if nbytes:
        _check(_lib.gsmart_copy_to_host(ctx, out.ctypes.data, dev_ptr, nbytes), ctx)
    return out


def gsmart_ingest_ntriples(ctx, text):
    """Parse + dictionary-encode an N-Triples document on the device and load
    it (f4).  text: bytes / bytearray / numpy uint8 (host) or a CUDA uint8
    tensor.  Returns (n_triples, n_entities, n_predicates)."""
    kind, keep = GSMART_PTR_HOST, None
    try:
        import torch
        if isinstance(text, torch.Tensor):
            if text.dtype != torch.uint8:
                raise TypeError("text tensor must be uint8")
            keep = text.contiguous()
            ptr, n = keep.data_ptr(), keep.numel()
            kind = GSMART_PTR_DEVICE if keep.is_cuda else GSMART_PTR_HOST
    except ImportError:
        pass
    if keep is None:
        keep = np.frombuffer(text, dtype=np.uint8) if isinstance(text, (bytes, bytearray, memoryview)) \
            else np.ascontiguousarray(text, dtype=np.uint8)
        ptr, n = (keep.ctypes.data if keep.size else None), keep.size
    nt, ne, npr = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint32()
    _check(_lib.gsmart_ingest_ntriples(ctx, ptr, n, kind, ctypes.byref(nt), ctypes.byref(ne), ctypes.byref(npr)), ctx)
    return nt.value, ne.value, npr.value


def gsmart_dict_lookup(ctx, kind, term):
    """Id of a term (bytes) or 0xFFFFFFFF when absent."""
    out = ctypes.c_uint32()
    _check(_lib.gsmart_dict_lookup(ctx, kind, bytes(term), len(term), ctypes.byref(out)), ctx)
    return out.value


def gsmart_dict_term(ctx, kind, term_id):
    """Bytes of the term with this id."""
    n = ctypes.c_uint64()
    _check(_lib.gsmart_dict_term(ctx, kind, term_id, None, 0, ctypes.byref(n)), ctx)
    buf = ctypes.create_string_buffer(max(n.value, 1))
    _check(_lib.gsmart_dict_term(ctx, kind, term_id, buf, n.value, ctypes.byref(n)), ctx)
    return buf.raw[:n.value]


def gsmart_triples_get(ctx):
    """Host copies of the loaded (s, p, o) id arrays."""
    s, p, o, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_uint64()
    _check(_lib.gsmart_triples_get(ctx, ctypes.byref(s), ctypes.byref(p), ctypes.byref(o), ctypes.byref(n)), ctx)
    return tuple(gsmart_copy_to_host(ctx, a.value, 4 * n.value) for a in (s, p, o))


# ------------------------------------------------------------------------ convenience
class Engine:
    """One context: load -> build -> query.  Thin sugar over the functions above."""

    def __init__(self, device=0, rank=0, world=1, nccl_id=None, stream=None, max_result_rows=0, local_comm=None,
                 exchange=GSMART_XCHG_PEER, alloc=None, free=None):
        self._hooks = (alloc, free)  # the C side holds raw function pointers
        self.ctx = gsmart_create(device, rank, world, nccl_id, stream, max_result_rows, local_comm, exchange,
                                 alloc, free)
        self.rank, self.world = rank, world

    def load(self, s, p, o, n_entities, n_predicates, keep=None):
        gsmart_load_triples(self.ctx, s, p, o, n_entities, n_predicates)
        gsmart_build_lspm(self.ctx, keep)

    def plan(self, q, traversal=GSMART_DEGREE):
        return Plan(self, q, traversal)

    def query_batch(self, queries, flags=0, traversal=GSMART_DEGREE):
        """Execute several queries concurrently (gsmart_execute_batch); returns rows per query."""
        plans = [Plan(self, q, traversal) for q in queries]
        try:
            res = gsmart_execute_batch(self.ctx, [p.h for p in plans], flags)
            out = []
            for r in res:
                try:
                    if flags & GSMART_COUNT_ONLY:
                        out.append(gsmart_result_shape(r)[0])
                    elif flags & GSMART_KEEP_ON_DEVICE:
                        out.append(None)
                    else:
                        out.append(gsmart_result_rows(r))
                finally:
                    gsmart_result_free(r)
            return out
        finally:
            for p in plans:
                p.close()

    def query(self, q, flags=0, with_stats=False, traversal=GSMART_DEGREE):
        with self.plan(q, traversal) as pl:
            return pl.run(flags, with_stats)

    def close(self):
        if self.ctx:
            gsmart_destroy(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Plan:
    def __init__(self, eng, q, traversal=GSMART_DEGREE):
        self.eng = eng
        self.h = gsmart_plan(eng.ctx, q, traversal)

    def describe(self):
        return gsmart_plan_describe(self.h)

    def run(self, flags=0, with_stats=False):
        r = gsmart_execute(self.eng.ctx, self.h, flags)
        try:
            if flags & GSMART_COUNT_ONLY:
                rows = gsmart_result_shape(r)[0]
            elif flags & GSMART_KEEP_ON_DEVICE or self.eng.rank != 0:
                rows = None  # with world > 1 the rows live on rank 0
            else:
                rows = gsmart_result_rows(r)
            stats = gsmart_result_stats(r) if with_stats else None
        finally:
            gsmart_result_free(r)
        return (rows, stats) if with_stats else rows

    def close(self):
        if self.h:
            gsmart_plan_free(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
