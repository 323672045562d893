"""ORACLE (test infrastructure only) — ctypes loader for oracle/liboracle.so
(built from oracle/bgp_oracle.c by `build_oracle()` / __graft_entry__.build())."""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build_oracle(force=False):
    src = os.path.join(_HERE, "bgp_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11",
                               "-o", _SO, src])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(_SO)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        lib.oracle_bgp.restype = ctypes.c_int
        lib.oracle_bgp.argtypes = [u32p, u32p, u32p, ctypes.c_uint64,
                                   ctypes.c_uint32, u32p, u32p,
                                   ctypes.c_uint32, u32p, u32p, u32p,
                                   ctypes.c_int, ctypes.POINTER(u32p),
                                   ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32)]
        lib.oracle_free.argtypes = [ctypes.c_void_p]
        lib.oracle_index_create.restype = ctypes.c_void_p
        lib.oracle_index_create.argtypes = [u32p, u32p, u32p, ctypes.c_uint64]
        lib.oracle_index_free.argtypes = [ctypes.c_void_p]
        lib.oracle_index_query.restype = ctypes.c_int
        lib.oracle_index_query.argtypes = [ctypes.c_void_p, ctypes.c_uint32, u32p, u32p,
                                           ctypes.c_uint32, u32p, u32p, u32p,
                                           ctypes.c_int, ctypes.POINTER(u32p),
                                           ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32)]
        _lib = lib
    return _lib


def _u32(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint32))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def oracle_bgp(s, p, o, q, n_threads=0):
    """Sorted distinct solution rows of query q (synth.Query) as a
    uint32 array [n_rows, n_vars] (variables in ascending vertex index)."""
    lib = _load()
    keep = []
    sa, sp_ = _u32(s); keep.append(sa)
    pa, pp_ = _u32(p); keep.append(pa)
    oa, op_ = _u32(o); keep.append(oa)
    nv = q.n_vertices
    ic, icp = _u32([0 if v is None else 1 for v in q.vertices] or [0])
    cid, cidp = _u32([0 if v is None else min(v, 0xFFFFFFFF) for v in q.vertices] or [0])
    es, esp = _u32([e[0] for e in q.edges] or [0])
    ep, epp = _u32([e[1] for e in q.edges] or [0])
    ed, edp = _u32([e[2] for e in q.edges] or [0])
    rows = ctypes.POINTER(ctypes.c_uint32)()
    nr = ctypes.c_uint64(0)
    nc = ctypes.c_uint32(0)
    rc = lib.oracle_bgp(sp_, pp_, op_, len(sa), nv, icp, cidp, len(q.edges), esp, epp, edp,
                        int(n_threads), ctypes.byref(rows), ctypes.byref(nr), ctypes.byref(nc))
    if rc != 0:
        raise RuntimeError(f"oracle_bgp failed rc={rc}")
    n, w = int(nr.value), int(nc.value)
    if n == 0 or w == 0:
        out = np.zeros((n, w), dtype=np.uint32)
    else:
        out = np.ctypeslib.as_array(rows, shape=(n * w,)).copy().reshape(n, w)
    lib.oracle_free(rows)
    return out


class OracleIndex:
    """Index build (sorted SPO/OPS) separated from queries, so the CPU baseline
    can time queries apart from loading (the paper separates loading time,
    Tables 2-4, from query time, Tables 5-6)."""

    def __init__(self, s, p, o):
        lib = _load()
        sa, sp_ = _u32(s)
        pa, pp_ = _u32(p)
        oa, op_ = _u32(o)
        self._h = lib.oracle_index_create(sp_, pp_, op_, len(sa))

    def query(self, q, n_threads=0):
        lib = _load()
        ic, icp = _u32([0 if v is None else 1 for v in q.vertices] or [0])
        cid, cidp = _u32([0 if v is None else min(v, 0xFFFFFFFF) for v in q.vertices] or [0])
        es, esp = _u32([e[0] for e in q.edges] or [0])
        ep, epp = _u32([e[1] for e in q.edges] or [0])
        ed, edp = _u32([e[2] for e in q.edges] or [0])
        rows = ctypes.POINTER(ctypes.c_uint32)()
        nr = ctypes.c_uint64(0)
        nc = ctypes.c_uint32(0)
        rc = lib.oracle_index_query(self._h, q.n_vertices, icp, cidp, len(q.edges), esp, epp, edp,
                                    int(n_threads), ctypes.byref(rows), ctypes.byref(nr),
                                    ctypes.byref(nc))
        if rc != 0:
            raise RuntimeError(f"oracle_index_query failed rc={rc}")
        n, w = int(nr.value), int(nc.value)
        if n == 0 or w == 0:
            out = np.zeros((n, w), dtype=np.uint32)
        else:
            out = np.ctypeslib.as_array(rows, shape=(n * w,)).copy().reshape(n, w)
        lib.oracle_free(rows)
        return out

    def close(self):
        if self._h:
            _load().oracle_index_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
