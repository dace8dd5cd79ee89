"""ORACLE -- TEST INFRASTRUCTURE ONLY.  ctypes loader for oracle/bfs_oracle.c.

``build()`` compiles the plain C BFS with gcc (building the checker is not
using it); ``bfs_sources`` calls it.  Shares nothing with the product path.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bfs_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_bfs.so")
_lib = None


def build(force=False):
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_bfs_sources.restype = ctypes.c_int
        L.oracle_bfs_sources.argtypes = [
            ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_num_threads.argtypes = [ctypes.c_int]
        L.oracle_graph_new.restype = ctypes.c_void_p
        L.oracle_graph_new.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_graph_free.restype = None
        L.oracle_graph_free.argtypes = [ctypes.c_void_p]
        L.oracle_graph_bfs.restype = ctypes.c_int
        L.oracle_graph_bfs.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
        _lib = L
    return _lib


def num_threads(threads=0):
    return lib().oracle_num_threads(int(threads))


def bfs_sources(V, E, sources, threads=0):
    """E: iterable of canonical (u, v) pairs or an (m,2) int array."""
    if isinstance(E, np.ndarray):
        arr = np.ascontiguousarray(E, dtype=np.int32).reshape(-1, 2)
    else:
        arr = np.array(sorted(E), dtype=np.int32).reshape(-1, 2)
    eu = np.ascontiguousarray(arr[:, 0])
    ev = np.ascontiguousarray(arr[:, 1])
    src = np.ascontiguousarray(sources, dtype=np.int32)
    S = np.zeros(len(src), np.uint64)
    k = np.zeros(len(src), np.int32)
    rc = lib().oracle_bfs_sources(int(V), int(len(eu)), eu.ctypes.data, ev.ctypes.data,
                                  src.ctypes.data, int(len(src)), S.ctypes.data, k.ctypes.data,
                                  int(threads))
    if rc != 0:
        raise RuntimeError(f"oracle_bfs_sources failed: {rc}")
    return S, k


class Graph:
    """Adjacency built once; ``bfs(sources)`` returns (S, k, seconds of the BFS loop)."""

    def __init__(self, V, E):
        arr = np.ascontiguousarray(E, dtype=np.int32).reshape(-1, 2)
        self._eu = np.ascontiguousarray(arr[:, 0])
        self._ev = np.ascontiguousarray(arr[:, 1])
        self.V = int(V)
        self.h = lib().oracle_graph_new(self.V, int(len(arr)), self._eu.ctypes.data, self._ev.ctypes.data)
        if not self.h:
            raise RuntimeError("oracle_graph_new failed")

    def bfs(self, sources, threads=0):
        src = np.ascontiguousarray(sources, dtype=np.int32)
        S = np.zeros(len(src), np.uint64)
        k = np.zeros(len(src), np.int32)
        secs = ctypes.c_double(0.0)
        rc = lib().oracle_graph_bfs(self.h, src.ctypes.data, int(len(src)), S.ctypes.data, k.ctypes.data,
                                    int(threads), ctypes.byref(secs))
        if rc != 0:
            raise RuntimeError(f"oracle_graph_bfs failed: {rc}")
        return S, k, secs.value

    def __del__(self):
        try:
            if self.h:
                lib().oracle_graph_free(self.h)
                self.h = None
        except Exception:
            pass
