"""Thin Python binding over the C ABI (include/hm.h): argument marshalling only.

Every step of the path -- CSR build, AND/OR aggregation, all-sources BFS
closeness, exact means, CC-node sets, composition and top-K -- runs in
libhm.so's CUDA kernels.  PyTorch is used for device memory and the stream.

Inputs may be numpy arrays (host) or torch CUDA tensors (device); outputs are
returned as numpy arrays by default, or written into caller-supplied torch
CUDA tensors (``out=``) without leaving the device.
"""
import ctypes

import numpy as np

from . import _lib
from ._lib import c_i32p
from ._lib import HM_CC1, HM_CC1_RARY, HM_CC2, HM_CC2_AVG, HM_NAIVE  # noqa: F401

HEURISTICS = {"naive": HM_NAIVE, "cc1": HM_CC1, "cc2": HM_CC2, "cc2_avg": HM_CC2_AVG, "cc1_rary": HM_CC1_RARY}


class HmError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_lib.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _ptr(x):
    """data pointer of a numpy array or torch tensor (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    # torch tensor
    assert x.is_contiguous()
    return x.data_ptr()


class Context:
    """One hm_ctx on ``device``, issuing work on ``stream`` (a torch.cuda.Stream,
    or None for a fresh torch stream kept in ``self.stream``).  Time or order
    torch work against the library with ``self.stream``."""

    def __init__(self, device=0, stream=None):
        self.L = _lib.load()
        import torch
        self.torch = torch
        torch.cuda.init()
        if stream is False:          # library-owned stream (debug)
            self.stream = None
            s = 0
        else:
            self.stream = torch.cuda.Stream(device) if stream is None else stream
            s = self.stream.cuda_stream
        self._stream = s
        h = ctypes.c_void_p()
        st = self.L.hm_create(ctypes.byref(h), int(device), ctypes.c_void_p(s) if s else None)
        if st != 0:
            raise HmError(st, "hm_create failed")
        self.h = h
        self.device = device
        self.V = None
        self.n_layers = 0

    # ------------------------------------------------------------ plumbing
    def _check(self, st):
        if st != 0:
            raise HmError(st, self.L.hm_last_error(self.h).decode(errors="replace"))

    def close(self):
        if getattr(self, "h", None):
            self.L.hm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_param(self, name, value):
        self._check(self.L.hm_set_param(self.h, name.encode(), int(value)))

    def sync(self):
        self._check(self.L.hm_sync(self.h))

    def debug_counts(self, n=335872):
        out = np.zeros(n, np.uint64)
        self._check(self.L.hm_debug_counts(self.h, _ptr(out), n))
        return out

    def stats(self, reset=False):
        s = _lib.HmStats()
        self._check(self.L.hm_get_stats(self.h, ctypes.byref(s), 1 if reset else 0))
        out = {k: getattr(s, k) for k, _ in _lib.HmStats._fields_}
        out["phase_ms"] = list(s.phase_ms)
        return out

    # ------------------------------------------------------------- graphs
    def load_layers(self, V, layers):
        """layers: list of (m,2) int32 arrays (numpy host or torch CUDA).
        Returns (layer ids, dropped counts)."""
        l = len(layers)
        keep = []
        ptrs = (ctypes.c_void_p * l)()
        ms = (ctypes.c_int64 * l)()
        for i, E in enumerate(layers):
            if isinstance(E, np.ndarray):
                E = np.ascontiguousarray(E, dtype=np.int32).reshape(-1, 2)
            else:
                assert E.dtype == self.torch.int32
                E = E.contiguous().reshape(-1, 2)
            keep.append(E)
            ptrs[i] = _ptr(E) if E.shape[0] else None
            ms[i] = E.shape[0]
        dropped = (ctypes.c_int64 * l)()
        self._check(self.L.hm_load_layers(self.h, int(V), l, ptrs, ms, dropped))
        self.V = int(V)
        self.n_layers = l
        return list(range(l)), [int(x) for x in dropped]

    def graph_info(self, g):
        """(V, m) of graph g.  For an AND aggregate the exact m is read from the device (one host
        round trip); hm_graph_info without the m output does not synchronise."""
        V = ctypes.c_int32()
        m = ctypes.c_int64()
        self._check(self.L.hm_graph_info(self.h, int(g), ctypes.byref(V), ctypes.byref(m), None, None))
        return V.value, m.value

    def _V(self, g):
        V = ctypes.c_int32()
        self._check(self.L.hm_graph_info(self.h, int(g), ctypes.byref(V), None, None, None))
        return V.value

    def graph_csr(self, g):
        V, m = self.graph_info(g)
        rp = np.zeros(V + 1, np.int32)
        col = np.zeros(max(2 * m, 1), np.int32)
        self._check(self.L.hm_graph_csr(self.h, int(g), _ptr(rp), _ptr(col)))
        return rp, col[:2 * m]

    def and_aggregate(self, ids):
        ids = (ctypes.c_int32 * len(ids))(*ids)
        out = ctypes.c_int32()
        self._check(self.L.hm_and_aggregate(self.h, ids, len(ids), ctypes.byref(out)))
        return out.value

    def or_aggregate(self, ids):
        ids = (ctypes.c_int32 * len(ids))(*ids)
        out = ctypes.c_int32()
        self._check(self.L.hm_or_aggregate(self.h, ids, len(ids), ctypes.byref(out)))
        return out.value

    def free_graph(self, g):
        self._check(self.L.hm_free_graph(self.h, int(g)))

    # ----------------------------------------------------------- analysis
    def closeness(self, g, out=None, want=("S", "k", "c", "pen")):
        """All-sources BFS closeness of graph g.  Returns dict of numpy arrays
        (S uint64, k int32, c float64, pen uint64) for the names in ``want``;
        with ``out`` (dict of torch CUDA tensors) writes there instead."""
        V = self._V(g)
        if out is None:
            res = {}
            if "S" in want:
                res["S"] = np.zeros(V, np.uint64)
            if "k" in want:
                res["k"] = np.zeros(V, np.int32)
            if "c" in want:
                res["c"] = np.zeros(V, np.float64)
            if "pen" in want:
                res["pen"] = np.zeros(V, np.uint64)
        else:
            res = out
        self._check(self.L.hm_closeness(self.h, int(g), _ptr(res.get("S")), _ptr(res.get("k")),
                                        _ptr(res.get("c")), _ptr(res.get("pen"))))
        return res

    def closeness_multi(self, gids):
        """Closeness of several graphs in one fused pass (results cached per graph)."""
        arr = (ctypes.c_int32 * len(gids))(*gids)
        self._check(self.L.hm_closeness_multi(self.h, arr, len(gids)))

    def closeness_partial(self, g, shard, nshards, out=None):
        """One shard's partial distance sums S_partial[V] (uint64; numpy, or into a
        device tensor `out`): batches shard, shard + nshards, ... (hm_closeness_partial)."""
        V = self._V(g)
        buf = np.zeros(V, np.uint64) if out is None else out
        self._check(self.L.hm_closeness_partial(self.h, int(g), int(shard), int(nshards), _ptr(buf)))
        return buf

    def closeness_combine(self, g, S_total):
        """Finalise graph g from the summed shard sums (numpy uint64 or device tensor)."""
        if isinstance(S_total, np.ndarray):
            S_total = np.ascontiguousarray(S_total, dtype=np.uint64)
        self._check(self.L.hm_closeness_combine(self.h, int(g), _ptr(S_total)))

    def closeness_results(self, g, out=None, want=("S", "k", "c", "pen")):
        """Cached closeness results of graph g (numpy by default, or into ``out``)."""
        V = self._V(g)
        if out is None:
            res = {}
            if "S" in want:
                res["S"] = np.zeros(V, np.uint64)
            if "k" in want:
                res["k"] = np.zeros(V, np.int32)
            if "c" in want:
                res["c"] = np.zeros(V, np.float64)
            if "pen" in want:
                res["pen"] = np.zeros(V, np.uint64)
        else:
            res = out
        self._check(self.L.hm_closeness_results(self.h, int(g), _ptr(res.get("S")), _ptr(res.get("k")),
                                                _ptr(res.get("c")), _ptr(res.get("pen"))))
        return res

    def cc_nodes(self, g):
        """(sorted numpy array of CC nodes, count, mean closeness)."""
        V = self._V(g)
        bm = np.zeros((V + 31) // 32, np.uint32)
        cnt = ctypes.c_int32()
        mu = ctypes.c_double()
        self._check(self.L.hm_cc_nodes(self.h, int(g), _ptr(bm), ctypes.byref(cnt), ctypes.byref(mu)))
        bits = np.unpackbits(bm.view(np.uint8), bitorder="little")[:V]
        return np.nonzero(bits)[0].astype(np.int64), cnt.value, mu.value

    def degrees(self, g):
        V = self._V(g)
        d = np.zeros(V, np.int32)
        self._check(self.L.hm_degrees(self.h, int(g), _ptr(d)))
        return d

    def topk_closeness(self, g, K, out=None):
        ids = np.zeros(K, np.int32) if out is None else out
        self._check(self.L.hm_topk_closeness(self.h, int(g), int(K), _ptr(ids)))
        return ids

    # -------------------------------------------------------- composition
    def compose(self, heuristic, ids, K, out=None, count_out=None):
        """heuristic in {'cc1','cc1_rary','cc2','cc2_avg','naive'}.  Returns (ranked ids, |result set|).
        With ``out`` (a device tensor of K int32) and ``count_out`` (a device tensor of 1 int32)
        the call is stream-ordered with no host synchronisation: ``out`` holds K entries,
        -1 past |R|, and (out, count_out) is returned."""
        h = HEURISTICS[heuristic] if isinstance(heuristic, str) else int(heuristic)
        arr = (ctypes.c_int32 * len(ids))(*ids)
        buf = np.zeros(K, np.int32) if out is None else out
        if count_out is not None:
            self._check(self.L.hm_compose(self.h, h, arr, len(ids), int(K), _ptr(buf),
                                          ctypes.cast(_ptr(count_out), c_i32p)))
            return buf, count_out
        cnt = ctypes.c_int32()
        self._check(self.L.hm_compose(self.h, h, arr, len(ids), int(K), _ptr(buf), ctypes.byref(cnt)))
        n = cnt.value
        if out is None:
            return buf[:min(K, n)], n
        return buf, n

    def exact_mean(self, x, mask=None):
        """hm_exact_mean: (RN(exact sum of the selected x) / count, count).  x: float64 numpy
        array or CUDA tensor; mask: None or uint8 of the same length."""
        if isinstance(x, np.ndarray):
            x = np.ascontiguousarray(x, dtype=np.float64)
        if isinstance(mask, np.ndarray):
            mask = np.ascontiguousarray(mask, dtype=np.uint8)
        n = int(x.shape[0])
        mu = ctypes.c_double()
        cnt = ctypes.c_int32()
        self._check(self.L.hm_exact_mean(self.h, _ptr(x) if n else None, n, _ptr(mask) if n else None,
                                         ctypes.byref(mu), ctypes.byref(cnt)))
        return mu.value, cnt.value

    # ------------------------------------------------------------ metrics
    def set_metrics(self, V, est, gt):
        """Accuracy of an estimated id list vs the ground truth:
        dict jaccard, precision, recall, f1, n_est, n_gt, n_common."""
        def arr(x):
            if x is None or (not isinstance(x, np.ndarray) and hasattr(x, "data_ptr")):
                return x
            return np.ascontiguousarray(np.asarray(x, dtype=np.int32).reshape(-1))
        est, gt = arr(est), arr(gt)
        ne = 0 if est is None else int(est.shape[0])
        ng = 0 if gt is None else int(gt.shape[0])
        out = (ctypes.c_double * 7)()
        self._check(self.L.hm_set_metrics(self.h, int(V), _ptr(est) if ne else None, ne,
                                          _ptr(gt) if ng else None, ng, out))
        keys = ("jaccard", "precision", "recall", "f1", "n_est", "n_gt", "n_common")
        return {k: (float(v) if i < 4 else int(v)) for i, (k, v) in enumerate(zip(keys, out))}
