"""Byte layouts and SHA-256 digests of full-size outputs.

Shared by ``tools/oracle_golden.py`` (which writes ``tests/golden/fullsize_*.json``
from the oracle alone) and ``tests/test_gpu_fullsize.py`` (which digests the
CUDA path's outputs the same way).  Serialisation only: no arithmetic of the
method lives here.

Layouts (all little-endian):
  S, pen      uint64[V]      k, deg   int32[V]      c   float64[V] (IEEE bits)
  id sets     sorted int32   ranked id lists   int32 in rank order
  edge sets   sorted int64 keys u*V + v with u < v
"""
import hashlib

import numpy as np

LAYOUT = {"S": "<u8", "pen": "<u8", "k": "<i4", "deg": "<i4", "c": "<f8",
          "ids": "<i4", "edges": "<i8"}


def sha(arr, kind):
    a = np.ascontiguousarray(np.asarray(arr).astype(LAYOUT[kind], copy=False))
    return hashlib.sha256(a.tobytes()).hexdigest()


def edge_keys(V, pairs):
    """sorted int64 keys of a canonical edge collection ((m,2) array or set of tuples)."""
    if isinstance(pairs, np.ndarray):
        p = pairs.astype(np.int64).reshape(-1, 2)
    else:
        p = np.array(sorted(pairs), dtype=np.int64).reshape(-1, 2)
    return np.sort(p[:, 0] * np.int64(V) + p[:, 1])


def input_sha(h):
    """SHA-256 of a HoMLN's inputs: V, K, every layer's canonical int32 pairs, the subsets."""
    m = hashlib.sha256()
    m.update(np.array([h.V, h.K, len(h.layers)], "<i8").tobytes())
    for L in h.layers:
        a = np.ascontiguousarray(np.asarray(L, dtype="<i4").reshape(-1, 2))
        m.update(np.array([a.shape[0]], "<i8").tobytes())
        m.update(a.tobytes())
    for T in h.subsets:
        m.update(np.array(list(T) + [-1], "<i8").tobytes())
    return m.hexdigest()
