"""Full-size oracle digests for the GPU parity tests (tests/golden/fullsize_<C>.json).

Calls ONLY ``oracle/`` (the plain CPU definition) and ``synth/`` (the seeded
input generator); nothing here touches the CUDA path.  For every BASELINE.json
config it runs the whole oracle at full size -- all-sources BFS on every layer
and on every AND subset (§4), WF closeness, n-penalty sums,
fsum means and CC nodes, the AND edge sets,
GT top-K, CC2 (Alg. 1), CC2 above-average,
CC1 with its full ranked set R (Eq. 2-3) and naive
 -- and stores SHA-256 digests of every output in the byte
layouts of tests/_digest.py, keyed by the SHA-256 of the inputs.  Short lists
(top-K) are stored verbatim as well.

    python tools/oracle_golden.py C1 C2 C3 C4 C5 [--threads N]

Runtime on 8 cores: C1/C2 seconds, C3 ~3 min, C4 ~8 min, C5 ~15 min.
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from synth import build_config  # noqa: E402
from _digest import sha, edge_keys, input_sha  # noqa: E402


def graph_record(V, res):
    CH = sorted(res["CH"])
    return {
        "S": sha(res["S"], "S"), "k": sha(res["k"], "k"), "c": sha(res["c"], "c"),
        "pen": sha(res["pen"], "pen"), "deg": sha(res["deg"], "deg"),
        "CH": sha(CH, "ids"), "n_CH": len(CH), "mu": float(res["mu"]).hex(),
        "sum_S": int(sum(res["S"])), "sum_k": int(sum(res["k"])),
        "fsum_c": math.fsum(res["c"]).hex(),
    }


def golden(name, threads):
    t0 = time.time()
    h = build_config(name)
    V, K = h.V, h.K
    out = {"config": h.name, "V": V, "K": K, "subsets": [list(T) for T in h.subsets],
           "input_sha256": input_sha(h),
           "generator": "tools/oracle_golden.py (oracle/ + synth/ only)",
           "layers": [], "ands": []}
    Es = [set(map(tuple, L.tolist())) for L in h.layers]
    res = []
    for i, E in enumerate(Es):
        r = O.analyze(V, E, threads=threads)
        res.append(r)
        rec = graph_record(V, r)
        rec["m"] = len(E)
        out["layers"].append(rec)
        print(f"[{name}] layer {i}: m={len(E)} ({time.time() - t0:.0f} s)", flush=True)
    for T in h.subsets:
        T = list(T)
        A = O.and_aggregate([Es[i] for i in T])
        ra = O.analyze(V, A, threads=threads)
        rs = [res[i] for i in T]
        rec = graph_record(V, ra)
        rec["T"] = T
        rec["m"] = len(A)
        rec["edges"] = sha(edge_keys(V, A), "edges")
        Or = O.or_aggregate([Es[i] for i in T])
        rec["or_m"] = len(Or)
        rec["or_edges"] = sha(edge_keys(V, Or), "edges")
        rec["gt_topk"] = O.topk_closeness(ra["c"], K)
        rec["cc2_topk"] = O.cc2(rs, K)[0]
        r1, n1, _ = O.cc1(rs, V)                          # the full ranked set R (K = V)
        rec["cc1_n"] = n1
        rec["cc1_ranked"] = sha(r1, "ids")
        rec["cc1_topk"] = r1[:K]
        nv = sorted(O.naive(rs, V)[2])
        rec["naive_n"] = len(nv)
        rec["naive"] = sha(nv, "ids")
        rec["naive_topk"] = nv[:K]
        av = sorted(O.cc2_above_average(rs))
        rec["cc2_avg_n"] = len(av)
        rec["cc2_avg"] = sha(av, "ids")
        rec["cc2_avg_topk"] = av[:K]
        out["ands"].append(rec)
        print(f"[{name}] AND{T}: m={len(A)} |R|={n1} ({time.time() - t0:.0f} s)", flush=True)
    out["oracle_seconds"] = round(time.time() - t0, 1)
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_{name}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"[{name}] wrote {path} ({out['oracle_seconds']} s)", flush=True)


def add_or(name):
    """add the OR aggregate's edge-set digest of every subset (oracle or_aggregate) to an
    existing digest file without re-running the BFS."""
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_{name}.json")
    out = json.load(open(path))
    h = build_config(name)
    assert out["input_sha256"] == input_sha(h)
    Es = [set(map(tuple, L.tolist())) for L in h.layers]
    for rec in out["ands"]:
        A = O.or_aggregate([Es[i] for i in rec["T"]])
        rec["or_m"] = len(A)
        rec["or_edges"] = sha(edge_keys(V=h.V, pairs=A), "edges")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"[{name}] OR digests added to {path}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--add-or", action="store_true", help="only add the OR edge-set digests to existing files")
    a = ap.parse_args()
    for c in a.configs:
        if a.add_or:
            add_or(c)
        else:
            golden(c, a.threads)


if __name__ == "__main__":
    main()
