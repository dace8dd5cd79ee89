"""dev tool (CPU, numpy): replay the visited-set MS-BFS level recurrence of one source batch on a
config's layer and count the row traffic in 32-byte sectors -- gathered neighbour rows, own rows read,
rows written -- with and without skipping the segments of V(v) that are all-zero or all-one.  This is
the estimate behind the segment-skipping experiment of DESIGN.md 6.1 (predicted: 26 % fewer sectors on
a C5 layer; measured on the B200: slower, the sparse levels are not byte-bound).

    python tools/segment_sim.py C5 262144 0      # config, V, layer (W = 64: 4096 sources per batch)
"""
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import build_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
V = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
layer = int(sys.argv[3]) if len(sys.argv) > 3 else 0
W, NSEC = 64, 16                        # 64 words per row, 16 sectors of 4 words
B = 64 * W
FULL = np.uint64(0xFFFFFFFFFFFFFFFF)

E = build_config(name, V=V).layers[layer]
src = np.concatenate([E[:, 0], E[:, 1]])
dst = np.concatenate([E[:, 1], E[:, 0]])
o = np.lexsort((dst, src))
src, dst = src[o], dst[o]
deg = np.bincount(src, minlength=V)
sources = np.nonzero(deg > 0)[0][:B]    # one batch window of non-isolated rows (community-contiguous)
Vis = np.zeros((V, W), np.uint64)
for j, s in enumerate(sources):
    Vis[s, j >> 6] |= np.uint64(1) << np.uint64(j & 63)
changed = np.zeros(V, bool)
changed[sources] = True
done = np.zeros(V, bool)
tot = dict(gather=0, gather_skip=0, own=0, own_skip=0, write=0, write_skip=0, masks=0)
d = 1
while True:
    m = changed[dst] & ~done[src]
    sv, su = src[m], dst[m]
    if len(sv) == 0:
        break
    rows, start = np.unique(sv, return_index=True)
    ng = np.diff(np.append(start, len(sv)))
    G = Vis[su]
    acc = np.bitwise_or.reduceat(G, start, axis=0)
    own = Vis[rows]
    new = acc & ~own
    ch = (new != 0).any(axis=1)
    osec = own.reshape(len(rows), NSEC, 4)
    ofull = (osec == FULL).all(axis=2)
    ozero = (osec == 0).all(axis=2)
    gsec = G.reshape(len(su), NSEC, 4)
    gmixed_or_full = ~(gsec == 0).all(axis=2)
    need = gmixed_or_full & np.repeat(~ofull, ng, axis=0)      # skip zero sectors and own-complete ones
    nv = (own | new)[ch].reshape(-1, NSEC, 4)
    nmixed = ~((nv == 0).all(axis=2) | (nv == FULL).all(axis=2))
    c = dict(gather=len(su) * NSEC, gather_skip=int(need.sum()), own=len(rows) * NSEC,
             own_skip=int((~ofull & ~ozero).sum()), write=int(ch.sum()) * NSEC, write_skip=int(nmixed.sum()),
             masks=len(su))
    for k, v in c.items():
        tot[k] += v
    print(f"d={d:2d} rows {len(rows):7d} changed {int(ch.sum()):7d} gathers {len(su):8d}  gathered sectors kept "
          f"{c['gather_skip'] / max(c['gather'], 1):.3f}  own {c['own_skip'] / max(c['own'], 1):.3f}  "
          f"written {c['write_skip'] / max(c['write'], 1):.3f}")
    Vis[rows] = own | new
    pc = np.unpackbits(np.ascontiguousarray(Vis[rows]).view(np.uint8), axis=1).sum(axis=1)
    done[rows[pc == B]] = True
    changed[:] = False
    changed[rows[ch]] = True
    d += 1
full = tot["gather"] + tot["own"] + tot["write"]
skip = tot["gather_skip"] + tot["own_skip"] + tot["write_skip"] + tot["masks"]    # + one mask sector per gather
print(f"sectors per batch: whole rows {full / 1e6:.1f} M, with segment skipping {skip / 1e6:.1f} M ({skip / full:.3f})")
