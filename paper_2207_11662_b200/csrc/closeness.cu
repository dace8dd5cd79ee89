// Psi (PAPER.md:121-122 §3; :209 §4): all-sources BFS closeness of one graph or of several graphs in one fused pass.
//
// Pipeline (all device-side, stream-ordered, no host synchronisation):
//   1. connected components (lock-free union-find, hooks larger root under
//      smaller, so the label is the smallest vertex id of the component);
//   2. relabel: components sorted by (size desc, smallest id asc), vertices by
//      (component rank, id); isolated vertices last and excluded from the BFS;
//   3. relabelled CSR + per-row component info + heavy-row list;
//   4. persistent MS-BFS (msbfs.cu) -> S per relabelled row;
//   5. finalize in original order: S, k, Wasserman-Faust closeness, n-penalty
//      sum, degree;
//   6. mu = RN(exact sum c) / V (exactsum.cu) and CH = {v : c(v) > mu}.
#include <cmath>
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "msbfs.cuh"
#include "exactsum.cuh"

namespace hm {
namespace {

constexpr int TB = 256;

__device__ __forceinline__ int cc_find(int32_t *p, int x) {
    while (true) {
        const int px = __ldcg(p + x);
        if (px == x) return x;
        const int ppx = __ldcg(p + px);
        if (ppx != px) p[x] = ppx;     // path halving: ppx is an ancestor of x
        x = px;
    }
}

__global__ void k_iota(int32_t *p, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}

// union-find start (as in ECL-CC): parent(u) = the smallest of u and its neighbours -- a valid
// forest (parents are smaller) that already joins most of each component; warp per row
__global__ void k_cc_init(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int32_t *p, int V) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = w0; u < V; u += nw) {
        const int rb = row_ptr[u], re = row_ptr[u + 1];
        int m = (int)u;
        for (int j = rb + lane; j < re; j += 32) m = min(m, col[j]);
        for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) p[u] = m;
    }
}

__device__ __forceinline__ void cc_unite(int32_t *p, int u, int v) {
    int ru = cc_find(p, u), rv = cc_find(p, v);
    while (ru != rv) {
        if (ru < rv) { const int t = ru; ru = rv; rv = t; }   // ru > rv: hook ru under rv
        const int old = atomicCAS(p + ru, ru, rv);
        if (old == ru) break;
        ru = cc_find(p, old);
        rv = cc_find(p, rv);
    }
}

// Sampled components (the Afforest scheme): (1) every vertex unites with its first CC_SAMPLE
// neighbours, which already joins most of the giant component; (2) the most frequent root after
// (1) is taken as the giant; (3) only rows not yet in the giant unite over their remaining arcs.
// Every edge is then either united or has both ends already joined to the giant.
constexpr int CC_SAMPLE = 2;
__global__ void k_cc_sample(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int32_t *p, int V) {
    for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < V; u += gridDim.x * blockDim.x) {
        const int rb = row_ptr[u], re = min(row_ptr[u + 1], row_ptr[u] + CC_SAMPLE);
        for (int j = rb; j < re; ++j) cc_unite(p, u, col[j]);
    }
}
// root counts (warp-aggregated) of the sampled forest
__global__ void k_cc_root_counts(int32_t *p, int32_t *cnt, int V) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        const int r = cc_find(p, v);
        const unsigned act = __activemask();
        const unsigned same = __match_any_sync(act, r);
        if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(cnt + r, __popc(same));
    }
}
__global__ void k_cc_giant(const int32_t *p, const int32_t *cnt, unsigned long long *best, int V) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
        if (cnt[v] > 0) atomicMax(best, ((unsigned long long)cnt[v] << 32) | (unsigned)(V - 1 - v));
}
// warp per row u not joined to the giant root: unite over the arcs after the sampled ones
__global__ void k_cc_rest(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int32_t *p, int V,
                          const unsigned long long *best) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int giant = V - 1 - (int)(*best & 0xffffffffull);
    for (int64_t u = w0; u < V; u += nw) {
        const int rb = row_ptr[u] + CC_SAMPLE, re = row_ptr[u + 1];
        if (rb >= re) continue;
        int in_giant = 0;
        if (lane == 0) in_giant = cc_find(p, (int)u) == giant;
        if (__shfl_sync(0xffffffffu, in_giant, 0)) continue;
        for (int j = rb + lane; j < re; j += 32) cc_unite(p, (int)u, col[j]);
    }
}

// warp per row u; unite(u, v) for arcs with v > u.  (An arc-parallel version spreads hub rows
// over more threads but was slower: thousands of threads then contend on the hub's root with
// CAS, 0.48 vs 0.31 ms per C3 graph.)
__global__ void k_cc_union(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                           int32_t *p, int V) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = w0; u < V; u += nw) {
        const int rb = row_ptr[u], re = row_ptr[u + 1];
        for (int j = rb + lane; j < re; j += 32) {
            const int v = col[j];
            if (v <= u) continue;
            int ru = cc_find(p, (int)u), rv = cc_find(p, v);
            while (ru != rv) {
                if (ru < rv) { const int t = ru; ru = rv; rv = t; }   // ru > rv: hook ru under rv
                const int old = atomicCAS(p + ru, ru, rv);
                if (old == ru) break;
                ru = cc_find(p, old);
                rv = cc_find(p, rv);
            }
        }
    }
}

// Components by min-label hooking and pointer jumping (Shiloach-Vishkin style), in one cooperative
// launch (cc_init 3, default).  f[v] <= v always holds (every update is an atomicMin to a vertex of
// the same component), so f is a forest whose roots are the smallest ids.  Per round: every edge
// hooks the larger of its endpoints' roots under the smaller (atomicMin: no retry loop under
// contention, unlike CAS unions on popular roots), then every vertex jumps to its root; rounds
// repeat until no hook changes anything.  The edges are walked a warp per 32-row group over the
// group's contiguous arcs (each arc's row found by a shuffle search over the group's row_ptr).
namespace cgk = cooperative_groups;
__global__ void k_cc_sv(const int32_t *__restrict__ rp, const int32_t *__restrict__ col, int V, int32_t *f,
                        int32_t *flags, int32_t *rowof) {
    cgk::grid_group grid = cgk::this_grid();
    const int lane = threadIdx.x & 31;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t gwarp = gtid >> 5, nwarps = nth >> 5;
    const int64_t nnz = rp[V];
    const int64_t ngroups = ((int64_t)V + 31) >> 5;
    // graphs with hub rows (rowof != null): the row of every arc (warp per row, coalesced writes), so
    // the rounds walk the arcs evenly over all threads and a hub row does not hold one warp for
    // thousands of arcs; otherwise a warp per 32-row group walks the group's contiguous arcs
    if (rowof)
        for (int64_t u = gwarp; u < V; u += nwarps)
            for (int j = rp[u] + lane; j < rp[u + 1]; j += 32) rowof[j] = (int)u;
    for (int64_t v = gtid; v < V; v += nth) f[v] = (int)v;
    if (gtid == 0) flags[0] = flags[1] = flags[2] = 0;
    grid.sync();
    for (int it = 0;; ++it) {
        // three rotating flags: the one reset here was last read two rounds ago, before the
        // grid barriers of the previous round
        int32_t *fl = flags + (it % 3);
        if (gtid == 0) flags[(it + 1) % 3] = 0;
        bool changed = false;
        if (rowof) {
            for (int64_t j = gtid; j < nnz; j += nth) {
                const int u = rowof[j], w = col[j];
                if (w <= u) continue;                                 // each edge once
                const int fu = f[u], fw = f[w];
                if (fu == fw) continue;
                const int hi = fu > fw ? fu : fw, lw = fu > fw ? fw : fu;
                if (atomicMin(f + hi, lw) > lw) changed = true;
            }
        } else {
            for (int64_t g = gwarp; g < ngroups; g += nwarps) {
                const int r0 = (int)(g * 32);
                const int rl = r0 + lane < V ? r0 + lane : V;
                const int rpl = rp[rl];                               // lane t: first arc of row r0 + t
                const int A0 = __shfl_sync(0xffffffffu, rpl, 0);
                const int A1 = rp[r0 + 32 < V ? r0 + 32 : V];
                for (int base = A0; base < A1; base += 32) {          // warp-uniform trip count
                    const int j = base + lane;
                    // row of arc j: the last lane t with rp[r0 + t] <= j (5-step shuffle search)
                    int lo = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const int x = __shfl_sync(0xffffffffu, rpl, lo + step);
                        if (lo + step < 32 && x <= j) lo += step;
                    }
                    if (j >= A1) continue;
                    const int u = r0 + lo, w = col[j];
                    if (w <= u) continue;                             // each edge once
                    const int fu = f[u], fw = f[w];
                    if (fu == fw) continue;
                    const int hi = fu > fw ? fu : fw, lw = fu > fw ? fw : fu;
                    if (atomicMin(f + hi, lw) > lw) changed = true;
                }
            }
        }
        if (changed) *fl = 1;
        grid.sync();
        for (int64_t v = gtid; v < V; v += nth) {                     // jump to the root
            int x = f[v];
            int y = f[x];
            while (x != y) {
                x = y;
                y = f[x];
            }
            f[v] = x;
        }
        grid.sync();
        if (*((volatile int32_t *)fl) == 0) break;
    }
}

// Final labels go to a separate array: concurrent path halving inside cc_find
// may still rewrite parent[] entries (to valid, less-compressed ancestors),
// so writing roots back into parent[] would race.
__global__ void k_cc_compress(int32_t *p, int32_t *label, int32_t *csize, int V) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        const int r = cc_find(p, v);
        label[v] = r;
        // warp-aggregated count (the giant component's root would serialise per-vertex atomics)
        const unsigned act = __activemask();
        const unsigned same = __match_any_sync(act, r);
        if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(csize + r, __popc(same));
    }
}

// component keys (stable 32-bit key/value radix sort; ids ascending within equal keys):
// roots -> key V - size, value root; others -> key V (sort last)
__global__ void k_comp_keys(const int32_t *label, const int32_t *csize, uint32_t *key, uint32_t *val, int V) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        key[v] = (label[v] == v) ? (uint32_t)(V - csize[v]) : (uint32_t)V;
        val[v] = (uint32_t)v;
    }
}

// sorted component table; scalars[1] = n_giant (if > 1), scalars[2] = n_comp
__global__ void k_comp_tables(const uint32_t *keys, const uint32_t *vals, int32_t *size_s, int32_t *rank_of_root,
                              int32_t *scalars, int V) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < V; i += gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        if (k < (uint32_t)V) {
            const int sz = V - (int)k;
            size_s[i] = sz;
            rank_of_root[vals[i]] = i;
            if (i == 0) scalars[1] = sz > 1 ? sz : 0;
            const bool last = (i + 1 == V) || (keys[i + 1] >= (uint32_t)V);
            if (last) scalars[2] = i + 1;
        } else {
            size_s[i] = 0;
        }
    }
}

// scalars[0] = n_live = first row of the first singleton component
__global__ void k_nlive(const int32_t *size_s, const int32_t *cstart, int32_t *scalars, int V) {
    const int n_comp = scalars[2];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_comp; i += gridDim.x * blockDim.x)
        if (size_s[i] > 1 && (i + 1 == n_comp || size_s[i + 1] <= 1)) scalars[0] = cstart[i] + size_s[i];
}

// vertex keys: component rank (value: the vertex; the stable sort keeps ids ascending inside a
// component); peeled vertices (rem[v] > 0) key V, after every component: no BFS row
// vertex keys: component rank (stable: vertex id within a component).  With tsz (pruned graphs) the key
// is rank << 8 | (255 - min(T, 255)) in the pruned (rank-0) component: its core rows sorted by hanging-tree
// size T descending, so a batch window's T is constant over long runs of sources (the MS-BFS then weighs
// a 128-source chunk by T x popc instead of T's bit planes)
__global__ void k_vert_keys(const int32_t *label, const int32_t *rank_of_root, const int32_t *rem,
                            const uint32_t *tsz, uint32_t *key, uint32_t *val, int V) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        if (tsz) {
            if (rem[v]) {
                key[v] = (uint32_t)V << 8;
            } else {
                const uint32_t r = (uint32_t)rank_of_root[label[v]];
                const uint32_t t = tsz[v] - 1u;
                key[v] = (r << 8) | (r == 0 ? 255u - (t < 255u ? t : 255u) : 0u);
            }
        } else {
            key[v] = (rem && rem[v]) ? (uint32_t)V : (uint32_t)rank_of_root[label[v]];
        }
        val[v] = (uint32_t)v;
    }
}

__global__ void k_perm(const uint32_t *rk, const uint32_t *olds, const int32_t *row_ptr, const int32_t *degl,
                       const int32_t *size_s, const int32_t *cstart, int32_t *new_to_old, int32_t *old_to_new,
                       int32_t *new_deg, int2 *cinfo, int V, int kshift) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < V; i += gridDim.x * blockDim.x) {
        const int old = (int)olds[i];
        const int r = (int)(rk[i] >> kshift);              // component rank (k_vert_keys)
        new_to_old[i] = old;
        old_to_new[old] = i;
        if (r >= V) {                       // peeled vertex: no row
            new_deg[i] = 0;
            cinfo[i] = make_int2(0, 0);
            continue;
        }
        // live degree: arcs to peeled vertices are dropped (degl counts live neighbours)
        new_deg[i] = degl ? degl[old] : row_ptr[old + 1] - row_ptr[old];
        cinfo[i] = make_int2(cstart[r], size_s[r]);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) new_deg[V] = 0;
}

// rows of more than RELABEL_BIG arcs (R-MAT hubs of 5-8 K arcs) would hold one warp for hundreds of
// dependent-load rounds: they are listed (scalars[15] counts them) and relabelled by k_relabel_big
constexpr int RELABEL_BIG = 1024;
__global__ void k_relabel_cols(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                               const int32_t *__restrict__ nrp, const int32_t *__restrict__ new_to_old,
                               const int32_t *__restrict__ old_to_new, int32_t *__restrict__ ncol,
                               int32_t *heavy, int32_t *scalars, const int32_t *rem, int V, int32_t *big) {
    const int lane = threadIdx.x & 31;
    const int heavy_deg = scalars[4];
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int n_live = scalars[0];
    for (int64_t i = w0; i < n_live; i += nw) {
        const int old = new_to_old[i];
        const int rb = row_ptr[old], re = row_ptr[old + 1];
        if (big && re - rb > RELABEL_BIG) {                 // hub row: a whole block (k_relabel_big)
            if (lane == 0) big[atomicAdd(scalars + 15, 1)] = (int)i;
            continue;
        }
        const int ob = nrp[i];
        // packed arc: (relabelled neighbour << 5) | (row index within its 32-row group);
        // with pruning only arcs to live (unpeeled) neighbours, order kept
        int outn = 0;
        for (int j0 = rb; j0 < re; j0 += 32) {
            const int j = j0 + lane;
            const int u = j < re ? col[j] : 0;
            const bool keep = j < re && !(rem && rem[u]);
            const unsigned b = __ballot_sync(0xffffffffu, keep);
            if (keep) ncol[ob + outn + __popc(b & ((1u << lane) - 1u))] = (old_to_new[u] << 5) | (int)(i & 31);
            outn += __popc(b);
        }
        if (lane == 0 && outn > heavy_deg) heavy[atomicAdd(scalars + 3, 1)] = (int)i;
    }
}

// the listed hub rows, a block per row: 1024 arcs per round, kept positions (pruning drops arcs to
// peeled vertices, order kept) from a block-wide ballot scan
__global__ void __launch_bounds__(1024) k_relabel_big(const int32_t *__restrict__ row_ptr,
                                                      const int32_t *__restrict__ col, const int32_t *__restrict__ nrp,
                                                      const int32_t *__restrict__ new_to_old,
                                                      const int32_t *__restrict__ old_to_new, int32_t *__restrict__ ncol,
                                                      int32_t *heavy, int32_t *scalars, const int32_t *rem,
                                                      const int32_t *big) {
    __shared__ int s_w[32];
    __shared__ int s_tot;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int heavy_deg = scalars[4];
    const int nbig = scalars[15];
    for (int b = blockIdx.x; b < nbig; b += gridDim.x) {
        const int i = big[b];
        const int old = new_to_old[i];
        const int rb = row_ptr[old], re = row_ptr[old + 1];
        const int ob = nrp[i];
        int outn = 0;
        for (int j0 = rb; j0 < re; j0 += 1024) {
            const int j = j0 + threadIdx.x;
            const int u = j < re ? col[j] : 0;
            const bool keep = j < re && !(rem && rem[u]);
            const int val = keep ? ((old_to_new[u] << 5) | (i & 31)) : 0;
            const unsigned bm = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) s_w[wib] = __popc(bm);
            __syncthreads();
            if (wib == 0) {
                const int x = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0;
                int incl = x;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                s_w[lane] = incl - x;
                if (lane == 31) s_tot = incl;
            }
            __syncthreads();
            if (keep) ncol[ob + outn + s_w[wib] + __popc(bm & ((1u << lane) - 1u))] = val;
            outn += s_tot;
            __syncthreads();
        }
        if (threadIdx.x == 0 && outn > heavy_deg) heavy[atomicAdd(scalars + 3, 1)] = i;
    }
}

// items per heavy row (in place of the prefix the MS-BFS kernel reads): ceil(deg / BFS_HEAVY_CHUNK)
// for h < n_heavy (device count, at most `bound`), 0 for n_heavy <= h <= bound
__global__ void k_heavy_items(const int32_t *heavy, const int32_t *nrp, const int32_t *n_heavy_dev, int bound,
                              int32_t *items) {
    const int n_heavy = min(*n_heavy_dev, bound);
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h <= bound; h += gridDim.x * blockDim.x) {
        int n = 0;
        if (h < n_heavy) {
            const int v = heavy[h];
            n = (nrp[v + 1] - nrp[v] + BFS_HEAVY_CHUNK - 1) / BFS_HEAVY_CHUNK;
        }
        items[h] = n;
    }
}

// heavy-row threshold into scalars[4]: `param`, or (param <= 0, auto) 256 on graphs of average degree
// >= 8 and 64 on sparser ones, from the exact arc count row_ptr[V] (on the device: an AND graph's
// count is not known on the host)
__global__ void k_heavy_threshold(const int32_t *row_ptr, int V, int param, int32_t *scalars) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    int h = param;
    if (h <= 0) h = ((int64_t)row_ptr[V] >= (int64_t)8 * V) ? 256 : 64;
    scalars[4] = h < BFS_MAX_LIGHT_DEG ? h : BFS_MAX_LIGHT_DEG;
}

// upper bound on the MS-BFS rows: vertices with an edge that were not peeled
__global__ void k_count_rows(const int32_t *row_ptr, const int32_t *rem, int V, int32_t *out) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        const bool live = row_ptr[v + 1] > row_ptr[v] && !(rem && rem[v]);
        const unsigned b = __ballot_sync(__activemask(), live);
        if ((threadIdx.x & 31) == __ffs(__activemask()) - 1 && b) atomicAdd(out, __popc(b));
    }
}

// hanging-tree size T of every BFS row (weights of the pruned MS-BFS)
__global__ void k_row_T(const int32_t *new_to_old, const uint32_t *tsz, const int32_t *scalars, uint32_t *T) {
    const int n_live = scalars[0];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_live; i += gridDim.x * blockDim.x)
        T[i] = tsz[new_to_old[i]] - 1u;
}

// union CSR of several graphs: graph g's vertex v becomes voff + v
// graph i of a fused union: its arcs start after the exact arc counts of graphs 0..i-1, read on the
// device (an AND graph's count lives only in its row_ptr[V]), so building the union needs no host
// round trip
constexpr int UNION_MAX = 64;
struct UnionEnds {
    const int32_t *end[UNION_MAX];   // &row_ptr_j[V_j] of the graphs before this one
    int n;
};
__global__ void k_union_copy(const int32_t *__restrict__ rp, const int32_t *__restrict__ col, int V, UnionEnds pre,
                             int voff, int32_t *rp_u, int32_t *col_u) {
    int64_t aoff = 0;
    for (int k = 0; k < pre.n; ++k) aoff += *pre.end[k];
    const int64_t nnz = rp[V];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= V; i += (int64_t)gridDim.x * blockDim.x)
        rp_u[voff + i] = (int32_t)(rp[i] + aoff);
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x)
        col_u[aoff + j] = col[j] + voff;
}

// per-graph finalize; union arrays are indexed at voff + v
// S from the relabelled accumulators (S_orig == nullptr) or given in original order
// (hm_closeness_combine: the sum of the shards' partial sums).
__global__ void k_finalize(const int32_t *old_to_new, const int32_t *label, const int32_t *csize,
                           const int32_t *row_ptr, const uint64_t *S_rel, const int32_t *scalars,
                           const uint64_t *S_orig,
                           uint64_t *S, int32_t *kk, double *c, uint64_t *pen, int32_t *deg, int V, int voff,
                           unsigned long long *acc, int32_t *cnt) {
    // the exact sum of c for the mean (reading Z6): block-local 16-bit-half limbs, flushed to acc
    // (at most EXACT_MAX_PER_BLOCK values per block)
    __shared__ unsigned s16[2 * EXACT_NLIMB];
    for (int i = threadIdx.x; i < 2 * EXACT_NLIMB; i += blockDim.x) s16[i] = 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) *cnt = 0;
    __syncthreads();
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        uint64_t s;
        if (S_orig) {
            s = S_orig[v];
        } else {
            const int i = old_to_new[voff + v];
            s = (i < scalars[0]) ? S_rel[i] : 0ull;
        }
        const int k = csize[label[voff + v]];
        // Wasserman-Faust closeness exactly as NetworkX evaluates it:
        // ((k-1)/S) * ((k-1)/(V-1)), binary64 RN, 0 if S == 0 or V <= 1.
        double cv = 0.0;
        if (s > 0ull && V > 1) {
            const double t1 = __ddiv_rn((double)(k - 1), (double)s);
            const double t2 = __ddiv_rn((double)(k - 1), (double)(V - 1));
            cv = __dmul_rn(t1, t2);
        }
        S[v] = s;
        kk[v] = k;
        c[v] = cv;
        pen[v] = s + (uint64_t)(V - k) * (uint64_t)V;   // n-penalty sum
        deg[v] = row_ptr[v + 1] - row_ptr[v];
        exact_add16(s16, cv);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < EXACT_NLIMB; i += blockDim.x) {
        const unsigned long long x = exact_limb16(s16, i);
        if (x) atomicAdd(&acc[i], x);
    }
}

// mu = RN(exact sum of c) / V (every block rounds the limbs itself; block 0 stores mu), then the CH
// bitmap: bit v set iff c[v] > mu (strict), popcount into *count
__global__ void k_mu_bitmap(const unsigned long long *acc, const double *c, uint32_t *bm, double *mu_out,
                            int32_t *count, int V) {
    __shared__ double s_mu;
    if (threadIdx.x == 0) {
        s_mu = __ddiv_rn(exact_round(acc), (double)V);
        if (blockIdx.x == 0) *mu_out = s_mu;
    }
    __syncthreads();
    const double m = s_mu;
    const int lane = threadIdx.x & 31;
    for (int64_t vb = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31LL; vb < V;
         vb += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = vb + lane;
        const bool in = v < V && c[v] > m;
        const unsigned b = __ballot_sync(0xffffffffu, in);
        if (lane == 0) {
            bm[vb >> 5] = b;
            if (b) atomicAdd(count, __popc(b));
        }
    }
}

// a shard's partial target-side sums in original vertex order (0 for isolated vertices)
__global__ void k_partial_sums(const int32_t *old_to_new, const uint64_t *S_rel, const int32_t *scalars,
                               uint64_t *S_out, int V) {
    const int n_live = scalars[0];
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        const int i = old_to_new[v];
        S_out[v] = (i < n_live) ? S_rel[i] : 0ull;
    }
}


// ---------------------------------------------------------------------------------------------
// Small graphs (V <= SMALL_V, one graph, no pruning): the whole pre-processing (components,
// component order, relabelling, packed CSR, heavy list) and the whole post-processing (finalize,
// exact mean, CC-node bitmap) each run in ONE CTA out of shared memory, instead of ~30 grid-wide
// launches that a 1000-vertex graph cannot fill (C1: the step is launch-bound).
constexpr int SMALL_V = 4096;
constexpr int SMALL_T = 1024;

__device__ __forceinline__ int s_find(int *p, int x) {
    while (true) {
        const int px = p[x];
        if (px == x) return x;
        const int ppx = p[px];
        if (ppx != px) p[x] = ppx;     // path halving: ppx is an ancestor of x
        x = px;
    }
}

// in-place exclusive scan of a[0..n) by one CTA of SMALL_T threads; returns the total
__device__ int s_excl_scan(int *a, int n, int *ws) {
    const int per = (n + SMALL_T - 1) / SMALL_T;
    const int b0 = threadIdx.x * per, b1 = min(n, b0 + per);
    int sum = 0;
    for (int i = b0; i < b1; ++i) sum += a[i];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) ws[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int w = ws[lane];                       // SMALL_T / 32 == 32 warps
        int wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        ws[lane] = wi - w;
        if (lane == 31) ws[32] = wi;
    }
    __syncthreads();
    int run = ws[wid] + incl - sum;
    for (int i = b0; i < b1; ++i) {
        const int x = a[i];
        a[i] = run;
        run += x;
    }
    const int total = ws[32];
    __syncthreads();
    return total;
}

// ascending bitonic sort of P (a power of two) 64-bit keys in shared memory
__device__ void s_bitonic(uint64_t *k, int P) {
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P; i += SMALL_T) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const uint64_t a = k[i], b = k[j];
                    if (up ? (a > b) : (a < b)) {
                        k[i] = b;
                        k[j] = a;
                    }
                }
            }
            __syncthreads();
        }
}

// Same outputs as steps 1-3 of closeness_multi (no pruning): label / csize by root id, the
// component table (size_s, cstart), n2o / o2n, cinfo, the relabelled packed CSR, the heavy list
// and scalars [0] n_live [1] n_giant [2] n_comp [3] n_heavy [4] heavy threshold.
__global__ void __launch_bounds__(SMALL_T) k_small_prep(const int32_t *__restrict__ rp, const int32_t *__restrict__ col,
                                                        int V, int P, int sh, int heavy_param, int32_t *label,
                                                        int32_t *csize, int32_t *size_s, int32_t *cstart,
                                                        int32_t *n2o, int32_t *o2n, int32_t *nrp, int2 *cinfo,
                                                        int32_t *ncol, int32_t *heavy, int32_t *scalars,
                                                        int32_t *hstart) {
    extern __shared__ unsigned long long s_mem[];
    uint64_t *key = reinterpret_cast<uint64_t *>(s_mem);             // [P]
    int *par = reinterpret_cast<int *>(key + P);                       // [V] parent, then label
    int *lab = par + V;                                                // [V] label
    int *csz = lab + V;                                                // [V] size by root id
    int *aux = csz + V;                                                // [V + 1] rank of root / degrees
    int *ssz = aux + V + 1;                                            // [V + 1] size by rank, then cstart
    int *ws = ssz + V + 1;                                             // [33] scan scratch
    __shared__ int s_ncomp, s_nlive;
    const uint64_t lo = (1ull << sh) - 1ull;
    for (int v = threadIdx.x; v < V; v += SMALL_T) {
        par[v] = v;
        csz[v] = 0;
    }
    if (threadIdx.x == 0) {
        s_ncomp = 0;
        s_nlive = 0;
    }
    __syncthreads();
    // 1. components: lock-free union in shared memory (larger root under smaller)
    for (int u = threadIdx.x; u < V; u += SMALL_T)
        for (int j = rp[u]; j < rp[u + 1]; ++j) {
            const int w = col[j];
            if (w <= u) continue;
            int ru = s_find(par, u), rw = s_find(par, w);
            while (ru != rw) {
                if (ru < rw) { const int t = ru; ru = rw; rw = t; }
                const int old = atomicCAS(par + ru, ru, rw);
                if (old == ru) break;
                ru = s_find(par, old);
                rw = s_find(par, rw);
            }
        }
    __syncthreads();
    for (int v = threadIdx.x; v < V; v += SMALL_T) lab[v] = s_find(par, v);
    __syncthreads();
    for (int v = threadIdx.x; v < V; v += SMALL_T) {
        atomicAdd(csz + lab[v], 1);
        label[v] = lab[v];
    }
    __syncthreads();
    // 2. component order: (size desc, root asc); non-roots sort last
    for (int i = threadIdx.x; i < P; i += SMALL_T)
        key[i] = i < V ? ((lab[i] == i) ? (((uint64_t)(V - csz[i]) << sh) | (uint64_t)i) : ((uint64_t)V << sh))
                       : ~0ull;
    __syncthreads();
    s_bitonic(key, P);
    for (int i = threadIdx.x; i < V; i += SMALL_T) {
        csize[i] = csz[i];
        const uint64_t k = key[i];
        if ((k >> sh) < (uint64_t)V) {
            ssz[i] = V - (int)(k >> sh);
            aux[(int)(k & lo)] = i;                                     // rank of the root
            if (i + 1 == V || (key[i + 1] >> sh) >= (uint64_t)V) s_ncomp = i + 1;
        } else {
            ssz[i] = 0;
        }
    }
    __syncthreads();
    const int n_comp = s_ncomp;
    for (int i = threadIdx.x; i < V; i += SMALL_T) size_s[i] = ssz[i];
    __syncthreads();
    s_excl_scan(ssz, V, ws);                                            // ssz := cstart
    for (int i = threadIdx.x; i < n_comp; i += SMALL_T) {
        const int sz = size_s[i];
        if (sz > 1 && (i + 1 == n_comp || size_s[i + 1] <= 1)) s_nlive = ssz[i] + sz;
    }
    for (int i = threadIdx.x; i < V; i += SMALL_T) cstart[i] = ssz[i];
    __syncthreads();
    // vertex order: (component rank, id)
    for (int i = threadIdx.x; i < P; i += SMALL_T)
        key[i] = i < V ? (((uint64_t)aux[lab[i]] << sh) | (uint64_t)i) : ~0ull;
    __syncthreads();
    s_bitonic(key, P);
    for (int i = threadIdx.x; i < V; i += SMALL_T) {
        const int old = (int)(key[i] & lo);
        const int r = (int)(key[i] >> sh);
        n2o[i] = old;
        o2n[old] = i;
        aux[i] = rp[old + 1] - rp[old];                                 // new degree
        cinfo[i] = make_int2(ssz[r], size_s[r]);
    }
    if (threadIdx.x == 0) aux[V] = 0;
    __syncthreads();
    const int nnz = s_excl_scan(aux, V + 1, ws);                        // aux := relabelled row_ptr
    for (int i = threadIdx.x; i <= V; i += SMALL_T) nrp[i] = aux[i];
    int hd = heavy_param;
    if (hd <= 0) hd = ((int64_t)nnz >= (int64_t)8 * V) ? 256 : 64;
    if (hd > BFS_MAX_LIGHT_DEG) hd = BFS_MAX_LIGHT_DEG;
    __syncthreads();
    // 3. packed arcs (relabelled neighbour << 5 | row & 31), heavy rows
    const int n_live = s_nlive;
    for (int i = threadIdx.x; i < n_live; i += SMALL_T) {
        const int old = (int)(key[i] & lo);
        const int rb = rp[old], re = rp[old + 1], ob = aux[i];
        for (int j = rb; j < re; ++j) ncol[ob + (j - rb)] = (o2n[col[j]] << 5) | (i & 31);
        if (re - rb > hd) heavy[atomicAdd(scalars + 3, 1)] = i;
    }
    if (threadIdx.x == 0) {
        scalars[0] = n_live;
        scalars[1] = size_s[0] > 1 ? size_s[0] : 0;
        scalars[2] = n_comp;
        scalars[4] = hd;
    }
    __syncthreads();
    if (hstart && threadIdx.x == 0) {                 // heavy-row work items: their prefix (few rows)
        const int nh = scalars[3];
        int acc = 0;
        hstart[0] = 0;
        for (int h = 0; h < nh; ++h) {
            const int v = heavy[h];
            acc += (aux[v + 1] - aux[v] + BFS_HEAVY_CHUNK - 1) / BFS_HEAVY_CHUNK;
            hstart[h + 1] = acc;
        }
    }
}

// finalize (S, k, WF closeness, n-penalty sum, degree), exact mean and CH bitmap in one CTA
__global__ void __launch_bounds__(SMALL_T) k_small_finish(const int32_t *o2n, const int32_t *label,
                                                          const int32_t *csize, const int32_t *row_ptr,
                                                          const uint64_t *S_rel, const int32_t *scalars,
                                                          uint64_t *S, int32_t *kk, double *c, uint64_t *pen,
                                                          int32_t *deg, uint32_t *bm, double *mu_out,
                                                          int32_t *cnt_out, int V) {
    __shared__ unsigned s16[2 * EXACT_NLIMB];
    __shared__ unsigned long long acc[EXACT_NLIMB];
    __shared__ double s_mu;
    __shared__ int s_cnt;
    for (int i = threadIdx.x; i < 2 * EXACT_NLIMB; i += SMALL_T) s16[i] = 0u;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    const int n_live = scalars[0];
    for (int v = threadIdx.x; v < V; v += SMALL_T) {
        const int i = o2n[v];
        const uint64_t sv = i < n_live ? S_rel[i] : 0ull;
        const int k = csize[label[v]];
        double cv = 0.0;                 // Wasserman-Faust, the NetworkX order
        if (sv > 0ull && V > 1) {
            const double t1 = __ddiv_rn((double)(k - 1), (double)sv);
            const double t2 = __ddiv_rn((double)(k - 1), (double)(V - 1));
            cv = __dmul_rn(t1, t2);
        }
        S[v] = sv;
        kk[v] = k;
        c[v] = cv;
        pen[v] = sv + (uint64_t)(V - k) * (uint64_t)V;      // n-penalty sum
        deg[v] = row_ptr[v + 1] - row_ptr[v];
        exact_add16(s16, cv);                                 // V <= SMALL_V < 2^16 values: exact
    }
    __syncthreads();
    for (int i = threadIdx.x; i < EXACT_NLIMB; i += SMALL_T) acc[i] = exact_limb16(s16, i);
    __syncthreads();
    if (threadIdx.x == 0) s_mu = __ddiv_rn(exact_round(acc), (double)V);   // mu = RN(sum c) / V (Z6)
    __syncthreads();
    const double m = s_mu;
    const int lane = threadIdx.x & 31;
    for (int vb = threadIdx.x & ~31; vb < V; vb += SMALL_T) {              // CH = {v : c(v) > mu}
        const int v = vb + lane;
        const bool in = v < V && c[v] > m;
        const unsigned b = __ballot_sync(0xffffffffu, in);
        if (lane == 0) {
            bm[vb >> 5] = b;
            if (b) atomicAdd(&s_cnt, __popc(b));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *mu_out = m;
        *cnt_out = s_cnt;
    }
}

inline int nbits(uint64_t x) {
    int b = 0;
    while (x) { ++b; x >>= 1; }
    return b;
}

}  // namespace

// 5.-6. finalize one graph: S, k, WF closeness, n-penalty sum, degree; exact mean; CH bitmap
static void finalize_graph(hm_ctx *ctx, Graph &G, const int32_t *o2n, const int32_t *label, const int32_t *csize,
                           const uint64_t *S_rel, const int32_t *scalars, const uint64_t *S_orig, int voff) {
    cudaStream_t s = ctx->stream;
    const int Vg = G.V;
    uint32_t *chbm = G.ch.as<uint32_t>();
    const size_t nbw = (size_t)(Vg + 31) / 32;
    double *d_mu = reinterpret_cast<double *>(reinterpret_cast<char *>(chbm) + ((nbw * 4 + 7) / 8) * 8);
    int32_t *d_cnt = reinterpret_cast<int32_t *>(d_mu + 1);
    Buf acc((size_t)EXACT_NLIMB * 8, s);
    HM_CUDA(cudaMemsetAsync(acc.p, 0, acc.bytes, s));
    int64_t nb = grid_for(Vg, TB, (int64_t)ctx->num_sms * 16);
    const int64_t need = ((int64_t)Vg + EXACT_MAX_PER_BLOCK - 1) / EXACT_MAX_PER_BLOCK;
    if (nb < need) nb = need;
    // finalize + the exact sum of c in one pass; then mu and the CC-node bitmap in one pass
    k_finalize<<<(unsigned)nb, TB, 0, s>>>(
        o2n, label, csize, G.row_ptr.as<int32_t>(), S_rel, scalars, S_orig, G.S.as<uint64_t>(), G.k.as<int32_t>(),
        G.c.as<double>(), G.pen.as<uint64_t>(), G.deg.as<int32_t>(), Vg, voff, acc.as<unsigned long long>(), d_cnt);
    check_launch("k_finalize");
    k_mu_bitmap<<<grid_for((int64_t)Vg, TB, (int64_t)ctx->num_sms * 8), TB, 0, s>>>(
        acc.as<unsigned long long>(), G.c.as<double>(), chbm, d_mu, d_cnt, Vg);
    check_launch("k_mu_bitmap");
    count_launch(ctx, 2);
    G.has_results = true;
}

void closeness(hm_ctx *ctx, Graph &G) { closeness_multi(ctx, std::vector<Graph *>{&G}); }

// Fusing pays while the graphs are too small to fill the GPU one at a time (C2, 4 graphs of 16 K
// vertices: 3.24 -> 1.77 ms per step; C1, 3 graphs of 1000 vertices: 0.55 ms with three one-CTA
// small-path passes, 0.42 ms fused).  Larger graphs fill the grid on their own and keep their own
// pruning (the fused pass does not prune): C3's 14 graphs fused take 57.8 ms, separately 39.9.  Among
// them, graphs whose (cached) pruning decision is "no pruning" still gain from sharing level steps in
// groups of <= 2^20 vertices (C3's two ER layers: 17.4 -> 13.6 ms fused; C5's three layers: 195.9 ->
// 189.0 ms), while pruned ones lose (C3's R-MAT layers 6.8 -> 8.8, C4's layers 48.7 -> 65.0) and run
// one pass each.
constexpr int64_t FUSE_AUTO_MAX_V = (int64_t)1 << 17;
constexpr int64_t FUSE_GROUP_MAX_V = (int64_t)1 << 20;
static bool known_unpruned(hm_ctx *ctx, const Graph &g) {
    if (ctx->params.bfs_prune == 0 || (ctx->params.bfs_prune == 2 && g.V < 4096)) return true;
    const PruneDecision *d = g.and_key.empty()
                                 ? &g.pdec
                                 : (ctx->and_pdec.count(g.and_key) ? &ctx->and_pdec[g.and_key] : nullptr);
    return d && d->valid && !d->active;
}
void closeness_group(hm_ctx *ctx, const std::vector<Graph *> &gs) {
    int64_t Vs = 0;
    for (const Graph *g : gs) Vs += g->V;
    const int f = ctx->params.bfs_fuse;
    if (gs.size() > 1 && (f == 1 || (f == 2 && Vs <= FUSE_AUTO_MAX_V))) {
        closeness_multi(ctx, gs);
        return;
    }
    if (f == 2) {
        // graphs met for the first time: their pruning decision first (components + peeling + one round trip
        // each, as their own pass would take), so they can join a fused group in this very call
        for (Graph *g : gs) {
            const bool want = ctx->params.bfs_prune == 1 || (ctx->params.bfs_prune == 2 && g->V >= 4096);
            const PruneDecision *d = g->and_key.empty()
                                         ? &g->pdec
                                         : (ctx->and_pdec.count(g->and_key) ? &ctx->and_pdec[g->and_key] : nullptr);
            if (want && g->V < FUSE_GROUP_MAX_V && !(d && d->valid))
                closeness_multi(ctx, std::vector<Graph *>{g}, 0, 1, nullptr, nullptr, true);
        }
    }
    std::vector<Graph *> grp;                      // f == 2: groups of known-unpruned graphs
    int64_t gv = 0;
    auto flush = [&]() {
        if (grp.size() > 1) closeness_multi(ctx, grp);
        else if (grp.size() == 1) closeness_multi(ctx, std::vector<Graph *>{grp[0]});
        grp.clear();
        gv = 0;
    };
    for (Graph *g : gs) {
        if (f == 2 && g->V < FUSE_GROUP_MAX_V && known_unpruned(ctx, *g)) {
            if (gv + g->V > FUSE_GROUP_MAX_V) flush();
            grp.push_back(g);
            gv += g->V;
        } else {
            closeness_multi(ctx, std::vector<Graph *>{g});
        }
    }
    flush();
}

void closeness_partial(hm_ctx *ctx, Graph &G, int shard, int nshards, uint64_t *d_S_out) {
    closeness_multi(ctx, std::vector<Graph *>{&G}, shard, nshards, d_S_out, nullptr);
}

void closeness_combine(hm_ctx *ctx, Graph &G, const uint64_t *d_S_total) {
    closeness_multi(ctx, std::vector<Graph *>{&G}, 0, 1, nullptr, d_S_total);
}

// Psi for several graphs in one fused pass over their disjoint union (each
// graph is its own set of components; the MS-BFS batches all of them
// together, so the per-level costs are shared).  Results are per graph.
//
// Sharding: with d_S_partial the MS-BFS runs only the batches
// i = shard, shard + nshards, ... and the raw partial sums are written out instead of
// being finalised; with d_S_total the MS-BFS is skipped and the graph is finalised from
// the given (summed) sums.  Both are single-graph modes.
// decide_only: one graph, components and the pruning decision only (cached with the graph), nothing else
void closeness_multi(hm_ctx *ctx, const std::vector<Graph *> &gs, int shard, int nshards, uint64_t *d_S_partial,
                     const uint64_t *d_S_total, bool decide_only) {
    cudaStream_t s = ctx->stream;
    HM_REQUIRE(!gs.empty(), HM_EINVAL, "no graphs");
    HM_REQUIRE(nshards >= 1 && shard >= 0 && shard < nshards, HM_EINVAL, "need 0 <= shard < nshards");
    HM_REQUIRE(!(d_S_partial || d_S_total) || gs.size() == 1, HM_EINVAL, "sharded closeness is per graph");
    int64_t Vu64 = 0, nnz_u = 0;
    for (Graph *g : gs) {
        Vu64 += g->V;
        // the union CSR concatenates arcs: sized by the host counts (an AND graph's is an upper bound;
        // the exact offsets are taken on the device, k_union_copy)
        nnz_u += g->nnz;
    }
    HM_REQUIRE(Vu64 < (1 << 26), HM_ERANGE, "hm_closeness supports sum V < 2^26 (packed arc format)");
    HM_REQUIRE(nnz_u < (int64_t)INT32_MAX, HM_ERANGE, "union of graphs too large for an int32 CSR");
    const int V = (int)Vu64;
    int W = ctx->params.bfs_words > 0 ? ctx->params.bfs_words : 64;   // 0 = auto (64, or 128 below)
    const unsigned gb = grid_for(V, TB, (int64_t)ctx->num_sms * 16);
    const unsigned gw = grid_for((int64_t)V * 32, TB, (int64_t)ctx->num_sms * 16);
    // sort keys are <= V: sh = bits of V (the small path packs (high << sh) | vertex in 2 sh bits)
    const int sh = nbits((uint64_t)V);

    // per-graph outputs
    for (Graph *g : gs) {
        const size_t Vg = (size_t)g->V;
        if (!g->S.p || g->S.bytes < Vg * 8) {
            g->S.alloc(Vg * 8, s);
            g->k.alloc(Vg * 4, s);
            g->c.alloc(Vg * 8, s);
            g->pen.alloc(Vg * 8, s);
            g->deg.alloc(Vg * 4, s);
            g->ch.alloc(((Vg + 31) / 32) * 4 + 8 + 8, s);   // bitmap + mu + count
        }
    }
    // union CSR (a single graph is used in place)
    Buf rp_ub, col_ub;
    const int32_t *rp_u = gs[0]->row_ptr.as<int32_t>();
    const int32_t *col_u = gs[0]->col.as<int32_t>();
    std::vector<int> voff(gs.size(), 0);
    if (gs.size() > 1) {
        rp_ub.alloc((size_t)(V + 1) * 4, s);
        col_ub.alloc((size_t)(nnz_u > 0 ? nnz_u : 1) * 4, s);
        HM_REQUIRE(gs.size() <= (size_t)UNION_MAX, HM_EINVAL, "hm_closeness_multi fuses at most 64 graphs");
        int vo = 0;
        UnionEnds pre{};
        for (size_t i = 0; i < gs.size(); ++i) {
            voff[i] = vo;
            const int64_t n = (int64_t)gs[i]->V + 1 > gs[i]->nnz ? (int64_t)gs[i]->V + 1 : gs[i]->nnz;
            pre.n = (int)i;
            k_union_copy<<<grid_for(n, TB, (int64_t)ctx->num_sms * 16), TB, 0, s>>>(
                gs[i]->row_ptr.as<int32_t>(), gs[i]->col.as<int32_t>(), gs[i]->V, pre, vo,
                rp_ub.as<int32_t>(), col_ub.as<int32_t>());
            pre.end[i] = gs[i]->row_ptr.as<int32_t>() + gs[i]->V;
            vo += gs[i]->V;
        }
        check_launch("k_union_copy");
        count_launch(ctx, (int)gs.size());
        rp_u = rp_ub.as<int32_t>();
        col_u = col_ub.as<int32_t>();
    }
    struct {
        int V;
        int64_t nnz;
        const int32_t *rp, *col;
    } U{V, nnz_u, rp_u, col_u};

    // pruning: on (1), off (0), or (2, default) on from V = 4096, below which its kernels and host
    // round trip cost more than the BFS they save (C1: 0.32 vs 0.26 ms per closeness call)
    const bool want_prune = ctx->params.bfs_prune == 1 || (ctx->params.bfs_prune == 2 && V >= 4096);
    // small graphs: one-CTA pre- and post-processing (k_small_prep / k_small_finish)
    const bool small = gs.size() == 1 && !d_S_partial && !d_S_total && V <= SMALL_V && !want_prune;
    // automatic batch width for small graphs: the narrowest rows whose batch still covers the graph
    // (C1, V = 1000: 1024 sources, 0.61 -> 0.57 ms per step)
    if (small && ctx->params.bfs_words == 0 && ctx->params.bfs_team == 0 && ctx->params.bfs_gd == 0 &&
        ctx->params.bfs_blocks_per_sm != 1)
        W = V <= 1024 ? 16 : V <= 2048 ? 32 : 64;

    bool t_ordered = false;               // the pruned core relabelled in T order (k_vert_keys)
    Buf parent((size_t)V * 4, s), label((size_t)V * 4, s), csize((size_t)V * 4, s);
    Buf key1((size_t)V * 8, s), key2((size_t)V * 8, s);
    Buf size_s((size_t)V * 4, s), cstart((size_t)V * 4, s), rank((size_t)V * 4, s);
    Buf n2o((size_t)V * 4, s), o2n((size_t)V * 4, s), ndeg((size_t)(V + 1) * 4, s);
    Buf nrp((size_t)(V + 1) * 4, s), cinfo((size_t)V * 8, s);
    Buf ncol((size_t)(U.nnz > 0 ? U.nnz : 1) * 4, s), heavy((size_t)V * 4, s);
    Buf scal(64, s);
    int32_t *scalars = scal.as<int32_t>();
    HM_CUDA(cudaMemsetAsync(scal.p, 0, 64, s));
    HM_CUDA(cudaMemsetAsync(csize.p, 0, csize.bytes, s));

    cudaEvent_t ph = phase_begin(ctx);
    Prune pr;
    const int32_t *rem = nullptr;
    const int heavy_param = ctx->params.bfs_heavy;
    // smallest threshold the device can pick (sizes the heavy-row bound below)
    const int heavy_min = heavy_param > 0 ? (heavy_param < BFS_MAX_LIGHT_DEG ? heavy_param : BFS_MAX_LIGHT_DEG) : 64;
    Buf hstart, hacc, hcnt;
    int32_t h_heavy_small = 0;
    if (small) {
        // heavy-row arrays sized by the bound nnz / (threshold + 1); the prep kernel fills the item prefix
        const int64_t bound = U.nnz / ((int64_t)heavy_min + 1);
        h_heavy_small = (int32_t)(bound < V ? bound : V);
        if (h_heavy_small > 0) hstart.alloc((size_t)(h_heavy_small + 1) * 4, s);
        int P = 1;
        while (P < V) P <<= 1;
        const size_t smem = (size_t)P * 8 + ((size_t)5 * V + 35) * 4;
        HM_CUDA(cudaFuncSetAttribute(k_small_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_small_prep<<<1, SMALL_T, smem, s>>>(U.rp, U.col, V, P, sh, heavy_param, label.as<int32_t>(),
                                              csize.as<int32_t>(), size_s.as<int32_t>(), cstart.as<int32_t>(),
                                              n2o.as<int32_t>(), o2n.as<int32_t>(), nrp.as<int32_t>(),
                                              cinfo.as<int2>(), ncol.as<int32_t>(), heavy.as<int32_t>(), scalars,
                                              h_heavy_small > 0 ? hstart.as<int32_t>() : nullptr);
        check_launch("k_small_prep");
        count_launch(ctx);
        phase_end(ctx, PH_RELABEL, ph);
        ph = phase_begin(ctx);
    } else {
    // 1. connected components (auto: the one-launch hooking pays from V = 32768 -- C5 layer 0.2 vs
    // 0.5-1.0 ms -- while its grid barriers cost more than they save on C2-sized graphs, 0.51 vs 0.30 ms)
    const int cc_init = ctx->params.cc_init == 4 ? (V >= 32768 ? 3 : 2) : ctx->params.cc_init;
    if (cc_init == 3) {
        // one cooperative launch (grid: what fits, at most 4 CTAs per SM)
        int per_sm = 0;
        HM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cc_sv, TB, 0));
        if (per_sm > 4) per_sm = 4;
        HM_REQUIRE(per_sm >= 1, HM_ECUDA, "k_cc_sv occupancy");
        int gc = (int)grid_for((int64_t)V * 2, TB, (int64_t)ctx->num_sms * per_sm);
        int32_t *fp = parent.as<int32_t>();
        int32_t *flg = scalars + 12;                                  // zeroed scalars block, [12..14]
        const int32_t *rpp = U.rp, *clp = U.col;
        int Vv = V;
        // arc-balanced rounds for graphs with hub rows (known from the graph's cached pruning round
        // trip: C3's R-MAT layers 360-470 -> 190-250 us), row groups otherwise (C5 layers 0.23 vs 0.30 ms)
        const PruneDecision *pd0 = gs.size() == 1 ? (gs[0]->and_key.empty() ? &gs[0]->pdec
                                                     : (ctx->and_pdec.count(gs[0]->and_key)
                                                            ? &ctx->and_pdec[gs[0]->and_key] : nullptr))
                                                  : nullptr;
        const bool hubs = pd0 && pd0->valid && pd0->maxdeg > 256;
        Buf rowof;
        if (hubs) rowof.alloc((size_t)(U.nnz > 0 ? U.nnz : 1) * 4, s);
        int32_t *rop = hubs ? rowof.as<int32_t>() : nullptr;
        void *args[] = {(void *)&rpp, (void *)&clp, (void *)&Vv, (void *)&fp, (void *)&flg, (void *)&rop};
        HM_CUDA(cudaLaunchCooperativeKernel((const void *)k_cc_sv, dim3(gc), dim3(TB), args, 0, s));
        count_launch(ctx);
    } else if (cc_init == 1) k_cc_init<<<gw, TB, 0, s>>>(U.rp, U.col, parent.as<int32_t>(), V);
    else k_iota<<<gb, TB, 0, s>>>(parent.as<int32_t>(), V);
    if (cc_init == 3) {
    } else if (cc_init == 2) {
        // csize doubles as the root-count scratch; scalars + 8 (zeroed) holds the giant pick
        unsigned long long *gbest = reinterpret_cast<unsigned long long *>(scalars + 8);
        k_cc_sample<<<gb, TB, 0, s>>>(U.rp, U.col, parent.as<int32_t>(), V);
        k_cc_root_counts<<<gb, TB, 0, s>>>(parent.as<int32_t>(), csize.as<int32_t>(), V);
        k_cc_giant<<<gb, TB, 0, s>>>(parent.as<int32_t>(), csize.as<int32_t>(), gbest, V);
        k_cc_rest<<<gw, TB, 0, s>>>(U.rp, U.col, parent.as<int32_t>(), V, gbest);
        HM_CUDA(cudaMemsetAsync(csize.p, 0, csize.bytes, s));
        count_launch(ctx, 3);
    } else {
        k_cc_union<<<gw, TB, 0, s>>>(U.rp, U.col, parent.as<int32_t>(), V);
    }
    k_cc_compress<<<gb, TB, 0, s>>>(parent.as<int32_t>(), label.as<int32_t>(), csize.as<int32_t>(), V);
    check_launch("cc");
    count_launch(ctx, 3);
    phase_end(ctx, PH_CC, ph);
    ph = phase_begin(ctx);

    // 1b. exact 2-core pruning of the largest component (prune.cu; single graph only)
    if (want_prune && gs.size() == 1) {
        Graph &G0 = *gs[0];
        PruneDecision *dec = G0.and_key.empty() ? &G0.pdec : &ctx->and_pdec[G0.and_key];
        prune_component(ctx, U.rp, U.col, label.as<int32_t>(), csize.as<int32_t>(), V, pr, dec);
    }
    if (decide_only) {
        phase_end(ctx, PH_PRUNE, ph);
        return;
    }
    rem = pr.active ? pr.rem.as<int32_t>() : nullptr;
    if (gs.size() > 1) {
        // a fused union's shape from its graphs' cached pruning decisions (all known: the automatic
        // grouping fuses only such graphs) -- the batch width and the lean kernel choice below
        bool all = true;
        int maxdeg = 0;
        int64_t arcs = 0, nonisol = 0;
        for (const Graph *g : gs) {
            const PruneDecision *d = g->and_key.empty()
                                         ? &g->pdec
                                         : (ctx->and_pdec.count(g->and_key) ? &ctx->and_pdec[g->and_key] : nullptr);
            if (!d || !d->valid) {
                all = false;
                break;
            }
            maxdeg = d->maxdeg > maxdeg ? d->maxdeg : maxdeg;
            arcs += d->arcs;
            nonisol += d->nonisolated;
        }
        if (all) {
            pr.shape_known = true;
            pr.maxdeg = maxdeg;
            pr.arcs = arcs;
            pr.nonisolated = (int)nonisol;
        }
    }
    phase_end(ctx, PH_PRUNE, ph);
    ph = phase_begin(ctx);

    if (d_S_total) {
        Graph &G = *gs[0];
        Buf Sfin((size_t)V * 8, s);
        HM_CUDA(cudaMemcpyAsync(Sfin.p, d_S_total, (size_t)V * 8, cudaMemcpyDeviceToDevice, s));
        if (pr.active) prune_finish(ctx, pr, label.as<int32_t>(), csize.as<int32_t>(), Sfin.as<uint64_t>(), V);
        finalize_graph(ctx, G, nullptr, label.as<int32_t>(), csize.as<int32_t>(), nullptr, scalars,
                       Sfin.as<uint64_t>(), 0);
        phase_end(ctx, PH_FINALIZE, ph);
        return;
    }

    // 2. component order and vertex order
    // (batching by live component sizes: the pruned component counts its core only)
    // (stable 32-bit key / 32-bit value radix sorts over nbits(V) bits: 3 passes at V = 2^16..2^24
    // instead of 64-bit composite keys over 2 nbits(V) bits)
    uint32_t *kin = key1.as<uint32_t>(), *vin = kin + V, *kout = key2.as<uint32_t>(), *vout = kout + V;
    k_comp_keys<<<gb, TB, 0, s>>>(label.as<int32_t>(), pr.active ? pr.lsize.as<int32_t>() : csize.as<int32_t>(),
                                  kin, vin, V);
    count_launch(ctx);
    {
        const int kbits = sh;                                      // keys <= V
        // pruned graphs: vertex keys carry the core's T order in 8 more bits (k_vert_keys) -- only without
        // hub rows: on R-MAT layers the large hanging trees hang off the hubs, and T order packs the hubs
        // into the first groups and source windows (C4's pruned layers 25.7 -> 30.6 ms with it)
        const int to = ctx->params.bfs_torder;
        const int kshift = (pr.active && sh + 8 <= 32 &&
                            (to == 2 || (to == 1 && pr.shape_known && pr.maxdeg <= 256))) ? 8 : 0;
        t_ordered = kshift != 0;
        size_t tb = 0;
        HM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, V, 0, kbits + kshift, s));
        size_t tb2 = 0;
        HM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, size_s.as<int32_t>(), cstart.as<int32_t>(), V + 1, s));
        if (tb2 > tb) tb = tb2;
        Buf tmp(tb, s);
        size_t tbs = tb;
        HM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tbs, kin, kout, vin, vout, V, 0, kbits, s));
        k_comp_tables<<<gb, TB, 0, s>>>(kout, vout, size_s.as<int32_t>(), rank.as<int32_t>(), scalars, V);
        tbs = tb;
        HM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tbs, size_s.as<int32_t>(), cstart.as<int32_t>(), V, s));
        k_nlive<<<gb, TB, 0, s>>>(size_s.as<int32_t>(), cstart.as<int32_t>(), scalars, V);
        k_vert_keys<<<gb, TB, 0, s>>>(label.as<int32_t>(), rank.as<int32_t>(), rem,
                                      kshift ? pr.tsz.as<uint32_t>() : nullptr, kin, vin, V);
        tbs = tb;
        HM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tbs, kin, kout, vin, vout, V, 0, kbits + kshift, s));
        k_perm<<<gb, TB, 0, s>>>(kout, vout, U.rp, pr.active ? pr.degl.as<int32_t>() : nullptr,
                                size_s.as<int32_t>(), cstart.as<int32_t>(), n2o.as<int32_t>(), o2n.as<int32_t>(),
                                ndeg.as<int32_t>(), cinfo.as<int2>(), V, kshift);
        tbs = tb;
        HM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tbs, ndeg.as<int32_t>(), nrp.as<int32_t>(), V + 1, s));
        check_launch("relabel");
        count_launch(ctx, 4 + 3 * 4 + 2);   // our kernels + CUB passes (approximate)
    }
    // 3. relabelled CSR + heavy list (rows heavier than the MS-BFS light path takes)
    // heavy-row threshold: bfs_heavy, or (0, auto) 256 on graphs of average degree >= 8 and 64 on
    // sparser ones, where a row of a few dozen arcs already stalls its warp's lock-step rounds
    // (heavy sweep over C2-C4 layers and AND graphs)
    k_heavy_threshold<<<1, 32, 0, s>>>(U.rp, V, heavy_param, scalars);
    {
        // hub rows to k_relabel_big -- unless the graph's cached shape says it has none
        const PruneDecision *pdh = gs.size() == 1 ? (gs[0]->and_key.empty() ? &gs[0]->pdec
                                                      : (ctx->and_pdec.count(gs[0]->and_key)
                                                             ? &ctx->and_pdec[gs[0]->and_key] : nullptr))
                                                   : nullptr;
        const bool may_big = !(pdh && pdh->valid && pdh->maxdeg <= RELABEL_BIG);
        Buf bigl;
        if (may_big) bigl.alloc((size_t)(U.nnz / RELABEL_BIG + 1) * 4, s);
        k_relabel_cols<<<gw, TB, 0, s>>>(U.rp, U.col, nrp.as<int32_t>(),
                                         n2o.as<int32_t>(), o2n.as<int32_t>(), ncol.as<int32_t>(),
                                         heavy.as<int32_t>(), scalars, rem, V, may_big ? bigl.as<int32_t>() : nullptr);
        check_launch("k_relabel_cols");
        count_launch(ctx, 2);
        if (may_big) {
            k_relabel_big<<<ctx->num_sms, 1024, 0, s>>>(U.rp, U.col, nrp.as<int32_t>(), n2o.as<int32_t>(),
                                                       o2n.as<int32_t>(), ncol.as<int32_t>(), heavy.as<int32_t>(),
                                                       scalars, rem, bigl.as<int32_t>());
            check_launch("k_relabel_big");
            count_launch(ctx);
        }
    }
    phase_end(ctx, PH_RELABEL, ph);
    ph = phase_begin(ctx);

    if (ctx->params.bfs_dbg & 2) {
        if (!ctx->dbgc.p) ctx->dbgc.alloc(335872 * 8, s);
        const size_t nn = (size_t)(V < 65536 ? V : 65536);
        HM_CUDA(cudaMemcpyAsync(ctx->dbgc.as<char>() + 139264 * 8, n2o.p, nn * 4, cudaMemcpyDeviceToDevice, s));
        HM_CUDA(cudaMemcpyAsync(ctx->dbgc.as<char>() + (139264 + 65536) * 8, nrp.p, nn * 4,
                                cudaMemcpyDeviceToDevice, s));
        HM_CUDA(cudaMemcpyAsync(ctx->dbgc.as<char>() + (139264 + 2 * 65536) * 8, key2.p, nn * 4,
                                cudaMemcpyDeviceToDevice, s));
    }
    }   // !small

    // 4. MS-BFS
    size_t rowb = (size_t)W * 8;
    // frontier rows only for vertices that can be BFS rows (an edge, not peeled): large sparse
    // graphs (many isolated vertices) need far less than V rows of state
    int64_t frows = V;
    int32_t h_heavy = 0;
    // graphs of <= 256 MB of visited-set rows at V rows -- or <= 4 GB when the graph's shape is known from its
    // (cached) pruning decision, e.g. a fused group of C5's layers -- skip the row count and its host round
    // trip: F is sized for V rows and the heavy-row arrays for the bound nnz / (heavy_deg + 1)
    const int64_t state_bytes = (int64_t)V * (int64_t)rowb * 2;
    const bool count_rows = state_bytes > ((int64_t)4 << 30) || (!pr.shape_known && state_bytes > ((int64_t)256 << 20));
    if (!count_rows) {
        if (frows < 32) frows = 32;                                  // as the counted path
        const int64_t bound = U.nnz / ((int64_t)heavy_min + 1);
        h_heavy = (int32_t)(bound < V ? bound : V);
        if (pr.shape_known) {
            // the pruning round trip read the graph's shape: with no row above the heavy threshold
            // the lean kernel runs (no heavy-row arrays), and the batch width can be chosen
            const int hd = heavy_param > 0 ? heavy_min : (pr.arcs >= (int64_t)8 * V ? 256 : 64);
            if (pr.maxdeg <= hd) {
                h_heavy = 0;
                if (ctx->params.bfs_words == 0 && ctx->params.bfs_team == 0 && ctx->params.bfs_gd == 0 &&
                    ctx->params.bfs_blocks_per_sm != 1 && pr.arcs < (int64_t)4 * pr.nonisolated && V >= 65536) {
                    W = 128;                                         // see the counted path below
                    rowb = (size_t)W * 8;
                }
            }
        }
    } else {
        Buf cntb(16, s);
        HM_CUDA(cudaMemsetAsync(cntb.p, 0, 16, s));
        k_count_rows<<<gb, TB, 0, s>>>(U.rp, rem, V, cntb.as<int32_t>());
        check_launch("k_count_rows");
        count_launch(ctx);
        int32_t h_rows = 0, h_arcs = 0;
        HM_CUDA(cudaMemcpyAsync(&h_rows, cntb.p, 4, cudaMemcpyDeviceToHost, s));
        HM_CUDA(cudaMemcpyAsync(&h_heavy, scalars + 3, 4, cudaMemcpyDeviceToHost, s));
        HM_CUDA(cudaMemcpyAsync(&h_arcs, U.rp + V, 4, cudaMemcpyDeviceToHost, s));
        host_sync(ctx);
        // automatic batch width (bfs_words 0): 8192 sources per batch for sparse graphs without heavy
        // rows (average degree < 4: long, thin BFS -- the C5 AND graph 58.3 -> 50.2 ms, half the batches
        // and level barriers), 4096 otherwise (the C5 layers: 65.3 vs 85.9 ms at 8192)
        if (ctx->params.bfs_words == 0 && ctx->params.bfs_team == 0 && ctx->params.bfs_gd == 0 &&
            ctx->params.bfs_blocks_per_sm != 1 && h_heavy == 0 && (int64_t)h_arcs < (int64_t)4 * h_rows &&
            V >= 65536) {
            W = 128;
            rowb = (size_t)W * 8;
        }
        frows = (int64_t)h_rows + 32;
        if (frows > V) frows = V;
        if (frows < 32) frows = 32;
    }
    const size_t bmw = (((size_t)(V + 31) / 32) + 4) & ~(size_t)3;   // multiple of 4 words (16-B rows for uint4 copies)
    Buf F0((size_t)frows * rowb, s), F1((size_t)frows * rowb, s);
    Buf bms(bmw * 8 * 4, s), Srel((size_t)V * 8, s), Kb((size_t)V * 2 + 16, s), flags(128, s);
    HM_CUDA(cudaMemsetAsync(Srel.p, 0, Srel.bytes, s));
    HM_CUDA(cudaMemsetAsync(flags.p, 0, flags.bytes, s));
    BfsArgs a;
    a.row_ptr = nrp.as<int32_t>();
    a.col = ncol.as<int32_t>();
    a.cinfo = cinfo.as<int2>();
    a.comp_size = size_s.as<int32_t>();
    a.comp_start = cstart.as<int32_t>();
    a.scalars = scalars;
    a.heavy = heavy.as<int32_t>();
    // heavy-row work items: ceil(deg / BFS_HEAVY_CHUNK) per heavy row, their prefix, and the
    // partial-row accumulators of rows with several items
    a.hstart = nullptr;
    a.hacc = nullptr;
    a.hcnt = nullptr;
    a.hclaim = nullptr;
    if (h_heavy > 0) {
        if (!small) hstart.alloc((size_t)(h_heavy + 1) * 4, s);   // small graphs: filled by k_small_prep
        hacc.alloc((size_t)h_heavy * W * 8, s);
        hcnt.alloc((size_t)h_heavy * 4 + 16, s);
        HM_CUDA(cudaMemsetAsync(hacc.p, 0, hacc.bytes, s));
        HM_CUDA(cudaMemsetAsync(hcnt.p, 0, hcnt.bytes, s));
        if (!small) {
        k_heavy_items<<<grid_for(h_heavy + 1, TB, (int64_t)ctx->num_sms * 4), TB, 0, s>>>(
            heavy.as<int32_t>(), nrp.as<int32_t>(), scalars + 3, h_heavy, hstart.as<int32_t>());
        check_launch("k_heavy_items");
        count_launch(ctx);
        size_t tb = 0;
        HM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, hstart.as<int32_t>(), hstart.as<int32_t>(), h_heavy + 1, s));
        Buf tmp(tb, s);
        HM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, hstart.as<int32_t>(), hstart.as<int32_t>(), h_heavy + 1, s));
        count_launch(ctx, 2);
        }
        a.hstart = hstart.as<int32_t>();
        a.hacc = hacc.as<unsigned long long>();
        a.hcnt = hcnt.as<int32_t>();
        a.hclaim = a.hcnt + h_heavy;    // 3 claim counters after the per-row item counts (zeroed)
    }
    a.F[0] = F0.as<uint64_t>();
    a.F[1] = F1.as<uint64_t>();
    uint32_t *bm = bms.as<uint32_t>();
    for (int i = 0; i < 3; ++i) a.chg[i] = bm + i * bmw;
    a.done = bm + 3 * bmw;
    a.has = bm + 4 * bmw;
    a.par = bm + 5 * bmw;
    a.cand[0] = bm + 6 * bmw;
    a.cand[1] = bm + 7 * bmw;
    a.td_div = ctx->params.bfs_td;
    a.K = Kb.as<uint16_t>();
    a.chg_words = (int)bmw;
    a.hints = ctx->params.bfs_hints;
    Buf Trow, planes, tconst;
    a.tw = nullptr;
    a.planes = nullptr;
    a.tconst = nullptr;
    if (pr.active) {                    // weights 1 + T(s) of the pruned MS-BFS (prune.cu (1))
        Trow.alloc((size_t)V * 4, s);
        planes.alloc((size_t)BFS_T_BITS * W * 8, s);
        if (t_ordered) tconst.alloc((size_t)(W / 2) * 4 + 16, s);
        k_row_T<<<gb, TB, 0, s>>>(n2o.as<int32_t>(), pr.tsz.as<uint32_t>(), scalars, Trow.as<uint32_t>());
        check_launch("k_row_T");
        count_launch(ctx);
        a.tw = Trow.as<uint32_t>();
        a.planes = planes.as<unsigned long long>();
        a.tconst = t_ordered ? tconst.as<int32_t>() : nullptr;
    }
    a.shard = shard;
    a.nshards = nshards;
    a.interleave = ctx->params.bfs_interleave;
    a.dbg_level = ctx->params.bfs_dbg >> 8;                   // bfs_dbg bits 8.. (profiling builds)
    a.count_rows = ctx->params.bfs_count_rows;
    // top-down push phase (bfs_push): graphs without heavy rows, default kernels, counting barrier
    Buf plist0, plist1;
    a.push_num = 0;
    a.plist[0] = a.plist[1] = nullptr;
    a.pcur = nullptr;
    a.pcap = 0;
    // automatic (-1): on for the 8192-source batches of sparse graphs (C5 AND launch 44.6 -> 42.5 ms: its first
    // four levels 242 -> 129 us per batch), off at 4096 (C5 layer 65.0 -> 66.4 ms at best: a push level of 237 K pairs
    // costs more than the bottom-up level it replaces, and level 0 writes every row)
    const int push_par = ctx->params.bfs_push >= 0 ? ctx->params.bfs_push : (W == 128 ? 8 : 0);
    if (push_par > 0 && h_heavy == 0 && !a.count_rows && ctx->params.bfs_fbar && a.td_div == 0 &&
        ctx->params.bfs_team == 0 && ctx->params.bfs_gd == 0 && ctx->params.bfs_blocks_per_sm != 1 &&
        (W == 64 || W == 128)) {
        const int64_t cap = 2 * ((frows * (int64_t)push_par) / 4) + 64 * (int64_t)W + 1024;
        if (cap < ((int64_t)1 << 30)) {
            plist0.alloc((size_t)cap * 8, s);
            plist1.alloc((size_t)cap * 8, s);
            a.push_num = push_par;
            a.plist[0] = plist0.as<unsigned long long>();
            a.plist[1] = plist1.as<unsigned long long>();
            a.pcap = (int)cap;
        }
    }
    {
        // rows per work unit: bfs_unit, or (0, auto) about a quarter of the live rows per warp of
        // a full grid (2 CTAs x 14 warps per SM), as a power of two in [2, 32], 16 taken as 32.
        // Small graphs need small units to occupy the grid; C5-sized graphs the whole 32-row
        // groups (unit sweep over C1..C5)
        int unit = ctx->params.bfs_unit;
        if (unit <= 0) {
            const double q = (double)(frows - 32) / ((double)ctx->num_sms * 28.0) / 4.0;
            const int e = q > 1.0 ? (int)std::lround(std::log2(q)) : 0;
            unit = 1 << (e < 1 ? 1 : e > 5 ? 5 : e);
            if (unit == 16) unit = 32;
        }
        int us = 0;
        while ((32 >> us) > unit && us < 4) ++us;     // 32 >> us rows per unit
        a.unit_shift = us;
    }
    a.chg_smem = (ctx->params.bfs_chg_smem && bmw * 4 <= 80 * 1024) ? 1 : 0;
    a.S = Srel.as<uint64_t>();
    a.flags = flags.as<int32_t>();
    // fused level barrier: two zeroed counters in the same (zeroed) 128-B flags block
    a.lbar = ctx->params.bfs_fbar ? (unsigned long long *)((char *)flags.p + 64) : nullptr;
    a.pcur = (unsigned *)((char *)flags.p + 96);                // 3 zeroed list cursors after the barrier counters
    a.counters = ctx->dstats.as<unsigned long long>();
    a.dbgc = nullptr;
    if (ctx->params.bfs_dbg & 2) {
        if (!ctx->dbgc.p) {
            ctx->dbgc.alloc(335872 * 8, s);
        }
        HM_CUDA(cudaMemsetAsync(ctx->dbgc.p, 0, 139264 * 8, s));
        a.dbgc = ctx->dbgc.as<unsigned long long>();
    }
    phase_end(ctx, PH_BFS_SETUP, ph);
    ph = phase_begin(ctx);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->params.timing) {
        HM_CUDA(cudaEventCreate(&e0));
        HM_CUDA(cudaEventCreate(&e1));
        HM_CUDA(cudaEventRecord(e0, s));
    }
    // small graphs: no more CTAs than one light unit per warp (cheaper level barriers)
    const int64_t units = small ? ((frows + 31) / 32) << a.unit_shift : 0;
    const int grid = launch_msbfs(W, ctx->params.bfs_team, ctx->params.bfs_gd, a, ctx->num_sms,
                                  ctx->params.bfs_blocks_per_sm, s, units);
    if (grid == -1)                     // no instantiation for this (words, team, gathers, CTAs/SM)
        throw Error(HM_EINVAL, "no MS-BFS kernel for bfs_words=" + std::to_string(W) + " bfs_team=" +
                                   std::to_string(ctx->params.bfs_team) + " bfs_gd=" + std::to_string(ctx->params.bfs_gd) +
                                   " bfs_blocks_per_sm=" + std::to_string(ctx->params.bfs_blocks_per_sm) +
                                   " (see launch_msbfs in msbfs.cu for the built combinations)");
    if (grid < 0) {
        cudaGetLastError();
        throw Error(HM_ECUDA, "msbfs launch failed (" + std::to_string(grid) + ")");
    }
    check_launch("msbfs");
    if (ctx->params.timing) {
        HM_CUDA(cudaEventRecord(e1, s));
        ctx->pending.push_back({e0, e1});   // resolved in hm_get_stats (no sync here)
    }
    count_launch(ctx);
    ctx->stats.bfs_launches += 1;
    phase_end(ctx, PH_BFS, ph);
    ph = phase_begin(ctx);

    if (small) {
        Graph &G = *gs[0];
        const size_t nbw = (size_t)(V + 31) / 32;
        double *d_mu = reinterpret_cast<double *>(G.ch.as<char>() + ((nbw * 4 + 7) / 8) * 8);
        k_small_finish<<<1, SMALL_T, 0, s>>>(o2n.as<int32_t>(), label.as<int32_t>(), csize.as<int32_t>(),
                                            G.row_ptr.as<int32_t>(), Srel.as<uint64_t>(), scalars,
                                            G.S.as<uint64_t>(), G.k.as<int32_t>(), G.c.as<double>(),
                                            G.pen.as<uint64_t>(), G.deg.as<int32_t>(), G.ch.as<uint32_t>(), d_mu,
                                            reinterpret_cast<int32_t *>(d_mu + 1), V);
        check_launch("k_small_finish");
        count_launch(ctx);
        G.has_results = true;
        phase_end(ctx, PH_FINALIZE, ph);
        return;
    }
    if (d_S_partial) {
        k_partial_sums<<<grid_for(V, TB, (int64_t)ctx->num_sms * 16), TB, 0, s>>>(o2n.as<int32_t>(), Srel.as<uint64_t>(),
                                                                                 scalars, d_S_partial, V);
        check_launch("k_partial_sums");
        count_launch(ctx);
        phase_end(ctx, PH_FINALIZE, ph);
        return;
    }
    if (gs.size() == 1) {
        // S in original order (weighted core sums with pruning), then (1) + (2), then finalize
        Buf Sfin((size_t)V * 8, s);
        k_partial_sums<<<grid_for(V, TB, (int64_t)ctx->num_sms * 16), TB, 0, s>>>(o2n.as<int32_t>(),
                                                                                 Srel.as<uint64_t>(), scalars,
                                                                                 Sfin.as<uint64_t>(), V);
        check_launch("k_partial_sums");
        count_launch(ctx);
        if (pr.active) prune_finish(ctx, pr, label.as<int32_t>(), csize.as<int32_t>(), Sfin.as<uint64_t>(), V);
        finalize_graph(ctx, *gs[0], nullptr, label.as<int32_t>(), csize.as<int32_t>(), nullptr, scalars,
                       Sfin.as<uint64_t>(), 0);
        phase_end(ctx, PH_FINALIZE, ph);
        return;
    }
    for (size_t gi = 0; gi < gs.size(); ++gi)
        finalize_graph(ctx, *gs[gi], o2n.as<int32_t>(), label.as<int32_t>(), csize.as<int32_t>(), Srel.as<uint64_t>(),
                       scalars, nullptr, voff[gi]);
}

}  // namespace hm
