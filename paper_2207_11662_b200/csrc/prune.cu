// Exact 2-core pruning for all-sources closeness (an exactness-preserving work
// reduction of Psi; it changes no result).
//
// Hanging trees of the largest connected component P are peeled off round by
// round (a degree-1 vertex x is removed together with its edge to its unique
// live neighbour, the parent p(x)); what is left of P is its 2-core (or, for a
// tree, one vertex).  Removing a vertex of degree 1 changes no distance between
// the remaining vertices, so with
//   T(c) = number of peeled vertices hanging below core vertex c,
//   A(c) = sum over those vertices x of d(x, c),
// every core vertex u of P has
//   S(u) = sum_{core s} (1 + T(s)) d(s, u)  +  sum_{core c} A(c)          (1)
// (each peeled x reaches u through its core root c: d(x,u) = d(x,c) + d(c,u)),
// and every peeled vertex x, re-rooted from its parent (x's subtree of size
// size(x) moves one step closer, the other k - size(x) one step farther),
//   S(x) = S(p(x)) + k - 2 size(x)                                          (2)
// with k = |P|.  The multi-source BFS therefore runs on the core only and sums
// (1 + T(s)) per reached source s (msbfs.cu: bit planes of T); (1) adds the
// component constant and (2) runs top-down over the peeling rounds.
//
// Determinism: a round first marks every live degree-1 vertex of P (of two
// such vertices joined by P's last edge only the larger id goes), then each
// marked vertex takes its unique live neighbour as parent.  Everything is
// integer arithmetic, so the result is the same bit for bit as without pruning.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "msbfs.cuh"

namespace cg = cooperative_groups;

namespace hm {
namespace {

constexpr int TB = 256;

// P = the largest component (ties: smallest root); key = size << 32 | (V - 1 - root)
// (warp max first: graphs with many isolated vertices have as many roots, and one global atomicMax
// per root serialises on `best`)
__global__ void k_pick_largest(const int32_t *label, const int32_t *csize, unsigned long long *best, int V) {
    const int stride = gridDim.x * blockDim.x;
    for (int v0 = blockIdx.x * blockDim.x; v0 < V; v0 += stride) {      // warp-uniform trip count
        const int v = v0 + threadIdx.x;
        unsigned long long k = 0ull;
        if (v < V && label[v] == v) k = ((unsigned long long)csize[v] << 32) | (unsigned)(V - 1 - v);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, k, o);
            k = y > k ? y : k;
        }
        if ((threadIdx.x & 31) == 0 && k) atomicMax(best, k);
    }
}

__device__ __forceinline__ int live_neighbour(const int32_t *rp, const int32_t *col, const int32_t *rem, int v,
                                              int also_live_round) {
    for (int j = rp[v]; j < rp[v + 1]; ++j) {
        const int u = col[j];
        const int ru = *((volatile const int32_t *)(rem + u));
        if (ru == 0 || ru == also_live_round) return u;
    }
    return -1;
}

// persistent cooperative peeling of component P; scal[0] = rounds R, scal[1] = peeled vertices
__global__ void k_peel(const int32_t *__restrict__ rp, const int32_t *__restrict__ col, const int32_t *label,
                       const unsigned long long *best, int V, int32_t *rem, int32_t *par, uint32_t *tsz,
                       unsigned long long *tD, int32_t *degl, int32_t *flags, int32_t *scal) {
    cg::grid_group grid = cg::this_grid();
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int P = V - 1 - (int)(*best & 0xffffffffull);
    for (int64_t v = gtid; v < V; v += nth) {
        degl[v] = rp[v + 1] - rp[v];
        rem[v] = 0;
        par[v] = -1;
        tsz[v] = 1u;
        tD[v] = 0ull;
    }
    if (gtid == 0) {
        flags[0] = flags[1] = 0;
        scal[0] = scal[1] = 0;
    }
    grid.sync();
    for (int r = 1;; ++r) {
        // A: mark the live degree-1 vertices of P (of a last edge, only the larger end)
        int marked = 0;
        for (int64_t v = gtid; v < V; v += nth) {
            if (label[v] != P || rem[v] != 0 || degl[v] != 1) continue;
            const int u = live_neighbour(rp, col, rem, (int)v, r);
            if (u < 0) continue;
            if (degl[u] == 1 && u > v) continue;          // the pair's smaller end stays
            rem[v] = r;
            ++marked;
        }
        if (marked) atomicAdd(flags + (r & 1), marked);
        grid.sync();
        const int nr = *((volatile int32_t *)(flags + (r & 1)));
        if (nr == 0) break;
        // B: hang each marked vertex (complete subtree) on its unique live neighbour
        for (int64_t v = gtid; v < V; v += nth) {
            if (rem[v] != r) continue;
            const int u = live_neighbour(rp, col, rem, (int)v, -1);
            par[v] = u;
            atomicSub(degl + u, 1);
            atomicAdd(tsz + u, tsz[v]);
            atomicAdd(tD + u, tD[v] + (unsigned long long)tsz[v]);
        }
        if (gtid == 0) {
            flags[(r + 1) & 1] = 0;
            scal[0] = r;
            scal[1] += nr;
        }
        grid.sync();
    }
}

// live size per component root; stats: [0] lsize of P, [1] largest other component, [2] max T in P
__global__ void k_prune_stats(const int32_t *label, const int32_t *csize, const int32_t *rem, const uint32_t *tsz,
                              const unsigned long long *best, int32_t *lsize, unsigned long long *Cc,
                              const unsigned long long *tD, int32_t *stats, int V) {
    const int P = V - 1 - (int)(*best & 0xffffffffull);
    const int lane = threadIdx.x & 31;
    const int stride = gridDim.x * blockDim.x;
    for (int v0 = blockIdx.x * blockDim.x; v0 < V; v0 += stride) {      // warp-uniform trip count
        const int v = v0 + threadIdx.x;
        const bool in = v < V;
        const int l = in ? label[v] : -1;
        const bool live = in && rem[v] == 0;
        if (live) {
            const unsigned act = __activemask();
            const unsigned same = __match_any_sync(act, l);                 // warp-aggregated count
            if (lane == __ffs(same) - 1) atomicAdd(lsize + l, __popc(same));
        }
        // warp-aggregated: max T over P's core, (1) the component constant of P, the largest other root
        const bool inP = live && l == P;
        const unsigned tmax = __reduce_max_sync(0xffffffffu, inP ? tsz[v] - 1u : 0u);
        unsigned long long td = inP ? tD[v] : 0ull;
        const unsigned omax = __reduce_max_sync(0xffffffffu, (in && l == v && v != P) ? (unsigned)csize[v] : 0u);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) td += __shfl_xor_sync(0xffffffffu, td, o);
        const bool anyP = __any_sync(0xffffffffu, inP);
        if (lane == 0) {
            if (anyP) atomicMax(stats + 2, (int)tmax);
            if (td) atomicAdd(Cc + P, td);
            if (omax) atomicMax(stats + 1, (int)omax);
        }
    }
}

// graph shape for the host decisions taken at the same round trip: [0] max degree, [1] vertices
// with an edge, [2] arcs
__global__ void k_graph_stats(const int32_t *rp, int V, int32_t *out) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        const int deg = rp[v + 1] - rp[v];
        const unsigned act = __activemask();
        const int mx = (int)__reduce_max_sync(act, (unsigned)deg);
        const unsigned ne = __ballot_sync(act, deg > 0);
        if ((threadIdx.x & 31) == __ffs(act) - 1) {
            atomicMax(out + 0, mx);
            if (ne) atomicAdd(out + 1, __popc(ne));
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[2] = rp[V];
}

// (1) constant, then (2) top-down over the peeling rounds; S in original order
__global__ void k_prune_finish(const int32_t *label, const int32_t *csize, const int32_t *rem, const int32_t *par,
                               const uint32_t *tsz, const unsigned long long *Cc, const int32_t *scal,
                               unsigned long long *S, int V) {
    cg::grid_group grid = cg::this_grid();
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = gtid; v < V; v += nth)
        if (rem[v] == 0) S[v] += Cc[label[v]];
    grid.sync();
    for (int r = scal[0]; r >= 1; --r) {
        for (int64_t v = gtid; v < V; v += nth) {
            if (rem[v] != r) continue;
            const unsigned long long k = (unsigned long long)csize[label[v]];
            S[v] = S[par[v]] + k - 2ull * (unsigned long long)tsz[v];
        }
        grid.sync();
    }
}

int coop_grid(const void *kern, int threads, int num_sms) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, 0) != cudaSuccess || b < 1) return -1;
    return num_sms * (b < 4 ? b : 4);
}

}  // namespace

bool prune_component(hm_ctx *ctx, const int32_t *rp, const int32_t *col, const int32_t *label, const int32_t *csize,
                     int V, Prune &pr, PruneDecision *dec) {
    cudaStream_t s = ctx->stream;
    pr.active = false;
    if (V < 3) return false;
    pr.rem.alloc((size_t)V * 4, s);
    pr.par.alloc((size_t)V * 4, s);
    pr.tsz.alloc((size_t)V * 4, s);
    pr.tD.alloc((size_t)V * 8, s);
    pr.degl.alloc((size_t)V * 4, s);
    pr.lsize.alloc((size_t)V * 4, s);
    pr.Cc.alloc((size_t)V * 8, s);
    pr.scal.alloc(64, s);
    HM_CUDA(cudaMemsetAsync(pr.scal.p, 0, 64, s));
    HM_CUDA(cudaMemsetAsync(pr.lsize.p, 0, pr.lsize.bytes, s));
    HM_CUDA(cudaMemsetAsync(pr.Cc.p, 0, pr.Cc.bytes, s));
    unsigned long long *best = reinterpret_cast<unsigned long long *>(pr.scal.as<char>() + 32);
    int32_t *scal = pr.scal.as<int32_t>();           // [0] R, [1] peeled, [2..3] flags, [4..6] stats
    const unsigned gb = grid_for(V, TB, (int64_t)ctx->num_sms * 16);
    k_pick_largest<<<gb, TB, 0, s>>>(label, csize, best, V);
    check_launch("k_pick_largest");
    const int g = coop_grid((const void *)k_peel, TB, ctx->num_sms);
    HM_REQUIRE(g > 0, HM_ECUDA, "k_peel occupancy");
    int32_t *rem = pr.rem.as<int32_t>(), *par = pr.par.as<int32_t>(), *degl = pr.degl.as<int32_t>();
    uint32_t *tsz = pr.tsz.as<uint32_t>();
    unsigned long long *tD = pr.tD.as<unsigned long long>();
    int32_t *flags = scal + 2;
    void *args[] = {(void *)&rp, (void *)&col, (void *)&label, (void *)&best, (void *)&V, (void *)&rem, (void *)&par,
                    (void *)&tsz, (void *)&tD, (void *)&degl, (void *)&flags, (void *)&scal};
    HM_CUDA(cudaLaunchCooperativeKernel((const void *)k_peel, dim3(g), dim3(TB), args, 0, s));
    k_prune_stats<<<gb, TB, 0, s>>>(label, csize, rem, tsz, best, pr.lsize.as<int32_t>(),
                                   pr.Cc.as<unsigned long long>(), tD, scal + 4, V);
    check_launch("k_prune_stats");
    k_graph_stats<<<gb, TB, 0, s>>>(rp, V, scal + 10);
    check_launch("k_graph_stats");
    count_launch(ctx, 4);
    PruneDecision d;
    if (dec && dec->valid) {
        d = *dec;                        // decided by an earlier call on the same graph: no round trip
    } else {
        // one host round trip decides whether the pruned BFS pays (and brings the graph's shape along)
        struct {
            int32_t R, peeled, f0, f1, lsizeP_unused, max_other, maxT, pad;
            unsigned long long best;
            int32_t maxdeg, nonisolated, arcs, pad2;
        } h;
        HM_CUDA(cudaMemcpyAsync(&h, pr.scal.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        host_sync(ctx);
        const int sizeP = (int)(h.best >> 32);
        const int coreP = sizeP - h.peeled;
        d.valid = true;
        d.P = V - 1 - (int)(h.best & 0xffffffffull);
        d.R = h.R;
        d.peeled = h.peeled;
        d.maxdeg = h.maxdeg;
        d.nonisolated = h.nonisolated;
        d.arcs = h.arcs;
        // worth it: >= 1 % of P peeled; P's core still the strictly largest live component
        // (so it stays the first, "giant" batch component); T fits the kernel's bit planes
        d.active = h.peeled > 0 && (int64_t)h.peeled * 100 >= sizeP && coreP > h.max_other &&
                   h.maxT < (1 << BFS_T_BITS);
        if (dec) *dec = d;
    }
    pr.R = d.R;
    pr.peeled = d.peeled;
    pr.P = d.P;
    pr.shape_known = true;
    pr.maxdeg = d.maxdeg;
    pr.nonisolated = d.nonisolated;
    pr.arcs = d.arcs;
    pr.active = d.active;
    return pr.active;
}

void prune_finish(hm_ctx *ctx, Prune &pr, const int32_t *label, const int32_t *csize, uint64_t *S_orig, int V) {
    cudaStream_t s = ctx->stream;
    const int g = coop_grid((const void *)k_prune_finish, TB, ctx->num_sms);
    HM_REQUIRE(g > 0, HM_ECUDA, "k_prune_finish occupancy");
    const int32_t *rem = pr.rem.as<int32_t>(), *par = pr.par.as<int32_t>(), *scal = pr.scal.as<int32_t>();
    const uint32_t *tsz = pr.tsz.as<uint32_t>();
    const unsigned long long *Cc = pr.Cc.as<unsigned long long>();
    unsigned long long *S = reinterpret_cast<unsigned long long *>(S_orig);
    void *args[] = {(void *)&label, (void *)&csize, (void *)&rem, (void *)&par, (void *)&tsz, (void *)&Cc,
                    (void *)&scal, (void *)&S, (void *)&V};
    HM_CUDA(cudaLaunchCooperativeKernel((const void *)k_prune_finish, dim3(g), dim3(TB), args, 0, s));
    count_launch(ctx);
}

}  // namespace hm
