// Persistent, cooperative, bit-parallel multi-source BFS (MS-BFS) for
// all-sources closeness on B200 (sm_100a).
//
// What it computes (§4): for every vertex v the distance sum
// S(v) = sum_w d(v,w) over reachable w.  The paper's tool runs one BFS per
// source, O(V(V+E)).  Here B = 64*W sources advance together, one bit per
// source in a W-word row per vertex, one level per grid-wide step.
//
// Target-side accumulation (exact, undirected graphs): since
// d(s,v) = d(v,s), summing d * popc(new bits of row v at level d) over all
// batches gives S(v) directly -- no transpose, one owner per row, no atomics
// on the sums.
//
// Work reduction, all exact:
//  * sources are batched per connected component (rows grouped by component,
//    components sorted by size descending, isolated vertices excluded); batch
//    `base` covers every component larger than `base`, each with its own
//    source window [start+base, start+base+B) -- so a row only ever sees bits
//    of sources in its own component and "complete" (all window sources
//    reached) is well defined per row;
//  * a row only gathers from neighbours that changed at the previous level
//    (row bitmap `chg`, L1-resident), and only the words it still misses;
//  * complete rows are skipped (bitmap `done`); a row whose neighbours did not
//    change reads only its column indices.
//
// Memory layout: state rows are W*8 bytes (128 B at W=16), row-major, so a
// team of W/2 lanes moves one row with 16-byte vector loads -- one L2 line.
// The frontier array read by the gathers (n_live * W * 8 bytes, 33.5 MB at
// V=2^18, W=16) stays L2-resident (126 MB).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "msbfs.cuh"

namespace cg = cooperative_groups;

namespace hm {
namespace {

constexpr int BLOCK = 512;

__device__ __forceinline__ ulonglong2 ld2(const uint64_t *p) {
    return *reinterpret_cast<const ulonglong2 *>(p);
}
__device__ __forceinline__ void st2(uint64_t *p, ulonglong2 v) {
    *reinterpret_cast<ulonglong2 *>(p) = v;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid barrier on a monotonically increasing arrival counter: generation g is
// complete when bar[0] reaches gridDim.x * g; the last arriver publishes g in
// bar[1].  Every thread fences its own writes before arriving and after
// leaving (release / acquire at gpu scope).
__device__ __forceinline__ void gbar(unsigned *bar, unsigned &gen) {
    __threadfence();
    __syncthreads();
    ++gen;
    if (threadIdx.x == 0) {
        const unsigned target = gen * gridDim.x;
        const unsigned arrived = atomicAdd(bar, 1u) + 1u;
        if (arrived == target) {
            __threadfence();
            atomicExch(bar + 1, gen);
        } else {
            while (ld_acquire_gpu(bar + 1) < gen) __nanosleep(32);
        }
    }
    __syncthreads();
    __threadfence();
}

// bits [0, nb) of a B-bit row, restricted to 64-bit word w
__device__ __forceinline__ uint64_t window_word(int w, int64_t nb) {
    const int64_t lo = (int64_t)w * 64;
    if (nb <= lo) return 0ull;
    if (nb >= lo + 64) return ~0ull;
    return (1ull << (nb - lo)) - 1ull;
}

// first row of the first component with size <= max(base, 1), clamped to n_live
__device__ int batch_hi(const BfsArgs &a, int64_t base, int n_comp, int n_live) {
    const int64_t t = base < 1 ? 1 : base;
    int lo = 0, hi = n_comp;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if ((int64_t)a.comp_size[mid] > t) lo = mid + 1;
        else hi = mid;
    }
    int r = (lo < n_comp) ? a.comp_start[lo] : n_live;
    return r < n_live ? r : n_live;
}

// Per-row context for one lane of a team (2 words per lane).
struct RowState {
    ulonglong2 vv;   // visited bits (lane's 2 words)
    ulonglong2 fw;   // full window mask
    bool tch;        // vis row valid in global memory
};

template <int W>
__device__ __forceinline__ RowState load_row_state(const BfsArgs &a, int v, int64_t base, int tl) {
    constexpr int64_t B = 64 * W;
    RowState r;
    const int2 ci = a.cinfo[v];
    int64_t nb = (int64_t)ci.y - base;
    if (nb > B) nb = B;
    r.fw = make_ulonglong2(window_word(2 * tl, nb), window_word(2 * tl + 1, nb));
    r.tch = (a.touched[v >> 5] >> (v & 31)) & 1u;
    if (r.tch) {
        r.vv = ld2(a.vis + (size_t)v * W + 2 * tl);
    } else {
        r.vv = make_ulonglong2(0ull, 0ull);
        const int64_t j = (int64_t)v - ci.x - base;
        if (j >= 0 && j < nb) {
            const int wj = (int)(j >> 6);
            if (wj == 2 * tl) r.vv.x = 1ull << (j & 63);
            else if (wj == 2 * tl + 1) r.vv.y = 1ull << (j & 63);
        }
    }
    return r;
}

// Gather step over one chunk of T neighbour slots: lanes hold candidate
// neighbour ids `u` (valid where bit set in m, team-relative), each lane loads
// its 16 bytes of every changed neighbour's frontier row unless the lane's
// words are already complete.  Up to 4 rows in flight per lane.
template <int W, int T>
__device__ __forceinline__ void gather_chunk(const uint64_t *__restrict__ Fc, unsigned m, int u,
                                             unsigned tmask, int tbase, int tl, bool need,
                                             ulonglong2 &acc) {
    while (m) {
        const int t0 = __ffs(m) - 1;
        m &= m - 1;
        int t1 = t0, t2 = t0, t3 = t0;
        bool h1 = false, h2 = false, h3 = false;
        if (m) { t1 = __ffs(m) - 1; m &= m - 1; h1 = true; }
        if (m) { t2 = __ffs(m) - 1; m &= m - 1; h2 = true; }
        if (m) { t3 = __ffs(m) - 1; m &= m - 1; h3 = true; }
        const int u0 = __shfl_sync(tmask, u, tbase + t0);
        const int u1 = __shfl_sync(tmask, u, tbase + t1);
        const int u2 = __shfl_sync(tmask, u, tbase + t2);
        const int u3 = __shfl_sync(tmask, u, tbase + t3);
        if (need) {
            const ulonglong2 x0 = ld2(Fc + (size_t)u0 * W + 2 * tl);
            ulonglong2 x1 = make_ulonglong2(0ull, 0ull), x2 = x1, x3 = x1;
            if (h1) x1 = ld2(Fc + (size_t)u1 * W + 2 * tl);
            if (h2) x2 = ld2(Fc + (size_t)u2 * W + 2 * tl);
            if (h3) x3 = ld2(Fc + (size_t)u3 * W + 2 * tl);
            acc.x |= x0.x | x1.x | x2.x | x3.x;
            acc.y |= x0.y | x1.y | x2.y | x3.y;
        }
    }
}

// Commit: new = acc & ~vis; write vis/frontier, accumulate S, set bitmaps.
// Executed by all T lanes of one team (team-uniform control flow).
template <int W, int T>
__device__ __forceinline__ void commit_row(const BfsArgs &a, int v, int d, const RowState &rs,
                                           ulonglong2 acc, uint64_t *__restrict__ Fn,
                                           uint32_t *chn, int32_t *flag, unsigned tmask, int tl) {
    const ulonglong2 nw = make_ulonglong2(acc.x & ~rs.vv.x, acc.y & ~rs.vv.y);
    int cnt = __popcll(nw.x) + __popcll(nw.y);
#pragma unroll
    for (int o = T / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(tmask, cnt, o);
    if (cnt == 0) return;
    const ulonglong2 nv = make_ulonglong2(rs.vv.x | nw.x, rs.vv.y | nw.y);
    st2(a.vis + (size_t)v * W + 2 * tl, nv);
    st2(Fn + (size_t)v * W + 2 * tl, nw);
    const bool complete = __all_sync(tmask, nv.x == rs.fw.x && nv.y == rs.fw.y);
    if (tl == 0) {
        const uint32_t vbit = 1u << (v & 31);
        a.S[v] += (uint64_t)d * (uint64_t)cnt;
        atomicOr(&chn[v >> 5], vbit);
        if (!rs.tch) atomicOr(&a.touched[v >> 5], vbit);
        if (complete) atomicOr(&a.done[v >> 5], vbit);
        *flag = 1;
        if (a.dbgc) {
            atomicAdd(a.dbgc + (d < 4095 ? d : 4095), 1ull);
            if (v < 65536 && d < 64) atomicOr(a.dbgc + 8192 + v, 1ull << d);
        }
    }
}

template <int W>
__global__ void __launch_bounds__(BLOCK, 2) msbfs_kernel(BfsArgs a) {
    constexpr int T = W / 2;           // lanes per row
    constexpr int64_t B = 64 * W;      // sources per batch
    constexpr int TPB = BLOCK / T;     // teams per block
    cg::grid_group grid = cg::this_grid();
    unsigned int gen = 0;
    __shared__ int s_hi;
    __shared__ ulonglong2 s_red[TPB][T];

    const int lane = threadIdx.x & 31;
    const int tl = lane % T;
    const int tbase = lane - tl;
    const unsigned tmask = (T == 32) ? 0xffffffffu : (((1u << T) - 1u) << tbase);
    const int64_t nthreads = (int64_t)gridDim.x * BLOCK;
    const int64_t gtid = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
    const int64_t team = gtid / T;
    const int64_t nteams = nthreads / T;
    const int tib = threadIdx.x / T;

    const int n_live = a.scalars[0];
    const int64_t n_giant = a.scalars[1];
    const int n_comp = a.scalars[2];
    const int n_heavy = a.scalars[3];
    const int heavy_deg = a.heavy_deg;

    for (int64_t base = 0; base < n_giant; base += B) {
        if (threadIdx.x == 0) s_hi = batch_hi(a, base, n_comp, n_live);
        __syncthreads();
        const int hi = s_hi;
        if (a.dbgc && threadIdx.x == 0 && base / B < 64) {
            atomicMax(a.dbgc + 6000 + base / B, (unsigned long long)hi);
            if (blockIdx.x == 0 && base == 0) {
                a.dbgc[6100] = n_live; a.dbgc[6101] = n_giant; a.dbgc[6102] = n_comp; a.dbgc[6103] = n_heavy;
            }
        }
        const int64_t nbw = (hi + 31) >> 5;

        // ---- level 0: sources of every component window; bitmaps reset
        for (int64_t vb = gtid & ~31LL; vb < hi; vb += nthreads) {
            const int v = (int)(vb + lane);
            bool src = false, dn = false;
            if (v < hi) {
                const int2 ci = a.cinfo[v];
                const int64_t j = (int64_t)v - ci.x - base;
                int64_t nb = (int64_t)ci.y - base;
                if (nb > B) nb = B;
                if (j >= 0 && j < nb) {
                    src = true;
                    dn = (nb == 1);
                    uint64_t *f = a.F0 + (size_t)v * W;
                    const int wj = (int)(j >> 6);
#pragma unroll
                    for (int w = 0; w < W; w += 2)
                        st2(f + w, make_ulonglong2(w == wj ? 1ull << (j & 63) : 0ull,
                                                   w + 1 == wj ? 1ull << (j & 63) : 0ull));
                }
            }
            const unsigned bs = __ballot_sync(0xffffffffu, src);
            const unsigned bd = __ballot_sync(0xffffffffu, dn);
            if (lane == 0) {
                const int64_t w = vb >> 5;
                a.chg0[w] = bs;
                a.chg1[w] = 0u;
                a.done[w] = bd;
                a.touched[w] = 0u;
            }
        }
        if (gtid == 0) a.flags[1] = 0;
        if (a.dbg & 1) __threadfence();
        if (a.dbg & 32) gbar(a.bar, gen); else grid.sync();

        int d = 1;
        for (;; ++d) {
            const uint64_t *__restrict__ Fc = (d & 1) ? a.F0 : a.F1;
            uint64_t *__restrict__ Fn = (d & 1) ? a.F1 : a.F0;
            const int r0 = (d - 1) % 3, r1 = d % 3, r2 = (d + 1) % 3;
            const uint32_t *chp = r0 == 0 ? a.chg0 : (r0 == 1 ? a.chg1 : a.chg2);
            uint32_t *chn = r1 == 0 ? a.chg0 : (r1 == 1 ? a.chg1 : a.chg2);
            uint32_t *chz = r2 == 0 ? a.chg0 : (r2 == 1 ? a.chg1 : a.chg2);
            int32_t *flag = a.flags + r1;
            for (int64_t w = gtid; w < nbw; w += nthreads) chz[w] = 0u;
            if (gtid == 0) a.flags[r2] = 0;

            // ---- heavy rows: one CTA per row, neighbour list split over teams
            for (int h = blockIdx.x; h < n_heavy; h += gridDim.x) {
                const int v = a.heavy[h];
                if (v >= hi) continue;                                   // block-uniform
                if ((a.done[v >> 5] >> (v & 31)) & 1u) continue;         // block-uniform
                const int rb = a.row_ptr[v], re = a.row_ptr[v + 1];
                const RowState rs = load_row_state<W>(a, v, base, tl);
                ulonglong2 acc = make_ulonglong2(0ull, 0ull);
                for (int j0 = rb + tib * T; j0 < re; j0 += BLOCK) {
                    const int j = j0 + tl;
                    int u = 0;
                    bool c = false;
                    if (j < re) {
                        u = a.col[j];
                        c = (chp[u >> 5] >> (u & 31)) & 1u;
                    }
                    const unsigned m = __ballot_sync(tmask, c) >> tbase;
                    if (!m) continue;
                    const bool need = ((acc.x | rs.vv.x) != rs.fw.x) || ((acc.y | rs.vv.y) != rs.fw.y);
                    if (!__any_sync(tmask, need)) break;
                    gather_chunk<W, T>(Fc, m, u, tmask, tbase, tl, need, acc);
                }
                s_red[tib][tl] = acc;
                __syncthreads();
                if (tib == 0) {
                    for (int t = 1; t < TPB; ++t) {
                        const ulonglong2 x = s_red[t][tl];
                        acc.x |= x.x;
                        acc.y |= x.y;
                    }
                    commit_row<W, T>(a, v, d, rs, acc, Fn, chn, flag, tmask, tl);
                }
                __syncthreads();
            }

            // ---- light rows: one team per row
            for (int64_t vv = team; vv < hi; vv += nteams) {
                const int v = (int)vv;
                if (!(a.dbg & 8) && ((a.done[v >> 5] >> (v & 31)) & 1u)) continue;         // team-uniform
                const int rb = a.row_ptr[v], re = a.row_ptr[v + 1];
                if (re - rb > heavy_deg) continue;
                ulonglong2 acc = make_ulonglong2(0ull, 0ull);
                RowState rs;
                bool have = false;
                int nm = 0;
                for (int j0 = rb; j0 < re; j0 += T) {
                    const int j = j0 + tl;
                    int u = 0;
                    bool c = false;
                    if (j < re) {
                        u = a.col[j];
                        c = (chp[u >> 5] >> (u & 31)) & 1u;
                    }
                    const unsigned m = __ballot_sync(tmask, c) >> tbase;
                    nm += __popc(m);
                    if (!m) continue;
                    if (!have) {
                        rs = load_row_state<W>(a, v, base, tl);
                        have = true;
                    }
                    const bool need = (a.dbg & 16) || ((acc.x | rs.vv.x) != rs.fw.x) || ((acc.y | rs.vv.y) != rs.fw.y);
                    if (!__any_sync(tmask, need)) break;
                    gather_chunk<W, T>(Fc, m, u, tmask, tbase, tl, need, acc);
                }
                if (a.dbgc && d == 1 && v < 65536) {
                    int ac = __popcll(acc.x) + __popcll(acc.y);
                    for (int o = T / 2; o > 0; o >>= 1) ac += __shfl_xor_sync(tmask, ac, o);
                    int fc = __popcll(Fc[(size_t)v * W + 2 * tl]) + __popcll(Fc[(size_t)v * W + 2 * tl + 1]);
                    for (int o = T / 2; o > 0; o >>= 1) fc += __shfl_xor_sync(tmask, fc, o);
                    if (tl == 0)
                        a.dbgc[73728 + v] = 1ull | (have ? 2ull : 0ull) | ((unsigned long long)nm << 8) |
                                            ((unsigned long long)(re - rb) << 16) | ((unsigned long long)ac << 24) |
                                            ((unsigned long long)fc << 40) | ((unsigned long long)blockIdx.x << 48);
                }
                if (have) commit_row<W, T>(a, v, d, rs, acc, Fn, chn, flag, tmask, tl);
            }
            if (a.dbg & 1) __threadfence();
            if (a.dbg & 32) gbar(a.bar, gen); else grid.sync();
            const int fv = *((volatile int32_t *)flag);
            if (a.dbgc && threadIdx.x == 0) atomicAdd(a.dbgc + 4096 + (d < 4095 ? d : 4095), (unsigned long long)fv);
            if (fv == 0) break;
        }
        if (gtid == 0) {
            a.counters[0] += (unsigned long long)d;
            a.counters[1] += 1ull;
        }
    }
}

}  // namespace

int launch_msbfs(int W, const BfsArgs &a, int num_sms, int blocks_per_sm, cudaStream_t s) {
    const void *kern = nullptr;
    switch (W) {
        case 8: kern = (const void *)msbfs_kernel<8>; break;
        case 16: kern = (const void *)msbfs_kernel<16>; break;
        case 32: kern = (const void *)msbfs_kernel<32>; break;
        default: return -1;
    }
    int maxb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, kern, BLOCK, 0) != cudaSuccess) return -2;
    if (maxb < 1) return -3;
    const int b = (blocks_per_sm > 0 && blocks_per_sm < maxb) ? blocks_per_sm : maxb;
    const int grid = num_sms * b;
    BfsArgs args = a;
    void *kargs[] = {(void *)&args};
    if (cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(BLOCK), kargs, 0, s) != cudaSuccess) return -4;
    return grid;
}

}  // namespace hm
