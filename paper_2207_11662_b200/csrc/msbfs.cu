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
// batches gives S(v) directly -- no transpose, one owner per row.
//
// Work reduction, all exact:
//  * sources are batched per connected component (rows grouped by component,
//    components sorted by size descending, isolated vertices excluded); batch
//    `base` covers every component larger than `base`, each with its own
//    source window [start+base, start+base+B) -- so a row only ever sees bits
//    of sources in its own component and "complete" is well defined per row;
//  * a row only gathers from neighbours that changed at the previous level
//    (row bitmap `chg`), and only the words it still misses;
//  * complete rows are skipped (bitmap `done`).
//
// Level step (one warp per 32-row group; the group's bitmap words belong to
// that warp for the level):
//  1. scan: the warp walks the group's arcs 32 at a time, coalesced; each lane
//     finds its arc's row by a shuffle binary search over the group's row
//     offsets and keeps arcs whose row is live and whose neighbour changed;
//     kept (row, neighbour) pairs are staged in shared memory in arc order,
//     hence grouped by row;
//  2. gather/commit: the warp's W/2-lane teams take one row segment each, in
//     lock-step, issue all the segment's 16-byte frontier gathers (4 in
//     flight), OR them, and commit new = acc & ~vis;
//  3. the group's chg / done / touched words are published with one atomicOr
//     each (rows of degree > heavy_deg are handled by whole CTAs first).
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
constexpr int NWARP = BLOCK / 32;
constexpr int CAP = 256;           // staged pairs per warp
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ ulonglong2 ld2(const uint64_t *p) {
    return *reinterpret_cast<const ulonglong2 *>(p);
}
__device__ __forceinline__ void st2(uint64_t *p, ulonglong2 v) {
    *reinterpret_cast<ulonglong2 *>(p) = v;
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
};

template <int W>
__device__ __forceinline__ RowState row_state(const BfsArgs &a, int v, int64_t base, int tl, bool tch) {
    constexpr int64_t B = 64 * W;
    RowState r;
    const int2 ci = a.cinfo[v];
    int64_t nb = (int64_t)ci.y - base;
    if (nb > B) nb = B;
    r.fw = make_ulonglong2(window_word(2 * tl, nb), window_word(2 * tl + 1, nb));
    if (tch) {
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

struct Smem {
    int hi;
    int32_t su[NWARP][CAP];         // staged neighbour ids
    uint8_t sr[NWARP][CAP];         // staged row index within the group
    int16_t seg[NWARP][34];         // segment starts (+ end sentinel)
};

template <int W>
__global__ void __launch_bounds__(BLOCK, 2) msbfs_kernel(BfsArgs a) {
    constexpr int T = W / 2;           // lanes per row
    constexpr int TPW = 32 / T;        // teams per warp
    constexpr int64_t B = 64 * W;      // sources per batch
    constexpr int TPB = BLOCK / T;     // teams per block
    cg::grid_group grid = cg::this_grid();
    __shared__ Smem sm;
    __shared__ ulonglong2 s_red[TPB][T];

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int tl = lane % T;
    const int team = lane / T;                  // team within warp
    const int tbase = lane - tl;
    const unsigned tmask = (T == 32) ? FULL : (((1u << T) - 1u) << tbase);
    const unsigned ltmask = (1u << lane) - 1u;
    const int64_t nthreads = (int64_t)gridDim.x * BLOCK;
    const int64_t gtid = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
    const int64_t gwarp = gtid >> 5;
    const int64_t nwarps = nthreads >> 5;
    const int tib = threadIdx.x / T;

    const int n_live = a.scalars[0];
    const int64_t n_giant = a.scalars[1];
    const int n_comp = a.scalars[2];
    const int n_heavy = a.scalars[3];
    const int heavy_deg = a.heavy_deg;
    int32_t *su = sm.su[wib];
    uint8_t *sr = sm.sr[wib];
    int16_t *seg = sm.seg[wib];

    for (int64_t base = 0; base < n_giant; base += B) {
        if (threadIdx.x == 0) sm.hi = batch_hi(a, base, n_comp, n_live);
        __syncthreads();
        const int hi = sm.hi;
        const int64_t ngroups = (hi + 31) >> 5;

        // ---- level 0: sources of every component window; bitmaps reset
        for (int64_t g = gwarp; g < ngroups; g += nwarps) {
            const int v = (int)(g * 32 + lane);
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
            const unsigned bs = __ballot_sync(FULL, src);
            const unsigned bd = __ballot_sync(FULL, dn);
            if (lane == 0) {
                a.chg0[g] = bs;
                a.chg1[g] = 0u;
                a.done[g] = bd;
                a.touched[g] = 0u;
            }
        }
        if (gtid == 0) a.flags[1] = 0;
        grid.sync();

        int d = 1;
        for (;; ++d) {
            const uint64_t *__restrict__ Fc = (d & 1) ? a.F0 : a.F1;
            uint64_t *__restrict__ Fn = (d & 1) ? a.F1 : a.F0;
            const int r0 = (d - 1) % 3, r1 = d % 3, r2 = (d + 1) % 3;
            const uint32_t *chp = r0 == 0 ? a.chg0 : (r0 == 1 ? a.chg1 : a.chg2);
            uint32_t *chn = r1 == 0 ? a.chg0 : (r1 == 1 ? a.chg1 : a.chg2);
            uint32_t *chz = r2 == 0 ? a.chg0 : (r2 == 1 ? a.chg1 : a.chg2);
            int32_t *flag = a.flags + r1;
            for (int64_t w = gtid; w < ngroups; w += nthreads) chz[w] = 0u;
            if (gtid == 0) a.flags[r2] = 0;

            // ---- heavy rows: one CTA per row, neighbour list split over teams
            for (int h = blockIdx.x; h < n_heavy; h += gridDim.x) {
                const int v = a.heavy[h];
                if (v >= hi) continue;                                   // block-uniform
                if ((a.done[v >> 5] >> (v & 31)) & 1u) continue;         // block-uniform
                const int rb = a.row_ptr[v], re = a.row_ptr[v + 1];
                const bool tch = (a.touched[v >> 5] >> (v & 31)) & 1u;
                const RowState rs = row_state<W>(a, v, base, tl, tch);
                ulonglong2 acc = make_ulonglong2(0ull, 0ull);
                for (int j0 = rb + tib * T; j0 < re; j0 += BLOCK) {
                    const int j = j0 + tl;
                    int u = 0;
                    bool c = false;
                    if (j < re) {
                        u = a.col[j];
                        c = (chp[u >> 5] >> (u & 31)) & 1u;
                    }
                    unsigned m = __ballot_sync(tmask, c) >> tbase;
                    const bool need = ((acc.x | rs.vv.x) != rs.fw.x) || ((acc.y | rs.vv.y) != rs.fw.y);
                    while (m) {
                        const int t0 = __ffs(m) - 1;
                        m &= m - 1;
                        const int u0 = __shfl_sync(tmask, u, tbase + t0);
                        if (need) {
                            const ulonglong2 x = ld2(Fc + (size_t)u0 * W + 2 * tl);
                            acc.x |= x.x;
                            acc.y |= x.y;
                        }
                    }
                }
                s_red[tib][tl] = acc;
                __syncthreads();
                if (tib == 0) {
                    for (int t = 1; t < TPB; ++t) {
                        const ulonglong2 x = s_red[t][tl];
                        acc.x |= x.x;
                        acc.y |= x.y;
                    }
                    const ulonglong2 nw = make_ulonglong2(acc.x & ~rs.vv.x, acc.y & ~rs.vv.y);
                    int cnt = __popcll(nw.x) + __popcll(nw.y);
#pragma unroll
                    for (int o = T / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(tmask, cnt, o);
                    if (cnt) {
                        const ulonglong2 nv = make_ulonglong2(rs.vv.x | nw.x, rs.vv.y | nw.y);
                        st2(a.vis + (size_t)v * W + 2 * tl, nv);
                        st2(Fn + (size_t)v * W + 2 * tl, nw);
                        const bool complete = __all_sync(tmask, nv.x == rs.fw.x && nv.y == rs.fw.y);
                        if (tl == 0) {
                            const uint32_t vbit = 1u << (v & 31);
                            a.S[v] += (uint64_t)d * (uint64_t)cnt;
                            atomicOr(&chn[v >> 5], vbit);
                            if (!tch) atomicOr(&a.touched[v >> 5], vbit);
                            if (complete) atomicOr(&a.done[v >> 5], vbit);
                            *flag = 1;
                        }
                    }
                }
                __syncthreads();
            }

            // ---- light rows: one warp per 32-row group
            for (int64_t g = gwarp; g < ngroups; g += nwarps) {
                const int r = (int)(g * 32 + lane);
                const bool valid = r < hi;
                const int rp = a.row_ptr[valid ? r : hi];
                const int rnext = __shfl_down_sync(FULL, rp, 1);
                const int rend = (lane == 31) ? a.row_ptr[r + 1 < hi ? r + 1 : hi] : rnext;
                const uint32_t dword = a.done[g];
                const bool act = valid && !((dword >> lane) & 1u) && (rend - rp) <= heavy_deg;
                const unsigned amask = __ballot_sync(FULL, act);
                if (!amask) continue;                                    // warp-uniform
                uint32_t tword = a.touched[g];
                uint32_t chg_bits = 0u, done_bits = 0u;
                const int A0 = __shfl_sync(FULL, rp, 0);
                const int A1 = __shfl_sync(FULL, rend, 31);
                int n = 0;
                for (int a0 = A0; a0 < A1; a0 += 32) {
                    const int aa = a0 + lane;
                    int lo = 0;
#pragma unroll
                    for (int s = 16; s > 0; s >>= 1) {
                        const int c = lo + s;
                        const int x = __shfl_sync(FULL, rp, c & 31);
                        if (c < 32 && x <= aa) lo = c;
                    }
                    bool ok = false;
                    int u = 0;
                    if (aa < A1 && ((amask >> lo) & 1u)) {
                        u = a.col[aa];
                        ok = (chp[u >> 5] >> (u & 31)) & 1u;
                    }
                    const unsigned bm = __ballot_sync(FULL, ok);
                    if (ok) {
                        const int pos = n + __popc(bm & ltmask);
                        su[pos] = u;
                        sr[pos] = (uint8_t)lo;
                    }
                    n += __popc(bm);
                    const bool flush = (n > CAP - 32) || (a0 + 32 >= A1);
                    if (flush && n > 0) {
                        __syncwarp();
                        // segments: runs of equal row index
                        int nseg = 0;
                        for (int k0 = 0; k0 < n; k0 += 32) {
                            const int k = k0 + lane;
                            const bool st = k < n && (k == 0 || sr[k] != sr[k - 1]);
                            const unsigned sb = __ballot_sync(FULL, st);
                            if (st) seg[nseg + __popc(sb & ltmask)] = (int16_t)k;
                            nseg += __popc(sb);
                        }
                        if (lane == 0) seg[nseg] = (int16_t)n;
                        __syncwarp();
                        // teams take segments in lock-step rounds
                        for (int s0 = 0; s0 < nseg; s0 += TPW) {
                            const int si = s0 + team;
                            const bool has = si < nseg;
                            const int kb = has ? seg[si] : 0;
                            const int ke = has ? seg[si + 1] : 0;
                            const int ri = has ? sr[kb] : 0;
                            const int v = (int)(g * 32 + ri);
                            const bool tch = (tword >> ri) & 1u;
                            RowState rs;
                            ulonglong2 acc = make_ulonglong2(0ull, 0ull);
                            if (has) rs = row_state<W>(a, v, base, tl, tch);
                            uint64_t Sv = 0;
                            if (has && tl == 0) Sv = a.S[v];
                            // round length: longest segment among the warp's teams
                            int len = ke - kb;
#pragma unroll
                            for (int o = T; o < 32; o <<= 1) len = max(len, __shfl_xor_sync(FULL, len, o));
                            for (int k = 0; k < len; k += 4) {
                                const int k0 = kb + k;
                                const bool need = has && (((acc.x | rs.vv.x) != rs.fw.x) ||
                                                          ((acc.y | rs.vv.y) != rs.fw.y));
                                ulonglong2 x0 = make_ulonglong2(0ull, 0ull), x1 = x0, x2 = x0, x3 = x0;
                                if (need) {
                                    if (k0 < ke) x0 = ld2(Fc + (size_t)su[k0] * W + 2 * tl);
                                    if (k0 + 1 < ke) x1 = ld2(Fc + (size_t)su[k0 + 1] * W + 2 * tl);
                                    if (k0 + 2 < ke) x2 = ld2(Fc + (size_t)su[k0 + 2] * W + 2 * tl);
                                    if (k0 + 3 < ke) x3 = ld2(Fc + (size_t)su[k0 + 3] * W + 2 * tl);
                                }
                                acc.x |= x0.x | x1.x | x2.x | x3.x;
                                acc.y |= x0.y | x1.y | x2.y | x3.y;
                            }
                            // commit
                            ulonglong2 nw = make_ulonglong2(0ull, 0ull);
                            if (has) nw = make_ulonglong2(acc.x & ~rs.vv.x, acc.y & ~rs.vv.y);
                            int cnt = __popcll(nw.x) + __popcll(nw.y);
#pragma unroll
                            for (int o = T / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
                            bool complete = false;
                            if (cnt) {
                                const ulonglong2 nv = make_ulonglong2(rs.vv.x | nw.x, rs.vv.y | nw.y);
                                st2(a.vis + (size_t)v * W + 2 * tl, nv);
                                ulonglong2 fw_out = nw;
                                if ((chg_bits >> ri) & 1u) {     // row split over staging flushes:
                                    const ulonglong2 f0 = ld2(Fn + (size_t)v * W + 2 * tl);   // merge
                                    fw_out.x |= f0.x;
                                    fw_out.y |= f0.y;
                                }
                                st2(Fn + (size_t)v * W + 2 * tl, fw_out);
                                complete = nv.x == rs.fw.x && nv.y == rs.fw.y;
                                if (tl == 0) a.S[v] = Sv + (uint64_t)d * (uint64_t)cnt;
                            }
                            // team-wide "complete" and warp-wide bit merge
                            unsigned cflag = complete ? 1u : 0u;
#pragma unroll
                            for (int o = T / 2; o > 0; o >>= 1) cflag &= __shfl_xor_sync(FULL, cflag, o);
                            uint32_t cb = (cnt && tl == 0) ? (1u << ri) : 0u;
                            uint32_t db = (cnt && tl == 0 && cflag) ? (1u << ri) : 0u;
#pragma unroll
                            for (int o = T; o < 32; o <<= 1) {
                                cb |= __shfl_xor_sync(FULL, cb, o);
                                db |= __shfl_xor_sync(FULL, db, o);
                            }
                            cb = __shfl_sync(FULL, cb, 0);
                            db = __shfl_sync(FULL, db, 0);
                            chg_bits |= cb;
                            done_bits |= db;
                            tword |= cb;
                        }
                        n = 0;
                        __syncwarp();
                    }
                }
                if (lane == 0) {
                    if (chg_bits) {
                        atomicOr(&chn[g], chg_bits);
                        atomicOr(&a.touched[g], chg_bits);
                        *flag = 1;
                    }
                    if (done_bits) atomicOr(&a.done[g], done_bits);
                }
            }
            grid.sync();
            const int fv = *((volatile int32_t *)flag);
            if (a.dbgc && gtid == 0) a.dbgc[d < 4095 ? d : 4095] += 1ull;
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
