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
// Visited sets, double-buffered, no frontier array.  V_d(v) = sources within
// distance d of v.  On an undirected graph
//   V_d(v) = V_{d-1}(v) | OR over neighbours u of V_{d-1}(u),
// and only neighbours that CHANGED at level d-1 can contribute a new source (a
// source s in V_{d-2}(u) has d(s,v) <= d-1, already in V_{d-1}(v)).  So
//   new_d(v) = (OR over u in N(v) changed at d-1 of V_{d-1}(u)) & ~V_{d-1}(v)
// is exactly the set of sources at distance d.  A row that changes at level d
// writes V_d(v) into buffer F[d & 1]; a row changed at d-1 is therefore gathered
// from F[(d-1) & 1], which nobody writes during level d, and a row reads its own
// V_{d-1} from the buffer of the level that last wrote it (bitmaps has / par).
// Per changed row and level: one own-row read and one row write (the frontier
// recurrence F_d = acc & ~F_{d-1} & ~F_{d-2} of round 1 needed two reads and
// three arrays).  Completion (every window source reached) comes from a 16-bit
// per-row count K.
//
// Work reduction, all exact:
//  * sources are batched per connected component (rows grouped by component,
//    components sorted by size descending, isolated vertices excluded); batch
//    `base` covers every component larger than `base`, each with its own
//    source window [start+base, start+base+B);
//  * a row only gathers from neighbours that changed at the previous level
//    (row bitmaps "changed at level d" rotate over 4 levels);
//  * complete rows are skipped (bitmap `done`).
//
// Level step, light rows (one warp per work unit of 32, 16, 8, 4 or 2 rows of a
// 32-row group; CTA b owns units b, b + grid, ... and its warps claim them
// dynamically, starting at the batch's source window):
//  1. scan: packed arcs (neighbour << 5 | row in group), SCAN_U x 32 at a time,
//     coalesced; pairs (row, changed neighbour) staged in shared memory in arc
//     order, hence grouped by row;
//  2. gather/commit: the row segments are sorted by length and dealt to the
//     warp's TL-lane teams in lock-step rounds; each row's state and frontier
//     gathers are issued together (VEC x 16 B per lane per row), OR-ed, committed;
//  3. the group's chg / done words are published with one atomicOr each.
// Rows of degree > heavy_deg (R-MAT hubs) are cut into items of BFS_HEAVY_CHUNK
// arcs that whole CTAs claim after their light units (heavy_items, out of line;
// the last item of a row commits it).  The level barrier is one atomic per CTA on
// per-parity counters that also sum the level's changed rows (the frontier size).
//
// (Variants measured and not kept -- two interleaved batch streams with split grid
// barriers, half-CTA stream parts, a warp-wide pipelined item stream, per-CTA owned
// rows, a level-1 push step -- are in git history up to commit 93c73e1.)
//
// Memory layout: visited-set rows are W*8 bytes (512 B at the default W=64), row-major.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "msbfs.cuh"

namespace cg = cooperative_groups;



namespace hm {
namespace {

// threads per CTA (2 CTAs per SM), measured: the plain kernel runs best at 448 (512: 2.7 %
// slower, 416: much slower); the weighted kernel (pruned graphs) keeps more live state and
// runs best at 384 (85 registers, no spills)
#ifndef HM_BLOCK_PLAIN
#define HM_BLOCK_PLAIN 448      // measured best for the plain kernel (2 CTAs x 14 warps, 73 registers)
#endif
#ifndef HM_BLOCK_WEIGHTED
#define HM_BLOCK_WEIGHTED 320   // weighted (pruned) kernel: measured best in round 2 (288: +28 %, 352: +4 %, 384: +3 %)
#endif
constexpr int BLOCK_PLAIN = HM_BLOCK_PLAIN, BLOCK_WEIGHTED = HM_BLOCK_WEIGHTED;
#ifndef HM_CAP
#define HM_CAP 384      // measured: 384 beats 256 by 3 % on the C5 layers
#endif
#ifndef HM_SCAN_U
#define HM_SCAN_U 4
#endif
constexpr int CAP = HM_CAP;         // staged pairs per warp
constexpr int SCAN_U = HM_SCAN_U;   // arc chunks (of 32) loaded per scan step
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ ulonglong2 ld2(const uint64_t *p) {
    return *reinterpret_cast<const ulonglong2 *>(p);
}
__device__ __forceinline__ void st2(uint64_t *p, ulonglong2 v) {
    *reinterpret_cast<ulonglong2 *>(p) = v;
}
__device__ __forceinline__ int ld_cs(const int32_t *p) {   // arcs: read once per level
    int v;
    asm volatile("ld.global.cs.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
// arcs kept L2-resident (HM_CSR_POLICY 1, default: evict_last hint; the CSR is read every level -- C5 layer
// 65.3 -> 65.0 ms, C4 layer 1 25.9 -> 24.8 ms against the streaming .cs load)
__device__ __forceinline__ int ld_pol(const int32_t *p, uint64_t pol) {
    if (!pol) return ld_cs(p);                      // no L2 policies (bfs_hints without bit 1)
    int v;
    asm volatile("ld.global.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
#ifndef HM_CSR_POLICY
#define HM_CSR_POLICY 1
#endif

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

// Component of row v: rows [0, n_giant) are the largest component.
__device__ __forceinline__ int2 comp_of(const BfsArgs &a, int v, int n_giant) {
    return v < n_giant ? make_int2(0, n_giant) : a.cinfo[v];
}

__device__ __forceinline__ bool bit_of(const uint32_t *bm, int v) { return (bm[v >> 5] >> (v & 31)) & 1u; }

// Optional per-phase cycle profile (build with HM_MSBFS_PROF=1, run with bfs_dbg = 2):
// lane 0 of every warp accumulates clock64() deltas per phase into dbgc[8192 + phase],
// and counts (flushes, items) into dbgc[8200..8201].
struct Prof {
#ifdef HM_MSBFS_PROF
    long long t;
    long long acc[9];    // [8]: cycles outside the profiled level (bfs_dbg_level > 0)
    long long cnt[2];
    bool on;
#endif
};
#ifdef HM_MSBFS_PROF
#define PROF_INIT(p) do { (p).t = clock64(); for (int _i = 0; _i < 9; ++_i) (p).acc[_i] = 0; (p).cnt[0] = (p).cnt[1] = 0; (p).on = true; } while (0)
#define PROF_LEVEL(p, d) do { (p).on = (a.dbg_level <= 0 || (d) == a.dbg_level); } while (0)
#define PROF_MARK(p, i) do { const long long _n = clock64(); (p).acc[(p).on ? (i) : 8] += _n - (p).t; (p).t = _n; } while (0)
#define PROF_COUNT(p, i, v) do { if ((p).on) (p).cnt[i] += (v); } while (0)
#define PROF_FLUSH(p, dst) do { if ((dst) && (threadIdx.x & 31) == 0) { for (int _i = 0; _i < 8; ++_i) \
        atomicAdd((dst) + 8192 + _i, (unsigned long long)(p).acc[_i]); \
        atomicAdd((dst) + 8200, (unsigned long long)(p).cnt[0]); atomicAdd((dst) + 8201, (unsigned long long)(p).cnt[1]); } } while (0)
#else
#define PROF_INIT(p) do { } while (0)
#define PROF_MARK(p, i) do { } while (0)
#define PROF_LEVEL(p, d) do { } while (0)
#define PROF_COUNT(p, i, v) do { } while (0)
#define PROF_FLUSH(p, dst) do { } while (0)
#endif

#ifndef HM_HEAVY_DYN
#define HM_HEAVY_DYN 1          // heavy items: 0 dealt before the light units, 1 claimed after them
#endif
#ifndef HM_HEAVY_GD
#define HM_HEAVY_GD 8
#endif
constexpr int HGD = HM_HEAVY_GD;    // heavy-row gathers in flight per team
#ifndef HM_PUSH_PU
#define HM_PUSH_PU 4
#endif

template <int NWARP>
struct Smem {
    int hi;
    int next;                       // next group to claim in this CTA's range
    int flag;
    unsigned long long lb[4];    // counting barrier (thread 0): expected arrivals [p], changed rows seen [2 + p]
    unsigned long long epoch;    // counting barriers passed (thread 0); parity p = epoch & 1
    int nchg;                    // rows this CTA changed in the current level
    unsigned ngat, nown;         // rows this CTA gathered / own rows it read in the current level
    long long nlast;             // rows the whole grid changed before the last counting barrier
    int push, emit;              // push phase: this level pushes pairs / appends the pairs it finds
    unsigned pn;                 // pairs in the list to read
    int pt;                      // list-producing levels (level 0s, push levels) run so far
    int32_t su[NWARP][CAP];         // staged neighbour ids
    uint8_t sr[NWARP][CAP];         // staged row index within the group
    int16_t seg[NWARP][34];         // segment starts (+ end sentinel)
};

// A state row split over TL lanes: lane l holds 16-byte chunks q*TL + l, q < VEC.
template <int VEC>
__device__ __forceinline__ void zero_row(ulonglong2 (&r)[VEC]) {
#pragma unroll
    for (int q = 0; q < VEC; ++q) r[q] = make_ulonglong2(0ull, 0ull);
}
template <int VEC>
__device__ __forceinline__ void or_row(ulonglong2 (&r)[VEC], const ulonglong2 (&x)[VEC]) {
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
        r[q].x |= x[q].x;
        r[q].y |= x[q].y;
    }
}
// L2 cache-policy variants (createpolicy + .L2::cache_hint); pol == 0 -> plain access
__device__ __forceinline__ ulonglong2 ld2p(const uint64_t *p, uint64_t pol) {
    if (!pol) return ld2(p);
    ulonglong2 v;
    // gathered rows are random and read once per SM: do not let them evict the bitmaps from L1
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;"
                 : "=l"(v.x), "=l"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st2p(uint64_t *p, ulonglong2 v, uint64_t pol) {
    if (!pol) {
        st2(p, v);
        return;
    }
    asm volatile("st.global.L2::cache_hint.v2.u64 [%0], {%1, %2}, %3;" ::"l"(p), "l"(v.x), "l"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

template <int W, int TL, int VEC>
__device__ __forceinline__ void ld_row(ulonglong2 (&r)[VEC], const uint64_t *F, int v, int l, uint64_t pol = 0) {
#pragma unroll
    for (int q = 0; q < VEC; ++q) r[q] = ld2p(F + (size_t)v * W + 2 * (q * TL + l), pol);
}
template <int W, int TL, int VEC>
__device__ __forceinline__ void st_row(uint64_t *F, int v, int l, const ulonglong2 (&r)[VEC], uint64_t pol = 0) {
#pragma unroll
    for (int q = 0; q < VEC; ++q) st2p(F + (size_t)v * W + 2 * (q * TL + l), r[q], pol);
}

// Grid barrier that also sums a per-CTA count (thread 0 only; the caller __syncthreads() after).
// Each CTA adds its count to the epoch parity's count counter, then (after a fence) 1 to the
// parity's arrival counter; once all grid arrivals are seen, the count counter holds every CTA's
// count: sm.nlast = the grid's total for this barrier, sm.flag = (total != 0).  64-bit counters,
// never reset within a launch.  (The next arrival on this parity needs every CTA past the next
// barrier, which needs this CTA's arrival there, so what is read here is final.)
template <class SM>
__device__ __forceinline__ void count_barrier(unsigned long long *lbar, SM &sm, int add) {
    const int p = (int)(sm.epoch & 1ull);
    ++sm.epoch;
    if (add) atomicAdd(lbar + 2 + p, (unsigned long long)add);
    __threadfence();
    atomicAdd(lbar + p, 1ull);
    const unsigned long long expect = sm.lb[p] + gridDim.x;
    sm.lb[p] = expect;
    unsigned long long v;
    while (true) {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(lbar + p) : "memory");
        if (v >= expect) break;
        __nanosleep(20);
    }
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(lbar + 2 + p) : "memory");
    sm.nlast = (long long)(v - sm.lb[2 + p]);
    sm.flag = (v != sm.lb[2 + p]) ? 1 : 0;
    sm.lb[2 + p] = v;
    __threadfence();
}

// Level guard (thread 0, after the level barrier): no BFS over hi rows runs deeper than hi levels, so
// a deeper level is a kernel bug -- stop the batch rather than loop on, and flag it (hm_get_stats fails)
template <class SM>
__device__ __forceinline__ void level_guard(SM &sm, int d, unsigned long long *counters) {
    if (d > sm.hi + 1) {
        sm.flag = 0;
        counters[7] = 1ull;
    }
}

// Top-down discovery for a sparse level (direction optimisation): every row that changed at
// d-1 (the frontier, bitmap chp) marks its neighbours that are not done as candidates; the
// level's pull step then visits candidate rows only.  Warp per 32-row frontier group, striding
// over the group's packed arcs (row index in the low 5 bits): coalesced and independent loads.
__device__ __noinline__ void td_discover(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                         const uint32_t *chp, const uint32_t *done, uint32_t *cand, int hi,
                                         int64_t ngroups, int64_t gwarp, int64_t nwarps) {
    const int lane = threadIdx.x & 31;
    for (int64_t g = gwarp; g < ngroups; g += nwarps) {
        const uint32_t fw = chp[g];
        if (!fw) continue;                                   // warp-uniform
        const int r0 = (int)(g * 32) + __ffs(fw) - 1;        // first and last frontier row of the group
        const int r1 = (int)(g * 32) + 32 - __clz(fw);
        const int A0 = row_ptr[r0], A1 = row_ptr[r1 < hi ? r1 : hi];
        for (int j0 = A0; j0 < A1; j0 += 32 * 4) {
            int x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = (j0 + 32 * q + lane < A1) ? col[j0 + 32 * q + lane] : -1;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (x[q] >= 0 && ((fw >> (x[q] & 31)) & 1u)) {
                    const int v = x[q] >> 5;
                    if (!bit_of(done, v)) atomicOr(&cand[v >> 5], 1u << (v & 31));
                }
            }
        }
    }
}

// ---- Top-down push phase (bfs_push, PS instantiations: graphs without heavy rows) ----
// The first levels of a batch are sparse: 64 W sources reach few rows, yet a bottom-up level visits every
// row.  While the (row, source) pairs found at the previous level are few, a level instead runs the
// per-source top-down step (the BFS the paper's tool runs once per source) on the batch's bit
// rows: each pair (v, s) ORs bit s into V(u) of every neighbour u (atomicOr); a first set is the discovery
// d(s, u) = d, which adds d (x the source's weight) to S(u), 1 to K(u), marks u changed and, while the next
// level will still push, appends (u, s).  All rows live in buffer F[0] during the phase (level 0 writes
// every row: zero, the sources' own bit set); the bottom-up levels take over with the buffer parity shifted
// so that the last push level's rows are the ones gathered.  Sums are integers: the result is identical.
//
// thread 0, after a level's barrier: the pairs that level appended (cursor lt % 3) decide whether the next
// level pushes, and whether it appends what it finds (predicted from the growth of the lists)
template <class SM>
__device__ __forceinline__ void push_decide(const BfsArgs &a, SM &sm, int lt, int hi, bool first) {
    unsigned n;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(n) : "l"(a.pcur + lt % 3) : "memory");
    const bool listed = first || sm.emit;
    const double lim = (double)hi * (double)a.push_num * 0.25;
    const bool push = listed && n > 0u && n <= (unsigned)a.pcap && (double)n <= lim;
    double g = first ? (double)a.row_ptr[hi] / (double)(hi > 0 ? hi : 1) : (double)n / (double)(sm.pn ? sm.pn : 1u);
    if (g < 1.0) g = 1.0;
    sm.emit = (push && (double)n * g <= lim) ? 1 : 0;
    sm.push = push ? 1 : 0;
    sm.pn = n;
}

// one push level d over the n pairs of Lr: 2^lps lanes per pair (short lists: a pair's arcs are dealt over its
// lanes, fewer dependent rounds), the arc loop warp-uniform; returns the rows this thread was first to mark changed
template <int W, bool WT>
__device__ __noinline__ int push_level(const BfsArgs &a, const unsigned long long *Lr, unsigned n,
                                       unsigned long long *Lw, unsigned *cur, bool emit, uint32_t *chn,
                                       int d, int64_t base, int n_giant, int64_t gwarp, int64_t nwarps, int lps) {
    constexpr int64_t B = 64 * W;
    constexpr int PU = HM_PUSH_PU;                           // row atomics in flight per lane
    const int lane = threadIdx.x & 31;
    const unsigned ltmask = (1u << lane) - 1u;
    uint64_t *Fp = a.F[0];
    unsigned *K32 = reinterpret_cast<unsigned *>(a.K);
    int nchg = 0;
    const int LP = 1 << lps, sub = lane & (LP - 1), ppw = 32 >> lps;     // lanes per pair, this lane's, pairs per warp
    for (int64_t p0 = gwarp * ppw; p0 < (int64_t)n; p0 += nwarps * ppw) {
        const int64_t p = p0 + (lane >> lps);
        int v = -1, j = 0, r0 = 0, deg = 0;
        if (p < (int64_t)n) {
            const unsigned long long pr = __ldcg(Lr + p);     // written by other CTAs at the previous level
            v = (int)(pr >> 16);
            j = (int)(pr & 0xffffull);
            r0 = a.row_ptr[v] + sub;                          // this lane's arcs: r0, r0 + LP, ...
            deg = (a.row_ptr[v + 1] - r0 + LP - 1) >> lps;
            if (deg < 0) deg = 0;
        }
        int2 ci = make_int2(0, 0);
        if (v >= 0) ci = comp_of(a, v, n_giant);
        int64_t nb = (int64_t)ci.y - base;
        if (nb > B) nb = B;
        unsigned long long wt = 1ull;                        // the source's weight 1 + T(s) (pruned core)
        if constexpr (WT)
            if (v >= 0 && v < n_giant) wt += (unsigned long long)a.tw[base + j];
        const unsigned long long bit = 1ull << (j & 63);
        const int word = j >> 6;
        const int dmax = __reduce_max_sync(FULL, deg);
        for (int a0 = 0; a0 < dmax; a0 += PU) {
            int u[PU];
            unsigned long long old[PU];
#pragma unroll
            for (int q = 0; q < PU; ++q) u[q] = (a0 + q < deg) ? (a.col[r0 + ((a0 + q) << lps)] >> 5) : -1;
#pragma unroll
            for (int q = 0; q < PU; ++q) {
                old[q] = bit;
                if (u[q] >= 0) old[q] = atomicOr(reinterpret_cast<unsigned long long *>(Fp + (size_t)u[q] * W + word), bit);
            }
            unsigned bm[PU], ko[PU], co[PU];
            int tot = 0;
            // the discoveries' updates are issued together (their returns overlap), then read
#pragma unroll
            for (int q = 0; q < PU; ++q) {
                const bool disc = u[q] >= 0 && !(old[q] & bit);
                ko[q] = co[q] = 0u;
                if (disc) {
                    const int uu = u[q];
                    atomicAdd(reinterpret_cast<unsigned long long *>(a.S + uu), (unsigned long long)d * wt);
                    ko[q] = atomicAdd(K32 + (uu >> 1), 1u << ((uu & 1) * 16));
                    co[q] = atomicOr(&chn[uu >> 5], 1u << (uu & 31));
                }
                bm[q] = emit ? __ballot_sync(FULL, disc) : 0u;
                tot += __popc(bm[q]);
            }
#pragma unroll
            for (int q = 0; q < PU; ++q) {
                if (u[q] >= 0 && !(old[q] & bit)) {
                    const int uu = u[q];
                    const int kn = (int)((ko[q] >> ((uu & 1) * 16)) & 0xffffu) + 1;
                    const unsigned ub = 1u << (uu & 31);
                    if (!(co[q] & ub)) ++nchg;
                    const int64_t ju = (int64_t)uu - ci.x - base;
                    if (kn + ((ju >= 0 && ju < nb) ? 1 : 0) == nb) atomicOr(&a.done[uu >> 5], ub);
                }
            }
            if (tot) {                                       // warp-uniform: one cursor reservation per round
                unsigned pos = 0;
                if (lane == 0) pos = atomicAdd(cur, (unsigned)tot);
                pos = __shfl_sync(FULL, pos, 0);
#pragma unroll
                for (int q = 0; q < PU; ++q) {
                    if ((bm[q] >> lane) & 1u) {
                        const unsigned at = pos + __popc(bm[q] & ltmask);
                        if (at < (unsigned)a.pcap) Lw[at] = ((unsigned long long)u[q] << 16) | (unsigned long long)j;
                    }
                    pos += __popc(bm[q]);
                }
            }
        }
    }
    return nchg;
}

// the push levels of one batch, after its level 0: returns the levels run (negative: the last one found nothing,
// the batch is complete).  Level d reads the list of list-level pt - 1, appends to list pt (cursor pt % 3) and
// zeroes cursor (pt + 1) % 3, whose readers all passed the previous barrier.
template <int W, bool WT, class SM>
__device__ __noinline__ int push_phase(const BfsArgs &a, SM &sm, int64_t base, int hi, int n_giant,
                                       unsigned long long *t_prev) {
    const int lane = threadIdx.x & 31;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ngroups = (hi + 31) >> 5;
    int d = 1;
    for (;; ++d) {
        if (!sm.push) return d - 1;                       // block-uniform (written before a __syncthreads)
        const int pt = sm.pt;
        const bool emit = sm.emit;
        const unsigned pairs = sm.pn;
        uint32_t *chn = a.chg[d % 3];
        uint32_t *chz = a.chg[(d + 1) % 3];
        for (int64_t w = gtid; w < ngroups; w += nthreads) chz[w] = 0u;
        if (gtid == 0) {
            a.flags[(d + 1) % 3] = 0;
            a.pcur[(pt + 1) % 3] = 0u;
        }
        if (threadIdx.x == 0) sm.nchg = 0;
        __syncthreads();
        int lps = 0;                                      // lanes per pair: as many as the grid has for the list (<= 8)
        while (lps < 3 && ((int64_t)pairs << (lps + 1)) <= nthreads) ++lps;
        int nchg = push_level<W, WT>(a, a.plist[(pt - 1) & 1], pairs, a.plist[pt & 1], a.pcur + pt % 3, emit, chn, d,
                                     base, n_giant, gtid >> 5, nthreads >> 5, lps);
        nchg = __reduce_add_sync(FULL, nchg);
        if (lane == 0 && nchg) atomicAdd(&sm.nchg, nchg);
        __syncthreads();
        if (threadIdx.x == 0) {
            count_barrier(a.lbar, sm, sm.nchg);           // sm.nlast = rows changed at d
            level_guard(sm, d, a.counters);
            push_decide(a, sm, pt, hi, false);
            sm.pt = pt + 1;
        }
        __syncthreads();
        const int fv = sm.flag;
        if (gtid == 0) {
            if (sm.nlast > 0) a.counters[3] += (unsigned long long)sm.nlast;    // rows changed
            a.counters[5] += 1ull;                                              // top-down levels
            if (a.dbgc) {
                unsigned long long now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                const int di = d < 4095 ? d : 4095;
                a.dbgc[di] += 1ull;
                a.dbgc[4096 + di] += now - *t_prev;
                if (sm.nlast > 0) a.dbgc[12288 + di] += (unsigned long long)sm.nlast;
                a.dbgc[16384 + di] += 1ull;
                *t_prev = now;
            }
        }
        if (fv == 0) return -d;
    }
}

// Heavy rows (degree > heavy_deg), out of line: items of BFS_HEAVY_CHUNK arcs (hstart: first item
// of each heavy row), claimed from the level's counter hclaim (nullptr: dealt round-robin over the
// CTAs), each item's arcs split over the CTA's teams of T = W/2 lanes.  A row of several items ORs its partial rows into hacc; the last item to
// arrive commits.  Returns whether this thread committed a change.
template <int W, int BLOCK, bool WT>
__device__ __noinline__ int heavy_items(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                         const int2 *__restrict__ cinfo, const int32_t *__restrict__ heavy,
                                         const int32_t *__restrict__ hstart, unsigned long long *hacc, int32_t *hcnt,
                                         uint32_t *done, uint16_t *K, uint64_t *S, int32_t *hclaim, ulonglong2 *s_red_,
                                 const unsigned long long *s_pl_, int s_nb, int n_items, int n_heavy,
                                 int hi, int n_giant, int64_t base, int d, const uint32_t *chp_s,
                                 uint32_t *has, uint32_t *par, const uint64_t *__restrict__ Fc,
                                 const uint64_t *F0, const uint64_t *F1, uint64_t *__restrict__ Fn,
                                 uint32_t *chn, const uint32_t *cand, unsigned *s_ngat) {
    // s_ngat: the CTA's gather and own-read counters (Smem ngat, nown)
    constexpr int T = W / 2;
    constexpr int TPB = BLOCK / T;
    constexpr int64_t B = 64 * W;
    const int lane = threadIdx.x & 31;
    const int tib = threadIdx.x / T;
    const int tl = lane % T;
    const int tbase = lane - tl;
    const unsigned tmask = ((T == 32) ? FULL : ((1u << T) - 1u)) << tbase;
    int ncommit = 0;                    // rows this thread committed (changed)
    __shared__ int sm_hh;               // heavy row of the current item
    __shared__ int sm_hlast;            // this CTA completed the heavy row (last item to arrive)
    __shared__ int sm_it;               // claimed item (hclaim: dynamic claims)
    for (int it_s = blockIdx.x;; it_s += gridDim.x) {
        if (threadIdx.x == 0) {
            const int it = hclaim ? atomicAdd(hclaim, 1) : it_s;
            sm_it = it;
            int lo = 0, hi2 = n_heavy - 1;                       // last h with hstart[h] <= it
            while (lo < hi2) {
                const int mid = (lo + hi2 + 1) >> 1;
                if (hstart[mid] <= it) lo = mid; else hi2 = mid - 1;
            }
            sm_hh = lo;
        }
        __syncthreads();
        const int it = sm_it;
        if (it >= n_items) break;                                // block-uniform
        const int h = sm_hh;
        const int v = heavy[h];
        const int i0 = hstart[h], nch = hstart[h + 1] - i0;
        __syncthreads();                                         // sm_hh reused next item
        if (v >= hi) continue;                                   // block-uniform
        if (bit_of(done, v)) continue;                         // block-uniform
        if (cand && !bit_of(cand, v)) continue;                // top-down level: not adjacent to the frontier
        const int rb = row_ptr[v] + (it - i0) * BFS_HEAVY_CHUNK;
        const int re = min(row_ptr[v + 1], rb + BFS_HEAVY_CHUNK);
        ulonglong2 acc = make_ulonglong2(0ull, 0ull);
        for (int j0 = rb + tib * T; j0 < re; j0 += BLOCK) {
            const int j = j0 + tl;
            int u = 0;
            bool c = false;
            if (j < re) {
                u = col[j] >> 5;
                c = bit_of(chp_s, u);
            }
            unsigned m = __ballot_sync(tmask, c) >> tbase;
            if (s_ngat && tl == 0 && m) atomicAdd(s_ngat, (unsigned)__popc(m));
            while (m) {                                          // HGD neighbour rows in flight
                int uq[HGD];
        #pragma unroll
                for (int q = 0; q < HGD; ++q) {
                    uq[q] = -1;
                    if (m) {
                        const int t0 = __ffs(m) - 1;
                        m &= m - 1;
                        uq[q] = __shfl_sync(tmask, u, tbase + t0);
                    }
                }
                ulonglong2 x[HGD];
        #pragma unroll
                for (int q = 0; q < HGD; ++q)
                    x[q] = uq[q] >= 0 ? ld2(Fc + (size_t)uq[q] * W + 2 * tl) : make_ulonglong2(0ull, 0ull);
        #pragma unroll
                for (int q = 0; q < HGD; ++q) {
                    acc.x |= x[q].x;
                    acc.y |= x[q].y;
                }
            }
        }
        s_red_[tib * T + tl] = acc;
        __syncthreads();
        if (tib == 0) {
            for (int t = 1; t < TPB; ++t) {
                const ulonglong2 x = s_red_[t * T + tl];
                acc.x |= x.x;
                acc.y |= x.y;
            }
        }
        if (nch > 1) {                                           // block-uniform
            unsigned long long *hp = hacc + (size_t)h * W + 2 * tl;
            if (tib == 0) {
                if (acc.x) atomicOr(hp, acc.x);
                if (acc.y) atomicOr(hp + 1, acc.y);
                __threadfence();
            }
            __syncthreads();
            if (threadIdx.x == 0) sm_hlast = (atomicAdd(hcnt + h, 1) == nch - 1) ? 1 : 0;
            __syncthreads();
            if (!sm_hlast) continue;                             // block-uniform
            if (tib == 0) {
                __threadfence();
                acc.x = __ldcg(hp);
                acc.y = __ldcg(hp + 1);
                hp[0] = 0ull;                                    // ready for the next level
                hp[1] = 0ull;
            }
            if (threadIdx.x == 0) hcnt[h] = 0;
        }
        if (tib == 0) {
            // own visited set V_{d-1}(v): in the buffer of the level that last wrote it
            ulonglong2 vv = make_ulonglong2(0ull, 0ull);
            if (bit_of(has, v)) {
                vv = ld2((bit_of(par, v) ? F1 : F0) + (size_t)v * W + 2 * tl);
                if (s_ngat && tl == 0) atomicAdd(s_ngat + 1, 1u);
            }
            const ulonglong2 nw = make_ulonglong2(acc.x & ~vv.x, acc.y & ~vv.y);
            int cnt = __popcll(nw.x) + __popcll(nw.y);
#pragma unroll
            for (int o = T / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(tmask, cnt, o);
            unsigned long long wsum = 0ull;     // sum of T over the new sources (pruned component)
            if constexpr (WT) {
                const int nbp = v < n_giant ? s_nb : 0;
                for (int b = 0; b < nbp; ++b)
                    wsum += (unsigned long long)(__popcll(nw.x & s_pl_[b * W + 2 * tl]) +
                                                 __popcll(nw.y & s_pl_[b * W + 2 * tl + 1])) << b;
#pragma unroll
                for (int o = T / 2; o > 0; o >>= 1) wsum += __shfl_xor_sync(tmask, wsum, o);
            }
            if (cnt) {
                st2(Fn + (size_t)v * W + 2 * tl, make_ulonglong2(nw.x | vv.x, nw.y | vv.y));   // V_d(v)
                if (tl == 0) {
                    const int2 ci = (v < n_giant ? make_int2(0, n_giant) : cinfo[v]);
                    int64_t nb = (int64_t)ci.y - base;
                    if (nb > B) nb = B;
                    const int64_t j = (int64_t)v - ci.x - base;
                    const int kn = (int)K[v] + cnt;
                    K[v] = (uint16_t)kn;
                    if constexpr (WT)
                        S[v] += (uint64_t)d * ((uint64_t)cnt + wsum);
                    else
                        S[v] += (uint64_t)d * (uint64_t)cnt;
                    const uint32_t vbit = 1u << (v & 31);
                    atomicOr(&chn[v >> 5], vbit);
                    atomicOr(&has[v >> 5], vbit);
                    if (d & 1) atomicOr(&par[v >> 5], vbit);
                    else atomicAnd(&par[v >> 5], ~vbit);
                    if (kn + ((j >= 0 && j < nb) ? 1 : 0) == nb) atomicOr(&done[v >> 5], vbit);
                    ++ncommit;
                }
            }
        }
        __syncthreads();
    }
    return ncommit;
}

// W words per row, TL lanes per light row, GD gathers in flight per lane, MINB CTAs per SM
// WT: weighted sums for the pruned component (prune.cu): S(v) += d * sum over the new
// sources s of (1 + T(s)), the T sum taken from per-batch bit planes of T in shared memory
// HV: heavy-row path compiled in (false only for graphs without heavy rows: a leaner kernel)
// CNT: count the row traffic (gathered rows, own rows read) into counters[8..9] -- a separate
// instantiation, so the timed kernels carry none of it (it costs them ~3 %)
// TC (with WT): the pruned core is in T order (closeness.cu k_vert_keys) -- chunks of one T are weighed by
// T x popc, the others by the planes; a separate instantiation, so graphs without T order run the plain
// plane code
// PS: top-down push phase on a batch's first levels (bfs_push; lean kernels only, see push_level)
template <int W, int TL, int GD, int MINB, bool WT, bool HV = true, bool CNT = false, bool TC = false,
          bool PS = false, int BLOCK = WT ? BLOCK_WEIGHTED : BLOCK_PLAIN>
__global__ void __launch_bounds__(BLOCK, MINB) msbfs_kernel(const __grid_constant__ BfsArgs a) {
    constexpr int T = W / 2 < 32 ? W / 2 : 32;   // lanes per row in the heavy path (W <= 64 with heavy rows)
    constexpr int TPB = BLOCK / T;     // heavy-path teams per block
    constexpr int64_t B = 64 * W;      // sources per batch
    // light rows: TL lanes per row, VEC 16-byte chunks per lane, GD gathers in flight per lane
    constexpr int VEC = W / (2 * TL);
    constexpr int LTPW = 32 / TL;
    cg::grid_group grid = cg::this_grid();
    __shared__ Smem<BLOCK / 32> sm;
    __shared__ unsigned long long s_pl[WT ? BFS_T_BITS : 1][WT ? W : 1];   // T bit planes of the batch window
    __shared__ int s_nb;
    __shared__ int s_tc[TC ? W / 2 : 1];   // T of each 128-source chunk of the window when constant, else -1
#ifdef HM_MSBFS_PROF
    __shared__ int s_tmin, s_tmax;
#endif
    __shared__ ulonglong2 s_red[TPB][T];
    extern __shared__ uint4 s_dyn[];

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int tl = lane % T;
    const int tbase = lane - tl;
    const unsigned tmask = ((T == 32) ? FULL : ((1u << T) - 1u)) << tbase;
    const unsigned ltmask = (1u << lane) - 1u;
    const int64_t nthreads = (int64_t)gridDim.x * BLOCK;
    const int64_t gtid = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
    const int64_t gwarp = gtid >> 5;
    const int64_t nwarps = nthreads >> 5;
    const int tib = threadIdx.x / T;
    const int ltl = lane % TL;
    const int lteam = lane / TL;

    const int n_live = a.scalars[0];
    const int n_giant = a.scalars[1];
    const int n_comp = a.scalars[2];
    const int n_heavy = a.scalars[3];
    const int n_items = (n_heavy > 0 && a.hstart) ? a.hstart[n_heavy] : 0;   // heavy-row items
    const int heavy_deg = a.scalars[4];
    int32_t *su = sm.su[wib];
    uint8_t *sr = sm.sr[wib];
    int16_t *seg = sm.seg[wib];
    // L2 eviction-priority policies (a.hints bits): gathered F_{d-1} rows, own F_{d-2} rows, F_d stores
    // (bit 4: use the hinted instructions with evict_normal where no other policy is set)
    const uint64_t pol_d = (a.hints & 16) ? policy_evict_normal() : 0ull;
    const uint64_t pol_c = (a.hints & 1) ? policy_evict_last() : pol_d;
    const uint64_t pol_p = (a.hints & 2) ? policy_evict_first() : pol_d;
    const uint64_t pol_n = (a.hints & 4) ? policy_evict_last() : (a.hints & 8) ? policy_evict_first() : pol_d;
    Prof pf;
    PROF_INIT(pf);
    (void)pf;
    if (threadIdx.x < 4) sm.lb[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) {
        sm.epoch = 0ull;
        sm.push = sm.emit = 0;
        sm.pn = 0u;
    }
    if (threadIdx.x == 0) sm.pt = 0;    // list-producing levels run by this launch: rotates the pair lists and cursors

    for (int64_t base = 0; base < n_giant; base += B) {
        if (a.nshards > 1 && (int)((base / B) % a.nshards) != a.shard) continue;   // another shard's batch
        if (threadIdx.x == 0) sm.hi = batch_hi(a, base, n_comp, n_live);
        __syncthreads();
        const int hi = sm.hi;
        const int64_t ngroups = (hi + 31) >> 5;

        // ---- level 0: sources of every component window (F_0); bitmaps and counts reset
        const int pt0 = PS ? sm.pt : 0;                              // this level's list index (push phase)
        int nsrc = 0;                                                // source rows (lane 0 counts its groups)
        for (int64_t g = gwarp; g < ngroups; g += nwarps) {
            const int v = (int)(g * 32 + lane);
            bool src = false, dn = false;
            int jsrc = -1;                                           // the row's own source bit, if it is a source
            if (v < hi) {
                const int2 ci = comp_of(a, v, n_giant);
                const int64_t j = (int64_t)v - ci.x - base;
                int64_t nb = (int64_t)ci.y - base;
                if (nb > B) nb = B;
                if (j >= 0 && j < nb) {
                    src = true;
                    dn = (nb == 1);
                    if constexpr (!PS) {
                    uint64_t *f = a.F[0] + (size_t)v * W;           // V_0(v) = {v}
                    const int wj = (int)(j >> 6);
#pragma unroll
                    for (int w = 0; w < W; w += 2)
                        st2(f + w, make_ulonglong2(w == wj ? 1ull << (j & 63) : 0ull,
                                                   w + 1 == wj ? 1ull << (j & 63) : 0ull));
                    }
                    if constexpr (PS) jsrc = (int)j;
                }
                a.K[v] = 0;
            }
            const unsigned bs = __ballot_sync(FULL, src);
            const unsigned bd = __ballot_sync(FULL, dn);
            if constexpr (PS) {
                const unsigned bv = __ballot_sync(FULL, v < hi);
                if (lane == 0) a.has[g] = bv;
                // push phase: every row of the batch holds a visited set from level 0 on (the pushes OR into
                // it): the group's rows are written whole, coalesced -- zero, the sources' own bit set
                constexpr int CPR = W / 2;                               // 16-byte chunks per row
                const int nrow = __popc(bv);
                uint64_t *fg = a.F[0] + (size_t)g * 32 * W;
                for (int i0 = 0; i0 < nrow * CPR; i0 += 32) {
                    const int i = i0 + lane;
                    const int row = i / CPR, w0 = 2 * (i % CPR);
                    const int js = __shfl_sync(FULL, jsrc, row & 31);
                    if (i < nrow * CPR)
                        st2(fg + (size_t)row * W + w0,
                            make_ulonglong2((js >> 6) == w0 ? 1ull << (js & 63) : 0ull,
                                            (js >> 6) == w0 + 1 ? 1ull << (js & 63) : 0ull));
                }
                // the sources are level 0's pairs
                if (bs) {
                    unsigned pos = 0;
                    if (lane == 0) pos = atomicAdd(a.pcur + pt0 % 3, (unsigned)__popc(bs));
                    pos = __shfl_sync(FULL, pos, 0) + __popc(bs & ltmask);
                    if (src && pos < (unsigned)a.pcap)
                        a.plist[pt0 & 1][pos] = ((unsigned long long)v << 16) | (unsigned long long)jsrc;
                }
            }
            if (lane == 0) {
                a.chg[0][g] = bs;     // changed at level 0: the sources
                a.chg[1][g] = 0u;     // written at level 1
                if (!PS) a.has[g] = bs;   // only the sources hold a visited set, in buffer 0 (push phase: every row)
                a.par[g] = 0u;
                a.cand[1][g] = 0u;    // level 1's top-down candidates (level d clears level d+1's)
                nsrc += __popc(bs);
                a.done[g] = bd;
            }
        }
        if (gtid == 0) a.flags[1] = 0;
        if (PS && gtid == 0) a.pcur[(pt0 + 1) % 3] = 0u;        // the next list's cursor
        if (HV && gtid == 0 && a.hclaim) a.hclaim[1] = 0;        // level 1's heavy-item claims
        if constexpr (WT) {
            // bit planes of T over the giant's source window: plane b, word w, bit j =
            // bit b of T(row base + 64 w + j) (rows outside [0, n_giant) weigh 1: T = 0)
            for (int64_t w = gwarp; w < W; w += nwarps) {
                const int64_t r0 = base + 64 * w + lane, r1 = r0 + 32;
                const uint32_t t0 = r0 < n_giant ? a.tw[r0] : 0u, t1 = r1 < n_giant ? a.tw[r1] : 0u;
                for (int b = 0; b < BFS_T_BITS; ++b) {
                    const unsigned lo = __ballot_sync(FULL, (t0 >> b) & 1u), hi1 = __ballot_sync(FULL, (t1 >> b) & 1u);
                    if (lane == 0) a.planes[(size_t)b * W + w] = (unsigned long long)lo | ((unsigned long long)hi1 << 32);
                }
            }
            // chunks of 128 sources (words 2c, 2c+1) with one T: the core rows are sorted by T (k_vert_keys),
            // so nearly all are, and a commit weighs them by T x popc instead of the planes
            if (TC)
            for (int64_t c = gwarp; c < W / 2; c += nwarps) {
                unsigned tmin = 0xffffffffu, tmax = 0u;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int64_t r = base + 128 * c + 32 * k + lane;
                    if (r < n_giant) {
                        const uint32_t t = a.tw[r];
                        tmin = min(tmin, t);
                        tmax = max(tmax, t);
                    }
                }
                tmin = __reduce_min_sync(FULL, tmin);
                tmax = __reduce_max_sync(FULL, tmax);
                if (lane == 0) a.tconst[c] = tmin == 0xffffffffu ? 0 : (tmin == tmax ? (int)tmin : -1);
            }
        }
        if (a.lbar) {                                                // the level-0 frontier: the sources
            if (threadIdx.x == 0) sm.nchg = 0;
            __syncthreads();
            nsrc = __reduce_add_sync(FULL, nsrc);
            if (lane == 0 && nsrc) atomicAdd(&sm.nchg, nsrc);
            __syncthreads();
            if (threadIdx.x == 0) {
                count_barrier(a.lbar, sm, sm.nchg);
                if constexpr (PS) {
                    push_decide(a, sm, pt0, hi, true);
                    sm.pt = pt0 + 1;
                }
            }
            __syncthreads();
        } else {
            grid.sync();
            if (threadIdx.x == 0) sm.nlast = -1;
        }
        int po = 0;                                                   // buffer parity offset after a push phase
        bool ended = false;                                           // the batch ended inside the push phase
        if constexpr (WT) {
            if (threadIdx.x == 0) s_nb = 0;
            __syncthreads();
            for (int i = threadIdx.x; i < BFS_T_BITS * W; i += BLOCK) {
                const unsigned long long x = a.planes[i];
                s_pl[i / W][i % W] = x;
                if (x) atomicMax(&s_nb, i / W + 1);
            }
            if (TC)
                for (int i = threadIdx.x; i < W / 2; i += BLOCK) s_tc[i] = a.tconst[i];
            __syncthreads();
        }

        int d = 1;
        unsigned long long t_prev = 0;
        if (a.dbgc && gtid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_prev));
        if constexpr (PS) {
            // push phase: levels 1 .. d-1 run top-down (push_phase); a negative count = the batch ended there
            const int np = push_phase<W, WT>(a, sm, base, hi, n_giant, &t_prev);
            d = np < 0 ? -np : np + 1;                                // (ended at level -np: that many levels ran)
            // pushes wrote F[0]: the first bottom-up level d gathers it as F[(d - 1 + po) & 1]
            po = (d - 1) & 1;
            ended = np < 0;
        }
        if (!ended)
        for (;; ++d) {
            PROF_LEVEL(pf, d);
            // rows changed at d-1 hold V_{d-1} in F[(d-1) & 1] (gathered); a row changing at d
            // writes V_d into F[d & 1]; a row's own V_{d-1} is in the buffer of its last change
            const uint64_t *__restrict__ Fc = a.F[(d - 1 + po) & 1];
            uint64_t *__restrict__ Fn = a.F[(d + po) & 1];
            const uint64_t *F0 = a.F[0], *F1 = a.F[1];
            const uint32_t *chp = a.chg[(d + 2) % 3];
            uint32_t *chn = a.chg[d % 3];
            uint32_t *chz = a.chg[(d + 1) % 3];
            uint32_t *cand_n = a.cand[(d + 1) & 1];
            for (int64_t w = gtid; w < ngroups; w += nthreads) {
                chz[w] = 0u;
                cand_n[w] = 0u;                                  // level d+1's top-down candidates
            }
            if (gtid == 0) a.flags[(d + 1) % 3] = 0;
            if (HV && gtid == 0 && a.hclaim) a.hclaim[(d + 1) % 3] = 0;   // next level's claims
            // stage the two previous change bitmaps in shared memory
            const uint32_t *chp_s = chp;
            if (threadIdx.x == 0) {
                sm.next = a.interleave ? 0 : (int)(((int64_t)blockIdx.x * (ngroups << a.unit_shift)) / gridDim.x);
                sm.nchg = 0;
                sm.ngat = 0u;
                sm.nown = 0u;
            }
            if (a.chg_smem) {
                const int nw4 = (int)((ngroups + 3) >> 2);
                uint4 *d0 = s_dyn;
                const uint4 *s0 = reinterpret_cast<const uint4 *>(chp);
                for (int i = threadIdx.x; i < nw4; i += BLOCK) d0[i] = s0[i];
                chp_s = reinterpret_cast<const uint32_t *>(d0);
            }
            // direction: top-down when the frontier (rows changed at d-1) is small against the batch's rows
            const long long frontier = sm.nlast;
            const bool td = a.td_div > 0 && a.lbar && frontier >= 0 && frontier * a.td_div <= (long long)hi;
            const uint32_t *cand = td ? a.cand[d & 1] : nullptr;
            __syncthreads();
            if (td) {
                td_discover(a.row_ptr, a.col, chp_s, a.done, a.cand[d & 1], hi, ngroups, gwarp, nwarps);
                __syncthreads();
                if (threadIdx.x == 0) count_barrier(a.lbar, sm, 0);
                __syncthreads();
            }
            PROF_MARK(pf, 0);
#ifdef HM_MSBFS_PROF
            const long long t_lvl0 = clock64();
            if (threadIdx.x == 0) {
                s_tmin = 0x7fffffff;
                s_tmax = 0;
            }
            __syncthreads();
#endif
            int nchg = 0;                 // rows changed by this thread (lane 0 of a unit / heavy committer)

            // ---- heavy rows (heavy_items): items of BFS_HEAVY_CHUNK arcs, claimed after the light
            // units (below); HM_HEAVY_DYN 0 deals them round-robin here instead
            if constexpr (HV && !HM_HEAVY_DYN)
                if (n_items > 0)
                nchg = heavy_items<W, BLOCK, WT>(a.row_ptr, a.col, a.cinfo, a.heavy, a.hstart, a.hacc, a.hcnt, a.done,
                                                a.K, a.S, nullptr, &s_red[0][0], &s_pl[0][0], s_nb, n_items, n_heavy,
                                                hi, n_giant, base, d, chp_s, a.has, a.par, Fc, F0, F1, Fn, chn,
                                                cand, CNT ? &sm.ngat : nullptr);
            PROF_MARK(pf, 1);

            // ---- light rows: one warp per unit of 32 >> unit_shift rows of a 32-row group;
            // each CTA owns a contiguous range of units and its warps claim them
            // dynamically (smaller units: less end-of-level quantisation)
            const int us = a.unit_shift;
            const int ur = 32 >> us;                                    // rows per unit
            const int64_t nunits = ngroups << us;
            // interleave (a.interleave): CTA b owns units b, b + grid, b + 2 grid, ... so a
            // cluster of busy rows (e.g. the batch's own source community at levels 2-3) is
            // spread over all CTAs instead of landing in a few contiguous ranges
            const int64_t u_end = a.interleave ? nunits : ((int64_t)(blockIdx.x + 1) * nunits) / gridDim.x;
            for (;;) {
                int64_t un = 0;
                if (lane == 0) un = (int64_t)atomicAdd(&sm.next, 1);
                un = __shfl_sync(FULL, un, 0);
                if (a.interleave) {
                    // ... and the claim order starts at the batch's source window, whose rows
                    // (one dense region of the graph) carry the most work in the first levels
                    un = un * gridDim.x + blockIdx.x;
                    if (un >= u_end) break;
                    un += ((int64_t)(base >> 5)) << us;
                    if (un >= nunits) un -= nunits;
                }
                if (un >= u_end) break;
                const int64_t g = un >> us;
                const int q0 = (int)(un & ((1 << us) - 1)) * ur;           // first row of the unit in the group
                const int r = (int)(g * 32 + lane);
                const bool valid = r < hi;
                const bool inunit = lane >= q0 && lane < q0 + ur;
                const int rp = a.row_ptr[valid ? r : hi];
                const int rlast = a.row_ptr[(int)(g * 32 + 32) < hi ? (int)(g * 32 + 32) : hi];
                const uint32_t dword = a.done[g] | (td ? ~cand[g] : 0u);   // top-down: candidates only
                const int rnext = __shfl_down_sync(FULL, rp, 1);
                const int rend = (lane == 31) ? rlast : rnext;
                const bool act = valid && inunit && !((dword >> lane) & 1u) && (rend - rp) <= heavy_deg;
                const unsigned amask = __ballot_sync(FULL, act);
                PROF_MARK(pf, 2);
                if (!amask) continue;                                    // warp-uniform
                const uint32_t hword = a.has[g], qword = a.par[g];     // own rows: state held, its buffer
                uint32_t chg_bits = 0u, done_bits = 0u;
                const int A0 = __shfl_sync(FULL, rp, q0);
                const int A1 = __shfl_sync(FULL, rend, q0 + ur - 1);    // end of the unit's last row
                int n = 0;
                for (int a0 = A0; a0 < A1; a0 += 32 * SCAN_U) {
                    int xx[SCAN_U];
        #pragma unroll
                    for (int q = 0; q < SCAN_U; ++q) {
                        const int aa = a0 + 32 * q + lane;
#if HM_CSR_POLICY
                        xx[q] = aa < A1 ? ld_pol(a.col + aa, pol_c) : -1;
#else
                        xx[q] = aa < A1 ? ld_cs(a.col + aa) : -1;
#endif
                    }
        #pragma unroll
                    for (int q = 0; q < SCAN_U; ++q) {
                        const int x = xx[q];
                        const int u = x >> 5, ri = x & 31;
                        const bool ok = x >= 0 && ((amask >> ri) & 1u) && bit_of(chp_s, u);
                        const unsigned bm = __ballot_sync(FULL, ok);
                        if (ok) {
                            const int pos = n + __popc(bm & ltmask);
                            su[pos] = u;
                            sr[pos] = (uint8_t)ri;
                        }
                        n += __popc(bm);
                    }
                    const bool flush = (n > CAP - 32 * SCAN_U) || (a0 + 32 * SCAN_U >= A1);
                    PROF_MARK(pf, 3);
                    if (!flush || n == 0) continue;
                    if (CNT && lane == 0) atomicAdd(&sm.ngat, (unsigned)n);  // this flush's gathers
                    __syncwarp();
                    // segments: runs of equal row index (at most 32)
                    int nseg = 0;
                    for (int k0 = 0; k0 < n; k0 += 32) {
                        const int k = k0 + lane;
                        const bool stt = k < n && (k == 0 || sr[k] != sr[k - 1]);
                        const unsigned sb = __ballot_sync(FULL, stt);
                        if (stt) seg[nseg + __popc(sb & ltmask)] = (int16_t)k;
                        nseg += __popc(sb);
                    }
                    if (lane == 0) seg[nseg] = (int16_t)n;
                    __syncwarp();
                    if constexpr (CNT) {                                       // own rows read this flush
                        const bool own = lane < nseg && (((hword | chg_bits) >> sr[seg[lane]]) & 1u);
                        const unsigned ob = __ballot_sync(FULL, own);
                        if (lane == 0 && ob) atomicAdd(&sm.nown, (unsigned)__popc(ob));
                    }
                    // sort the segments by length (descending) so the TPW rows of a
                    // lock-step round have similar neighbour counts
                    int key = lane < nseg ? (((seg[lane + 1] - seg[lane]) << 5) | lane) : -1;
        #pragma unroll
                    for (int k = 2; k <= 32; k <<= 1) {
        #pragma unroll
                        for (int j = k >> 1; j > 0; j >>= 1) {
                            const int other = __shfl_xor_sync(FULL, key, j);
                            const bool keep_max = (((lane & k) == 0) == ((lane & j) == 0));
                            key = keep_max ? max(key, other) : min(key, other);
                        }
                    }
                    PROF_MARK(pf, 4);
                    uint32_t cb_team = 0u, db_team = 0u;   // per-team-leader bits of this flush
                    for (int s0 = 0; s0 < nseg; s0 += LTPW) {
                        const int mykey = __shfl_sync(FULL, key, (s0 + lteam) & 31);
                        const int rlen = __shfl_sync(FULL, key, s0) >> 5;        // longest in round
                        const bool has = s0 + lteam < nseg;
                        const int sg = mykey & 31;
                        const int kb = has ? seg[sg] : 0;
                        const int ke = has ? seg[sg + 1] : 0;
                        const int ri = has ? sr[kb] : 0;
                        const int v = (int)(g * 32 + ri);
                        // row state, issued with the gathers: own V_{d-1} (or the V_d an earlier
                        // staging flush of this unit wrote), K, S
                        ulonglong2 vv[VEC];
                        zero_row<VEC>(vv);
                        if (has && ((chg_bits >> ri) & 1u)) {
                            ld_row<W, TL, VEC>(vv, Fn, v, ltl);
                        } else if (has && ((hword >> ri) & 1u)) {
                            const bool q = (qword >> ri) & 1u;
                            // written at d-1: also gathered by the neighbours this level
                            ld_row<W, TL, VEC>(vv, q ? F1 : F0, v, ltl, q == (bool)((d - 1 + po) & 1) ? pol_c : pol_p);
                        }
                        int Kv = 0;
                        uint64_t Sv = 0;
                        if (has && ltl == 0) {
                            Kv = a.K[v];
                            Sv = a.S[v];
                        }
                        ulonglong2 acc[VEC];
                        zero_row<VEC>(acc);
                        PROF_COUNT(pf, 0, 1);
                        for (int k0 = kb; k0 < kb + rlen; k0 += GD) {
                            PROF_COUNT(pf, 1, 1);
                            ulonglong2 x[GD][VEC];
        #pragma unroll
                            for (int q = 0; q < GD; ++q) {
                                zero_row<VEC>(x[q]);
                                if (k0 + q < ke) ld_row<W, TL, VEC>(x[q], Fc, su[k0 + q], ltl, pol_c);
                            }
        #pragma unroll
                            for (int q = 0; q < GD; ++q) or_row<VEC>(acc, x[q]);
                        }
                        int cnt = 0;
        #pragma unroll
                        for (int q = 0; q < VEC; ++q) {
                            acc[q].x &= ~vv[q].x;
                            acc[q].y &= ~vv[q].y;
                            cnt += __popcll(acc[q].x) + __popcll(acc[q].y);
                        }
        #pragma unroll
                        for (int o = TL / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
                        unsigned long long wsum = 0ull;   // sum of T over the new sources (pruned component)
                        if constexpr (WT) {
                            // chunks of one T: T x popc; the others by T's bit planes (rows without new
                            // sources skip both: cnt is team-uniform here)
                            int needp = 0;
                            if (TC && has && cnt && v < n_giant) {
        #pragma unroll
                                for (int q = 0; q < VEC; ++q) {
                                    const int t = s_tc[q * TL + ltl];
                                    if (t >= 0) wsum += (unsigned long long)t * (unsigned)(__popcll(acc[q].x) + __popcll(acc[q].y));
                                    else needp = 1;
                                }
                            }
                            const int nbp = (TC ? needp : (has && cnt && v < n_giant)) ? s_nb : 0;
                            const int nbw = __reduce_max_sync(FULL, (unsigned)nbp);   // warp-uniform trip count
                            for (int b = 0; b < nbw; ++b) {
                                unsigned c2 = 0;
        #pragma unroll
                                for (int q = 0; q < VEC; ++q) {
                                    const int wi = 2 * (q * TL + ltl);
                                    if (!TC || s_tc[q * TL + ltl] < 0)
                                        c2 += __popcll(acc[q].x & s_pl[b][wi]) + __popcll(acc[q].y & s_pl[b][wi + 1]);
                                }
                                if (b < nbp) wsum += (unsigned long long)c2 << b;
                            }
        #pragma unroll
                            for (int o = TL / 2; o > 0; o >>= 1) wsum += __shfl_xor_sync(FULL, wsum, o);
                        }
                        if (cnt) {
                            or_row<VEC>(acc, vv);                         // V_d(v) = V_{d-1}(v) | new
                            st_row<W, TL, VEC>(Fn, v, ltl, acc, pol_n);
                            if (ltl == 0) {
                                const int2 ci = comp_of(a, v, n_giant);
                                int64_t nb = (int64_t)ci.y - base;
                                if (nb > B) nb = B;
                                const int64_t j = (int64_t)v - ci.x - base;
                                const int kn = Kv + cnt;
                                a.K[v] = (uint16_t)kn;
                                if constexpr (WT)
                                    a.S[v] = Sv + (uint64_t)d * ((uint64_t)cnt + wsum);
                                else
                                    a.S[v] = Sv + (uint64_t)d * (uint64_t)cnt;
                                cb_team |= 1u << ri;
                                if (kn + ((j >= 0 && j < nb) ? 1 : 0) == nb) db_team |= 1u << ri;
                            }
                        }
                    }
                    // merge the team leaders' bits: warp-uniform
        #pragma unroll
                    for (int o = TL; o < 32; o <<= 1) {
                        cb_team |= __shfl_xor_sync(FULL, cb_team, o);
                        db_team |= __shfl_xor_sync(FULL, db_team, o);
                    }
                    cb_team = __shfl_sync(FULL, cb_team, 0);
                    db_team = __shfl_sync(FULL, db_team, 0);
                    chg_bits |= cb_team;
                    PROF_MARK(pf, 5);
                    done_bits |= db_team;
                    n = 0;
                    __syncwarp();
                }
                if (lane == 0) {
                    if (chg_bits) {
                        atomicOr(&chn[g], chg_bits);
                        atomicOr(&a.has[g], chg_bits);
                        if ((d + po) & 1) atomicOr(&a.par[g], chg_bits);
                        else atomicAnd(&a.par[g], ~chg_bits);
                        nchg += __popc(chg_bits);
                    }
                    if (done_bits) atomicOr(&a.done[g], done_bits);
                }
                PROF_MARK(pf, 2);
            }
#ifdef HM_MSBFS_PROF
            if (pf.on && lane == 0) {          // spread of the warps' exit times from the unit loop
                const int te = (int)((clock64() - t_lvl0) >> 4);
                atomicMin(&s_tmin, te);
                atomicMax(&s_tmax, te);
            }
#endif
            // heavy items claimed dynamically by the CTAs as they finish their light units (a CTA
            // holding a hub no longer finishes last; C4 layers -5 %, C3 -6 % against dealing them
            // round-robin before the light units; compiling both placements in is slower than either)
            if constexpr (HV && HM_HEAVY_DYN)
                if (n_items > 0)
                nchg += heavy_items<W, BLOCK, WT>(a.row_ptr, a.col, a.cinfo, a.heavy, a.hstart, a.hacc, a.hcnt, a.done,
                                                 a.K, a.S, a.hclaim + (d % 3), &s_red[0][0], &s_pl[0][0], s_nb, n_items,
                                                 n_heavy, hi, n_giant, base, d, chp_s, a.has, a.par, Fc, F0, F1, Fn,
                                                 chn, cand, CNT ? &sm.ngat : nullptr);
            // rows changed by this CTA: warp sums, one shared atomic per warp
            nchg = __reduce_add_sync(FULL, nchg);
            if (lane == 0 && nchg) atomicAdd(&sm.nchg, nchg);
            __syncthreads();
            const int nchg_cta = sm.nchg;
            if (CNT && threadIdx.x == 0) {                               // row traffic of this CTA's level
                if (sm.ngat) atomicAdd(a.counters + 8, (unsigned long long)sm.ngat);
                if (sm.nown) atomicAdd(a.counters + 9, (unsigned long long)sm.nown);
            }
            // one flag write per CTA (same-address stores from every group serialise in L2)
            if (nchg_cta && threadIdx.x == 0 && !a.lbar) a.flags[d % 3] = 1;
#ifdef HM_MSBFS_PROF
            if (pf.on && threadIdx.x == 0 && a.dbgc) {
                atomicAdd(a.dbgc + 8202, (unsigned long long)s_tmin << 4);
                atomicAdd(a.dbgc + 8203, (unsigned long long)s_tmax << 4);
                atomicAdd(a.dbgc + 8204, 1ull);
            }
#endif
            PROF_MARK(pf, 6);
            if (a.lbar) {
                if (threadIdx.x == 0) {
                    count_barrier(a.lbar, sm, nchg_cta);                      // sm.nlast = rows changed at d
                    level_guard(sm, d, a.counters);
                }
                __syncthreads();
            } else {
                grid.sync();
                if (threadIdx.x == 0) {
                    sm.flag = *((volatile int32_t *)(a.flags + (d % 3)));
                    sm.nlast = -1;                                   // unknown without the counting barrier
                    level_guard(sm, d, a.counters);
                }
                __syncthreads();
            }
            PROF_MARK(pf, 7);
            const int fv = sm.flag;
            if (gtid == 0) {
                if (sm.nlast > 0) {
                    a.counters[3] += (unsigned long long)sm.nlast;                  // row commits
                    a.counters[6] += (unsigned long long)sm.nlast * 2ull * 8ull * W;   // own read + row write
                }
                if (td) a.counters[5] += 1ull;                                      // top-down levels
            }
            if (a.dbgc && gtid == 0) {
                unsigned long long now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                const int di = d < 4095 ? d : 4095;
                a.dbgc[di] += 1ull;
                a.dbgc[4096 + di] += now - t_prev;
                if (sm.nlast > 0) a.dbgc[12288 + di] += (unsigned long long)sm.nlast;   // rows changed at d
                if (td) a.dbgc[16384 + di] += 1ull;                                      // top-down at d
                t_prev = now;
            }
            if (fv == 0) break;
        }
        if (gtid == 0) {
            a.counters[0] += (unsigned long long)d;
            a.counters[1] += 1ull;
            // dense-level model bytes of this batch: rows [0, hi) and their arcs
            const unsigned long long arcs = (unsigned long long)a.row_ptr[hi];
            a.counters[2] += (unsigned long long)d *
                             (4ull * (hi + 1) + 4ull * arcs + 2ull * 8ull * W * (unsigned long long)hi);
            a.counters[4] += (unsigned long long)d * (4ull * (hi + 1) + 4ull * arcs);   // CSR bytes per level
        }
    }
    PROF_FLUSH(pf, a.dbgc);
}

}  // namespace

int launch_msbfs(int W, int TL, int GD, const BfsArgs &a, int num_sms, int blocks_per_sm, cudaStream_t s,
                 int64_t units) {
    const void *kern = nullptr;
    int block = BLOCK_PLAIN;
    if (TL == 0) TL = (W >= 64) ? 16 : W / 2;
    const int vec = W / (2 * TL);
    const int minb = blocks_per_sm == 1 ? 1 : 2;
    const bool push = a.push_num > 0 && a.plist[0] && a.lbar && !a.hstart && !a.count_rows && a.td_div == 0;
    // gathers in flight per lane: 4 at W = 64 with 2 CTAs/SM (round 2, visited-set rows: C5 layer
    // 68.8 -> 64.8 ms, AND 62.2 -> 58.6 ms against 2)
    if (GD == 0) GD = (minb == 1) ? (vec == 1 ? 8 : 4) : (vec == 1 ? 4 : (vec == 2 && W == 64 ? 4 : 2));
#define HM_MSBFS_CASE(w, tl, gd, mb)                                                                     \
    case ((w * 100 + tl) * 100 + gd * 10 + mb):                                                          \
        kern = a.tw ? (const void *)msbfs_kernel<w, tl, gd, mb, true> : (const void *)msbfs_kernel<w, tl, gd, mb, false>; \
        block = a.tw ? BLOCK_WEIGHTED : BLOCK_PLAIN;                                                     \
        break;
    switch ((W * 100 + TL) * 100 + GD * 10 + minb) {
        HM_MSBFS_CASE(8, 4, 4, 2)
        HM_MSBFS_CASE(8, 4, 8, 1)
        HM_MSBFS_CASE(16, 8, 8, 1)
        HM_MSBFS_CASE(16, 8, 4, 2)
        HM_MSBFS_CASE(16, 4, 2, 2)
        HM_MSBFS_CASE(32, 16, 4, 2)
        HM_MSBFS_CASE(32, 16, 8, 1)
        HM_MSBFS_CASE(32, 8, 2, 2)
        HM_MSBFS_CASE(64, 32, 4, 2)
    case ((64 * 100 + 16) * 100 + 4 * 10 + 2):                 // default: lean variants without heavy rows
        if (a.count_rows) {                                     // row-traffic counting instantiations
            if (a.hstart)
                kern = a.tw ? (const void *)msbfs_kernel<64, 16, 4, 2, true, true, true>
                            : (const void *)msbfs_kernel<64, 16, 4, 2, false, true, true>;
            else
                kern = a.tw ? (const void *)msbfs_kernel<64, 16, 4, 2, true, false, true>
                            : (const void *)msbfs_kernel<64, 16, 4, 2, false, false, true>;
        } else if (push) {                                      // top-down push phase on the first levels
            kern = !a.tw ? (const void *)msbfs_kernel<64, 16, 4, 2, false, false, false, false, true>
                 : a.tconst ? (const void *)msbfs_kernel<64, 16, 4, 2, true, false, false, true, true>
                            : (const void *)msbfs_kernel<64, 16, 4, 2, true, false, false, false, true>;
        } else if (a.tw && a.tconst) {                         // weighted, T-ordered core
            kern = a.hstart ? (const void *)msbfs_kernel<64, 16, 4, 2, true, true, false, true>
                            : (const void *)msbfs_kernel<64, 16, 4, 2, true, false, false, true>;
        } else if (a.hstart)
            kern = a.tw ? (const void *)msbfs_kernel<64, 16, 4, 2, true> : (const void *)msbfs_kernel<64, 16, 4, 2, false>;
        else
            kern = a.tw ? (const void *)msbfs_kernel<64, 16, 4, 2, true, false>
                        : (const void *)msbfs_kernel<64, 16, 4, 2, false, false>;
        block = a.tw ? BLOCK_WEIGHTED : BLOCK_PLAIN;
        break;
        HM_MSBFS_CASE(64, 16, 2, 2)
    case ((128 * 100 + 16) * 100 + 2 * 10 + 2):               // W = 128: graphs without heavy rows only
        if (a.hstart) return -1;
        if (a.count_rows)
            kern = a.tw ? (const void *)msbfs_kernel<128, 16, 2, 2, true, false, true>
                        : (const void *)msbfs_kernel<128, 16, 2, 2, false, false, true>;
        else if (push)
            kern = !a.tw ? (const void *)msbfs_kernel<128, 16, 2, 2, false, false, false, false, true>
                 : a.tconst ? (const void *)msbfs_kernel<128, 16, 2, 2, true, false, false, true, true>
                            : (const void *)msbfs_kernel<128, 16, 2, 2, true, false, false, false, true>;
        else if (a.tw && a.tconst)
            kern = (const void *)msbfs_kernel<128, 16, 2, 2, true, false, false, true>;
        else
            kern = a.tw ? (const void *)msbfs_kernel<128, 16, 2, 2, true, false>
                        : (const void *)msbfs_kernel<128, 16, 2, 2, false, false>;
        block = a.tw ? BLOCK_WEIGHTED : BLOCK_PLAIN;
        break;
    case ((128 * 100 + 16) * 100 + 4 * 10 + 2):
        if (a.hstart) return -1;
        kern = a.tw ? (const void *)msbfs_kernel<128, 16, 4, 2, true, false>
                    : (const void *)msbfs_kernel<128, 16, 4, 2, false, false>;
        block = a.tw ? BLOCK_WEIGHTED : BLOCK_PLAIN;
        break;
        HM_MSBFS_CASE(64, 16, 4, 1)
        HM_MSBFS_CASE(64, 16, 8, 2)
        HM_MSBFS_CASE(64, 16, 8, 1)
        HM_MSBFS_CASE(64, 32, 8, 1)
        default: return -1;
    }
#undef HM_MSBFS_CASE
    size_t dyn = a.chg_smem ? (size_t)a.chg_words * 4 : 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn) != cudaSuccess) return -5;
    int maxb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, kern, block, dyn) != cudaSuccess) return -2;
    if (maxb < 1) return -3;
    const int b = (minb < maxb) ? minb : maxb;
    int grid = num_sms * b;
    if (units > 0) {
        const int64_t need = (units + block / 32 - 1) / (block / 32);
        if (need < grid) grid = need < 1 ? 1 : (int)need;
    }
    BfsArgs args = a;
    void *kargs[] = {(void *)&args};
    if (cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(block), kargs, dyn, s) != cudaSuccess) return -4;
    return grid;
}

}  // namespace hm
