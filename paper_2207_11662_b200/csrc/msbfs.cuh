// Multi-source bit-parallel BFS (MS-BFS) for all-sources closeness -- interface.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace hm {

// Rows of degree > min(heavy_deg, BFS_MAX_LIGHT_DEG) are processed by whole CTAs.
constexpr int BFS_MAX_LIGHT_DEG = 1 << 30;
constexpr int BFS_T_BITS = 24;
#ifndef HM_HEAVY_CHUNK
#define HM_HEAVY_CHUNK 1024
#endif
constexpr int BFS_HEAVY_CHUNK = HM_HEAVY_CHUNK;   // arcs per heavy-row work item (one CTA each)        // pruned MS-BFS: hanging-tree sizes T < 2^24 (weight bit planes)

// Device-resident description of one relabelled graph for the MS-BFS kernel.
// Rows 0..n_live-1 are the non-isolated vertices, grouped by connected
// component, components sorted by size descending (see closeness.cu).
struct BfsArgs {
    const int32_t *row_ptr;      // relabelled CSR (rows >= n_live have degree 0)
    const int32_t *col;          // packed arcs: (neighbour << 5) | (row & 31)
    const int2 *cinfo;           // per live row: (first row of its component, component size)
    const int32_t *comp_size;    // per component rank (descending sizes)
    const int32_t *comp_start;   // per component rank: first row
    const int32_t *scalars;      // [0] n_live, [1] n_giant (largest size), [2] n_comp, [3] n_heavy,
                                 // [4] heavy-row degree threshold
    const int32_t *heavy;        // rows with degree > heavy_deg (any order)
    const int32_t *hstart;       // [n_heavy + 1] first item of each heavy row (ceil(deg / BFS_HEAVY_CHUNK) items)
    unsigned long long *hacc;    // [n_heavy][W] zeroed: partial OR rows of multi-item heavy rows
    int32_t *hcnt;               // [n_heavy] zeroed: items of the row done this level
    int32_t *hclaim;             // [3] heavy-item claim counters, rotated by level
    uint64_t *F[2];              // [n_live][W] visited-set rows V(v), double-buffered: a row that
                                 // changes at level d writes V_d(v) into F[d & 1]
    uint32_t *chg[3];            // row bitmaps "changed at level", rotating over 3 levels
    uint32_t *done;              // row bitmap: all sources of the row's window reached it
    uint32_t *has;               // row bitmap: the row holds a visited set in this batch
    uint32_t *par;               // row bitmap: parity of the level that last wrote the row (its buffer)
    uint32_t *cand[2];           // top-down levels: rows adjacent to the frontier ("candidates"), by level parity
    int td_div;                  // direction switch: a level runs top-down (frontier-driven candidate rows)
                                 // when frontier rows * td_div <= the batch's rows; 0 = always bottom-up
    uint16_t *K;                 // [n_live] window sources reached so far in this batch (self excluded)
    uint64_t *S;                 // [n_live] distance-sum accumulators (target side)
    int32_t *flags;              // [3] any-change flags, rotated by level
    unsigned long long *counters;  // [0] levels, [1] batches, [2] model bytes, [3] row commits,
                                   // [4] CSR bytes, [5] top-down levels, [6] state bytes of the commits,
                                   // [7] level guard tripped (hm_get_stats fails), [8] rows gathered,
                                   // [9] own rows read
    unsigned long long *dbgc;    // debug (bfs_dbg & 2): per-level counts and times (+ phase cycles)
    int chg_smem;                // 1: stage the previous level's change bitmap in dynamic shared memory
    int chg_words;               // bitmap words (multiple of 4)
    int unit_shift;              // light-path work unit = 32 >> unit_shift rows of a 32-row group
    int shard, nshards;          // run batches i = shard, shard + nshards, ... only
    int interleave;              // 1: CTA b owns units b, b + grid, ...; 0: a contiguous range
    const uint32_t *tw;          // pruned MS-BFS: hanging-tree size T per row (nullptr: unweighted)
    unsigned long long *planes;  // [BFS_T_BITS][W] scratch: T bit planes of the batch window
    int32_t *tconst;             // [W/2] scratch: per 128-source chunk of the window, its T if constant, else -1
    int hints;                   // L2 policy bits: 1 gathers evict_last, 2 own F_{d-2} evict_first,
                                 // 4 F_d stores evict_last, 8 F_d stores evict_first, 16 evict_normal
    unsigned long long *lbar;    // [4] counting grid-barrier counters (zeroed): arrivals [p] and changed rows
                                 // [2 + p] by barrier-epoch parity p; nullptr: grid.sync + flag (no top-down)
    int dbg_level;               // HM_MSBFS_PROF builds: profile only this level (<= 0: all)
    int count_rows;              // 1: run the row-traffic counting instantiation (default kernels; counters[8..9])
    // top-down push phase of a batch's first (sparse) levels (bfs_push; lean default kernels only):
    int push_num;                // a level pushes when the pairs (row, source) found at the previous level
                                 // number <= rows * push_num / 4; 0 = off (no push instantiation)
    unsigned long long *plist[2];  // [pcap] pair lists (row << 16 | source bit), alternating by level
    unsigned *pcur;              // [3] list cursors (zeroed), rotating over the launch's levels
    int pcap;                    // list capacity in pairs
};

// Launches the persistent cooperative kernel for W words (64*W sources per
// batch).  Returns the grid size (< 0: no instantiation / launch failure).
// TL = lanes per state row in the light path (0 = default: W/2, 16 at W = 64);
// GD = gathers in flight per lane (0 = default for the occupancy);
// blocks_per_sm == 1 selects the 1-CTA/SM (128-register) instantiations, else 2 CTAs/SM.
// units > 0: the light-path work units of the largest batch; the grid is capped at one unit per warp
// (small graphs: fewer CTAs in every level barrier).
int launch_msbfs(int W, int TL, int GD, const BfsArgs &a, int num_sms, int blocks_per_sm, cudaStream_t s,
                 int64_t units = 0);

}  // namespace hm
