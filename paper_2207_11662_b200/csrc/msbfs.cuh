// Multi-source bit-parallel BFS (MS-BFS) for all-sources closeness -- interface.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace hm {

// Device-resident description of one relabelled graph for the MS-BFS kernel.
// Rows 0..n_live-1 are the non-isolated vertices, grouped by connected
// component, components sorted by size descending (see closeness.cu).
struct BfsArgs {
    const int32_t *row_ptr;      // relabelled CSR (rows >= n_live have degree 0)
    const int32_t *col;
    const int2 *cinfo;           // per live row: (first row of its component, component size)
    const int32_t *comp_size;    // per component rank (descending sizes)
    const int32_t *comp_start;   // per component rank: first row
    const int32_t *scalars;      // [0] n_live, [1] n_giant (largest size), [2] n_comp, [3] n_heavy
    const int32_t *heavy;        // rows with degree > heavy_deg (any order)
    int32_t heavy_deg;
    uint64_t *vis;               // [n_live][W]  visited bits (valid where "touched")
    uint64_t *F0, *F1;           // [n_live][W]  frontier (new bits of the level), ping-pong
    uint32_t *chg0, *chg1, *chg2;  // row bitmaps: row changed at a level (3-way rotation)
    uint32_t *done;              // row bitmap: all sources of the row's window reached it
    uint32_t *touched;           // row bitmap: vis row has been written in this batch
    uint64_t *S;                 // [n_live] distance-sum accumulators (target side)
    int32_t *flags;              // [3] any-change flags, rotated by level
    unsigned long long *counters;  // [0] levels, [1] batches
    unsigned long long *dbgc;    // debug: [d] rows changed at level d, [4096+d] blocks that saw the flag set
    unsigned *bar;               // [2] grid-barrier state (zeroed before launch)
    int dbg;                     // debug bits: 1 = per-thread fence before each grid barrier
};

// Launches the persistent cooperative kernel for W words (64*W sources per
// batch).  blocks_per_sm == 0 -> occupancy maximum.  Returns the grid size.
int launch_msbfs(int W, const BfsArgs &a, int num_sms, int blocks_per_sm, cudaStream_t s);

}  // namespace hm
