/*
 * hm.h -- C ABI of the B200 (sm_100a) closeness-centrality library for
 * homogeneous multilayer networks (arXiv 2207.11662, "Closeness Centrality
 * Detection in Homogeneous Multilayer Networks").
 *
 * Problem statement followed (§1): given the layers
 * G_1(V,E_1) ... G_l(V,E_l) of a HoMLN over one vertex set V, identify the
 * closeness-centrality (CC) nodes of the Boolean-AND aggregate of any r <= l
 * layers, from per-layer partial results computed once (the decoupling
 * approach, §3).
 *
 * Every entry point is stream-ordered on the context's CUDA stream.  All
 * compute runs in this library's own CUDA kernels; there is no CPU fallback.
 * Pointers called "host or device" are classified with
 * cudaPointerGetAttributes; host outputs are complete when the call returns,
 * device outputs are complete in stream order.
 *
 * Errors: no exception crosses the ABI.  A non-zero status leaves every output
 * untouched, stores a message retrievable with hm_last_error(), and leaves the
 * context usable (except after HM_ECUDA from a sticky device fault).
 *
 * Threading: one context is used by one host thread at a time; distinct
 * contexts are independent.  Results are bit-identical across runs and do not
 * depend on tuning parameters (hm_set_param).
 */
#ifndef HM_H
#define HM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hm_ctx hm_ctx;      /* opaque: owns device memory and (optionally) a stream */
typedef int32_t hm_status;

enum {
    HM_OK = 0,
    HM_EINVAL = -1,   /* bad argument: V <= 0, l < 1, r < 2, K not in [1, V], null pointer, unknown enum */
    HM_ERANGE = -2,   /* vertex id outside [0, V), or 2m >= 2^31 arcs (int32 CSR)                          */
    HM_ENOMEM = -3,   /* device allocation failed                                                          */
    HM_ECUDA = -4,    /* CUDA runtime / kernel error (message has cudaGetErrorString)                       */
    HM_ESTATE = -5    /* unknown / freed graph id, compose before closeness, free of a layer              */
};

enum { HM_NAIVE = 0, HM_CC1 = 1, HM_CC2 = 2, HM_CC2_AVG = 3, HM_CC1_RARY = 4 };   /* hm_compose heuristics */

/* ---------------------------------------------------------------- context */

/* Create a context on CUDA device `device`.  cuda_stream: a cudaStream_t to
 * issue all work on (borrowed, e.g. torch.cuda.current_stream().cuda_stream),
 * or NULL for a context-owned non-blocking stream.  *out receives the context. */
hm_status hm_create(hm_ctx **out, int device, void *cuda_stream);

/* Release every device buffer and the owned stream.  NULL is a no-op. */
void hm_destroy(hm_ctx *ctx);

/* Message for the last non-OK status on ctx (owned by ctx; "" if none). */
const char *hm_last_error(const hm_ctx *ctx);

/* Tuning knobs (results never depend on them):
 *   "bfs_words"   : 64-bit words per bit-parallel state row (8, 16, 32, 64 or 128; sources per batch =
 *                   64*words; 128 only for graphs without heavy rows); 0 (default) = automatic: 128 for
 *                   sparse graphs (average degree < 4) without heavy rows whose state exceeds 256 MB, else 64
 *   "bfs_heavy"   : degree above which a row goes to the MS-BFS heavy path (work items of 1024 arcs
 *                   claimed by whole CTAs); 0 = default: 256, or 64 on graphs of average degree < 8
 *   "bfs_blocks_per_sm" : CTAs per SM of the persistent MS-BFS kernel (1, or 0 / 2 = two)
 *   "bfs_gd"      : MS-BFS neighbour-row gathers in flight per lane (0 = default, 2, 4, 8)
 *   "bfs_prune"   : exact 2-core pruning of the largest component before the MS-BFS (hanging
 *                   trees restored by weights and re-rooting; results unchanged): 1 on, 0 off,
 *                   2 (default) on for V >= 4096
 *   "bfs_interleave": 1 (default) CTAs own interleaved light-path units, 0 contiguous ranges
 *   "bfs_fbar": 0 MS-BFS levels end in the cooperative grid barrier plus an any-change
 *              flag; 1 (default) one counter atomic per CTA carries both (arrival and "row changed")
 *   "bfs_hints"   : MS-BFS L2 eviction-priority bits (1 gathers evict_last, 2 own F_{d-2} evict_first,
 *                   4 F_d stores evict_last, 8 F_d stores evict_first; default 11)
 *   "cc_init"     : connected components: 4 (default) = 3 from V = 32768, else 2; 3 min-label hooking (atomicMin of the larger root
 *                   under the smaller) and pointer jumping, rounds until no hook changes, in one
 *                   cooperative launch; 2 sampled union-find (unite each vertex with its first 2
 *                   neighbours, then only rows outside the most frequent root unite over the rest);
 *                   0 union over every arc; 1 as 0 starting from parent = smallest neighbour
 *   "bfs_unit"    : rows per MS-BFS light-path work unit (32, 16, 8, 4 or 2; 0 = default: chosen from
 *                   the live rows per warp of the grid, 32 on C5-sized graphs)
 *   "bfs_team"    : lanes per state row in the MS-BFS light path (0 = default, 4, 8, 16, 32; <= words/2)
 *   "bfs_td"      : direction optimisation (north_star; the BFS of PAPER.md:209): a level runs top-down --
 *                   the frontier (rows changed at the previous level) marks its neighbours as candidates,
 *                   then only candidate rows pull -- when frontier rows * bfs_td <= the batch's rows, else
 *                   bottom-up over every row not yet complete; 0 = always bottom-up
 *   "bfs_push"    : direction optimisation, push form (the per-source top-down BFS step of PAPER.md:209 on the
 *                   batch's first, sparse levels): while the (row, source) pairs found at the previous level
 *                   number <= rows * bfs_push / 4, a level pushes each pair's source bit into its neighbours'
 *                   visited sets (atomic OR; a first set is a discovery at exactly this distance), then the
 *                   bit-parallel bottom-up levels take over; 0 = off; -1 (default) = automatic: 8 for graphs
 *                   run at 8192 sources per batch, else off.  Graphs without heavy rows, default kernel
 *                   shape.  Results are identical either way.
 *   "bfs_fuse"    : hm_closeness_multi: 0 one pass per graph, 1 one fused pass over the disjoint union,
 *                   2 (default) fused when sum of V <= 2^17 (graphs too small to fill the GPU alone), else
 *                   graphs known to run unpruned fused in groups of <= 2^20 vertices, the rest one pass each
 *   "bfs_count_rows": 1 runs the default MS-BFS kernels in a counting instantiation that fills hm_stats
 *                   bfs_gathers / bfs_own_reads (the row traffic; ~3 % slower), 0 (default) the timed ones
 *   "bfs_torder"  : pruned graphs: relabel the pruned core in order of hanging-tree size T so the MS-BFS weighs
 *                   128-source chunks by T x popc (0 never, 1 (default) graphs without rows above degree 256,
 *                   2 always)
 *   "topk_tiles"  : top-K lists (K <= 4096, n > 4096): 1 (default) one launch -- per-tile block-local radix
 *                   selects, then the last tile merges and sorts -- where the G = ceil(n / 8192) tiles' K
 *                   candidates fit one block (G * K <= 16384), 0 the cooperative 12-pass radix select
 *   "bfs_chg_smem": 1 stages the per-level change bitmaps in shared memory, 0 (default) reads them via L1
 *   "timing"      : 1 = record CUDA events around the MS-BFS kernel, 2 = also around every phase of
 *                   closeness / compose / top-K / aggregation (see hm_get_stats)
 *   "bfs_dbg"     : debug: bit 1 (value 2) = per-level counters and times (hm_debug_counts);
 *                   bits 8.. = the one level to profile in HM_MSBFS_PROF builds
 * Unknown name -> HM_EINVAL. */
hm_status hm_set_param(hm_ctx *ctx, const char *name, int64_t value);

/* --------------------------------------------------------------- graphs */

/* Load the l layers of a HoMLN (§1).  Vertices are 0..V-1 in every
 * layer.  edges[i] points to 2*m[i] int32 values (u0,v0,u1,v1,...), host or
 * device.  Undirected: either or both directions may be given; self-loops and
 * duplicates are dropped (count in dropped_out[i] if non-NULL, host array of l).
 * Builds one CSR per layer on the device (rows ascending).  Assigns graph ids
 * 0..l-1 in order; replaces any previously loaded HoMLN in ctx.
 * Errors: V <= 0 or l < 1 -> EINVAL; id outside [0,V) or 2*m[i] >= 2^31 -> ERANGE. */
hm_status hm_load_layers(hm_ctx *ctx, int32_t V, int32_t l, const int32_t *const *edges,
                         const int64_t *m, int64_t *dropped_out);

/* Shape and borrowed device views of graph g's CSR (row_ptr: V+1, col: 2m),
 * valid until g is freed.  Any out pointer may be NULL. */
hm_status hm_graph_info(hm_ctx *ctx, int32_t g, int32_t *V, int64_t *m_undirected,
                        const int32_t **d_row_ptr, const int32_t **d_col);

/* Copy graph g's CSR into caller buffers (host or device): row_ptr V+1, col 2m. */
hm_status hm_graph_csr(hm_ctx *ctx, int32_t g, int32_t *row_ptr, int32_t *col);

/* Boolean AND aggregation (PAPER.md:150 §3.1; :205 §4 ground truth step i):
 * an edge is in the result iff it is in every one of the r >= 2 distinct graphs
 * graph_ids[0..r-1] (host array).  Vertex set stays V.  *g_out receives the new
 * graph id (>= l).  Computed by a sorted-adjacency intersection kernel.
 * Errors: r < 2 or repeated id -> EINVAL; unknown id -> ESTATE. */
hm_status hm_and_aggregate(hm_ctx *ctx, const int32_t *graph_ids, int32_t r, int32_t *g_out);

/* Boolean OR aggregation (§3.1): edge in at least one graph. */
hm_status hm_or_aggregate(hm_ctx *ctx, const int32_t *graph_ids, int32_t r, int32_t *g_out);

/* Release an aggregated graph (ids >= l) and its cached results.  Layers -> ESTATE. */
hm_status hm_free_graph(hm_ctx *ctx, int32_t g);

/* ------------------------------------------------------------ analysis */

/* All-sources unweighted BFS closeness of graph g (§4; the
 * analysis function Psi of PAPER.md:121-122).  For every vertex v:
 *   dist_sum[v]  S(v) = sum of d(v,w) over vertices w reachable from v (uint64)
 *   reach[v]     k(v) = number of vertices reachable from v, v included
 *   closeness[v] Wasserman-Faust closeness as NetworkX computes it
 *                (PAPER.md:186, :209): ((k-1)/S) * ((k-1)/(V-1)) in binary64,
 *                0 when S == 0 or V <= 1; equals Eq. 1 when k == V
 *   pen_sum[v]   n-penalty sum sumDist(v) (§5.1): S + (V-k)*V
 * Also caches, for hm_compose / hm_topk_closeness / hm_cc_nodes: degrees, the
 * mean closeness mu = (correctly rounded sum of c) / V and the CC-node set
 * CH = {v : c(v) > mu}.  Any output pointer may be NULL; each
 * is host or device, length V.  Re-running on a graph recomputes.  Host round
 * trips (context-stream synchronisations) inside the call: one with pruning on
 * ("bfs_prune" 1, or 2 with V >= 4096), to decide whether the exact 2-core
 * pruning of the largest component pays; one when V * 8 * bfs_words * 3 bytes
 * exceed 256 MB, to size the frontier rows by the live rows. */
hm_status hm_closeness(hm_ctx *ctx, int32_t g, uint64_t *dist_sum, int32_t *reach,
                       double *closeness, uint64_t *pen_sum);

/* hm_closeness for n >= 1 distinct graphs: the graphs are independent problems
 * (the layers of a HoMLN, analysed "in parallel", plus any
 * aggregate).  Fused ("bfs_fuse" 1, or 2 = default when sum of V <= 2^17):
 * their all-sources BFS runs over the disjoint union in ONE pass and shares
 * every level step (no pruning, no host round trip); otherwise (default) the
 * graphs known not to be pruned (an earlier call's cached decision) are fused
 * in groups of <= 2^20 vertices and every other graph gets its own
 * hm_closeness pass.  Results are per graph, identical to n separate hm_closeness
 * calls either way, cached for hm_compose / hm_topk_closeness / hm_cc_nodes and
 * readable with hm_closeness_results.  graph_ids: host array.  Errors: n < 1 or
 * repeated id -> EINVAL; unknown id -> ESTATE; fused with n > 64 -> EINVAL;
 * fused with sum of V >= 2^26 -> ERANGE. */
hm_status hm_closeness_multi(hm_ctx *ctx, const int32_t *graph_ids, int32_t n);

/* Sharded Psi (source batches split over GPUs, one sum
 * reduction).  hm_closeness_partial runs the all-sources BFS of graph g for the
 * source batches i = shard, shard + nshards, ... only (the batch order is fixed by
 * the graph) and writes that shard's partial target-side sums, uint64[V] in
 * original vertex order, to S_partial (host or device).  The element-wise sum
 * over all nshards shards (e.g. an NCCL all-reduce) is the graph's
 * pre-finalisation sum vector, the same for every nshards (each batch
 * contributes once): S itself when pruning is off, else the pruned core's
 * weighted sums (peeled vertices 0).  Only that sum is meaningful, through
 * hm_closeness_combine.
 * hm_closeness_combine finalises graph g from that sum S_total (host or device,
 * uint64[V]): k, closeness, n-penalty sum, degrees, mean and CC nodes, cached
 * exactly as hm_closeness caches them (hm_closeness_results / hm_compose /
 * hm_topk_closeness then work unchanged).  Errors: nshards < 1 or shard outside
 * [0, nshards) or NULL buffer -> EINVAL; unknown graph -> ESTATE. */
hm_status hm_closeness_partial(hm_ctx *ctx, int32_t g, int32_t shard, int32_t nshards, uint64_t *S_partial);
hm_status hm_closeness_combine(hm_ctx *ctx, int32_t g, const uint64_t *S_total);

/* Copy the cached hm_closeness results of graph g (ESTATE if none); the same
 * four outputs as hm_closeness, each NULL-able, host or device, length V. */
hm_status hm_closeness_results(hm_ctx *ctx, int32_t g, uint64_t *dist_sum, int32_t *reach,
                               double *closeness, uint64_t *pen_sum);

/* CC nodes of graph g (needs hm_closeness(g) first, else ESTATE):
 * bitmap (ceil(V/32) uint32 words, bit v%32 of word v/32; host or device, may
 * be NULL), *count (may be NULL) and *mean = mu (host, may be NULL). */
hm_status hm_cc_nodes(hm_ctx *ctx, int32_t g, uint32_t *bitmap, int32_t *count, double *mean);

/* Degrees deg(v) = |NBD(v)| of graph g, V int32, host or device. */
hm_status hm_degrees(hm_ctx *ctx, int32_t g, int32_t *deg);

/* Ground-truth style ranking: the K vertices of largest
 * closeness, ties by lower id, in rank order.  1 <= K <= V.  ids_out: K int32,
 * host or device.  Needs hm_closeness(g) (ESTATE otherwise). */
hm_status hm_topk_closeness(hm_ctx *ctx, int32_t g, int32_t K, int32_t *ids_out);

/* -------------------------------------------------------- composition */

/* Composition Theta over r >= 2 distinct layer/graph ids (host array), each of
 * which must have had hm_closeness run (ESTATE otherwise).  Reads only the
 * cached per-graph results and the graphs' own adjacency (NBD), never the AND
 * aggregate (the decoupling contract).
 *   HM_CC2  (Alg. 1): est(v) = max_i pen_i(v); the K
 *           vertices of largest Eq. 1 score (V-1)/est, i.e. smallest (est, id);
 *           writes exactly K ids, *count_out = K.
 *   HM_CC1  (Eq. 2, Eq. 3; pseudocode :477-507): the paper
 *           defines CC1 for a PAIR of layers only, so r must be 2 (r > 2 ->
 *           HM_EINVAL).  Result set R, ranked by RN(est/mindeg) ascending then
 *           id; writes min(K, |R|) ids, *count_out = |R|.
 *   HM_CC1_RARY (explicit opt-in, reading Z12 of DESIGN.md §3): CC1 for any
 *           2 <= r <= 8 in the flat r-ary form -- mindeg = min_i deg_i,
 *           avgAND = max_i avg_i, I(u) = the intersection over all r layers
 *           of the candidate neighbourhoods.  Identical to HM_CC1 when r = 2.
 *   HM_NAIVE: intersection of the CC-node sets, ranked by id;
 *           writes min(K, |R|) ids, *count_out = |R|.
 *   HM_CC2_AVG ("above average" form of CC2): score(v) =
 *           (V-1)/est(v) (Eq. 1, binary64, 0 if est == 0); R = {v : score(v) >
 *           mean score}, the mean being the correctly rounded sum / V; ids
 *           ascending; writes min(K, |R|) ids, *count_out = |R|.
 * 1 <= K <= V.  ids_out host or device; count_out host or device (may be NULL).
 * With device ids_out AND (device or NULL) count_out the call never
 * synchronises the stream: ids_out receives K entries, those past |R| set to -1. */
hm_status hm_compose(hm_ctx *ctx, int32_t heuristic, const int32_t *layer_ids, int32_t r,
                     int32_t K, int32_t *ids_out, int32_t *count_out);

/* Accuracy of an estimated CC-node list against the ground truth
 * (§6: precision, recall, F1; Jaccard similarity): est_ids[n_est]
 * and gt_ids[n_gt] are vertex ids (host or device; duplicates count once; n = 0
 * allowed, the pointer may then be NULL).  out (host, 7 doubles) receives
 * Jaccard |A∩B|/|A∪B| (1 if both empty), precision |A∩B|/|A| (1 if both empty,
 * 0 if only A is empty), recall |A∩B|/|B| (1 if B empty), F1 2PR/(P+R) (0 if
 * P+R == 0), then |A|, |B|, |A∩B|.  Each ratio is one IEEE binary64 division.
 * Errors: V <= 0 or n < 0 -> EINVAL; an id outside [0, V) -> ERANGE. */
hm_status hm_set_metrics(hm_ctx *ctx, int32_t V, const int32_t *est_ids, int64_t n_est,
                         const int32_t *gt_ids, int64_t n_gt, double *out);

/* Exact mean of non-negative doubles, the reducer behind every "average" of
 * the method: the CC-node threshold "higher than the average",
 * the layer averages of Eq. 3 and the CC2
 * above-average threshold.  Reading Z6:
 * mean = RN(exact sum of the selected x[i]) / count, one IEEE division, i.e.
 * Python's math.fsum(x) / count, independent of summation order.  x: n
 * doubles, host or device; mask: NULL (all selected) or n bytes (nonzero =
 * selected), host or device; *mean_out (host) = 0.0 when nothing is selected;
 * *count_out (host, may be NULL) = the number selected.  Exposed so the tests
 * can pin the device reducer on adversarial arrays.  Errors: n < 0 or NULL
 * x (n > 0) or NULL mean_out -> EINVAL; a selected value negative, inf or nan
 * -> EINVAL (outside the contract; nothing written). */
hm_status hm_exact_mean(hm_ctx *ctx, const double *x, int64_t n, const uint8_t *mask, double *mean_out,
                        int32_t *count_out);

/* ------------------------------------------------------------ utilities */

/* Wait for all work issued on the context stream. */
hm_status hm_sync(hm_ctx *ctx);

/* Counters since the last reset (reset=1 zeroes them after reading):
 *   launches       number of this library's kernel launches
 *   bfs_launches   launches of the persistent MS-BFS kernel
 *   bfs_ms         summed CUDA-event time of those launches (needs param timing=1)
 *   bfs_levels     BFS levels executed (sum over batches)
 *   bfs_batches    source batches executed */
typedef struct {
    int64_t launches;
    int64_t bfs_launches;
    double bfs_ms;
    int64_t bfs_levels;
    int64_t bfs_batches;
    double bfs_model_bytes;   /* SURVEY §8(d) dense-level bytes of the MS-BFS launches, summed per batch:
                                 levels * (4 (rows + 1) + 4 arcs + 2 * 8 W * rows) over the batch's
                                 BFS rows and arcs (the pruned core when 2-core pruning applies); 2 state
                                 rows per row and level: the own visited set read and the new one written */
    int64_t bfs_row_commits;  /* rows changed, summed over levels and batches (each one own-row read and one
                                 8 W-byte row write: the compulsory state traffic); needs bfs_fbar = 1 */
    double bfs_csr_bytes;     /* CSR bytes of the same model: levels * (4 (rows + 1) + 4 arcs) per batch */
    int64_t bfs_td_levels;    /* levels run top-down (frontier-driven candidate rows, parameter bfs_td) */
    double bfs_state_bytes;   /* compulsory state bytes: 2 * 8 W per row commit (own visited set read, new one
                                 written), summed over levels and batches; needs bfs_fbar = 1 */
    int64_t host_syncs;       /* host round trips (stream synchronisations) made inside library calls: a
                                 sequence of calls with none can be captured in a CUDA graph */
    double phase_ms[10];      /* with timing = 2: CUDA-event time per phase -- [0] components, [1] pruning
                                 decision, [2] relabel, [3] MS-BFS setup, [4] MS-BFS, [5] finalize + mean +
                                 CC nodes, [6] compose, [7] top-K, [8] aggregation, [9] other */
    int64_t bfs_gathers;      /* neighbour rows gathered (one 8 W-byte row read each), summed over levels and
                                 batches: with bfs_own_reads and bfs_row_commits the MS-BFS's row traffic
                                 through L2, 8 W (gathers + own reads + commits) bytes; counted only with
                                 "bfs_count_rows" 1 (default kernels), else 0 */
    int64_t bfs_own_reads;    /* own visited-set rows read (rows with a state and a changed neighbour) */
} hm_stats;
hm_status hm_get_stats(hm_ctx *ctx, hm_stats *out, int reset);

/* Debug: copy the counters of the last MS-BFS launch made with
 * hm_set_param("bfs_dbg", 2): out[d] = source batches that ran level d,
 * out[4096+d] = nanoseconds spent in level d (summed over batches),
 * out[12288+d] = rows changed at level d (summed over batches), and in
 * HM_MSBFS_PROF builds out[8192..8204] = per-phase warp cycles and counts.
 * n <= 335872 uint64 (host).  ESTATE if no such launch happened. */
hm_status hm_debug_counts(hm_ctx *ctx, uint64_t *out, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* HM_H */
