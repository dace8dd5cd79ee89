// Shared internals of libhm (B200 / sm_100a).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <utility>
#include <vector>
#include <map>
#include <stdexcept>

#include "../../include/hm.h"

namespace hm {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    hm_status code;
    Error(hm_status c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define HM_CUDA(call)                                                                  \
    do {                                                                               \
        cudaError_t _e = (call);                                                       \
        if (_e != cudaSuccess)                                                         \
            throw ::hm::Error(_e == cudaErrorMemoryAllocation ? HM_ENOMEM : HM_ECUDA,  \
                              std::string(#call) + ": " + cudaGetErrorString(_e));     \
    } while (0)

#define HM_REQUIRE(cond, code, msg)                 \
    do {                                            \
        if (!(cond)) throw ::hm::Error(code, msg);  \
    } while (0)

// ------------------------------------------------------- device buffers
// Stream-ordered allocation (cudaMallocAsync) owned by RAII handles.
struct Buf {
    void *p = nullptr;
    size_t bytes = 0;
    cudaStream_t s = nullptr;
    Buf() = default;
    Buf(size_t n, cudaStream_t st) { alloc(n, st); }
    Buf(const Buf &) = delete;
    Buf &operator=(const Buf &) = delete;
    Buf(Buf &&o) noexcept { *this = std::move(o); }
    Buf &operator=(Buf &&o) noexcept {
        if (this != &o) {
            release();
            p = o.p; bytes = o.bytes; s = o.s;
            o.p = nullptr; o.bytes = 0;
        }
        return *this;
    }
    ~Buf() { release(); }
    void alloc(size_t n, cudaStream_t st) {
        release();
        s = st;
        bytes = n;
        if (n) HM_CUDA(cudaMallocAsync(&p, n, st));
    }
    // grow-only scratch
    void ensure(size_t n, cudaStream_t st) {
        if (n > bytes || p == nullptr) alloc(n < 64 ? 64 : n, st);
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        bytes = 0;
    }
    template <class T> T *as() const { return static_cast<T *>(p); }
};

// The host-side outcome of the pruning round trip (prune.cu): a pure function of the graph, so it is
// kept with the graph (layers: for their lifetime; AND aggregates: keyed by their layer set until
// the next hm_load_layers) and later closeness calls skip the round trip.  All device work
// (peeling, relabelling, the BFS) still runs on every call.
struct PruneDecision {
    bool valid = false;
    bool active = false;
    int P = -1, R = 0, peeled = 0;
    int maxdeg = 0, nonisolated = 0;
    int64_t arcs = 0;
};

// ------------------------------------------------------- per-graph state
struct Graph {
    bool alive = false;
    bool is_layer = false;
    int32_t V = 0;
    int64_t nnz = 0;          // arcs = 2 m (an upper bound while !nnz_exact: AND aggregates, whose exact
                              // count stays on the device in row_ptr[V] until exact_nnz() reads it)
    bool nnz_exact = true;
    Buf row_ptr, col;         // CSR, rows ascending
    // cached Psi results (valid when has_results)
    bool has_results = false;
    Buf S, k, c, pen, deg, ch;   // uint64, int32, double, uint64, int32, uint32 bitmap
    double mu = 0.0;
    int32_t ch_count = 0;
    PruneDecision pdec;              // cached pruning decision (see PruneDecision)
    std::vector<int32_t> and_key;    // AND aggregates: the sorted layer ids (decision cache key)
};

struct Params {
    int bfs_words = 0;         // 0 = auto: 64 words (4096 sources per batch), 128 for sparse graphs without heavy rows
    int bfs_heavy = 0;         // MS-BFS heavy-row degree threshold (0 = auto: 256, or 64 below average degree 8)
    int bfs_blocks_per_sm = 0;
    int bfs_chg_smem = 0;      // 1: stage the change bitmaps in shared memory each level; 0: read them via L1
    int bfs_prune = 2;         // exact 2-core pruning before the MS-BFS: 1 on, 0 off, 2 on from V = 4096
    int bfs_interleave = 1;    // MS-BFS: CTAs own interleaved units (1) or contiguous ranges (0)
    int bfs_fbar = 1;          // MS-BFS level barrier with the any-change flag folded in
    int bfs_hints = 11;        // MS-BFS L2 eviction-priority bits (msbfs.cuh BfsArgs::hints)
    int cc_init = 4;           // components: 0 union over all arcs, 1 from parent = smallest neighbour, 2 sampled
                               // (Afforest), 3 min-label hooking + pointer jumping in one cooperative launch,
                               // 4 (default) = 3 from V = 32768, else 2
    int bfs_unit = 0;          // MS-BFS light-path rows per work unit (0 = auto by rows per warp; 32 ... 2)
    int bfs_gd = 0;            // MS-BFS gathers in flight per lane (0 = default)
    int bfs_team = 0;          // MS-BFS lanes per light state row (0 = default)      // stage the change bitmaps in shared memory each level
    int bfs_fuse = 2;          // hm_closeness_multi: 0 one pass per graph, 1 one fused pass, 2 (auto) fused when
                               // sum of V <= 2^17 (small graphs that cannot fill the GPU alone)
    int bfs_count_rows = 0;    // MS-BFS: 1 = counting instantiation (hm_stats bfs_gathers / bfs_own_reads)
    int bfs_torder = 1;        // pruned core rows in T order: 0 never, 1 graphs without hub rows, 2 always
    int topk_tiles = 1;        // top-K: 1 two-phase tile select (one launch) where it fits, 0 cooperative radix select
    int bfs_td = 0;            // direction switch: top-down levels when frontier * bfs_td <= rows (0 = off)
    int bfs_push = -1;         // top-down push phase: first levels of a batch push (row, source) pairs while the
                               // pairs number <= rows * bfs_push / 4 (0 = off; -1 = automatic: 8 at 8192 sources
                               // per batch, else off; lean default kernels only)
    int timing = 0;
    int bfs_dbg = 0;
};

struct Stats {
    int64_t launches = 0;
    int64_t host_syncs = 0;   // host round trips (stream synchronisations) inside library calls
    int64_t bfs_launches = 0;
    double bfs_ms = 0;
};

}  // namespace hm

struct hm_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    std::vector<hm::Graph> graphs;
    std::map<std::vector<int32_t>, hm::PruneDecision> and_pdec;   // AND graphs' pruning decisions by layer set
    int32_t n_layers = 0;
    hm::Params params;
    hm::Stats stats;
    hm::Buf dbgc;             // debug counters of the last MS-BFS launch (bfs_dbg & 2)
    hm::Buf dstats;           // device counters: [0] levels, [1] batches (uint64)
    int num_sms = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;   // MS-BFS launch events (timing=1)
    struct PhaseEv { int id; cudaEvent_t e0, e1; };
    std::vector<PhaseEv> phase_pending;                          // per-phase events (timing=2)
    double phase_ms[10] = {0};
};

namespace hm {

inline void count_launch(hm_ctx *ctx, int n = 1) { ctx->stats.launches += n; }

// per-phase CUDA-event timing (param timing >= 2; resolved in hm_get_stats, no synchronisation here)
enum { PH_CC = 0, PH_PRUNE, PH_RELABEL, PH_BFS_SETUP, PH_BFS, PH_FINALIZE, PH_COMPOSE, PH_TOPK, PH_AGGREGATE, PH_OTHER };
inline cudaEvent_t phase_begin(hm_ctx *ctx) {
    if (ctx->params.timing < 2) return nullptr;
    cudaEvent_t e;
    HM_CUDA(cudaEventCreate(&e));
    HM_CUDA(cudaEventRecord(e, ctx->stream));
    return e;
}
inline void phase_end(hm_ctx *ctx, int id, cudaEvent_t &e0) {
    if (!e0) return;
    cudaEvent_t e1;
    HM_CUDA(cudaEventCreate(&e1));
    HM_CUDA(cudaEventRecord(e1, ctx->stream));
    ctx->phase_pending.push_back({id, e0, e1});
    e0 = nullptr;
}

// a host round trip inside a library call (counted: a step without any can be captured in a CUDA graph)
inline void host_sync(hm_ctx *ctx) {
    ++ctx->stats.host_syncs;
    HM_CUDA(cudaStreamSynchronize(ctx->stream));
}

// Row of arc j of a CSR (row_ptr[0..V], V >= 1, 0 <= j < row_ptr[V]): the largest u with
// row_ptr[u] <= j.  Arc-parallel kernels use it so that a hub row is spread over many threads
// instead of serialising one warp (R-MAT hubs of 5-8 K arcs).
__device__ __forceinline__ int csr_row_of(const int32_t *__restrict__ row_ptr, int V, int64_t j) {
    int lo = 0, hi = V - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (row_ptr[mid] <= j) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

inline void check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(HM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

inline unsigned grid_for(int64_t n, int threads, int64_t cap = 148LL * 32) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (unsigned)b;
}

Graph &graph(hm_ctx *ctx, int32_t g);                 // throws ESTATE
int64_t exact_nnz(hm_ctx *ctx, Graph &G);             // reads row_ptr[V] (one host round trip) if not known
bool is_device_ptr(const void *p);
void copy_out(hm_ctx *ctx, void *dst, const void *dsrc, size_t bytes);  // host or device dst

// module entry points (each file)
void build_csr(hm_ctx *ctx, int32_t V, const int32_t *edges_host_or_dev, int64_t m, Graph &G,
               int64_t *dropped);
void and_or_aggregate(hm_ctx *ctx, const std::vector<Graph *> &in, bool is_and, Graph &out);
void closeness(hm_ctx *ctx, Graph &G);
void closeness_multi(hm_ctx *ctx, const std::vector<Graph *> &gs, int shard = 0, int nshards = 1,
                     uint64_t *d_S_partial = nullptr, const uint64_t *d_S_total = nullptr,
                     bool decide_only = false);
void closeness_partial(hm_ctx *ctx, Graph &G, int shard, int nshards, uint64_t *d_S_out);
// hm_closeness_multi: one fused pass or one pass per graph (Params::bfs_fuse)
void closeness_group(hm_ctx *ctx, const std::vector<Graph *> &gs);

// exact 2-core pruning of the largest component (prune.cu)
struct Prune {
    bool active = false;
    int P = -1, R = 0, peeled = 0;
    bool shape_known = false;         // the decision round trip also read: max degree, vertices with an
    int maxdeg = 0, nonisolated = 0;  // edge, arcs (for the host's batch-width / heavy-path choices)
    int64_t arcs = 0;
    Buf rem, par, tsz, tD, degl, lsize, Cc, scal;   // per vertex / per component root
};
bool prune_component(hm_ctx *ctx, const int32_t *rp, const int32_t *col, const int32_t *label, const int32_t *csize,
                     int V, Prune &pr, PruneDecision *dec);
void prune_finish(hm_ctx *ctx, Prune &pr, const int32_t *label, const int32_t *csize, uint64_t *S_orig, int V);
void closeness_combine(hm_ctx *ctx, Graph &G, const uint64_t *d_S_total);
// exact (correctly rounded) sum of masked non-negative doubles, then mean = sum / count;
// result written to device double *d_mean (count taken from mask popcount or n)
void exact_mean(hm_ctx *ctx, const double *d_x, int64_t n, const uint8_t *d_mask_or_null,
                double *d_mean_out, int32_t *d_count_out, int32_t *d_bad_out = nullptr);
void degrees(hm_ctx *ctx, const Graph &G, int32_t *d_deg);
// keys ordering closeness descending: ~bits(c) (c >= 0, so bit patterns are monotone)
void closeness_desc_keys(hm_ctx *ctx, const double *d_c, int32_t V, uint64_t *d_keys);
void topk(hm_ctx *ctx, const uint64_t *d_keys, int32_t n, int32_t K, int32_t *d_ids_out);
void compose(hm_ctx *ctx, int heuristic, const std::vector<Graph *> &gs, int32_t K,
             int32_t *ids_out, int32_t *count_out);
// Jaccard, precision, recall, F1, |est|, |gt|, |est ∩ gt| of two id lists (device)
void set_metrics(hm_ctx *ctx, int32_t V, const int32_t *d_est, int64_t n_est, const int32_t *d_gt,
                 int64_t n_gt, double *d_out7, int32_t *d_bad);

}  // namespace hm
