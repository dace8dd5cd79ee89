// C ABI entry points (include/hm.h).  Argument checking, graph registry,
// host/device output handling; every computation is delegated to the kernels
// in graph.cu, closeness.cu, msbfs.cu, exactsum.cu, topk.cu and compose.cu.
#include <cuda_runtime.h>
#include <string.h>
#include <algorithm>
#include <set>

#include "common.cuh"

namespace hm {

Graph &graph(hm_ctx *ctx, int32_t g) {
    HM_REQUIRE(g >= 0 && g < (int32_t)ctx->graphs.size() && ctx->graphs[g].alive, HM_ESTATE,
               "unknown or freed graph id " + std::to_string(g));
    return ctx->graphs[g];
}

bool is_device_ptr(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

void copy_out(hm_ctx *ctx, void *dst, const void *dsrc, size_t bytes) {
    if (!dst || !bytes) return;
    if (is_device_ptr(dst)) {
        HM_CUDA(cudaMemcpyAsync(dst, dsrc, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
        HM_CUDA(cudaMemcpyAsync(dst, dsrc, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        host_sync(ctx);
    }
}

}  // namespace hm

using namespace hm;

#define HM_API_BEGIN(ctx)                                   \
    if (!(ctx)) return HM_EINVAL;                           \
    try {                                                   \
        HM_CUDA(cudaSetDevice((ctx)->device));
#define HM_API_END(ctx)                                     \
        (ctx)->err.clear();                                 \
        return HM_OK;                                       \
    } catch (const hm::Error &e) {                          \
        (ctx)->err = e.what();                              \
        return e.code;                                      \
    } catch (const std::exception &e) {                    \
        (ctx)->err = e.what();                              \
        return HM_ECUDA;                                    \
    }

extern "C" {

hm_status hm_create(hm_ctx **out, int device, void *cuda_stream) {
    if (!out) return HM_EINVAL;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        return HM_ECUDA;
    }
    hm_ctx *ctx = new hm_ctx();
    ctx->device = device;
    try {
        HM_CUDA(cudaSetDevice(device));
        if (cuda_stream) {
            ctx->stream = (cudaStream_t)cuda_stream;
        } else {
            HM_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
            ctx->own_stream = true;
        }
        HM_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
        int coop = 0;
        HM_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
        HM_REQUIRE(coop, HM_ECUDA, "device lacks cooperative launch");
        // keep freed stream-ordered memory in the pool (no release at sync points)
        cudaMemPool_t pool;
        HM_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        HM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        HM_CUDA(cudaEventCreate(&ctx->ev0));
        HM_CUDA(cudaEventCreate(&ctx->ev1));
        ctx->dstats.alloc(128, ctx->stream);
        HM_CUDA(cudaMemsetAsync(ctx->dstats.p, 0, 128, ctx->stream));
        HM_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (const hm::Error &) {
        hm_destroy(ctx);
        return HM_ECUDA;
    }
    *out = ctx;
    return HM_OK;
}

void hm_destroy(hm_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    ctx->graphs.clear();
    ctx->dstats.release();
    ctx->dbgc.release();
    for (auto &pe : ctx->pending) {
        cudaEventDestroy(pe.first);
        cudaEventDestroy(pe.second);
    }
    for (auto &pe : ctx->phase_pending) {
        cudaEventDestroy(pe.e0);
        cudaEventDestroy(pe.e1);
    }
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char *hm_last_error(const hm_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

hm_status hm_set_param(hm_ctx *ctx, const char *name, int64_t value) {
    HM_API_BEGIN(ctx)
    HM_REQUIRE(name, HM_EINVAL, "null name");
    const std::string n(name);
    if (n == "bfs_words") {
        HM_REQUIRE(value == 0 || value == 8 || value == 16 || value == 32 || value == 64 || value == 128, HM_EINVAL,
                   "bfs_words must be 0 (auto), 8, 16, 32, 64 or 128 (128: graphs without heavy rows)");
        ctx->params.bfs_words = (int)value;
    } else if (n == "bfs_heavy") {
        HM_REQUIRE(value >= 0, HM_EINVAL, "bfs_heavy must be >= 0 (0 = automatic)");
        ctx->params.bfs_heavy = (int)value;
    } else if (n == "bfs_blocks_per_sm") {
        HM_REQUIRE(value >= 0 && value <= 2, HM_EINVAL, "bfs_blocks_per_sm must be 0 (= 2), 1 or 2");
        ctx->params.bfs_blocks_per_sm = (int)value;
    } else if (n == "bfs_prune") {
        HM_REQUIRE(value >= 0 && value <= 2, HM_EINVAL, "bfs_prune must be 0, 1 or 2 (auto)");
        ctx->params.bfs_prune = (int)value;
    } else if (n == "bfs_count_rows") {
        ctx->params.bfs_count_rows = value ? 1 : 0;
    } else if (n == "bfs_torder") {
        HM_REQUIRE(value >= 0 && value <= 2, HM_EINVAL, "bfs_torder must be 0, 1 or 2");
        ctx->params.bfs_torder = (int)value;
    } else if (n == "topk_tiles") {
        HM_REQUIRE(value == 0 || value == 1 || value == 1024 || value == 2048 || value == 4096 || value == 8192,
                   HM_EINVAL, "topk_tiles must be 0, 1 (default tile), 1024, 2048, 4096 or 8192");
        ctx->params.topk_tiles = (int)value;
    } else if (n == "bfs_fuse") {
        HM_REQUIRE(value >= 0 && value <= 2, HM_EINVAL, "bfs_fuse must be 0, 1 or 2 (auto)");
        ctx->params.bfs_fuse = (int)value;
    } else if (n == "cc_init") {
        HM_REQUIRE(value >= 0 && value <= 4, HM_EINVAL, "cc_init must be 0, 1, 2, 3 or 4 (auto)");
        ctx->params.cc_init = (int)value;
    } else if (n == "bfs_fbar") {
        ctx->params.bfs_fbar = value ? 1 : 0;
    } else if (n == "bfs_interleave") {
        ctx->params.bfs_interleave = value ? 1 : 0;
    } else if (n == "bfs_hints") {
        HM_REQUIRE(value >= 0 && value <= 31, HM_EINVAL, "bfs_hints must be in [0, 31]");
        ctx->params.bfs_hints = (int)value;
    } else if (n == "bfs_unit") {
        HM_REQUIRE(value == 0 || value == 2 || value == 4 || value == 8 || value == 16 || value == 32, HM_EINVAL,
                   "bfs_unit must be 0 (auto), 2, 4, 8, 16 or 32");
        ctx->params.bfs_unit = (int)value;
    } else if (n == "bfs_gd") {
        HM_REQUIRE(value == 0 || value == 2 || value == 4 || value == 8, HM_EINVAL, "bfs_gd must be 0, 2, 4 or 8");
        ctx->params.bfs_gd = (int)value;
    } else if (n == "bfs_team") {
        HM_REQUIRE(value == 0 || value == 4 || value == 8 || value == 16 || value == 32, HM_EINVAL,
                   "bfs_team must be 0 (default), 4, 8, 16 or 32 (and at most words/2)");
        ctx->params.bfs_team = (int)value;
    } else if (n == "bfs_push") {
        HM_REQUIRE(value >= -1 && value <= 4096, HM_EINVAL, "bfs_push must be in [-1, 4096]");
        ctx->params.bfs_push = (int)value;
    } else if (n == "bfs_td") {
        HM_REQUIRE(value >= 0 && value <= (1 << 20), HM_EINVAL, "bfs_td must be in [0, 2^20]");
        ctx->params.bfs_td = (int)value;
    } else if (n == "bfs_chg_smem") {
        ctx->params.bfs_chg_smem = value ? 1 : 0;
    } else if (n == "bfs_dbg") {
        ctx->params.bfs_dbg = (int)value;
    } else if (n == "timing") {
        HM_REQUIRE(value >= 0 && value <= 2, HM_EINVAL, "timing must be 0, 1 or 2");
        ctx->params.timing = (int)value;
    } else {
        throw Error(HM_EINVAL, "unknown parameter " + n);
    }
    HM_API_END(ctx)
}

hm_status hm_load_layers(hm_ctx *ctx, int32_t V, int32_t l, const int32_t *const *edges, const int64_t *m,
                         int64_t *dropped_out) {
    HM_API_BEGIN(ctx)
    HM_REQUIRE(V > 0 && l >= 1, HM_EINVAL, "need V > 0 and l >= 1");
    HM_REQUIRE(edges && m, HM_EINVAL, "null edges / m");
    for (int i = 0; i < l; ++i) {
        HM_REQUIRE(m[i] >= 0, HM_EINVAL, "negative edge count");
        HM_REQUIRE(m[i] == 0 || edges[i], HM_EINVAL, "null edge array");
        HM_REQUIRE(2 * m[i] < (int64_t)INT32_MAX, HM_ERANGE, "2*m >= 2^31 arcs does not fit an int32 CSR");
    }
    std::vector<Graph> gs(l);
    std::vector<int64_t> dropped(l, 0);
    for (int i = 0; i < l; ++i) {
        build_csr(ctx, V, edges[i], m[i], gs[i], &dropped[i]);
        gs[i].alive = true;
        gs[i].is_layer = true;
    }
    HM_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->graphs = std::move(gs);
    ctx->n_layers = l;
    ctx->and_pdec.clear();                 // decisions of AND aggregates of the previous layers
    if (dropped_out)
        for (int i = 0; i < l; ++i) dropped_out[i] = dropped[i];
    HM_API_END(ctx)
}

hm_status hm_graph_info(hm_ctx *ctx, int32_t g, int32_t *V, int64_t *m_undirected, const int32_t **d_row_ptr,
                        const int32_t **d_col) {
    HM_API_BEGIN(ctx)
    Graph &G = graph(ctx, g);
    if (V) *V = G.V;
    if (m_undirected) *m_undirected = exact_nnz(ctx, G) / 2;
    if (d_row_ptr) *d_row_ptr = G.row_ptr.as<int32_t>();
    if (d_col) *d_col = G.col.as<int32_t>();
    HM_API_END(ctx)
}

hm_status hm_graph_csr(hm_ctx *ctx, int32_t g, int32_t *row_ptr, int32_t *col) {
    HM_API_BEGIN(ctx)
    Graph &G = graph(ctx, g);
    copy_out(ctx, row_ptr, G.row_ptr.p, (size_t)(G.V + 1) * 4);
    copy_out(ctx, col, G.col.p, (size_t)exact_nnz(ctx, G) * 4);
    HM_API_END(ctx)
}

static hm_status aggregate(hm_ctx *ctx, const int32_t *ids, int32_t r, int32_t *g_out, bool is_and) {
    HM_API_BEGIN(ctx)
    HM_REQUIRE(ids && g_out, HM_EINVAL, "null argument");
    HM_REQUIRE(r >= 2, HM_EINVAL, "aggregation needs r >= 2");
    HM_REQUIRE(r <= 8, HM_EINVAL, "aggregation supports r <= 8");
    std::set<int32_t> seen(ids, ids + r);
    HM_REQUIRE((int32_t)seen.size() == r, HM_EINVAL, "repeated graph id");
    std::vector<Graph *> in;
    for (int i = 0; i < r; ++i) in.push_back(&graph(ctx, ids[i]));
    for (int i = 1; i < r; ++i) HM_REQUIRE(in[i]->V == in[0]->V, HM_EINVAL, "graphs differ in V");
    Graph out;
    cudaEvent_t ph = phase_begin(ctx);
    and_or_aggregate(ctx, in, is_and, out);
    phase_end(ctx, PH_AGGREGATE, ph);
    if (is_and) {   // the aggregate is a function of its layer set: the key of its cached decisions
        bool layers_only = true;
        for (int i = 0; i < r; ++i) layers_only = layers_only && ids[i] < ctx->n_layers;
        if (layers_only) {
            out.and_key.assign(ids, ids + r);
            std::sort(out.and_key.begin(), out.and_key.end());
        }
    }
    // reuse a freed slot, else append (pointers in `in` are not used after this)
    int32_t slot = -1;
    for (int32_t i = ctx->n_layers; i < (int32_t)ctx->graphs.size(); ++i)
        if (!ctx->graphs[i].alive) { slot = i; break; }
    if (slot < 0) {
        ctx->graphs.emplace_back();
        slot = (int32_t)ctx->graphs.size() - 1;
    }
    ctx->graphs[slot] = std::move(out);
    *g_out = slot;
    HM_API_END(ctx)
}

hm_status hm_and_aggregate(hm_ctx *ctx, const int32_t *graph_ids, int32_t r, int32_t *g_out) {
    return aggregate(ctx, graph_ids, r, g_out, true);
}

hm_status hm_or_aggregate(hm_ctx *ctx, const int32_t *graph_ids, int32_t r, int32_t *g_out) {
    return aggregate(ctx, graph_ids, r, g_out, false);
}

hm_status hm_free_graph(hm_ctx *ctx, int32_t g) {
    HM_API_BEGIN(ctx)
    Graph &G = graph(ctx, g);
    HM_REQUIRE(!G.is_layer, HM_ESTATE, "layers cannot be freed individually");
    G = Graph();
    HM_API_END(ctx)
}

hm_status hm_closeness(hm_ctx *ctx, int32_t g, uint64_t *dist_sum, int32_t *reach, double *closeness_out,
                       uint64_t *pen_sum) {
    HM_API_BEGIN(ctx)
    Graph &G = graph(ctx, g);
    closeness(ctx, G);
    const size_t V = (size_t)G.V;
    copy_out(ctx, dist_sum, G.S.p, V * 8);
    copy_out(ctx, reach, G.k.p, V * 4);
    copy_out(ctx, closeness_out, G.c.p, V * 8);
    copy_out(ctx, pen_sum, G.pen.p, V * 8);
    HM_API_END(ctx)
}

hm_status hm_closeness_multi(hm_ctx *ctx, const int32_t *graph_ids, int32_t n) {
    HM_API_BEGIN(ctx)
    HM_REQUIRE(graph_ids && n >= 1, HM_EINVAL, "need n >= 1 graph ids");
    std::set<int32_t> seen(graph_ids, graph_ids + n);
    HM_REQUIRE((int32_t)seen.size() == n, HM_EINVAL, "repeated graph id");
    std::vector<Graph *> gs;
    for (int i = 0; i < n; ++i) gs.push_back(&graph(ctx, graph_ids[i]));
    closeness_group(ctx, gs);
    HM_API_END(ctx)
}

hm_status hm_closeness_partial(hm_ctx *ctx, int32_t g, int32_t shard, int32_t nshards, uint64_t *S_partial) {
    HM_API_BEGIN(ctx)
    HM_REQUIRE(S_partial, HM_EINVAL, "null S_partial");
    HM_REQUIRE(nshards >= 1 && shard >= 0 && shard < nshards, HM_EINVAL, "need 0 <= shard < nshards");
    Graph &G = graph(ctx, g);
    const size_t V = (size_t)G.V;
    if (is_device_ptr(S_partial)) {
        closeness_partial(ctx, G, shard, nshards, S_partial);
    } else {
        Buf tmp(V * 8, ctx->stream);
        closeness_partial(ctx, G, shard, nshards, tmp.as<uint64_t>());
        copy_out(ctx, S_partial, tmp.p, V * 8);
    }
    HM_API_END(ctx)
}

hm_status hm_closeness_combine(hm_ctx *ctx, int32_t g, const uint64_t *S_total) {
    HM_API_BEGIN(ctx)
    HM_REQUIRE(S_total, HM_EINVAL, "null S_total");
    Graph &G = graph(ctx, g);
    const size_t V = (size_t)G.V;
    if (is_device_ptr(S_total)) {
        closeness_combine(ctx, G, S_total);
    } else {
        Buf tmp(V * 8, ctx->stream);
        HM_CUDA(cudaMemcpyAsync(tmp.p, S_total, V * 8, cudaMemcpyHostToDevice, ctx->stream));
        closeness_combine(ctx, G, tmp.as<uint64_t>());
        host_sync(ctx);   // the host buffer may be reused on return
    }
    HM_API_END(ctx)
}

hm_status hm_closeness_results(hm_ctx *ctx, int32_t g, uint64_t *dist_sum, int32_t *reach, double *closeness_out,
                               uint64_t *pen_sum) {
    HM_API_BEGIN(ctx)
    Graph &G = graph(ctx, g);
    HM_REQUIRE(G.has_results, HM_ESTATE, "hm_closeness_results before hm_closeness");
    const size_t V = (size_t)G.V;
    copy_out(ctx, dist_sum, G.S.p, V * 8);
    copy_out(ctx, reach, G.k.p, V * 4);
    copy_out(ctx, closeness_out, G.c.p, V * 8);
    copy_out(ctx, pen_sum, G.pen.p, V * 8);
    HM_API_END(ctx)
}

hm_status hm_cc_nodes(hm_ctx *ctx, int32_t g, uint32_t *bitmap, int32_t *count, double *mean) {
    HM_API_BEGIN(ctx)
    Graph &G = graph(ctx, g);
    HM_REQUIRE(G.has_results, HM_ESTATE, "hm_cc_nodes before hm_closeness");
    const size_t nbw = (size_t)(G.V + 31) / 32;
    copy_out(ctx, bitmap, G.ch.p, nbw * 4);
    const char *base = G.ch.as<char>() + ((nbw * 4 + 7) / 8) * 8;
    struct { double mu; int32_t cnt; int32_t pad; } h;
    HM_CUDA(cudaMemcpyAsync(&h, base, 12, cudaMemcpyDeviceToHost, ctx->stream));
    host_sync(ctx);
    if (count) *count = h.cnt;
    if (mean) *mean = h.mu;
    HM_API_END(ctx)
}

hm_status hm_degrees(hm_ctx *ctx, int32_t g, int32_t *deg) {
    HM_API_BEGIN(ctx)
    Graph &G = graph(ctx, g);
    HM_REQUIRE(deg, HM_EINVAL, "null deg");
    Buf tmp((size_t)G.V * 4, ctx->stream);
    degrees(ctx, G, tmp.as<int32_t>());
    copy_out(ctx, deg, tmp.p, (size_t)G.V * 4);
    HM_API_END(ctx)
}

hm_status hm_topk_closeness(hm_ctx *ctx, int32_t g, int32_t K, int32_t *ids_out) {
    HM_API_BEGIN(ctx)
    Graph &G = graph(ctx, g);
    HM_REQUIRE(G.has_results, HM_ESTATE, "hm_topk_closeness before hm_closeness");
    HM_REQUIRE(K >= 1 && K <= G.V, HM_EINVAL, "K must be in [1, V]");
    HM_REQUIRE(ids_out, HM_EINVAL, "null ids_out");
    Buf keys((size_t)G.V * 8, ctx->stream), ids((size_t)K * 4, ctx->stream);
    cudaEvent_t ph = phase_begin(ctx);
    closeness_desc_keys(ctx, G.c.as<double>(), G.V, keys.as<uint64_t>());
    topk(ctx, keys.as<uint64_t>(), G.V, K, ids.as<int32_t>());
    phase_end(ctx, PH_TOPK, ph);
    copy_out(ctx, ids_out, ids.p, (size_t)K * 4);
    HM_API_END(ctx)
}

hm_status hm_compose(hm_ctx *ctx, int32_t heuristic, const int32_t *layer_ids, int32_t r, int32_t K,
                     int32_t *ids_out, int32_t *count_out) {
    HM_API_BEGIN(ctx)
    HM_REQUIRE(layer_ids && ids_out, HM_EINVAL, "null argument");
    HM_REQUIRE(heuristic == HM_NAIVE || heuristic == HM_CC1 || heuristic == HM_CC2 ||
                   heuristic == HM_CC2_AVG || heuristic == HM_CC1_RARY,
               HM_EINVAL, "unknown heuristic");
    HM_REQUIRE(r >= 2 && r <= 8, HM_EINVAL, "compose needs 2 <= r <= 8");
    std::set<int32_t> seen(layer_ids, layer_ids + r);
    HM_REQUIRE((int32_t)seen.size() == r, HM_EINVAL, "repeated graph id");
    std::vector<Graph *> gs;
    for (int i = 0; i < r; ++i) gs.push_back(&graph(ctx, layer_ids[i]));
    cudaEvent_t ph = phase_begin(ctx);
    compose(ctx, heuristic, gs, K, ids_out, count_out);
    phase_end(ctx, PH_COMPOSE, ph);
    HM_API_END(ctx)
}

hm_status hm_set_metrics(hm_ctx *ctx, int32_t V, const int32_t *est_ids, int64_t n_est,
                         const int32_t *gt_ids, int64_t n_gt, double *out) {
    HM_API_BEGIN(ctx)
    HM_REQUIRE(out && V > 0 && n_est >= 0 && n_gt >= 0, HM_EINVAL, "bad argument");
    HM_REQUIRE((n_est == 0 || est_ids) && (n_gt == 0 || gt_ids), HM_EINVAL, "null id list");
    cudaStream_t s = ctx->stream;
    // host id lists are staged to the device; device ones are read in place
    Buf stage((size_t)(n_est + n_gt) * 4 + 4, s), res(7 * 8 + 8, s);
    const int32_t *de = est_ids, *dg = gt_ids;
    if (n_est && !is_device_ptr(est_ids)) {
        HM_CUDA(cudaMemcpyAsync(stage.p, est_ids, (size_t)n_est * 4, cudaMemcpyHostToDevice, s));
        de = stage.as<int32_t>();
    }
    if (n_gt && !is_device_ptr(gt_ids)) {
        HM_CUDA(cudaMemcpyAsync(stage.as<int32_t>() + n_est, gt_ids, (size_t)n_gt * 4, cudaMemcpyHostToDevice, s));
        dg = stage.as<int32_t>() + n_est;
    }
    HM_CUDA(cudaMemsetAsync(res.p, 0, res.bytes, s));
    int32_t *d_bad = reinterpret_cast<int32_t *>(res.as<double>() + 7);
    set_metrics(ctx, V, de, n_est, dg, n_gt, res.as<double>(), d_bad);
    double h[8];
    HM_CUDA(cudaMemcpyAsync(h, res.p, sizeof h, cudaMemcpyDeviceToHost, s));
    host_sync(ctx);
    int32_t bad;
    memcpy(&bad, &h[7], 4);
    HM_REQUIRE(!bad, HM_ERANGE, "vertex id outside [0, V)");
    memcpy(out, h, 7 * sizeof(double));
    HM_API_END(ctx)
}

hm_status hm_exact_mean(hm_ctx *ctx, const double *x, int64_t n, const uint8_t *mask, double *mean_out,
                        int32_t *count_out) {
    HM_API_BEGIN(ctx)
    HM_REQUIRE(n >= 0 && mean_out && (n == 0 || x), HM_EINVAL, "bad argument");
    cudaStream_t s = ctx->stream;
    Buf stage((size_t)n * 9 + 16, s), res(32, s);
    const double *dx = x;
    const uint8_t *dm = mask;
    if (n && !is_device_ptr(x)) {
        HM_CUDA(cudaMemcpyAsync(stage.p, x, (size_t)n * 8, cudaMemcpyHostToDevice, s));
        dx = stage.as<double>();
    }
    if (n && mask && !is_device_ptr(mask)) {
        HM_CUDA(cudaMemcpyAsync(stage.as<char>() + (size_t)n * 8, mask, (size_t)n, cudaMemcpyHostToDevice, s));
        dm = reinterpret_cast<const uint8_t *>(stage.as<char>() + (size_t)n * 8);
    }
    HM_CUDA(cudaMemsetAsync(res.p, 0, res.bytes, s));
    int32_t *d_cnt_bad = reinterpret_cast<int32_t *>(res.as<double>() + 1);
    exact_mean(ctx, dx, n, dm, res.as<double>(), d_cnt_bad, d_cnt_bad + 1);
    struct { double mu; int32_t cnt, bad; } h;
    HM_CUDA(cudaMemcpyAsync(&h, res.p, 16, cudaMemcpyDeviceToHost, s));
    host_sync(ctx);
    HM_REQUIRE(!h.bad, HM_EINVAL, "a selected value is negative, inf or nan");
    *mean_out = h.mu;
    if (count_out) *count_out = h.cnt;
    HM_API_END(ctx)
}

hm_status hm_debug_counts(hm_ctx *ctx, uint64_t *out, int32_t n) {
    HM_API_BEGIN(ctx)
    HM_REQUIRE(out && n > 0 && n <= 335872, HM_EINVAL, "bad debug buffer");
    HM_REQUIRE(ctx->dbgc.p, HM_ESTATE, "no debug counters (set bfs_dbg bit 2 and run hm_closeness)");
    HM_CUDA(cudaMemcpyAsync(out, ctx->dbgc.p, (size_t)n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    HM_CUDA(cudaStreamSynchronize(ctx->stream));
    HM_API_END(ctx)
}

hm_status hm_sync(hm_ctx *ctx) {
    HM_API_BEGIN(ctx)
    HM_CUDA(cudaStreamSynchronize(ctx->stream));
    HM_API_END(ctx)
}

hm_status hm_get_stats(hm_ctx *ctx, hm_stats *out, int reset) {
    HM_API_BEGIN(ctx)
    HM_REQUIRE(out, HM_EINVAL, "null out");
    unsigned long long dv[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    HM_CUDA(cudaMemcpyAsync(dv, ctx->dstats.p, 80, cudaMemcpyDeviceToHost, ctx->stream));
    HM_CUDA(cudaStreamSynchronize(ctx->stream));
    // the MS-BFS level guard (a level deeper than the batch's rows): results since the last reset are wrong
    HM_REQUIRE(dv[7] == 0, HM_ECUDA, "MS-BFS level guard tripped: a BFS ran deeper than its rows (kernel bug)");
    for (auto &pe : ctx->pending) {
        float ms = 0.f;
        HM_CUDA(cudaEventElapsedTime(&ms, pe.first, pe.second));
        ctx->stats.bfs_ms += ms;
        cudaEventDestroy(pe.first);
        cudaEventDestroy(pe.second);
    }
    ctx->pending.clear();
    for (auto &pe : ctx->phase_pending) {
        float ms = 0.f;
        HM_CUDA(cudaEventElapsedTime(&ms, pe.e0, pe.e1));
        ctx->phase_ms[pe.id] += ms;
        cudaEventDestroy(pe.e0);
        cudaEventDestroy(pe.e1);
    }
    ctx->phase_pending.clear();
    for (int i = 0; i < 10; ++i) out->phase_ms[i] = ctx->phase_ms[i];
    out->launches = ctx->stats.launches;
    out->host_syncs = ctx->stats.host_syncs;
    out->bfs_launches = ctx->stats.bfs_launches;
    out->bfs_ms = ctx->stats.bfs_ms;
    out->bfs_levels = (int64_t)dv[0];
    out->bfs_batches = (int64_t)dv[1];
    out->bfs_model_bytes = (double)dv[2];
    out->bfs_row_commits = (int64_t)dv[3];
    out->bfs_csr_bytes = (double)dv[4];
    out->bfs_td_levels = (int64_t)dv[5];
    out->bfs_state_bytes = (double)dv[6];
    out->bfs_gathers = (int64_t)dv[8];
    out->bfs_own_reads = (int64_t)dv[9];
    if (reset) {
        ctx->stats = Stats();
        for (int i = 0; i < 10; ++i) ctx->phase_ms[i] = 0.0;
        HM_CUDA(cudaMemsetAsync(ctx->dstats.p, 0, 128, ctx->stream));
        HM_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    HM_API_END(ctx)
}

}  // extern "C"
