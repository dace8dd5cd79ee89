// Device graph store: CSR construction from edge pairs, and Boolean layer
// aggregation (§3.1) by sorted-adjacency intersection / union.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace hm {
namespace {

constexpr int TB = 256;

inline int nbits(uint64_t x) {
    int b = 0;
    while (x) { ++b; x >>= 1; }
    return b;
}

// both directions of every non-loop pair as (u << 32 | v); loops and bad ids -> sentinel V << 32
__global__ void k_pair_keys(const int32_t *__restrict__ e, int64_t m, int32_t V, uint64_t *keys, int32_t *bad) {
    const uint64_t sent = (uint64_t)V << 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t u = e[2 * i], v = e[2 * i + 1];
        if (u < 0 || u >= V || v < 0 || v >= V) {
            *bad = 1;
            keys[2 * i] = keys[2 * i + 1] = sent;
        } else if (u == v) {
            keys[2 * i] = keys[2 * i + 1] = sent;
        } else {
            keys[2 * i] = ((uint64_t)(uint32_t)u << 32) | (uint32_t)v;
            keys[2 * i + 1] = ((uint64_t)(uint32_t)v << 32) | (uint32_t)u;
        }
    }
}

// flag first occurrences of valid keys in a sorted array
__global__ void k_unique_flags(const uint64_t *__restrict__ k, int64_t n, uint64_t sent, int32_t *flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = (k[i] < sent && (i == 0 || k[i] != k[i - 1])) ? 1 : 0;
}

__global__ void k_compact_keys(const uint64_t *__restrict__ k, const int32_t *__restrict__ flag,
                               const int32_t *__restrict__ pos, int64_t n, uint64_t *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (flag[i]) out[pos[i]] = k[i];
}

// CSR from sorted unique keys: row_ptr[w] = first index with row >= w
__global__ void k_keys_to_csr(const uint64_t *__restrict__ k, int64_t nnz, int32_t V, int32_t *row_ptr,
                              int32_t *col) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const int u = (int)(k[i] >> 32);
        const int prev = (i == 0) ? -1 : (int)(k[i - 1] >> 32);
        for (int w = prev + 1; w <= u; ++w) row_ptr[w] = (int32_t)i;
        col[i] = (int32_t)(k[i] & 0xffffffffull);
        if (i == nnz - 1)
            for (int w = u + 1; w <= V; ++w) row_ptr[w] = (int32_t)nnz;
    }
}

__device__ __forceinline__ bool bsearch_row(const int32_t *__restrict__ col, int lo, int hi, int v) {
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int x = col[mid];
        if (x == v) return true;
        if (x < v) lo = mid + 1;
        else hi = mid;
    }
    return false;
}

struct AggIn {
    const int32_t *rp[8];
    const int32_t *cl[8];
    int r;
    int drv;   // driver graph (fewest arcs)
};

// AND pass 1 (arc-parallel): keep[j] = 1 iff driver arc j = (u, v) is in every other graph's
// sorted row u
__global__ void k_and_keep(AggIn in, int32_t V, int64_t nd, int32_t *keep) {
    const int32_t *rpd = in.rp[in.drv];
    const int32_t *cld = in.cl[in.drv];
    const int64_t na = rpd[V];         // the driver's arcs (nd may be an upper bound: an AND input)
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nd; j += (int64_t)gridDim.x * blockDim.x) {
        if (j >= na) {
            keep[j] = 0;
            continue;
        }
        const int u = csr_row_of(rpd, V, j);
        const int v = cld[j];
        bool ok = true;
        for (int g = 0; g < in.r && ok; ++g) {
            if (g == in.drv) continue;
            ok = bsearch_row(in.cl[g], in.rp[g][u], in.rp[g][u + 1], v);
        }
        keep[j] = ok ? 1 : 0;
    }
}

// AND pass 2: kept arcs to their exclusive-scan positions (CSR order is arc order), and
// row_ptr[u] = pos[first driver arc of u]
__global__ void k_and_fill(AggIn in, int32_t V, int64_t nd, const int32_t *__restrict__ keep,
                           const int32_t *__restrict__ pos, int32_t *orp, int32_t *ocol) {
    const int32_t *rpd = in.rp[in.drv];
    const int32_t *cld = in.cl[in.drv];
    const int64_t n = nd > (int64_t)V + 1 ? nd : (int64_t)V + 1;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        if (j < nd && keep[j]) ocol[pos[j]] = cld[j];
        if (j <= V) orp[j] = pos[rpd[j]];
    }
}

// OR: all arcs of all graphs as keys (warp per row)
__global__ void k_or_keys(AggIn in, int32_t V, const int64_t *off, uint64_t *keys) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int g = 0; g < in.r; ++g) {
        const int32_t *rp = in.rp[g];
        const int32_t *cl = in.cl[g];
        for (int64_t u = w0; u < V; u += nw)
            for (int j = rp[u] + lane; j < rp[u + 1]; j += 32)
                keys[off[g] + j] = ((uint64_t)u << 32) | (uint32_t)cl[j];
    }
}

// sorted keys (with possible duplicates / sentinels) -> G's CSR; returns nnz
int64_t csr_from_sorted_keys(hm_ctx *ctx, const uint64_t *d_sorted, int64_t n, int32_t V, Graph &G) {
    cudaStream_t s = ctx->stream;
    const uint64_t sent = (uint64_t)V << 32;
    Buf flag((size_t)(n + 1) * 4, s), pos((size_t)(n + 1) * 4, s);
    const unsigned g = grid_for(n, TB, (int64_t)ctx->num_sms * 16);
    k_unique_flags<<<g, TB, 0, s>>>(d_sorted, n, sent, flag.as<int32_t>());
    HM_CUDA(cudaMemsetAsync(flag.as<int32_t>() + n, 0, 4, s));
    size_t tb = 0;
    HM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.as<int32_t>(), pos.as<int32_t>(), n + 1, s));
    Buf tmp(tb, s);
    HM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, flag.as<int32_t>(), pos.as<int32_t>(), n + 1, s));
    int32_t nnz32 = 0;
    HM_CUDA(cudaMemcpyAsync(&nnz32, pos.as<int32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
    host_sync(ctx);
    const int64_t nnz = nnz32;
    Buf ukeys((size_t)(nnz > 0 ? nnz : 1) * 8, s);
    k_compact_keys<<<g, TB, 0, s>>>(d_sorted, flag.as<int32_t>(), pos.as<int32_t>(), n, ukeys.as<uint64_t>());
    G.V = V;
    G.nnz = nnz;
    G.row_ptr.alloc((size_t)(V + 1) * 4, s);
    G.col.alloc((size_t)(nnz > 0 ? nnz : 1) * 4, s);
    if (nnz == 0) {
        HM_CUDA(cudaMemsetAsync(G.row_ptr.p, 0, G.row_ptr.bytes, s));
    } else {
        k_keys_to_csr<<<grid_for(nnz, TB, (int64_t)ctx->num_sms * 16), TB, 0, s>>>(
            ukeys.as<uint64_t>(), nnz, V, G.row_ptr.as<int32_t>(), G.col.as<int32_t>());
    }
    check_launch("csr_from_sorted_keys");
    count_launch(ctx, 3);
    return nnz;
}

void sort_keys(hm_ctx *ctx, Buf &keys, Buf &sorted, int64_t n, int end_bit) {
    cudaStream_t s = ctx->stream;
    size_t tb = 0;
    HM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.as<uint64_t>(), sorted.as<uint64_t>(), (int)n, 0,
                                           end_bit, s));
    Buf tmp(tb, s);
    HM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys.as<uint64_t>(), sorted.as<uint64_t>(), (int)n, 0,
                                           end_bit, s));
    count_launch(ctx, 4);
}

}  // namespace

int64_t exact_nnz(hm_ctx *ctx, Graph &G) {
    if (!G.nnz_exact) {
        int32_t n = 0;
        HM_CUDA(cudaMemcpyAsync(&n, G.row_ptr.as<int32_t>() + G.V, 4, cudaMemcpyDeviceToHost, ctx->stream));
        host_sync(ctx);
        G.nnz = n;
        G.nnz_exact = true;
    }
    return G.nnz;
}

namespace {

__global__ void k_degrees(const int32_t *row_ptr, int32_t V, int32_t *deg) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
        deg[v] = row_ptr[v + 1] - row_ptr[v];
}

}  // namespace

void degrees(hm_ctx *ctx, const Graph &G, int32_t *d_deg) {
    k_degrees<<<grid_for(G.V, TB, (int64_t)ctx->num_sms * 16), TB, 0, ctx->stream>>>(G.row_ptr.as<int32_t>(), G.V,
                                                                                        d_deg);
    check_launch("k_degrees");
    count_launch(ctx);
}

void build_csr(hm_ctx *ctx, int32_t V, const int32_t *edges, int64_t m, Graph &G, int64_t *dropped) {
    cudaStream_t s = ctx->stream;
    HM_REQUIRE(m >= 0, HM_EINVAL, "negative edge count");
    HM_REQUIRE(2 * m < (int64_t)INT32_MAX, HM_ERANGE, "2*m >= 2^31 arcs does not fit an int32 CSR");
    const int64_t n = 2 * m;
    Buf dev_edges;
    const int32_t *d_e = edges;
    if (m > 0 && !is_device_ptr(edges)) {
        dev_edges.alloc((size_t)n * 4, s);
        HM_CUDA(cudaMemcpyAsync(dev_edges.p, edges, (size_t)n * 4, cudaMemcpyHostToDevice, s));
        d_e = dev_edges.as<int32_t>();
    }
    Buf keys((size_t)(n > 0 ? n : 1) * 8, s), sorted((size_t)(n > 0 ? n : 1) * 8, s), bad(8, s);
    HM_CUDA(cudaMemsetAsync(bad.p, 0, 8, s));
    if (m > 0) {
        k_pair_keys<<<grid_for(m, TB, (int64_t)ctx->num_sms * 16), TB, 0, s>>>(d_e, m, V, keys.as<uint64_t>(),
                                                                               bad.as<int32_t>());
        check_launch("k_pair_keys");
        count_launch(ctx);
    }
    int32_t h_bad = 0;
    HM_CUDA(cudaMemcpyAsync(&h_bad, bad.p, 4, cudaMemcpyDeviceToHost, s));
    host_sync(ctx);
    HM_REQUIRE(!h_bad, HM_ERANGE, "edge endpoint outside [0, V)");
    if (n > 0) sort_keys(ctx, keys, sorted, n, 32 + nbits((uint64_t)V));
    const int64_t nnz = csr_from_sorted_keys(ctx, sorted.as<uint64_t>(), n, V, G);
    if (dropped) *dropped = m - nnz / 2;
}

void and_or_aggregate(hm_ctx *ctx, const std::vector<Graph *> &in, bool is_and, Graph &out) {
    cudaStream_t s = ctx->stream;
    const int r = (int)in.size();
    HM_REQUIRE(r >= 2 && r <= 8, HM_EINVAL, "aggregation needs 2 <= r <= 8 graphs");
    const int32_t V = in[0]->V;
    AggIn a;
    a.r = r;
    a.drv = 0;
    for (int i = 0; i < r; ++i) {
        a.rp[i] = in[i]->row_ptr.as<int32_t>();
        a.cl[i] = in[i]->col.as<int32_t>();
        if (in[i]->nnz < in[a.drv]->nnz) a.drv = i;
    }
    const unsigned gw = grid_for((int64_t)V * 32, TB, (int64_t)ctx->num_sms * 16);
    if (is_and) {
        const int64_t nd = in[a.drv]->nnz;
        HM_REQUIRE(nd < (int64_t)INT32_MAX, HM_ERANGE, "AND aggregate too large for an int32 CSR");
        // keep flags (+ a zero sentinel at nd), their exclusive scan = output positions
        Buf keep((size_t)(nd + 1) * 4, s), pos((size_t)(nd + 1) * 4, s), orp((size_t)(V + 1) * 4, s);
        HM_CUDA(cudaMemsetAsync(keep.as<int32_t>() + nd, 0, 4, s));
        const unsigned ga = grid_for(nd > V ? nd : (int64_t)V + 1, TB, (int64_t)ctx->num_sms * 16);
        if (nd > 0) k_and_keep<<<ga, TB, 0, s>>>(a, V, nd, keep.as<int32_t>());
        size_t tb = 0;
        HM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, keep.as<int32_t>(), pos.as<int32_t>(), nd + 1, s));
        Buf tmp(tb, s);
        HM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, keep.as<int32_t>(), pos.as<int32_t>(), nd + 1, s));
        // no host round trip: the output is sized by the driver's arcs (an upper bound; the
        // exact count stays on the device in row_ptr[V] and is read only when a caller asks)
        out.V = V;
        out.nnz = nd;
        out.nnz_exact = false;
        out.col.alloc((size_t)(nd > 0 ? nd : 1) * 4, s);
        k_and_fill<<<ga, TB, 0, s>>>(a, V, nd, keep.as<int32_t>(), pos.as<int32_t>(), orp.as<int32_t>(),
                                     out.col.as<int32_t>());
        out.row_ptr = std::move(orp);
        check_launch("and_aggregate");
        count_launch(ctx, 3);
    } else {
        std::vector<int64_t> off(r + 1, 0);
        for (int i = 0; i < r; ++i) off[i + 1] = off[i] + exact_nnz(ctx, *in[i]);
        const int64_t n = off[r];
        HM_REQUIRE(n < (int64_t)INT32_MAX, HM_ERANGE, "OR aggregate too large for an int32 CSR");
        Buf doff((size_t)(r + 1) * 8, s), keys((size_t)(n > 0 ? n : 1) * 8, s), sorted((size_t)(n > 0 ? n : 1) * 8, s);
        HM_CUDA(cudaMemcpyAsync(doff.p, off.data(), (size_t)(r + 1) * 8, cudaMemcpyHostToDevice, s));
        k_or_keys<<<gw, TB, 0, s>>>(a, V, doff.as<int64_t>(), keys.as<uint64_t>());
        check_launch("k_or_keys");
        count_launch(ctx);
        if (n > 0) sort_keys(ctx, keys, sorted, n, 32 + nbits((uint64_t)V));
        csr_from_sorted_keys(ctx, sorted.as<uint64_t>(), n, V, out);
        host_sync(ctx);   // host vector `off` lifetime
    }
    out.alive = true;
    out.is_layer = false;
}

}  // namespace hm
