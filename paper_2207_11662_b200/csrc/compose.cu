// Composition Theta (§5): CC2 (Alg. 1), CC1 (Eq. 2, Eq. 3 and
// its pseudocode) and the naive baseline, over r >= 2 layers' cached Psi
// results.  Only per-layer results and the layers' own neighbourhoods (NBD,
// PAPER.md:431) are read -- never an AND aggregate.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "exactsum.cuh"

namespace hm {
namespace {

constexpr int TB = 256;
constexpr int RMAX = 8;

struct LayerPtrs {
    const uint64_t *pen[RMAX];
    const int32_t *deg[RMAX];
    const uint32_t *ch[RMAX];
    const int32_t *rp[RMAX];
    const int32_t *cl[RMAX];
    int r;
};

// CC2 (Alg. 1): estSumDist(u) = max_i sumDist_i(u) (n-penalty
// sums, reading Z3).  Ranking by Eq. 1 (n-1)/est descending == est ascending.
__global__ void k_cc2_keys(LayerPtrs L, int V, uint64_t *key, int32_t *count, int K) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *count = K;      // CC2 ranks every vertex
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        uint64_t e = L.pen[0][v];
        for (int i = 1; i < L.r; ++i) e = max(e, L.pen[i][v]);
        key[v] = e;
    }
}

// naive: common CC nodes; key 0 for members (ranked by id), ~0 otherwise
__global__ void k_naive_keys(LayerPtrs L, int V, uint64_t *key, int32_t *count) {
    const int lane = threadIdx.x & 31;
    for (int64_t vb = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31LL; vb < V;
         vb += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = vb + lane;
        uint32_t w = 0xffffffffu;
        for (int i = 0; i < L.r; ++i) w &= L.ch[i][vb >> 5];
        if (vb + 32 > V) w &= (V - vb >= 32) ? 0xffffffffu : ((1u << (V - vb)) - 1u);
        if (v < V) key[v] = ((w >> lane) & 1u) ? 0ull : ~0ull;
        if (lane == 0 && w) atomicAdd(count, __popc(w));
    }
}

// CC1 step 1 (Eq. 2): mindeg, ratio_i = pen_i / mindeg (+inf if mindeg = 0, Z8),
// fused with the exact sums of Eq. 3's layer averages (reading Z6: RN(exact sum) / count over
// the finite ratios, Z8) and the zeroing of the main loop's counters and bitmap: one pass instead of
// a ratio kernel, r exact-mean reductions and two memsets.  acc: r x EXACT_NLIMB zeroed 64-bit limbs,
// then the finite count.  At most EXACT_MAX_PER_BLOCK vertices per block.
__global__ void __launch_bounds__(256) k_cc1_ratios_sums(LayerPtrs L, int V, int32_t *mindeg, double *ratio,
                                                         unsigned long long *acc, int32_t *icnt, uint32_t *R) {
    __shared__ unsigned s16[RMAX][2 * EXACT_NLIMB];
    __shared__ int s_cnt;
    for (int i = threadIdx.x; i < L.r * 2 * EXACT_NLIMB; i += blockDim.x) s16[i / (2 * EXACT_NLIMB)][i % (2 * EXACT_NLIMB)] = 0u;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    int my = 0;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        int md = L.deg[0][v];
        for (int i = 1; i < L.r; ++i) md = min(md, L.deg[i][v]);
        mindeg[v] = md;
        icnt[v] = 0;
        if ((v & 31) == 0) R[v >> 5] = 0u;
        for (int i = 0; i < L.r; ++i) {
            const double q = md >= 1 ? __ddiv_rn((double)L.pen[i][v], (double)md) : (double)INFINITY;
            ratio[(size_t)i * V + v] = q;
            if (md >= 1) exact_add16(s16[i], q);
        }
        my += md >= 1;
    }
    my = __reduce_add_sync(0xffffffffu, my);
    if ((threadIdx.x & 31) == 0 && my) atomicAdd(&s_cnt, my);
    __syncthreads();
    for (int i = threadIdx.x; i < L.r * EXACT_NLIMB; i += blockDim.x) {
        const unsigned long long x = exact_limb16(s16[i / EXACT_NLIMB], i % EXACT_NLIMB);
        if (x) atomicAdd(&acc[i], x);
    }
    if (threadIdx.x == 0 && s_cnt) atomicAdd(&acc[(size_t)L.r * EXACT_NLIMB], (unsigned long long)s_cnt);
}

// avg_i = RN(exact sum of finite ratio_i) / |F| (0 if F is empty), then Eq. 3: avgAND = max_i avg_i
__global__ void k_cc1_avgs(const unsigned long long *acc, int r, double *avgs) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const unsigned long long n = acc[(size_t)r * EXACT_NLIMB];
    double m = 0.0;
    for (int i = 0; i < r; ++i) {
        const double a = n ? __ddiv_rn(exact_round(acc + (size_t)i * EXACT_NLIMB), (double)n) : 0.0;
        avgs[i] = a;
        m = i == 0 ? a : fmax(m, a);
    }
    avgs[r] = m;
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

// CC1 main loop (pseudocode PAPER.md:486-507, flat r-ary, Z7-Z12), arc-parallel over the
// arcs (u, v) of layer 0 (the intersection is symmetric in the layers, so any layer can drive;
// CC nodes are often hubs, whose rows would serialise a warp):
//   v ∈ I(u) iff ratio_i(v) < avgAND and v ∈ NBD_i(u) for every layer i.
// pass 0 counts |I(u)| (warp-aggregated per row); pass 1 adds I(u) when |I(u)| > 1 and adds
// every common u.  R is a bitmap (atomicOr -- set union is order-free).
__device__ __forceinline__ bool cc1_common(const LayerPtrs &L, int u) {
    bool common = true;
    for (int i = 0; i < L.r; ++i) common = common && ((L.ch[i][u >> 5] >> (u & 31)) & 1u);
    return common;
}
__global__ void k_cc1_main(LayerPtrs L, int V, int64_t nnz0, const double *ratio, const double *avg_and_p,
                           int32_t *icnt, uint32_t *R, int pass) {
    const double avg_and = *avg_and_p;
    const int64_t n = nnz0 > V ? nnz0 : V;
    const int64_t na = L.rp[0][V];     // layer 0's arcs (nnz0 may be an upper bound: an AND graph)
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        if (pass == 1 && j < V && cc1_common(L, (int)j)) atomicOr(&R[j >> 5], 1u << (j & 31));
        bool in = false;
        int u = -1;
        if (j < na) {
            u = csr_row_of(L.rp[0], V, j);
            if (cc1_common(L, u) && (pass == 0 || icnt[u] > 1)) {
                const int v = L.cl[0][j];
                in = true;
                for (int i = 0; i < L.r && in; ++i) {
                    in = ratio[(size_t)i * V + v] < avg_and;
                    if (in && i != 0) in = bsearch_row(L.cl[i], L.rp[i][u], L.rp[i][u + 1], v);
                }
                if (in && pass == 1) atomicOr(&R[v >> 5], 1u << (v & 31));
            }
        }
        if (pass == 0) {
            const unsigned act = __activemask();
            const unsigned inm = __ballot_sync(act, in);
            if (in) {
                const unsigned same = __match_any_sync(inm, u);
                if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(icnt + u, __popc(same));
            }
        }
    }
}

// CC1 ranking (Z13): members keyed by the bits of RN(est/mindeg) (positive
// doubles order as their bit patterns), others ~0; |R| into *count.
__global__ void k_cc1_keys(LayerPtrs L, int V, const uint32_t *R, const int32_t *mindeg, uint64_t *key,
                           int32_t *count) {
    const int lane = threadIdx.x & 31;
    for (int64_t vb = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31LL; vb < V;
         vb += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = vb + lane;
        const uint32_t w = R[vb >> 5];
        if (v < V) {
            if ((w >> lane) & 1u) {
                uint64_t e = L.pen[0][v];
                for (int i = 1; i < L.r; ++i) e = max(e, L.pen[i][v]);
                const double q = __ddiv_rn((double)e, (double)mindeg[v]);
                key[v] = (uint64_t)__double_as_longlong(q);
            } else {
                key[v] = ~0ull;
            }
        }
        if (lane == 0 && w) atomicAdd(count, __popc(w));
    }
}

// CC2 with the "above-average" selection: Eq. 1 on estSumDist,
// score = (V-1) / est in binary64 (est > 0 whenever V > 1).
__global__ void k_cc2_scores(LayerPtrs L, int V, double *score) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        uint64_t e = L.pen[0][v];
        for (int i = 1; i < L.r; ++i) e = max(e, L.pen[i][v]);
        score[v] = e > 0 ? __ddiv_rn((double)(V - 1), (double)e) : 0.0;
    }
}

// members: score > mean (strict, Z4); key 0 for members (ranked by id), ~0 otherwise
__global__ void k_above_keys(const double *score, const double *mu, int V, uint64_t *key, int32_t *count) {
    const int lane = threadIdx.x & 31;
    const double m = *mu;
    for (int64_t vb = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31LL; vb < V;
         vb += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = vb + lane;
        const bool in = v < V && score[v] > m;
        if (v < V) key[v] = in ? 0ull : ~0ull;
        const unsigned b = __ballot_sync(0xffffffffu, in);
        if (lane == 0 && b) atomicAdd(count, __popc(b));
    }
}

// id list -> membership bitmap (duplicates collapse: set semantics); an id
// outside [0, V) sets *bad
__global__ void k_ids_to_bitmap(const int32_t *ids, int64_t n, int V, uint32_t *bm, int32_t *bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = ids[i];
        if (v < 0 || v >= V) {
            *bad = 1;
            continue;
        }
        atomicOr(bm + (v >> 5), 1u << (v & 31));
    }
}

// |A|, |B|, |A ∩ B| of two vertex bitmaps, then Jaccard / precision / recall /
// F1 (PAPER.md:372; empty-set conventions SPEC.md:370, :379) in one thread.
__global__ void k_set_counts(const uint32_t *a, const uint32_t *b, int nw, unsigned long long *cnt) {
    unsigned long long ca = 0, cb = 0, cab = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += gridDim.x * blockDim.x) {
        ca += __popc(a[i]);
        cb += __popc(b[i]);
        cab += __popc(a[i] & b[i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        ca += __shfl_xor_sync(0xffffffffu, ca, o);
        cb += __shfl_xor_sync(0xffffffffu, cb, o);
        cab += __shfl_xor_sync(0xffffffffu, cab, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(cnt + 0, ca);
        atomicAdd(cnt + 1, cb);
        atomicAdd(cnt + 2, cab);
    }
}

__global__ void k_set_metrics(const unsigned long long *cnt, double *out) {
    if (threadIdx.x != 0) return;
    const double na = (double)cnt[0], nb = (double)cnt[1], nab = (double)cnt[2];
    const double uni = na + nb - nab;
    const double jac = uni > 0 ? nab / uni : 1.0;
    const double p = na > 0 ? nab / na : (nb == 0 ? 1.0 : 0.0);
    const double r = nb > 0 ? nab / nb : 1.0;
    const double f = (p + r) > 0 ? 2.0 * p * r / (p + r) : 0.0;
    out[0] = jac;
    out[1] = p;
    out[2] = r;
    out[3] = f;
    out[4] = na;
    out[5] = nb;
    out[6] = nab;
}

// ids past the set size become -1 (device outputs of the sync-free path)
__global__ void k_pad_ids(int32_t *ids, int K, const int32_t *count) {
    const int n = *count;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x)
        if (i >= n) ids[i] = -1;
}

}  // namespace

void set_metrics(hm_ctx *ctx, int32_t V, const int32_t *d_est, int64_t n_est, const int32_t *d_gt,
                 int64_t n_gt, double *d_out7, int32_t *d_bad) {
    cudaStream_t s = ctx->stream;
    const int nw = (V + 31) / 32;
    Buf bm((size_t)nw * 8, s), cnt(32, s);
    HM_CUDA(cudaMemsetAsync(bm.p, 0, bm.bytes, s));
    HM_CUDA(cudaMemsetAsync(cnt.p, 0, 32, s));
    uint32_t *a = bm.as<uint32_t>(), *b = a + nw;
    if (n_est > 0) {
        k_ids_to_bitmap<<<grid_for(n_est, TB, (int64_t)ctx->num_sms * 4), TB, 0, s>>>(d_est, n_est, V, a, d_bad);
        count_launch(ctx);
    }
    if (n_gt > 0) {
        k_ids_to_bitmap<<<grid_for(n_gt, TB, (int64_t)ctx->num_sms * 4), TB, 0, s>>>(d_gt, n_gt, V, b, d_bad);
        count_launch(ctx);
    }
    k_set_counts<<<grid_for(nw, TB, (int64_t)ctx->num_sms * 4), TB, 0, s>>>(a, b, nw,
                                                                           cnt.as<unsigned long long>());
    k_set_metrics<<<1, 32, 0, s>>>(cnt.as<unsigned long long>(), d_out7);
    check_launch("set_metrics");
    count_launch(ctx, 2);
}

void compose(hm_ctx *ctx, int heuristic, const std::vector<Graph *> &gs, int32_t K, int32_t *ids_out,
             int32_t *count_out) {
    cudaStream_t s = ctx->stream;
    const int r = (int)gs.size();
    HM_REQUIRE(r >= 2 && r <= RMAX, HM_EINVAL, "compose needs 2 <= r <= 8 layers");
    // CC1 is defined for a pair of layers; the flat r-ary form (Z12) is opt-in
    HM_REQUIRE(heuristic != HM_CC1 || r == 2, HM_EINVAL,
               "CC1 is defined for two layers only (PAPER.md:477-507); use HM_CC1_RARY for the flat r-ary "
               "reading Z12");
    const int V = gs[0]->V;
    HM_REQUIRE(K >= 1 && K <= V, HM_EINVAL, "K must be in [1, V]");
    LayerPtrs L;
    L.r = r;
    for (int i = 0; i < r; ++i) {
        HM_REQUIRE(gs[i]->has_results, HM_ESTATE, "compose before hm_closeness on an input graph");
        HM_REQUIRE(gs[i]->V == V, HM_EINVAL, "graphs differ in V");
        L.pen[i] = gs[i]->pen.as<uint64_t>();
        L.deg[i] = gs[i]->deg.as<int32_t>();
        L.ch[i] = gs[i]->ch.as<uint32_t>();
        L.rp[i] = gs[i]->row_ptr.as<int32_t>();
        L.cl[i] = gs[i]->col.as<int32_t>();
    }
    const unsigned g = grid_for(V, TB, (int64_t)ctx->num_sms * 16);
    // ids[0..K) ranked ids, ids[K] = |result set| (one D2H for host outputs)
    Buf keys((size_t)V * 8, s), ids((size_t)(K + 1) * 4, s);
    int32_t *d_ids = ids.as<int32_t>();
    int32_t *d_cnt = d_ids + K;
    HM_CUDA(cudaMemsetAsync(d_cnt, 0, 4, s));
    if (heuristic == HM_CC2) {
        k_cc2_keys<<<g, TB, 0, s>>>(L, V, keys.as<uint64_t>(), d_cnt, K);
        check_launch("k_cc2_keys");
        count_launch(ctx);
    } else if (heuristic == HM_NAIVE) {
        k_naive_keys<<<g, TB, 0, s>>>(L, V, keys.as<uint64_t>(), d_cnt);
        check_launch("k_naive_keys");
        count_launch(ctx);
    } else if (heuristic == HM_CC2_AVG) {
        Buf score((size_t)V * 8, s), mu(16, s);
        k_cc2_scores<<<g, TB, 0, s>>>(L, V, score.as<double>());
        exact_mean(ctx, score.as<double>(), V, nullptr, mu.as<double>(), nullptr);
        k_above_keys<<<g, TB, 0, s>>>(score.as<double>(), mu.as<double>(), V, keys.as<uint64_t>(), d_cnt);
        check_launch("cc2 above-average");
        count_launch(ctx, 2);
    } else if (heuristic == HM_CC1 || heuristic == HM_CC1_RARY) {
        Buf mindeg((size_t)V * 4, s), ratio((size_t)V * r * 8, s);
        Buf avgs((size_t)(r + 1) * 8, s), R((size_t)((V + 31) / 32) * 4, s), icnt((size_t)V * 4, s);
        Buf acc(((size_t)r * EXACT_NLIMB + 1) * 8, s);
        HM_CUDA(cudaMemsetAsync(acc.p, 0, acc.bytes, s));
        int64_t nb = grid_for(V, TB, (int64_t)ctx->num_sms * 16);
        const int64_t need = ((int64_t)V + EXACT_MAX_PER_BLOCK - 1) / EXACT_MAX_PER_BLOCK;
        if (nb < need) nb = need;
        // ratios (Eq. 2), the exact layer sums, zeroed counters and bitmap in one pass; then Eq. 3
        k_cc1_ratios_sums<<<(unsigned)nb, TB, 0, s>>>(L, V, mindeg.as<int32_t>(), ratio.as<double>(),
                                                     acc.as<unsigned long long>(), icnt.as<int32_t>(),
                                                     R.as<uint32_t>());
        k_cc1_avgs<<<1, 32, 0, s>>>(acc.as<unsigned long long>(), r, avgs.as<double>());
        count_launch(ctx, 2);
        const int64_t nnz0 = gs[0]->nnz;
        const unsigned ga = grid_for(nnz0 > V ? nnz0 : (int64_t)V, TB, (int64_t)ctx->num_sms * 16);
        for (int pass = 0; pass < 2; ++pass)
            k_cc1_main<<<ga, TB, 0, s>>>(L, V, nnz0, ratio.as<double>(), avgs.as<double>() + r,
                                         icnt.as<int32_t>(), R.as<uint32_t>(), pass);
        k_cc1_keys<<<g, TB, 0, s>>>(L, V, R.as<uint32_t>(), mindeg.as<int32_t>(), keys.as<uint64_t>(), d_cnt);
        check_launch("cc1");
        count_launch(ctx, 4);
    } else {
        throw Error(HM_EINVAL, "unknown heuristic");
    }
    // Top-K over all V keys: members' keys are below ~0 (non-members), so the first
    // min(K, |R|) ranked ids are the members and no host round trip is needed before it.
    topk(ctx, keys.as<uint64_t>(), V, K, d_ids);
    const bool dev_ids = is_device_ptr(ids_out);
    const bool dev_cnt = count_out == nullptr || is_device_ptr(count_out);
    if (dev_ids && dev_cnt) {                         // fully stream-ordered: no synchronisation
        k_pad_ids<<<grid_for(K, TB, (int64_t)ctx->num_sms * 4), TB, 0, s>>>(d_ids, K, d_cnt);
        check_launch("k_pad_ids");
        count_launch(ctx);
        HM_CUDA(cudaMemcpyAsync(ids_out, d_ids, (size_t)K * 4, cudaMemcpyDeviceToDevice, s));
        if (count_out) HM_CUDA(cudaMemcpyAsync(count_out, d_cnt, 4, cudaMemcpyDeviceToDevice, s));
        return;
    }
    std::vector<int32_t> h((size_t)K + 1);
    HM_CUDA(cudaMemcpyAsync(h.data(), d_ids, (size_t)(K + 1) * 4, cudaMemcpyDeviceToHost, s));
    host_sync(ctx);
    const int32_t nR = h[K];
    const int32_t Kout = nR < K ? nR : K;
    if (dev_ids) {
        if (Kout > 0) HM_CUDA(cudaMemcpyAsync(ids_out, d_ids, (size_t)Kout * 4, cudaMemcpyDeviceToDevice, s));
    } else {
        for (int i = 0; i < Kout; ++i) ids_out[i] = h[i];
    }
    if (count_out) {
        if (dev_cnt) HM_CUDA(cudaMemcpyAsync(count_out, d_cnt, 4, cudaMemcpyDeviceToDevice, s));
        else *count_out = nR;
    }
}

}  // namespace hm
