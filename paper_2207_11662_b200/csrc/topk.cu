// Top-K selection: the K smallest (key, id) pairs of n 64-bit keys, in order.
//
// Used by every ranking of the paper's outputs: ground truth by closeness
// (PAPER.md:205-209), CC2 by estSumDist, CC1 and naive result
// sets.  Ties go to the lower vertex id, so the
// composite (key << 32 | id) is unique and the answer is well defined.
//
// Radix select over the 96-bit composite, 8 bits per pass from the most
// significant: per pass a grid histogram of the digit among elements whose
// higher digits match the prefix found so far, then one small kernel picks
// the digit holding the K-th element.  After 12 passes the exact K-th
// composite T is known; every element <= T (exactly K) is gathered and sorted
// in shared memory (bitonic, K <= 4096) -- larger K use a stable device sort.
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace hm {
namespace {
namespace cg = cooperative_groups;

constexpr int TB = 256;
constexpr int SORT_MAX = 4096;

struct SelState {
    unsigned long long pkey;   // prefix of key bits found so far
    unsigned int pid;          // prefix of id bits found so far
    int rem;                   // rank still to find inside the current prefix group (1-based)
    unsigned int hist[256];
    int count;                 // gathered elements
    int done;                  // k_select_coop: the K-th element is fixed early (its key's group fits whole)
};

// digit p (0..11) of composite (key, id): p < 8 -> key byte (7-p), else id byte (11-p)
__device__ __forceinline__ unsigned digit_of(uint64_t key, uint32_t id, int p) {
    return p < 8 ? (unsigned)((key >> (8 * (7 - p))) & 0xff) : (unsigned)((id >> (8 * (11 - p))) & 0xff);
}

__device__ __forceinline__ bool prefix_match(uint64_t key, uint32_t id, uint64_t pkey, uint32_t pid, int p) {
    // digits 0..p-1 must match
    if (p == 0) return true;
    if (p <= 8) {
        const int sh = 64 - 8 * p;
        return (sh >= 64) ? true : ((key >> sh) == (pkey >> sh));
    }
    if (key != pkey) return false;
    const int sh = 32 - 8 * (p - 8);
    return (sh >= 32) ? true : ((id >> sh) == (pid >> sh));
}

__global__ void k_hist(const uint64_t *__restrict__ keys, int n, SelState *st, int p) {
    __shared__ unsigned h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint64_t pkey = st->pkey;
    const uint32_t pid = st->pid;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        if (prefix_match(k, (uint32_t)i, pkey, pid, p)) atomicAdd(&h[digit_of(k, (uint32_t)i, p)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (h[i]) atomicAdd(&st->hist[i], h[i]);
}

__global__ void k_sel_init(SelState *st, int K) {
    if (threadIdx.x == 0) st->rem = K;
}

__global__ void k_pick(SelState *st, int p) {
    if (threadIdx.x != 0) return;
    int rem = st->rem;
    unsigned b = 0;
    for (; b < 256; ++b) {
        const int c = (int)st->hist[b];
        if (rem <= c) break;
        rem -= c;
    }
    if (b > 255) b = 255;   // unreachable when K <= n
    st->rem = rem;
    if (p < 8) st->pkey |= (unsigned long long)b << (8 * (7 - p));
    else st->pid |= b << (8 * (11 - p));
    for (int i = 0; i < 256; ++i) st->hist[i] = 0;
}

__global__ void k_gather(const uint64_t *__restrict__ keys, int n, SelState *st, uint64_t *ok, uint32_t *oid) {
    const uint64_t tk = st->pkey;
    const uint32_t ti = st->pid;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        if (k < tk || (k == tk && (uint32_t)i <= ti)) {
            const int pos = atomicAdd(&st->count, 1);
            ok[pos] = k;
            oid[pos] = (uint32_t)i;
        }
    }
}

// The whole select in one cooperative launch: per pass a block histogram of the digit among the
// prefix-matching elements, merged into st->hist; after a grid barrier warp 0 of block 0 finds the
// digit holding the rem-th element (prefix sums over 8 bins per lane) and extends the prefix; after
// the 12th pass every block gathers its elements <= T.  (The multi-launch path below is kept for
// grids the cooperative launch cannot place.)
__global__ void __launch_bounds__(TB) k_select_coop(const uint64_t *__restrict__ keys, int n, SelState *st,
                                                    uint64_t *ok, uint32_t *oid, int K) {
    cg::grid_group grid = cg::this_grid();
    __shared__ unsigned h[256];
    __shared__ unsigned long long s_pkey;
    __shared__ unsigned s_pid;
    if (blockIdx.x == 0) {                       // the selection state (no separate memset / init launches)
        for (int i = threadIdx.x; i < 256; i += blockDim.x) st->hist[i] = 0u;
        if (threadIdx.x == 0) {
            st->pkey = 0ull;
            st->pid = 0u;
            st->rem = K;
            st->count = 0;
            st->done = 0;
        }
    }
    grid.sync();
    for (int p = 0; p < 12; ++p) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
        if (threadIdx.x == 0) {
            s_pkey = __ldcg(&st->pkey);
            s_pid = __ldcg(&st->pid);
        }
        __syncthreads();
        const uint64_t pkey = s_pkey;
        const uint32_t pid = s_pid;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            const uint64_t k = keys[i];
            if (prefix_match(k, (uint32_t)i, pkey, pid, p)) atomicAdd(&h[digit_of(k, (uint32_t)i, p)], 1u);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < 256; i += blockDim.x)
            if (h[i]) atomicAdd(&st->hist[i], h[i]);
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x < 32) {
            const int lane = threadIdx.x;
            unsigned c[8], tot = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c[q] = __ldcg(&st->hist[lane * 8 + q]);
                tot += c[q];
            }
            unsigned incl = tot;                         // inclusive prefix over lanes
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int rem = st->rem;
            const unsigned excl = incl - tot;
            // the lane whose bins hold the rem-th element: excl < rem <= incl
            const bool mine = (int)excl < rem && rem <= (int)incl;
            const unsigned who = __ballot_sync(0xffffffffu, mine);
            if (mine) {
                int r = rem - (int)excl;
                int b = 0;
                for (; b < 7; ++b) {
                    if (r <= (int)c[b]) break;
                    r -= (int)c[b];
                }
                const unsigned dg = (unsigned)(lane * 8 + b);
                st->rem = r;
                if (p < 8) st->pkey |= (unsigned long long)dg << (8 * (7 - p));
                else st->pid |= dg << (8 * (11 - p));
                if (p == 7 && r == (int)c[b]) {              // every element of key T is in: no id passes
                    st->pid = 0xffffffffu;
                    st->done = 1;
                }
            }
            if (!who && lane == 0) {                     // unreachable when K <= n
                if (p < 8) st->pkey |= 255ull << (8 * (7 - p));
                else st->pid |= 255u << (8 * (11 - p));
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) st->hist[lane * 8 + q] = 0;
        }
        grid.sync();
        if (p == 7 && __ldcg(&st->done)) break;                 // grid-uniform
    }
    const uint64_t tk = __ldcg(&st->pkey);
    const uint32_t ti = __ldcg(&st->pid);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        if (k < tk || (k == tk && (uint32_t)i <= ti)) {
            const int pos = atomicAdd(&st->count, 1);
            ok[pos] = k;
            oid[pos] = (uint32_t)i;
        }
    }
}

__device__ __forceinline__ bool less_kv(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// one block, K <= SORT_MAX: bitonic sort of (key, id) then write ids
// sort the first n (key, id) pairs (ids = positions when oid is null) in shared memory and write
// the first K ids; P = the power of two >= n
__global__ void __launch_bounds__(1024) k_sort_small(const uint64_t *ok, const uint32_t *oid, int n, int K, int P,
                                                     int32_t *out) {
    extern __shared__ unsigned char smem[];
    uint64_t *sk = reinterpret_cast<uint64_t *>(smem);
    uint32_t *si = reinterpret_cast<uint32_t *>(sk + P);
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        sk[i] = i < n ? ok[i] : ~0ull;
        si[i] = i < n ? (oid ? oid[i] : (uint32_t)i) : 0xffffffffu;
    }
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const bool sw = up ? less_kv(sk[j], si[j], sk[i], si[i]) : less_kv(sk[i], si[i], sk[j], si[j]);
                    if (sw) {
                        const uint64_t tk = sk[i]; sk[i] = sk[j]; sk[j] = tk;
                        const uint32_t ti = si[i]; si[i] = si[j]; si[j] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < K; i += blockDim.x) out[i] = (int32_t)si[i];
}

// ---- two-phase tile select (n > SORT_MAX, K <= SORT_MAX): no grid barrier.
// Phase A: block b selects the K smallest of its TILE_E pairs in shared memory (a block-local radix
// select, stopping at the first digit whose bin is taken whole) and writes them, padded to K with the
// sentinel (~0, ~0) that exceeds every real pair, to its candidate slot.  Phase B: the last block to
// finish (ticket) selects the K smallest of the G*K candidates the same way, sorts them (bitonic) and
// writes their ids.  One launch instead of a 12-pass cooperative select (C3: 40 top-K lists per step).
constexpr int TT = 1024;            // threads per block
constexpr int TILE_MAX = 8192;      // pairs per phase-A block (at most)
constexpr int CAND_MAX = 16384;     // candidates phase B holds in shared memory (G * K)

__device__ __forceinline__ bool le_depth(uint64_t k, uint32_t id, uint64_t tk, uint32_t ti, int p) {
    // the first p + 1 digits of (k, id) <= those of (tk, ti)
    if (p < 8) {
        const int sh = 8 * (7 - p);
        return (k >> sh) <= (tk >> sh);
    }
    if (k != tk) return k < tk;
    const int sh = 8 * (11 - p);
    return (id >> sh) <= (ti >> sh);
}

struct BlkSel {
    unsigned hist[256];
    unsigned long long pkey;
    unsigned pid;
    int rem, pend, cnt;
};

// block radix select over n pairs in shared memory: afterwards exactly K pairs satisfy
// le_depth(x, (bs.pkey, bs.pid), bs.pend)
__device__ void block_select(const uint64_t *sk, const uint32_t *si, int n, int K, BlkSel &bs) {
    if (threadIdx.x == 0) {
        bs.pkey = 0ull;
        bs.pid = 0u;
        bs.rem = K;
        bs.pend = -1;
    }
    for (int p = 0; p < 12; ++p) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) bs.hist[i] = 0u;
        __syncthreads();
        const uint64_t pk = bs.pkey;
        const uint32_t pi = bs.pid;
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            if (prefix_match(sk[i], si[i], pk, pi, p)) atomicAdd(&bs.hist[digit_of(sk[i], si[i], p)], 1u);
        __syncthreads();
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            unsigned c[8], tot = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c[q] = bs.hist[lane * 8 + q];
                tot += c[q];
            }
            unsigned incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int rem = bs.rem;
            const unsigned excl = incl - tot;
            if ((int)excl < rem && rem <= (int)incl) {           // exactly one lane (K <= n)
                int r = rem - (int)excl, b = 0;
                for (; b < 7; ++b) {
                    if (r <= (int)c[b]) break;
                    r -= (int)c[b];
                }
                const unsigned dg = (unsigned)(lane * 8 + b);
                if (p < 8) bs.pkey |= (unsigned long long)dg << (8 * (7 - p));
                else bs.pid |= dg << (8 * (11 - p));
                bs.rem = r;
                if (r == (int)c[b]) bs.pend = p;                  // the whole bin is taken: done
            }
        }
        __syncthreads();
        if (bs.pend >= 0) break;                                  // block-uniform
    }
}

// the first K pairs of (sk, si) -- P >= K a power of two, slots [K, P) padded by the caller -- sorted
__device__ void block_bitonic(uint64_t *sk, uint32_t *si, int P) {
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const bool sw = up ? less_kv(sk[j], si[j], sk[i], si[i]) : less_kv(sk[i], si[i], sk[j], si[j]);
                    if (sw) {
                        const uint64_t tk = sk[i]; sk[i] = sk[j]; sk[j] = tk;
                        const uint32_t ti = si[i]; si[i] = si[j]; si[j] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// selected pairs of (sk, si)[0, n) -> (ok, oi) at positions from the block counter bs.cnt (unordered)
__device__ void block_compact(const uint64_t *sk, const uint32_t *si, int n, const BlkSel &bs, uint64_t *ok,
                              uint32_t *oi, int *cnt) {
    const uint64_t tk = bs.pkey;
    const uint32_t ti = bs.pid;
    const int pe = bs.pend;
    const int lane = threadIdx.x & 31;
    for (int i0 = 0; i0 < n; i0 += blockDim.x) {                 // block-uniform trip count
        const int i = i0 + threadIdx.x;
        const bool sel = i < n && le_depth(sk[i], si[i], tk, ti, pe);
        const unsigned b = __ballot_sync(0xffffffffu, sel);
        int base = 0;
        if (lane == 0 && b) base = atomicAdd(cnt, __popc(b));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (sel) {
            const int pos = base + __popc(b & ((1u << lane) - 1u));
            ok[pos] = sk[i];
            oi[pos] = si[i];
        }
    }
}

__global__ void __launch_bounds__(TT) k_topk_tiles(const uint64_t *__restrict__ keys, int n, int K,
                                                  uint64_t *cand_k, uint32_t *cand_i, unsigned *ticket,
                                                  int32_t *out, int TILE_E) {
    extern __shared__ unsigned char smem[];
    __shared__ BlkSel bs;
    __shared__ int s_last;
    const int G = gridDim.x;
    const int nsm = max(min(n, TILE_E), G * K);                  // pairs the shared arrays hold
    uint64_t *sk = reinterpret_cast<uint64_t *>(smem);
    uint32_t *si = reinterpret_cast<uint32_t *>(sk + nsm);
    // phase A: this block's tile
    const int i0 = blockIdx.x * TILE_E;
    const int nb = min(TILE_E, n - i0);
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        sk[i] = keys[i0 + i];
        si[i] = (uint32_t)(i0 + i);
    }
    if (threadIdx.x == 0) bs.cnt = 0;
    __syncthreads();
    uint64_t *ck = cand_k + (size_t)blockIdx.x * K;
    uint32_t *ci = cand_i + (size_t)blockIdx.x * K;
    if (nb <= K) {
        for (int i = threadIdx.x; i < K; i += blockDim.x) {
            ck[i] = i < nb ? sk[i] : ~0ull;
            ci[i] = i < nb ? si[i] : 0xffffffffu;
        }
    } else {
        block_select(sk, si, nb, K, bs);
        block_compact(sk, si, nb, bs, ck, ci, &bs.cnt);          // exactly K
    }
    // the last block to finish merges
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == (unsigned)(G - 1)) ? 1 : 0;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int nc = G * K;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
        sk[i] = __ldcg(cand_k + i);
        si[i] = __ldcg(cand_i + i);
    }
    if (threadIdx.x == 0) bs.cnt = 0;
    __syncthreads();
    block_select(sk, si, nc, K, bs);
    // the K selected to the front of the candidate buffer (block 0's slot is re-read below)
    uint64_t *rk = cand_k + nc;
    uint32_t *ri = cand_i + nc;
    block_compact(sk, si, nc, bs, rk, ri, &bs.cnt);
    __threadfence_block();
    __syncthreads();
    int P = 1;
    while (P < K) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        sk[i] = i < K ? __ldcg(rk + i) : ~0ull;
        si[i] = i < K ? __ldcg(ri + i) : 0xffffffffu;
    }
    __syncthreads();
    block_bitonic(sk, si, P);
    for (int i = threadIdx.x; i < K; i += blockDim.x) out[i] = (int32_t)si[i];
    if (threadIdx.x == 0) *ticket = 0u;
}

__global__ void k_iota_u32(uint32_t *p, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = (uint32_t)i;
}
__global__ void k_copy_ids(const uint32_t *src, int K, int32_t *out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x) out[i] = (int32_t)src[i];
}

__global__ void k_desc_keys(const double *c, int V, uint64_t *key) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
        key[v] = ~(uint64_t)__double_as_longlong(c[v]);
}

}  // namespace

void closeness_desc_keys(hm_ctx *ctx, const double *d_c, int32_t V, uint64_t *d_keys) {
    k_desc_keys<<<grid_for(V, TB, (int64_t)ctx->num_sms * 16), TB, 0, ctx->stream>>>(d_c, V, d_keys);
    check_launch("k_desc_keys");
    count_launch(ctx);
}

void topk(hm_ctx *ctx, const uint64_t *d_keys, int32_t n, int32_t K, int32_t *d_ids_out) {
    cudaStream_t s = ctx->stream;
    HM_REQUIRE(K >= 1 && K <= n, HM_EINVAL, "top-K needs 1 <= K <= n");
    if (K > SORT_MAX) {
        // stable radix sort of all (key, id) pairs; ids ascending on ties
        Buf ids((size_t)n * 4, s), ko((size_t)n * 8, s), io((size_t)n * 4, s);
        k_iota_u32<<<grid_for(n, TB), TB, 0, s>>>(ids.as<uint32_t>(), n);
        size_t tb = 0;
        HM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, d_keys, ko.as<uint64_t>(), ids.as<uint32_t>(),
                                                io.as<uint32_t>(), n, 0, 64, s));
        Buf tmp(tb, s);
        HM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, d_keys, ko.as<uint64_t>(), ids.as<uint32_t>(),
                                                io.as<uint32_t>(), n, 0, 64, s));
        k_copy_ids<<<grid_for(K, TB), TB, 0, s>>>(io.as<uint32_t>(), K, d_ids_out);
        check_launch("topk large");
        count_launch(ctx, 10);
        return;
    }
    if (n <= SORT_MAX) {
        // small inputs: one CTA sorts all n (key, id) pairs in shared memory (one launch instead of
        // the select pipeline; C1: 4 top-K lists per step)
        int P = 1;
        while (P < n) P <<= 1;
        k_sort_small<<<1, 1024, (size_t)P * 12, s>>>(d_keys, nullptr, n, K, P, d_ids_out);
        check_launch("topk small");
        count_launch(ctx, 1);
        return;
    }
    {
        // two-phase tile select: one launch, no grid barrier (see k_topk_tiles)
        // tile: topk_tiles = 1 -> 8192 pairs per block; > 1 -> that many (a power of two, 1024 .. 8192)
        const int TILE_E = ctx->params.topk_tiles > 1 ? ctx->params.topk_tiles : TILE_MAX;
        const int G = (int)((n + TILE_E - 1) / TILE_E);
        if (ctx->params.topk_tiles && (int64_t)G * K <= CAND_MAX && G <= ctx->num_sms) {
            const int nsm = (n < TILE_E ? n : TILE_E) > G * K ? (n < TILE_E ? n : TILE_E) : G * K;
            const size_t sm = (size_t)nsm * 12;
            Buf cb((size_t)(G + 1) * K * 12 + 16, s);
            uint64_t *ck = cb.as<uint64_t>();
            uint32_t *ci = reinterpret_cast<uint32_t *>(ck + (size_t)(G + 1) * K);
            unsigned *ticket = reinterpret_cast<unsigned *>(ci + (size_t)(G + 1) * K);
            HM_CUDA(cudaMemsetAsync(ticket, 0, 4, s));
            HM_CUDA(cudaFuncSetAttribute(k_topk_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            k_topk_tiles<<<G, TT, sm, s>>>(d_keys, n, K, ck, ci, ticket, d_ids_out, TILE_E);
            check_launch("k_topk_tiles");
            count_launch(ctx, 1);
            return;
        }
    }
    Buf stb(sizeof(SelState), s), ok((size_t)K * 8, s), oid((size_t)K * 4, s);
    SelState *st = stb.as<SelState>();
    // one cooperative launch (grid: one CTA per 1 K keys, at most 4 per SM and what fits)
    int per_sm = 0;
    HM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_select_coop, TB, 0));
    if (per_sm > 4) per_sm = 4;
    int gc = (int)grid_for(n, TB * 4, (int64_t)ctx->num_sms * per_sm);
    if (gc < 1) gc = 1;
    if (per_sm >= 1) {
        const uint64_t *kp = d_keys;
        uint64_t *okp = ok.as<uint64_t>();
        uint32_t *oip = oid.as<uint32_t>();
        int Kk = K;
        void *args[] = {(void *)&kp, (void *)&n, (void *)&st, (void *)&okp, (void *)&oip, (void *)&Kk};
        HM_CUDA(cudaLaunchCooperativeKernel((const void *)k_select_coop, dim3(gc), dim3(TB), args, 0, s));
        count_launch(ctx, 1);
    } else {
        HM_CUDA(cudaMemsetAsync(st, 0, sizeof(SelState), s));
        k_sel_init<<<1, 32, 0, s>>>(st, K);
        const unsigned g = grid_for(n, TB, (int64_t)ctx->num_sms * 4);
        for (int p = 0; p < 12; ++p) {
            k_hist<<<g, TB, 0, s>>>(d_keys, n, st, p);
            k_pick<<<1, 32, 0, s>>>(st, p);
        }
        k_gather<<<g, TB, 0, s>>>(d_keys, n, st, ok.as<uint64_t>(), oid.as<uint32_t>());
        count_launch(ctx, 25);
    }
    int P = 1;
    while (P < K) P <<= 1;
    const size_t sm = (size_t)P * 12;
    if (sm > 48 * 1024)
        HM_CUDA(cudaFuncSetAttribute(k_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_sort_small<<<1, 1024, sm, s>>>(ok.as<uint64_t>(), oid.as<uint32_t>(), K, K, P, d_ids_out);
    check_launch("topk");
    count_launch(ctx, 1);
}

}  // namespace hm
