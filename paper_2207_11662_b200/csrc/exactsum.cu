// Exact, correctly rounded sums of non-negative doubles.
//
// The paper averages closeness (CC nodes: "higher than the average",
// PAPER.md:186) and degree-distance ratios (Eq. 3) without
// fixing an evaluation order.  The reading here is: mean = RN(exact sum) / n,
// i.e. Python's math.fsum(x) / n -- independent of summation order, so the GPU
// result does not depend on the grid shape.
//
// Method: every finite double x = m * 2^e (m < 2^53, e >= -1074) is added,
// exactly, into a fixed-point accumulator of 32-bit limbs held in 64-bit
// counters; limb i weighs 2^(32 i + LO) with LO = -1088, so a value touches at
// most three limbs.  Counters cannot overflow for n < 2^31 values (each adds
// < 2^32 per limb).  A single thread then normalises carries and rounds the
// integer once to binary64 (round half to even) and divides by the count with
// one IEEE division.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace hm {
namespace {

constexpr int LO = -1088;
constexpr int NLIMB = 70;     // covers 2^-1088 .. 2^1152
constexpr int BLOCK = 256;

__global__ void __launch_bounds__(BLOCK) k_exact_accum(const double *__restrict__ x, int64_t n,
                                                       const uint8_t *__restrict__ mask,
                                                       unsigned long long *acc,
                                                       unsigned long long *count,
                                                       int32_t *bad) {
    __shared__ unsigned long long s[NLIMB];
    __shared__ unsigned long long s_cnt;
    for (int i = threadIdx.x; i < NLIMB; i += BLOCK) s[i] = 0ull;
    if (threadIdx.x == 0) s_cnt = 0ull;
    __syncthreads();
    unsigned long long my_cnt = 0;
    for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
        if (mask && !mask[i]) continue;
        const double v = x[i];
        ++my_cnt;
        const uint64_t bits = (uint64_t)__double_as_longlong(v);
        const int ef = (int)((bits >> 52) & 0x7ff);
        if ((bits >> 63) || ef == 0x7ff) {   // negative, inf or nan: outside the contract
            *bad = 1;
            continue;
        }
        uint64_t m = bits & ((1ull << 52) - 1);
        int e;
        if (ef == 0) {
            e = -1074;
        } else {
            m |= (1ull << 52);
            e = ef - 1075;
        }
        if (m == 0) continue;
        const int pos = e - LO;               // >= 14
        const int li = pos >> 5, off = pos & 31;
        const unsigned __int128 t = (unsigned __int128)m << off;
        const uint64_t l0 = (uint64_t)t & 0xffffffffull;
        const uint64_t l1 = (uint64_t)(t >> 32) & 0xffffffffull;
        const uint64_t l2 = (uint64_t)(t >> 64) & 0xffffffffull;
        if (l0) atomicAdd(&s[li], (unsigned long long)l0);
        if (l1) atomicAdd(&s[li + 1], (unsigned long long)l1);
        if (l2) atomicAdd(&s[li + 2], (unsigned long long)l2);
    }
    // count: warp reduce then shared atomic
    for (int o = 16; o > 0; o >>= 1) my_cnt += __shfl_xor_sync(0xffffffffu, my_cnt, o);
    if ((threadIdx.x & 31) == 0 && my_cnt) atomicAdd(&s_cnt, my_cnt);
    __syncthreads();
    for (int i = threadIdx.x; i < NLIMB; i += BLOCK)
        if (s[i]) atomicAdd(&acc[i], s[i]);
    if (threadIdx.x == 0 && s_cnt) atomicAdd(count, s_cnt);
}

// One thread: carry-normalise, round to nearest even, divide by count.
__global__ void k_exact_finish(const unsigned long long *acc_in, const unsigned long long *count,
                               double *mean_out, int32_t *count_out, const int32_t *bad, int32_t *bad_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (bad_out) *bad_out = *bad;
    uint32_t L[NLIMB + 2];
    unsigned long long carry = 0;
    for (int i = 0; i < NLIMB; ++i) {
        const unsigned long long v = acc_in[i] + carry;   // < 2^64 (acc < 2^63, carry < 2^32)
        L[i] = (uint32_t)(v & 0xffffffffull);
        carry = v >> 32;
    }
    L[NLIMB] = (uint32_t)(carry & 0xffffffffull);
    L[NLIMB + 1] = (uint32_t)(carry >> 32);
    int t = NLIMB + 1;
    while (t >= 0 && L[t] == 0) --t;
    double sum = 0.0;
    if (t >= 0) {
        const uint32_t hi = L[t];
        const uint32_t mid = t >= 1 ? L[t - 1] : 0u;
        const uint32_t lo = t >= 2 ? L[t - 2] : 0u;
        bool sticky = false;
        for (int i = t - 3; i >= 0; --i)
            if (L[i]) { sticky = true; break; }
        const unsigned __int128 X = ((unsigned __int128)hi << 64) | ((unsigned __int128)mid << 32) | lo;
        const int p = 64 + (31 - __clz((int)hi));           // index of X's top bit
        const int shift = p - 52;                             // >= 12
        uint64_t q = (uint64_t)(X >> shift);
        const unsigned __int128 rem = X & ((((unsigned __int128)1) << shift) - 1);
        const unsigned __int128 half = ((unsigned __int128)1) << (shift - 1);
        if (rem > half || (rem == half && (sticky || (q & 1ull)))) ++q;
        // value = q * 2^(shift + 32 (t-2) + LO); q <= 2^53 is exact in binary64
        const int e2 = shift + 32 * (t - 2) + LO;
        sum = ldexp((double)q, e2);
    }
    const unsigned long long n = *count;
    if (count_out) *count_out = (int32_t)n;
    *mean_out = n ? __ddiv_rn(sum, (double)n) : 0.0;
}

}  // namespace

void exact_mean(hm_ctx *ctx, const double *d_x, int64_t n, const uint8_t *d_mask_or_null,
                double *d_mean_out, int32_t *d_count_out, int32_t *d_bad_out) {
    cudaStream_t s = ctx->stream;
    Buf acc((NLIMB + 2) * sizeof(unsigned long long), s);
    HM_CUDA(cudaMemsetAsync(acc.p, 0, acc.bytes, s));
    unsigned long long *d_acc = acc.as<unsigned long long>();
    unsigned long long *d_cnt = d_acc + NLIMB;
    int32_t *d_bad = reinterpret_cast<int32_t *>(d_acc + NLIMB + 1);
    if (n > 0) {
        k_exact_accum<<<grid_for(n, BLOCK, (int64_t)ctx->num_sms * 8), BLOCK, 0, s>>>(
            d_x, n, d_mask_or_null, d_acc, d_cnt, d_bad);
        check_launch("k_exact_accum");
        count_launch(ctx);
    }
    k_exact_finish<<<1, 32, 0, s>>>(d_acc, d_cnt, d_mean_out, d_count_out, d_bad, d_bad_out);
    check_launch("k_exact_finish");
    count_launch(ctx);
}

}  // namespace hm
