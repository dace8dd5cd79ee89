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
#include "exactsum.cuh"

namespace hm {
namespace {

constexpr int NLIMB = EXACT_NLIMB;
constexpr int BLOCK = 256;

__global__ void __launch_bounds__(BLOCK) k_exact_accum(const double *__restrict__ x, int64_t n,
                                                       const uint8_t *__restrict__ mask,
                                                       unsigned long long *acc,
                                                       unsigned long long *count,
                                                       int32_t *bad) {
    __shared__ unsigned s16[2 * NLIMB];
    __shared__ unsigned long long s_cnt;
    for (int i = threadIdx.x; i < 2 * NLIMB; i += BLOCK) s16[i] = 0u;
    if (threadIdx.x == 0) s_cnt = 0ull;
    __syncthreads();
    unsigned long long my_cnt = 0;
    for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
        if (mask && !mask[i]) continue;
        const double v = x[i];
        ++my_cnt;
        const uint64_t bits = (uint64_t)__double_as_longlong(v);
        if ((bits >> 63) || ((bits >> 52) & 0x7ff) == 0x7ff) {   // negative, inf or nan: outside the contract
            *bad = 1;
            continue;
        }
        exact_add16(s16, v);
    }
    // count: warp reduce then shared atomic
    for (int o = 16; o > 0; o >>= 1) my_cnt += __shfl_xor_sync(0xffffffffu, my_cnt, o);
    if ((threadIdx.x & 31) == 0 && my_cnt) atomicAdd(&s_cnt, my_cnt);
    __syncthreads();
    for (int i = threadIdx.x; i < NLIMB; i += BLOCK) {
        const unsigned long long x = exact_limb16(s16, i);
        if (x) atomicAdd(&acc[i], x);
    }
    if (threadIdx.x == 0 && s_cnt) atomicAdd(count, s_cnt);
}

// One thread: carry-normalise, round to nearest even, divide by count.
__global__ void k_exact_finish(const unsigned long long *acc_in, const unsigned long long *count,
                               double *mean_out, int32_t *count_out, const int32_t *bad, int32_t *bad_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (bad_out) *bad_out = *bad;
    const double sum = exact_round(acc_in);
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
        // blocks: at most EXACT_MAX_PER_BLOCK values each (the 16-bit-half counters stay exact)
        int64_t nb = grid_for(n, BLOCK, (int64_t)ctx->num_sms * 8);
        const int64_t need = (n + EXACT_MAX_PER_BLOCK - 1) / EXACT_MAX_PER_BLOCK;
        if (nb < need) nb = need;
        k_exact_accum<<<(unsigned)nb, BLOCK, 0, s>>>(
            d_x, n, d_mask_or_null, d_acc, d_cnt, d_bad);
        check_launch("k_exact_accum");
        count_launch(ctx);
    }
    k_exact_finish<<<1, 32, 0, s>>>(d_acc, d_cnt, d_mean_out, d_count_out, d_bad, d_bad_out);
    check_launch("k_exact_finish");
    count_launch(ctx);
}

}  // namespace hm
