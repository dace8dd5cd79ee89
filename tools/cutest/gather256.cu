// random 256-B row gathers (the MS-BFS F_{d-1} pattern at W=32): cp.async.bulk into smem
// (double-buffered, mbarrier) vs LDG (16 lanes x 16 B per row, D rows in flight per team)
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int RPW>
__global__ void k_bulk(const uint4 *__restrict__ F, long nrows, int iters, uint4 *out) {
  extern __shared__ uint4 sm[];
  __shared__ uint64_t mbar[32][2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint4 *buf = sm + w * 2 * RPW * 16;
  if (lane == 0) { asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(smem_u32(&mbar[w][0]))); asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(smem_u32(&mbar[w][1]))); }
  __syncwarp();
  unsigned s = (blockIdx.x * 1024 + threadIdx.x) * 2654435761u;
  uint4 acc = make_uint4(0,0,0,0);
  auto issue = [&](int b) {
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(smem_u32(&mbar[w][b])), "r"(RPW * 256));
    __syncwarp();
    for (int k = 0; k < RPW / 32; ++k) {
      const int row = k * 32 + lane;
      s = s * 1664525u + 1013904223u;
      const uint4 *src = F + (long)(s % (unsigned)nrows) * 16;
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                   :: "r"(smem_u32(buf + (b * RPW + row) * 16)), "l"(src), "r"(smem_u32(&mbar[w][b])) : "memory");
    }
  };
  unsigned ph[2] = {0, 0};
  issue(0);
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    if (it + 1 < iters) issue(b ^ 1);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" :: "r"(smem_u32(&mbar[w][b])), "r"(ph[b]) : "memory");
    ph[b] ^= 1;
    for (int k = 0; k < RPW / 2; ++k) { uint4 x = buf[(b * RPW) * 16 + k * 32 + lane]; acc.x |= x.x; acc.y ^= x.y; }
    __syncwarp();
  }
  if ((acc.x ^ acc.y) == 0x12345678) out[0] = acc;
}
template <int D>
__global__ void k_ldg(const uint4 *__restrict__ F, long nrows, int iters, uint4 *out) {
  const int lane = threadIdx.x & 31, tl = lane & 15;
  unsigned s = (blockIdx.x * 1024 + threadIdx.x) * 2654435761u;
  uint4 acc = make_uint4(0,0,0,0);
  for (int it = 0; it < iters; ++it) {
    uint4 x[D];
#pragma unroll
    for (int q = 0; q < D; ++q) { unsigned r = __shfl_sync(0xffffffff, (s = s * 1664525u + 1013904223u), lane & ~15); x[q] = F[(long)(r % (unsigned)nrows) * 16 + tl]; }
#pragma unroll
    for (int q = 0; q < D; ++q) { acc.x |= x[q].x; acc.y ^= x[q].y; }
  }
  if ((acc.x ^ acc.y) == 0x12345678) out[0] = acc;
}
int main() {
  uint4 *F, *out; const long maxrows = 1L << 20; cudaMalloc(&F, maxrows * 256); cudaMemset(F, 1, maxrows * 256); cudaMalloc(&out, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (long nrows : {131072L, 262144L, 524288L}) {
    printf("footprint %ld MB\n", nrows * 256 >> 20);
    for (int threads : {256, 512}) {
      const int blocks = 148;
      {  // bulk, RPW=32 rows per stage per warp, 2 stages
        const int smem = (threads / 32) * 2 * 32 * 256; const int iters = 256;
        cudaFuncSetAttribute(k_bulk<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_bulk<32><<<blocks, threads, smem>>>(F, nrows, iters, out);
        cudaEventRecord(e0); k_bulk<32><<<blocks, threads, smem>>>(F, nrows, iters, out); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("  threads %d bulk32x2 (smem %d KB): %.0f GB/s [%s]\n", threads, smem >> 10, (double)blocks * threads / 32 * 32 * 256.0 * iters / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
      if (threads == 256) {
        const int smem = (threads / 32) * 2 * 64 * 256; const int iters = 128;
        cudaFuncSetAttribute(k_bulk<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_bulk<64><<<blocks, threads, smem>>>(F, nrows, iters, out);
        cudaEventRecord(e0); k_bulk<64><<<blocks, threads, smem>>>(F, nrows, iters, out); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("  threads %d bulk64x2 (smem %d KB): %.0f GB/s [%s]\n", threads, smem >> 10, (double)blocks * threads / 32 * 64 * 256.0 * iters / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
      for (int bps : {1, 2, 4}) {
        const int iters = 1024;
        k_ldg<4><<<blocks * bps, threads>>>(F, nrows, iters, out);
        cudaEventRecord(e0); k_ldg<4><<<blocks * bps, threads>>>(F, nrows, iters, out); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        double b4 = (double)blocks * bps * threads / 16 * 4 * 256.0 * iters / ms / 1e6;
        k_ldg<8><<<blocks * bps, threads>>>(F, nrows, iters, out);
        cudaEventRecord(e0); k_ldg<8><<<blocks * bps, threads>>>(F, nrows, iters, out); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        double b8 = (double)blocks * bps * threads / 16 * 8 * 256.0 * iters / ms / 1e6;
        printf("  threads %d x %d blk/SM ldg D=4 %.0f GB/s, D=8 %.0f GB/s [%s]\n", threads, bps, b4, b8, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
}
