// random 128-B row gathers into shared memory: cp.async (16 B/lane) vs cp.async.bulk (128 B/lane) vs LDG
#include <cstdio>
#include <cstdint>
#define ROWS_PER_WARP 64
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k_cpasync(const uint4 *__restrict__ F, long nrows, int iters, uint4 *out) {
  extern __shared__ uint4 sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint4 *buf = sm + w * ROWS_PER_WARP * 8;
  unsigned s = (blockIdx.x * 1024 + threadIdx.x) * 2654435761u;
  uint4 acc = make_uint4(0,0,0,0);
  for (int it = 0; it < iters; ++it) {
    // 64 rows x 8 chunks = 512 copies, 16 per lane; lane -> (row = idx/8, chunk = idx%8)
    for (int k = 0; k < 16; ++k) {
      const int idx = k * 32 + lane, row = idx >> 3, ch = idx & 7;
      unsigned r = __shfl_sync(0xffffffff, (s = s * 1664525u + 1013904223u), (idx >> 3) & 31);
      const uint4 *src = F + (long)(r % (unsigned)nrows) * 8 + ch;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_u32(buf + row * 8 + ch)), "l"(src));
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    for (int k = 0; k < 16; ++k) { uint4 x = buf[k * 32 + lane]; acc.x |= x.x; acc.y ^= x.y; }
    __syncwarp();
  }
  if ((acc.x ^ acc.y) == 0x12345678) out[0] = acc;
}
__global__ void k_bulk(const uint4 *__restrict__ F, long nrows, int iters, uint4 *out) {
  extern __shared__ uint4 sm[];
  __shared__ uint64_t mbar[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint4 *buf = sm + w * ROWS_PER_WARP * 8;
  if (lane == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(smem_u32(&mbar[w])));
  __syncwarp();
  unsigned s = (blockIdx.x * 1024 + threadIdx.x) * 2654435761u;
  uint4 acc = make_uint4(0,0,0,0);
  unsigned phase = 0;
  for (int it = 0; it < iters; ++it) {
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(smem_u32(&mbar[w])), "r"(ROWS_PER_WARP * 128));
    __syncwarp();
    for (int k = 0; k < ROWS_PER_WARP / 32; ++k) {
      const int row = k * 32 + lane;
      s = s * 1664525u + 1013904223u;
      const uint4 *src = F + (long)(s % (unsigned)nrows) * 8;
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];"
                   :: "r"(smem_u32(buf + row * 8)), "l"(src), "r"(smem_u32(&mbar[w])) : "memory");
    }
    // wait
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" :: "r"(smem_u32(&mbar[w])), "r"(phase) : "memory");
    phase ^= 1;
    for (int k = 0; k < 16; ++k) { uint4 x = buf[k * 32 + lane]; acc.x |= x.x; acc.y ^= x.y; }
    __syncwarp();
  }
  if ((acc.x ^ acc.y) == 0x12345678) out[0] = acc;
}
__global__ void k_ldg(const uint4 *__restrict__ F, long nrows, int iters, uint4 *out) {
  const int lane = threadIdx.x & 31, tl = lane & 7;
  unsigned s = (blockIdx.x * 1024 + threadIdx.x) * 2654435761u;
  uint4 acc = make_uint4(0,0,0,0);
  for (int it = 0; it < iters * ROWS_PER_WARP / 16; ++it) {
    uint4 x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) { unsigned r = __shfl_sync(0xffffffff, (s = s * 1664525u + 1013904223u), lane & ~7); x[q] = F[(long)(r % (unsigned)nrows) * 8 + tl]; }
#pragma unroll
    for (int q = 0; q < 4; ++q) { acc.x |= x[q].x; acc.y ^= x[q].y; }
  }
  if ((acc.x ^ acc.y) == 0x12345678) out[0] = acc;
}
int main() {
  uint4 *F, *out; const long nrows = 262144; cudaMalloc(&F, nrows * 128); cudaMemset(F, 1, nrows * 128); cudaMalloc(&out, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 64;
  for (int threads : {256, 512}) for (int bps : {1, 2}) {
    const int blocks = 148 * bps; const int smem = (threads / 32) * ROWS_PER_WARP * 128;
    cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const double bytes = (double)blocks * (threads / 32) * ROWS_PER_WARP * 128.0 * iters;
    float ms;
    k_cpasync<<<blocks, threads, smem>>>(F, nrows, iters, out);
    cudaEventRecord(e0); k_cpasync<<<blocks, threads, smem>>>(F, nrows, iters, out); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("threads %d bps %d smem %dKB: cp.async %.0f GB/s", threads, bps, smem / 1024, bytes / ms / 1e6);
    k_bulk<<<blocks, threads, smem>>>(F, nrows, iters, out);
    cudaEventRecord(e0); k_bulk<<<blocks, threads, smem>>>(F, nrows, iters, out); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf(" | bulk %.0f GB/s", bytes / ms / 1e6);
    k_ldg<<<blocks, threads>>>(F, nrows, iters, out);
    cudaEventRecord(e0); k_ldg<<<blocks, threads>>>(F, nrows, iters, out); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf(" | ldg(4 in flight/team) %.0f GB/s  [%s]\n", bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
}
