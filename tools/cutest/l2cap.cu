// effective L2 capacity for random 128-B row gathers: bandwidth vs array size
#include <cstdio>
#include <cstdint>
__global__ void k_gather(const uint4 *__restrict__ F, long nrows, long iters, uint4 *out, unsigned seed) {
  const int lane = threadIdx.x & 31, tl = lane & 7;
  const long team = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  uint4 acc = make_uint4(0, 0, 0, 0);
  unsigned s = seed ^ (unsigned)(team * 2654435761u);
  for (long k = 0; k < iters; k += 4) {
    uint4 x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) { s = s * 1664525u + 1013904223u; long r = (long)((s >> 4) % (unsigned)nrows); x[q] = F[r * 8 + tl]; }
#pragma unroll
    for (int q = 0; q < 4; ++q) { acc.x |= x[q].x; acc.y ^= x[q].y; }
  }
  if ((acc.x ^ acc.y) == 0x12345678) out[0] = acc;
}
int main() {
  uint4 *F, *out; size_t maxb = 256ull << 20;
  cudaMalloc(&F, maxb); cudaMemset(F, 1, maxb); cudaMalloc(&out, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 4, threads = 512; const long teams = (long)blocks * threads / 8; const long iters = 256;
  for (int mb : {8, 16, 24, 32, 40, 48, 56, 64, 80, 96, 112, 128, 160, 256}) {
    long nrows = ((long)mb << 20) / 128;
    k_gather<<<blocks, threads>>>(F, nrows, iters, out, 1);
    cudaEventRecord(e0);
    k_gather<<<blocks, threads>>>(F, nrows, iters, out, 7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("array %4d MB: %7.1f GB/s (%.3f ms)\n", mb, teams * iters * 128.0 / ms / 1e6, ms);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
