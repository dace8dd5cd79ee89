// grid barrier cost: CG grid.sync vs a monotonic-counter barrier
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned ld_acq(const unsigned *p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__global__ void k_cg(int n, int *out) { cg::grid_group g = cg::this_grid(); int x = 0; for (int i = 0; i < n; ++i) { x += threadIdx.x; g.sync(); } if (x == 12345) *out = x; }
__global__ void k_my(int n, unsigned *bar, int *out) {
  unsigned gen = 0; int x = 0;
  for (int i = 0; i < n; ++i) {
    x += threadIdx.x;
    __syncthreads(); ++gen;
    if (threadIdx.x == 0) { __threadfence(); unsigned t = gen * gridDim.x; unsigned a = atomicAdd(bar, 1u) + 1u;
      if (a == t) { atomicExch(bar + 1, gen); } else { while (ld_acq(bar + 1) < gen) { } } }
    __syncthreads();
  }
  if (x == 12345) *out = x;
}
int main() {
  int *out; unsigned *bar; cudaMalloc(&out, 4); cudaMalloc(&bar, 8);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int bps : {1, 2}) for (int threads : {256, 512}) {
    int grid = nsm * bps; int n = 20000;
    void *args1[] = {&n, &out};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args1, 0, 0); cudaDeviceSynchronize();
    cudaEventRecord(e0); cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args1, 0, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemset(bar, 0, 8);
    void *args2[] = {&n, &bar, &out};
    cudaEventRecord(e0); cudaLaunchCooperativeKernel((void*)k_my, grid, threads, args2, 0, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms2; cudaEventElapsedTime(&ms2, e0, e1);
    printf("grid %d x %d: cg %.3f us/sync, custom %.3f us/sync (%s)\n", grid, threads, ms * 1000 / n, ms2 * 1000 / n, cudaGetErrorString(cudaGetLastError()));
  }
}
