// levelmix inside a persistent cooperative kernel (grid.sync per level) vs one launch per level;
// 3 rotating frontier arrays (own F_{d-1}, F_{d-2} reads + gathers + F_d write), as in MS-BFS v5/v6
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;
struct Args { uint4 *F[3]; const int *nbr; int nrows; int levels; int own; };
__device__ __forceinline__ void level(const Args &a, int d) {
  const int lane = threadIdx.x & 31, tl = lane & 7;
  const long team = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const long nteams = ((long)gridDim.x * blockDim.x) >> 3;
  const uint4 *Fc = a.F[(d + 2) % 3], *Fp = a.F[(d + 1) % 3]; uint4 *Fn = a.F[d % 3];
  for (long v = team; v < a.nrows; v += nteams) {
    uint4 acc = make_uint4(0,0,0,0), x[8], o1 = acc, o2 = acc;
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = Fc[(long)a.nbr[v * 8 + q] * 8 + tl];
    if (a.own) { o1 = Fc[v * 8 + tl]; o2 = Fp[v * 8 + tl]; }
#pragma unroll
    for (int q = 0; q < 8; ++q) { acc.x |= x[q].x; acc.y |= x[q].y; acc.z |= x[q].z; acc.w |= x[q].w; }
    Fn[v * 8 + tl] = make_uint4(acc.x & ~(o1.x | o2.x), acc.y & ~(o1.y | o2.y), acc.z & ~(o1.z | o2.z), acc.w & ~(o1.w | o2.w));
  }
}
__global__ void k_persist(Args a) { cg::grid_group g = cg::this_grid(); for (int d = 1; d <= a.levels; ++d) { level(a, d); g.sync(); } }
__global__ void k_one(Args a, int d) { level(a, d); }
int main() {
  const int nrows = 262144;
  Args a; for (int i = 0; i < 3; ++i) { cudaMalloc(&a.F[i], nrows * 128L); cudaMemset(a.F[i], 0x11 * (i + 1), nrows * 128L); }
  int *nbr; cudaMalloc(&nbr, nrows * 8 * 4L);
  int *h = new int[nrows * 8]; unsigned s = 1; for (long i = 0; i < nrows * 8L; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) % nrows; }
  cudaMemcpy(nbr, h, nrows * 8 * 4L, cudaMemcpyHostToDevice);
  a.nbr = nbr; a.nrows = nrows; a.levels = 40;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int own : {0, 1}) for (int bps : {2, 4}) {
    a.own = own; const int blocks = 148 * bps;
    void *args[] = {&a};
    cudaLaunchCooperativeKernel((void *)k_persist, blocks, 512, args, 0, 0); cudaDeviceSynchronize();
    cudaEventRecord(e0); cudaLaunchCooperativeKernel((void *)k_persist, blocks, 512, args, 0, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaEventRecord(e0); for (int d = 1; d <= a.levels; ++d) k_one<<<blocks, 512>>>(a, d); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms2; cudaEventElapsedTime(&ms2, e0, e1);
    printf("own=%d blocks/SM %d: persistent+grid.sync %.1f us/level | launch per level %.1f us/level  [%s]\n", own, bps, ms * 1000 / a.levels, ms2 * 1000 / a.levels, cudaGetErrorString(cudaGetLastError()));
  }
}
