// L2 random row-gather bandwidth: teams of T lanes each load one R-byte row (16 B per lane)
#include <cstdio>
#include <cstdint>
template <int T, int U>
__global__ void k_gather(const uint4 *__restrict__ F, const int *__restrict__ idx, int n, int rows_per_team, uint4 *out) {
  const int lane = threadIdx.x & 31, tl = lane % T;
  const long team = ((long)blockIdx.x * blockDim.x + threadIdx.x) / T;
  uint4 acc = make_uint4(0, 0, 0, 0);
  const int *ip = idx + team * rows_per_team;
  for (int k = 0; k < rows_per_team; k += U) {
    uint4 x[U];
#pragma unroll
    for (int q = 0; q < U; ++q) x[q] = F[(long)ip[k + q] * T + tl];
#pragma unroll
    for (int q = 0; q < U; ++q) { acc.x |= x[q].x; acc.y |= x[q].y; acc.z |= x[q].z; acc.w |= x[q].w; }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678) out[0] = acc;
}
int main() {
  const int nrows = 262144; 
  for (int T : {8, 16}) {
    const int R = T * 16;
    uint4 *F, *out; int *idx;
    cudaMalloc(&F, (size_t)nrows * R); cudaMemset(F, 1, (size_t)nrows * R); cudaMalloc(&out, 64);
    const int blocks = 148 * 4, threads = 512, teams = blocks * threads / T, rpt = 64;
    const long nidx = (long)teams * rpt;
    int *h = new int[nidx]; unsigned s = 12345; for (long i = 0; i < nidx; ++i) { s = s * 1664525u + 1013904223u; h[i] = s % nrows; }
    cudaMalloc(&idx, nidx * 4); cudaMemcpy(idx, h, nidx * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int u : {1, 4, 8}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (T == 8) { if (u == 1) k_gather<8,1><<<blocks, threads>>>(F, idx, nrows, rpt, out); else if (u == 4) k_gather<8,4><<<blocks, threads>>>(F, idx, nrows, rpt, out); else k_gather<8,8><<<blocks, threads>>>(F, idx, nrows, rpt, out); }
        else { if (u == 1) k_gather<16,1><<<blocks, threads>>>(F, idx, nrows, rpt, out); else if (u == 4) k_gather<16,4><<<blocks, threads>>>(F, idx, nrows, rpt, out); else k_gather<16,8><<<blocks, threads>>>(F, idx, nrows, rpt, out); }
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("T=%d row=%dB unroll=%d: %.1f GB/s gathered (%.2f ms, array %.1f MB)\n", T, R, u, (double)nidx * R / ms / 1e6, ms, nrows * R / 1e6);
      }
    }
    cudaFree(F); cudaFree(idx); delete[] h;
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
