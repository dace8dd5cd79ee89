// Bare memory pattern of one dense MS-BFS level on a C5-like layer (V = 262144 rows, 8 random
// neighbours per row), W = 64 (512-B rows, 134 MB per array) vs the same level split into two
// half-row passes (256-B halves, a 67 MB gathered working set per pass).  16 lanes per row,
// 2 x 16 B per lane; own F_{d-1} / F_{d-2} reads and the F_d write included.
#include <cstdio>
#include <cstdint>
template <int HALVES>
__global__ void k_level(const uint4 *__restrict__ Fc, const uint4 *__restrict__ Fp, uint4 *Fn,
                        const int *__restrict__ nbr, int nrows, int pass) {
  const int lane = threadIdx.x & 31, tl = lane & 15;
  const long team = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 4;
  const long nteams = ((long)gridDim.x * blockDim.x) >> 4;
  constexpr int CH = 32 / HALVES;                // 16-B chunks per row handled in this pass
  constexpr int VEC = CH / 16;                   // chunks per lane
  for (long v = team; v < nrows; v += nteams) {
    uint4 acc[VEC], own[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) { acc[q] = make_uint4(0, 0, 0, 0); }
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      uint4 x0[VEC], x1[VEC];
      const long u0 = nbr[v * 8 + k], u1 = nbr[v * 8 + k + 1];
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        x0[q] = Fc[u0 * 32 + pass * CH + q * 16 + tl];
        x1[q] = Fc[u1 * 32 + pass * CH + q * 16 + tl];
      }
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        acc[q].x |= x0[q].x | x1[q].x; acc[q].y |= x0[q].y | x1[q].y;
        acc[q].z |= x0[q].z | x1[q].z; acc[q].w |= x0[q].w | x1[q].w;
      }
    }
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      const uint4 a = Fc[v * 32 + pass * CH + q * 16 + tl], b = Fp[v * 32 + pass * CH + q * 16 + tl];
      own[q] = make_uint4(a.x | b.x, a.y | b.y, a.z | b.z, a.w | b.w);
      Fn[v * 32 + pass * CH + q * 16 + tl] = make_uint4(acc[q].x & ~own[q].x, acc[q].y & ~own[q].y,
                                                        acc[q].z & ~own[q].z, acc[q].w & ~own[q].w);
    }
  }
}
int main() {
  const int nrows = 262144;
  uint4 *F[3]; int *nbr;
  for (int i = 0; i < 3; ++i) { cudaMalloc(&F[i], nrows * 512L); cudaMemset(F[i], 0x11 * (i + 1), nrows * 512L); }
  cudaMalloc(&nbr, nrows * 8 * 4L);
  int *h = new int[nrows * 8L]; unsigned s = 7;
  for (long i = 0; i < nrows * 8L; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) % nrows; }
  cudaMemcpy(nbr, h, nrows * 8 * 4L, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bps : {2, 3, 4}) {
    const int blocks = 148 * bps, threads = 448;
    float best1 = 1e9, best2 = 1e9, ms;
    for (int rep = 0; rep < 6; ++rep) {
      const int d = rep % 3;
      cudaEventRecord(e0);
      k_level<1><<<blocks, threads>>>(F[(d + 2) % 3], F[(d + 1) % 3], F[d], nbr, nrows, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best1) best1 = ms;
      cudaEventRecord(e0);
      k_level<2><<<blocks, threads>>>(F[(d + 2) % 3], F[(d + 1) % 3], F[d], nbr, nrows, 0);
      k_level<2><<<blocks, threads>>>(F[(d + 2) % 3], F[(d + 1) % 3], F[d], nbr, nrows, 1);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best2) best2 = ms;
    }
    const double gb = nrows * (8 + 3) * 512.0 / 1e9;
    printf("blocks/SM %d: one pass %.1f us (%.0f GB/s of row traffic), two half passes %.1f us (%.0f GB/s)\n",
           bps, best1 * 1e3, gb / (best1 / 1e3), best2 * 1e3, gb / (best2 / 1e3));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
