// Memory-pattern floor of one dense level of the visited-set MS-BFS (round 2) on a C5-sized layer:
// V = 262144 rows of 512 B (W = 64), every row gathers G random neighbour rows from the gathered
// buffer Fc, reads its own row (Fc too: at a dense level every row changed at d-1) and writes its
// new row into Fn -- no scan, staging, sorting or bookkeeping.  16-lane teams, 2 x 16 B per lane,
// 4 rows in flight per lane, 2 CTAs x 448 threads per SM: the access pattern of msbfs_kernel's
// light path.  Also the same pattern on a buffer that fits L2 (pure L2 gather throughput).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o level_floor level_floor.cu && ./level_floor
#include <cstdio>
#include <cstdint>

template <int G>
__global__ void __launch_bounds__(448, 2) k_level(const uint4 *__restrict__ Fc, uint4 *__restrict__ Fn,
                                                  const int *__restrict__ nbr, int nrows) {
  const int lane = threadIdx.x & 31, tl = lane & 15;
  const long team = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 4;
  const long nteams = ((long)gridDim.x * blockDim.x) >> 4;
  for (long v = team; v < nrows; v += nteams) {
    uint4 acc[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
    const uint4 o0 = Fc[v * 32 + tl], o1 = Fc[v * 32 + 16 + tl];
#pragma unroll
    for (int k = 0; k < G; k += 4) {
      uint4 x[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long u = nbr[v * G + k + q];
        x[q][0] = Fc[u * 32 + tl];
        x[q][1] = Fc[u * 32 + 16 + tl];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          acc[c].x |= x[q][c].x; acc[c].y |= x[q][c].y; acc[c].z |= x[q][c].z; acc[c].w |= x[q][c].w;
        }
    }
    Fn[v * 32 + tl] = make_uint4(acc[0].x | o0.x, acc[0].y | o0.y, acc[0].z | o0.z, acc[0].w | o0.w);
    Fn[v * 32 + 16 + tl] = make_uint4(acc[1].x | o1.x, acc[1].y | o1.y, acc[1].z | o1.z, acc[1].w | o1.w);
  }
}

int main() {
  const int G = 8;
  for (int nrows : {262144, 32768}) {           // 134 MB per buffer (C5 layer), 16.8 MB (L2-resident)
    uint4 *F[2];
    int *nbr;
    for (int i = 0; i < 2; ++i) {
      cudaMalloc(&F[i], nrows * 512L);
      cudaMemset(F[i], 0x11 * (i + 1), nrows * 512L);
    }
    cudaMalloc(&nbr, (long)nrows * G * 4);
    int *h = new int[(long)nrows * G];
    unsigned s = 7;
    for (long i = 0; i < (long)nrows * G; ++i) {
      s = s * 1664525u + 1013904223u;
      h[i] = (s >> 8) % nrows;
    }
    cudaMemcpy(nbr, h, (long)nrows * G * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9, ms;
    for (int rep = 0; rep < 8; ++rep) {
      // level rep reads the rows level rep - 1 wrote (what L2 still holds of them, as in the kernel)
      cudaEventRecord(e0);
      k_level<G><<<148 * 2, 448>>>(F[rep & 1], F[(rep + 1) & 1], nbr, nrows);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep >= 2 && ms < best) best = ms;
    }
    const double l2b = nrows * (G + 2) * 512.0;     // gathered + own rows read, new rows written
    printf("rows %6d (%.1f MB per buffer), %d gathers per row: %.1f us per level, %.2f TB/s of row traffic\n",
           nrows, nrows * 512.0 / 1e6, G, best * 1e3, l2b / (best / 1e3) / 1e12);
    cudaFree(F[0]);
    cudaFree(F[1]);
    cudaFree(nbr);
    delete[] h;
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
