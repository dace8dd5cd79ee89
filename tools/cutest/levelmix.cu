// memory floor of one dense MS-BFS level (W=16): per row 8 random 128-B gathers from F (33.5 MB),
// read+write of its vis row (33.5 MB), write of its new frontier row (33.5 MB)
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint4 ldcs(const uint4 *p) { uint4 v; asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p)); return v; }
__device__ __forceinline__ void stcs(uint4 *p, uint4 v) { asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory"); }
template <int MODE>
__global__ void k_level(const uint4 *__restrict__ F, uint4 *vis, uint4 *Fn, const int *__restrict__ nbr, int nrows, int deg) {
  const int lane = threadIdx.x & 31, tl = lane & 7;
  const long team = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const long nteams = ((long)gridDim.x * blockDim.x) >> 3;
  for (long v = team; v < nrows; v += nteams) {
    uint4 acc = make_uint4(0,0,0,0), x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = (q < deg) ? F[(long)nbr[v * 8 + q] * 8 + tl] : make_uint4(0,0,0,0);
    uint4 vv = make_uint4(0,0,0,0);
    if (MODE >= 1) vv = (MODE == 2) ? ldcs(vis + v * 8 + tl) : vis[v * 8 + tl];
#pragma unroll
    for (int q = 0; q < 8; ++q) { acc.x |= x[q].x; acc.y |= x[q].y; acc.z |= x[q].z; acc.w |= x[q].w; }
    uint4 nw = make_uint4(acc.x & ~vv.x, acc.y & ~vv.y, acc.z & ~vv.z, acc.w & ~vv.w);
    if (MODE >= 1) { uint4 nv = make_uint4(vv.x | nw.x, vv.y | nw.y, vv.z | nw.z, vv.w | nw.w); if (MODE == 2) stcs(vis + v * 8 + tl, nv); else vis[v * 8 + tl] = nv; }
    Fn[v * 8 + tl] = nw;
  }
}
int main() {
  const int nrows = 262144;
  uint4 *F, *vis, *Fn; int *nbr;
  cudaMalloc(&F, nrows * 128L); cudaMalloc(&vis, nrows * 128L); cudaMalloc(&Fn, nrows * 128L); cudaMalloc(&nbr, nrows * 8 * 4L);
  cudaMemset(F, 0x11, nrows * 128L); cudaMemset(vis, 0, nrows * 128L);
  int *h = new int[nrows * 8]; unsigned s = 1; for (long i = 0; i < nrows * 8L; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) % nrows; }
  cudaMemcpy(nbr, h, nrows * 8 * 4L, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bps : {2, 4}) for (int mode : {0, 1, 2}) {
    const int blocks = 148 * bps, threads = 512;
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k_level<0><<<blocks, threads>>>(F, vis, Fn, nbr, nrows, 8);
      if (mode == 1) k_level<1><<<blocks, threads>>>(F, vis, Fn, nbr, nrows, 8);
      if (mode == 2) k_level<2><<<blocks, threads>>>(F, vis, Fn, nbr, nrows, 8);
      cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      uint4 *t = F; F = Fn; Fn = t;
    }
    printf("blocks/SM %d mode %d (0: gathers+Fn, 1: +vis rw, 2: +vis rw .cs): %.1f us per level\n", bps, mode, best * 1000);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
