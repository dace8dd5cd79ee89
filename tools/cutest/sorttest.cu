// standalone check of CUB radix sort as used in closeness.cu
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
int main() {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    int fails = 0;
    for (int V : {1500, 1024, 5000, 262144}) {
        for (int rep = 0; rep < 10; ++rep) {
            std::vector<unsigned long long> h(V);
            for (int i = 0; i < V; ++i) h[i] = i;
            std::shuffle(h.begin(), h.end(), std::mt19937(rep));
            unsigned long long *a, *b; void* t = nullptr;
            cudaMallocAsync(&a, V * 8, s); cudaMallocAsync(&b, V * 8, s);
            cudaMemcpyAsync(a, h.data(), V * 8, cudaMemcpyHostToDevice, s);
            size_t tb = 0; int nb = 0; for (unsigned x = V; x; x >>= 1) ++nb;
            cub::DeviceRadixSort::SortKeys(nullptr, tb, a, b, V, 0, 32 + nb, s);
            cudaMallocAsync(&t, tb, s);
            cub::DeviceRadixSort::SortKeys(t, tb, a, b, V, 0, 32 + nb, s);
            std::vector<unsigned long long> o(V);
            cudaMemcpyAsync(o.data(), b, V * 8, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            int bad = 0; for (int i = 0; i < V; ++i) bad += (o[i] != (unsigned long long)i);
            if (bad) { ++fails; printf("V=%d rep=%d bad=%d\n", V, rep, bad); }
            cudaFreeAsync(a, s); cudaFreeAsync(b, s); cudaFreeAsync(t, s);
        }
    }
    printf("sort fails %d  (%s)\n", fails, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
