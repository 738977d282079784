// Microbenchmark: dependent-access latency (one warp, lane 0 chases a random
// permutation) for loads and atomics over buffers of different sizes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 lat_bench.cu -o lat_bench
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void chase(const unsigned *next, int steps, unsigned *out, long long *cyc, int mode, unsigned *acc,
                      unsigned start) {
    unsigned p = start;
    long long t0 = clock64();
    for (int i = 0; i < steps; ++i) {
        if (mode == 0) p = __ldg(next + p);
        else if (mode == 1) p = __ldcg(next + p);
        else p = atomicAdd(acc + p, 0u) ^ 0u, p = next[p];  // atomic then load (2 dependent)
    }
    long long t1 = clock64();
    *out = p;
    *cyc = t1 - t0;
}

int main() {
    for (size_t mb : {16, 256, 2048, 16384}) {
        const size_t n = mb * (1u << 20) / 4;
        std::vector<unsigned> h(n);
        // random cycle with stride >= 4 KB jumps
        std::vector<unsigned> perm(n / 1024);
        for (size_t i = 0; i < perm.size(); ++i) perm[i] = (unsigned)i;
        srand(1);
        for (size_t i = perm.size() - 1; i > 0; --i) std::swap(perm[i], perm[rand() % (i + 1)]);
        for (size_t i = 0; i < perm.size(); ++i) h[(size_t)perm[i] * 1024] = perm[(i + 1) % perm.size()] * 1024;
        unsigned *d, *o, *acc;
        long long *c;
        if (cudaMalloc(&d, n * 4) != cudaSuccess) { printf("alloc %zu MB failed\n", mb); continue; }
        cudaMalloc(&acc, n * 4);
        cudaMemset(acc, 0, n * 4);
        cudaMalloc(&o, 4);
        cudaMalloc(&c, 8);
        cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
        const char *nm[] = {"ldg", "ldcg", "atom+ld"};
        unsigned start = 0;
        for (int mode = 0; mode < 3; ++mode) {
            const int steps = 2000;
            start = h[start];
            for (int k = 0; k < 3000; ++k) start = h[start];  // a fresh part of the cycle
            chase<<<1, 1>>>(d, steps, o, c, mode, acc, start);
            long long cy, cw;
            cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
            chase<<<1, 1>>>(d, steps, o, c, mode, acc, start);  // again: warm in L2
            cudaMemcpy(&cw, c, 8, cudaMemcpyDeviceToHost);
            printf("%6zu MB  %-8s cold %.0f  warm %.0f cycles per step\n", mb, nm[mode], (double)cy / steps,
                   (double)cw / steps);
        }
        cudaFree(d); cudaFree(acc); cudaFree(o); cudaFree(c);
    }
    return 0;
}
