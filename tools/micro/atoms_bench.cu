// Microbenchmark: shared-memory atomicOr / atomicXor / plain load+store
// throughput per SM on random word indices (the window replay's bitmap ops).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 atoms_bench.cu -o atoms_bench
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(unsigned *out, int iters) {
    __shared__ unsigned bm[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    unsigned x = threadIdx.x * 2654435761u + blockIdx.x, acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x = x * 1664525u + 1013904223u;
            const unsigned w = (x >> 8) & 8191, b = 1u << (x & 31);
            if (MODE == 0) acc += atomicOr(&bm[w], b) & b;
            if (MODE == 1) atomicXor(&bm[w], b);
            if (MODE == 2) acc += bm[w] & b;
            if (MODE == 3) bm[w] = acc + u;
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned)(t1 - t0);
    if (acc == 12345) out[1000] = acc;
}

int main() {
    unsigned *d;
    cudaMalloc(&d, 4096 * 4);
    const char *names[] = {"atomicOr(ret)", "atomicXor(noret)", "lds", "sts"};
    for (int bs : {512, 1024}) {
        for (int mode = 0; mode < 4; ++mode) {
            int iters = 1000;
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            auto launch = [&]() {
                if (mode == 0) k<0><<<148 * (2048 / bs), bs>>>(d, iters);
                if (mode == 1) k<1><<<148 * (2048 / bs), bs>>>(d, iters);
                if (mode == 2) k<2><<<148 * (2048 / bs), bs>>>(d, iters);
                if (mode == 3) k<3><<<148 * (2048 / bs), bs>>>(d, iters);
            };
            launch();
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double ops_per_sm = 2048.0 * iters * 8;  // lane-ops per SM
            const double cyc = ms * 1e-3 * 1.9e9;
            printf("bs %d %-18s %.3f ms  %.2f lane-ops/cycle/SM  (%.1f cycles per warp-instr)\n", bs, names[mode], ms,
                   ops_per_sm / cyc, cyc / (ops_per_sm / 32));
        }
    }
    return 0;
}
