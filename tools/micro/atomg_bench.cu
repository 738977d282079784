// Microbenchmark: global atomics on random addresses in an L2-resident array
// (the window plan's blocker decrements), per-SM throughput.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 atomg_bench.cu -o atomg_bench
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE, int U>
__global__ void k(int *arr, unsigned n, int iters, int *sink) {
    unsigned x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
    int acc = 0;
    for (int it = 0; it < iters; ++it) {
        int r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            x = x * 1664525u + 1013904223u;
            const unsigned i = (x >> 4) % n;
            if (MODE == 0) r[u] = atomicSub(&arr[i], 1);          // ATOM with return
            if (MODE == 1) { atomicAdd(&arr[i], 1); r[u] = 0; }  // RED
            if (MODE == 2) r[u] = __ldcg(&arr[i]);               // load
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += r[u] == 1;
    }
    if (acc == 123456) *sink = acc;
}

int main() {
    const unsigned n = 64u << 20;  // elements spread over 256 MB (L2-miss) or small
    int *arr, *sink;
    cudaMalloc(&arr, (size_t)n * 4);
    cudaMalloc(&sink, 4);
    cudaMemset(arr, 0, (size_t)n * 4);
    const char *names[] = {"ATOM ret", "RED", "LDG.cg"};
    for (unsigned span : {150000u, 64u << 20}) {
        for (int blocks_per_sm : {1, 2, 4}) {
            for (int mode = 0; mode < 3; ++mode) {
                const int bs = 512, iters = 200;
                const int grid = 148 * blocks_per_sm;
                auto launch = [&]() {
                    if (mode == 0) k<0, 8><<<grid, bs>>>(arr, span, iters, sink);
                    if (mode == 1) k<1, 8><<<grid, bs>>>(arr, span, iters, sink);
                    if (mode == 2) k<2, 8><<<grid, bs>>>(arr, span, iters, sink);
                };
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                launch();
                cudaEventRecord(a);
                launch();
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double lane_ops = (double)grid * bs * iters * 8;
                const double cyc = ms * 1e-3 * 1.9e9;
                printf("span %9u  %d x 512 thr/SM  %-8s %.3f ms  %.3f lane-ops/cycle/SM  chip %.1f G/s\n", span,
                       blocks_per_sm, names[mode], ms, lane_ops / cyc / 148, lane_ops / (ms * 1e-3) / 1e9);
            }
        }
    }
    return 0;
}
