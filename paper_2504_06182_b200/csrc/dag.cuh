// Occupancy DAG kernels (dag.cu).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

namespace rb {

struct DagArgs {
    int W, H, P;
    const int32_t *src, *dst;        // device, P one-bend paths
    int32_t *source_of, *target_of;  // device, W*H each
    int32_t *cnt;                    // device, P
    int64_t *off;                    // device, P+1
    unsigned long long *keys, *keys_alt;  // device, max edges each
    void *temp;
    size_t temp_bytes;
};

size_t dag_temp_bytes(int64_t max_edges, int P);
// counts edges (synchronizes the stream)
cudaError_t dag_count(const DagArgs &d, cudaStream_t st, int64_t *n_edges_host);
// writes the sorted edge list into device arrays ea/eb
cudaError_t dag_emit(const DagArgs &d, int64_t n_edges, cudaStream_t st, int32_t *ea, int32_t *eb);

}  // namespace rb
