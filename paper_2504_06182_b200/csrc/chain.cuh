// Chain (exact 1D) kernels: chain.cu (band mode, warp per chain) and
// chain_general.cu (arbitrary targets, one CTA).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rb {

struct ChainBandParams {
    const uint64_t *occ;  // count chains, (n+63)/64 words each
    int count, n, t_lo, t_hi;
    int32_t *path_src, *path_dst;  // [count * k]
    int64_t *total_displacement;
    int32_t *displaced, *status, *detail;
    int32_t *use_first;  // optional: index of the first used sorted source
    int b_off, be_off, hole_off, warp_smem;  // set by launch_chain_band
};

cudaError_t launch_chain_band(const ChainBandParams &p, int sms, cudaStream_t st);

// General assignment on sorted inputs (device arrays).  Sources carry
// [min_use, max_use] and a position; chains use {0, 1}.  Blocks: when
// `certify` is set the reference's candidate/certified blocks
// (exact1d.cpp:219-297) are applied (chain mode: sources are vertices).
struct ChainGeneralParams {
    int n;                   // chain length (chain mode)
    int ns, nt;
    const int64_t *pos;      // [ns] ascending
    const int32_t *min_use;  // [ns] (nullptr = 0)
    const int32_t *max_use;  // [ns] (nullptr = 1)
    const int64_t *tgt;      // [nt] ascending
    int certify;             // chain mode: candidate + certified blocks
    // workspace (device)
    int64_t *dp_a, *dp_b, *cprefix;  // [nt + 1] each
    uint16_t *choice;                // [max block sources * (nt + 1)] run length per cell
    int32_t *blocks;                 // [4 * (n + 2)] (s0, s1, t0, t1)
    int64_t *wts;                    // [n + 2] block costs
    int32_t *scratch;                // [n + 2]
    // outputs
    int32_t *use;                    // [ns]
    int64_t *pair_src, *pair_dst;    // [nt]
    int64_t *weight;                 // [1]
    int32_t *status;                 // [1]
};

cudaError_t launch_chain_general(const ChainGeneralParams &p, cudaStream_t st);

// solve_1d tail on device: paths are the matching pairs in target order.
// Writes path_order (rights by target desc, lefts asc, isolated by index,
// exact1d.cpp:494-515) and the span-overlap DAG in the reference's emission
// order (exact1d.cpp:529-560).
struct ChainOrderParams {
    int P;
    const int32_t *src, *dst;   // device [P]
    int32_t *order;             // [P]
    int32_t *rank;              // [P] scratch
    unsigned long long *keys_a, *keys_b;  // [P] scratch
    int64_t *cnt;               // [P + 1] scratch
    int32_t *sweep_id;          // [P] span id at sweep position
    int32_t *q_pos;             // [P] sweep positions sorted by (hi, pos)
    int64_t *q_hi;              // [P]
    int32_t *ea, *eb;           // [edges]
    void *temp;
    size_t temp_bytes;
};

size_t chain_order_temp_bytes(int P);
cudaError_t chain_order_count(const ChainOrderParams &p, cudaStream_t st, int64_t *n_edges);
cudaError_t chain_order_emit(const ChainOrderParams &p, cudaStream_t st);

}  // namespace rb
