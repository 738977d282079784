// batch_moves kernels (batching.cu) and the fused solve -> DAG -> batching
// pipeline (pipeline.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rb {

// per-instance device scratch of the batching warp
struct BatchScratch {
    uint32_t *occ;      // W*H bits (vertex id), initialised from the sources
    uint32_t *inb;      // W*H bits, zero
    int32_t *next;      // [P]
    int32_t *blockers;  // [P] initialised to the in-degree
    uint8_t *done;      // [P]
    int32_t *ready, *ready2, *newly, *mem, *mfr, *mto;  // [P] each
    int32_t *counter;   // [1], zero
    uint32_t *blk_sm;   // pipeline: blocker counts in shared memory (u16 pairs), or null
    int32_t *newly_sm;  // pipeline leap mode: the warp's shared buffer of released ids
};

constexpr int NEWLY_SM = 128;  // released ids per warp kept in shared memory (leap mode)

struct PipeRecords {  // one instance's ready records (batch_warp_pipe)
    int4 *rec, *rec2;
    int32_t *rb, *rb2;
};

struct BatchJob {
    int P, W, H, preset, edge_level;
    const int64_t *soff;  // [P+1] successor CSR offsets (global edge index)
    const int32_t *succ;
    const int4 *prec;     // pipeline: [P+1] {xs|ys<<16, xt|yt<<16, move base, soff - e0} per path
    int64_t e0;           // pipeline: soff[0]
    const int32_t *slen;  // pipeline (global DAG walk): list lengths, p's list = [soff[p], soff[p] + slen[p]);
                          // null: [soff[p], soff[p + 1])
    const int64_t *in_off;  // edge-level only: incoming CSR
    const int32_t *in_src;
    const int64_t *in_need;
    BatchScratch s;
    int32_t *move_batch;  // path-major, one per elementary move
    // move log (pipeline): {path-major slot, batch} of the accepted moves in
    // batch order; the warp scatters it into move_batch when its instance
    // finishes.  Null: move_batch is written directly.
    int2 *mlog;
    int32_t *nlog;
    int32_t *batch_count, *status, *detail;
};

cudaError_t launch_batch_explicit(const BatchJob &J, const int64_t *off, const int32_t *verts, cudaStream_t st);

// kernels used by the general C-ABI call
__global__ void edges_check_kernel(int P, int64_t E, const int32_t *es, const int32_t *ed, int32_t *bad,
                                   int32_t *outdeg, int32_t *indeg);
__global__ void csr_fill_kernel(int64_t E, const int32_t *key, const int32_t *val, const int64_t *off, int32_t *fill,
                                int32_t *out, const int64_t *need_in, int64_t *need_out);
__global__ void kahn_kernel(int P, const int64_t *soff, const int32_t *succ, int32_t *indeg, int32_t *frontier,
                            int32_t *next_frontier, int32_t *processed);
__global__ void need_kernel(int64_t E, const int32_t *es, const int32_t *ed, const int64_t *off, const int32_t *verts,
                            int64_t *need);

// fused pipeline over `count` grid instances already solved on the device
struct PipelineArgs {
    int count, W, H, k, preset;
    int leap;                            // leap mode (preset none): batching.cu
    int wide;                            // wide phase first (batch_wide.cu)
    int64_t *wstate;                     // [count * 4] wide -> warp hand-off {phase, nb, left, nready}
    int32_t *wnext;                      // window kernel: next instance to take (zeroed before the launch)
    int32_t *vmin;                       // [count * W*H] wide: per-vertex min id (0x7f7f7f7f = empty)
    const int32_t *path_src, *path_dst;  // [count * W*k] (instance stride W*k)
    const int32_t *path_count;           // [count]
    const int32_t *solve_status;         // [count]
    const int32_t *solve_detail;         // [count] (may be null)
    int64_t move_stride;
    int32_t *move_batch;                 // [count * move_stride]
    int32_t *batch_count, *status, *detail;
    // scratch (device), per instance strides: maps W*H, paths W*k
    int32_t *source_of, *target_of;      // [count * W*H]
    int32_t *outdeg, *indeg, *fill;      // [count * W*k]
    const int32_t *slen;                 // list lengths (= outdeg after pl_compact_kernel), or null (small DAG)
    int64_t *soff;                       // [count * W*k + 1]
    int64_t *mbase;                      // [count * W*k + 1]
    int32_t *succ;                       // [edge capacity]
    int64_t edge_capacity;
    uint32_t *occ, *inb;                 // [count * ceil(W*H/32)]
    int32_t *newly, *mem, *mfr, *mto;    // [count * W*k]
    int32_t *counter;                    // [count] move-log length
    int2 *mlog;                          // [total moves] move log, instance i at mbase[i*W*k]
    // small instances (pipeline_small_dag): per-instance edge / move totals and
    // their exclusive scans over instances, [count + 1] each
    int small_dag;
    int4 *rec, *rec2;    // [count * W*k] ready-path records (batch_warp_pipe)
    int4 *prec;          // [count * (W*k + 1)] path records {xs|ys<<16, xt|yt<<16, move base, soff} (leap / wide)
    int32_t *rb, *rb2;   // [count * W*k] their move bases
    int64_t *inst_edges, *inst_moves, *ebase, *mvbase;
    const uint64_t *grid_occ;            // [count * W * wpc] initial occupancy (occ bits)
    void *temp;
    size_t temp_bytes;
};

size_t pipeline_temp_bytes(int64_t n);
// counts_host[0] = DAG edges, counts_host[1] = elementary moves (all instances)
cudaError_t pipeline_dag_count(const PipelineArgs &a, cudaStream_t st, int64_t *counts_host, int64_t *launches);
// pev (may be null): events [2] after the DAG, [3] after the wide phase, [4] after batching
cudaError_t pipeline_run_batching(const PipelineArgs &a, int sms, cudaStream_t st, cudaEvent_t *pev, int64_t *launches);
// shared memory of the per-instance DAG builder, or 0 when an instance does not fit
int64_t pipeline_small_dag_smem(int W, int H, int k);

// wide phase (batch_wide.cu): CTA per instance while the ready set exceeds a warp
bool pipeline_wide_config(int W, int H, int64_t smem_budget, int *rmax, int *hbits, size_t *smem);
cudaError_t launch_batch_wide(const PipelineArgs &a, int sms, int rmax, int hbits, size_t smem, cudaStream_t st);
// preset none: the wide phase in windows of batches (batch_window.cu)
bool pipeline_window_config(int W, int H, int64_t smem_budget, int *rmax, size_t *smem);
cudaError_t launch_batch_window(const PipelineArgs &a, int sms, int rmax, size_t smem, cudaStream_t st);

// occ bits (column-major, bit y) -> vertex-id bitmap
__global__ void occ_to_vertex_bits(int count, int W, int H, const uint64_t *occ, uint32_t *bits);

}  // namespace rb
