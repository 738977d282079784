// Host/device interface of the grid-solver kernels (grid_solver.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rb {

// Instance shape and derived sizes (host computes, device reads).
struct GridShape {
    int W, H, k;      // width, height, band height h'
    int wpd;          // u64 words per column
    int B;            // bits per lane chunk in warp engines (8/16/32)
    int LK;           // list capacity (k + 2)
    int LT, LB;       // level-table sizes (top / bottom), multiples of 64
    int nchunk;       // 32-slot chunks covering 2W-1 group-order slots
    int nwarps;
    int lo, hi;       // band depths (rows from the top)
    int solver;       // executor the shared-memory layout is for: 0 red-rec, 1 bird
    int64_t smem_bytes;
};

struct GridSmem {
    int64_t dep, keys, bal, sigma, ev_count, ev_off, wave_off, lvl_t, lvl_b, scal, lists, plists, mark_next, mark_head,
        ev_col, ev_aux, ev_a, wave_list, ev_type, solved, total;
};

// red-rec plans in global memory (redrec_plan_kernel -> redrec_kernel), per
// instance: W event types / columns / aux columns / wave list, W+2 wave
// offsets, 8 meta ints (n1, n2, nlev, status, detail)
struct RedrecPlans {
    uint8_t *ev_type;
    int16_t *ev_col, *ev_aux, *wave_list;
    int32_t *wave_off, *meta;
};

struct GridParams {
    GridShape shape;
    const uint64_t *occ;
    int count;
    int32_t *path_src, *path_dst, *path_event;
    int32_t *path_count;
    int64_t *total_displacement;
    int32_t *status, *detail, *events;
    uint32_t *stage;         // red-rec: per-CTA packed path staging, W*k words per CTA (grid-sized)
    RedrecPlans plans;       // red-rec: [count] plans
    long long *phase_clock;  // optional: clock64 at phase boundaries of instance 0 (profiling)
    int *work;               // optional: zeroed instance counter (dynamic instance scheduling)
};

bool grid_shape(int W, int H, int k, int nwarps, int solver, GridShape &s);
// ev (optional): events recorded before the planner, before and after the
// executor (bird: the last two)
cudaError_t launch_grid_solver(int solver, const GridParams &p, int grid, cudaStream_t stream,
                               cudaEvent_t *ev = nullptr);
int grid_occupancy(int solver, const GridShape &s);
// per-event staging stride (ints): k rounded up to a 128-byte line
__host__ __device__ inline int stage_stride(int k) { return (k + 31) & ~31; }
size_t grid_stage_ints(const GridShape &s);
size_t redrec_plan_bytes(int W);  // global plan bytes per instance
RedrecPlans redrec_plans_carve(void *base, int W, int count);

}  // namespace rb
