/*
 * recon_b200.h — C-ABI of the B200-native atom-reconfiguration core.
 *
 * This is the drop-in boundary between the reference's C++ API
 * (the headers under /root/reference/proj/include/recon, unchanged) and the sm_100a
 * kernels in paper_2504_06182_b200/csrc.  Every entry point takes plain
 * pointers and sizes; no C++ or torch types cross it.  The reference-side
 * binding (the C++ shim that re-implements the reference's free functions on
 * top of these calls) is paper_2504_06182_b200/shim/recon_shim.cpp and is
 * described in INTEGRATION.md.
 *
 * Which reference interface each entry point replaces:
 *
 *   recon_redrec_solve         Solution red_rec(const Problem&, std::vector<RedRecEvent>*)
 *                                  reference proj/include/recon/redrec.hpp:67-68,
 *                                  proj/src/redrec.cpp:205-232
 *   recon_bird_solve           Solution bird(const Problem&, std::vector<int>*)
 *                                  bird.hpp:40-41, bird.cpp:107-123
 *   recon_occupancy_dag        MoveDag occupancy_dag(const std::vector<Path>&)
 *                                  virtual_line.hpp:104, virtual_line.cpp:241-268
 *   recon_assign_1d            Matching1D assign_1d(int, std::vector<int>, std::vector<int>)
 *                                  exact1d.hpp:21, exact1d.cpp:342-372
 *   recon_assign_1d_generalized Matching1D assign_1d_generalized(const Generalized1DInstance&)
 *                                  exact1d.hpp:39, exact1d.cpp:374-407
 *   recon_solve_1d             Solution solve_1d(int, const std::vector<int>&, const std::vector<int>&)
 *                                  exact1d.hpp:82, exact1d.cpp:564-572
 *   recon_batch_moves          BatchSchedule batch_moves(const Problem&, const Solution&, const BatchOptions&)
 *                                  batching.hpp:58-59, batching.cpp:28-159
 *
 * plus batched device-resident variants (recon_*_batch) that take `count`
 * independent instances already in HBM and write per-instance outputs at a
 * fixed stride, and host-buffer batched variants (recon_*_batch_host) that
 * include the host<->device copies.
 *
 * Occupancy layout ("occ bits"): column-major bit planes.  A W x H grid uses
 * words_per_column = (H + 63) / 64 uint64 words per column; the token on
 * vertex (x, y) (y counted from the bottom row, vertex id x*H + y, reference
 * geometry.hpp:89-92) is bit (y % 64) of word [x * words_per_column + y / 64].
 * A chain of n vertices is the W = n, H = 1 case written densely: bit v of
 * word v / 64 (words_per_chain = (n + 63) / 64).
 *
 * Errors: every call returns a recon_status that maps 1:1 onto the reference
 * exception types (geometry.hpp:18-30 plus std::logic_error from
 * redrec.cpp:82-84); *detail selects the exact reference message, available
 * from recon_detail_message().  Per-instance statuses of batched calls use the
 * same codes.
 *
 * Threading: no hidden global mutable state.  A recon_ctx owns a CUDA stream
 * and a device workspace; calls on distinct contexts may run concurrently.
 * Passing ctx == NULL uses a context private to the calling host thread.
 */
#ifndef RECON_B200_H
#define RECON_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RECON_ABI_VERSION 1

typedef enum recon_status {
    RECON_OK = 0,
    RECON_ERR_INPUT = 1,      /* recon::InputError */
    RECON_ERR_INFEASIBLE = 2, /* recon::InfeasibleError */
    RECON_ERR_COLLISION = 3,  /* recon::CollisionError */
    RECON_ERR_LOGIC = 4,      /* std::logic_error */
    RECON_ERR_CAPACITY = 5,   /* a caller buffer is too small; the *_count out-param holds the need */
    RECON_ERR_CUDA = 6,       /* CUDA runtime failure (no device, launch failure, ...) */
    RECON_ERR_ARGUMENT = 7    /* null pointer / nonsensical size passed to the C-ABI */
} recon_status;

/* Exact reference messages (file:line of the throw in the reference). */
typedef enum recon_detail {
    RECON_D_NONE = 0,
    RECON_D_FEWER_SOURCES = 1,         /* "fewer sources than targets (|S| < |T|)" problem.hpp:115, exact1d.cpp:311 */
    RECON_D_BAND_NOT_CENTERED = 2,     /* "targets must form a centered full-width band" virtual_line.cpp:32-45 */
    RECON_D_BAND_HEIGHT = 3,           /* "target band height must be in (0, H)" virtual_line.cpp:48-49 */
    RECON_D_BAND_EMPTY = 4,            /* "target band is empty" virtual_line.cpp:25 */
    RECON_D_NO_DEFICIT = 5,            /* "select_best_pair: no deficit column remains" redrec.cpp:82 */
    RECON_D_NO_DONOR = 6,              /* "select_best_pair: deficit column with no admissible donor" redrec.cpp:83-84 */
    RECON_D_BATCH_NO_PROGRESS = 7,     /* "batching made no progress (blocked dependency structure)" batching.cpp:127-128 */
    RECON_D_BATCH_CYCLIC = 8,          /* "batching requires an acyclic dependency dag" batching.cpp:34 */
    RECON_D_CHAIN_LENGTH = 9,          /* "chain length must be positive" exact1d.cpp:300 */
    RECON_D_SOURCE_OOB = 10,           /* "source vertex out of bounds" exact1d.cpp:303-304 */
    RECON_D_SOURCE_ORDER = 11,         /* "source vertices must be strictly increasing" exact1d.cpp:305-306 */
    RECON_D_TARGET_OOB = 12,           /* "target vertex out of bounds" */
    RECON_D_TARGET_ORDER = 13,         /* "target vertices must be strictly increasing" */
    RECON_D_GEN_MULTIPLICITY = 14,     /* "source multiplicity must be at least 1" exact1d.cpp:379 */
    RECON_D_GEN_MIN_USE = 15,          /* "source min_use outside [0, multiplicity]" exact1d.cpp:380-381 */
    RECON_D_GEN_SOURCE_ORDER = 16,     /* "source positions must be strictly increasing" exact1d.cpp:382-383 */
    RECON_D_GEN_TARGET_ORDER = 17,     /* "target positions must be strictly increasing" exact1d.cpp:389 */
    RECON_D_GEN_SUPPLY = 18,           /* "insufficient tokens for targets" exact1d.cpp:391 */
    RECON_D_GEN_MANDATORY = 19,        /* "mandatory draws exceed target count" exact1d.cpp:392 */
    RECON_D_GEN_NO_ASSIGNMENT = 20,    /* "no assignment satisfies the usage bounds" exact1d.cpp:395 */
    RECON_D_DAG_EDGE_RANGE = 21,       /* "dag edge endpoint out of range" path_system.cpp:12 */
    RECON_D_GRID_DIMENSIONS = 22,      /* "grid dimensions must be positive" geometry.hpp */
    RECON_D_INFEASIBLE_SUPPLY = 23,    /* "fewer sources than targets" exact1d.cpp:70 (certifier) */
    RECON_D_CUDA = 24                  /* CUDA runtime failure; see recon_last_cuda_error() */
} recon_detail;

const char *recon_detail_message(int32_t detail);
const char *recon_last_cuda_error(void);
int32_t recon_abi_version(void);

/* ------------------------------------------------------------------------- */
/* Contexts                                                                   */
/* ------------------------------------------------------------------------- */

typedef struct recon_ctx recon_ctx;

/* Creates a context bound to CUDA device `device` with its own stream. */
recon_status recon_ctx_create(int32_t device, recon_ctx **out);
void recon_ctx_destroy(recon_ctx *ctx);
/* The context's cudaStream_t (as void*). */
void *recon_ctx_stream(recon_ctx *ctx);
/* Number of kernel launches this context has issued (for bench accounting). */
int64_t recon_ctx_launch_count(recon_ctx *ctx);
/* Profiling (no reference counterpart): with timing enabled, the grid
   solvers record CUDA events on the context stream around their kernels;
   recon_ctx_kernel_times waits for the last solve and writes ms[0] = red-rec
   planner, ms[1] = red-rec executor or bird kernel (0 when not launched). */
recon_status recon_ctx_set_kernel_timing(recon_ctx *ctx, int32_t enable);
recon_status recon_ctx_kernel_times(recon_ctx *ctx, float *ms, int32_t n);
/* With kernel timing on: the last device pipeline run's phases in ms (CUDA
 * events on the context stream): [0] solve, [1] occupancy DAG + path records,
 * [2] wide batching phase, [3] warp batching phase.  Zeros otherwise. */
recon_status recon_ctx_phase_times(recon_ctx *ctx, float *ms, int32_t n);

/* ------------------------------------------------------------------------- */
/* Grid solvers (red-rec, bird): single instance, host buffers                */
/* ------------------------------------------------------------------------- */

/*
 * Paths come out in the reference's canonical order (the path order of
 * Solution::path_system, which is also the schedule order: red_rec/bird use
 * the identity path order, virtual_line.cpp:270-277).  Each path is a
 * one-bend staircase fully determined by (src, dst): horizontal along the
 * source row to the destination column, then vertical (virtual_line.cpp:150-173).
 * Every grid path has length > 0.
 *
 * `path_capacity` >= width * h_prime always suffices.
 * `events`: red-rec writes 4 int32 per event {event_id, column, donor,
 * mark_destination} (redrec.hpp:56-65); bird writes 1 int32 per event, the
 * filled column (the solved_order of bird.hpp:41).  Both emit exactly
 * `width` events; capacity counts int32 elements.  May be NULL.
 * `dag_*`: optional occupancy DAG (virtual_line.cpp:241-268), edges sorted by
 * (src, dst); pass dag_src == NULL to skip.  On RECON_ERR_CAPACITY the
 * required edge count is in dag_count.
 */
typedef struct recon_grid_solution {
    int32_t *path_src;
    int32_t *path_dst;
    int32_t *path_event; /* may be NULL */
    int64_t path_capacity;
    int64_t path_count;           /* out */
    int64_t displaced_tokens;     /* out: SolutionStats::displaced_tokens */
    int64_t total_displacement;   /* out: SolutionStats::total_displacement */
    int32_t *events;              /* may be NULL */
    int32_t event_capacity;
    int32_t event_count;          /* out (number of events, not int32s) */
    int32_t *dag_src;             /* may be NULL */
    int32_t *dag_dst;
    int64_t dag_capacity;
    int64_t dag_count;            /* out */
} recon_grid_solution;

recon_status recon_redrec_solve(recon_ctx *ctx, const uint64_t *occ, int32_t width,
                                int32_t height, int32_t h_prime, recon_grid_solution *out,
                                int32_t *detail);
recon_status recon_bird_solve(recon_ctx *ctx, const uint64_t *occ, int32_t width,
                              int32_t height, int32_t h_prime, recon_grid_solution *out,
                              int32_t *detail);

/* occupancy_dag over an explicit path list given as (src, dst) one-bend paths
 * on a width x height grid.  Edges sorted by (src, dst). */
recon_status recon_occupancy_dag(recon_ctx *ctx, int32_t width, int32_t height,
                                 const int32_t *path_src, const int32_t *path_dst,
                                 int64_t path_count, int32_t *dag_src, int32_t *dag_dst,
                                 int64_t dag_capacity, int64_t *dag_count, int32_t *detail);

/* ------------------------------------------------------------------------- */
/* Grid solvers: batched, device-resident                                     */
/* ------------------------------------------------------------------------- */

/*
 * `count` independent instances of one (width, height, h_prime) shape.  All
 * pointers are device pointers.  Instance i reads occ + i*width*wpc and writes
 * its paths at [i * path_stride, i * path_stride + path_count[i]) with
 * path_stride = width * h_prime.
 */
typedef struct recon_grid_batch {
    const uint64_t *occ;
    int32_t count;
    int32_t width;
    int32_t height;
    int32_t h_prime;
    int32_t *path_src;           /* [count * width * h_prime] */
    int32_t *path_dst;           /* [count * width * h_prime] */
    int32_t *path_event;         /* may be NULL */
    int32_t *path_count;         /* [count] */
    int64_t *total_displacement; /* [count] */
    int32_t *status;             /* [count] recon_status */
    int32_t *detail;             /* [count] recon_detail */
    int32_t *events;             /* may be NULL: red-rec [count*width*4], bird [count*width] */
} recon_grid_batch;

recon_status recon_redrec_solve_batch(recon_ctx *ctx, const recon_grid_batch *batch);
recon_status recon_bird_solve_batch(recon_ctx *ctx, const recon_grid_batch *batch);

/* Same, but every pointer in `batch` is HOST memory (pinned or pageable): the
 * call copies the inputs in, solves, and copies the outputs back. */
recon_status recon_redrec_solve_batch_host(recon_ctx *ctx, const recon_grid_batch *batch);
recon_status recon_bird_solve_batch_host(recon_ctx *ctx, const recon_grid_batch *batch);

/* Same as *_batch_host, but the path list comes back packed: one uint32 per
 * path slot, src | dst << 16, in path_packed[count * width * h_prime] (slot
 * layout as path_src).  Grids of at most 65,536 cells (RECON_ERR_ARGUMENT
 * otherwise); batch->path_src / path_dst are not used and may be NULL.  The
 * device-to-host copy of the path lists bounds the host call (8 bytes per
 * path over the host link), and this halves it.  Same paths, same order:
 * a caller decodes src = v & 0xffff, dst = v >> 16. */
recon_status recon_redrec_solve_batch_host_packed(recon_ctx *ctx, const recon_grid_batch *batch,
                                                  uint32_t *path_packed);
recon_status recon_bird_solve_batch_host_packed(recon_ctx *ctx, const recon_grid_batch *batch,
                                                uint32_t *path_packed);

/* occupancy_dag over explicit vertex lists (paths of any shape, CSR
 * off[P+1] into verts); edges sorted by (src, dst), deduplicated. */
recon_status recon_occupancy_dag_paths(recon_ctx *ctx, int32_t width, int32_t height, int32_t path_count,
                                       const int64_t *path_offsets, const int32_t *path_vertices,
                                       int32_t *dag_src, int32_t *dag_dst, int64_t dag_capacity,
                                       int64_t *dag_count, int32_t *detail);

/* ------------------------------------------------------------------------- */
/* Exact 1D                                                                   */
/* ------------------------------------------------------------------------- */

/* min_assignment_cost_1d (exact1d.hpp:48-49): exact optimum of assigning the
 * (unsorted, possibly repeated) sources onto the targets; virtual (negative)
 * positions allowed. */
recon_status recon_min_cost_1d(recon_ctx *ctx, int32_t ns, const int64_t *sources, int32_t nt,
                               const int64_t *targets, int64_t *cost, int32_t *detail);

/*
 * assign_1d: S and T need not be sorted (the reference sorts them,
 * exact1d.cpp:343-344).  Outputs: weight; pairs (src, dst) sorted by target,
 * exactly nt of them; use_count[ns] indexed by the SORTED S.
 */
recon_status recon_assign_1d(recon_ctx *ctx, int32_t n, const int32_t *S, int32_t ns,
                             const int32_t *T, int32_t nt, int64_t *weight, int64_t *pair_src,
                             int64_t *pair_dst, int32_t *use_count, int32_t *detail);

/* assign_1d_generalized: sources as parallel arrays (pos strictly increasing),
 * targets strictly increasing; pairs [nt], use_count [nsrc]. */
recon_status recon_assign_1d_generalized(recon_ctx *ctx, int32_t nsrc, const int64_t *pos,
                                         const int32_t *multiplicity, const int32_t *min_use,
                                         int32_t nt, const int64_t *targets, int64_t *weight,
                                         int64_t *pair_src, int64_t *pair_dst,
                                         int32_t *use_count, int32_t *detail);

/*
 * solve_1d: paths in the reference's path order (the order of
 * paths_from_matching after resolve_nesting, exact1d.cpp:564-572), i.e. one
 * straight path per target including zero-length ones; path_order is
 * order_moves_1d's execution order (exact1d.cpp:517-528); the DAG is the
 * span-overlap edge list in the reference's emission order
 * (exact1d.cpp:529-560).  dag_src == NULL skips the DAG; on
 * RECON_ERR_CAPACITY dag_count holds the need.
 */
recon_status recon_solve_1d(recon_ctx *ctx, int32_t n, const int32_t *S, int32_t ns,
                            const int32_t *T, int32_t nt, int32_t *path_src, int32_t *path_dst,
                            int32_t *path_order, int32_t *dag_src, int32_t *dag_dst,
                            int64_t dag_capacity, int64_t *dag_count,
                            int64_t *total_displacement, int32_t *displaced, int32_t *detail);

/*
 * Batched chains, device-resident: `count` chains of length n, sources given
 * as dense bits (words_per_chain = (n+63)/64 per chain), targets the
 * contiguous band [t_lo, t_hi] shared by every chain.  Instance i writes its
 * nt = t_hi - t_lo + 1 paths at [i*nt, (i+1)*nt) in solve_1d path order
 * (target ascending); its DAG stays implicit (span overlap, exact1d.cpp:529-560).
 */
typedef struct recon_chain_batch {
    const uint64_t *occ;
    int32_t count;
    int32_t n;
    int32_t t_lo;
    int32_t t_hi;
    int32_t *path_src;           /* [count * nt] */
    int32_t *path_dst;           /* [count * nt] */
    int64_t *total_displacement; /* [count] */
    int32_t *displaced;          /* [count] */
    int32_t *status;             /* [count] */
    int32_t *detail;             /* [count] */
} recon_chain_batch;

recon_status recon_solve_1d_batch(recon_ctx *ctx, const recon_chain_batch *batch);
recon_status recon_solve_1d_batch_host(recon_ctx *ctx, const recon_chain_batch *batch);

/* ------------------------------------------------------------------------- */
/* Batching                                                                   */
/* ------------------------------------------------------------------------- */

typedef enum recon_preset {
    RECON_PRESET_NONE = 0,             /* ConstraintPreset::none */
    RECON_PRESET_COLUMN_DIRECTION = 1  /* ConstraintPreset::column_direction */
} recon_preset;

/*
 * batch_moves over an explicit solution: initial occupancy (problem.sources)
 * as occ bits, paths as a CSR vertex list (path_offsets[P+1], int64), DAG
 * edges.  Output: move_batch[path_offsets[P] - P] — for path p, its k-th move
 * (vertices[k] -> vertices[k+1]) lands at index path_offsets[p] - p + k and
 * receives its batch number.  Batch b holds the moves tagged b in ascending
 * path id (batching.cpp:107-125); axis/dir tags follow from the batch's first
 * move when preset != none (batching.cpp:150-155).
 */
recon_status recon_batch_moves(recon_ctx *ctx, int32_t width, int32_t height,
                               const uint64_t *occ, int32_t path_count,
                               const int64_t *path_offsets, const int32_t *path_vertices,
                               int64_t edge_count, const int32_t *edge_src,
                               const int32_t *edge_dst, int32_t preset, int32_t edge_level,
                               int32_t *move_batch, int64_t *batch_count, int32_t *detail);

/*
 * Fused grid pipeline, device-resident: solve (red-rec or bird) + occupancy
 * DAG + batching for `count` instances.  Outputs of the solve as in
 * recon_grid_batch; move_batch holds, per instance, one batch index per
 * elementary move in canonical schedule order (path-major), at stride
 * move_stride; batch_count[i] = number of batches.
 */
typedef struct recon_pipeline_batch {
    recon_grid_batch grid;
    int32_t solver;              /* 0 = red-rec, 1 = bird */
    int32_t preset;              /* recon_preset */
    int64_t move_stride;         /* >= max total displacement per instance */
    int32_t *move_batch;         /* [count * move_stride] */
    int32_t *batch_count;        /* [count] */
} recon_pipeline_batch;

recon_status recon_pipeline_batch_run(recon_ctx *ctx, const recon_pipeline_batch *batch);
/* Same with every pointer in `batch` in host memory. */
recon_status recon_pipeline_batch_run_host(recon_ctx *ctx, const recon_pipeline_batch *batch);

/*
 * Per-instance result record of a pipeline run (device): SolutionStats
 * {displaced_tokens, total_displacement} (path_system.hpp:74-77), the batch
 * count (BatchSchedule::batches.size(), batching.hpp:23-27), the status and
 * digest64, a 64-bit fingerprint of the canonical path list and the whole
 * batch schedule (identical across GPU counts and chunkings):
 *   mix(z)       = splitmix64 finaliser (z += 0x9e3779b97f4a7c15; ...)
 *   e(tag, i, v) = mix(mix((tag << 48) ^ i) ^ (uint32)v)
 *   status == 0: digest = mix( sum_i e(1,i,src[i]) + e(2,i,dst[i])  (i < P)
 *                              + sum_j e(3,j,move_batch[j])          (j < D)
 *                              + e(5,0,P) + e(6,0,D & 0xffffffff) + e(7,0,D >> 32) + e(8,0,nb) )  (mod 2^64)
 *   else:        digest = mix(e(4,0,status))
 * (tests/digest.py is the same formula in numpy.)
 */
typedef struct recon_instance_stats {
    int32_t status;              /* recon_status of the instance (solve or batching) */
    int32_t detail;              /* recon_detail */
    int32_t path_count;          /* P */
    int32_t displaced_tokens;    /* paths of length > 0 (PathSystem::displaced_count) */
    int64_t total_displacement;  /* D */
    int64_t batch_count;         /* nb */
    uint64_t digest;             /* digest64 */
} recon_instance_stats;

/*
 * Run-length form of a batch schedule (a lossless wire format of move_batch,
 * SURVEY.md §8(f) 3): the path-major move list of an instance split into
 * maximal runs whose batch indices rise by one per move.  Run r covers moves
 * [run_slot[r], run_slot[r+1]) (the last run ends at the instance's total
 * displacement D), and move j of it is in batch run_batch[r] + (j - run_slot[r]).
 * A path that never waits is one run, so an instance needs about P runs
 * (~1.3 MB for C5) instead of D batch indices (~43 MB).  Instances whose
 * status is not RECON_OK have 0 runs.
 */
typedef struct recon_schedule_runs {
    int64_t run_stride;   /* run capacity per instance */
    int32_t *run_slot;    /* [count * run_stride] first move of each run */
    int32_t *run_batch;   /* [count * run_stride] its batch index */
    int64_t *run_count;   /* [count] runs per instance (> run_stride: RECON_ERR_CAPACITY) */
} recon_schedule_runs;

/* Runs of a finished recon_pipeline_batch_run (device pointers in both). */
recon_status recon_pipeline_schedule_runs(recon_ctx *ctx, const recon_pipeline_batch *batch, recon_schedule_runs *runs);
/* recon_pipeline_batch_run_host returning the schedule as runs (host pointers;
 * batch->move_batch may be NULL): the host link carries ~P runs instead of D
 * batch indices per instance.  Page-locked, device-mapped run_slot/run_batch
 * arrays (cudaHostAlloc, torch pin_memory) are written by a kernel over the host
 * link; other host memory is filled with one copy per instance and array. */
recon_status recon_pipeline_batch_run_host_runs(recon_ctx *ctx, const recon_pipeline_batch *batch,
                                                recon_schedule_runs *runs);

/* Stats of a finished recon_pipeline_batch_run: `batch` holds the run's device
 * pointers, `stats` is a device array of batch->grid.count records.  Enqueued
 * on the context's stream. */
recon_status recon_pipeline_stats(recon_ctx *ctx, const recon_pipeline_batch *batch, recon_instance_stats *stats);

/* ------------------------------------------------------------------------- */
/* Validators (device)                                                        */
/* ------------------------------------------------------------------------- */

/*
 * Batched, on-device restatement of the reference's solution checks for grid
 * solutions in this ABI's path format (one-bend paths from (src, dst), the
 * identity schedule = paths in order, each path's moves in order):
 *   validate_solution        executor.hpp:38, executor.cpp:142-183
 *   check_one_move_per_token executor.hpp:43, executor.cpp:185-219
 *   validate_batches         batching.hpp:64-65, batching.cpp:161-252
 * Each report keeps the reference's check order and early returns; the
 * verdict is a bit set of the failure categories the reference would report
 * (0 = every check passes).  Batch checks run when move_batch != NULL.  A
 * path endpoint off the grid yields exactly RECON_V_PATH_BOUNDS (the path
 * cannot be drawn, so nothing else is evaluated).
 */
typedef enum recon_verdict {
    RECON_V_PATH_BOUNDS = 1u << 0,          /* "path i leaves the grid" */
    RECON_V_SHARED_SOURCE = 1u << 1,        /* "two paths share source vertex v" */
    RECON_V_SHARED_TARGET = 1u << 2,        /* "two paths share target vertex v" */
    RECON_V_DAG_CYCLE = 1u << 3,            /* "dependency dag has a cycle" */
    RECON_V_STATS_DISPLACEMENT = 1u << 4,   /* stats.total_displacement != weight */
    RECON_V_STATS_DISPLACED = 1u << 5,      /* stats.displaced_tokens != displaced count */
    RECON_V_EXECUTION = 1u << 6,            /* "execution failed: ..." (collision) */
    RECON_V_TARGETS = 1u << 7,              /* final configuration misses a target */
    RECON_V_DAG_ORDER = 1u << 8,            /* "schedule violates dag edge i->j" */
    RECON_V_TOKEN_EMPTY = 1u << 9,          /* one-move check: move from an empty vertex */
    RECON_V_TOKEN_SECOND_PATH = 1u << 10,   /* one-move check: token begins a second path */
    RECON_V_BATCH_CONSERVATION = 1u << 11,  /* batched moves != path-system edge multiset */
    RECON_V_BATCH_BOUND = 1u << 12,         /* more batches than elementary moves */
    RECON_V_BATCH_EMPTY = 1u << 13,         /* "batch b is empty" */
    RECON_V_BATCH_DISJOINT = 1u << 14,      /* "batch b is not vertex-disjoint" */
    RECON_V_BATCH_CONSTRAINT = 1u << 15,    /* "batch b violates the constraint set" */
    RECON_V_BATCH_COLLISION = 1u << 16,     /* batch moves from an empty / into an occupied vertex */
    RECON_V_BATCH_TARGETS = 1u << 17,       /* batched execution misses a target */
    RECON_V_BATCH_DAG = 1u << 18,           /* "batch order violates dag edge i->j" */
    RECON_V_BATCH_ORDER = 1u << 19,         /* a path's move precedes its earlier move (match_schedule fails) */
    RECON_V_TOKEN_MATCH = 1u << 20          /* one-move check: match_schedule attributes the moves to
                                               other paths and then fails (colliding schedules only) */
} recon_verdict;

typedef enum recon_dag_mode {
    RECON_DAG_NONE = 0,       /* solution without dependency edges */
    RECON_DAG_EXPLICIT = 1,   /* edges (dag_a[e], dag_b[e]) for e in [dag_offset[i], dag_offset[i+1]) */
    RECON_DAG_OCCUPANCY = 2   /* occupancy_dag of the paths (virtual_line.cpp:241-268), derived on the device */
} recon_dag_mode;

typedef struct recon_validate_batch {
    const uint64_t *occ;                 /* initial configurations, count * width * wpc words */
    int32_t count, width, height, h_prime;
    const int32_t *path_src, *path_dst;  /* instance i at i * path_stride */
    int64_t path_stride;
    const int32_t *path_count;           /* [count] */
    const int64_t *total_displacement;   /* claimed stats [count], NULL = not checked */
    const int32_t *displaced;            /* claimed displaced_tokens [count], NULL = not checked */
    int32_t dag_mode;                    /* recon_dag_mode */
    const int32_t *dag_a, *dag_b;        /* RECON_DAG_EXPLICIT: edge lists (global edge index) */
    const int64_t *dag_offset;           /* [count + 1] */
    const int32_t *move_batch;           /* batch per move, path-major, instance i at i * move_stride; NULL = no batch checks */
    int64_t move_stride;
    const int32_t *batch_count;          /* [count] */
    int32_t preset;                      /* recon_preset of the batch schedule */
    uint32_t *verdict;                   /* [count] recon_verdict bits */
} recon_validate_batch;

recon_status recon_validate_batch_run(recon_ctx *ctx, const recon_validate_batch *batch);
/* Same with every pointer in `batch` in host memory. */
recon_status recon_validate_batch_run_host(recon_ctx *ctx, const recon_validate_batch *batch);

/* ------------------------------------------------------------------------- */
/* Wire formats (device)                                                      */
/* ------------------------------------------------------------------------- */

/*
 * The reference's JSON text, byte for byte, formatted on the device:
 *   recon_solution_json        solution_to_json       (io.hpp:21-22, io.cpp:81-101)
 *   recon_batch_schedule_json  batch_schedule_to_json (io.hpp:25-27, io.cpp:140-164)
 * Layout of the reference's nlohmann::ordered_json::dump(2) (stock library):
 * one value per line, two spaces per level, "[]" for empty arrays, plus the
 * trailing newline io.cpp adds.  Paths are one-bend paths from (src, dst);
 * the schedule is the paths' moves in path_order (NULL = identity, as
 * red_rec / bird emit it).  Batches are the moves tagged with each batch
 * index in ascending path id; axis/dir tags come from a batch's first move
 * when preset != none, else null.  *length receives the byte count (no NUL);
 * RECON_ERR_CAPACITY when capacity < *length (nothing written).
 */
recon_status recon_solution_json(recon_ctx *ctx, int32_t width, int32_t height, int32_t path_count,
                                 const int32_t *path_src, const int32_t *path_dst, const int32_t *path_order,
                                 int64_t dag_count, const int32_t *dag_a, const int32_t *dag_b,
                                 int64_t displaced_tokens, int64_t total_displacement, char *out,
                                 int64_t capacity, int64_t *length);
recon_status recon_batch_schedule_json(recon_ctx *ctx, int32_t width, int32_t height, int32_t path_count,
                                       const int32_t *path_src, const int32_t *path_dst,
                                       const int32_t *move_batch, int32_t batch_count, int32_t preset,
                                       char *out, int64_t capacity, int64_t *length);
/* Same with every pointer in host memory. */
recon_status recon_solution_json_host(recon_ctx *ctx, int32_t width, int32_t height, int32_t path_count,
                                      const int32_t *path_src, const int32_t *path_dst, const int32_t *path_order,
                                      int64_t dag_count, const int32_t *dag_a, const int32_t *dag_b,
                                      int64_t displaced_tokens, int64_t total_displacement, char *out,
                                      int64_t capacity, int64_t *length);
recon_status recon_batch_schedule_json_host(recon_ctx *ctx, int32_t width, int32_t height, int32_t path_count,
                                            const int32_t *path_src, const int32_t *path_dst,
                                            const int32_t *move_batch, int32_t batch_count, int32_t preset,
                                            char *out, int64_t capacity, int64_t *length);

/* ------------------------------------------------------------------------- */
/* Multi-cycle loss simulation (SPEC.md module `sim`; no reference code)      */
/* ------------------------------------------------------------------------- */

/*
 * Monte Carlo trials of repeated reconfiguration under atom loss (SPEC.md
 * [MODULE] sim: LossModel, run_trial, estimate_success).  Trial i starts from
 * occ[i] (sample_initial: recon_sample_occ gives the reference's Rng draws)
 * and repeats cycles: solve (red-rec or bird), optionally batch, execute the
 * schedule with per-operation survival draws, let every atom decay over the
 * cycle's elapsed time, re-measure.  A trial succeeds when the centered band
 * is full, and fails when fewer than W*h' atoms remain, when the solver or the
 * batching fails, or after max_cycles cycles.
 *
 * Execution model (SPEC design decisions and invariants):
 *  - every displaced token is extracted (p_alpha), makes its k moves (p_nu
 *    each) and is implanted (p_alpha); a token lost mid-path vanishes and
 *    skips its remaining operations; N_nu / N_alpha count the operations
 *    performed, so they are the same with and without batching (SPEC:
 *    "batching conservation");
 *  - unbatched, each displaced token is one EDI cycle (elapsed 2 t_alpha +
 *    k t_nu); batched, an EDI cycle is a maximal run of consecutive batches
 *    moving the same token set (elapsed 2 t_alpha + #batches t_nu);
 *  - NB_nu / NB_alpha count the scheduled displacement / transfer sequences
 *    (batched: batches / runs; unbatched: moves / displaced tokens);
 *  - after the moves every atom survives with exp(-(elapsed + t_meas) / tau)
 *    (tau <= 0: no decay).
 * Draws: include/recon_sim_rng.h (counter-based, order-independent).
 */
typedef struct recon_loss_model {
    double p_nu, p_alpha; /* per-displacement / per-transfer survival */
    double tau;           /* trapping lifetime (s); <= 0 disables decay */
    double t_nu, t_alpha, t_meas;
} recon_loss_model;

typedef struct recon_sim_batch {
    const uint64_t *occ;       /* initial configurations, count * width * wpc words (host) */
    int32_t count;             /* trials */
    int32_t width, height, h_prime;
    uint64_t seed_base;        /* trial i draws with seed_base + i */
    int32_t solver;            /* 0 = red-rec, 1 = bird */
    int32_t batching;          /* 0 = off, 1 = on */
    int32_t preset;            /* recon_preset when batching */
    int32_t max_cycles;
    recon_loss_model loss;
    /* outputs, [count] each, host memory */
    int32_t *success;          /* 1 = target reached */
    int32_t *cycles;           /* reconfiguration cycles run */
    int32_t *status;           /* RECON_OK, or the solver / batching status that ended the trial */
    int64_t *n_nu, *n_alpha, *nb_nu, *nb_alpha, *atoms_lost;
    double *elapsed;           /* model time (s) */
} recon_sim_batch;

recon_status recon_sim_run_host(recon_ctx *ctx, const recon_sim_batch *batch);

/* ------------------------------------------------------------------------- */
/* Synthetic inputs (host)                                                    */
/* ------------------------------------------------------------------------- */

/*
 * Instance i = Rng(seed_base + i).sample_without_replacement(width*height, k)
 * (reference rng.hpp:14-59, bit-identical), packed as occ bits: layout 0 =
 * grid (column-major words), layout 1 = dense chain (height must be 1).
 * threads <= 0 uses every hardware thread.
 */
recon_status recon_sample_occ(uint64_t seed_base, int32_t count, int32_t width, int32_t height,
                              int64_t k, int32_t layout, uint64_t *occ, int32_t threads);

#ifdef __cplusplus
}
#endif

#endif /* RECON_B200_H */
