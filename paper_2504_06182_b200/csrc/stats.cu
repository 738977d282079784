// Per-instance result record of a pipeline run, on the device:
// SolutionStats {displaced_tokens, total_displacement} (path_system.hpp:74-77,
// path_system.cpp:41-44), the batch count (BatchSchedule::batches.size(),
// batching.hpp:23-27), the status, and digest64 over the canonical path list
// and the whole batch schedule (the digest definition is in
// include/recon_b200.h).  One CTA per instance; the element hashes are summed
// (mod 2^64) by a block reduction, so the value is independent of the
// reduction order.  SURVEY.md §5 / §8(d): the 32-byte stats record, plus the
// digest that cross-GPU-count identity is checked with.

#include <climits>

#include "capi_internal.cuh"
#include "common.cuh"

namespace {

using namespace rb;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t elem(uint64_t tag, uint64_t i, int32_t v) {
    return mix64(mix64((tag << 48) ^ i) ^ (uint64_t)(uint32_t)v);
}

constexpr int ST = 256;

__global__ void __launch_bounds__(ST) pipeline_stats_kernel(recon_pipeline_batch pb, recon_instance_stats *out) {
    __shared__ unsigned long long s_sum;
    __shared__ int s_disp;
    const recon_grid_batch &g = pb.grid;
    const int64_t S = (int64_t)g.width * g.h_prime;
    for (int inst = blockIdx.x; inst < g.count; inst += gridDim.x) {
        const int32_t st = g.status[inst];
        recon_instance_stats r{};
        r.status = st;
        r.detail = g.detail ? g.detail[inst] : 0;
        if (st != RECON_OK) {
            if (threadIdx.x == 0) {
                r.digest = mix64(elem(4, 0, st));
                out[inst] = r;
            }
            continue;
        }
        const int P = g.path_count[inst];
        const int64_t D = g.total_displacement[inst];
        const int32_t nb = pb.batch_count[inst];
        if (threadIdx.x == 0) {
            s_sum = 0;
            s_disp = 0;
        }
        __syncthreads();
        const int32_t *src = g.path_src + inst * S, *dst = g.path_dst + inst * S;
        const int32_t *mb = pb.move_batch + inst * pb.move_stride;
        uint64_t acc = 0;
        int disp = 0;
        for (int i = threadIdx.x; i < P; i += ST) {
            const int32_t s = __ldg(src + i), t = __ldg(dst + i);
            acc += elem(1, i, s) + elem(2, i, t);
            disp += s != t;
        }
        for (int64_t j = threadIdx.x; j < D; j += ST) acc += elem(3, (uint64_t)j, __ldcs(mb + j));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            acc += __shfl_xor_sync(FULL, acc, o);
            disp += __shfl_xor_sync(FULL, disp, o);
        }
        if (lane_id() == 0) {
            atomicAdd(&s_sum, (unsigned long long)acc);
            atomicAdd(&s_disp, disp);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t a = s_sum;
            a += elem(5, 0, P) + elem(6, 0, (int32_t)(uint32_t)(D & 0xffffffffll)) + elem(7, 0, (int32_t)(D >> 32)) +
                 elem(8, 0, nb);
            r.path_count = P;
            r.displaced_tokens = s_disp;
            r.total_displacement = D;
            r.batch_count = nb;
            r.digest = mix64(a);
            out[inst] = r;
        }
        __syncthreads();
    }
}

// ---- run-length schedule: one CTA per instance, RI consecutive moves per
// thread (two 16-byte loads, the next tile's issued before this tile's scan),
// a run starts where the batch index does not continue the previous move's
// (+1); a block scan over the run-start counts places the runs (one barrier
// per tile: the warp totals are double-buffered).  HBM-bound: 4 B read per
// move (C5: 54 GB per 1,536-instance chunk)
constexpr int RI = 8, RT = 1024;

// v = p[j, j + RI) (0 past D); 16-byte loads while inside [0, lim)
__device__ __forceinline__ void load8(const int32_t *p, int64_t j, int64_t lim, int64_t D, int32_t *v) {
    if (j + RI <= lim) {
        const int4 x = __ldcs(reinterpret_cast<const int4 *>(p + j));
        const int4 y = __ldcs(reinterpret_cast<const int4 *>(p + j + 4));
        v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w, v[4] = y.x, v[5] = y.y, v[6] = y.z, v[7] = y.w;
    } else {
#pragma unroll
        for (int i = 0; i < RI; ++i) v[i] = j + i < D ? p[j + i] : 0;
    }
}

__global__ void __launch_bounds__(RT, 2) schedule_runs_kernel(recon_pipeline_batch pb, recon_schedule_runs runs) {
    __shared__ int wsum[2][RT / 32];
    const recon_grid_batch &g = pb.grid;
    const int lane = lane_id(), warp = warp_id();
    constexpr int64_t TILE = (int64_t)RT * RI;
    for (int inst = blockIdx.x; inst < g.count; inst += gridDim.x) {
        const int64_t D = g.status[inst] == RECON_OK ? g.total_displacement[inst] : 0;
        const int32_t *mb = pb.move_batch + inst * pb.move_stride;
        int32_t *rs = runs.run_slot + inst * runs.run_stride, *rb = runs.run_batch + inst * runs.run_stride;
        // (vector loads only when aligned, and inside the instance's move_stride;
        // moves past D are masked)
        const int64_t ms4 = pb.move_stride - (pb.move_stride & 3);
        const int64_t lim = ((uintptr_t)mb & 15u) == 0 && ms4 >= D ? ms4 : -1;
        int64_t base = 0;
        int32_t nx[RI];
        if (D > 0) load8(mb, (int64_t)threadIdx.x * RI, lim, D, nx);
        int par = 0;
        for (int64_t t0 = 0; t0 < D; t0 += TILE, par ^= 1) {
            const int64_t j0 = t0 + (int64_t)threadIdx.x * RI;
            int32_t v[RI];
#pragma unroll
            for (int i = 0; i < RI; ++i) v[i] = nx[i];
            if (t0 + TILE < D) load8(mb, j0 + TILE, lim, D, nx);
            // the move before this thread's first: the lane below's last, or
            // (lane 0) the previous warp's / tile's, loaded
            int32_t pv = __shfl_up_sync(FULL, v[RI - 1], 1);
            if (lane == 0) pv = (j0 > 0 && j0 - 1 < D) ? mb[j0 - 1] : INT_MIN;
            unsigned starts = 0;
#pragma unroll
            for (int i = 0; i < RI; ++i) {
                const int32_t prev = i == 0 ? pv : v[i - 1];
                if (j0 + i < D && (j0 + i == 0 || v[i] != prev + 1)) starts |= 1u << i;
            }
            int tot;
            const int ex = warp_excl_scan(__popc(starts), &tot);
            if (lane == 0) wsum[par][warp] = tot;
            __syncthreads();
            int wt;
            const int wex = warp_excl_scan(wsum[par][lane], &wt);  // (RT / 32 == 32 warps)
            int64_t at = base + __shfl_sync(FULL, wex, warp) + ex;
#pragma unroll
            for (int i = 0; i < RI; ++i)
                if ((starts >> i) & 1u) {
                    if (at < runs.run_stride) {
                        rs[at] = (int32_t)(j0 + i);
                        rb[at] = v[i];
                    }
                    ++at;
                }
            base += wt;
        }
        if (threadIdx.x == 0) runs.run_count[inst] = base;
        __syncthreads();  // (wsum of this instance's last tiles)
    }
}

}  // namespace

namespace rb {
// enqueues the run extraction of a device pipeline batch on `st`
cudaError_t launch_schedule_runs(const recon_pipeline_batch &pb, const recon_schedule_runs &runs, int sms,
                                 cudaStream_t st) {
    const int grid = pb.grid.count < sms * 2 ? pb.grid.count : sms * 2;
    schedule_runs_kernel<<<grid, RT, 0, st>>>(pb, runs);
    return cudaGetLastError();
}
}  // namespace rb

extern "C" recon_status recon_pipeline_schedule_runs(recon_ctx *ctx, const recon_pipeline_batch *pb,
                                                     recon_schedule_runs *runs) {
    int32_t *detail = nullptr;
    if (!pb || !runs || !runs->run_slot || !runs->run_batch || !runs->run_count || !pb->move_batch ||
        !pb->grid.status || !pb->grid.total_displacement)
        return RECON_ERR_ARGUMENT;
    if (pb->grid.count <= 0) return RECON_OK;
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice", detail);
    e = launch_schedule_runs(*pb, *runs, c->sms, c->stream);
    c->launches += 1;
    if (e != cudaSuccess) return cuda_fail(e, "schedule runs", detail);
    return RECON_OK;
}

extern "C" recon_status recon_pipeline_stats(recon_ctx *ctx, const recon_pipeline_batch *pb, recon_instance_stats *stats) {
    int32_t *detail = nullptr;
    if (!pb || !stats || !pb->grid.status || !pb->grid.path_count || !pb->grid.path_src || !pb->grid.path_dst ||
        !pb->grid.total_displacement || !pb->move_batch || !pb->batch_count)
        return RECON_ERR_ARGUMENT;
    if (pb->grid.count <= 0) return RECON_OK;
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice", detail);
    const int grid = pb->grid.count < c->sms * 8 ? pb->grid.count : c->sms * 8;
    pipeline_stats_kernel<<<grid, ST, 0, c->stream>>>(*pb, stats);
    c->launches += 1;
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "pipeline stats", detail);
    return RECON_OK;
}
