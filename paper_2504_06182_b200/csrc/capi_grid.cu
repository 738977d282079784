// C-ABI: grid solvers (red-rec, bird) and the occupancy DAG.
//
// recon_redrec_solve / recon_bird_solve replace red_rec / bird
// (reference redrec.hpp:67-68, bird.hpp:40-41); recon_occupancy_dag replaces
// occupancy_dag (virtual_line.hpp:104).

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "capi_internal.cuh"
#include "dag.cuh"
#include "grid_solver.cuh"

using namespace rb;

namespace {

constexpr int kWarps = 8;

#define CK(call, where)                                   \
    do {                                                  \
        cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, where, detail); \
    } while (0)

recon_status validate_grid(int W, int H, int hp, int32_t *detail) {
    if (W <= 0 || H <= 0) {  // Geometry::grid (geometry.hpp:72-73)
        if (detail) *detail = RECON_D_GRID_DIMENSIONS;
        return RECON_ERR_INPUT;
    }
    if (hp <= 0 || hp >= H) {  // TargetRegion::expand (problem.hpp:82-83)
        if (detail) *detail = RECON_D_BAND_HEIGHT;
        return RECON_ERR_INPUT;
    }
    return RECON_OK;
}

// Warps per CTA.  Batches: more, smaller CTAs keep more instances in flight
// per SM and wait less at the wave / window barriers: 2 warps up to 128^2
// (red-rec: 1 up to 64^2; bird needs 2 for its top / bottom halves), 4 up to
// 256^2, 8 beyond (measured r01 with the per-solver shared-memory layouts).  A batch with no more instances than SMs runs one
// CTA per SM anyway, so it takes up to 32 warps (bird: 16) to shorten the
// instance's own critical path.  RECON_GRID_WARPS overrides.
bool shape_for(Ctx *c, int solver, int W, int H, int hp, int count, GridShape &s) {
    const long long cells = (long long)W * H;
    int w = cells <= 128 * 128 ? 2 : (cells <= 256 * 256 ? 4 : kWarps);
    if (solver == 0 && cells <= 64 * 64) w = 1;  // red-rec: one warp per tiny instance
    if (count <= c->sms) w = solver == 0 ? 32 : 16;  // latency: more warps on the instance
    if (const char *e = getenv("RECON_GRID_WARPS")) w = std::max(1, std::min(32, atoi(e)));
    if (solver == 1) w = std::max(2, std::min(w, 16));  // bird: 2..16 warps (top/bottom halves, 512 threads)
    const int floor_w = std::min(kWarps, w);  // (shape retries halve w down to this)
    for (; w >= floor_w; w /= 2)
        if (grid_shape(W, H, hp, w, solver, s)) return true;
    return grid_shape(W, H, hp, kWarps, solver, s);
}

int grid_blocks(Ctx *c, int solver, const GridShape &s, int count) {
    const int occ = std::max(1, grid_occupancy(solver, s));
    return std::max(1, std::min(count, occ * c->sms));
}

// launches with the per-CTA staging scratch and the plans the red-rec kernels need
cudaError_t launch(Ctx *c, int solver, GridParams &p, int grid) {
    // dynamic instance scheduling when CTAs take more than one instance
    p.work = nullptr;
    if (p.count > grid) {
        p.work = c->dev<int>(S_WORK, 1);
        if (!p.work) return cudaErrorMemoryAllocation;
        cudaError_t e = cudaMemsetAsync(p.work, 0, sizeof(int), c->stream);
        if (e != cudaSuccess) return e;
    }
    if (solver == 0) {
        p.stage = c->dev<uint32_t>(S_STAGE, (size_t)grid * grid_stage_ints(p.shape));
        if (!p.stage) return cudaErrorMemoryAllocation;
        void *pl = c->get(S_PLAN, (size_t)p.count * redrec_plan_bytes(p.shape.W) + 1024);
        if (!pl) return cudaErrorMemoryAllocation;
        p.plans = redrec_plans_carve(pl, p.shape.W, p.count);
    }
    c->launches += solver == 0 ? 2 : 1;
    c->timed_plan = solver == 0;
    return launch_grid_solver(solver, p, grid, c->stream, c->timing ? c->tev : nullptr);
}

// runs the DAG over `P` device-resident paths; copies edges to host arrays
recon_status run_dag(Ctx *c, int W, int H, const int32_t *d_src, const int32_t *d_dst, int64_t P,
                     int32_t *h_a, int32_t *h_b, int64_t cap, int64_t *count, int32_t *detail) {
    DagArgs d{};
    d.W = W;
    d.H = H;
    d.P = (int)P;
    d.src = d_src;
    d.dst = d_dst;
    d.source_of = c->dev<int32_t>(S_SRCOF, (size_t)W * H);
    d.target_of = c->dev<int32_t>(S_TGTOF, (size_t)W * H);
    d.cnt = c->dev<int32_t>(S_DCNT, (size_t)P + 1);
    d.off = c->dev<int64_t>(S_DOFF, (size_t)P + 2);
    d.temp_bytes = dag_temp_bytes(1, (int)P + 1);
    d.temp = c->get(S_TEMP, d.temp_bytes);
    if (!d.source_of || !d.target_of || !d.cnt || !d.off || !d.temp)
        return cuda_fail(cudaErrorMemoryAllocation, "dag workspace", detail);
    int64_t n = 0;
    CK(dag_count(d, c->stream, &n), "dag_count");
    c->launches += 4;
    *count = n;
    if (n > cap) return RECON_ERR_CAPACITY;
    if (n == 0) return RECON_OK;
    d.keys = c->dev<unsigned long long>(S_KEYS, (size_t)n);
    d.keys_alt = c->dev<unsigned long long>(S_KEYS2, (size_t)n);
    d.temp_bytes = dag_temp_bytes(n, (int)P + 1);
    d.temp = c->get(S_TEMP, d.temp_bytes);
    int32_t *ea = c->dev<int32_t>(S_EA, (size_t)n), *eb = c->dev<int32_t>(S_EB, (size_t)n);
    if (!d.keys || !d.keys_alt || !d.temp || !ea || !eb)
        return cuda_fail(cudaErrorMemoryAllocation, "dag workspace", detail);
    CK(dag_emit(d, n, c->stream, ea, eb), "dag_emit");
    c->launches += 3;
    CK(cudaMemcpyAsync(h_a, ea, (size_t)n * 4, cudaMemcpyDeviceToHost, c->stream), "dag D2H");
    CK(cudaMemcpyAsync(h_b, eb, (size_t)n * 4, cudaMemcpyDeviceToHost, c->stream), "dag D2H");
    CK(cudaStreamSynchronize(c->stream), "dag sync");
    return RECON_OK;
}

recon_status grid_single(int solver, recon_ctx *ctx, const uint64_t *occ, int W, int H, int hp,
                         recon_grid_solution *out, int32_t *detail) {
    if (detail) *detail = 0;
    if (!occ || !out) return RECON_ERR_ARGUMENT;
    recon_status st = validate_grid(W, H, hp, detail);
    if (st != RECON_OK) return st;
    Ctx *c = resolve(ctx);
    if (!c) {
        if (detail) *detail = RECON_D_CUDA;
        return RECON_ERR_CUDA;
    }
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    GridShape s;
    if (!shape_for(c, solver, W, H, hp, 1, s)) return RECON_ERR_ARGUMENT;
    const size_t words = (size_t)W * s.wpd, stride = (size_t)W * hp;
    GridParams p{};
    p.shape = s;
    p.count = 1;
    uint64_t *d_occ = c->dev<uint64_t>(S_OCC, words);
    p.occ = d_occ;
    p.path_src = c->dev<int32_t>(S_PSRC, stride);
    p.path_dst = c->dev<int32_t>(S_PDST, stride);
    p.path_event = c->dev<int32_t>(S_PEV, stride);
    p.path_count = c->dev<int32_t>(S_PCNT, 1);
    p.total_displacement = c->dev<int64_t>(S_TDISP, 1);
    p.status = c->dev<int32_t>(S_STATUS, 1);
    p.detail = c->dev<int32_t>(S_DETAIL, 1);
    p.events = c->dev<int32_t>(S_EVENTS, (size_t)W * 4);
    if (!d_occ || !p.path_src || !p.path_dst || !p.path_event || !p.path_count || !p.total_displacement ||
        !p.status || !p.detail || !p.events)
        return cuda_fail(cudaErrorMemoryAllocation, "grid workspace", detail);
    CK(cudaMemcpyAsync(d_occ, occ, words * 8, cudaMemcpyHostToDevice, c->stream), "occ H2D");
    CK(launch(c, solver, p, 1), "grid kernel launch");
    int32_t h_cnt = 0, h_st = 0, h_det = 0;
    int64_t h_td = 0;
    CK(cudaMemcpyAsync(&h_cnt, p.path_count, 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaMemcpyAsync(&h_st, p.status, 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaMemcpyAsync(&h_det, p.detail, 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaMemcpyAsync(&h_td, p.total_displacement, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaStreamSynchronize(c->stream), "grid kernel");
    if (h_st != RECON_OK) {
        if (detail) *detail = h_det;
        return (recon_status)h_st;
    }
    out->path_count = h_cnt;
    out->displaced_tokens = h_cnt;  // every grid path has length > 0 (virtual_line.cpp:219)
    out->total_displacement = h_td;
    out->event_count = W;
    if (out->path_capacity < h_cnt) return RECON_ERR_CAPACITY;
    if (h_cnt > 0) {
        CK(cudaMemcpyAsync(out->path_src, p.path_src, (size_t)h_cnt * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        CK(cudaMemcpyAsync(out->path_dst, p.path_dst, (size_t)h_cnt * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        if (out->path_event)
            CK(cudaMemcpyAsync(out->path_event, p.path_event, (size_t)h_cnt * 4, cudaMemcpyDeviceToHost, c->stream),
               "D2H");
    }
    if (out->events) {
        const int per = solver == 0 ? 4 : 1;
        if (out->event_capacity < W * per) return RECON_ERR_CAPACITY;
        CK(cudaMemcpyAsync(out->events, p.events, (size_t)W * per * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    }
    CK(cudaStreamSynchronize(c->stream), "D2H");
    if (out->dag_src) {
        return run_dag(c, W, H, p.path_src, p.path_dst, h_cnt, out->dag_src, out->dag_dst, out->dag_capacity,
                       &out->dag_count, detail);
    }
    return RECON_OK;
}

// Packed path list for the host copy: one u32 per path slot, src | dst << 16
// (grids of at most 65,536 cells).  Streaming loads/stores; the 8-byte
// {src, dst} slots are read once and 4 bytes go back over the host link.
__global__ void __launch_bounds__(256) pack_paths_kernel(const int32_t *__restrict__ src,
                                                         const int32_t *__restrict__ dst,
                                                         uint32_t *__restrict__ out, size_t n) {
    const size_t t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x, step = (size_t)gridDim.x * blockDim.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) |
                       reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    size_t done = 0;
    if (vec) {
        const size_t n4 = n / 4;
        const int4 *s4 = reinterpret_cast<const int4 *>(src), *d4 = reinterpret_cast<const int4 *>(dst);
        uint4 *o4 = reinterpret_cast<uint4 *>(out);
        for (size_t i = t0; i < n4; i += step) {
            const int4 a = __ldcs(s4 + i), b = __ldcs(d4 + i);
            __stcs(o4 + i, make_uint4((uint32_t)a.x | (uint32_t)b.x << 16, (uint32_t)a.y | (uint32_t)b.y << 16,
                                      (uint32_t)a.z | (uint32_t)b.z << 16, (uint32_t)a.w | (uint32_t)b.w << 16));
        }
        done = n4 * 4;
    }
    for (size_t i = done + t0; i < n; i += step) out[i] = (uint32_t)src[i] | (uint32_t)dst[i] << 16;
}

recon_status grid_batch(int solver, recon_ctx *ctx, const recon_grid_batch *b, bool host, uint32_t *packed = nullptr) {
    int32_t *detail = nullptr;
    if (!b || !b->occ || !b->path_count || !b->total_displacement || !b->status) return RECON_ERR_ARGUMENT;
    if (!packed && (!b->path_src || !b->path_dst)) return RECON_ERR_ARGUMENT;
    int32_t dummy = 0;
    recon_status st = validate_grid(b->width, b->height, b->h_prime, &dummy);
    if (st != RECON_OK) return st;
    if (packed && (int64_t)b->width * b->height > 65536) return RECON_ERR_ARGUMENT;
    if (b->count <= 0) return RECON_OK;
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    GridShape s;
    if (!shape_for(c, solver, b->width, b->height, b->h_prime, b->count, s)) return RECON_ERR_ARGUMENT;
    const size_t n = (size_t)b->count, words = (size_t)b->width * s.wpd, stride = (size_t)b->width * b->h_prime;
    const int per = solver == 0 ? 4 : 1;
    GridParams p{};
    p.shape = s;
    p.count = b->count;
    if (!host) {
        p.occ = b->occ;
        p.path_src = b->path_src;
        p.path_dst = b->path_dst;
        p.path_event = b->path_event;
        p.path_count = b->path_count;
        p.total_displacement = b->total_displacement;
        p.status = b->status;
        p.detail = b->detail;
        p.events = b->events;
        CK(launch(c, solver, p, grid_blocks(c, solver, s, b->count)), "grid kernel launch");
        return RECON_OK;
    }
    uint64_t *d_occ = c->dev<uint64_t>(S_OCC, n * words);
    p.occ = d_occ;
    p.path_src = c->dev<int32_t>(S_PSRC, n * stride);
    p.path_dst = c->dev<int32_t>(S_PDST, n * stride);
    p.path_event = b->path_event ? c->dev<int32_t>(S_PEV, n * stride) : nullptr;
    p.path_count = c->dev<int32_t>(S_PCNT, n);
    p.total_displacement = c->dev<int64_t>(S_TDISP, n);
    p.status = c->dev<int32_t>(S_STATUS, n);
    p.detail = c->dev<int32_t>(S_DETAIL, n);
    p.events = b->events ? c->dev<int32_t>(S_EVENTS, n * b->width * per) : nullptr;
    uint32_t *d_pack = packed ? c->dev<uint32_t>(S_PPACK, n * stride) : nullptr;
    if (!d_occ || !p.path_src || !p.path_dst || (packed && !d_pack) || (b->path_event && !p.path_event) || !p.path_count ||
        !p.total_displacement || !p.status || !p.detail || (b->events && !p.events))
        return cuda_fail(cudaErrorMemoryAllocation, "grid batch workspace", detail);
    // Chunks: chunk k's results go back on the copy stream while chunk k + 1
    // solves (the device-to-host copy of the path lists dominates, so it
    // overlaps the solve instead of following it).  Chunk sizes start at one
    // instance per SM and double up to a wave of CTAs, so the copy engine
    // starts after a short first solve; each chunk's inputs go up just
    // before its launch (the other direction of the link).
    if (!c->copy_stream) CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "copy stream");
    const size_t wave = (size_t)grid_blocks(c, solver, s, b->count);
    const size_t chunk_max = std::max<size_t>(wave, (n + 7) / 8);
    size_t chunk = std::min<size_t>(std::max(c->sms, 1), chunk_max);
    cudaStream_t cs = c->copy_stream;
    // any failure after the first copy: drain both streams before returning, so
    // no device-to-host copy of an earlier chunk is still writing into the
    // caller's buffers when the call returns
    auto drain = [&](recon_status st) {
        cudaStreamSynchronize(cs);
        cudaStreamSynchronize(c->stream);
        return st;
    };
#define CKD(call, where)                                                          \
    do {                                                                          \
        cudaError_t e_ = (call);                                                  \
        if (e_ != cudaSuccess) return drain(cuda_fail(e_, where, detail));        \
    } while (0)
    for (size_t i0 = 0, m = 0; i0 < n; i0 += m, chunk = std::min(chunk * 2, chunk_max)) {
        m = std::min(chunk, n - i0);
        CKD(cudaMemcpyAsync(d_occ + i0 * words, b->occ + i0 * words, m * words * 8, cudaMemcpyHostToDevice, c->stream),
           "occ H2D");
        GridParams q = p;
        q.count = (int)m;
        // the first chunk (one instance per SM) takes the lone-instance shape
        // (more warps per instance, shorter critical path): the copy engine
        // starts sooner; later chunks overlap copies and keep the batch shape
        GridShape sq = s;
        if (i0 == 0 && m <= (size_t)c->sms && m < n && !shape_for(c, solver, b->width, b->height, b->h_prime, (int)m, sq))
            sq = s;
        q.shape = sq;
        q.occ = d_occ + i0 * words;
        q.path_src = p.path_src + i0 * stride;
        q.path_dst = p.path_dst + i0 * stride;
        q.path_event = p.path_event ? p.path_event + i0 * stride : nullptr;
        q.path_count = p.path_count + i0;
        q.total_displacement = p.total_displacement + i0;
        q.status = p.status + i0;
        q.detail = p.detail + i0;
        q.events = p.events ? p.events + i0 * b->width * per : nullptr;
        CKD(launch(c, solver, q, grid_blocks(c, solver, sq, (int)m)), "grid kernel launch");
        if (packed) {
            pack_paths_kernel<<<c->sms * 8, 256, 0, c->stream>>>(q.path_src, q.path_dst, d_pack + i0 * stride, m * stride);
            ++c->launches;
            CKD(cudaGetLastError(), "pack kernel launch");
        }
        cudaEvent_t ev = c->chunk_event();
        if (!ev) return drain(cuda_fail(cudaErrorMemoryAllocation, "chunk event", detail));
        CKD(cudaEventRecord(ev, c->stream), "event");
        CKD(cudaStreamWaitEvent(cs, ev, 0), "wait");
        if (packed) {
            CKD(cudaMemcpyAsync(packed + i0 * stride, d_pack + i0 * stride, m * stride * 4, cudaMemcpyDeviceToHost, cs),
               "D2H");
        } else {
            CKD(cudaMemcpyAsync(b->path_src + i0 * stride, q.path_src, m * stride * 4, cudaMemcpyDeviceToHost, cs), "D2H");
            CKD(cudaMemcpyAsync(b->path_dst + i0 * stride, q.path_dst, m * stride * 4, cudaMemcpyDeviceToHost, cs), "D2H");
        }
        if (b->path_event)
            CKD(cudaMemcpyAsync(b->path_event + i0 * stride, q.path_event, m * stride * 4, cudaMemcpyDeviceToHost, cs),
               "D2H");
        CKD(cudaMemcpyAsync(b->path_count + i0, q.path_count, m * 4, cudaMemcpyDeviceToHost, cs), "D2H");
        CKD(cudaMemcpyAsync(b->total_displacement + i0, q.total_displacement, m * 8, cudaMemcpyDeviceToHost, cs), "D2H");
        CKD(cudaMemcpyAsync(b->status + i0, q.status, m * 4, cudaMemcpyDeviceToHost, cs), "D2H");
        if (b->detail) CKD(cudaMemcpyAsync(b->detail + i0, q.detail, m * 4, cudaMemcpyDeviceToHost, cs), "D2H");
        if (b->events)
            CKD(cudaMemcpyAsync(b->events + i0 * b->width * per, q.events, m * b->width * per * 4,
                               cudaMemcpyDeviceToHost, cs),
               "D2H");
    }
#undef CKD
    CK(cudaStreamSynchronize(c->stream), "grid batch");
    CK(cudaStreamSynchronize(cs), "grid batch D2H");
    return RECON_OK;
}

}  // namespace

extern "C" {

recon_status recon_redrec_solve(recon_ctx *ctx, const uint64_t *occ, int32_t width, int32_t height,
                                int32_t h_prime, recon_grid_solution *out, int32_t *detail) {
    return grid_single(0, ctx, occ, width, height, h_prime, out, detail);
}

recon_status recon_bird_solve(recon_ctx *ctx, const uint64_t *occ, int32_t width, int32_t height,
                              int32_t h_prime, recon_grid_solution *out, int32_t *detail) {
    return grid_single(1, ctx, occ, width, height, h_prime, out, detail);
}

recon_status recon_redrec_solve_batch(recon_ctx *ctx, const recon_grid_batch *b) { return grid_batch(0, ctx, b, false); }
recon_status recon_bird_solve_batch(recon_ctx *ctx, const recon_grid_batch *b) { return grid_batch(1, ctx, b, false); }
recon_status recon_redrec_solve_batch_host(recon_ctx *ctx, const recon_grid_batch *b) { return grid_batch(0, ctx, b, true); }
recon_status recon_bird_solve_batch_host(recon_ctx *ctx, const recon_grid_batch *b) { return grid_batch(1, ctx, b, true); }
recon_status recon_redrec_solve_batch_host_packed(recon_ctx *ctx, const recon_grid_batch *b, uint32_t *path_packed) {
    if (!path_packed) return RECON_ERR_ARGUMENT;
    return grid_batch(0, ctx, b, true, path_packed);
}
recon_status recon_bird_solve_batch_host_packed(recon_ctx *ctx, const recon_grid_batch *b, uint32_t *path_packed) {
    if (!path_packed) return RECON_ERR_ARGUMENT;
    return grid_batch(1, ctx, b, true, path_packed);
}

recon_status recon_occupancy_dag(recon_ctx *ctx, int32_t width, int32_t height, const int32_t *path_src,
                                 const int32_t *path_dst, int64_t path_count, int32_t *dag_src, int32_t *dag_dst,
                                 int64_t dag_capacity, int64_t *dag_count, int32_t *detail) {
    if (detail) *detail = 0;
    if (!dag_count || (path_count > 0 && (!path_src || !path_dst))) return RECON_ERR_ARGUMENT;
    if (width <= 0 || height <= 0) {
        if (detail) *detail = RECON_D_GRID_DIMENSIONS;
        return RECON_ERR_INPUT;
    }
    *dag_count = 0;
    if (path_count == 0) return RECON_OK;
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    int32_t *ds = c->dev<int32_t>(S_PSRC, (size_t)path_count), *dd = c->dev<int32_t>(S_PDST, (size_t)path_count);
    if (!ds || !dd) return cuda_fail(cudaErrorMemoryAllocation, "dag paths", detail);
    CK(cudaMemcpyAsync(ds, path_src, (size_t)path_count * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
    CK(cudaMemcpyAsync(dd, path_dst, (size_t)path_count * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
    return run_dag(c, width, height, ds, dd, path_count, dag_src, dag_dst, dag_capacity, dag_count, detail);
}

}  // extern "C"

// Profiling hook (not part of the public ABI): solves one instance and
// returns clock64 stamps at the kernel's phase boundaries (plan, phase 1 +
// pairing loop, phase 3) plus the phase-1 / loop event counts.
extern "C" recon_status recon_debug_grid_phases(int32_t solver, const uint64_t *occ, int32_t W, int32_t H,
                                                int32_t hp, long long *out6, int32_t nout) {
    int32_t *detail = nullptr;
    Ctx *c = resolve(nullptr);
    if (!c) return RECON_ERR_CUDA;
    GridShape s;
    if (!shape_for(c, solver, W, H, hp, 1, s)) return RECON_ERR_ARGUMENT;
    const size_t words = (size_t)W * s.wpd, stride = (size_t)W * hp;
    GridParams p{};
    p.shape = s;
    p.count = 1;
    uint64_t *d_occ = c->dev<uint64_t>(S_OCC, words);
    p.occ = d_occ;
    p.path_src = c->dev<int32_t>(S_PSRC, stride);
    p.path_dst = c->dev<int32_t>(S_PDST, stride);
    p.path_count = c->dev<int32_t>(S_PCNT, 1);
    p.total_displacement = c->dev<int64_t>(S_TDISP, 1);
    p.status = c->dev<int32_t>(S_STATUS, 1);
    p.detail = c->dev<int32_t>(S_DETAIL, 1);
    p.phase_clock = c->dev<long long>(S_KEYS, (size_t)(nout > 8 ? nout : 8));
    CK(cudaMemsetAsync(p.phase_clock, 0, (size_t)(nout > 8 ? nout : 8) * 8, c->stream), "memset");
    CK(cudaMemcpyAsync(d_occ, occ, words * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    CK(launch(c, solver, p, 1), "launch");
    CK(cudaMemcpyAsync(out6, p.phase_clock, (size_t)(nout > 6 ? nout : 6) * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaStreamSynchronize(c->stream), "sync");
    return RECON_OK;
}
