// C-ABI: batch_moves (batching.hpp:58-59) and the fused solve -> DAG ->
// batching pipeline over device-resident instances.

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cub/device/device_scan.cuh>
#include <vector>

#include "batching.cuh"
#include "capi_internal.cuh"
#include "grid_solver.cuh"

using namespace rb;

namespace {

#define CK(call, where)                                             \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return cuda_fail(e_, where, detail); \
    } while (0)

__global__ void copy_i32(int64_t n, const int32_t *a, int32_t *b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

// every instance's runs [0, min(count, stride)) straight into the caller's
// page-locked host arrays (device-mapped): one launch instead of two copies
// per instance; a CTA per instance, coalesced writes over the host link
__global__ void runs_to_host_kernel(int64_t n, int64_t rst, const int64_t *rc, const int32_t *rs, const int32_t *rb,
                                    int32_t *hs, int32_t *hb) {
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const int64_t R = min(rc[i], rst);
        const int32_t *s = rs + i * rst, *b = rb + i * rst;
        int32_t *ds = hs + i * rst, *db = hb + i * rst;
        for (int64_t j = threadIdx.x; j < R; j += blockDim.x) {
            ds[j] = s[j];
            db[j] = b[j];
        }
    }
}

// the device view of a page-locked, device-mapped host pointer (else NULL)
void *mapped_host(void *p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

// solved != NULL: recorded on the context stream once the solve's outputs
// (paths, counts, displacements) are final, before the DAG and batching
recon_status pipeline_impl(recon_ctx *ctx, const recon_pipeline_batch *pb, cudaEvent_t solved = nullptr) {
    int32_t *detail = nullptr;
    if (!pb) return RECON_ERR_ARGUMENT;
    const recon_grid_batch *b = &pb->grid;
    if (!b->occ || !b->path_src || !b->path_dst || !b->path_count || !b->total_displacement || !b->status ||
        !pb->move_batch || !pb->batch_count)
        return RECON_ERR_ARGUMENT;
    if (b->count <= 0) return RECON_OK;
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    // 1. solve on device
    recon_grid_batch g = *b;
    const size_t n = (size_t)b->count, S = (size_t)b->width * b->h_prime, WH = (size_t)b->width * b->height;
    cudaEvent_t *pev = (c->timing && c->pev[0]) ? c->pev : nullptr;
    c->timed_pipeline = pev != nullptr;
    if (pev) cudaEventRecord(pev[0], c->stream);
    // (a timed pipeline keeps the solve's own planner/executor events off)
    const bool kt = c->timing;
    if (pev) c->timing = false;
    recon_status st = pb->solver == 1 ? recon_bird_solve_batch(ctx, &g) : recon_redrec_solve_batch(ctx, &g);
    c->timing = kt;
    if (st != RECON_OK) return st;
    if (pev) cudaEventRecord(pev[1], c->stream);
    if (solved) CK(cudaEventRecord(solved, c->stream), "event");
    // 2. DAG + batching scratch
    PipelineArgs a{};
    a.count = b->count;
    a.W = b->width;
    a.H = b->height;
    a.k = b->h_prime;
    a.preset = pb->preset;
    a.path_src = g.path_src;
    a.path_dst = g.path_dst;
    a.path_count = g.path_count;
    a.solve_status = g.status;
    a.solve_detail = g.detail;
    a.move_stride = pb->move_stride;
    a.grid_occ = g.occ;
    // leap mode (batching.cu) for preset none on large grids;
    // RECON_BATCH_LEAP=0 forces the batch-by-batch loop, 2 forces leap mode
    static const int leap_env = [] {
        const char *e = getenv("RECON_BATCH_LEAP");
        return e ? atoi(e) : 1;
    }();
    // (small grids: the batch-by-batch loop with the move log and the
    // blocker counts in shared memory is faster, 7.0 vs 9.2 ms on C3)
    a.leap = pb->preset == 0 && (leap_env == 1 ? S >= 16384 : leap_env == 2);
    // wide phase (batch_wide.cu) for large instances; RECON_BATCH_WIDE=0/1 forces
    static const int wide_env = [] {
        const char *e = getenv("RECON_BATCH_WIDE");
        return e ? atoi(e) : -1;
    }();
    a.wide = wide_env >= 0 ? wide_env : (S >= 16384 ? 1 : 0);
    // path records (packed coordinates, move base, successor offset): the DAG
    // walk, the wide phase and leap mode read them
    a.prec = c->dev<int4>(S_BM_PREC, n * (S + 1));
    if (!a.prec) return cuda_fail(cudaErrorMemoryAllocation, "pipeline prec", detail);
    if (a.wide) {
        a.wstate = c->dev<int64_t>(S_BM_WSTATE, n * 4 + 1);
        a.wnext = a.wstate ? reinterpret_cast<int32_t *>(a.wstate + n * 4) : nullptr;
        a.vmin = c->dev<int32_t>(S_BM_VMIN, n * WH);
        if (!a.wstate || !a.vmin) return cuda_fail(cudaErrorMemoryAllocation, "pipeline wide", detail);
    }
    const size_t nwb = (WH + 31) / 32;
    static const int small_env = [] {
        const char *e = getenv("RECON_SMALL_DAG");
        return e ? atoi(e) : 1;
    }();
    a.small_dag = small_env && pipeline_small_dag_smem(a.W, a.H, a.k) > 0;
    // per-instance vertex maps only for the global DAG walk: {source, target}
    // owner per vertex, column-major and row-major
    // + the coverage difference arrays (batching.cu pl_mark2_kernel)
    const size_t maps = a.small_dag ? 0 : n * WH * 8 + n * ((size_t)b->height * (b->width + 1) + (size_t)b->width * (b->height + 1));
    int32_t *i32 = c->dev<int32_t>(S_BM_AUX0, maps + n * S * 9 + n * 2 + 8);
    int64_t *i64 = c->dev<int64_t>(S_BM_AUX1, (n * S + 1) * 2 + 4 * (n + 1) + 4);
    uint32_t *bits = c->dev<uint32_t>(S_BM_AUX2, n * nwb * 2 + 4);
    int4 *rec = c->dev<int4>(S_BM_AUX7, n * S * 2 + 4);
    int32_t *mb = pb->move_batch;
    int32_t *bc = pb->batch_count;
    int32_t *bst = g.status;  // batching status (overwrites the solve status)
    int32_t *bdet = g.detail;
    if (!i32 || !i64 || !bits || !rec) return cuda_fail(cudaErrorMemoryAllocation, "pipeline", detail);
    a.source_of = maps ? i32 : nullptr;  // int2 maps (batching.cu pl_mark2_kernel)
    a.target_of = nullptr;
    int32_t *q = i32 + maps;
    a.outdeg = q;
    a.slen = a.small_dag ? nullptr : a.outdeg;  // (pl_compact_kernel's list lengths)
    a.indeg = q + n * S;
    a.fill = q + 2 * n * S;
    a.newly = q + 3 * n * S;
    a.mem = q + 4 * n * S;
    a.mfr = q + 5 * n * S;
    a.mto = q + 6 * n * S;
    a.rb = q + 7 * n * S;   // ready records' move bases (batch_warp_pipe)
    a.rb2 = q + 8 * n * S;
    a.counter = q + 9 * n * S;
    a.rec = rec;  // ready records
    a.rec2 = rec + n * S;
    a.soff = i64;
    a.mbase = i64 + n * S + 1;
    a.inst_edges = i64 + 2 * (n * S + 1);
    a.inst_moves = a.inst_edges + (n + 1);
    a.ebase = a.inst_moves + (n + 1);
    a.mvbase = a.ebase + (n + 1);
    a.occ = bits;
    a.inb = bits + n * nwb;
    a.move_batch = mb;
    a.batch_count = bc;
    a.status = bst;
    a.detail = bdet;
    a.temp_bytes = pipeline_temp_bytes((int64_t)(n * S + 1));
    a.temp = c->get(S_TEMP, a.temp_bytes);
    if (!a.temp) return cuda_fail(cudaErrorMemoryAllocation, "pipeline temp", detail);
    int64_t counts[2] = {0, 0};
    CK(pipeline_dag_count(a, c->stream, counts, &c->launches), "pipeline dag");
    const int64_t edges = counts[0];
    a.succ = c->dev<int32_t>(S_BM_AUX5, (size_t)edges + 1);
    a.edge_capacity = edges;
    if (!a.succ) return cuda_fail(cudaErrorMemoryAllocation, "pipeline succ", detail);
    // move log (scattered into move_batch by each warp when its instance
    // finishes) for many small instances, whose scattered move_batch stores
    // otherwise miss L2 one 4-byte store at a time; large instances (whose log
    // would cost 8 B per move of HBM) write move_batch directly.
    // RECON_BATCH_LOG=0/1 forces.
    static const int log_env = [] {
        const char *e = getenv("RECON_BATCH_LOG");
        return e ? atoi(e) : -1;
    }();
    const bool use_log = !a.leap && (log_env >= 0 ? log_env == 1 : (n >= (size_t)c->sms * 4 && 2 * nwb * 4 <= 32 * 1024));
    a.mlog = nullptr;
    if (use_log) {
        a.mlog = c->dev<int2>(S_BM_AUX6, (size_t)counts[1] + 1);
        if (!a.mlog) return cuda_fail(cudaErrorMemoryAllocation, "pipeline move log", detail);
    }
    CK(pipeline_run_batching(a, c->sms, c->stream, pev, &c->launches), "pipeline batching");
    return RECON_OK;
}

// Host buffers: the instances go through the device pipeline in sub-chunks
// sized to free HBM.  Each sub-chunk's outputs sit in one of
// two device slots; its device-to-host copies (per instance only the used
// [0, D) of the schedule) run on the copy stream while the next sub-chunk is
// solved and batched on the context stream.
// runs != NULL: the schedule comes back as runs (recon_schedule_runs, host
// pointers) instead of move_batch, which may then be NULL.
recon_status pipeline_host_chunked(recon_ctx *ctx, const recon_pipeline_batch *pb, recon_schedule_runs *runs) {
    int32_t *detail = nullptr;
    if (!pb) return RECON_ERR_ARGUMENT;
    const recon_grid_batch *b = &pb->grid;
    if (!b->occ || !b->path_src || !b->path_dst || !b->path_count || !b->total_displacement || !b->status ||
        (!pb->move_batch && !runs) || !pb->batch_count)
        return RECON_ERR_ARGUMENT;
    if (runs && (!runs->run_slot || !runs->run_batch || !runs->run_count || runs->run_stride <= 0))
        return RECON_ERR_ARGUMENT;
    if (b->count <= 0) return RECON_OK;
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    if (!c->copy_stream) CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "copy stream");
    cudaStream_t cs = c->copy_stream;
    const size_t S = (size_t)b->width * b->h_prime, WH = (size_t)b->width * b->height;
    const int wpc = (b->height + 63) / 64;
    const size_t occ_words = (size_t)b->width * wpc;
    // sub-chunk: what free memory holds (two output slots + the pipeline
    // workspace, ~48 successor edges per path); RECON_PIPE_HOST_CHUNK forces
    // runs: the copies are small, so one output slot (the next sub-chunk waits
    // for them); per-move schedules: two slots, copies overlap the next solve
    const int nslots = runs ? 1 : 2;
    // the pipeline workspace (grow-only) counts only when it must still grow:
    // the ready-record slot holds 32 B per path slot
    const bool warm = c->buf[S_BM_AUX7].bytes >= (size_t)b->count * S * 32;
    const size_t per = nslots * (occ_words * 8 + 8 * S + 32 + (size_t)pb->move_stride * 4) +
                       (warm ? 0 : (40 * WH + 36 * S + 16 * S + 32 * S + 16 * S + WH / 4 + 4 * WH + 192 * S));
    static const int env_chunk = [] {
        const char *e = getenv("RECON_PIPE_HOST_CHUNK");
        return e ? atoi(e) : 0;
    }();
    size_t sub = env_chunk > 0 ? (size_t)env_chunk : 0;
    if (!sub) {
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot), "cudaMemGetInfo");
        // the output slots this context already holds count as available
        size_t have = 0;
        for (int sl_ = S_PH_OCC0; sl_ <= S_PH_RC1; ++sl_) have += c->buf[sl_].bytes;
        sub = std::max<size_t>(1, (size_t)(0.8 * (double)fr + (double)have) / per);
        // two sub-chunks at least, so that copies overlap the next solve
        // (runs: the copies are small, one sub-chunk pays the batching
        // latency once)
        if ((size_t)b->count > 1 && !runs) sub = std::min(sub, ((size_t)b->count + 1) / 2);
    }
    sub = std::min(sub, (size_t)b->count);
    // the two device output slots
    struct Slot {
        uint64_t *occ;
        int32_t *src, *dst, *ev, *i32, *mb, *rs, *rb;
        int64_t *i64, *rc;
        cudaEvent_t done = nullptr;  // its copies are finished
    } sl[2];
    // (out of memory: release the output slots and halve the sub-chunk)
    for (int k = 0; k < nslots; ++k) {
        sl[k].occ = c->dev<uint64_t>(S_PH_OCC0 + k, sub * occ_words);
        sl[k].src = c->dev<int32_t>(S_PH_SRC0 + k, sub * S);
        sl[k].dst = c->dev<int32_t>(S_PH_DST0 + k, sub * S);
        sl[k].ev = b->path_event ? c->dev<int32_t>(S_PH_EV0 + k, sub * S) : nullptr;
        sl[k].i32 = c->dev<int32_t>(S_PH_I32_0 + k, sub * 4);  // path_count | status | detail | batch_count
        sl[k].i64 = c->dev<int64_t>(S_PH_I64_0 + k, sub);
        sl[k].mb = c->dev<int32_t>(S_PH_MB0 + k, sub * (size_t)pb->move_stride);
        sl[k].rs = sl[k].rb = nullptr;
        sl[k].rc = nullptr;
        if (runs) {
            sl[k].rs = c->dev<int32_t>(S_PH_RS0 + k, sub * (size_t)runs->run_stride * 2);
            sl[k].rb = sl[k].rs ? sl[k].rs + sub * (size_t)runs->run_stride : nullptr;
            sl[k].rc = c->dev<int64_t>(S_PH_RC0 + k, sub);
        }
        if (!sl[k].occ || !sl[k].src || !sl[k].dst || (b->path_event && !sl[k].ev) || !sl[k].i32 || !sl[k].i64 ||
            !sl[k].mb || (runs && (!sl[k].rs || !sl[k].rc))) {
            if (sub == 1) return cuda_fail(cudaErrorMemoryAllocation, "pipeline host slots", detail);
            for (int sl_ = S_PH_OCC0; sl_ <= S_PH_RC1; ++sl_) {
                if (c->buf[sl_].p) cudaFree(c->buf[sl_].p);
                c->buf[sl_].p = nullptr;
                c->buf[sl_].bytes = 0;
            }
            sub = (sub + 1) / 2;
            k = -1;  // (the loop's ++k restarts at slot 0)
        }
    }
    std::vector<int64_t> hD(sub), hR(sub);
    // page-locked, device-mapped run arrays: written by a kernel, not copied
    int32_t *hs_map = runs ? static_cast<int32_t *>(mapped_host(runs->run_slot)) : nullptr;
    int32_t *hb_map = runs ? static_cast<int32_t *>(mapped_host(runs->run_batch)) : nullptr;
    bool over = false;  // some instance had more runs than run_stride
    // on any failure after copies were issued: drain both streams before returning
    auto fail = [&](recon_status st) {
        cudaStreamSynchronize(cs);
        cudaStreamSynchronize(c->stream);
        return st;
    };
#define CKF(call, where)                                                         \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess) return fail(cuda_fail(e_, where, detail));        \
    } while (0)
    int k = 0;
    for (size_t j0 = 0; j0 < (size_t)b->count; j0 += sub, k = (k + 1) % nslots) {
        const size_t n = std::min(sub, (size_t)b->count - j0);
        Slot &o = sl[k];
        if (o.done) CKF(cudaStreamWaitEvent(c->stream, o.done, 0), "wait slot");
        CKF(cudaMemcpyAsync(o.occ, b->occ + j0 * occ_words, n * occ_words * 8, cudaMemcpyHostToDevice, c->stream),
            "H2D");
        recon_pipeline_batch d = *pb;
        d.grid.occ = o.occ;
        d.grid.count = (int32_t)n;
        d.grid.path_src = o.src;
        d.grid.path_dst = o.dst;
        d.grid.path_event = o.ev;
        d.grid.path_count = o.i32;
        d.grid.status = o.i32 + n;
        d.grid.detail = o.i32 + 2 * n;
        d.grid.total_displacement = o.i64;
        d.grid.events = nullptr;
        d.batch_count = o.i32 + 3 * n;
        d.move_batch = o.mb;
        static const bool trace = getenv("RECON_PIPE_HOST_TRACE") != nullptr;
        auto stamp = [&](const char *what) {
            if (!trace) return;
            cudaStreamSynchronize(c->stream);
            fprintf(stderr, "[pipe host] sub-chunk %zu (n=%zu): %s %.3f ms\n", j0, n, what,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count());
        };
        stamp("start");
        cudaEvent_t solved = c->chunk_event();
        if (!solved) return fail(cuda_fail(cudaErrorUnknown, "event", detail));
        const recon_status st = pipeline_impl(ctx, &d, solved);
        if (st != RECON_OK) return fail(st);
        stamp("pipeline");
        // the solve's outputs are final: their copies (most of the bytes, 8 B
        // per path slot) overlap the DAG and the batching still running
        CKF(cudaStreamWaitEvent(cs, solved, 0), "wait");
        CKF(cudaMemcpyAsync(b->path_src + j0 * S, o.src, n * S * 4, cudaMemcpyDeviceToHost, cs), "D2H");
        CKF(cudaMemcpyAsync(b->path_dst + j0 * S, o.dst, n * S * 4, cudaMemcpyDeviceToHost, cs), "D2H");
        if (b->path_event) CKF(cudaMemcpyAsync(b->path_event + j0 * S, o.ev, n * S * 4, cudaMemcpyDeviceToHost, cs), "D2H");
        CKF(cudaMemcpyAsync(b->path_count + j0, o.i32, n * 4, cudaMemcpyDeviceToHost, cs), "D2H");
        CKF(cudaMemcpyAsync(b->total_displacement + j0, o.i64, n * 8, cudaMemcpyDeviceToHost, cs), "D2H");
        recon_schedule_runs dr{};
        if (runs) {
            dr = recon_schedule_runs{runs->run_stride, o.rs, o.rb, o.rc};
            CKF(launch_schedule_runs(d, dr, c->sms, c->stream), "schedule runs");
            ++c->launches;
            CKF(cudaMemcpyAsync(hR.data(), o.rc, n * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
        }
        // every instance's displacement, then only [0, D) of its schedule
        CKF(cudaMemcpyAsync(hD.data(), o.i64, n * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
        CKF(cudaStreamSynchronize(c->stream), "pipeline sub-chunk");
        stamp("runs + counts");
        cudaEvent_t batched = c->chunk_event();
        if (!batched) return fail(cuda_fail(cudaErrorUnknown, "event", detail));
        CKF(cudaEventRecord(batched, c->stream), "event");
        CKF(cudaStreamWaitEvent(cs, batched, 0), "wait");
        CKF(cudaMemcpyAsync(b->status + j0, o.i32 + n, n * 4, cudaMemcpyDeviceToHost, cs), "D2H");
        if (b->detail) CKF(cudaMemcpyAsync(b->detail + j0, o.i32 + 2 * n, n * 4, cudaMemcpyDeviceToHost, cs), "D2H");
        CKF(cudaMemcpyAsync(pb->batch_count + j0, o.i32 + 3 * n, n * 4, cudaMemcpyDeviceToHost, cs), "D2H");
        for (size_t i = 0; i < n && pb->move_batch; ++i) {
            const int64_t D = std::min<int64_t>(std::max<int64_t>(hD[i], 0), pb->move_stride);
            if (D > 0)
                CKF(cudaMemcpyAsync(pb->move_batch + (j0 + i) * (size_t)pb->move_stride,
                                    o.mb + i * (size_t)pb->move_stride, (size_t)D * 4, cudaMemcpyDeviceToHost, cs),
                    "D2H");
        }
        if (runs) {
            const size_t rst = (size_t)runs->run_stride;
            CKF(cudaMemcpyAsync(runs->run_count + j0, o.rc, n * 8, cudaMemcpyDeviceToHost, cs), "D2H");
            for (size_t i = 0; i < n; ++i) over |= hR[i] > runs->run_stride;
            if (hs_map && hb_map) {
                runs_to_host_kernel<<<(int)std::min<size_t>(n, (size_t)c->sms * 8), 256, 0, cs>>>(
                    (int64_t)n, (int64_t)rst, o.rc, o.rs, o.rb, hs_map + j0 * rst, hb_map + j0 * rst);
                CKF(cudaGetLastError(), "runs to host");
                ++c->launches;
            }
            for (size_t i = 0; i < n && !(hs_map && hb_map); ++i) {
                const int64_t R = std::min<int64_t>(hR[i], runs->run_stride);
                if (R <= 0) continue;
                CKF(cudaMemcpyAsync(runs->run_slot + (j0 + i) * rst, o.rs + i * rst, (size_t)R * 4,
                                    cudaMemcpyDeviceToHost, cs), "D2H");
                CKF(cudaMemcpyAsync(runs->run_batch + (j0 + i) * rst, o.rb + i * rst, (size_t)R * 4,
                                    cudaMemcpyDeviceToHost, cs), "D2H");
            }
        }
        o.done = c->chunk_event();
        if (!o.done) return fail(cuda_fail(cudaErrorUnknown, "event", detail));
        CKF(cudaEventRecord(o.done, cs), "event");
    }
#undef CKF
    CK(cudaStreamSynchronize(cs), "pipeline copies");
    if (getenv("RECON_PIPE_HOST_TRACE"))
        fprintf(stderr, "[pipe host] copies done %.3f ms (sub=%zu)\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(), sub);
    return over ? RECON_ERR_CAPACITY : RECON_OK;
}

}  // namespace

extern "C" {

recon_status recon_batch_moves(recon_ctx *ctx, int32_t width, int32_t height, const uint64_t *occ, int32_t P,
                               const int64_t *off, const int32_t *verts, int64_t E, const int32_t *es,
                               const int32_t *ed, int32_t preset, int32_t edge_level, int32_t *move_batch,
                               int64_t *batch_count, int32_t *detail) {
    if (detail) *detail = 0;
    if (!batch_count || (P > 0 && (!off || !verts || !occ)) || (E > 0 && (!es || !ed))) return RECON_ERR_ARGUMENT;
    if (width <= 0 || height <= 0) {
        if (detail) *detail = RECON_D_GRID_DIMENSIONS;
        return RECON_ERR_INPUT;
    }
    *batch_count = 0;
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    cudaStream_t st = c->stream;
    const int64_t WH = (int64_t)width * height, nwb = (WH + 31) / 32;
    const int64_t nverts = P > 0 ? off[P] : 0, moves = nverts - P;
    const int wpc = (height + 63) / 64;
    // device buffers
    int64_t *d_off = c->dev<int64_t>(S_BM_OFF, (size_t)P + 2);
    int32_t *d_verts = c->dev<int32_t>(S_BM_VERT, (size_t)nverts + 1);
    int32_t *d_es = c->dev<int32_t>(S_BM_ES, (size_t)E + 1), *d_ed = c->dev<int32_t>(S_BM_ED, (size_t)E + 1);
    int32_t *d_out = c->dev<int32_t>(S_BM_OUT, (size_t)moves + 1);
    uint64_t *d_occ = c->dev<uint64_t>(S_OCC, (size_t)width * wpc);
    // i32: outdeg[P+1] indeg[P+1] fill[P+1] fill2[P+1] succ[E] in_src[E] misc[16] ar[12P]
    const size_t n32 = 4 * ((size_t)P + 1) + 2 * (size_t)E + 16 + 12 * (size_t)P + 16;
    int32_t *i32 = c->dev<int32_t>(S_BM_AUX0, n32);
    int64_t *i64 = c->dev<int64_t>(S_BM_AUX1, 2 * ((size_t)P + 2) + 2 * ((size_t)E + 1) + 4);
    uint32_t *bits = c->dev<uint32_t>(S_BM_AUX2, 2 * (size_t)nwb + 2);
    uint8_t *done = c->dev<uint8_t>(S_BM_AUX3, (size_t)P + 16);
    if (!d_off || !d_verts || !d_es || !d_ed || !d_out || !d_occ || !i32 || !i64 || !bits || !done)
        return cuda_fail(cudaErrorMemoryAllocation, "batch_moves workspace", detail);
    int32_t *outdeg = i32, *indeg = outdeg + (P + 1), *fill = indeg + (P + 1), *fill2 = fill + (P + 1);
    int32_t *succ = fill2 + (P + 1), *in_src = succ + E, *misc = in_src + E, *ar = misc + 16;
    int32_t *bad = misc, *processed = misc + 1, *counter = misc + 2, *res = misc + 4;
    int64_t *soff = i64, *in_off = soff + (P + 2), *need = in_off + (P + 2), *need_sorted = need + (E + 1);
    CK(cudaMemsetAsync(i32, 0, n32 * 4, st), "memset");
    if (P > 0) {
        CK(cudaMemcpyAsync(d_off, off, ((size_t)P + 1) * 8, cudaMemcpyHostToDevice, st), "H2D");
        CK(cudaMemcpyAsync(d_verts, verts, (size_t)nverts * 4, cudaMemcpyHostToDevice, st), "H2D");
    }
    if (E > 0) {
        CK(cudaMemcpyAsync(d_es, es, (size_t)E * 4, cudaMemcpyHostToDevice, st), "H2D");
        CK(cudaMemcpyAsync(d_ed, ed, (size_t)E * 4, cudaMemcpyHostToDevice, st), "H2D");
    }
    CK(cudaMemcpyAsync(d_occ, occ, (size_t)width * wpc * 8, cudaMemcpyHostToDevice, st), "H2D");
    const int blocks = 148 * 4;
    // MoveDag::is_acyclic (batching.cpp:34): endpoint range + Kahn
    edges_check_kernel<<<blocks, 256, 0, st>>>(P, E, d_es, d_ed, bad, outdeg, indeg);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, (const int32_t *)nullptr, (int64_t *)nullptr, P + 1);
    void *temp = c->get(S_TEMP, tb);
    if (!temp) return cuda_fail(cudaErrorMemoryAllocation, "temp", detail);
    // soff = exclusive scan of outdeg (widened)
    {
        std::vector<int32_t> h_bad(1);
        CK(cudaMemcpyAsync(h_bad.data(), bad, 4, cudaMemcpyDeviceToHost, st), "D2H");
        CK(cudaStreamSynchronize(st), "check");
        if (h_bad[0]) {
            if (detail) *detail = RECON_D_BATCH_CYCLIC;
            return RECON_ERR_INPUT;
        }
    }
    auto widen_scan = [&](const int32_t *deg, int64_t *out) -> cudaError_t {
        size_t t2 = tb;
        return cub::DeviceScan::ExclusiveSum(temp, t2, deg, out, P + 1, st);
    };
    CK(cudaMemsetAsync(outdeg + P, 0, 4, st), "memset");
    CK(widen_scan(outdeg, soff), "scan");
    csr_fill_kernel<<<blocks, 256, 0, st>>>(E, d_es, d_ed, soff, fill, succ, nullptr, nullptr);
    // Kahn on a copy of the in-degrees
    int32_t *indeg_copy = ar + 10 * P;  // ar[10P, 11P)
    copy_i32<<<blocks, 256, 0, st>>>(P, indeg, indeg_copy);
    kahn_kernel<<<1, 1024, 0, st>>>(P, soff, succ, indeg_copy, ar, ar + P, processed);
    c->launches += 5;
    int32_t h_proc = 0;
    CK(cudaMemcpyAsync(&h_proc, processed, 4, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaStreamSynchronize(st), "kahn");
    if (h_proc != P) {
        if (detail) *detail = RECON_D_BATCH_CYCLIC;
        return RECON_ERR_INPUT;
    }
    BatchJob J{};
    J.P = P;
    J.W = width;
    J.H = height;
    J.preset = preset;
    J.edge_level = edge_level ? 1 : 0;
    J.soff = soff;
    J.succ = succ;
    if (edge_level) {
        // incoming CSR with release thresholds (batching.cpp:38-59)
        need_kernel<<<blocks, 256, 0, st>>>(E, d_es, d_ed, d_off, d_verts, need);
        CK(cudaMemsetAsync(indeg + P, 0, 4, st), "memset");
        size_t t2 = tb;
        CK(cub::DeviceScan::ExclusiveSum(temp, t2, indeg, in_off, P + 1, st), "scan");
        csr_fill_kernel<<<blocks, 256, 0, st>>>(E, d_ed, d_es, in_off, fill2, in_src, need, need_sorted);
        J.in_off = in_off;
        J.in_src = in_src;
        J.in_need = need_sorted;
        c->launches += 2;
    }
    J.s.occ = bits;
    J.s.inb = bits + nwb;
    occ_to_vertex_bits<<<blocks, 256, 0, st>>>(1, width, height, d_occ, bits);
    CK(cudaMemsetAsync(bits + nwb, 0, (size_t)nwb * 4, st), "memset");
    J.s.next = ar;
    J.s.blockers = indeg;
    J.s.done = done;
    J.s.ready = ar + P;
    J.s.ready2 = ar + 2 * P;
    J.s.newly = ar + 3 * P;
    J.s.mem = ar + 4 * P;
    J.s.mfr = ar + 5 * P;
    J.s.mto = ar + 6 * P;
    J.s.counter = counter;
    J.move_batch = d_out;
    J.batch_count = res;
    J.status = res + 1;
    J.detail = res + 2;
    CK(launch_batch_explicit(J, d_off, d_verts, st), "batch launch");
    c->launches += 2;
    int32_t h_res[3];
    CK(cudaMemcpyAsync(h_res, res, 12, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaStreamSynchronize(st), "batching");
    if (h_res[1] != RECON_OK) {
        if (detail) *detail = h_res[2];
        return (recon_status)h_res[1];
    }
    *batch_count = h_res[0];
    if (moves > 0) {
        CK(cudaMemcpyAsync(move_batch, d_out, (size_t)moves * 4, cudaMemcpyDeviceToHost, st), "D2H");
        CK(cudaStreamSynchronize(st), "D2H");
    }
    return RECON_OK;
}

recon_status recon_pipeline_batch_run(recon_ctx *ctx, const recon_pipeline_batch *pb) {
    return pipeline_impl(ctx, pb);
}

recon_status recon_pipeline_batch_run_host(recon_ctx *ctx, const recon_pipeline_batch *pb) {
    return pipeline_host_chunked(ctx, pb, nullptr);
}

recon_status recon_pipeline_batch_run_host_runs(recon_ctx *ctx, const recon_pipeline_batch *pb,
                                                recon_schedule_runs *runs) {
    if (!runs) return RECON_ERR_ARGUMENT;
    return pipeline_host_chunked(ctx, pb, runs);
}

}  // extern "C"
