// C-ABI entry points (include/recon_b200.h) over the sm_100a kernels.
//
// Host code only: argument validation in the reference's error order,
// device workspace management per context, host<->device copies for the
// host-buffer entry points, kernel launches.  There is no CPU compute path:
// without a usable CUDA device every solver returns RECON_ERR_CUDA.

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "capi_internal.cuh"

thread_local std::string g_last_cuda_error;

namespace rb {

void set_cuda_error(cudaError_t e, const char *where) {
    g_last_cuda_error = std::string(where) + ": " + cudaGetErrorString(e);
}

void *Ctx::get(int slot, size_t bytes) {
    DevBuf &b = buf[slot];
    if (b.bytes >= bytes && b.p) return b.p;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    size_t want = bytes < 256 ? 256 : bytes;
    if (cudaMalloc(&b.p, want) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    b.bytes = want;
    return b.p;
}

void *Ctx::host(int slot, size_t bytes) {
    HostBuf &b = hbuf[slot];
    if (b.bytes >= bytes && b.p) return b.p;
    if (b.p) cudaFreeHost(b.p);
    b.p = nullptr;
    b.bytes = 0;
    size_t want = bytes < 256 ? 256 : bytes;
    if (cudaMallocHost(&b.p, want) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    b.bytes = want;
    return b.p;
}

Ctx::~Ctx() {
    for (auto &b : buf)
        if (b.p) cudaFree(b.p);
    for (auto &b : hbuf)
        if (b.p) cudaFreeHost(b.p);
    for (auto &e : tev)
        if (e) cudaEventDestroy(e);
    for (auto &e : cev)
        if (e) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (stream) cudaStreamDestroy(stream);
}

static thread_local Ctx *tl_default = nullptr;

Ctx *resolve(recon_ctx *ctx) {
    if (ctx) return reinterpret_cast<Ctx *>(ctx);
    if (!tl_default) {
        recon_ctx *c = nullptr;
        if (recon_ctx_create(-1, &c) != RECON_OK) return nullptr;
        tl_default = reinterpret_cast<Ctx *>(c);
    }
    return tl_default;
}

recon_status cuda_fail(cudaError_t e, const char *where, int32_t *detail) {
    set_cuda_error(e, where);
    if (detail) *detail = RECON_D_CUDA;
    return RECON_ERR_CUDA;
}

}  // namespace rb

using namespace rb;

extern "C" {

const char *recon_detail_message(int32_t detail) {
    switch (detail) {
        case RECON_D_FEWER_SOURCES: return "fewer sources than targets (|S| < |T|)";
        case RECON_D_BAND_NOT_CENTERED: return "targets must form a centered full-width band";
        case RECON_D_BAND_HEIGHT: return "target band height must be in (0, H)";
        case RECON_D_BAND_EMPTY: return "target band is empty";
        case RECON_D_NO_DEFICIT: return "select_best_pair: no deficit column remains";
        case RECON_D_NO_DONOR: return "select_best_pair: deficit column with no admissible donor";
        case RECON_D_BATCH_NO_PROGRESS: return "batching made no progress (blocked dependency structure)";
        case RECON_D_BATCH_CYCLIC: return "batching requires an acyclic dependency dag";
        case RECON_D_CHAIN_LENGTH: return "chain length must be positive";
        case RECON_D_SOURCE_OOB: return "source vertex out of bounds";
        case RECON_D_SOURCE_ORDER: return "source vertices must be strictly increasing";
        case RECON_D_TARGET_OOB: return "target vertex out of bounds";
        case RECON_D_TARGET_ORDER: return "target vertices must be strictly increasing";
        case RECON_D_GEN_MULTIPLICITY: return "source multiplicity must be at least 1";
        case RECON_D_GEN_MIN_USE: return "source min_use outside [0, multiplicity]";
        case RECON_D_GEN_SOURCE_ORDER: return "source positions must be strictly increasing";
        case RECON_D_GEN_TARGET_ORDER: return "target positions must be strictly increasing";
        case RECON_D_GEN_SUPPLY: return "insufficient tokens for targets";
        case RECON_D_GEN_MANDATORY: return "mandatory draws exceed target count";
        case RECON_D_GEN_NO_ASSIGNMENT: return "no assignment satisfies the usage bounds";
        case RECON_D_DAG_EDGE_RANGE: return "dag edge endpoint out of range";
        case RECON_D_GRID_DIMENSIONS: return "grid dimensions must be positive";
        case RECON_D_INFEASIBLE_SUPPLY: return "fewer sources than targets";
        case RECON_D_CUDA: return "CUDA runtime failure";
        default: return "";
    }
}

const char *recon_last_cuda_error(void) { return g_last_cuda_error.c_str(); }
int32_t recon_abi_version(void) { return RECON_ABI_VERSION; }

recon_status recon_ctx_create(int32_t device, recon_ctx **out) {
    if (!out) return RECON_ERR_ARGUMENT;
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        g_last_cuda_error = std::string("no CUDA device: ") + (e != cudaSuccess ? cudaGetErrorString(e) : "count 0");
        return RECON_ERR_CUDA;
    }
    if (device < 0) {
        if (cudaGetDevice(&device) != cudaSuccess) device = 0;
    }
    if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice", nullptr);
    Ctx *c = new Ctx();
    c->device = device;
    if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaStreamCreate", nullptr);
    }
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, device);
    c->sms = prop.multiProcessorCount;
    *out = reinterpret_cast<recon_ctx *>(c);
    return RECON_OK;
}

void recon_ctx_destroy(recon_ctx *ctx) { delete reinterpret_cast<Ctx *>(ctx); }

void *recon_ctx_stream(recon_ctx *ctx) {
    Ctx *c = resolve(ctx);
    return c ? (void *)c->stream : nullptr;
}

int64_t recon_ctx_launch_count(recon_ctx *ctx) {
    Ctx *c = resolve(ctx);
    return c ? c->launches : 0;
}

recon_status recon_ctx_set_kernel_timing(recon_ctx *ctx, int32_t enable) {
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    if (enable && !c->tev[0]) {
        for (auto &e : c->tev) {
            cudaError_t err = cudaEventCreate(&e);
            if (err != cudaSuccess) return cuda_fail(err, "cudaEventCreate", nullptr);
        }
        for (auto &e : c->pev) {
            cudaError_t err = cudaEventCreate(&e);
            if (err != cudaSuccess) return cuda_fail(err, "cudaEventCreate", nullptr);
        }
    }
    c->timing = enable != 0;
    return RECON_OK;
}

recon_status recon_ctx_phase_times(recon_ctx *ctx, float *ms, int32_t n) {
    Ctx *c = resolve(ctx);
    if (!c || !ms) return RECON_ERR_ARGUMENT;
    for (int32_t i = 0; i < n; ++i) ms[i] = 0.0f;
    if (!c->pev[0] || !c->timed_pipeline) return RECON_OK;
    cudaError_t e = cudaEventSynchronize(c->pev[4]);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize", nullptr);
    for (int32_t i = 0; i < n && i < 4; ++i) cudaEventElapsedTime(&ms[i], c->pev[i], c->pev[i + 1]);
    return RECON_OK;
}

recon_status recon_ctx_kernel_times(recon_ctx *ctx, float *ms, int32_t n) {
    Ctx *c = resolve(ctx);
    if (!c || !ms) return RECON_ERR_ARGUMENT;
    for (int32_t i = 0; i < n; ++i) ms[i] = 0.0f;
    if (!c->tev[0]) return RECON_OK;
    cudaError_t e = cudaEventSynchronize(c->tev[2]);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize", nullptr);
    float t[2] = {0.0f, 0.0f};
    if (c->timed_plan) cudaEventElapsedTime(&t[0], c->tev[0], c->tev[1]);
    cudaEventElapsedTime(&t[1], c->tev[1], c->tev[2]);
    for (int32_t i = 0; i < n && i < 2; ++i) ms[i] = t[i];
    return RECON_OK;
}

}  // extern "C"
