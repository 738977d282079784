// Host side of the grid solvers: shape/shared-memory sizing and launches of
// redrec_kernel (redrec.cu) and bird_kernel (bird.cu).

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "grid_common.cuh"

namespace rb {

template <int MINB>
__global__ void redrec_kernel(GridParams p);

// executor variant: 32-warp CTAs for lone instances, else 8-warp CTAs with
// MINB per SM (RECON_REDREC_MINB = 3 trades occupancy for 85 registers)
static void (*redrec_exec(const GridShape &s))(GridParams) {
    if (s.nwarps > 8) return redrec_kernel<1>;
    static const int minb = [] {
        const char *e = getenv("RECON_REDREC_MINB");
        return e ? atoi(e) : 4;
    }();
    return minb == 3 ? redrec_kernel<3> : redrec_kernel<4>;
}
__global__ void redrec_plan_kernel(GridParams p);
int64_t redrec_plan_smem(int W);
template <int MODE>
__global__ void bird_kernel(GridParams p);
static void (*bird_exec(const GridShape &s))(GridParams) {
    if (s.nwarps > 8) return bird_kernel<1>;
    return (long long)s.W * s.H >= 128 * 128 ? bird_kernel<2> : bird_kernel<0>;
}

// Launch-attribute caches: a lone small instance's latency is a few kernel
// durations, so per-call cudaFuncSetAttribute / occupancy / attribute queries
// (each a driver round trip) are done once per (device, kernel, size).
namespace {
std::mutex g_attr_mu;
std::map<std::pair<int, const void *>, int> g_smem_set;
std::map<std::tuple<int, const void *, int, int64_t>, int> g_occ;
std::map<int, int> g_sms;

int cur_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

cudaError_t ensure_smem(const void *kern, int64_t smem) {
    const int dev = cur_device();
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int &have = g_smem_set[{dev, kern}];
    if (smem <= have) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) have = (int)smem;
    return e;
}

int occupancy(const void *kern, int threads, int64_t smem) {
    const int dev = cur_device();
    {
        std::lock_guard<std::mutex> lk(g_attr_mu);
        auto it = g_occ.find({dev, kern, threads, smem});
        if (it != g_occ.end()) return it->second;
    }
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem);
    std::lock_guard<std::mutex> lk(g_attr_mu);
    g_occ[{dev, kern, threads, smem}] = nb;
    return nb;
}

int sm_count() {
    const int dev = cur_device();
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = g_sms.find(dev);
    if (it != g_sms.end()) return it->second;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = sms;
    return sms;
}
}  // namespace

bool grid_shape(int W, int H, int k, int nwarps, int solver, GridShape &s) {
    if (W <= 0 || H <= 0 || W > 1024 || H > 1024) return false;
    s.W = W;
    s.H = H;
    s.k = k;
    s.wpd = (H + 63) / 64;
    const int need = (H + 31) / 32;
    s.B = need <= 8 ? 8 : (need <= 16 ? 16 : 32);
    s.LK = k + 2;
    const int ylo = (H - k) / 2, yhi = ylo + k - 1;
    const int lo = H - 1 - yhi, hi = H - 1 - ylo;
    s.LT = (int)align_up(lo + W - 1 + 64, 64);
    s.LB = (int)align_up((H - 1 - hi) + W - 1 + 64, 64);
    s.nchunk = (2 * W - 1 + 31) / 32;
    s.nwarps = nwarps;
    s.solver = solver;
    s.lo = lo;
    s.hi = hi;
    GridSmem o;
    grid_smem_layout(s, o);
    s.smem_bytes = o.total;
    return s.smem_bytes <= 227 * 1024;
}

size_t grid_stage_ints(const GridShape &s) { return (size_t)s.W * stage_stride(s.k); }

size_t redrec_plan_bytes(int W) {
    return (size_t)align_up(W, 16) + 3 * (size_t)align_up(2 * W, 16) + (size_t)align_up(4 * (W + 2), 16) + 32;
}

RedrecPlans redrec_plans_carve(void *base, int W, int count) {
    unsigned char *b = (unsigned char *)base;
    RedrecPlans pl;
    const size_t n = (size_t)count;
    pl.ev_type = (uint8_t *)b;
    b += align_up(n * W, 16);
    pl.ev_col = (int16_t *)b;
    b += align_up(n * W * 2, 16);
    pl.ev_aux = (int16_t *)b;
    b += align_up(n * W * 2, 16);
    pl.wave_list = (int16_t *)b;
    b += align_up(n * W * 2, 16);
    pl.wave_off = (int32_t *)b;
    b += align_up(n * (W + 2) * 4, 16);
    pl.meta = (int32_t *)b;
    return pl;
}

cudaError_t launch_grid_solver(int solver, const GridParams &p, int grid, cudaStream_t stream, cudaEvent_t *ev) {
    const int threads = 32 * p.shape.nwarps;
    void (*kern)(GridParams) = solver == 0 ? redrec_exec(p.shape) : bird_exec(p.shape);
    cudaError_t e;
    if (solver == 0) {
        // plans first: one warp per instance, all instances in parallel
        // 2-warp CTAs spread the latency-bound planner warps evenly over the
        // SMs (4-warp CTAs: 0.34 ms per 2,048 256^2 grids, 2-warp: 0.31 ms)
        static const int pw = [] {
            const char *e = getenv("RECON_PLAN_WARPS");
            return e ? std::max(1, std::min(4, atoi(e))) : 2;
        }();
        const int64_t psmem = pw * redrec_plan_smem(p.shape.W);
        e = ensure_smem((const void *)redrec_plan_kernel, psmem);
        if (e != cudaSuccess) return e;
        const int per_sm = occupancy((const void *)redrec_plan_kernel, 32 * pw, psmem);
        const int sms = sm_count();
        const int pgrid = std::max(1, std::min((p.count + pw - 1) / pw, std::max(1, per_sm) * sms));
        if (ev) cudaEventRecord(ev[0], stream);
        redrec_plan_kernel<<<pgrid, 32 * pw, psmem, stream>>>(p);
    }
    e = ensure_smem((const void *)kern, p.shape.smem_bytes);
    if (e != cudaSuccess) return e;
    if (ev) cudaEventRecord(ev[1], stream);
    if (solver == 0 && !ev && p.count <= grid) {
        // programmatic dependent launch: executor CTAs start as planner CTAs
        // trigger, load and transpose their first instance, and wait for the
        // plans (griddepcontrol.wait) only before reading them.  Only when
        // every CTA takes one instance (latency: C4 h'128 67 -> 62 us); on
        // large batches the executor CTAs cannot co-reside with the planner
        // and the step was not faster.
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = p.shape.smem_bytes;
        cfg.stream = stream;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, p);
        if (e != cudaSuccess) return e;
    } else {
        kern<<<grid, threads, p.shape.smem_bytes, stream>>>(p);
    }
    if (ev) cudaEventRecord(ev[2], stream);
    return cudaGetLastError();
}

int grid_occupancy(int solver, const GridShape &s) {
    void (*kern)(GridParams) = solver == 0 ? redrec_exec(s) : bird_exec(s);
    ensure_smem((const void *)kern, s.smem_bytes);
    return occupancy((const void *)kern, 32 * s.nwarps, s.smem_bytes);
}

}  // namespace rb
