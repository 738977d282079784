// C-ABI helpers behind two more reference functions:
//   recon_min_cost_1d        min_assignment_cost_1d (exact1d.hpp:48-49)
//   recon_occupancy_dag_paths occupancy_dag over arbitrary vertex lists
//                             (virtual_line.hpp:104; used by aro's assembly)

#include <algorithm>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <vector>

#include "capi_internal.cuh"
#include "chain.cuh"

namespace rb {
__global__ void dagx_mark_kernel(int P, const int64_t *off, const int32_t *verts, int32_t *source_of,
                                 int32_t *target_of);
template <bool WRITE>
__global__ void dagx_walk_kernel(int P, const int64_t *off, const int32_t *verts, const int32_t *source_of,
                                 const int32_t *target_of, int32_t *cnt, const int64_t *eoff,
                                 unsigned long long *keys);
__global__ void unique_flags_kernel(int64_t n, const unsigned long long *k, int32_t *flag);
__global__ void unique_scatter_kernel(int64_t n, const unsigned long long *k, const int32_t *flag,
                                      const int64_t *pos, int32_t *a, int32_t *b);
}  // namespace rb

using namespace rb;

#define CK(call, where)                                             \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return cuda_fail(e_, where, detail); \
    } while (0)

__global__ void widen_i32_kernel(int n, const int32_t *in, int64_t *out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[i];
}

extern "C" {

recon_status recon_min_cost_1d(recon_ctx *ctx, int32_t ns, const int64_t *sources, int32_t nt, const int64_t *targets,
                               int64_t *cost, int32_t *detail) {
    if (detail) *detail = 0;
    if (!cost || (ns > 0 && !sources) || (nt > 0 && !targets)) return RECON_ERR_ARGUMENT;
    *cost = 0;
    if (nt == 0) return RECON_OK;  // certifier_cost (exact1d.cpp:107)
    if (ns < nt) {                 // exact1d.cpp:108
        if (detail) *detail = RECON_D_INFEASIBLE_SUPPLY;
        return RECON_ERR_INFEASIBLE;
    }
    std::vector<int64_t> s(sources, sources + ns), t(targets, targets + nt);
    std::sort(s.begin(), s.end());
    std::sort(t.begin(), t.end());
    std::vector<int64_t> pos;
    std::vector<int32_t> mn, mx;
    for (int64_t v : s) {
        if (!pos.empty() && pos.back() == v) {
            ++mx.back();
        } else {
            pos.push_back(v);
            mn.push_back(0);
            mx.push_back(1);
        }
    }
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    const int np = (int)pos.size();
    ChainGeneralParams p{};
    p.n = 0;
    p.ns = np;
    p.nt = nt;
    p.certify = 0;
    int64_t *d_pos = c->dev<int64_t>(S_CHAIN_A, (size_t)np + 1);
    int64_t *d_tg = c->dev<int64_t>(S_CHAIN_B, (size_t)nt + 1);
    int32_t *d_mm = c->dev<int32_t>(S_CHAIN_C, 2 * (size_t)np + 2);
    int64_t *d_dp = c->dev<int64_t>(S_CHAIN_D, 5 * ((size_t)nt + 1) + 4);
    uint16_t *d_choice = c->dev<uint16_t>(S_CHAIN_E, (size_t)np * ((size_t)nt + 1));
    int32_t *d_i32 = c->dev<int32_t>(S_BM_AUX0, 4 * 4 + 4 + (size_t)np + 4);
    if (!d_pos || !d_tg || !d_mm || !d_dp || !d_choice || !d_i32)
        return cuda_fail(cudaErrorMemoryAllocation, "min_cost workspace", detail);
    p.pos = d_pos;
    p.tgt = d_tg;
    p.min_use = d_mm;
    p.max_use = d_mm + np + 1;
    p.dp_a = d_dp;
    p.dp_b = d_dp + (nt + 1);
    p.cprefix = d_dp + 2 * (nt + 1);
    p.pair_src = d_dp + 3 * (nt + 1);
    p.pair_dst = d_dp + 4 * (nt + 1);
    p.weight = d_dp + 5 * (nt + 1);
    p.wts = p.weight + 1;
    p.choice = d_choice;
    p.blocks = d_i32;
    p.scratch = d_i32 + 16;
    p.use = d_i32 + 20;
    p.status = d_i32 + 20 + np + 1;
    cudaStream_t st = c->stream;
    CK(cudaMemcpyAsync(d_pos, pos.data(), (size_t)np * 8, cudaMemcpyHostToDevice, st), "H2D");
    CK(cudaMemcpyAsync(d_tg, t.data(), (size_t)nt * 8, cudaMemcpyHostToDevice, st), "H2D");
    CK(cudaMemcpyAsync(d_mm, mn.data(), (size_t)np * 4, cudaMemcpyHostToDevice, st), "H2D");
    CK(cudaMemcpyAsync(d_mm + np + 1, mx.data(), (size_t)np * 4, cudaMemcpyHostToDevice, st), "H2D");
    CK(launch_chain_general(p, st), "min_cost launch");
    c->launches += 1;
    CK(cudaMemcpyAsync(cost, p.weight, 8, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaStreamSynchronize(st), "min_cost");
    return RECON_OK;
}

recon_status recon_occupancy_dag_paths(recon_ctx *ctx, int32_t width, int32_t height, int32_t P, const int64_t *off,
                                       const int32_t *verts, int32_t *dag_src, int32_t *dag_dst,
                                       int64_t dag_capacity, int64_t *dag_count, int32_t *detail) {
    if (detail) *detail = 0;
    if (!dag_count || (P > 0 && (!off || !verts))) return RECON_ERR_ARGUMENT;
    *dag_count = 0;
    if (P == 0) return RECON_OK;
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    cudaStream_t st = c->stream;
    const size_t WH = (size_t)width * height, nv = (size_t)off[P];
    int64_t *d_off = c->dev<int64_t>(S_BM_OFF, (size_t)P + 2);
    int32_t *d_v = c->dev<int32_t>(S_BM_VERT, nv + 1);
    int32_t *so = c->dev<int32_t>(S_SRCOF, WH), *to = c->dev<int32_t>(S_TGTOF, WH);
    int32_t *cnt = c->dev<int32_t>(S_DCNT, (size_t)P + 1);
    int64_t *eoff = c->dev<int64_t>(S_DOFF, (size_t)P + 2);
    if (!d_off || !d_v || !so || !to || !cnt || !eoff) return cuda_fail(cudaErrorMemoryAllocation, "dag", detail);
    CK(cudaMemcpyAsync(d_off, off, ((size_t)P + 1) * 8, cudaMemcpyHostToDevice, st), "H2D");
    CK(cudaMemcpyAsync(d_v, verts, nv * 4, cudaMemcpyHostToDevice, st), "H2D");
    CK(cudaMemsetAsync(so, 0xff, WH * 4, st), "memset");
    CK(cudaMemsetAsync(to, 0xff, WH * 4, st), "memset");
    const int blocks = (P + 255) / 256 + 1;
    dagx_mark_kernel<<<blocks, 256, 0, st>>>(P, d_off, d_v, so, to);
    dagx_walk_kernel<false><<<blocks, 256, 0, st>>>(P, d_off, d_v, so, to, cnt, nullptr, nullptr);
    widen_i32_kernel<<<blocks, 256, 0, st>>>(P, cnt, eoff);
    CK(cudaMemsetAsync(eoff + P, 0, 8, st), "memset");
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, eoff, eoff, P + 1);
    void *temp = c->get(S_TEMP, tb);
    if (!temp) return cuda_fail(cudaErrorMemoryAllocation, "temp", detail);
    CK(cub::DeviceScan::ExclusiveSum(temp, tb, eoff, eoff, P + 1, st), "scan");
    int64_t n = 0;
    CK(cudaMemcpyAsync(&n, eoff + P, 8, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaStreamSynchronize(st), "dag count");
    c->launches += 4;
    if (n == 0) return RECON_OK;
    unsigned long long *k1 = c->dev<unsigned long long>(S_KEYS, (size_t)n), *k2 = c->dev<unsigned long long>(S_KEYS2, (size_t)n);
    int32_t *flag = c->dev<int32_t>(S_BM_AUX1, (size_t)n + 1);
    int64_t *pos = c->dev<int64_t>(S_BM_AUX2, (size_t)n + 1);
    int32_t *ea = c->dev<int32_t>(S_EA, (size_t)n), *eb = c->dev<int32_t>(S_EB, (size_t)n);
    if (!k1 || !k2 || !flag || !pos || !ea || !eb) return cuda_fail(cudaErrorMemoryAllocation, "dag keys", detail);
    dagx_walk_kernel<true><<<blocks, 256, 0, st>>>(P, d_off, d_v, so, to, nullptr, eoff, k1);
    size_t tb2 = 0, tb3 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb2, k1, k2, (int)n);
    cub::DeviceScan::ExclusiveSum(nullptr, tb3, flag, pos, (int)n + 1);
    temp = c->get(S_TEMP, std::max(tb2, tb3));
    if (!temp) return cuda_fail(cudaErrorMemoryAllocation, "temp", detail);
    CK(cub::DeviceRadixSort::SortKeys(temp, tb2, k1, k2, (int)n, 0, 64, st), "sort");
    const int eb_ = (int)std::min<int64_t>((n + 255) / 256 + 1, 148 * 16);
    unique_flags_kernel<<<eb_, 256, 0, st>>>(n, k2, flag);
    CK(cudaMemsetAsync(flag + n, 0, 4, st), "memset");
    CK(cub::DeviceScan::ExclusiveSum(temp, tb3, flag, pos, (int)n + 1, st), "scan");
    unique_scatter_kernel<<<eb_, 256, 0, st>>>(n, k2, flag, pos, ea, eb);
    c->launches += 5;
    int64_t u = 0;
    CK(cudaMemcpyAsync(&u, pos + n, 8, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaStreamSynchronize(st), "dag unique");
    *dag_count = u;
    if (u > dag_capacity) return RECON_ERR_CAPACITY;
    CK(cudaMemcpyAsync(dag_src, ea, (size_t)u * 4, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaMemcpyAsync(dag_dst, eb, (size_t)u * 4, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaStreamSynchronize(st), "D2H");
    return RECON_OK;
}

}  // extern "C"
