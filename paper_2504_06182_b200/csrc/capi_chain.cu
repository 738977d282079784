// C-ABI: exact 1D (assign_1d, assign_1d_generalized, solve_1d, batched chains).
//
// Replaces exact1d.hpp:21 (assign_1d), :39 (assign_1d_generalized), :82
// (solve_1d).  Host side only marshals: it sorts the by-value inputs and runs
// the reference's argument checks in the reference's order
// (exact1d.cpp:299-312, 374-396); every assignment, block certification,
// ordering and DAG is computed on the device.

#include <algorithm>
#include <vector>

#include "capi_internal.cuh"
#include "chain.cuh"

using namespace rb;

namespace {

#define CK(call, where)                                             \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return cuda_fail(e_, where, detail); \
    } while (0)

recon_status fail(int32_t *detail, recon_status st, int32_t d) {
    if (detail) *detail = d;
    return st;
}

// validate_chain_instance (exact1d.cpp:299-312) on sorted inputs
recon_status validate_chain(int n, const std::vector<int> &S, const std::vector<int> &T, int32_t *detail) {
    if (n <= 0) return fail(detail, RECON_ERR_INPUT, RECON_D_CHAIN_LENGTH);
    for (int pass = 0; pass < 2; ++pass) {
        const std::vector<int> &v = pass ? T : S;
        for (size_t i = 0; i < v.size(); ++i) {
            if (v[i] < 0 || v[i] >= n)
                return fail(detail, RECON_ERR_INPUT, pass ? RECON_D_TARGET_OOB : RECON_D_SOURCE_OOB);
            if (i > 0 && v[i] <= v[i - 1])
                return fail(detail, RECON_ERR_INPUT, pass ? RECON_D_TARGET_ORDER : RECON_D_SOURCE_ORDER);
        }
    }
    if (S.size() < T.size()) return fail(detail, RECON_ERR_INFEASIBLE, RECON_D_FEWER_SOURCES);
    return RECON_OK;
}

struct Matching {
    int64_t weight = 0;
    // device arrays (valid until the next call on the context)
    int64_t *d_psrc = nullptr, *d_pdst = nullptr;
    int32_t *d_use = nullptr;
};

// General DP path on device; inputs sorted.
recon_status run_general(Ctx *c, int n, int ns, int nt, const std::vector<int64_t> &pos,
                         const std::vector<int32_t> *mn, const std::vector<int32_t> *mx, const std::vector<int64_t> &tg,
                         bool certify, Matching &m, int32_t *detail) {
    ChainGeneralParams p{};
    p.n = n;
    p.ns = ns;
    p.nt = nt;
    p.certify = certify ? 1 : 0;
    const size_t nn = (size_t)std::max(n, 1) + 2;
    int64_t *d_pos = c->dev<int64_t>(S_CHAIN_A, (size_t)ns + 1);
    int64_t *d_tg = c->dev<int64_t>(S_CHAIN_B, (size_t)nt + 1);
    int32_t *d_mm = c->dev<int32_t>(S_CHAIN_C, 2 * (size_t)ns + 2);
    int64_t *d_dp = c->dev<int64_t>(S_CHAIN_D, 3 * ((size_t)nt + 1) + nn + 2 * ((size_t)nt + 1) + 2);
    uint16_t *d_choice = c->dev<uint16_t>(S_CHAIN_E, (size_t)std::max(ns, 1) * ((size_t)nt + 1));
    int32_t *d_i32 = c->dev<int32_t>(S_BM_AUX0, 4 * nn + nn + (size_t)ns + 4);
    if (!d_pos || !d_tg || !d_mm || !d_dp || !d_choice || !d_i32)
        return cuda_fail(cudaErrorMemoryAllocation, "chain workspace", detail);
    p.pos = d_pos;
    p.tgt = d_tg;
    p.min_use = mn ? d_mm : nullptr;
    p.max_use = mx ? d_mm + ns + 1 : nullptr;
    p.dp_a = d_dp;
    p.dp_b = d_dp + (nt + 1);
    p.cprefix = d_dp + 2 * (nt + 1);
    p.wts = d_dp + 3 * (nt + 1);
    p.pair_src = p.wts + nn;
    p.pair_dst = p.pair_src + (nt + 1);
    p.weight = p.pair_dst + (nt + 1);
    p.choice = d_choice;
    p.blocks = d_i32;
    p.scratch = d_i32 + 4 * nn;
    p.use = p.scratch + nn;
    p.status = p.use + ns + 1;
    cudaStream_t st = c->stream;
    if (ns) CK(cudaMemcpyAsync(d_pos, pos.data(), (size_t)ns * 8, cudaMemcpyHostToDevice, st), "H2D");
    if (nt) CK(cudaMemcpyAsync(d_tg, tg.data(), (size_t)nt * 8, cudaMemcpyHostToDevice, st), "H2D");
    if (mn && ns) CK(cudaMemcpyAsync(d_mm, mn->data(), (size_t)ns * 4, cudaMemcpyHostToDevice, st), "H2D");
    if (mx && ns) CK(cudaMemcpyAsync(d_mm + ns + 1, mx->data(), (size_t)ns * 4, cudaMemcpyHostToDevice, st), "H2D");
    CK(launch_chain_general(p, st), "chain_general launch");
    c->launches += 1;
    int32_t h_st = 0;
    CK(cudaMemcpyAsync(&h_st, p.status, 4, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaMemcpyAsync(&m.weight, p.weight, 8, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaStreamSynchronize(st), "chain_general");
    if (h_st != RECON_OK) return fail(detail, RECON_ERR_INFEASIBLE, RECON_D_GEN_NO_ASSIGNMENT);
    m.d_psrc = p.pair_src;
    m.d_pdst = p.pair_dst;
    m.d_use = p.use;
    return RECON_OK;
}

__global__ void band_to_matching(int k, int ns, const int32_t *ps, const int32_t *pd, const int32_t *first,
                                 int64_t *msrc, int64_t *mdst, int32_t *use) {
    const int f = *first;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x)
        use[i] = (i >= f && i < f + k) ? 1 : 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
        msrc[i] = ps[i];
        mdst[i] = pd[i];
    }
}

// Band path (contiguous T) through the batched warp kernel with count = 1.
recon_status run_band(Ctx *c, int n, const std::vector<int> &S, int tl, int th, Matching &m, int32_t *detail) {
    const int k = th - tl + 1, ns = (int)S.size();
    const size_t words = (size_t)(n + 63) / 64;
    std::vector<uint64_t> occ(words, 0ull);
    for (int v : S) occ[(size_t)v / 64] |= 1ull << (v % 64);
    uint64_t *d_occ = c->dev<uint64_t>(S_OCC, words);
    int32_t *d_i = c->dev<int32_t>(S_CHAIN_C, 2 * (size_t)k + 8 + (size_t)ns + 1);
    int64_t *d_l = c->dev<int64_t>(S_CHAIN_D, 2 * (size_t)k + 2);
    if (!d_occ || !d_i || !d_l) return cuda_fail(cudaErrorMemoryAllocation, "chain workspace", detail);
    ChainBandParams p{};
    p.occ = d_occ;
    p.count = 1;
    p.n = n;
    p.t_lo = tl;
    p.t_hi = th;
    p.path_src = d_i;
    p.path_dst = d_i + k;
    p.displaced = d_i + 2 * k;
    p.status = d_i + 2 * k + 1;
    p.detail = d_i + 2 * k + 2;
    p.use_first = d_i + 2 * k + 3;
    int32_t *use = d_i + 2 * k + 8;
    p.total_displacement = d_l;
    cudaStream_t st = c->stream;
    CK(cudaMemcpyAsync(d_occ, occ.data(), words * 8, cudaMemcpyHostToDevice, st), "H2D");
    CK(launch_chain_band(p, c->sms, st), "chain_band launch");
    band_to_matching<<<4, 256, 0, st>>>(k, ns, p.path_src, p.path_dst, p.use_first, d_l + 1, d_l + 1 + k, use);
    c->launches += 2;
    int32_t h[2];
    CK(cudaMemcpyAsync(h, p.status, 8, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaMemcpyAsync(&m.weight, d_l, 8, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaStreamSynchronize(st), "chain_band");
    if (h[0] != RECON_OK) return fail(detail, (recon_status)h[0], h[1]);
    m.d_psrc = d_l + 1;
    m.d_pdst = d_l + 1 + k;
    m.d_use = use;
    return RECON_OK;
}

recon_status assign_chain(Ctx *c, int n, std::vector<int> &S, std::vector<int> &T, Matching &m, int32_t *detail) {
    std::sort(S.begin(), S.end());  // assign_1d takes S, T by value and sorts (exact1d.cpp:343-344)
    std::sort(T.begin(), T.end());
    recon_status st = validate_chain(n, S, T, detail);
    if (st != RECON_OK) return st;
    if (T.empty()) return RECON_OK;
    const bool band = T.back() - T.front() + 1 == (int)T.size() && n <= 4096;
    if (band) return run_band(c, n, S, T.front(), T.back(), m, detail);
    std::vector<int64_t> pos(S.begin(), S.end()), tg(T.begin(), T.end());
    return run_general(c, n, (int)S.size(), (int)T.size(), pos, nullptr, nullptr, tg, true, m, detail);
}

}  // namespace

extern "C" {

recon_status recon_assign_1d(recon_ctx *ctx, int32_t n, const int32_t *S, int32_t ns, const int32_t *T, int32_t nt,
                             int64_t *weight, int64_t *pair_src, int64_t *pair_dst, int32_t *use_count,
                             int32_t *detail) {
    if (detail) *detail = 0;
    if ((ns > 0 && !S) || (nt > 0 && !T) || !weight) return RECON_ERR_ARGUMENT;
    Ctx *c = resolve(ctx);
    if (!c) return fail(detail, RECON_ERR_CUDA, RECON_D_CUDA);
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    std::vector<int> s(S, S + ns), t(T, T + nt);
    Matching m;
    recon_status st = assign_chain(c, n, s, t, m, detail);
    if (st != RECON_OK) return st;
    *weight = m.weight;
    if (nt == 0) {
        for (int i = 0; i < ns; ++i) use_count[i] = 0;
        return RECON_OK;
    }
    CK(cudaMemcpyAsync(pair_src, m.d_psrc, (size_t)nt * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaMemcpyAsync(pair_dst, m.d_pdst, (size_t)nt * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    if (ns) CK(cudaMemcpyAsync(use_count, m.d_use, (size_t)ns * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaStreamSynchronize(c->stream), "D2H");
    return RECON_OK;
}

recon_status recon_assign_1d_generalized(recon_ctx *ctx, int32_t nsrc, const int64_t *pos,
                                         const int32_t *multiplicity, const int32_t *min_use, int32_t nt,
                                         const int64_t *targets, int64_t *weight, int64_t *pair_src,
                                         int64_t *pair_dst, int32_t *use_count, int32_t *detail) {
    if (detail) *detail = 0;
    if ((nsrc > 0 && (!pos || !multiplicity || !min_use)) || (nt > 0 && !targets) || !weight)
        return RECON_ERR_ARGUMENT;
    // argument checks in the reference's order (exact1d.cpp:374-396)
    long long supply = 0, mandatory = 0;
    for (int i = 0; i < nsrc; ++i) {
        if (multiplicity[i] < 1) return fail(detail, RECON_ERR_INPUT, RECON_D_GEN_MULTIPLICITY);
        if (min_use[i] < 0 || min_use[i] > multiplicity[i]) return fail(detail, RECON_ERR_INPUT, RECON_D_GEN_MIN_USE);
        if (i > 0 && pos[i] <= pos[i - 1]) return fail(detail, RECON_ERR_INPUT, RECON_D_GEN_SOURCE_ORDER);
        supply += multiplicity[i];
        mandatory += min_use[i];
    }
    for (int i = 1; i < nt; ++i)
        if (targets[i] <= targets[i - 1]) return fail(detail, RECON_ERR_INPUT, RECON_D_GEN_TARGET_ORDER);
    if (supply < nt) return fail(detail, RECON_ERR_INFEASIBLE, RECON_D_GEN_SUPPLY);
    if (mandatory > nt) return fail(detail, RECON_ERR_INFEASIBLE, RECON_D_GEN_MANDATORY);
    Ctx *c = resolve(ctx);
    if (!c) return fail(detail, RECON_ERR_CUDA, RECON_D_CUDA);
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    std::vector<int64_t> p(pos, pos + nsrc), tg(targets, targets + nt);
    std::vector<int32_t> mn(min_use, min_use + nsrc), mx(multiplicity, multiplicity + nsrc);
    Matching m;
    if (nt == 0) {
        // window_dp over zero targets: every source uses min_use == 0
        *weight = 0;
        for (int i = 0; i < nsrc; ++i) use_count[i] = 0;
        return RECON_OK;
    }
    recon_status st = run_general(c, 0, nsrc, nt, p, &mn, &mx, tg, false, m, detail);
    if (st != RECON_OK) return st;
    *weight = m.weight;
    CK(cudaMemcpyAsync(pair_src, m.d_psrc, (size_t)nt * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaMemcpyAsync(pair_dst, m.d_pdst, (size_t)nt * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    if (nsrc) CK(cudaMemcpyAsync(use_count, m.d_use, (size_t)nsrc * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaStreamSynchronize(c->stream), "D2H");
    return RECON_OK;
}

__global__ void narrow_pairs(int k, const int64_t *a, const int64_t *b, int32_t *x, int32_t *y) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
        x[i] = (int32_t)a[i];
        y[i] = (int32_t)b[i];
    }
}

recon_status recon_solve_1d(recon_ctx *ctx, int32_t n, const int32_t *S, int32_t ns, const int32_t *T, int32_t nt,
                            int32_t *path_src, int32_t *path_dst, int32_t *path_order, int32_t *dag_src,
                            int32_t *dag_dst, int64_t dag_capacity, int64_t *dag_count, int64_t *total_displacement,
                            int32_t *displaced, int32_t *detail) {
    if (detail) *detail = 0;
    if ((ns > 0 && !S) || (nt > 0 && !T) || !total_displacement || !displaced) return RECON_ERR_ARGUMENT;
    Ctx *c = resolve(ctx);
    if (!c) return fail(detail, RECON_ERR_CUDA, RECON_D_CUDA);
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    std::vector<int> s(S, S + ns), t(T, T + nt);
    Matching m;
    recon_status st = assign_chain(c, n, s, t, m, detail);
    if (st != RECON_OK) return st;
    if (dag_count) *dag_count = 0;
    *total_displacement = 0;
    *displaced = 0;
    if (nt == 0) return RECON_OK;
    const int P = nt;
    int32_t *d_i = c->dev<int32_t>(S_BM_AUX1, 6 * (size_t)P + 4);
    unsigned long long *d_k = c->dev<unsigned long long>(S_BM_AUX2, 2 * (size_t)P + 2);
    int64_t *d_cnt = c->dev<int64_t>(S_BM_AUX3, (size_t)P + 2);
    ChainOrderParams o{};
    o.P = P;
    o.temp_bytes = chain_order_temp_bytes(P);
    o.temp = c->get(S_TEMP, o.temp_bytes);
    if (!d_i || !d_k || !d_cnt || !o.temp) return cuda_fail(cudaErrorMemoryAllocation, "solve_1d workspace", detail);
    int32_t *d_src = d_i, *d_dst = d_i + P;
    o.src = d_src;
    o.dst = d_dst;
    o.order = d_i + 2 * P;
    o.rank = d_i + 3 * P;
    o.sweep_id = d_i + 4 * P;
    o.keys_a = d_k;
    o.keys_b = d_k + P + 1;
    o.cnt = d_cnt;
    // paths = pairs in target order (paths_from_matching + resolve_nesting,
    // which is the identity on order-preserving pairs, exact1d.cpp:430-492)
    narrow_pairs<<<(P + 255) / 256, 256, 0, c->stream>>>(P, m.d_psrc, m.d_pdst, d_src, d_dst);
    int64_t ne = 0;
    CK(chain_order_count(o, c->stream, &ne), "chain order");
    c->launches += 6;
    CK(cudaMemcpyAsync(path_src, d_src, (size_t)P * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaMemcpyAsync(path_dst, d_dst, (size_t)P * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    if (path_order) CK(cudaMemcpyAsync(path_order, o.order, (size_t)P * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaStreamSynchronize(c->stream), "D2H");
    long long tot = 0;
    int disp = 0;
    for (int i = 0; i < P; ++i) {
        tot += path_src[i] > path_dst[i] ? path_src[i] - path_dst[i] : path_dst[i] - path_src[i];
        disp += path_src[i] != path_dst[i];
    }
    *total_displacement = tot;  // make_solution stats (path_system.cpp:43-44)
    *displaced = disp;
    if (dag_count) *dag_count = ne;
    if (dag_src) {
        if (ne > dag_capacity) return RECON_ERR_CAPACITY;
        if (ne > 0) {
            o.ea = c->dev<int32_t>(S_EA, (size_t)ne);
            o.eb = c->dev<int32_t>(S_EB, (size_t)ne);
            if (!o.ea || !o.eb) return cuda_fail(cudaErrorMemoryAllocation, "solve_1d dag", detail);
            CK(chain_order_emit(o, c->stream), "chain dag");
            c->launches += 1;
            CK(cudaMemcpyAsync(dag_src, o.ea, (size_t)ne * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
            CK(cudaMemcpyAsync(dag_dst, o.eb, (size_t)ne * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
            CK(cudaStreamSynchronize(c->stream), "D2H");
        }
    }
    return RECON_OK;
}

static recon_status chain_batch(recon_ctx *ctx, const recon_chain_batch *b, bool host) {
    int32_t *detail = nullptr;
    if (!b || !b->occ || !b->path_src || !b->path_dst || !b->total_displacement || !b->displaced || !b->status)
        return RECON_ERR_ARGUMENT;
    if (b->n <= 0 || b->n > 4096 || b->t_lo < 0 || b->t_hi < b->t_lo || b->t_hi >= b->n) return RECON_ERR_ARGUMENT;
    if (b->count <= 0) return RECON_OK;
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    const size_t n = (size_t)b->count, k = (size_t)(b->t_hi - b->t_lo + 1), words = (size_t)(b->n + 63) / 64;
    ChainBandParams p{};
    p.count = b->count;
    p.n = b->n;
    p.t_lo = b->t_lo;
    p.t_hi = b->t_hi;
    if (!host) {
        p.occ = b->occ;
        p.path_src = b->path_src;
        p.path_dst = b->path_dst;
        p.total_displacement = b->total_displacement;
        p.displaced = b->displaced;
        p.status = b->status;
        p.detail = b->detail;
        CK(launch_chain_band(p, c->sms, c->stream), "chain_band launch");
        c->launches += 1;
        return RECON_OK;
    }
    uint64_t *d_occ = c->dev<uint64_t>(S_OCC, n * words);
    int32_t *d_ps = c->dev<int32_t>(S_PSRC, n * k), *d_pd = c->dev<int32_t>(S_PDST, n * k);
    int64_t *d_td = c->dev<int64_t>(S_TDISP, n);
    int32_t *d_misc = c->dev<int32_t>(S_STATUS, 3 * n);
    if (!d_occ || !d_ps || !d_pd || !d_td || !d_misc) return cuda_fail(cudaErrorMemoryAllocation, "chain batch", detail);
    p.occ = d_occ;
    p.path_src = d_ps;
    p.path_dst = d_pd;
    p.total_displacement = d_td;
    p.displaced = d_misc;
    p.status = d_misc + n;
    p.detail = d_misc + 2 * n;
    cudaStream_t st = c->stream;
    CK(cudaMemcpyAsync(d_occ, b->occ, n * words * 8, cudaMemcpyHostToDevice, st), "H2D");
    CK(launch_chain_band(p, c->sms, st), "chain_band launch");
    c->launches += 1;
    CK(cudaMemcpyAsync(b->path_src, d_ps, n * k * 4, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaMemcpyAsync(b->path_dst, d_pd, n * k * 4, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaMemcpyAsync(b->total_displacement, d_td, n * 8, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaMemcpyAsync(b->displaced, d_misc, n * 4, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaMemcpyAsync(b->status, d_misc + n, n * 4, cudaMemcpyDeviceToHost, st), "D2H");
    if (b->detail) CK(cudaMemcpyAsync(b->detail, d_misc + 2 * n, n * 4, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaStreamSynchronize(st), "chain batch");
    return RECON_OK;
}

recon_status recon_solve_1d_batch(recon_ctx *ctx, const recon_chain_batch *b) { return chain_batch(ctx, b, false); }
recon_status recon_solve_1d_batch_host(recon_ctx *ctx, const recon_chain_batch *b) { return chain_batch(ctx, b, true); }

}  // extern "C"
