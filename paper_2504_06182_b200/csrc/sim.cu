// Multi-cycle loss simulation (SPEC.md [MODULE] sim):
// recon_sim_run_host.  All live trials advance one reconfiguration cycle at
// a time: the batched solver (+ batching) runs on every live trial at once,
// then one CTA per trial executes its schedule under loss and one CTA per
// trial applies lifetime decay and re-measures.  Draws are counter-based
// (include/recon_sim_rng.h), so every token's operations are simulated in
// parallel and still match the sequential restatement (oracle/sim_common.h)
// bit for bit.

#include <cmath>
#include <cub/block/block_scan.cuh>
#include <vector>

#include "capi_internal.cuh"
#include "recon_sim_rng.h"

using namespace rb;

namespace {

#define CK(call, where)                                             \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return cuda_fail(e_, where, detail); \
    } while (0)

constexpr int kThreads = 256;
using BlockScan = cub::BlockScan<int, kThreads>;

struct SimArgs {
    int W, H, hp, wpc, S;
    int batching;
    recon_loss_model L;
    uint64_t seed_base;
    int cyc;
    const int32_t *live;               // [m] trial ids
    const uint64_t *occ;               // [m] configurations at the cycle start
    uint64_t *nxt;                     // [m] after the moves
    const int32_t *src, *dst, *pc, *st;  // solver outputs [m]
    const int32_t *mb, *nb;            // batching outputs [m]
    int64_t ms;                        // move stride
    int32_t *off;                      // [m][S + 1] move offsets
    int32_t *bcnt, *runid;             // [m][nbmax]
    uint8_t *allc;
    int nbmax;
    double *cyc_el;                    // [m]
    // per-trial accumulators [count]
    int32_t *cycles, *status, *success;
    long long *n_nu, *n_al, *nb_nu, *nb_al, *lost;
    double *elapsed;
    int32_t *code;                     // [m] 0 continue, 1 success, 2 failure
    const double *pdec;                // [m]
};

// one CTA per live trial: the cycle's schedule under per-operation loss
__global__ void __launch_bounds__(kThreads) k_transport(SimArgs a) {
    __shared__ typename BlockScan::TempStorage scan;
    __shared__ long long s_nu, s_al;
    __shared__ int s_run;
    const int j = blockIdx.x, tid = threadIdx.x;
    const int trial = a.live[j];
    const size_t words = (size_t)a.W * a.wpc;
    const uint64_t *occ = a.occ + j * words;
    uint64_t *nxt = a.nxt + j * words;
    if (a.st[j] != RECON_OK) {  // the solver / batching failed: the trial ends
        if (tid == 0) {
            a.status[trial] = a.st[j];
            a.code[j] = 2;
            a.cyc_el[j] = 0.0;
        }
        return;
    }
    const int P = a.pc[j], H = a.H;
    const int32_t *src = a.src + (size_t)j * a.S, *dst = a.dst + (size_t)j * a.S;
    int32_t *off = a.off + (size_t)j * (a.S + 1);
    if (tid == 0) {
        s_nu = s_al = 0;
        a.code[j] = 0;
        a.cycles[trial] += 1;
    }
    // move offsets (block scan in chunks) and the moved-path count
    int run = 0, moved = 0;
    for (int p0 = 0; p0 < P; p0 += kThreads) {
        const int p = p0 + tid;
        int len = 0;
        if (p < P) {
            const int dx = src[p] / H - dst[p] / H, dy = src[p] % H - dst[p] % H;
            len = (dx < 0 ? -dx : dx) + (dy < 0 ? -dy : dy);
        }
        int ex, tot;
        BlockScan(scan).ExclusiveSum(len, ex, tot);
        if (p < P) off[p] = run + ex;
        run += tot;
        __syncthreads();
        int mv;
        BlockScan(scan).ExclusiveSum(len > 0 ? 1 : 0, ex, mv);
        moved += mv;
        __syncthreads();
    }
    const int D = run;
    if (tid == 0) off[P] = D;
    // EDI runs: consecutive batches moving the same token set
    int nruns = 0, nbc = 0;
    const int32_t *mb = a.batching ? a.mb + (size_t)j * a.ms : nullptr;
    int32_t *bcnt = a.bcnt + (size_t)j * a.nbmax, *runid = a.runid + (size_t)j * a.nbmax;
    uint8_t *allc = a.allc + (size_t)j * a.nbmax;
    if (a.batching) {
        nbc = a.nb[j];
        for (int k = tid; k < nbc; k += kThreads) {
            bcnt[k] = 0;
            allc[k] = 1;
        }
        __syncthreads();
        for (int p = tid; p < P; p += kThreads)
            for (int k = off[p]; k < off[p + 1]; ++k) {
                const int b = mb[k];
                atomicAdd(&bcnt[b], 1);
                if (!(k + 1 < off[p + 1] && mb[k + 1] == b + 1)) allc[b] = 0;
            }
        __syncthreads();
        int base = 0;
        for (int k0 = 0; k0 < nbc; k0 += kThreads) {
            const int k = k0 + tid;
            const int start = k < nbc && k > 0 && !(bcnt[k - 1] == bcnt[k] && allc[k - 1]) ? 1 : 0;
            int ex, tot;
            BlockScan(scan).InclusiveSum(start, ex, tot);
            if (k < nbc) runid[k] = base + ex;
            base += tot;
            __syncthreads();
        }
        nruns = nbc ? base + 1 : 0;
    }
    // no fused multiply-add: the same rounding as the host checkers
    const double el = a.batching ? __dadd_rn(__dmul_rn(2.0 * a.L.t_alpha, (double)nruns), __dmul_rn(a.L.t_nu, (double)nbc))
                                 : __dadd_rn(__dmul_rn(2.0 * a.L.t_alpha, (double)moved), __dmul_rn(a.L.t_nu, (double)D));
    if (tid == 0) {
        a.cyc_el[j] = el;
        a.nb_nu[trial] += a.batching ? nbc : D;
        a.nb_al[trial] += a.batching ? nruns : moved;
    }
    // the configuration minus the sources, then the surviving tokens at their targets
    for (size_t w = tid; w < words; w += kThreads) nxt[w] = occ[w];
    __syncthreads();
    for (int p = tid; p < P; p += kThreads) {
        const int v = src[p];
        atomicAnd((unsigned long long *)&nxt[(size_t)(v / H) * a.wpc + (v % H) / 64], ~(1ull << ((v % H) & 63)));
    }
    __syncthreads();
    const uint64_t seed = a.seed_base + (uint64_t)trial;
    const double pa = a.L.p_alpha, pn = a.L.p_nu;
    long long nu = 0, al = 0;
    for (int p = tid; p < P; p += kThreads) {  // extract, k moves, implant
        const int len = off[p + 1] - off[p];
        const uint64_t b4 = (uint64_t)p * 4096;
        bool alive = true;
        if (len > 0) {
            ++al;
            alive = recon_sim_u01(seed, (uint32_t)a.cyc, RECON_DRAW_EXTRACT, b4) < pa;
        }
        for (int k = 0; k < len && alive; ++k) {
            ++nu;
            alive = recon_sim_u01(seed, (uint32_t)a.cyc, RECON_DRAW_MOVE, b4 + (uint64_t)k) < pn;
        }
        if (len > 0 && alive) {
            ++al;
            alive = recon_sim_u01(seed, (uint32_t)a.cyc, RECON_DRAW_IMPLANT, b4) < pa;
        }
        if (alive) {
            const int v = dst[p];
            atomicOr((unsigned long long *)&nxt[(size_t)(v / H) * a.wpc + (v % H) / 64], 1ull << ((v % H) & 63));
        }
    }
    atomicAdd((unsigned long long *)&s_nu, (unsigned long long)nu);
    atomicAdd((unsigned long long *)&s_al, (unsigned long long)al);
    __syncthreads();
    if (tid == 0) {
        a.n_nu[trial] += s_nu;
        a.n_al[trial] += s_al;
    }
}

// one CTA per live trial: lifetime decay, re-measurement, next state
__global__ void __launch_bounds__(kThreads) k_decay(SimArgs a, uint64_t *occ_all) {
    __shared__ long long s_before, s_after;
    __shared__ int s_hole;
    const int j = blockIdx.x, tid = threadIdx.x;
    if (a.code[j] == 2) return;
    const int trial = a.live[j];
    const size_t words = (size_t)a.W * a.wpc;
    const uint64_t *occ = a.occ + j * words;
    uint64_t *nxt = a.nxt + j * words;
    if (tid == 0) {
        s_before = s_after = 0;
        s_hole = 0;
    }
    __syncthreads();
    const uint64_t seed = a.seed_base + (uint64_t)trial;
    const double pd = a.pdec[j];
    long long before = 0, after = 0;
    for (size_t w = tid; w < words; w += kThreads) {
        before += __popcll(occ[w]);
        uint64_t m = nxt[w];
        const int x = (int)(w / a.wpc), y0 = (int)(w % a.wpc) * 64;
        for (uint64_t t = m; t; t &= t - 1) {
            const int y = y0 + __ffsll((long long)t) - 1;
            if (!(recon_sim_u01(seed, (uint32_t)a.cyc, RECON_DRAW_DECAY, (uint64_t)x * a.H + y) < pd))
                m &= ~(1ull << (y - y0));
        }
        nxt[w] = m;
        occ_all[(size_t)trial * words + w] = m;
        after += __popcll(m);
    }
    atomicAdd((unsigned long long *)&s_before, (unsigned long long)before);
    atomicAdd((unsigned long long *)&s_after, (unsigned long long)after);
    __syncthreads();
    // the centered band full?
    const int ylo = (a.H - a.hp) / 2, n = a.W * a.hp;
    for (int c = tid; c < n; c += kThreads) {
        const int x = c / a.hp, y = ylo + c % a.hp;
        if (!((nxt[(size_t)x * a.wpc + y / 64] >> (y & 63)) & 1ull)) s_hole = 1;
    }
    __syncthreads();
    if (tid == 0) {
        a.lost[trial] += s_before - s_after;
        a.elapsed[trial] = __dadd_rn(a.elapsed[trial], __dadd_rn(a.cyc_el[j], a.L.t_meas));
        if (!s_hole) {
            a.success[trial] = 1;
            a.code[j] = 1;
        } else if (s_after < (long long)a.W * a.hp) {
            a.code[j] = 2;
        }
    }
}

__global__ void k_gather(const int32_t *live, int m, const uint64_t *occ_all, uint64_t *occ, size_t words) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (size_t)m * words; i += (size_t)gridDim.x * blockDim.x)
        occ[i] = occ_all[(size_t)live[i / words] * words + i % words];
}

template <class T>
T *alloc_zero(Ctx *c, int slot, size_t n, bool *ok) {
    T *p = c->dev<T>(slot, n ? n : 1);
    if (!p || cudaMemsetAsync(p, 0, (n ? n : 1) * sizeof(T), c->stream) != cudaSuccess) *ok = false;
    return p;
}

}  // namespace

extern "C" recon_status recon_sim_run_host(recon_ctx *ctx, const recon_sim_batch *b) {
    int32_t *detail = nullptr;
    if (!b || !b->occ || !b->success || !b->cycles || !b->status || !b->n_nu || !b->n_alpha || !b->nb_nu ||
        !b->nb_alpha || !b->atoms_lost || !b->elapsed || b->width <= 0 || b->height <= 0 || b->h_prime <= 0 ||
        b->h_prime >= b->height || b->count < 0)
        return RECON_ERR_ARGUMENT;
    const int n = b->count, W = b->width, H = b->height, hp = b->h_prime, wpc = (H + 63) / 64, S = W * hp;
    for (int i = 0; i < n; ++i) {
        b->success[i] = b->cycles[i] = b->status[i] = 0;
        b->n_nu[i] = b->n_alpha[i] = b->nb_nu[i] = b->nb_alpha[i] = b->atoms_lost[i] = 0;
        b->elapsed[i] = 0.0;
    }
    if (!n) return RECON_OK;
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    const size_t words = (size_t)W * wpc;
    const int64_t ms = (int64_t)W * hp * (W + H) + 1;
    bool ok = true;
    uint64_t *occ_all = c->dev<uint64_t>(S_SIM_OCC, (size_t)n * words);
    uint64_t *occ = c->dev<uint64_t>(S_SIM_CUR, (size_t)n * words), *nxt = c->dev<uint64_t>(S_SIM_NXT, (size_t)n * words);
    int32_t *cycles = alloc_zero<int32_t>(c, S_SIM_CYC, n, &ok), *status = alloc_zero<int32_t>(c, S_SIM_ST, n, &ok);
    int32_t *success = alloc_zero<int32_t>(c, S_SIM_SUC, n, &ok);
    long long *acc = alloc_zero<long long>(c, S_SIM_ACC, (size_t)5 * n, &ok);
    double *elapsed = alloc_zero<double>(c, S_SIM_EL, n, &ok);
    int32_t *live_d = c->dev<int32_t>(S_SIM_LIVE, n), *code = c->dev<int32_t>(S_SIM_CODE, n);
    double *cyc_el = c->dev<double>(S_SIM_CEL, n), *pdec = c->dev<double>(S_SIM_PDEC, n);
    // solver outputs for up to n live trials
    int32_t *src = c->dev<int32_t>(S_SIM_SRC, (size_t)n * S), *dst = c->dev<int32_t>(S_SIM_DST, (size_t)n * S);
    int32_t *pc = c->dev<int32_t>(S_SIM_PC, n), *st = c->dev<int32_t>(S_SIM_PST, n);
    int32_t *det = c->dev<int32_t>(S_SIM_DET, n), *nbv = c->dev<int32_t>(S_SIM_NB, n);
    int64_t *td = c->dev<int64_t>(S_SIM_TD, n);
    int32_t *off = c->dev<int32_t>(S_SIM_OFF, (size_t)n * (S + 1));
    int32_t *mb = b->batching ? c->dev<int32_t>(S_SIM_MB, (size_t)n * ms) : nullptr;
    if (!ok || !occ_all || !occ || !nxt || !live_d || !code || !cyc_el || !pdec || !src || !dst || !pc || !st ||
        !det || !nbv || !td || !off || (b->batching && !mb))
        return cuda_fail(cudaErrorMemoryAllocation, "sim workspace", detail);
    CK(cudaMemcpyAsync(occ_all, b->occ, (size_t)n * words * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    // trials that start short of atoms fail before any cycle
    std::vector<int32_t> live;
    for (int i = 0; i < n; ++i) {
        long long a = 0;
        for (size_t w = 0; w < words; ++w) a += __builtin_popcountll(b->occ[(size_t)i * words + w]);
        if (a >= (long long)W * hp) live.push_back(i);
    }
    std::vector<double> el, pd;
    std::vector<int32_t> codes, nbh;
    for (int cyc = 0; cyc < b->max_cycles && !live.empty(); ++cyc) {
        const int m = (int)live.size();
        CK(cudaMemcpyAsync(live_d, live.data(), m * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
        k_gather<<<(int)std::min<size_t>(((size_t)m * words + 255) / 256, (size_t)c->sms * 8), 256, 0, c->stream>>>(
            live_d, m, occ_all, occ, words);
        recon_grid_batch g{};
        g.occ = occ;
        g.count = m;
        g.width = W;
        g.height = H;
        g.h_prime = hp;
        g.path_src = src;
        g.path_dst = dst;
        g.path_count = pc;
        g.total_displacement = td;
        g.status = st;
        g.detail = det;
        recon_status rs;
        if (b->batching) {
            recon_pipeline_batch pb{g, b->solver, b->preset, ms, mb, nbv};
            rs = recon_pipeline_batch_run(ctx, &pb);
        } else {
            rs = b->solver == 1 ? recon_bird_solve_batch(ctx, &g) : recon_redrec_solve_batch(ctx, &g);
        }
        if (rs != RECON_OK) return rs;
        SimArgs a{};
        a.W = W;
        a.H = H;
        a.hp = hp;
        a.wpc = wpc;
        a.S = S;
        a.batching = b->batching;
        a.L = b->loss;
        a.seed_base = b->seed_base;
        a.cyc = cyc;
        a.live = live_d;
        a.occ = occ;
        a.nxt = nxt;
        a.src = src;
        a.dst = dst;
        a.pc = pc;
        a.st = st;
        a.mb = mb;
        a.nb = nbv;
        a.ms = ms;
        a.off = off;
        a.cyc_el = cyc_el;
        a.cycles = cycles;
        a.status = status;
        a.success = success;
        a.n_nu = acc;
        a.n_al = acc + n;
        a.nb_nu = acc + 2 * n;
        a.nb_al = acc + 3 * n;
        a.lost = acc + 4 * n;
        a.elapsed = elapsed;
        a.code = code;
        a.pdec = pdec;
        a.nbmax = 1;
        if (b->batching) {  // per-trial batch scratch, sized by this cycle's largest schedule
            nbh.resize(m);
            CK(cudaMemcpyAsync(nbh.data(), nbv, m * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
            CK(cudaStreamSynchronize(c->stream), "D2H");
            for (int x : nbh) a.nbmax = std::max(a.nbmax, x + 1);
        }
        a.bcnt = c->dev<int32_t>(S_SIM_BCNT, (size_t)m * a.nbmax);
        a.runid = c->dev<int32_t>(S_SIM_RUN, (size_t)m * a.nbmax);
        a.allc = c->dev<uint8_t>(S_SIM_ALLC, (size_t)m * a.nbmax);
        if (!a.bcnt || !a.runid || !a.allc) return cuda_fail(cudaErrorMemoryAllocation, "sim batches", detail);
        k_transport<<<m, kThreads, 0, c->stream>>>(a);
        // decay probabilities on the host (the same libm exp as the checkers)
        el.resize(m);
        pd.resize(m);
        CK(cudaMemcpyAsync(el.data(), cyc_el, m * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
        CK(cudaStreamSynchronize(c->stream), "D2H");
        for (int k = 0; k < m; ++k) pd[k] = b->loss.tau > 0.0 ? std::exp(-(el[k] + b->loss.t_meas) / b->loss.tau) : 1.0;
        CK(cudaMemcpyAsync(pdec, pd.data(), m * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
        k_decay<<<m, kThreads, 0, c->stream>>>(a, occ_all);
        c->launches += 3;
        codes.resize(m);
        CK(cudaMemcpyAsync(codes.data(), code, m * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        CK(cudaStreamSynchronize(c->stream), "sim cycle");
        std::vector<int32_t> next;
        for (int k = 0; k < m; ++k)
            if (codes[k] == 0) next.push_back(live[k]);
        live.swap(next);
    }
    std::vector<long long> hacc((size_t)5 * n);
    CK(cudaMemcpyAsync(b->success, success, n * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaMemcpyAsync(b->cycles, cycles, n * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaMemcpyAsync(b->status, status, n * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaMemcpyAsync(hacc.data(), acc, (size_t)5 * n * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaMemcpyAsync(b->elapsed, elapsed, n * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaStreamSynchronize(c->stream), "D2H");
    for (int i = 0; i < n; ++i) {
        b->n_nu[i] = hacc[i];
        b->n_alpha[i] = hacc[n + i];
        b->nb_nu[i] = hacc[2 * n + i];
        b->nb_alpha[i] = hacc[3 * n + i];
        b->atoms_lost[i] = hacc[4 * n + i];
    }
    return RECON_OK;
}
