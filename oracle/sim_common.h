/*
 * oracle/sim_common.h — TEST INFRASTRUCTURE (checker), shared by the C oracle
 * and the reference-backed library: a sequential restatement of the loss
 * simulation documented in include/recon_b200.h (SPEC.md [MODULE] sim), one
 * trial at a time, on top of a solver callback (the oracle's own solvers, or
 * the compiled reference's red_rec / bird / batch_moves).  The B200 library
 * implements the same model independently (csrc/sim.cu).
 */
#ifndef RECON_SIM_COMMON_H
#define RECON_SIM_COMMON_H

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "recon_b200.h"
#include "recon_sim_rng.h"

/* solve (+ batch) one instance: fills g's outputs, *nb and mb when batching */
typedef recon_status (*sim_solve_fn)(int batching, int solver, int preset, recon_grid_batch *g, int64_t ms,
                                     int32_t *mb, int32_t *nb);

static inline int simc_getbit(const uint64_t *m, int d) { return (int)((m[d >> 6] >> (d & 63)) & 1ULL); }

static inline void *simc_alloc(size_t n) {
    void *p = calloc(n ? n : 1, 1);
    if (!p) abort();
    return p;
}

static inline int simc_band_full(const uint64_t *occ, int W, int H, int hp) {
    const int wpc = (H + 63) / 64, ylo = (H - hp) / 2;
    for (int x = 0; x < W; ++x)
        for (int y = ylo; y < ylo + hp; ++y)
            if (!simc_getbit(occ + (size_t)x * wpc, y)) return 0;
    return 1;
}

static inline int64_t simc_atoms(const uint64_t *occ, int W, int H) {
    int64_t n = 0;
    for (int64_t i = 0; i < (int64_t)W * ((H + 63) / 64); ++i) n += __builtin_popcountll(occ[i]);
    return n;
}

static inline void simc_trial(const recon_sim_batch *b, int i, sim_solve_fn solve) {
    const int W = b->width, H = b->height, hp = b->h_prime, wpc = (H + 63) / 64;
    const int64_t S = (int64_t)W * hp, ms = (int64_t)W * hp * (W + H) + 1, nt = (int64_t)W * hp;
    const uint64_t seed = b->seed_base + (uint64_t)i;
    const recon_loss_model L = b->loss;
    const size_t words = (size_t)W * wpc;
    uint64_t *occ = (uint64_t *)simc_alloc(words * 8), *nxt = (uint64_t *)simc_alloc(words * 8);
    memcpy(occ, b->occ + (size_t)i * words, words * 8);
    int32_t *ps = (int32_t *)simc_alloc((size_t)S * 4), *pt = (int32_t *)simc_alloc((size_t)S * 4);
    int32_t *mb = (int32_t *)simc_alloc((size_t)ms * 4), *bcnt = (int32_t *)simc_alloc((size_t)ms * 4);
    int32_t *runid = (int32_t *)simc_alloc((size_t)ms * 4);
    int64_t *off = (int64_t *)simc_alloc(((size_t)S + 1) * 8);
    char *allc = (char *)simc_alloc((size_t)ms);
    int success = 0, cycles = 0, status = RECON_OK;
    int64_t n_nu = 0, n_al = 0, nb_nu = 0, nb_al = 0, lost = 0;
    double elapsed = 0.0;
    int64_t atoms = simc_atoms(occ, W, H);
    for (int cyc = 0; atoms >= nt && cyc < b->max_cycles; ++cyc) {
        int32_t pc = 0, st = 0, det = 0, nbc = 0;
        int64_t td = 0;
        recon_grid_batch g;
        memset(&g, 0, sizeof g);
        g.occ = occ;
        g.count = 1;
        g.width = W;
        g.height = H;
        g.h_prime = hp;
        g.path_src = ps;
        g.path_dst = pt;
        g.path_count = &pc;
        g.total_displacement = &td;
        g.status = &st;
        g.detail = &det;
        recon_status rs = solve(b->batching, b->solver, b->preset, &g, ms, mb, &nbc);
        if (rs != RECON_OK) st = rs;
        if (st != RECON_OK) {
            status = st;
            break;
        }
        ++cycles;
        int64_t D = 0, moved = 0;
        for (int32_t p = 0; p < pc; ++p) {
            const int dx = ps[p] / H - pt[p] / H, dy = ps[p] % H - pt[p] % H;
            const int64_t len = (dx < 0 ? -dx : dx) + (dy < 0 ? -dy : dy);
            off[p] = D;
            D += len;
            moved += len > 0;
        }
        off[pc] = D;
        int64_t nruns = 0;
        if (b->batching) { /* EDI runs: consecutive batches moving the same token set */
            for (int32_t k = 0; k < nbc; ++k) {
                bcnt[k] = 0;
                allc[k] = 1;
            }
            for (int32_t p = 0; p < pc; ++p)
                for (int64_t k = off[p]; k < off[p + 1]; ++k) {
                    const int32_t bb = mb[k];
                    bcnt[bb]++;
                    if (!(k + 1 < off[p + 1] && mb[k + 1] == bb + 1)) allc[bb] = 0;
                }
            for (int32_t k = 0; k < nbc; ++k)
                runid[k] = k == 0 ? 0 : runid[k - 1] + !(bcnt[k - 1] == bcnt[k] && allc[k - 1]);
            nruns = nbc ? runid[nbc - 1] + 1 : 0;
        }
        const double cyc_el = b->batching ? 2.0 * L.t_alpha * (double)nruns + L.t_nu * (double)nbc
                                          : 2.0 * L.t_alpha * (double)moved + L.t_nu * (double)D;
        nb_nu += b->batching ? nbc : D;
        nb_al += b->batching ? nruns : moved;
        const int64_t before = atoms;
        memcpy(nxt, occ, words * 8);
        for (int32_t p = 0; p < pc; ++p) nxt[(size_t)(ps[p] / H) * wpc + (ps[p] % H) / 64] &= ~(1ULL << ((ps[p] % H) & 63));
        for (int32_t p = 0; p < pc; ++p) { /* extract, k moves, implant (N counts are batching-independent) */
            const int64_t len = off[p + 1] - off[p];
            const uint64_t base = (uint64_t)p * 4096;
            int alive = 1;
            if (len > 0) {
                n_al++;
                alive = recon_sim_u01(seed, (uint32_t)cyc, RECON_DRAW_EXTRACT, base) < L.p_alpha;
            }
            for (int64_t k = 0; k < len && alive; ++k) {
                n_nu++;
                alive = recon_sim_u01(seed, (uint32_t)cyc, RECON_DRAW_MOVE, base + (uint64_t)k) < L.p_nu;
            }
            if (len > 0 && alive) {
                n_al++;
                alive = recon_sim_u01(seed, (uint32_t)cyc, RECON_DRAW_IMPLANT, base) < L.p_alpha;
            }
            if (alive) nxt[(size_t)(pt[p] / H) * wpc + (pt[p] % H) / 64] |= 1ULL << ((pt[p] % H) & 63);
        }
        const double pdec = L.tau > 0.0 ? exp(-(cyc_el + L.t_meas) / L.tau) : 1.0;
        for (int64_t v = 0; v < (int64_t)W * H; ++v) {
            uint64_t *w = nxt + (size_t)(v / H) * wpc + (v % H) / 64;
            const uint64_t bit = 1ULL << ((v % H) & 63);
            if ((*w & bit) && !(recon_sim_u01(seed, (uint32_t)cyc, RECON_DRAW_DECAY, (uint64_t)v) < pdec)) *w &= ~bit;
        }
        elapsed += cyc_el + L.t_meas;
        memcpy(occ, nxt, words * 8);
        atoms = simc_atoms(occ, W, H);
        lost += before - atoms;
        if (simc_band_full(occ, W, H, hp)) {
            success = 1;
            break;
        }
    }
    b->success[i] = success;
    b->cycles[i] = cycles;
    b->status[i] = status;
    b->n_nu[i] = n_nu;
    b->n_alpha[i] = n_al;
    b->nb_nu[i] = nb_nu;
    b->nb_alpha[i] = nb_al;
    b->atoms_lost[i] = lost;
    b->elapsed[i] = elapsed;
    free(occ);
    free(nxt);
    free(ps);
    free(pt);
    free(mb);
    free(bcnt);
    free(runid);
    free(off);
    free(allc);
}

static inline recon_status sim_run_checked(const recon_sim_batch *b, sim_solve_fn solve) {
    if (!b || !b->occ || !b->success || !b->cycles || !b->status || !b->n_nu || !b->n_alpha || !b->nb_nu ||
        !b->nb_alpha || !b->atoms_lost || !b->elapsed || b->width <= 0 || b->height <= 0 || b->h_prime <= 0 ||
        b->h_prime >= b->height)
        return RECON_ERR_ARGUMENT;
    for (int32_t i = 0; i < b->count; ++i) simc_trial(b, i, solve);
    return RECON_OK;
}

#endif
