/* TEST INFRASTRUCTURE: recon_pipeline_stats for the CPU checkers (the C
 * oracle and the compiled reference behind the same C-ABI; pointers are host
 * memory).  The digest64 definition is in include/recon_b200.h; the device
 * computes it in paper_2504_06182_b200/csrc/stats.cu. */
#ifndef RECON_DIGEST_CPU_H
#define RECON_DIGEST_CPU_H

#include <stdint.h>

#include "recon_b200.h"

static inline uint64_t recon_dg_mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t recon_dg_elem(uint64_t tag, uint64_t i, int32_t v) {
    return recon_dg_mix(recon_dg_mix((tag << 48) ^ i) ^ (uint64_t)(uint32_t)v);
}

static inline recon_status recon_dg_stats(const recon_pipeline_batch *pb, recon_instance_stats *out) {
    if (!pb || !out || !pb->grid.status || !pb->grid.path_count || !pb->grid.path_src || !pb->grid.path_dst ||
        !pb->grid.total_displacement || !pb->move_batch || !pb->batch_count)
        return RECON_ERR_ARGUMENT;
    const recon_grid_batch *g = &pb->grid;
    const int64_t S = (int64_t)g->width * g->h_prime;
    for (int32_t inst = 0; inst < g->count; ++inst) {
        recon_instance_stats r;
        r.status = g->status[inst];
        r.detail = g->detail ? g->detail[inst] : 0;
        r.path_count = 0;
        r.displaced_tokens = 0;
        r.total_displacement = 0;
        r.batch_count = 0;
        if (r.status != RECON_OK) {
            r.digest = recon_dg_mix(recon_dg_elem(4, 0, r.status));
            out[inst] = r;
            continue;
        }
        const int32_t P = g->path_count[inst];
        const int64_t D = g->total_displacement[inst];
        const int32_t nb = pb->batch_count[inst];
        const int32_t *src = g->path_src + inst * S, *dst = g->path_dst + inst * S;
        const int32_t *mb = pb->move_batch + inst * pb->move_stride;
        uint64_t acc = 0;
        int32_t disp = 0;
        for (int32_t i = 0; i < P; ++i) {
            acc += recon_dg_elem(1, (uint64_t)i, src[i]) + recon_dg_elem(2, (uint64_t)i, dst[i]);
            disp += src[i] != dst[i];
        }
        for (int64_t j = 0; j < D; ++j) acc += recon_dg_elem(3, (uint64_t)j, mb[j]);
        acc += recon_dg_elem(5, 0, P) + recon_dg_elem(6, 0, (int32_t)(uint32_t)(D & 0xffffffffll)) +
               recon_dg_elem(7, 0, (int32_t)(D >> 32)) + recon_dg_elem(8, 0, nb);
        r.path_count = P;
        r.displaced_tokens = disp;
        r.total_displacement = D;
        r.batch_count = nb;
        r.digest = recon_dg_mix(acc);
        out[inst] = r;
    }
    return RECON_OK;
}

/* recon_pipeline_schedule_runs over host pointers */
static inline recon_status recon_dg_runs(const recon_pipeline_batch *pb, recon_schedule_runs *runs) {
    if (!pb || !runs || !runs->run_slot || !runs->run_batch || !runs->run_count || !pb->move_batch ||
        !pb->grid.status || !pb->grid.total_displacement)
        return RECON_ERR_ARGUMENT;
    int over = 0;
    for (int32_t inst = 0; inst < pb->grid.count; ++inst) {
        const int64_t D = pb->grid.status[inst] == RECON_OK ? pb->grid.total_displacement[inst] : 0;
        const int32_t *mb = pb->move_batch + inst * pb->move_stride;
        int32_t *rs = runs->run_slot + inst * runs->run_stride, *rb = runs->run_batch + inst * runs->run_stride;
        int64_t r = 0;
        for (int64_t j = 0; j < D; ++j)
            if (j == 0 || mb[j] != mb[j - 1] + 1) {
                if (r < runs->run_stride) {
                    rs[r] = (int32_t)j;
                    rb[r] = mb[j];
                }
                ++r;
            }
        runs->run_count[inst] = r;
        over |= r > runs->run_stride;
    }
    return over ? RECON_ERR_CAPACITY : RECON_OK;
}

#endif
