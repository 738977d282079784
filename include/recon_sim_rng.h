/*
 * recon_sim_rng.h — the loss simulation's random draws (recon_sim_run).
 *
 * Counter-based: a draw is a pure function of (trial seed, cycle, kind,
 * index), so trials, tokens and operations can be evaluated in any order or
 * in parallel and still give bit-identical outcomes.  splitmix64 finalizer
 * (Steele, Lea, Flood 2014); 53-bit uniform in [0, 1).  An operation with
 * survival probability p succeeds iff recon_sim_u01(...) < p.
 */
#ifndef RECON_SIM_RNG_H
#define RECON_SIM_RNG_H

#include <stdint.h>

#ifdef __CUDACC__
#define RECON_SIM_HD __host__ __device__ __forceinline__
#else
#define RECON_SIM_HD static inline
#endif

enum { RECON_DRAW_EXTRACT = 0, RECON_DRAW_MOVE = 1, RECON_DRAW_IMPLANT = 2, RECON_DRAW_DECAY = 3 };

RECON_SIM_HD uint64_t recon_sim_mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* token draws: idx = path * 4096 + step (moves) or run ordinal (transfers);
   decay draws: idx = the atom's vertex after the cycle's moves */
RECON_SIM_HD double recon_sim_u01(uint64_t seed, uint32_t cycle, uint32_t kind, uint64_t idx) {
    const uint64_t h = recon_sim_mix(seed ^ recon_sim_mix((((uint64_t)cycle) << 8 | kind) ^ recon_sim_mix(idx)));
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

#endif
