// Shared device helpers for the recon B200 kernels (sm_100a).
//
// Everything on this path is integer bit/scan work: column occupancies are
// u64 bit planes in shared memory, counts come from popc, ranks from warp
// ballots and shuffle scans.  No tensor cores (nothing is a contraction).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "recon_b200.h"

namespace rb {

// Device-side invariant checks of the checked build (-DRECON_CHECKED,
// tools/checked_run.sh): a failed check prints and traps, so the launch
// fails loudly.  They compile to nothing in the product build.
#ifdef RECON_CHECKED
#define RB_CHECK(cond, what)                                                                          \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            printf("RB_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,       \
                   (int)blockIdx.x, (int)threadIdx.x);                                                \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define RB_CHECK(cond, what) (void)0
#endif

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// exclusive warp scan; *total receives the warp sum
__device__ __forceinline__ int warp_excl_scan(int v, int *total) {
    const int lane = lane_id();
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    *total = __shfl_sync(FULL, x, 31);
    return x - v;
}

// predicated atomic add that returns the old value without a branch: a run of
// these issues back to back (a conditional atomicAdd becomes a branch, and
// ptxas then places the first use of each result right after its atomic,
// one round trip per atomic)
__device__ __forceinline__ uint32_t atom_add_if(bool p, uint32_t *addr, uint32_t v) {
    uint32_t r = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q atom.global.add.u32 %0, [%1], %3;\n\t}"
                 : "+r"(r)
                 : "l"(addr), "r"((uint32_t)p), "r"(v)
                 : "memory");
    return r;
}

// grid-stride position over count x S items as (instance, index), advanced
// without a 64-bit division per step
struct InstIter {
    int64_t t, inst, S, q;  // q, r: the stride in instances and items
    int i, r;
    int64_t stride;
    __device__ __forceinline__ InstIter(int64_t start, int64_t S_, int64_t stride_) : t(start), S(S_), stride(stride_) {
        inst = start / S_;
        i = (int)(start - inst * S_);
        q = stride_ / S_;
        r = (int)(stride_ - q * S_);
    }
    __device__ __forceinline__ void next() {
        t += stride;
        inst += q;
        i += r;
        if (i >= S) {
            i -= (int)S;
            ++inst;
        }
    }
};

// pulls [p, p + bytes) into L2 ahead of use (no register result, never stalls)
__device__ __forceinline__ void prefetch_l2(const void *p, int bytes) {
    const char *c = static_cast<const char *>(p);
    for (int o = 0; o < bytes; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(c + o));
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

__device__ __forceinline__ long long warp_sum64(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(FULL, v, o);
        v = y < v ? y : v;
    }
    return v;
}

__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

// bits [a, b) of a 32-bit chunk whose bit 0 is depth `base`
__device__ __forceinline__ uint32_t chunk_range(int base, int B, int a, int b) {
    const int lo = max(a - base, 0), hi = min(b - base, B);
    if (hi <= lo) return 0u;
    const uint32_t top = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
    return top & ~((1u << lo) - 1u);
}

// bits [a, b) of a 64-bit word whose bit 0 is depth `base`
__device__ __forceinline__ uint64_t word_range(int base, int a, int b) {
    const int lo = max(a - base, 0), hi = min(b - base, 64);
    if (hi <= lo) return 0ull;
    const uint64_t top = hi >= 64 ? ~0ull : ((1ull << hi) - 1ull);
    return top & ~((1ull << lo) - 1ull);
}

// 64 bits of a depth mask starting at depth `start` (may be negative or past
// the end; missing bits read as 0)
__device__ __forceinline__ uint64_t extract64(const uint64_t *m, int wpd, int start) {
    if (start >= wpd * 64 || start <= -64) return 0ull;
    if (start < 0) return m[0] << (-start);
    const int w = start >> 6, s = start & 63;
    const uint64_t lo = m[w] >> s;
    if (s == 0 || w + 1 >= wpd) return lo;
    return lo | (m[w + 1] << (64 - s));
}

// lane chunk of B bits (B in {8,16,32}) starting at depth lane*B
__device__ __forceinline__ uint32_t lane_chunk(const uint64_t *m, int wpd, int lane, int B) {
    const int bit = lane * B;
    if (bit >= wpd * 64) return 0u;
    const uint64_t w = m[bit >> 6] >> (bit & 63);
    return B == 32 ? (uint32_t)w : (uint32_t)(w & ((1ull << B) - 1ull));
}

// n-th (0-based) set bit of x, x has more than n set bits
__device__ __forceinline__ int nth_set_bit(uint32_t x, int n) {
    for (int i = 0; i < n; ++i) x &= x - 1;
    return __ffs(x) - 1;
}

}  // namespace rb
