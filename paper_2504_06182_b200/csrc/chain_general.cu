// General line assignment on sm_100a: arbitrary targets (assign_1d with any T,
// assign_1d_generalized, solve_1d's ordering and DAG).  Single instance, one
// CTA of 1024 threads.
//
// Reference: exact1d.cpp:155-207 (window_dp), :219-297 (candidate and
// certified blocks), :342-407 (assign_1d / assign_1d_generalized),
// :494-560 (order_1d_intervals, order_moves_1d).
//
// The DP runs one source row per step with every target column in parallel:
//   cur[j] = min_{s in [lo, hi], s <= j} prev[j-s] + C(j) - C(j-s),
// C = prefix sums of |pos - t|.  The reference's sliding-window deque keeps,
// among equal keys, the newest candidate (it pops while back >= new), i.e.
// the SMALLEST run s; the device keeps the first s reaching the strict
// minimum in ascending s, the same choice.  Backtracking from the last row
// then yields the lexicographically smallest use vector read from the end.

#include <climits>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "chain.cuh"
#include "common.cuh"

namespace rb {

constexpr long long INF = LLONG_MAX / 4;
constexpr int GT = 512;  // threads of the general kernel (128 registers, no spills; 1024 spilled 728 B)

using BScan = cub::BlockScan<long long, GT>;
using BScanI = cub::BlockScan<int, GT>;

struct GenShared {
    typename BScan::TempStorage scan;
    typename BScanI::TempStorage scani;
    long long carry;
    int icarry, icarry2, icarry3, imax;
    int nb, nbtot;
    long long global, wt;
    int flag;
};

// CTA-wide window DP over sources [s0, s1) and targets [t0, t1).  Returns the
// optimum (INF if infeasible); records per-cell run choices when `record`.
__device__ long long window_dp_cta(const ChainGeneralParams &p, GenShared &sh, int s0, int s1, int t0, int t1,
                                   bool record) {
    const int k = t1 - t0, tid = threadIdx.x;
    int64_t *prev = p.dp_a, *cur = p.dp_b;
    for (int j = tid; j <= k; j += GT) prev[j] = j == 0 ? 0 : INF;
    __syncthreads();
    for (int i = s0; i < s1; ++i) {
        const long long pos = p.pos[i];
        const int lo = p.min_use ? p.min_use[i] : 0;
        const int hi = p.max_use ? p.max_use[i] : 1;
        uint16_t *crow = record ? p.choice + (size_t)(i - s0) * (k + 1) : nullptr;
        if (lo == 0 && hi == 1) {
            for (int j = tid; j <= k; j += GT) {
                long long best = prev[j];
                int bs = 0;
                if (j >= 1 && prev[j - 1] < INF) {
                    const long long d = pos - p.tgt[t0 + j - 1];
                    const long long v = prev[j - 1] + (d < 0 ? -d : d);
                    if (v < best) {
                        best = v;
                        bs = 1;
                    }
                }
                cur[j] = best;
                if (record) crow[j] = (uint16_t)bs;
            }
        } else {
            // C[j] = sum_{q<j} |pos - t_q|, chunked block scan
            if (tid == 0) sh.carry = 0;
            __syncthreads();
            for (int j0 = 0; j0 <= k; j0 += GT) {
                const int j = j0 + tid;
                long long v = 0;
                if (j >= 1 && j <= k) {
                    const long long d = pos - p.tgt[t0 + j - 1];
                    v = d < 0 ? -d : d;
                }
                long long incl, tot;
                BScan(sh.scan).InclusiveSum(v, incl, tot);
                if (j <= k) p.cprefix[j] = sh.carry + incl;
                __syncthreads();
                if (tid == 0) sh.carry += tot;
                __syncthreads();
            }
            for (int j = tid; j <= k; j += GT) {
                long long best = INF;
                int bs = 0;
                for (int s = lo; s <= hi && s <= j; ++s) {
                    if (prev[j - s] >= INF) continue;
                    const long long v = prev[j - s] + p.cprefix[j] - p.cprefix[j - s];
                    if (v < best) {
                        best = v;
                        bs = s;
                    }
                }
                cur[j] = best;
                if (record) crow[j] = (uint16_t)bs;
            }
        }
        __syncthreads();
        int64_t *t = prev;
        prev = cur;
        cur = t;
    }
    const long long res = prev[k];
    __syncthreads();
    return res;
}

// backtrack (thread 0) -> use[s0..s1)
__device__ void backtrack(const ChainGeneralParams &p, int s0, int s1, int t0, int t1) {
    const int k = t1 - t0;
    int j = k;
    for (int i = s1 - 1; i >= s0; --i) {
        const int s = p.choice[(size_t)(i - s0) * (k + 1) + j];
        p.use[i] = s;
        j -= s;
    }
}

__global__ void __launch_bounds__(GT) chain_general_kernel(ChainGeneralParams p) {
    __shared__ GenShared sh;
    const int tid = threadIdx.x;
    int32_t *B = p.blocks;  // block i: B[4i..4i+3] = s0, s1, t0, t1
    for (int i = tid; i < p.ns; i += GT) p.use[i] = 0;
    if (tid == 0) {
        sh.flag = 0;
        *p.weight = 0;
        *p.status = RECON_OK;
    }
    __syncthreads();
    if (p.nt == 0) return;
    if (p.certify) {
        // ---- candidate_blocks (exact1d.cpp:219-247)
        const int n = p.n;
        for (int v = tid; v < n; v += GT) p.scratch[v] = 0;
        __syncthreads();
        for (int i = tid; i < p.ns; i += GT) atomicOr(&p.scratch[p.pos[i]], 1);
        for (int i = tid; i < p.nt; i += GT) atomicOr(&p.scratch[p.tgt[i]], 2);
        __syncthreads();
        const int E = p.ns - p.nt;
        if (tid == 0) {
            sh.icarry = 0;   // #S before chunk
            sh.icarry2 = 0;  // #T before chunk
            sh.icarry3 = 0;  // #cuts before chunk
            sh.imax = 0;     // max(0, eligible D) so far
        }
        __syncthreads();
        // cuts stored as boundaries (PS, PT) in scratch-free area: B rows 1..
        for (int v0 = 0; v0 < n; v0 += GT) {
            const int v = v0 + tid;
            const int f = v < n ? p.scratch[v] : 0;
            const int s = f & 1, t = (f >> 1) & 1;
            int ps, pt, tot_s, tot_t;
            BScanI(sh.scani).ExclusiveSum(s, ps, tot_s);
            __syncthreads();
            BScanI(sh.scani).ExclusiveSum(t, pt, tot_t);
            __syncthreads();
            ps += sh.icarry;
            pt += sh.icarry2;
            const int D = ps - pt;
            const bool elig = v < n && !s && !t && D <= E;
            int em;
            int dummy;
            BScanI(sh.scani).ExclusiveScan(elig ? D : INT_MIN, em, cub::Max(), dummy);
            __syncthreads();
            if (tid == 0) em = INT_MIN;
            const int bar = max(sh.imax, em);
            const bool cut = elig && D >= bar;
            int cidx, ncut;
            BScanI(sh.scani).ExclusiveSum(cut ? 1 : 0, cidx, ncut);
            __syncthreads();
            if (cut) {
                const int c = sh.icarry3 + cidx + 1;  // boundary index (0 is the chain start)
                B[4 * c + 0] = ps;
                B[4 * c + 2] = pt;
            }
            int mx = elig ? D : INT_MIN;
            mx = __reduce_max_sync(FULL, mx);
            if ((tid & 31) == 0 && mx > INT_MIN) atomicMax(&sh.imax, mx);
            __syncthreads();
            if (tid == 0) {
                sh.icarry += tot_s;
                sh.icarry2 += tot_t;
                sh.icarry3 += ncut;
            }
            __syncthreads();
        }
        // boundaries 0 .. ncut+1 -> non-empty blocks (thread 0)
        if (tid == 0) {
            const int ncut = sh.icarry3;
            B[0] = 0;
            B[2] = 0;
            B[4 * (ncut + 1) + 0] = p.ns;
            B[4 * (ncut + 1) + 2] = p.nt;
            int nb = 0;
            int ps0 = B[0], pt0 = B[2];
            // compact into (s0, s1, t0, t1) rows in place (row nb <= row q)
            for (int q = 0; q <= ncut; ++q) {
                const int s1 = B[4 * (q + 1) + 0], t1 = B[4 * (q + 1) + 2];
                if (s1 > ps0 || t1 > pt0) {
                    B[4 * nb + 0] = ps0;
                    B[4 * nb + 1] = s1;
                    B[4 * nb + 2] = pt0;
                    B[4 * nb + 3] = t1;
                    ++nb;
                }
                ps0 = s1;
                pt0 = t1;
            }
            sh.nb = nb;
        }
        __syncthreads();
        // ---- certified_blocks (exact1d.cpp:255-297)
        if (sh.nb > 1) {
            const long long global = window_dp_cta(p, sh, 0, p.ns, 0, p.nt, false);
            long long sum = 0;
            for (int i = 0; i < sh.nb; ++i) {
                const long long w = B[4 * i + 3] > B[4 * i + 2]
                                        ? window_dp_cta(p, sh, B[4 * i], B[4 * i + 1], B[4 * i + 2], B[4 * i + 3], false)
                                        : 0;
                if (tid == 0) p.wts[i] = w;
                sum += w;
            }
            __syncthreads();
            if (sum != global) {
                int i = 0;
                while (i + 1 < sh.nb) {
                    const int a0 = B[4 * i], a2 = B[4 * i + 2];
                    const int b1 = B[4 * (i + 1) + 1], b3 = B[4 * (i + 1) + 3];
                    const long long wj = b3 > a2 ? window_dp_cta(p, sh, a0, b1, a2, b3, false) : 0;
                    const bool merge = wj < p.wts[i] + p.wts[i + 1];
                    __syncthreads();
                    if (merge) {
                        if (tid == 0) {
                            B[4 * i + 1] = b1;
                            B[4 * i + 3] = b3;
                            p.wts[i] = wj;
                            for (int q = i + 1; q + 1 < sh.nb; ++q) {
                                for (int r = 0; r < 4; ++r) B[4 * q + r] = B[4 * (q + 1) + r];
                                p.wts[q] = p.wts[q + 1];
                            }
                            sh.nb -= 1;
                        }
                        __syncthreads();
                        if (i > 0) --i;
                    } else {
                        ++i;
                    }
                }
                sum = 0;
                for (int q = 0; q < sh.nb; ++q) sum += p.wts[q];
                if (sum != global) {
                    if (tid == 0) {
                        B[0] = 0;
                        B[1] = p.ns;
                        B[2] = 0;
                        B[3] = p.nt;
                        sh.nb = 1;
                    }
                }
                __syncthreads();
            }
        }
    } else {
        if (tid == 0) {
            B[0] = 0;
            B[1] = p.ns;
            B[2] = 0;
            B[3] = p.nt;
            sh.nb = 1;
        }
        __syncthreads();
    }
    // ---- per-block window DP with the reference tie rule
    long long total = 0;
    for (int q = 0; q < sh.nb; ++q) {
        const int s0 = B[4 * q], s1 = B[4 * q + 1], t0 = B[4 * q + 2], t1 = B[4 * q + 3];
        if (t1 <= t0) continue;
        const long long w = window_dp_cta(p, sh, s0, s1, t0, t1, true);
        if (w >= INF) {
            if (tid == 0) *p.status = RECON_ERR_INFEASIBLE;
            break;
        }
        total += w;
        if (tid == 0) backtrack(p, s0, s1, t0, t1);
        __syncthreads();
    }
    if (tid == 0 && *p.status == RECON_OK) {
        *p.weight = total;
        // pairs in source order (= target order): exact1d.cpp:362-367, :398-405
        int tp = 0;
        for (int i = 0; i < p.ns; ++i)
            for (int u = 0; u < p.use[i]; ++u) {
                p.pair_src[tp] = p.pos[i];
                p.pair_dst[tp] = p.tgt[tp];
                ++tp;
            }
    }
}

cudaError_t launch_chain_general(const ChainGeneralParams &p, cudaStream_t st) {
    chain_general_kernel<<<1, GT, 0, st>>>(p);
    return cudaGetLastError();
}

// --------------------------------------------------------------------------
// solve_1d ordering + span-overlap DAG
// --------------------------------------------------------------------------

// order: rights (t > s) by target desc, lefts by target asc, isolated by index.
// Paths arrive in target order, so rights desc = reverse index order.
__global__ void chain_order_kernel(int P, const int32_t *src, const int32_t *dst, int32_t *order, int32_t *rank,
                                   unsigned long long *sweep_keys, unsigned long long *hi_keys) {
    __shared__ int cnt[3];
    if (threadIdx.x < 3) cnt[threadIdx.x] = 0;
    __syncthreads();
    // counts (single CTA)
    int r = 0, l = 0;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        r += dst[i] > src[i];
        l += dst[i] < src[i];
    }
    atomicAdd(&cnt[0], r);
    atomicAdd(&cnt[1], l);
    __syncthreads();
    const int nr = cnt[0], nl = cnt[1];
    // stable positions via a sequential-per-class prefix (P small, single instance)
    if (threadIdx.x == 0) {
        int ri = 0, li = 0, ii = 0;
        for (int i = 0; i < P; ++i) {
            int slot;
            if (dst[i] > src[i]) slot = nr - 1 - ri++;
            else if (dst[i] < src[i]) slot = nr + li++;
            else slot = nr + nl + ii++;
            order[slot] = i;
            rank[i] = slot;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const long long lo = min(src[i], dst[i]), hi = max(src[i], dst[i]);
        sweep_keys[i] = ((unsigned long long)lo << 32) | (unsigned)i;  // sweep order (lo, id)
        (void)hi;
        (void)hi_keys;
    }
}

// after sorting sweep_keys: sweep_id[pos] = id; hi-keys (hi << 32 | pos)
__global__ void chain_sweep_kernel(int P, const unsigned long long *sweep_sorted, const int32_t *src,
                                   const int32_t *dst, int32_t *sweep_id, unsigned long long *hi_keys) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < P; q += gridDim.x * blockDim.x) {
        const int id = (int)(sweep_sorted[q] & 0xffffffffull);
        sweep_id[q] = id;
        const long long hi = max(src[id], dst[id]);
        hi_keys[q] = ((unsigned long long)hi << 32) | (unsigned)q;
    }
}

// span at sweep position q: edges to earlier spans with hi >= lo, iterated by
// (hi, sweep position) — the multimap order of exact1d.cpp:548-559
template <bool WRITE>
__global__ void chain_edges_kernel(int P, const int32_t *src, const int32_t *dst, const int32_t *sweep_id,
                                   const unsigned long long *hi_sorted, const int32_t *rank, int64_t *cnt,
                                   int32_t *ea, int32_t *eb) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < P; q += gridDim.x * blockDim.x) {
        const int me = sweep_id[q];
        const long long lo = min(src[me], dst[me]);
        // first index in hi_sorted with hi >= lo
        int a = 0, b = P;
        while (a < b) {
            const int m = (a + b) >> 1;
            if ((long long)(hi_sorted[m] >> 32) < lo) a = m + 1;
            else b = m;
        }
        int64_t o = WRITE ? cnt[q] : 0;
        int64_t c = 0;
        for (int m = a; m < P; ++m) {
            const int qp = (int)(hi_sorted[m] & 0xffffffffull);
            if (qp >= q) continue;
            if (WRITE) {
                const int other = sweep_id[qp];
                const int x = rank[other] < rank[me] ? other : me;
                const int y = x == other ? me : other;
                ea[o] = x;
                eb[o] = y;
                ++o;
            }
            ++c;
        }
        if (!WRITE) cnt[q] = c;
    }
}

size_t chain_order_temp_bytes(int P) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, a, (unsigned long long *)nullptr, (unsigned long long *)nullptr, P);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t *)nullptr, (int64_t *)nullptr, P + 1);
    return a > b ? a : b;
}

cudaError_t chain_order_count(const ChainOrderParams &p, cudaStream_t st, int64_t *n_edges) {
    const int P = p.P;
    chain_order_kernel<<<1, 256, 0, st>>>(P, p.src, p.dst, p.order, p.rank, p.keys_a, p.keys_b);
    size_t tb = p.temp_bytes;
    cub::DeviceRadixSort::SortKeys(p.temp, tb, p.keys_a, p.keys_b, P, 0, 64, st);
    const int blocks = (P + 255) / 256 + 1;
    chain_sweep_kernel<<<blocks, 256, 0, st>>>(P, p.keys_b, p.src, p.dst, p.sweep_id, p.keys_a);
    tb = p.temp_bytes;
    cub::DeviceRadixSort::SortKeys(p.temp, tb, p.keys_a, p.keys_b, P, 0, 64, st);  // keys_b = hi-sorted
    chain_edges_kernel<false><<<blocks, 256, 0, st>>>(P, p.src, p.dst, p.sweep_id, p.keys_b, p.rank, p.cnt, nullptr,
                                                      nullptr);
    cudaMemsetAsync(p.cnt + P, 0, 8, st);
    tb = p.temp_bytes;
    cub::DeviceScan::ExclusiveSum(p.temp, tb, p.cnt, p.cnt, P + 1, st);
    cudaError_t e = cudaMemcpyAsync(n_edges, p.cnt + P, 8, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t chain_order_emit(const ChainOrderParams &p, cudaStream_t st) {
    const int blocks = (p.P + 255) / 256 + 1;
    chain_edges_kernel<true><<<blocks, 256, 0, st>>>(p.P, p.src, p.dst, p.sweep_id, p.keys_b, p.rank, p.cnt, p.ea,
                                                     p.eb);
    return cudaGetLastError();
}

}  // namespace rb
