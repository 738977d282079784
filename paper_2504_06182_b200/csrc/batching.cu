// batch_moves on sm_100a: one WARP per instance.
//
// Reference: /root/reference/proj/src/batching.cpp:28-159 (Alg. 4).
//
// State per instance (global scratch): occupancy bitmap, per-path next edge,
// per-path blocker counts, a SORTED ready list (the reference's std::set).
// Each batch:
//   1. the ready list is scanned in ascending id, 32 candidates per step; a
//      candidate's next move (from -> to) needs `to` free in the PRE-batch
//      occupancy, no vertex shared with an accepted move, and the constraint
//      predicate against every accepted move (batching.cpp:107-125).  Inside
//      a step the greedy ascending acceptance is resolved with a 32-round
//      shuffle over per-lane conflict masks; earlier steps are seen through
//      an in-batch vertex bitmap and the batch's first move;
//   2. no acceptance while moves remain -> InputError "batching made no
//      progress" (batching.cpp:127-128);
//   3. atomic application (sources vacated, then destinations filled);
//   4. finished paths release successors, which join the ready list for the
//      NEXT batch (batching.cpp:138-148): ready = (ready - finished) merged
//      with the sorted newly-released ids, by rank.
// The batch index of every move is written at its path-major slot.

#include <algorithm>
#include <climits>
#include <type_traits>
#include <cub/device/device_scan.cuh>

#include "batching.cuh"
#include "common.cuh"

#include "leap.cuh"

namespace rb {

struct ExplicitPaths {
    const int64_t *off;
    const int32_t *verts;
    __device__ __forceinline__ int len(int p) const { return (int)(off[p + 1] - off[p] - 1); }
    __device__ __forceinline__ int32_t v(int p, int k) const { return verts[off[p] + k]; }
    __device__ __forceinline__ int64_t move_base(int p) const { return off[p] - p; }
};

// one-bend staircase: horizontal along the source row, then vertical
// (virtual_line.cpp:150-173)
struct ImplicitPaths {
    const int32_t *src, *dst;
    const int64_t *base;  // [P] path-major move offsets (minus base0)
    int64_t base0;
    int H;
    __device__ __forceinline__ int len(int p) const {
        const int s = src[p], t = dst[p];
        return abs(s / H - t / H) + abs(s % H - t % H);
    }
    __device__ __forceinline__ int32_t v(int p, int k) const {
        const int s = src[p], t = dst[p];
        const int xs = s / H, ys = s % H, xt = t / H, yt = t % H;
        const int dx = abs(xt - xs);
        if (k <= dx) return (xs + (xt > xs ? k : -k)) * H + ys;
        const int m = k - dx;
        return xt * H + ys + (yt > ys ? m : -m);
    }
    __device__ __forceinline__ int64_t move_base(int p) const { return base[p] - base0; }
};

// one ready path cached in a lane's registers (register-resident frontier)
struct LanePath {
    int p, k, len, xs, ys, xt, yt;
    int64_t base;
    int64_t q0, q1;  // successor CSR range, prefetched when the lane is filled (leap mode)
    int pf;          // leap mode: the successors' records and blocker counts still to prefetch
    int pn;          // leap mode: new since the cached pair meetings (leap_delta's cache)
    __device__ __forceinline__ int32_t v(int H, int kk) const {
        const int dx = abs(xt - xs);
        if (kk <= dx) return (xs + (xt > xs ? kk : -kk)) * H + ys;
        const int m = kk - dx;
        return xt * H + ys + (yt > ys ? m : -m);
    }
};

// vertex bitmaps (occupancy, in-batch); SM = in shared memory, accessed with
// ld.shared / atom.shared (a generic pointer would take the generic path)
template <bool SM>
struct Bits {
    uint32_t *p;
    uint32_t sa;  // shared-window address of p when SM
    __device__ explicit Bits(uint32_t *q) : p(q), sa(SM ? (uint32_t)__cvta_generic_to_shared(q) : 0u) {}
    __device__ __forceinline__ bool get(int v) const {
        uint32_t x;
        if (SM) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(sa + ((uint32_t)(v >> 5) << 2)));
        else x = p[v >> 5];
        return (x >> (v & 31)) & 1u;
    }
    __device__ __forceinline__ void set(int v) const {
        if (SM) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(sa + ((uint32_t)(v >> 5) << 2)), "r"(1u << (v & 31)) : "memory");
        else atomicOr(&p[v >> 5], 1u << (v & 31));
    }
    __device__ __forceinline__ void clr(int v) const {
        if (SM) asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(sa + ((uint32_t)(v >> 5) << 2)), "r"(~(1u << (v & 31))) : "memory");
        else atomicAnd(&p[v >> 5], ~(1u << (v & 31)));
    }
};

// move_dir (batching.cpp:9-15): 0 up, 1 down, 2 left, 3 right
__device__ __forceinline__ int move_dir(int H, int32_t a, int32_t b) {
    const int ay = a % H, by = b % H;
    if (by > ay) return 0;
    if (by < ay) return 1;
    if (b / H < a / H) return 2;
    return 3;
}

// ConstraintSet::compatible (batching.cpp:17-24)
__device__ __forceinline__ bool compatible(int preset, int H, int32_t af, int32_t at, int32_t bf, int32_t bt) {
    if (preset == 0) return true;
    const int da = move_dir(H, af, at), db = move_dir(H, bf, bt);
    if (da != db) return false;
    if (da <= 1) return af / H == bf / H;
    return af % H == bf % H;
}

// sorts up to 32 ints held one per lane (INT_MAX = empty), ascending
__device__ __forceinline__ int warp_sort32(int v) {
    const int lane = lane_id();
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const int o = __shfl_xor_sync(FULL, v, j);
            const bool up = (lane & k) == 0;
            const bool lower = (lane & j) == 0;
            const int mn = min(v, o), mx = max(v, o);
            v = (lower == up) ? mn : mx;
        }
    }
    return v;
}

// #elements < x in a sorted array
__device__ __forceinline__ int lower_bound_i32(const int32_t *a, int n, int x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (a[m] < x) lo = m + 1;
        else hi = m;
    }
    return lo;
}

// The general entry point (arbitrary paths, given dag): the literal
// pairwise checks.  (The solver pipeline runs batch_warp_pipe below.)
// end of path p's successor list
__device__ __forceinline__ int64_t list_end(const BatchJob &J, int p) {
    return J.slen ? J.soff[p] + J.slen[p] : J.soff[p + 1];
}

template <class Paths>
__device__ void batch_warp(const BatchJob &J, const Paths &paths) {
    const int lane = lane_id();
    const int P = J.P, H = J.H;
    BatchScratch s = J.s;
    const Bits<false> occ(s.occ), inb(s.inb);
    // ---- init: next = 0, blockers = in-degree (given), finish zero-length paths
    long long left = 0;
    for (int p = lane; p < P; p += 32) {
        s.next[p] = 0;
        s.done[p] = 0;
        left += paths.len(p);
    }
    left = warp_sum64(left);
    __syncwarp();
    for (int p = lane; p < P; p += 32)
        if (paths.len(p) == 0) {
            s.done[p] = 1;
            for (int64_t q = J.soff[p]; q < list_end(J, p); ++q) atomicSub(&s.blockers[J.succ[q]], 1);
        }
    __syncwarp();
    __threadfence_block();
    int nready = 0;
    for (int p0 = 0; p0 < P; p0 += 32) {
        const int p = p0 + lane;
        const bool r = p < P && !s.done[p] && s.blockers[p] == 0;
        const unsigned m = __ballot_sync(FULL, r);
        if (r) s.ready[nready + __popc(m & lanemask_lt())] = p;
        nready += __popc(m);
    }
    __syncwarp();
    int32_t *ready = s.ready, *ready2 = s.ready2;
    int nb = 0, status = RECON_OK;
    while (left > 0) {
        // ---- 1. candidate scan (ascending id), greedy acceptance
        int nacc = 0;
        int32_t f_from = -1, f_to = -1;  // first accepted move of the batch
        if (J.edge_level) {
            // queue = every unfinished path whose edge-level release holds
            // (batching.cpp:84-102); rebuilt in ascending id
            nready = 0;
            for (int p0 = 0; p0 < P; p0 += 32) {
                const int p = p0 + lane;
                bool ok = p < P && !s.done[p];
                if (ok)
                    for (int64_t q = J.in_off[p]; q < J.in_off[p + 1] && ok; ++q) {
                        const int pred = J.in_src[q];
                        if (!s.done[pred] && s.next[pred] < J.in_need[q]) ok = false;
                    }
                const unsigned m = __ballot_sync(FULL, ok);
                if (ok) ready[nready + __popc(m & lanemask_lt())] = p;
                nready += __popc(m);
            }
            __syncwarp();
        }
        for (int c0 = 0; c0 < nready; c0 += 32) {
            const int idx = c0 + lane;
            const bool valid = idx < nready;
            int p = -1, k = 0;
            int32_t fr = -1, to = -1;
            bool cand = false;
            if (valid) {
                p = ready[idx];
                k = s.next[p];
                fr = paths.v(p, k);
                to = paths.v(p, k + 1);
                cand = !occ.get(to) && !inb.get(fr) && !inb.get(to);
                if (cand && f_from >= 0) cand = compatible(J.preset, H, fr, to, f_from, f_to);
            }
            const unsigned cm_all = __ballot_sync(FULL, cand);
            if (!cm_all) continue;
            unsigned acc = 0;
            // literal batching.cpp:107-125 greedy: pairwise vertex-disjointness
            // and the constraint predicate against earlier accepted lanes
            unsigned cm = 0;
            for (unsigned m = cm_all; m; m &= m - 1) {
                const int i = __ffs(m) - 1;
                const int32_t ofr = __shfl_sync(FULL, fr, i), oto = __shfl_sync(FULL, to, i);
                if (i < lane && cand) {
                    const bool share = ofr == fr || ofr == to || oto == fr || oto == to;
                    if (share || !compatible(J.preset, H, fr, to, ofr, oto)) cm |= 1u << i;
                }
            }
            for (unsigned m = cm_all; m; m &= m - 1) {
                const int i = __ffs(m) - 1;
                const bool a = __shfl_sync(FULL, cand && !(cm & acc), i);
                if (a) acc |= 1u << i;
            }
            if ((acc >> lane) & 1u) {
                inb.set(fr);
                inb.set(to);
                // advance the accepted path here, while its state is in registers
                const int slot = nacc + __popc(acc & lanemask_lt());
                J.move_batch[paths.move_base(p) + k] = nb;
                s.next[p] = k + 1;
                const bool fin = k + 1 == paths.len(p);
                if (fin) s.done[p] = 1;
                s.mem[slot] = fin ? (int)(0x80000000u | (unsigned)p) : p;  // bit 31: path finished
                s.mfr[slot] = fr;
                s.mto[slot] = to;
            }
            if (acc && f_from < 0) {
                const int first = __ffs(acc) - 1;
                f_from = __shfl_sync(FULL, fr, first);
                f_to = __shfl_sync(FULL, to, first);
            }
            nacc += __popc(acc);
            __syncwarp();
        }
        if (nacc == 0) {
            status = RECON_ERR_INPUT;  // batching.cpp:127-128
            break;
        }
        // ---- 3. atomic application
        for (int i = lane; i < nacc; i += 32) {
            occ.clr(s.mfr[i]);
            inb.clr(s.mfr[i]);
            inb.clr(s.mto[i]);
        }
        __syncwarp();
        for (int i = lane; i < nacc; i += 32) occ.set(s.mto[i]);
        __syncwarp();
        // ---- 4. finish and release (newly -> next batch); the moves were
        // recorded and the paths advanced during the scan
        int nnew = 0, nfin = 0;
        for (int i0 = 0; i0 < nacc; i0 += 32) {
            const int i = i0 + lane;
            bool fin = false;
            int p = -1;
            int64_t q0 = 0, q1 = 0;
            if (i < nacc) {
                const int m = s.mem[i];
                p = m & 0x7fffffff;
                fin = m < 0;
                if (fin) {
                    q0 = J.soff[p];
                    q1 = list_end(J, p);
                }
            }
            nfin += __popc(__ballot_sync(FULL, fin));
            // successors of the finished members, flattened across the warp
            int tot;
            const int base = warp_excl_scan((int)(q1 - q0), &tot);
            for (int t0 = 0; t0 < tot; t0 += 32) {
                const int t = t0 + lane;
                int owner = 0;  // largest lane with base <= t
#pragma unroll
                for (int st = 16; st > 0; st >>= 1) {
                    const int cand_l = owner + st;
                    const int b = __shfl_sync(FULL, base, cand_l);
                    if (b <= t) owner = cand_l;
                }
                const int64_t oq0 = __shfl_sync(FULL, q0, owner);
                const int ob = __shfl_sync(FULL, base, owner);
                bool released = false;
                int sc = -1;
                if (t < tot) {
                    sc = J.succ[oq0 + (t - ob)];
                    released = atomicSub(&s.blockers[sc], 1) == 1;
                }
                const unsigned rm = __ballot_sync(FULL, released);
                if (released) s.newly[nnew + __popc(rm & lanemask_lt())] = sc;
                nnew += __popc(rm);
            }
            __syncwarp();
        }
        left -= nacc;
        __syncwarp();
        if (!J.edge_level && (nfin > 0 || nnew > 0)) {
            // ready' = (ready - finished) U newly, sorted
            int nkeep = 0;
            for (int c0 = 0; c0 < nready; c0 += 32) {
                const int idx = c0 + lane;
                const int x = idx < nready ? ready[idx] : 0;
                const bool keep = idx < nready && !s.done[x];
                const unsigned m = __ballot_sync(FULL, keep);
                if (keep) ready2[nkeep + __popc(m & lanemask_lt())] = x;
                nkeep += __popc(m);
            }
            // sorted newly (in place)
            if (nnew <= 32) {
                int v = lane < nnew ? s.newly[lane] : INT_MAX;
                v = warp_sort32(v);
                if (lane < nnew) s.newly[lane] = v;
            } else {
                for (int q = lane; q < nnew; q += 32) {
                    const int x = s.newly[q];
                    int lt = 0;
                    for (int r2 = 0; r2 < nnew; ++r2) lt += s.newly[r2] < x;
                    s.mem[lt] = x;  // mem is free at this point
                }
                __syncwarp();
                for (int q = lane; q < nnew; q += 32) s.newly[q] = s.mem[q];
            }
            __syncwarp();
            // merge by rank: kept x -> i + #newly<x ; newly y -> j + #kept<y
            for (int i = lane; i < nkeep; i += 32) {
                const int x = ready2[i];
                ready[i + lower_bound_i32(s.newly, nnew, x)] = x;
            }
            for (int j = lane; j < nnew; j += 32) {
                const int y = s.newly[j];
                ready[j + lower_bound_i32(ready2, nkeep, y)] = y;
            }
            __syncwarp();
            nready = nkeep + nnew;
        }
        ++nb;
    }
    if (lane == 0) {
        *J.batch_count = status == RECON_OK ? nb : 0;
        *J.status = status;
        if (J.detail) *J.detail = status == RECON_OK ? 0 : RECON_D_BATCH_NO_PROGRESS;
    }
}

__global__ void batch_explicit_kernel(BatchJob J, ExplicitPaths paths) {
    if (threadIdx.x < 32) batch_warp<ExplicitPaths>(J, paths);
}

cudaError_t launch_batch_explicit(const BatchJob &J, const int64_t *off, const int32_t *verts, cudaStream_t st) {
    ExplicitPaths ep{off, verts};
    batch_explicit_kernel<<<1, 32, 0, st>>>(J, ep);
    return cudaGetLastError();
}

// ---- DAG preparation for the general call: CSR by source, blockers, range
// and acyclicity check (MoveDag::is_acyclic, path_system.cpp:7-39)

__global__ void edges_check_kernel(int P, int64_t E, const int32_t *es, const int32_t *ed, int32_t *bad,
                                   int32_t *outdeg, int32_t *indeg) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
        const int a = es[e], b = ed[e];
        if (a < 0 || a >= P || b < 0 || b >= P) {
            atomicExch(bad, 1);
            continue;
        }
        atomicAdd(&outdeg[a], 1);
        atomicAdd(&indeg[b], 1);
    }
}

__global__ void csr_fill_kernel(int64_t E, const int32_t *key, const int32_t *val, const int64_t *off, int32_t *fill,
                                int32_t *out, const int64_t *need_in, int64_t *need_out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
        const int a = key[e];
        const int slot = atomicAdd(&fill[a], 1);
        out[off[a] + slot] = val[e];
        if (need_out) need_out[off[a] + slot] = need_in[e];
    }
}

// layered Kahn on one CTA: counts processed nodes
__global__ void kahn_kernel(int P, const int64_t *soff, const int32_t *succ, int32_t *indeg, int32_t *frontier,
                            int32_t *next_frontier, int32_t *processed) {
    __shared__ int nf, nn, tot;
    if (threadIdx.x == 0) {
        nf = 0;
        tot = 0;
    }
    __syncthreads();
    for (int p = threadIdx.x; p < P; p += blockDim.x)
        if (indeg[p] == 0) frontier[atomicAdd(&nf, 1)] = p;
    __syncthreads();
    while (nf > 0) {
        if (threadIdx.x == 0) {
            nn = 0;
            tot += nf;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nf; i += blockDim.x) {
            const int p = frontier[i];
            for (int64_t q = soff[p]; q < soff[p + 1]; ++q)
                if (atomicSub(&indeg[succ[q]], 1) == 1) next_frontier[atomicAdd(&nn, 1)] = succ[q];
        }
        __syncthreads();
        int32_t *t = frontier;
        frontier = next_frontier;
        next_frontier = t;
        if (threadIdx.x == 0) nf = nn;
        __syncthreads();
    }
    if (threadIdx.x == 0) *processed = tot;
}

// edge-level release thresholds (batching.cpp:38-59): for dag edge i->j, the
// number of edges of P_i up to its last edge touching a vertex of P_j
__global__ void need_kernel(int64_t E, const int32_t *es, const int32_t *ed, const int64_t *off,
                            const int32_t *verts, int64_t *need) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
        const int i = es[e], j = ed[e];
        const int64_t li = off[i + 1] - off[i] - 1;
        int64_t nd = 0;
        for (int64_t k = 0; k < li; ++k) {
            const int32_t a = verts[off[i] + k], b = verts[off[i] + k + 1];
            bool touch = false;
            for (int64_t q = off[j]; q < off[j + 1] && !touch; ++q) touch = verts[q] == a || verts[q] == b;
            if (touch) nd = k + 1;
        }
        need[e] = nd;
    }
}


// --------------------------------------------------------------------------
// fused pipeline: per-instance occupancy DAG as a successor CSR + batching
// --------------------------------------------------------------------------

__global__ void occ_to_vertex_bits(int count, int W, int H, const uint64_t *occ, uint32_t *bits) {
    const int wpc = (H + 63) / 64;
    const int64_t nw = ((int64_t)W * H + 31) / 32;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)count * nw;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t inst = t / nw, w = t % nw;
        uint32_t out = 0;
        for (int b = 0; b < 32; ++b) {
            const int64_t v = w * 32 + b;
            if (v >= (int64_t)W * H) break;
            const int x = (int)(v / H), y = (int)(v % H);
            const uint64_t word = occ[(inst * W + x) * wpc + y / 64];
            out |= (uint32_t)((word >> (y % 64)) & 1ull) << b;
        }
        bits[t] = out;
    }
}

// packed coordinates x | y << 16 (path records)
__device__ __forceinline__ bool on_path2p(int ps, int pt, int x, int y) {
    const int xs = ps & 0xffff, ys = ps >> 16, xt = pt & 0xffff, yt = pt >> 16;
    if (y == ys && x >= min(xs, xt) && x <= max(xs, xt)) return true;
    if (x == xt && y >= min(ys, yt) && y <= max(ys, yt)) return true;
    return false;
}

__device__ __forceinline__ bool on_path2(int H, int32_t s, int32_t t, int32_t v) {
    const int xs = s / H, ys = s % H, xt = t / H, yt = t % H, x = v / H, y = v % H;
    if (y == ys && x >= min(xs, xt) && x <= max(xs, xt)) return true;
    if (x == xt && y >= min(ys, yt) && y <= max(ys, yt)) return true;
    return false;
}

// ---- large instances: one WARP per path, lanes over the route's vertices.
// The source/target owners of every vertex sit in one int2 map, column-major
// (x*H + y, read along vertical segments) and row-major (y*W + x, read along
// horizontal segments), so a route is read with contiguous 256-byte warp
// loads instead of one scattered load per vertex and thread.  Path i's
// out-list is [rule-2 edges (i, pb), written by i itself | rule-1 edges
// (i, j), appended by the paths j that cross source(i)], so only rule-1 edges
// need a fill counter (virtual_line.cpp:241-268 edge rules; order inside a
// list is irrelevant to batching).

// Per-vertex route coverage (how many routes contain a vertex) and target
// bitmaps give every path's out-degree without walking (below).  Coverage is
// counted as a horizontal part (row y, columns [x0, x1], the bend included)
// and a vertical part (column x, the rows past the bend): difference arrays
// rowc[y][W+1] and colc[x][H+1] per instance, prefix-summed by cover_scan_kernel.
struct CoverArrays {
    int32_t *rowc;     // [count * H * (W + 1)]
    int32_t *colc;     // [count * W * (H + 1)]
    uint32_t *rowT;    // [count * ceil(W*H/32)] target bits, row-major (y*W + x)
    uint32_t *colT;    // [count * ceil(W*H/32)] target bits, column-major (x*H + y)
};

// the cover arrays live after the two int2 maps (capi_batch.cu sizes the region)
static inline CoverArrays pipeline_cover_arrays(const PipelineArgs &a) {
    const size_t WH = (size_t)a.W * a.H;
    int32_t *base = a.source_of + (size_t)a.count * WH * 8;
    CoverArrays cv;
    cv.rowc = base;
    cv.colc = base + (size_t)a.count * a.H * (a.W + 1);
    cv.colT = a.occ;
    cv.rowT = a.inb;
    return cv;
}

__global__ void pl_mark2_kernel(PipelineArgs a, int32_t *mc, int32_t *mr, CoverArrays cv) {
    const int64_t S = (int64_t)a.W * a.k, WH = (int64_t)a.W * a.H, nwb = (WH + 31) / 32;
    const int W = a.W, H = a.H;
    int64_t cinst = -1;  // the instance whose path count is held in cP
    int cP = 0;
    for (InstIter it(blockIdx.x * (int64_t)blockDim.x + threadIdx.x, S, (int64_t)gridDim.x * blockDim.x);
         it.t < (int64_t)a.count * S; it.next()) {
        const int64_t t = it.t, inst = it.inst;
        const int p = it.i;
        if (inst != cinst) {
            cinst = inst;
            cP = a.solve_status[inst] != 0 ? 0 : a.path_count[inst];
        }
        if (p >= cP) continue;
        const int s = a.path_src[t], d = a.path_dst[t];
        const int xs = s / H, ys = s - xs * H, xd = d / H, yd = d - xd * H;
        // owner maps, 16 B per vertex: {source owner, the source owner's
        // target coordinates, target owner, the target owner's source
        // coordinates},
        // so the walk's duplicate-edge checks need no gather
        int2 *c = reinterpret_cast<int2 *>(mc + inst * WH * 4), *r = reinterpret_cast<int2 *>(mr + inst * WH * 4);
        const int ps = xs | (ys << 16), pd = xd | (yd << 16);
        int2 *pc = reinterpret_cast<int2 *>(a.prec + inst * (S + 1) + p);  // (prec .x/.y)
        *pc = make_int2(ps, pd);
        c[2 * (int64_t)s] = make_int2(p, pd);
        c[2 * (int64_t)d + 1] = make_int2(p, ps);
        r[2 * ((int64_t)ys * W + xs)] = make_int2(p, pd);
        r[2 * ((int64_t)yd * W + xd) + 1] = make_int2(p, ps);
        // coverage: horizontal part, then the vertical part past the bend
        int32_t *rc = cv.rowc + inst * (int64_t)H * (W + 1) + (int64_t)ys * (W + 1);
        atomicAdd(rc + min(xs, xd), 1);
        atomicSub(rc + max(xs, xd) + 1, 1);
        if (yd != ys) {
            int32_t *cc = cv.colc + inst * (int64_t)W * (H + 1) + (int64_t)xd * (H + 1);
            const int y0 = yd > ys ? ys + 1 : yd, y1 = yd > ys ? yd : ys - 1;
            atomicAdd(cc + y0, 1);
            atomicSub(cc + y1 + 1, 1);
        }
        const int64_t vr = (int64_t)yd * W + xd;
        atomicOr(cv.rowT + inst * nwb + (vr >> 5), 1u << (vr & 31));
        atomicOr(cv.colT + inst * nwb + ((int64_t)d >> 5), 1u << (d & 31));
    }
}

// in-place inclusive prefix sums of every row (length W+1) of rowc and every
// column (length H+1) of colc: one warp per line
__global__ void cover_scan_kernel(int count, int W, int H, CoverArrays cv) {
    const int lane = lane_id();
    const int64_t lines = (int64_t)count * (H + W);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t l = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp_id(); l < lines; l += nwarps) {
        const int64_t inst = l / (H + W), j = l % (H + W);
        int32_t *a;
        int n;
        if (j < H) {
            a = cv.rowc + inst * (int64_t)H * (W + 1) + j * (W + 1);
            n = W + 1;
        } else {
            a = cv.colc + inst * (int64_t)W * (H + 1) + (j - H) * (H + 1);
            n = H + 1;
        }
        int carry = 0;
        for (int i0 = 0; i0 < n; i0 += 32) {
            const int i = i0 + lane;
            int v = i < n ? a[i] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULL, v, o);
                if (lane >= o) v += y;
            }
            v += carry;
            if (i < n) a[i] = v;
            carry = __shfl_sync(FULL, v, 31);
        }
    }
}

__device__ __forceinline__ int cover_at(const CoverArrays &cv, int64_t inst, int W, int H, int x, int y) {
    return cv.rowc[inst * (int64_t)H * (W + 1) + (int64_t)y * (W + 1) + x] +
           cv.colc[inst * (int64_t)W * (H + 1) + (int64_t)x * (H + 1) + y];
}

// set bits of bitmap b over bit positions [lo, hi]
__device__ __forceinline__ int popc_range(const uint32_t *b, int64_t lo, int64_t hi) {
    int c = 0;
    for (int64_t w = lo >> 5; w <= (hi >> 5); ++w) {
        uint32_t m = b[w];
        if (w == (lo >> 5)) m &= ~0u << (lo & 31);
        if (w == (hi >> 5)) m &= ~0u >> (31 - (hi & 31));
        c += __popc(m);
    }
    return c;
}

// per path: rule-1 out-degree = the routes through its source but its own;
// rule-2 capacity = the targets on its route but its own (the rule-1
// duplicates among them become holes, -1); move count
__global__ void pl_degree_kernel(PipelineArgs a, CoverArrays cv) {
    const int64_t S = (int64_t)a.W * a.k, WH = (int64_t)a.W * a.H, nwb = (WH + 31) / 32;
    const int W = a.W, H = a.H;
    for (InstIter it(blockIdx.x * (int64_t)blockDim.x + threadIdx.x, S, (int64_t)gridDim.x * blockDim.x);
         it.t < (int64_t)a.count * S; it.next()) {
        const int64_t t = it.t, inst = it.inst;
        const int p = it.i;
        if (a.solve_status[inst] != 0 || p >= a.path_count[inst]) {
            a.outdeg[t] = 0;
            a.mfr[t] = 0;
            a.mbase[t] = 0;
            continue;
        }
        const int2 me = *reinterpret_cast<const int2 *>(a.prec + inst * (S + 1) + p);
        const int xs = me.x & 0xffff, ys = me.x >> 16, xt = me.y & 0xffff, yt = me.y >> 16;
        a.outdeg[t] = cover_at(cv, inst, W, H, xs, ys) - 1;
        int tg = popc_range(cv.rowT + inst * nwb, (int64_t)ys * W + min(xs, xt), (int64_t)ys * W + max(xs, xt));
        if (yt != ys) {
            const int y0 = yt > ys ? ys + 1 : yt, y1 = yt > ys ? yt : ys - 1;
            tg += popc_range(cv.colT + inst * nwb, (int64_t)xt * H + y0, (int64_t)xt * H + y1);
        }
        a.mfr[t] = tg - 1;
        a.mbase[t] = abs(xt - xs) + abs(yt - ys);
    }
}

// Path i's out-list is [rule-1 edges (i, j), appended through i's fill
// pointer by the paths j that cross source(i) | rule-2 edges (i, pb), written
// by i itself]; pl_compact_kernel then closes the gap between the two parts.
// The same walk counts i's in-degree: the sources on its route (rule 1) plus
// the routes through its target (rule 2) minus the pairs both rules give.
//
// Rule-1 edges implied by two others are dropped: the batches depend only on
// the DAG's reachability (a path is ready once all its predecessors are done,
// and a dropped predecessor reaches a kept one), and an edge (u, w) implied by
// a path u -> x -> w of the full DAG can go, because by induction over the
// edges' spans in a topological order every justifying edge is kept or
// itself implied.  For the rule-1 edge (s_b, i) at source(s_b) on i's route,
// x is the owner s_a of the previous (or next) source on i's route when s_a's
// route crosses source(s_b): then (s_b, s_a) is a rule-1 edge and (s_a, i)
// is one.  In a column of tokens that move up one after another this drops
// all but the nearest predecessor (C5: 7.4 M -> ~3.0 M edges per instance).
#ifndef RECON_WALK_MINB
#define RECON_WALK_MINB 4
#endif
__global__ void __launch_bounds__(256, RECON_WALK_MINB) pl_walk_warp_kernel(PipelineArgs a, const int4 *mc, const int4 *mr,
                                                                             CoverArrays cv) {
    const int lane = lane_id();
    const int W = a.W, H = a.H;
    const int64_t S = (int64_t)W * a.k, WH = (int64_t)W * H, N = (int64_t)a.count * S;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    unsigned long long *fillp = reinterpret_cast<unsigned long long *>(a.rec);  // next free rule-1 slot per path
    for (InstIter it(blockIdx.x * (int64_t)(blockDim.x >> 5) + warp_id(), S, nwarps); it.t < N; it.next()) {
        const int64_t t = it.t, inst = it.inst, o = inst * S;
        const int i = it.i;
        if (a.solve_status[inst] != 0 || i >= a.path_count[inst]) continue;
        const int4 *pc = a.prec + inst * (S + 1);  // packed coordinates in .x / .y
        const int2 me = *reinterpret_cast<const int2 *>(pc + i);
        const int xs = me.x & 0xffff, ys = me.x >> 16, xt = me.y & 0xffff, yt = me.y >> 16;
        const int dx = abs(xt - xs), len = dx + abs(yt - ys), sx = xt > xs ? 1 : -1, sy = yt > ys ? 1 : -1;
        const int4 *mci = mc + inst * WH, *mri = mr + inst * WH;
        int in1 = 0, dup = 0, out2 = 0;
        const int64_t r2base = a.soff[t] + a.outdeg[t];
        const int cov = lane == 0 ? cover_at(cv, inst, W, H, xt, yt) : 0;  // (issued early, used at the end)
        // the route's owner maps, up to RG chunks of 32 vertices loaded at once
#ifndef RECON_WALK_RG
#define RECON_WALK_RG 2
#endif
        constexpr int RG = RECON_WALK_RG;
        // the last rule-1 vertex of the route so far: its packed coordinates and
        // its owner's target (warp-uniform)
        int cpv = -1, cz = 0;
        for (int g0 = 0; g0 <= len; g0 += 32 * RG) {
            int4 m[RG];
            int pv[RG];  // the route vertex's packed coordinates
#pragma unroll
            for (int c = 0; c < RG; ++c) {
                const int j = g0 + 32 * c + lane;
                m[c] = make_int4(-1, 0, -1, 0);  // {source owner, its target, target owner, its source}
                const int x = j <= dx ? xs + sx * j : xt, y = j <= dx ? ys : ys + sy * (j - dx);
                pv[c] = x | (y << 16);
                if (j <= len) m[c] = j <= dx ? mri[(int64_t)y * W + x] : mci[(int64_t)x * H + y];
            }
            unsigned b1[RG];  // rule-1 lanes of each chunk
#pragma unroll
            for (int c = 0; c < RG; ++c) b1[c] = __ballot_sync(FULL, m[c].x >= 0 && m[c].x != i);
#pragma unroll
            for (int c = 0; c < RG; ++c) {
                if (g0 + 32 * c > len) break;
                // (m.x, i): i crosses source(m.x); both rules give it when m.x's
                // route (from here to m.z) crosses target(i)
                const bool r1 = b1[c] >> lane & 1u;
                // the neighbouring rule-1 vertices on the route (previous: this
                // chunk or the carry; next: this chunk or the next one loaded)
                const unsigned below = b1[c] & lanemask_lt(), above = b1[c] & ~lanemask_lt() & ~(1u << lane);
                const int pl = below ? 31 - __clz(below) : 0;
                int ppv = __shfl_sync(FULL, pv[c], pl), pz = __shfl_sync(FULL, m[c].y, pl);
                if (!below) {
                    ppv = cpv;
                    pz = cz;
                }
                int npv = -1, nz = 0;
#ifndef RECON_WALK_NONEXT
                {
                    const int nl = above ? __ffs(above) - 1 : (c + 1 < RG && b1[c + 1] ? __ffs(b1[c + 1]) - 1 : 0);
                    const int v0 = __shfl_sync(FULL, pv[c], nl), z0 = __shfl_sync(FULL, m[c].y, nl);
                    const int v1 = __shfl_sync(FULL, pv[c + 1 < RG ? c + 1 : c], nl);
                    const int z1 = __shfl_sync(FULL, m[c + 1 < RG ? c + 1 : c].y, nl);
                    if (above) {
                        npv = v0;
                        nz = z0;
                    } else if (c + 1 < RG && b1[c + 1] && g0 + 32 * (c + 1) <= len) {
                        npv = v1;
                        nz = z1;
                    }
                }
#endif
                if (b1[c]) {
                    const int last = 31 - __clz(b1[c]);
                    cpv = __shfl_sync(FULL, pv[c], last);
                    cz = __shfl_sync(FULL, m[c].y, last);
                }
                if (r1) {
                    const int bx = pv[c] & 0xffff, by = pv[c] >> 16;
                    const bool implied = (ppv >= 0 && on_path2p(ppv, pz, bx, by)) || (npv >= 0 && on_path2p(npv, nz, bx, by));
                    if (!implied) {
                        a.succ[atomicAdd(&fillp[o + m[c].x], 1ull)] = i;
                        ++in1;
                    }
                    dup += on_path2p(pv[c], m[c].y, xt, yt);
                }
                // (i, m.y): i crosses target(m.y), unless m.y's route (from m.w to
                // here) crosses source(i), which rule 1 already gives
                const bool r2 = m[c].z >= 0 && m[c].z != i && !on_path2p(m[c].w, pv[c], xs, ys);
                const unsigned b2 = __ballot_sync(FULL, r2);
                if (r2) a.succ[r2base + out2 + __popc(b2 & lanemask_lt())] = m[c].z;
                out2 += __popc(b2);
            }
        }
        in1 = warp_sum(in1);
        dup = warp_sum(dup);
        if (lane == 0) {
            a.indeg[t] = in1 + cov - 1 - dup;
            a.mfr[t] = out2;  // (the compaction's rule-2 count)
        }
    }
}

// pl_walk_warp_kernel with GW lanes per path (32 / GW paths per warp): a
// route (~69 vertices on C5) is walked GW * RG vertices at a time, so a
// route's last chunk idles fewer lanes, and a warp carries several routes'
// independent loads and atomics.  Same lists, counts and implied-edge rule;
// every collective runs on the whole warp, each group keeping to its own
// GW bits.
// The same implied-edge rule for rule-2 edges (C5: 2.9 M -> ~1.9 M edges,
// identical schedules): measured the leap phase 17 ms faster per 1,536-instance
// step but this walk 26 ms slower (its neighbour shuffles and the in-degree
// correction atomics), so off (experiments: -DRECON_RULE2_IMPLIED=1)
#ifndef RECON_RULE2_IMPLIED
#define RECON_RULE2_IMPLIED 0
#endif
constexpr bool RULE2_IMPLIED = RECON_RULE2_IMPLIED;  // (newly: the dropped rule-2 in-edges per path, zeroed)
template <int GW>  // lanes per path
__global__ void __launch_bounds__(256, RECON_WALK_MINB) pl_walk_half_kernel(PipelineArgs a, const int4 *mc, const int4 *mr,
                                                                            CoverArrays cv) {
    constexpr unsigned GM = (1u << GW) - 1u;
    const int lane = lane_id(), hl = lane & (GW - 1), hs = lane & ~(GW - 1);
    const unsigned hlt = (lanemask_lt() >> hs) & GM;  // the lanes below me in my group
    const int W = a.W, H = a.H;
    const int64_t S = (int64_t)W * a.k, WH = (int64_t)W * H, N = (int64_t)a.count * S;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    unsigned long long *fillp = reinterpret_cast<unsigned long long *>(a.rec);
    constexpr int RG = RECON_WALK_RG;
    for (InstIter it((32 / GW) * (blockIdx.x * (int64_t)(blockDim.x >> 5) + warp_id()) + hs / GW, S, (32 / GW) * nwarps);
         __any_sync(FULL, it.t < N); it.next()) {
        const int64_t t = it.t, inst = it.inst, o = inst * S;
        const int i = it.i;
        const bool act = t < N && a.solve_status[inst] == 0 && i < a.path_count[inst];
        int xs = 0, ys = 0, xt = 0, yt = 0, len = -1;
        int64_t r2base = 0;
        int cov = 0;
        const int4 *mci = mc, *mri = mr;
        if (act) {
            const int2 me = *reinterpret_cast<const int2 *>(a.prec + inst * (S + 1) + i);
            xs = me.x & 0xffff, ys = me.x >> 16, xt = me.y & 0xffff, yt = me.y >> 16;
            len = abs(xt - xs) + abs(yt - ys);
            r2base = a.soff[t] + a.outdeg[t];
            if (hl == 0) cov = cover_at(cv, inst, W, H, xt, yt);
            mci = mc + inst * WH;
            mri = mr + inst * WH;
        }
        const int dx = abs(xt - xs), sx = xt > xs ? 1 : -1, sy = yt > ys ? 1 : -1;
        const int glen = (int)__reduce_max_sync(FULL, (unsigned)(len + 1)) - 1;  // (both halves' loop)
        int in1 = 0, dup = 0, out2 = 0;
        int cpv = -1, cz = 0;  // the group's last rule-1 vertex so far and its owner's target
        int ctw = -1, cts = 0;  // (RULE2_IMPLIED) its last target vertex and that target owner's source
        for (int g0 = 0; g0 <= glen; g0 += GW * RG) {
            int4 m[RG];
            int pv[RG];
#pragma unroll
            for (int c = 0; c < RG; ++c) {
                const int j = g0 + GW * c + hl;
                m[c] = make_int4(-1, 0, -1, 0);
                const int x = j <= dx ? xs + sx * j : xt, y = j <= dx ? ys : ys + sy * (j - dx);
                pv[c] = x | (y << 16);
                if (j <= len) m[c] = j <= dx ? mri[(int64_t)y * W + x] : mci[(int64_t)x * H + y];
            }
            unsigned b1[RG];  // the group's rule-1 lanes of each chunk (GW bits)
#pragma unroll
            for (int c = 0; c < RG; ++c) b1[c] = (__ballot_sync(FULL, m[c].x >= 0 && m[c].x != i) >> hs) & GM;
            unsigned bt[RG];  // the group's lanes on another path's target
#pragma unroll
            for (int c = 0; c < RG; ++c) bt[c] = (__ballot_sync(FULL, m[c].z >= 0 && m[c].z != i) >> hs) & GM;
#pragma unroll
            for (int c = 0; c < RG; ++c) {
                const bool on = g0 + GW * c <= len;  // (this half still has vertices here)
                const bool r1 = b1[c] >> hl & 1u;
                const unsigned below = b1[c] & hlt, above = b1[c] & ~hlt & ~(1u << hl);
                const int pl = below ? 31 - __clz(below) : 0;
                int ppv = __shfl_sync(FULL, pv[c], hs + pl), pz = __shfl_sync(FULL, m[c].y, hs + pl);
                if (!below) {
                    ppv = cpv;
                    pz = cz;
                }
                int npv = -1, nz = 0;
                {
                    const int nl = above ? __ffs(above) - 1 : (c + 1 < RG && b1[c + 1] ? __ffs(b1[c + 1]) - 1 : 0);
                    const int v0 = __shfl_sync(FULL, pv[c], hs + nl), z0 = __shfl_sync(FULL, m[c].y, hs + nl);
                    const int v1 = __shfl_sync(FULL, pv[c + 1 < RG ? c + 1 : c], hs + nl);
                    const int z1 = __shfl_sync(FULL, m[c + 1 < RG ? c + 1 : c].y, hs + nl);
                    if (above) {
                        npv = v0;
                        nz = z0;
                    } else if (c + 1 < RG && b1[c + 1] && g0 + GW * (c + 1) <= len) {
                        npv = v1;
                        nz = z1;
                    }
                }
                {
                    const int last = b1[c] ? 31 - __clz(b1[c]) : 0;
                    const int lv = __shfl_sync(FULL, pv[c], hs + last), lz = __shfl_sync(FULL, m[c].y, hs + last);
                    if (b1[c]) {
                        cpv = lv;
                        cz = lz;
                    }
                }
                if (r1) {
                    const int bx = pv[c] & 0xffff, by = pv[c] >> 16;
                    const bool implied = (ppv >= 0 && on_path2p(ppv, pz, bx, by)) || (npv >= 0 && on_path2p(npv, nz, bx, by));
                    if (!implied) {
                        a.succ[atomicAdd(&fillp[o + m[c].x], 1ull)] = i;
                        ++in1;
                    }
                    dup += on_path2p(pv[c], m[c].y, xt, yt);
                }
                bool r2 = on && m[c].z >= 0 && m[c].z != i && !on_path2p(m[c].w, pv[c], xs, ys);
                if (RULE2_IMPLIED) {
                    // (i, t1) at target(t1) is implied by (i, t2) and (t2, t1) when t2,
                    // the owner of the previous or next target on i's route, passes
                    // target(t1) on its way (from its source to its target); t1's
                    // in-degree (counted from the routes through its target) loses it
                    const unsigned tb = bt[c] & hlt, ta = bt[c] & ~hlt & ~(1u << hl);
                    const int tl = tb ? 31 - __clz(tb) : 0;
                    int pw2 = __shfl_sync(FULL, pv[c], hs + tl), ps2 = __shfl_sync(FULL, m[c].w, hs + tl);
                    if (!tb) {
                        pw2 = ctw;
                        ps2 = cts;
                    }
                    int nw2 = -1, ns2 = 0;
                    {
                        const int nl = ta ? __ffs(ta) - 1 : (c + 1 < RG && bt[c + 1] ? __ffs(bt[c + 1]) - 1 : 0);
                        const int v0 = __shfl_sync(FULL, pv[c], hs + nl), s0 = __shfl_sync(FULL, m[c].w, hs + nl);
                        const int v1 = __shfl_sync(FULL, pv[c + 1 < RG ? c + 1 : c], hs + nl);
                        const int s1 = __shfl_sync(FULL, m[c + 1 < RG ? c + 1 : c].w, hs + nl);
                        if (ta) {
                            nw2 = v0;
                            ns2 = s0;
                        } else if (c + 1 < RG && bt[c + 1] && g0 + GW * (c + 1) <= len) {
                            nw2 = v1;
                            ns2 = s1;
                        }
                    }
                    {
                        const int last = bt[c] ? 31 - __clz(bt[c]) : 0;
                        const int lw = __shfl_sync(FULL, pv[c], hs + last), ls = __shfl_sync(FULL, m[c].w, hs + last);
                        if (bt[c]) {
                            ctw = lw;
                            cts = ls;
                        }
                    }
                    if (r2) {
                        const int bx = pv[c] & 0xffff, by = pv[c] >> 16;
                        if ((pw2 >= 0 && on_path2p(ps2, pw2, bx, by)) || (nw2 >= 0 && on_path2p(ns2, nw2, bx, by))) {
                            atomicAdd(&a.newly[o + m[c].z], 1);
                            r2 = false;
                        }
                    }
                }
                const unsigned b2 = (__ballot_sync(FULL, r2) >> hs) & GM;
                if (r2) a.succ[r2base + out2 + __popc(b2 & hlt)] = m[c].z;
                out2 += __popc(b2);
            }
        }
#pragma unroll
        for (int d = GW / 2; d > 0; d >>= 1) {
            in1 += __shfl_xor_sync(FULL, in1, d);
            dup += __shfl_xor_sync(FULL, dup, d);
        }
        if (act && hl == 0) {
            a.indeg[t] = in1 + cov - 1 - dup;
            a.mfr[t] = out2;
        }
    }
}

// rule-1 fill pointers: each list starts with its rule-1 part
__global__ void fillptr_kernel(int64_t n, const int64_t *soff, unsigned long long *fp) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        fp[i] = (unsigned long long)soff[i];
}

// closes each list's gap: the rule-2 part moves down to the end of the kept
// rule-1 part; slen (the out-degree array, free after the walk) = the list's
// length.  Lists stay at their offsets, so paths are independent.
__global__ void pl_compact_kernel(PipelineArgs a) {
    const int64_t S = (int64_t)a.W * a.k, N = (int64_t)a.count * S;
    const unsigned long long *fillp = reinterpret_cast<const unsigned long long *>(a.rec);
    for (InstIter it(blockIdx.x * (int64_t)blockDim.x + threadIdx.x, S, (int64_t)gridDim.x * blockDim.x); it.t < N;
         it.next()) {
        const int64_t t = it.t, inst = it.inst;
        if (a.solve_status[inst] != 0 || it.i >= a.path_count[inst]) continue;
        const int64_t s0 = a.soff[t];
        const int n1 = (int)((int64_t)fillp[t] - s0), cap1 = a.outdeg[t], n2 = a.mfr[t];
        a.indeg[t] -= a.newly[t];  // (rule-2 in-edges the walk dropped; zero for the warp-per-path walk)
        if (n1 < cap1)  // (ascending: a destination never overlaps a later source)
            for (int r = 0; r < n2; ++r) a.succ[s0 + n1 + r] = a.succ[s0 + cap1 + r];
        a.outdeg[t] = n1 + n2;
    }
}

// per-path records for the batching kernels: {xs | ys << 16, xt | yt << 16,
// move base, successor offset} relative to the instance (coordinates already
// split, so no division by H on the release path); entry P closes the last
// path's ranges
__global__ void prec_kernel(PipelineArgs a) {
    const int64_t S = (int64_t)a.W * a.k, S1 = S + 1;
    for (InstIter it(blockIdx.x * (int64_t)blockDim.x + threadIdx.x, S1, (int64_t)gridDim.x * blockDim.x);
         it.t < (int64_t)a.count * S1; it.next()) {
        const int64_t t = it.t, inst = it.inst;
        const int p = it.i;
        const int P = a.solve_status[inst] != 0 ? 0 : a.path_count[inst];
        if (p > P) continue;
        const int64_t o = inst * S;
        const int64_t e0 = a.soff[o], m0 = a.mbase[o];
        int ps = 0, pd = 0;
        if (p < P) {
            const int s = a.path_src[o + p], d = a.path_dst[o + p];
            const int xs = s / a.H, xd = d / a.H;
            ps = xs | ((s - xs * a.H) << 16);
            pd = xd | ((d - xd * a.H) << 16);
        }
        a.prec[t] = make_int4(ps, pd, (int)(a.mbase[o + p] - m0), (int)(a.soff[o + p] - e0));
    }
}

__global__ void sum2_widen_kernel(int64_t n, const int32_t *a, const int32_t *b, int64_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)a[i] + b[i];
}

// ---- small instances: the occupancy DAG per instance in one CTA, with the
// source / target maps and the degree counters in shared memory (the global
// variant above walks every path twice through L2-missing maps and atomics).
// PASS 0 counts degrees (indeg, outdeg to global) and the instance's edge and
// move totals; PASS 1 lays out soff / mbase from the instance bases and fills
// the successor lists.

__host__ __device__ inline int64_t al16(int64_t x) { return (x + 15) / 16 * 16; }

int64_t pipeline_small_dag_smem(int W, int H, int k) {
    const int64_t WH = (int64_t)W * H, S = (int64_t)W * k;
    if (S >= 32768) return 0;  // int16 maps
    const int64_t bytes = al16(WH * 2 * 2) + (2 * S + 2) * 4 + 64;
    return bytes <= 160 * 1024 ? bytes : 0;
}

// exclusive scan of v over the CTA (256 threads) in chunk order; returns the
// chunk total through *tot (all threads)
__device__ __forceinline__ int cta_excl_scan256(int v, int *wsum, int *tot) {
    const int lane = lane_id(), warp = warp_id();
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        before += w < warp ? wsum[w] : 0;
        all += wsum[w];
    }
    __syncthreads();
    *tot = all;
    return before + incl - v;
}

template <int PASS>
__global__ void __launch_bounds__(256) pl_dag_small_kernel(PipelineArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ int wsum[8];
    const int W = a.W, H = a.H, WH = W * H, S = W * a.k;
    int16_t *so = (int16_t *)dsm, *to = so + WH;
    int *deg0 = (int *)(dsm + al16((int64_t)WH * 4)), *deg1 = deg0 + S + 1;
    for (int inst = blockIdx.x; inst < a.count; inst += gridDim.x) {
        const int64_t o = (int64_t)inst * S;
        const int P = a.solve_status[inst] != 0 ? 0 : a.path_count[inst];
        const int32_t *src = a.path_src + o, *dst = a.path_dst + o;
        for (int v = threadIdx.x; v < WH; v += blockDim.x) so[v] = to[v] = -1;
        for (int p = threadIdx.x; p <= S; p += blockDim.x) deg0[p] = deg1[p] = 0;
        __syncthreads();
        for (int p = threadIdx.x; p < P; p += blockDim.x) {
            so[src[p]] = (int16_t)p;
            to[dst[p]] = (int16_t)p;
        }
        if (PASS == 1) {
            // local CSR offsets (deg0) from the out-degrees of pass 0
            int run = 0;
            for (int p0 = 0; p0 < P; p0 += blockDim.x) {
                const int p = p0 + threadIdx.x;
                int tot;
                const int ex = cta_excl_scan256(p < P ? a.outdeg[o + p] : 0, wsum, &tot);
                if (p < P) deg0[p] = run + ex;
                run += tot;
            }
        }
        __syncthreads();
        const int64_t eb = PASS == 1 ? a.ebase[inst] : 0;
        int moves = 0;
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
            const int32_t s = src[i], tt = dst[i];
            const int xs = s / H, ys = s % H, xt = tt / H, yt = tt % H;
            moves += abs(xt - xs) + abs(yt - ys);
            const int dx = xt > xs ? 1 : -1, dy = yt > ys ? 1 : -1;
            int x = xs, y = ys;
            for (;;) {
                const int v = x * H + y;
                const int pa = so[v];
                if (pa >= 0 && pa != i) {  // (pa, i)
                    if (PASS == 0) {
                        atomicAdd(&deg0[pa], 1);
                        atomicAdd(&deg1[i], 1);
                    } else {
                        a.succ[eb + deg0[pa] + atomicAdd(&deg1[pa], 1)] = i;
                    }
                }
                const int pb = to[v];
                if (pb >= 0 && pb != i && !on_path2(H, src[pb], dst[pb], s)) {  // (i, pb)
                    if (PASS == 0) {
                        atomicAdd(&deg0[i], 1);
                        atomicAdd(&deg1[pb], 1);
                    } else {
                        a.succ[eb + deg0[i] + atomicAdd(&deg1[i], 1)] = pb;
                    }
                }
                if (x != xt) x += dx;
                else if (y != yt) y += dy;
                else break;
            }
        }
        __syncthreads();
        if (PASS == 0) {
            int edges = 0;
            for (int p = threadIdx.x; p < P; p += blockDim.x) {
                a.outdeg[o + p] = deg0[p];
                a.indeg[o + p] = deg1[p];
                edges += deg0[p];
            }
            edges = warp_sum(edges);
            moves = warp_sum(moves);
            if (lane_id() == 0) wsum[warp_id()] = edges;
            __syncthreads();
            if (threadIdx.x == 0) {
                int e = 0;
                for (int w = 0; w < 8; ++w) e += wsum[w];
                a.inst_edges[inst] = e;
            }
            __syncthreads();
            if (lane_id() == 0) wsum[warp_id()] = moves;
            __syncthreads();
            if (threadIdx.x == 0) {
                int m = 0;
                for (int w = 0; w < 8; ++w) m += wsum[w];
                a.inst_moves[inst] = m;
            }
        } else {
            // soff / mbase: instance base + local prefix, for p in [0, P]
            // (p = P is the instance's end, which the batching reads)
            const int64_t mb = a.mvbase[inst];
            int run = 0;
            for (int p0 = 0; p0 <= P; p0 += blockDim.x) {
                const int p = p0 + threadIdx.x;
                int len = 0;
                if (p < P) {
                    const int32_t s = src[p], tt = dst[p];
                    len = abs(tt / H - s / H) + abs(tt % H - s % H);
                }
                int tot;
                const int ex = cta_excl_scan256(len, wsum, &tot);
                if (p <= P) {
                    a.soff[o + p] = eb + (p < P ? deg0[p] : a.inst_edges[inst]);
                    a.mbase[o + p] = mb + run + ex;
                }
                run += tot;
            }
        }
        __syncthreads();
    }
}

__global__ void widen32_kernel(int64_t n, const int32_t *in, int64_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

size_t pipeline_temp_bytes(int64_t n) {
    size_t t = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t, (int64_t *)nullptr, (int64_t *)nullptr, (int)n);
    return t;
}

cudaError_t pipeline_dag_count(const PipelineArgs &a, cudaStream_t st, int64_t *counts_host, int64_t *launches) {
    const int64_t S = (int64_t)a.W * a.k, WH = (int64_t)a.W * a.H, N = (int64_t)a.count * S;
    if (a.small_dag) {
        const int64_t smem = pipeline_small_dag_smem(a.W, a.H, a.k);
        cudaFuncSetAttribute(pl_dag_small_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(pl_dag_small_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int grid = (int)std::min<int64_t>(a.count, 148 * 16);
        pl_dag_small_kernel<0><<<grid, 256, smem, st>>>(a);
        *launches += 3;  // + two scans
        cudaMemsetAsync(a.inst_edges + a.count, 0, 8, st);
        cudaMemsetAsync(a.inst_moves + a.count, 0, 8, st);
        size_t tb = a.temp_bytes;
        cub::DeviceScan::ExclusiveSum(a.temp, tb, a.inst_edges, a.ebase, a.count + 1, st);
        tb = a.temp_bytes;
        cub::DeviceScan::ExclusiveSum(a.temp, tb, a.inst_moves, a.mvbase, a.count + 1, st);
        cudaError_t e = cudaMemcpyAsync(counts_host, a.ebase + a.count, 8, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return e;
        e = cudaMemcpyAsync(counts_host + 1, a.mvbase + a.count, 8, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return e;
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return e;
        return cudaGetLastError();
    }
    // maps: {source owner, target owner} per vertex, column-major then row-major;
    // coverage difference arrays after them; target bitmaps in occ / inb
    // (rewritten by pipeline_run_batching before the batching reads them)
    int32_t *mc = a.source_of, *mr = a.source_of + (size_t)a.count * WH * 4;
    const CoverArrays cv = pipeline_cover_arrays(a);
    cudaMemsetAsync(mc, 0xff, (size_t)a.count * WH * 32, st);
    cudaMemsetAsync(cv.rowc, 0, (size_t)a.count * ((size_t)a.H * (a.W + 1) + (size_t)a.W * (a.H + 1)) * 4, st);
    cudaMemsetAsync(cv.rowT, 0, (size_t)a.count * ((WH + 31) / 32) * 4, st);
    cudaMemsetAsync(cv.colT, 0, (size_t)a.count * ((WH + 31) / 32) * 4, st);
    const int blocks = 148 * 8;
    pl_mark2_kernel<<<blocks, 256, 0, st>>>(a, mc, mr, cv);
    cover_scan_kernel<<<blocks, 256, 0, st>>>(a.count, a.W, a.H, cv);
    pl_degree_kernel<<<blocks, 256, 0, st>>>(a, cv);
    *launches += 7;  // mark, cover scan, degrees, widen, two scans, fill pointers
    // soff = exclusive scan of the list capacities (rule 1 + rule 2); mbase = exclusive scan of lengths
    sum2_widen_kernel<<<blocks, 256, 0, st>>>(N, a.outdeg, a.mfr, a.soff);
    cudaMemsetAsync(a.soff + N, 0, 8, st);
    size_t tb = a.temp_bytes;
    cub::DeviceScan::ExclusiveSum(a.temp, tb, a.soff, a.soff, (int)(N + 1), st);
    cudaMemsetAsync(a.mbase + N, 0, 8, st);
    tb = a.temp_bytes;
    cub::DeviceScan::ExclusiveSum(a.temp, tb, a.mbase, a.mbase, (int)(N + 1), st);
    fillptr_kernel<<<blocks, 256, 0, st>>>(N, a.soff, reinterpret_cast<unsigned long long *>(a.rec));
    cudaError_t e = cudaMemcpyAsync(counts_host, a.soff + N, 8, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(counts_host + 1, a.mbase + N, 8, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// --------------------------------------------------------------------------
// pipeline batching with the ready list as records
// --------------------------------------------------------------------------
// A ready path is a record {p (-1 once finished), k | len << 16,
// xs | ys << 16, xt | yt << 16} plus its move base in a parallel array, kept
// in ascending p.  A batch reads its candidates with coalesced loads and
// advances them in place; only newly released paths touch the per-path
// arrays (src, dst, mbase).  Acceptance: the paths are solver output (every
// source occupied, distinct tokens), so the only possible vertex conflict
// inside a batch is a shared destination and the minimum id wins (under
// column_direction, the class of the batch's first move); application and
// release as in batch_warp.  With <= 32 ready paths, lane i keeps path i in
// registers (register-resident frontier).

__device__ __forceinline__ int4 make_rec(const ImplicitPaths &ip, int p, int *base) {
    const int s = ip.src[p], t = ip.dst[p];
    const int xs = s / ip.H, ys = s - xs * ip.H, xt = t / ip.H, yt = t - xt * ip.H;
    const int len = abs(xt - xs) + abs(yt - ys);
    *base = (int)ip.move_base(p);
    return make_int4(p, len << 16, xs | (ys << 16), xt | (yt << 16));
}

__device__ __forceinline__ LanePath rec_lane(int4 r, int base) {
    LanePath l;
    l.p = r.x;
    l.k = r.y & 0xffff;
    l.len = r.y >> 16;
    l.xs = r.z & 0xffff;
    l.ys = r.z >> 16;
    l.xt = r.w & 0xffff;
    l.yt = r.w >> 16;
    l.base = base;
    l.pf = 1;
    l.pn = 1;
    return l;
}

__device__ __forceinline__ int4 lane_rec(const LanePath &l) {
    return make_int4(l.p, l.k | (l.len << 16), l.xs | (l.ys << 16), l.xt | (l.yt << 16));
}

// #records with p < x in a p-ascending record array
__device__ __forceinline__ int lower_bound_rec(const int4 *a, int n, int x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (a[m].x < x) lo = m + 1;
        else hi = m;
    }
    return lo;
}

// per-path blocker counts: global int32, or (BSM) u16 halves of u32 words in
// shared memory, decremented with a 32-bit atomic add of -(1 << 16*half) (a
// count is >= 1 before each decrement, so no borrow crosses halves)
template <bool BSM>
struct Blockers {
    int32_t *g;
    uint32_t sa;
    __device__ Blockers(int32_t *gp, uint32_t *sp) : g(gp), sa(BSM ? (uint32_t)__cvta_generic_to_shared(sp) : 0u) {}
    __device__ __forceinline__ int get(int p) const {
        if (!BSM) return g[p];
        uint32_t x;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(sa + ((uint32_t)(p >> 1) << 2)));
        return (int)((x >> ((p & 1) * 16)) & 0xffffu);
    }
    // one predecessor of p finished; true when it was the last
    // the count before a decrement (compare with 1 later: the atomic's round
    // trip then overlaps other work)
    __device__ __forceinline__ int release_raw(int p) const {
        if (!BSM) return atomicSub(&g[p], 1);
        const uint32_t sh = (uint32_t)(p & 1) * 16u;
        uint32_t old;
        asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                     : "=r"(old)
                     : "r"(sa + ((uint32_t)(p >> 1) << 2)), "r"(0u - (1u << sh))
                     : "memory");
        return (int)((old >> sh) & 0xffffu);
    }
    // release_raw when `pred`, else 0: global counts issue back to back
    // (atom_add_if), so a run of these costs one round trip
    __device__ __forceinline__ int release_raw_if(bool pred, int p) const {
        if (!BSM) return (int)atom_add_if(pred, reinterpret_cast<uint32_t *>(g + max(p, 0)), 0xffffffffu);
        return pred ? release_raw(p) : 0;
    }
    __device__ __forceinline__ bool release(int p) const {
        if (!BSM) return atomicSub(&g[p], 1) == 1;
        const uint32_t sh = (uint32_t)(p & 1) * 16u;
        uint32_t old;
        asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                     : "=r"(old)
                     : "r"(sa + ((uint32_t)(p >> 1) << 2)), "r"(0u - (1u << sh))
                     : "memory");
        return ((old >> sh) & 0xffffu) == 1u;
    }
};

// successors of the finished paths (fin lanes, CSR range [q0, q1)) lose one
// blocker; the released ones are appended to newly; returns the new count
template <class BL>
__device__ __forceinline__ int release_successors(const BatchJob &J, const BL &blockers, int32_t *newly, int nnew,
                                                  bool fin, int64_t q0, int64_t q1) {
    const int lane = lane_id();
    if (!fin) q0 = q1 = 0;
    int tot;
    const int base = warp_excl_scan((int)(q1 - q0), &tot);
    for (int t0 = 0; t0 < tot; t0 += 32) {
        const int t = t0 + lane;
        int owner = 0;  // largest lane with base <= t
#pragma unroll
        for (int st = 16; st > 0; st >>= 1) {
            const int cl = owner + st;
            if (__shfl_sync(FULL, base, cl) <= t) owner = cl;
        }
        const int64_t oq0 = __shfl_sync(FULL, q0, owner);
        const int ob = __shfl_sync(FULL, base, owner);
        bool released = false;
        int sc = -1;
        if (t < tot) {
            sc = J.succ[oq0 + (t - ob)];
            released = sc >= 0 && blockers.release(sc);  // (-1: a hole of the list)
        }
        const unsigned rm = __ballot_sync(FULL, released);
        if (released) newly[nnew + __popc(rm & lanemask_lt())] = sc;
        nnew += __popc(rm);
    }
    return nnew;
}

// sorts newly[0, n) ascending in place (mem: scratch of n)
__device__ __forceinline__ void sort_newly(int32_t *newly, int32_t *mem, int n) {
    const int lane = lane_id();
    if (n <= 32) {
        int v = lane < n ? newly[lane] : INT_MAX;
        v = warp_sort32(v);
        if (lane < n) newly[lane] = v;
    } else {
        for (int q = lane; q < n; q += 32) {
            const int x = newly[q];
            int lt = 0;
            for (int r2 = 0; r2 < n; ++r2) lt += newly[r2] < x;
            mem[lt] = x;
        }
        __syncwarp();
        for (int q = lane; q < n; q += 32) newly[q] = mem[q];
    }
    __syncwarp();
}

// ready = (kept records rec2[0, nkeep)) U (records of newly[0, nnew)), by rank
// (kr: scratch of >= 32 ints.)  With <= 32 newly released paths, their ids
// stay in registers: a kept record's rank among them is a shuffle binary
// search, and the kept ranks place each newly released record, so neither
// side searches global memory.
__device__ __forceinline__ void merge_ready(const ImplicitPaths &paths, const PipeRecords &R, const int32_t *newly,
                                            int nkeep, int nnew, int32_t *kr) {
    const int lane = lane_id();
    if (nnew <= 32) {
        const int ny = lane < nnew ? newly[lane] : INT_MAX;  // ascending, INT_MAX padded
        if (lane < nnew) kr[lane] = nkeep;  // #kept below newly j (default: all)
        __syncwarp();
        const int ny31 = __shfl_sync(FULL, ny, 31);
        int prev_r = 0;
        for (int i0 = 0; i0 < nkeep; i0 += 32) {
            const int i = i0 + lane;
            int4 x = make_int4(INT_MAX, 0, 0, 0);
            int xb = 0;
            if (i < nkeep) {
                x = R.rec2[i];
                xb = R.rb2[i];
            }
            int r = 0;  // #newly < x.x
#pragma unroll
            for (int st = 16; st; st >>= 1)
                if (__shfl_sync(FULL, ny, r + st - 1) < x.x) r += st;
            if (r == 31 && ny31 < x.x) r = 32;
            int rp = __shfl_up_sync(FULL, r, 1);
            if (lane == 0) rp = prev_r;
            if (i < nkeep) {
                R.rec[i + r] = x;
                R.rb[i + r] = xb;
                for (int j = rp; j < r; ++j) kr[j] = i;  // newly j sits right before kept i
            }
            prev_r = __shfl_sync(FULL, r, 31);
        }
        __syncwarp();
        if (lane < nnew) {
            int b;
            const int4 rr = make_rec(paths, ny, &b);
            const int at = lane + kr[lane];
            R.rec[at] = rr;
            R.rb[at] = b;
        }
        __syncwarp();
        return;
    }
    for (int i = lane; i < nkeep; i += 32) {
        const int4 x = R.rec2[i];
        const int at = i + lower_bound_i32(newly, nnew, x.x);
        R.rec[at] = x;
        R.rb[at] = R.rb2[i];
    }
    for (int j = lane; j < nnew; j += 32) {
        const int y = newly[j];
        int b;
        const int4 r = make_rec(paths, y, &b);
        const int at = j + lower_bound_rec(R.rec2, nkeep, y);
        R.rec[at] = r;
        R.rb[at] = b;
    }
    __syncwarp();
}

// a lane path moved between lanes (q0/q1 only in leap mode)
__device__ __forceinline__ LanePath shfl_lane(const LanePath &lp, int src, bool with_succ) {
    LanePath q;
    q.p = __shfl_sync(FULL, lp.p, src);
    q.k = __shfl_sync(FULL, lp.k, src);
    q.len = __shfl_sync(FULL, lp.len, src);
    q.xs = __shfl_sync(FULL, lp.xs, src);
    q.ys = __shfl_sync(FULL, lp.ys, src);
    q.xt = __shfl_sync(FULL, lp.xt, src);
    q.yt = __shfl_sync(FULL, lp.yt, src);
    q.base = __shfl_sync(FULL, lp.base, src);
    if (with_succ) {
        q.q0 = __shfl_sync(FULL, lp.q0, src);
        q.q1 = __shfl_sync(FULL, lp.q1, src);
        q.pf = __shfl_sync(FULL, lp.pf, src);
    } else {
        q.q0 = q.q1 = 0;
        q.pf = 0;
    }
    q.pn = 1;
    return q;
}

// release_successors for leap mode: every successor id of the chunk group is
// loaded first, then every blocker decremented, so a finish costs two
// dependent round trips instead of two per 32 successors.  Released ids go to
// the warp's shared buffer (cap entries) when every successor fits, else to
// the global one; *out = the buffer used.
template <class BL>
__device__ __forceinline__ int release_successors_buf(const BatchJob &J, const BL &blockers, int32_t *sm, int cap,
                                                      int32_t *g, bool fin, int64_t q0, int64_t q1, int32_t **out) {
    constexpr int G = 8;  // chunks of 32 successors in flight
    const int lane = lane_id();
    if (!fin) q0 = q1 = 0;
    int tot;
    const int base = warp_excl_scan((int)(q1 - q0), &tot);
    int32_t *buf = tot <= cap ? sm : g;
    *out = buf;
    int nnew = 0;
    for (int g0 = 0; g0 < tot; g0 += 32 * G) {
        int sc[G];
#pragma unroll
        for (int c = 0; c < G; ++c) {
            const int t = g0 + c * 32 + lane;
            int owner = 0;  // largest lane with base <= t
#pragma unroll
            for (int st = 16; st > 0; st >>= 1) {
                const int cl = owner + st;
                if (__shfl_sync(FULL, base, cl) <= t) owner = cl;
            }
            const int64_t oq0 = __shfl_sync(FULL, q0, owner);
            const int ob = __shfl_sync(FULL, base, owner);
            sc[c] = t < tot ? __ldg(J.succ + oq0 + (t - ob)) : -1;
        }
        int old[G];
#pragma unroll
        for (int c = 0; c < G; ++c) old[c] = blockers.release_raw_if(sc[c] >= 0, sc[c]);
        bool rel[G];
#pragma unroll
        for (int c = 0; c < G; ++c) rel[c] = sc[c] >= 0 && old[c] == 1;
#pragma unroll
        for (int c = 0; c < G; ++c) {
            const unsigned rm = __ballot_sync(FULL, rel[c]);
            if (rel[c]) buf[nnew + __popc(rm & lanemask_lt())] = sc[c];
            nnew += __popc(rm);
        }
    }
    return nnew;
}

// phase cycle counters of batch_warp_pipe (experiments: -DRECON_BATCH_PROF)
__device__ unsigned long long g_batch_prof[16];

// Leap-mode finish: the finished lanes' successors are released as in
// release_successors_buf, and every successor's path record
// {source, target coordinates, move base, successor offset} (prec) is loaded
// together with its blocker decrement, so a released path needs no further
// round trip: it goes straight into an empty lane (lanes are not kept in id
// order in leap mode).  Released ids also go to `buf` for the rare spill.
// Returns the number released; *filled = whether every one got a lane.
template <class BL>
__device__ __forceinline__ int release_into_lanes(const BatchJob &J, const BL &blockers, int32_t *sm, int cap,
                                                  int32_t *g, bool fin, int64_t q0, int64_t q1, int32_t **out,
                                                  LanePath &lp, bool *filled) {
    constexpr int G = 8;  // chunks of 32 successors in flight
    const int lane = lane_id();
    const unsigned fmask = __ballot_sync(FULL, fin);
    const int tot = __reduce_add_sync(FULL, fin ? (unsigned)(q1 - q0) : 0u);
    int32_t *buf = tot <= cap ? sm : g;
    *out = buf;
    const unsigned empty = __ballot_sync(FULL, lp.p == INT_MAX);
    const int erank = __popc(empty & lanemask_lt());  // my rank among the empty lanes
    const int nempty = __popc(empty);
    const bool is_empty = (empty >> lane) & 1u;
    bool took = false;
    int nnew = 0;
    int sc[G];
    int nsl = 0;  // chunks loaded (warp-uniform)
    // decrement, prefetch and hand out the loaded chunks
    auto flush = [&]() {
        int4 pr[G];
        int qe[G];
        bool rel[G];
        int old[G];
#pragma unroll
        for (int c = 0; c < G; ++c) {
            const bool ok = c < nsl && sc[c] >= 0;
            pr[c] = make_int4(0, 0, 0, 0);
            qe[c] = 0;
            if (ok) {
                pr[c] = __ldg(J.prec + sc[c]);
                qe[c] = J.slen ? __ldg(J.slen + sc[c]) : __ldg(&J.prec[sc[c] + 1].w);
            }
            old[c] = blockers.release_raw_if(ok, sc[c]);
        }
#pragma unroll
        for (int c = 0; c < G; ++c) rel[c] = c < nsl && sc[c] >= 0 && old[c] == 1;
#pragma unroll
        for (int c = 0; c < G; ++c) {
            if (c >= nsl) break;
            const unsigned rm = __ballot_sync(FULL, rel[c]);
            if (!rm) continue;
            RB_CHECK(buf != sm || nnew + __popc(rm) <= cap, "released ids overflow the shared buffer");
            if (rel[c]) buf[nnew + __popc(rm & lanemask_lt())] = sc[c];
            // the empty lane of rank e takes released item e - nnew of this chunk
            const int j = erank - nnew;
            const bool take = is_empty && j >= 0 && j < __popc(rm);
            const int srcl = take ? (int)__fns(rm, 0, j + 1) : lane;
            const int np = __shfl_sync(FULL, sc[c], srcl);
            const int4 r = make_int4(__shfl_sync(FULL, pr[c].x, srcl), __shfl_sync(FULL, pr[c].y, srcl),
                                     __shfl_sync(FULL, pr[c].z, srcl), __shfl_sync(FULL, pr[c].w, srcl));
            const int e = __shfl_sync(FULL, qe[c], srcl);
            if (take) {
                took = true;
                lp.p = np;
                lp.k = 0;
                lp.xs = r.x & 0xffff;
                lp.ys = r.x >> 16;
                lp.xt = r.y & 0xffff;
                lp.yt = r.y >> 16;
                lp.len = abs(lp.xt - lp.xs) + abs(lp.yt - lp.ys);
                lp.base = r.z;
                lp.q0 = J.e0 + r.w;
                lp.q1 = J.e0 + (J.slen ? r.w + e : e);
                lp.pf = 1;
                lp.pn = 1;
            }
            nnew += __popc(rm);
        }
        nsl = 0;
    };
#ifdef RECON_BATCH_PROF
    const long long rt0 = clock64();
#endif
    // successor ids, finished lane by finished lane, 32 at a time
    for (unsigned m = fmask; m; m &= m - 1) {
        const int f = __ffs(m) - 1;
        const int64_t fq0 = __shfl_sync(FULL, q0, f);
        const int fn = (int)(__shfl_sync(FULL, q1, f) - fq0);
        for (int j0 = 0; j0 < fn; j0 += 32) {
            const int v = j0 + lane < fn ? __ldg(J.succ + fq0 + j0 + lane) : -1;
#pragma unroll
            for (int c = 0; c < G; ++c)
                if (c == nsl) sc[c] = v;
            if (++nsl == G) flush();
        }
    }
#ifdef RECON_BATCH_PROF
    const long long rt1 = clock64();
#endif
    if (nsl) flush();
#ifdef RECON_BATCH_PROF
    if (lane == 0) {
        atomicAdd(&g_batch_prof[10], (unsigned long long)(rt1 - rt0));
        atomicAdd(&g_batch_prof[11], (unsigned long long)(clock64() - rt1));
        atomicAdd(&g_batch_prof[12], 1ull);
    }
#endif
    *filled = nnew <= nempty;
    if (!*filled && took) lp.p = INT_MAX;  // the spill takes every released id from buf
    return nnew;
}


// Leap-mode finish issued early: the lanes that finish with this leap are
// known as soon as `delta` is, so their successor ids are loaded before the
// leap's schedule stores and their blocker decrements and path records are
// issued after them; release_fill then waits for the results.  Up to
// 32 * EG successors (the caller falls back to release_into_lanes beyond).
#ifndef RECON_EG
#define RECON_EG 6
#endif
constexpr int EG = RECON_EG;
struct EarlyRelease {
    int sc[EG];
    int4 pr[EG];
    int qe[EG];
    int old[EG];
};

__device__ __forceinline__ void release_load(const BatchJob &J, bool fin, int64_t q0, int64_t q1, EarlyRelease &er) {
    const int lane = lane_id();
    const unsigned fm = __ballot_sync(FULL, fin);
    if (!(fm & (fm - 1))) {  // one finishing lane (the common case): no owner search
        const int f = __ffs(fm) - 1;
        const int64_t oq0 = __shfl_sync(FULL, q0, f);
        const int n = (int)(__shfl_sync(FULL, q1, f) - oq0);
#pragma unroll
        for (int c = 0; c < EG; ++c) {
            const int t = c * 32 + lane;
            er.sc[c] = t < n ? __ldcg(J.succ + oq0 + t) : -1;
        }
        return;
    }
    if (!fin) q0 = q1 = 0;
    int tot;
    const int base = warp_excl_scan((int)(q1 - q0), &tot);
#pragma unroll
    for (int c = 0; c < EG; ++c) {
        const int t = c * 32 + lane;
        int owner = 0;  // largest lane with base <= t
#pragma unroll
        for (int st = 16; st > 0; st >>= 1) {
            const int cl = owner + st;
            if (__shfl_sync(FULL, base, cl) <= t) owner = cl;
        }
        const int64_t oq0 = __shfl_sync(FULL, q0, owner);
        const int ob = __shfl_sync(FULL, base, owner);
        er.sc[c] = t < tot ? __ldcg(J.succ + oq0 + (t - ob)) : -1;
    }
}

template <class BL>
__device__ __forceinline__ void release_issue(const BatchJob &J, const BL &blockers, EarlyRelease &er) {
#pragma unroll
    for (int c = 0; c < EG; ++c) {
        er.pr[c] = make_int4(0, 0, 0, 0);
        er.qe[c] = 0;
        if (er.sc[c] >= 0) {
            er.pr[c] = __ldcg(J.prec + er.sc[c]);
            er.qe[c] = J.slen ? __ldcg(J.slen + er.sc[c]) : __ldcg(&J.prec[er.sc[c] + 1].w);
        }
        er.old[c] = blockers.release_raw_if(er.sc[c] >= 0, er.sc[c]);
    }
}

// the released paths of an early release into the empty lanes (and `sm`);
// returns the number released, *filled = whether every one got a lane
__device__ __forceinline__ int release_fill(const BatchJob &J, const EarlyRelease &er, int32_t *sm, LanePath &lp,
                                            bool *filled) {
    const int lane = lane_id();
    const unsigned empty = __ballot_sync(FULL, lp.p == INT_MAX);
    const int erank = __popc(empty & lanemask_lt());
    const int nempty = __popc(empty);
    const bool is_empty = (empty >> lane) & 1u;
    bool took = false;
    int nnew = 0;
#pragma unroll
    for (int c = 0; c < EG; ++c) {
        const bool rel = er.sc[c] >= 0 && er.old[c] == 1;
        const unsigned rm = __ballot_sync(FULL, rel);
        if (!rm) continue;
        if (rel) sm[nnew + __popc(rm & lanemask_lt())] = er.sc[c];
        const int j = erank - nnew;
        const bool take = is_empty && j >= 0 && j < __popc(rm);
        const int srcl = take ? (int)__fns(rm, 0, j + 1) : lane;
        const int np = __shfl_sync(FULL, er.sc[c], srcl);
        const int4 r = make_int4(__shfl_sync(FULL, er.pr[c].x, srcl), __shfl_sync(FULL, er.pr[c].y, srcl),
                                 __shfl_sync(FULL, er.pr[c].z, srcl), __shfl_sync(FULL, er.pr[c].w, srcl));
        const int e = __shfl_sync(FULL, er.qe[c], srcl);
        if (take) {
            took = true;
            lp.p = np;
            lp.k = 0;
            lp.xs = r.x & 0xffff;
            lp.ys = r.x >> 16;
            lp.xt = r.y & 0xffff;
            lp.yt = r.y >> 16;
            lp.len = abs(lp.xt - lp.xs) + abs(lp.yt - lp.ys);
            lp.base = r.z;
            lp.q0 = J.e0 + r.w;
            lp.q1 = J.e0 + (J.slen ? r.w + e : e);
            lp.pf = 1;
            lp.pn = 1;
        }
        nnew += __popc(rm);
    }
    *filled = nnew <= nempty;
    if (!*filled && took) lp.p = INT_MAX;  // the spill takes every released id from sm
    return nnew;
}

// occupancy update without ordering: a token moving a -> b toggles both bits
// (red.xor commutes, so a vacated and a refilled vertex need no fence)
template <bool SM>
__device__ __forceinline__ void occ_toggle(const Bits<SM> &b, int v) {
    if (SM) asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(b.sa + ((uint32_t)(v >> 5) << 2)), "r"(1u << (v & 31)) : "memory");
    else asm volatile("red.global.xor.b32 [%0], %1;" ::"l"(b.p + (v >> 5)), "r"(1u << (v & 31)) : "memory");
}

#ifdef RECON_BATCH_PROF
#define BPROF_T0() long long bp_t0_ = clock64()
#define BPROF_ADD(i)                  \
    do {                              \
        const long long t_ = clock64(); \
        bprof[i] += t_ - bp_t0_;      \
        bp_t0_ = t_;                  \
    } while (0)
#define BPROF_CNT(i) (bprof[i] += 1)
#else
#define BPROF_T0() (void)0
#define BPROF_ADD(i) (void)0
#define BPROF_CNT(i) (void)0
#endif

// ---- leap mode (preset none, register frontier): the batches in which
// every ready path moves are skipped in one step.
//
// Between two "events" — a path's final move, or a ready path that is not
// accepted — every ready path advances one vertex per batch, so batch
// nb + t moves every live path's (k + t)-th edge.  An event is found without
// stepping:
//  * path p's final move happens at offset f_p = len_p - k_p - 1;
//  * p is not accepted at offset t iff its destination P(t+1) is occupied
//    pre-batch, or another ready path q wants the same vertex
//    (batching.cpp:111-113).  Occupied means a ready path's current vertex,
//    P(t+1) == Q(t), or a stationary token.  A stationary token can never
//    lie on a ready path's remaining route under the occupancy dag
//    (virtual_line.cpp:241-268): an unstarted path's source on p's route is a
//    dag predecessor of p (so it already left), a finished path's target on
//    p's route is a dag successor of p (so it has not arrived), and a token
//    no path moves cannot lie on any route of a collision-free solution.
// With one-bend routes (horizontal, then vertical; virtual_line.cpp:150-173)
// P(t) and Q(t) are two linear pieces each, so the first meeting time is a
// small integer solve per piece pair.  delta = min over live paths of
// min(f_p + 1, first stall) batches are applied at once; delta == 0 runs the
// literal batch.  Bit-identical to the literal loop (tests/test_batching_gpu.py).
// Deadlocked lanes.  A lane whose next vertex holds another lane's token is
// blocked; the blocked lanes whose blocker is itself blocked, closed under
// that relation, form cycles (head-on riders, batching.cpp:127-128's
// no-progress case) plus the lanes queued behind them.  None of them can ever
// move again, so they are frozen: their tokens act as fixed obstacles and the
// leap runs over the remaining lanes (the movers).  A lane blocked by a mover
// only waits one batch: delta = 0 then.
// Returns delta (0: run the batch literally) and the movers' lane mask.
__device__ __forceinline__ int leap_delta(const LanePath &lp, int H, int32_t fr, int32_t to, unsigned *movers,
                                          int *ppair, int *pwith) {
    *ppair = INT_MAX;
    *pwith = -1;
    const int lane = lane_id();
    const bool valid = lp.p != INT_MAX;
    const unsigned vm = __ballot_sync(FULL, valid);
    int blocker = -1;
    for (unsigned m = vm; m; m &= m - 1) {
        const int q = __ffs(m) - 1;
        if (__shfl_sync(FULL, fr, q) == to) blocker = q;
    }
    bool frozen = valid && blocker >= 0;
    unsigned fm = __ballot_sync(FULL, frozen);
    const unsigned blocked = fm;
    if (fm) {
        for (;;) {  // greatest set closed under "blocked by a member"
            frozen = frozen && ((fm >> blocker) & 1u);
            const unsigned nfm = __ballot_sync(FULL, frozen);
            if (nfm == fm) break;
            fm = nfm;
        }
        if (blocked != fm) {  // someone waits for a mover: one literal batch
            *movers = vm & ~fm;
            return 0;
        }
    }
    const unsigned mv = vm & ~fm;
    *movers = mv;
    if (!mv) return 0;  // only frozen lanes: the literal batch reports no progress
    const bool mover = (mv >> lane) & 1u;
    int best = mover ? lp.len - lp.k : INT_MAX;  // f + 1
    Seg mine[2];
    lane_segs(lp.k, lp.len, lp.xs, lp.ys, lp.xt, lp.yt, mine[0], mine[1]);
    // remaining route's bounding box: no meeting outside both boxes
    const int xc = mine[0].t1 >= 0 ? mine[0].x0 : lp.xt;  // column now
    const int bx0 = min(xc, lp.xt), bx1 = max(xc, lp.xt);
    const int yc = mine[1].y0 + mine[1].vy * mine[1].t0;  // row at the bend (or now)
    const int by0 = min(yc, lp.yt), by1 = max(yc, lp.yt);
    const int pk = lp.k | (lp.len << 16), pxs = lp.xs | (lp.ys << 16), pxt = lp.xt | (lp.yt << 16);
    const int pb0 = bx0 | (by0 << 16), pb1 = bx1 | (by1 << 16);
    const unsigned others = __popc(vm) > 1 ? vm : 0u;
    for (unsigned m = others; m; m &= m - 1) {
        const int q = __ffs(m) - 1;
        const int qk = __shfl_sync(FULL, pk, q), qxs = __shfl_sync(FULL, pxs, q), qxt = __shfl_sync(FULL, pxt, q);
        const int qb0 = __shfl_sync(FULL, pb0, q), qb1 = __shfl_sync(FULL, pb1, q);
        const int qfr = __shfl_sync(FULL, fr, q);
        const bool qfrozen = (fm >> q) & 1u;
        if (!mover || q == lane) continue;
        if (qfrozen) {
            // a frozen token is a fixed obstacle: the first t with P(t+1) on it
            const int qx = qfr / H, qy = qfr - qx * H;
            if (qx >= bx0 && qx <= bx1 && qy >= by0 && qy <= by1) {
                const Seg pt[2] = {Seg{qx, qy, 0, 0, 0, INT_MAX / 2}, Seg{qx, qy, 0, 0, 0, INT_MAX / 2}};
                best = min(best, pair_event(mine, pt, 0, lp.len - lp.k - 1));
            }
            continue;
        }
        const bool overlap = (qb0 & 0xffff) <= bx1 && (qb1 & 0xffff) >= bx0 && (qb0 >> 16) <= by1 && (qb1 >> 16) >= by0;
        if (overlap) {
            const int k = qk & 0xffff, len = qk >> 16;
            Seg other[2];
            lane_segs(k, len, qxs & 0xffff, qxs >> 16, qxt & 0xffff, qxt >> 16, other[0], other[1]);
            const int e = pair_event(mine, other, 0, min(lp.len - lp.k - 1, len - k - 1));
            if (e < *ppair) {
                *ppair = e;
                *pwith = q;
            }
            best = min(best, e);
        }
    }
    return __reduce_min_sync(FULL, mover ? best : INT_MAX);
}

template <bool SM, bool SMI, bool LOG, bool BSM, bool LEAP = false>
__device__ void batch_warp_pipe(const BatchJob &J, const ImplicitPaths &paths, PipeRecords R, const int64_t *wst) {
    const int lane = lane_id();
    const int P = J.P, H = J.H;
    BatchScratch s = J.s;
    const Bits<SM> occ(s.occ);
    const Bits<SMI> inb(s.inb);
    const Blockers<BSM> blk(s.blockers, s.blk_sm);  // BSM: filled by the caller
    // the wide phase (batch_wide.cu) ran the first batches: continue from its
    // ready records, bitmap, blocker counts and counters
    const bool resumed = wst && wst[0] == 1;
    long long left = 0;
    int nready = 0;
    int nb = 0, nlog = 0, status = RECON_OK;
    if (resumed) {
        nb = (int)wst[1];
        left = wst[2];
        nready = (int)wst[3];
    }
    // ---- init: blockers = in-degree (given); zero-length paths finish at once
    for (int p = lane; p < P && !resumed; p += 32) {
        const int len = paths.len(p);
        left += len;
        if (len == 0)
            for (int64_t q = J.soff[p]; q < list_end(J, p); ++q)
                if (J.succ[q] >= 0) blk.release(J.succ[q]);  // (-1: a hole of the list)
    }
    if (!resumed) left = warp_sum64(left);
    __syncwarp();
    __threadfence_block();
    for (int p0 = 0; p0 < P && !resumed; p0 += 32) {
        const int p = p0 + lane;
        const bool r = p < P && blk.get(p) == 0 && paths.len(p) > 0;
        const unsigned m = __ballot_sync(FULL, r);
        if (r) {
            int b;
            const int4 rc = make_rec(paths, p, &b);
            const int at = nready + __popc(m & lanemask_lt());
            R.rec[at] = rc;
            R.rb[at] = b;
        }
        nready += __popc(m);
    }
    __syncwarp();
#ifdef RECON_BATCH_PROF
    long long bprof[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    const long long bp_start = clock64();
#endif
    // register-resident frontier (<= 32 ready paths), as in batch_warp
    bool regmode = false;
    LanePath lp;
    lp.p = INT_MAX;
    lp.pf = 0;
    lp.pn = 0;
    // leap mode: each lane's earliest meeting with another lane (batches from
    // now, or INT_MAX) and that lane, kept across leaps while no lane is
    // frozen and no literal batch runs: every lane then moves each batch, so a
    // meeting only shifts by the leap; lanes that enter add their pairs, a
    // lane whose partner left holds a lower bound (pst) until it binds
    int pm = INT_MAX, pw = -1;
    bool pst = false, pv_ok = false;
    // the lane's current move (fr -> to), advanced incrementally on acceptance
    int32_t fr = -1, to = -1;
    auto lane_move = [&]() {
        if (lp.p != INT_MAX) {
            fr = lp.v(H, lp.k);
            to = lp.v(H, lp.k + 1);
        }
    };
    auto enter_regmode = [&]() {
        lp.p = INT_MAX;
        if (lane < nready) {
            lp = rec_lane(R.rec[lane], R.rb[lane]);
            if (LEAP) {
                lp.q0 = J.soff[lp.p];
                lp.q1 = list_end(J, lp.p);
            }
        }
        lane_move();
        regmode = true;
        pv_ok = false;
    };
    auto put_move = [&](int64_t slot, int rank_in_batch) {
        if (LOG) J.mlog[nlog + rank_in_batch] = make_int2((int)slot, nb);
        else J.move_batch[slot] = nb;
    };
    if (nready <= 32) enter_regmode();
    while (left > 0) {
        if (regmode) {
            bool fin = false;
            int64_t q0 = 0, q1 = 0;
            bool early = false;  // (uniform) the finish was issued with the leap
            EarlyRelease er;
            BPROF_T0();
            unsigned movers = 0;
            // a lane that entered since the last leap: its successor ids now,
            // and after leap_delta their path records and blocker counts
            // into L2, so its finish (>= one leap away) decrements in L2
            int pfv0 = -1, pfv1 = -1, pff = -1, pfn = 0;  // (pff: the lane, pfn: its successor count)
            if (LEAP) {
                const unsigned pfm = __ballot_sync(FULL, lp.p != INT_MAX && lp.pf);
                if (pfm) {
                    pff = __ffs(pfm) - 1;
                    const int64_t fq = __shfl_sync(FULL, lp.q0, pff);
                    pfn = (int)(__shfl_sync(FULL, lp.q1, pff) - fq);
                    pfv0 = lane < pfn ? __ldcg(J.succ + fq + lane) : -1;
                    pfv1 = 32 + lane < pfn ? __ldcg(J.succ + fq + 32 + lane) : -1;
                    if (lane == pff) lp.pf = 0;
                }
            }
            int delta = 0;
            bool fast = false;
            if (LEAP && pv_ok) {
                const bool valid_l = lp.p != INT_MAX;
                Seg mine[2];
                lane_segs(lp.k, lp.len, lp.xs, lp.ys, lp.xt, lp.yt, mine[0], mine[1]);
                for (unsigned nm = __ballot_sync(FULL, valid_l && lp.pn); nm; nm &= nm - 1) {
                    // an entered lane n: the pairs (i, n) and (n, i)
                    const int n = __ffs(nm) - 1;
                    const int nk = __shfl_sync(FULL, lp.k, n), nlen = __shfl_sync(FULL, lp.len, n);
                    const int nxs = __shfl_sync(FULL, lp.xs, n), nys = __shfl_sync(FULL, lp.ys, n);
                    const int nxt = __shfl_sync(FULL, lp.xt, n), nyt = __shfl_sync(FULL, lp.yt, n);
                    Seg sn[2];
                    lane_segs(nk, nlen, nxs, nys, nxt, nyt, sn[0], sn[1]);
                    // remaining routes' bounding boxes: no meeting outside both
                    const int nxc = sn[0].t1 >= 0 ? sn[0].x0 : nxt, nyc = sn[1].y0 + sn[1].vy * sn[1].t0;
                    const int mxc = mine[0].t1 >= 0 ? mine[0].x0 : lp.xt, myc = mine[1].y0 + mine[1].vy * mine[1].t0;
                    const bool olap = max(min(nxc, nxt), min(mxc, lp.xt)) <= min(max(nxc, nxt), max(mxc, lp.xt)) &&
                                      max(min(nyc, nyt), min(myc, lp.yt)) <= min(max(nyc, nyt), max(myc, lp.yt));
                    int en = INT_MAX;
                    if (valid_l && lane != n && olap) {
                        const int T = min(lp.len - lp.k - 1, nlen - nk - 1);
                        const int e = pair_event(mine, sn, 0, T);
                        if (e < pm) {
                            pm = e;
                            pw = n;
                        }
                        en = pair_event(sn, mine, 0, T);
                    }
                    const int m = (int)__reduce_min_sync(FULL, (unsigned)en);
                    const unsigned wm = __ballot_sync(FULL, en == m && m != INT_MAX);
                    if (lane == n) {
                        pm = m;
                        pw = wm ? __ffs(wm) - 1 : -1;
                        pst = false;
                        lp.pn = 0;
                    }
                }
                const int cand = valid_l ? min(lp.len - lp.k, pm) : INT_MAX;
                const int d0 = (int)__reduce_min_sync(FULL, (unsigned)cand);
                if (d0 > 0 && d0 != INT_MAX && !__any_sync(FULL, valid_l && pst && pm <= d0)) {
                    delta = d0;
                    movers = __ballot_sync(FULL, valid_l);
                    fast = true;
                }
            }
            if (LEAP && !fast) {
#ifdef RECON_BATCH_PROF
                if (lane == 0) atomicAdd(&g_batch_prof[15], 1ull);
#endif
                int pp, pwi;
                delta = leap_delta(lp, H, fr, to, &movers, &pp, &pwi);
                const unsigned vmask = __ballot_sync(FULL, lp.p != INT_MAX);
                pv_ok = delta > 0 && movers == vmask;  // (no frozen lane)
                pm = pp;
                pw = pwi;
                pst = false;
                lp.pn = 0;
            }
            if (LEAP) {
                auto pf1 = [&](int v) {
                    if (v < 0) return;
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(J.prec + v));
                    if (J.slen) asm volatile("prefetch.global.L2 [%0];" ::"l"(J.slen + v));
                    if (!BSM) asm volatile("prefetch.global.L2 [%0];" ::"l"(s.blockers + v));
                };
                pf1(pfv0);
                pf1(pfv1);
            }
            BPROF_ADD(0);
            if (delta > 0) {
                BPROF_CNT(5);
                // batches nb .. nb+delta-1 move every mover one vertex each
                // (frozen lanes stay put)
                const bool valid = (movers >> lane) & 1u;
                // lanes finishing with this leap: their successor ids now,
                // their decrements after the schedule stores (EarlyRelease)
                const bool willfin = valid && lp.len - lp.k == delta;
                early = LEAP && __reduce_add_sync(FULL, willfin ? (unsigned)(lp.q1 - lp.q0) : 0u) <= 32u * EG &&
                        __any_sync(FULL, willfin);
                if (early) release_load(J, willfin, lp.q0, lp.q1, er);
                else if (willfin) prefetch_l2(J.succ + lp.q0, (int)(lp.q1 - lp.q0) * 4);
#ifdef RECON_CHECKED
                // the leap invariant: no token outside the movers blocks a
                // mover's next `delta` vertices (frozen tokens are fixed
                // obstacles, stationary ones cannot lie on a route)
                for (unsigned m = movers; m; m &= m - 1) {
                    const int o = __ffs(m) - 1;
                    LanePath q = shfl_lane(lp, o, false);
                    for (int t0 = 0; t0 < delta; t0 += 32) {
                        const int t = t0 + lane;
                        const int32_t v = t < delta ? q.v(H, q.k + t + 1) : -1;
                        bool mover_token = false;  // a mover's current vertex: it leaves at offset 0
                        for (unsigned mm = movers; mm; mm &= mm - 1) {
                            const int32_t c = __shfl_sync(FULL, fr, __ffs(mm) - 1);
                            mover_token |= c == v && t >= 1;
                        }
                        RB_CHECK(v < 0 || !occ.get(v) || mover_token, "leap: a stationary token blocks a mover");
                    }
                }
#endif
                const unsigned vm = movers;
                if (valid) {  // the mover's run of `delta` slots, 16 bytes at a time where aligned
                    int32_t *d = J.move_batch + lp.base + lp.k;
                    int j = 0;
                    for (; j < delta && ((uintptr_t)(d + j) & 15u); ++j) __stcs(d + j, nb + j);
                    for (; j + 4 <= delta; j += 4)
                        __stcs(reinterpret_cast<int4 *>(d + j), make_int4(nb + j, nb + j + 1, nb + j + 2, nb + j + 3));
                    for (; j < delta; ++j) __stcs(d + j, nb + j);
                }
                if (early) release_issue(J, blk, er);
                if (valid) {
                    occ_toggle(occ, fr);
                    lp.k += delta;
                    fr = lp.v(H, lp.k);
                    occ_toggle(occ, fr);
                    fin = lp.k == lp.len;
                    if (fin) {
                        q0 = lp.q0;
                        q1 = lp.q1;
                    } else {
                        to = lp.v(H, lp.k + 1);
                    }
                }
                nb += delta;
                left -= (long long)__popc(vm) * delta;
                if (LEAP && pm != INT_MAX) pm -= delta;
                BPROF_ADD(1);
            } else {
                BPROF_CNT(6);
                pv_ok = false;
                const bool valid = lp.p != INT_MAX;
                bool cand;
                if (LEAP) {
                    bool held = false;  // a ready path's token sits on my destination
                    for (unsigned m = __ballot_sync(FULL, valid); m; m &= m - 1)
                        held |= __shfl_sync(FULL, fr, __ffs(m) - 1) == to;
                    cand = valid && !held;
                } else {
                    cand = valid && !occ.get(to);
                }
                const unsigned cm = __ballot_sync(FULL, cand);
                if (!cm) {
                    status = RECON_ERR_INPUT;  // batching.cpp:127-128
                    break;
                }
                bool a;
                if (J.preset != 0) {
                    const int first = __ffs(cm) - 1;
                    const int32_t ff = __shfl_sync(FULL, fr, first), ft = __shfl_sync(FULL, to, first);
                    a = cand && compatible(J.preset, H, fr, to, ff, ft);
                } else if (LEAP) {
                    // lanes are not in id order in leap mode: the minimum id of
                    // each destination group wins (batching.cpp:112-113)
                    const unsigned same = __match_any_sync(FULL, cand ? to : -2 - lane);
                    a = cand && __reduce_min_sync(same, (unsigned)lp.p) == (unsigned)lp.p;
                } else {
                    const unsigned same = __match_any_sync(FULL, cand ? to : -2 - lane);
                    a = cand && (same & lanemask_lt()) == 0;
                }
                const unsigned acc = __ballot_sync(FULL, a);
                if (LEAP) {
                    if (a) {
                        occ_toggle(occ, fr);
                        occ_toggle(occ, to);
                    }
                } else {
                    if (a) occ.clr(fr);
                    __syncwarp();
                    if (a) occ.set(to);
                }
                if (a) {
                    put_move(lp.base + lp.k, __popc(acc & lanemask_lt()));
                    ++lp.k;
                    fin = lp.k == lp.len;
                    if (fin) {
                        q0 = LEAP ? lp.q0 : J.soff[lp.p];
                        q1 = LEAP ? lp.q1 : list_end(J, lp.p);
                    }
                    // next move: horizontal steps first (virtual_line.cpp:150-173)
                    const int dx = abs(lp.xt - lp.xs);
                    fr = to;
                    to += lp.k < dx ? (lp.xt > lp.xs ? H : -H) : (lp.yt > lp.ys ? 1 : -1);
                }
                nlog += __popc(acc);
                left -= __popc(acc);
                ++nb;
                BPROF_ADD(2);
            }
            const unsigned fm = __ballot_sync(FULL, fin);
            if (LEAP && pw >= 0 && (fm >> pw & 1u)) pst = true;  // (the partner left: pm is a lower bound)
            if (fm) {
                BPROF_CNT(8);
                int32_t *newly = s.newly;
                int nnew;
                bool filled = false;
                if (LEAP && early) {
                    if (fin) lp.p = INT_MAX;
#ifdef RECON_BATCH_PROF
                    const long long ft0 = clock64();
#endif
                    nnew = release_fill(J, er, s.newly_sm, lp, &filled);
#ifdef RECON_BATCH_PROF
                    if (lane == 0) {
                        atomicAdd(&g_batch_prof[13], (unsigned long long)(clock64() - ft0));
                        atomicAdd(&g_batch_prof[14], 1ull);
                    }
#endif
                    newly = s.newly_sm;
                } else if (LEAP) {
                    if (fin) lp.p = INT_MAX;
                    nnew = release_into_lanes(J, blk, s.newly_sm, NEWLY_SM, s.newly, fin, q0, q1, &newly, lp, &filled);
                } else {
                    nnew = release_successors(J, blk, s.newly, 0, fin, q0, q1);
                    if (fin) lp.p = INT_MAX;
                }
                __syncwarp();
                if (LEAP && filled) {
                    // released paths already sit in the empty lanes
                } else if (LEAP) {
                    // more ready paths than lanes (release_into_lanes emptied
                    // the lanes it had filled): the live lanes in id order and
                    // the released ids become the sorted record list
                    int key = lp.p != INT_MAX ? (lp.p << 5) | lane : INT_MAX;
                    key = warp_sort32(key);
                    const int srcl = key == INT_MAX ? lane : (key & 31);
                    const LanePath q = shfl_lane(lp, srcl, true);
                    const int nlive = __popc(__ballot_sync(FULL, key != INT_MAX));
                    if (lane < nlive) {
                        R.rec2[lane] = lane_rec(q);
                        R.rb2[lane] = (int)q.base;
                    }
                    __syncwarp();
                    sort_newly(newly, s.mem, nnew);
                    merge_ready(paths, R, newly, nlive, nnew, s.mfr);
                    nready = nlive + nnew;
                    regmode = false;
                    __threadfence();  // the general path reads the toggled bitmap
                } else {
                const unsigned live = __ballot_sync(FULL, lp.p != INT_MAX);
                const int nlive = __popc(live);
                if (nlive + nnew > 32) {
                    // spill to the record list: live lanes are ascending
                    if (lp.p != INT_MAX) {
                        const int at = __popc(live & lanemask_lt());
                        R.rec2[at] = lane_rec(lp);
                        R.rb2[at] = (int)lp.base;
                    }
                    __syncwarp();
                    sort_newly(newly, s.mem, nnew);
                    merge_ready(paths, R, newly, nlive, nnew, s.mfr);
                    nready = nlive + nnew;
                    regmode = false;
                } else if (nnew > 0) {
                    // newly released paths take the empty lanes, then sort lanes by id
                    const int erank = __popc(~live & lanemask_lt());
                    if (lp.p == INT_MAX && erank < nnew) {
                        int b;
                        const int np = newly[erank];
                        const int4 r = make_rec(paths, np, &b);
                        lp = rec_lane(r, b);
                    }
                    int key = lp.p == INT_MAX ? INT_MAX : (lp.p << 5) | lane;
                    key = warp_sort32(key);
                    const int src = key == INT_MAX ? lane : (key & 31);
                    LanePath q = shfl_lane(lp, src, false);
                    if (key == INT_MAX) q.p = INT_MAX;
                    lp = q;
                } else {
                    // finished lanes leave gaps: lane L takes the L-th live lane
                    const int src = lane < nlive ? (int)__fns(live, 0, lane + 1) : lane;
                    LanePath q = shfl_lane(lp, src, false);
                    if (lane >= nlive) q.p = INT_MAX;
                    lp = q;
                }
                }
                lane_move();  // lanes were reloaded / reordered
                BPROF_ADD(3);
            }
            __syncwarp();
            continue;
        }
        BPROF_T0();
        BPROF_CNT(7);
        // ---- general: candidate scan over the records (ascending id)
        int nacc = 0;
        int32_t f_from = -1, f_to = -1;  // first accepted move of the batch
        // large grids (no move log): records one chunk ahead (a chunk only
        // rewrites its own records); small grids keep their registers
        constexpr bool PREFETCH = !LOG;
        int4 nrec = make_int4(0, 0, 0, 0);
        int nrb = 0;
        if (PREFETCH && lane < nready) {
            nrec = R.rec[lane];
            nrb = R.rb[lane];
        }
        for (int c0 = 0; c0 < nready; c0 += 32) {
            const int idx = c0 + lane;
            const bool valid = idx < nready;
            int4 crec = nrec;
            int crb = nrb;
            if (PREFETCH) {
                if (idx + 32 < nready) {
                    nrec = R.rec[idx + 32];
                    nrb = R.rb[idx + 32];
                }
            } else if (valid) {
                crec = R.rec[idx];
                crb = R.rb[idx];
            }
            LanePath l;
            l.p = -1;
            int32_t fr = -1, to = -1;
            bool cand = false;
            if (valid) {
                l = rec_lane(crec, crb);
                fr = l.v(H, l.k);
                to = l.v(H, l.k + 1);
                cand = !occ.get(to) && !inb.get(fr) && !inb.get(to);
                if (cand && f_from >= 0) cand = compatible(J.preset, H, fr, to, f_from, f_to);
            }
            const unsigned cm_all = __ballot_sync(FULL, cand);
            if (!cm_all) continue;
            bool a;
            if (J.preset != 0) {
                const int first = __ffs(cm_all) - 1;
                const int32_t ff = f_from >= 0 ? f_from : __shfl_sync(FULL, fr, first);
                const int32_t ft = f_from >= 0 ? f_to : __shfl_sync(FULL, to, first);
                a = cand && compatible(J.preset, H, fr, to, ff, ft);
            } else {
                const unsigned same = __match_any_sync(FULL, cand ? to : -2 - lane);
                a = cand && (same & lanemask_lt()) == 0;
            }
            const unsigned acc = __ballot_sync(FULL, a);
            if (a) {
                inb.set(fr);
                inb.set(to);
                const int slot = nacc + __popc(acc & lanemask_lt());
                put_move(l.base + l.k, slot);
                const bool fin = l.k + 1 == l.len;
                int *rw = reinterpret_cast<int *>(R.rec + idx);
                if (fin) rw[0] = -1;  // finished: dropped at the next merge
                else rw[1] = (l.k + 1) | (l.len << 16);
                s.mem[slot] = fin ? (int)(0x80000000u | (unsigned)l.p) : l.p;
                s.mfr[slot] = fr;
                s.mto[slot] = to;
            }
            if (acc && f_from < 0) {
                const int first = __ffs(acc) - 1;
                f_from = __shfl_sync(FULL, fr, first);
                f_to = __shfl_sync(FULL, to, first);
            }
            nacc += __popc(acc);
            __syncwarp();
        }
        if (nacc == 0) {
            status = RECON_ERR_INPUT;  // batching.cpp:127-128
            break;
        }
        // ---- atomic application and release (newly -> next batch), one pass:
        // the accepted moves' sources are occupied and their destinations
        // empty, so the sets are disjoint and each update is independent
        int nnew = 0, nfin = 0;
        for (int i0 = 0; i0 < nacc; i0 += 32) {
            const int i = i0 + lane;
            bool fin = false;
            int64_t q0 = 0, q1 = 0;
            if (i < nacc) {
                const int m = s.mem[i], fr = s.mfr[i], to = s.mto[i];
                occ.clr(fr);
                occ.set(to);
                inb.clr(fr);
                inb.clr(to);
                fin = m < 0;
                if (fin) {
                    const int p = m & 0x7fffffff;
                    q0 = J.soff[p];
                    q1 = list_end(J, p);
                }
            }
            nfin += __popc(__ballot_sync(FULL, fin));
            nnew = release_successors(J, blk, s.newly, nnew, fin, q0, q1);
            __syncwarp();
        }
        left -= nacc;
        nlog += nacc;
        __syncwarp();
        if ((nfin > 0 || nnew > 0) && nnew <= 32) {
            // ready' = (ready - finished) U newly in one pass into the other
            // record buffer (then the buffers swap): a kept record goes to its
            // kept index + its rank among the newly released ids (registers,
            // shuffle search); kept ranks place the newly released records
            sort_newly(s.newly, s.mem, nnew);
            int32_t *kr = s.mfr;  // free after the application step
            const int ny = lane < nnew ? s.newly[lane] : INT_MAX;
            if (lane < nnew) kr[lane] = -1;  // -> all kept below: set after the pass
            __syncwarp();
            const int ny31 = __shfl_sync(FULL, ny, 31);
            int nkeep = 0, prev_r = 0;
            for (int c0 = 0; c0 < nready; c0 += 32) {
                const int idx = c0 + lane;
                int4 x = make_int4(-1, 0, 0, 0);
                int b = 0;
                if (idx < nready) {
                    x = R.rec[idx];
                    b = R.rb[idx];
                }
                const bool keep = x.x >= 0;
                const unsigned m = __ballot_sync(FULL, keep);
                const int key = keep ? x.x : INT_MAX;
                int r = 0;  // #newly < key
#pragma unroll
                for (int st = 16; st; st >>= 1)
                    if (__shfl_sync(FULL, ny, r + st - 1) < key) r += st;
                if (r == 31 && ny31 < key) r = 32;
                const int ki = nkeep + __popc(m & lanemask_lt());
                // rank of the previous kept element (this chunk's, else the last one's)
                const unsigned before = m & lanemask_lt();
                const int rsh = __shfl_sync(FULL, r, before ? 31 - __clz(before) : lane);
                const int rp = before ? rsh : prev_r;
                if (keep) {
                    R.rec2[ki + r] = x;
                    R.rb2[ki + r] = b;
                    for (int j = rp; j < r; ++j) kr[j] = ki;  // newly j sits right before kept ki
                }
                if (m) prev_r = __shfl_sync(FULL, r, 31 - __clz(m));
                nkeep += __popc(m);
            }
            __syncwarp();
            if (lane < nnew) {
                int bb;
                const int4 rr = make_rec(paths, ny, &bb);
                const int k = kr[lane] < 0 ? nkeep : kr[lane];
                R.rec2[lane + k] = rr;
                R.rb2[lane + k] = bb;
            }
            __syncwarp();
            int4 *tr = R.rec;
            R.rec = R.rec2;
            R.rec2 = tr;
            int32_t *tb = R.rb;
            R.rb = R.rb2;
            R.rb2 = tb;
            nready = nkeep + nnew;
        } else if (nfin > 0 || nnew > 0) {
            // ready' = (ready - finished) U newly, by rank
            int nkeep = 0;
            for (int c0 = 0; c0 < nready; c0 += 32) {
                const int idx = c0 + lane;
                int4 x = make_int4(-1, 0, 0, 0);
                int b = 0;
                if (idx < nready) {
                    x = R.rec[idx];
                    b = R.rb[idx];
                }
                const bool keep = x.x >= 0;
                const unsigned m = __ballot_sync(FULL, keep);
                if (keep) {
                    const int at = nkeep + __popc(m & lanemask_lt());
                    R.rec2[at] = x;
                    R.rb2[at] = b;
                }
                nkeep += __popc(m);
            }
            __syncwarp();
            sort_newly(s.newly, s.mem, nnew);
            merge_ready(paths, R, s.newly, nkeep, nnew, s.mfr);
            nready = nkeep + nnew;
        }
        ++nb;
        if (nready <= 32) enter_regmode();
        BPROF_ADD(4);
    }
#ifdef RECON_BATCH_PROF
    bprof[9] = clock64() - bp_start;
    if (lane == 0)
        for (int i = 0; i < 10; ++i) atomicAdd(&g_batch_prof[i], (unsigned long long)bprof[i]);
#endif
    if (LOG) {
        // the instance's log -> move_batch in one burst: its region is written
        // back to back, so L2 merges the scattered 4-byte stores into sectors
        __syncwarp();
        for (int i = lane; i < nlog; i += 32) {
            const int2 e = __ldcs(J.mlog + i);
            J.move_batch[e.x] = e.y;
        }
    }
    if (lane == 0) {
        if (J.nlog) *J.nlog = nlog;
        *J.batch_count = status == RECON_OK ? nb : 0;
        *J.status = status;
        if (J.detail) *J.detail = status == RECON_OK ? 0 : RECON_D_BATCH_NO_PROGRESS;
    }
}

// MODE bits: 1 = occupancy / in-batch bitmaps in shared memory, 2 = move log,
// 4 = blocker counts in shared memory (u16, after the bitmaps; needs 1),
// 8 = the in-batch bitmap stays in global memory (only the candidate scan of
// the general path touches it), halving a large grid's shared memory,
// 16 = leap mode (preset none; no move log)
template <int MODE>
// (mode 16, one warp per CTA: <= 168 registers keep 3 warps per SM sub-partition)
__global__ void __launch_bounds__(MODE == 16 ? 32 : 256, MODE == 16 ? 12 : ((MODE & 2) ? 4 : 1)) batch_pipeline_kernel(PipelineArgs a) {
    constexpr bool occ_in_smem = MODE & 1, LOG = MODE & 2, BSM = MODE & 4, INB_SM = occ_in_smem && !(MODE & 8);
    constexpr bool LEAP = MODE & 16;
    static_assert(!(LEAP && LOG), "leap mode writes move_batch directly");
    extern __shared__ __align__(16) uint32_t bsmem[];
    __shared__ int32_t newly_buf[LEAP ? 8 : 1][LEAP ? NEWLY_SM : 1];
    const int64_t S = (int64_t)a.W * a.k, nwb = ((int64_t)a.W * a.H + 31) / 32;
    const int nw = blockDim.x >> 5;
    for (int inst = blockIdx.x * nw + warp_id(); inst < a.count; inst += gridDim.x * nw) {
        if (a.solve_status[inst] != 0) {
            if (lane_id() == 0) {
                a.status[inst] = a.solve_status[inst];
                a.batch_count[inst] = 0;
                if (a.detail && a.solve_detail && a.detail != a.solve_detail) a.detail[inst] = a.solve_detail[inst];
            }
            continue;
        }
        const int64_t *wst = a.wstate ? a.wstate + (int64_t)inst * 4 : nullptr;
        if (wst && wst[0] == 2) continue;  // the wide phase finished the instance
        const int64_t o = (int64_t)inst * S;
        const int64_t moves = a.mbase[o + a.path_count[inst]] - a.mbase[o];
        if (moves > a.move_stride || moves >= INT_MAX) {  // (records hold 32-bit move slots)
            if (lane_id() == 0) {
                a.status[inst] = RECON_ERR_CAPACITY;
                a.batch_count[inst] = 0;
                if (a.detail) a.detail[inst] = RECON_D_NONE;
            }
            continue;
        }
        BatchJob J{};
        J.P = a.path_count[inst];
        J.W = a.W;
        J.H = a.H;
        J.preset = a.preset;
        J.edge_level = 0;
        J.soff = a.soff + o;
        J.prec = a.prec ? a.prec + (int64_t)inst * (S + 1) : nullptr;
        J.e0 = a.soff[o];
        J.succ = a.succ;
        J.slen = a.slen ? a.slen + o : nullptr;
        J.s.occ = a.occ + inst * nwb;
        J.s.inb = a.inb + inst * nwb;
        const int64_t nbw = BSM ? (S + 1) / 2 : 0, nib = INB_SM ? nwb : 0, per = nwb + nib + nbw;
        if (occ_in_smem) {  // the instance's occupancy (and in-batch) bitmaps live in this warp's shared memory
            uint32_t *mine = bsmem + (size_t)warp_id() * per;
            for (int64_t w = lane_id(); w < nwb; w += 32) {
                mine[w] = J.s.occ[w];
                if (INB_SM) mine[nwb + w] = 0u;
            }
            __syncwarp();
            J.s.occ = mine;
            if (INB_SM) J.s.inb = mine + nwb;
        }
        J.s.blockers = a.indeg + o;
        J.s.newly = a.newly + o;
        J.s.newly_sm = LEAP ? newly_buf[warp_id()] : nullptr;
        J.s.mem = a.mem + o;
        J.s.mfr = a.mfr + o;
        J.s.mto = a.mto + o;
        J.s.counter = a.counter + inst;
        J.move_batch = a.move_batch + (int64_t)inst * a.move_stride;
        if (LOG) {
            J.mlog = a.mlog + a.mbase[o];
            J.nlog = a.counter + inst;
        }
        J.batch_count = a.batch_count + inst;
        J.status = a.status + inst;
        J.detail = a.detail ? a.detail + inst : nullptr;
        ImplicitPaths ip{a.path_src + o, a.path_dst + o, a.mbase + o, a.mbase[o], a.H};
        const PipeRecords R{a.rec + o, a.rec2 + o, a.rb + o, a.rb2 + o};
        if (BSM) {
            uint32_t *bw = bsmem + (size_t)warp_id() * per + nwb + nib;
            const int P = J.P;
            for (int64_t w = lane_id(); w < nbw; w += 32) {
                const int p = (int)(2 * w);
                const uint32_t lo = p < P ? (uint32_t)J.s.blockers[p] : 0u;
                const uint32_t hi = p + 1 < P ? (uint32_t)J.s.blockers[p + 1] : 0u;
                bw[w] = lo | (hi << 16);
            }
            __syncwarp();
            J.s.blk_sm = bw;
        }
        batch_warp_pipe<occ_in_smem, INB_SM, LOG, BSM, LEAP>(J, ip, R, wst);
    }
}

cudaError_t pipeline_run_batching(const PipelineArgs &a, int sms, cudaStream_t st, cudaEvent_t *pev, int64_t *launches) {
    const int64_t S = (int64_t)a.W * a.k, N = (int64_t)a.count * S, nwb = ((int64_t)a.W * a.H + 31) / 32;
    const int blocks = 148 * 8;
    if (a.small_dag) {
        const int64_t smem = pipeline_small_dag_smem(a.W, a.H, a.k);
        pl_dag_small_kernel<1><<<(int)std::min<int64_t>(a.count, 148 * 16), 256, smem, st>>>(a);
    } else {
        const int32_t *mc = a.source_of, *mr = a.source_of + (size_t)a.count * a.W * a.H * 4;
        // lanes per path of the walk (RECON_WALK_LANES: 32 = a warp per path;
        // C5 walk time at 256 instances, ms: 40.8 / 32.8 / 28.0 / 26.0 / 27.3 /
        // 30.0 for 32 / 16 / 8 / 4 / 2 / 1; a lane-per-path walk whose lanes
        // take a new path as soon as their route ends, without shuffles:
        // 37.8 vs 26.0 ms for the 4-lane walk, its per-lane map reads touch a
        // line each)
        static const int lanes_env = [] {
            const char *e = getenv("RECON_WALK_LANES");
            return e ? atoi(e) : 4;
        }();
        const CoverArrays cva = pipeline_cover_arrays(a);
        cudaMemsetAsync(a.newly, 0, (size_t)a.count * (size_t)a.W * a.k * sizeof(int32_t), st);
        const int4 *mc4 = (const int4 *)mc, *mr4 = (const int4 *)mr;
        switch (lanes_env) {
            case 1: pl_walk_half_kernel<1><<<blocks, 256, 0, st>>>(a, mc4, mr4, cva); break;
            case 2: pl_walk_half_kernel<2><<<blocks, 256, 0, st>>>(a, mc4, mr4, cva); break;
            case 8: pl_walk_half_kernel<8><<<blocks, 256, 0, st>>>(a, mc4, mr4, cva); break;
            case 16: pl_walk_half_kernel<16><<<blocks, 256, 0, st>>>(a, mc4, mr4, cva); break;
            case 32: pl_walk_warp_kernel<<<blocks, 256, 0, st>>>(a, mc4, mr4, cva); break;
            default: pl_walk_half_kernel<4><<<blocks, 256, 0, st>>>(a, mc4, mr4, cva); break;
        }
        pl_compact_kernel<<<blocks, 256, 0, st>>>(a);
        *launches += 1;
    }
    if (a.prec) prec_kernel<<<blocks, 256, 0, st>>>(a);
    occ_to_vertex_bits<<<blocks, 256, 0, st>>>(a.count, a.W, a.H, a.grid_occ, a.occ);
    *launches += a.prec ? 3 : 2;  // dag fill (+ path records) + bitmap
    cudaMemsetAsync(a.inb, 0, (size_t)a.count * nwb * 4, st);
    cudaMemsetAsync(a.counter, 0, (size_t)a.count * 4, st);
    (void)N;
    if (pev) cudaEventRecord(pev[2], st);
    if (a.wide) {
        // wide phase first: the batches whose ready set exceeds a warp
        int rmax = 0, hbits = 0;
        size_t wsmem = 0;
        static const int wide_smem_env = [] {
            const char *e = getenv("RECON_WIDE_SMEM_KB");
            return e ? atoi(e) : 0;
        }();
        const int64_t budget = wide_smem_env > 0 ? (int64_t)wide_smem_env * 1024 : 113 * 1024;  // 2 CTAs per SM
        // preset none: windows of batches (RECON_WIDE_WINDOW=0: batch by batch)
        static const int window_env = [] {
            const char *e = getenv("RECON_WIDE_WINDOW");
            return e ? atoi(e) : 1;
        }();
        if (a.preset == 0 && window_env && a.prec &&
            (pipeline_window_config(a.W, a.H, budget, &rmax, &wsmem) ||
             pipeline_window_config(a.W, a.H, 220 * 1024, &rmax, &wsmem))) {
            cudaMemsetAsync(a.vmin, 0x7f, (size_t)a.count * a.W * a.H * 4, st);
            cudaMemsetAsync(a.wnext, 0, sizeof(int32_t), st);
            cudaError_t e = launch_batch_window(a, sms, rmax, wsmem, st);
            if (e != cudaSuccess) return e;
            *launches += 1;
        } else if (pipeline_wide_config(a.W, a.H, budget, &rmax, &hbits, &wsmem) ||
            pipeline_wide_config(a.W, a.H, 220 * 1024, &rmax, &hbits, &wsmem)) {
            cudaMemsetAsync(a.vmin, 0x7f, (size_t)a.count * a.W * a.H * 4, st);
            cudaError_t e = launch_batch_wide(a, sms, rmax, hbits, wsmem, st);
            if (e != cudaSuccess) return e;
            *launches += 1;
        } else {
            cudaMemsetAsync(a.wstate, 0, (size_t)a.count * 32, st);
        }
    }
    // occupancy + in-batch bitmaps in shared memory when a few warps' worth fits
    // bitmaps in shared memory when a few warps' worth fits; then the blocker
    // counts too when they fit in u16 and the CTA keeps at least two warps
    const int64_t bm_bytes = 2 * nwb * 4, blk_bytes = (S + 1) / 2 * 4;
    static const int bsm_env = [] {
        const char *e = getenv("RECON_BATCH_BSM");
        return e ? atoi(e) : 1;
    }();
    int warps = 4, mode = 0;
    size_t smem = 0;
    static const int occ_env = [] {
        const char *e = getenv("RECON_BATCH_OCC_SMEM");
        return e ? atoi(e) : 1;
    }();
    if (a.leap) {
        // leap mode reads the bitmaps only in literal batches and the general
        // (> 32 ready) path: shared memory only when it costs no warps
        mode = 16;
        int64_t per = bm_bytes + (S < 65536 ? blk_bytes : 0);
        if (occ_env && per <= 24 * 1024) {
            mode |= 1 | ((bsm_env && S < 65536) ? 4 : 0);
            if (!(mode & 4)) per = bm_bytes;
            warps = 8;
            smem = (size_t)warps * per;
        } else {
            // one warp (instance) per CTA: ~180 registers per thread still
            // keep 11 instances per SM resident
            warps = 1;
        }
    } else if (occ_env && bm_bytes <= 96 * 1024) {
        mode = 1 | (a.mlog ? 2 : 0);
        if (bsm_env && S < 65536 && bm_bytes + blk_bytes <= 100 * 1024) mode |= 4;
        int64_t per = bm_bytes + ((mode & 4) ? blk_bytes : 0);
        warps = (int)std::max<int64_t>(1, std::min<int64_t>(8, (200 * 1024) / per));
        // more instances than the SMs hold with both bitmaps: keep only the
        // occupancy in shared memory, for twice the warps per SM
        if (mode == 1 && warps < 8 && a.count > (int64_t)warps * sms) {
            mode |= 8;
            per = bm_bytes / 2;
            warps = (int)std::max<int64_t>(1, std::min<int64_t>(8, (200 * 1024) / per));
        }
        smem = (size_t)warps * per;
    }
    void (*kern)(PipelineArgs) = mode == 0 ? batch_pipeline_kernel<0> : mode == 1 ? batch_pipeline_kernel<1>
                               : mode == 9 ? batch_pipeline_kernel<9> : mode == 3 ? batch_pipeline_kernel<3>
                               : mode == 5 ? batch_pipeline_kernel<5> : mode == 16 ? batch_pipeline_kernel<16>
                               : mode == 17 ? batch_pipeline_kernel<17> : mode == 21 ? batch_pipeline_kernel<21>
                               : batch_pipeline_kernel<7>;
    if (smem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = (int)std::min<int64_t>(((int64_t)a.count + warps - 1) / warps, (int64_t)sms * 32);
    if (pev) cudaEventRecord(pev[3], st);
    kern<<<grid, warps * 32, smem, st>>>(a);
    *launches += 1;
    if (pev) cudaEventRecord(pev[4], st);
    return cudaGetLastError();
}

}  // namespace rb

// experiments: the phase counters above (zero unless built with -DRECON_BATCH_PROF)
extern "C" int recon_debug_batch_prof(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, rb::g_batch_prof, sizeof(rb::g_batch_prof)) != cudaSuccess) return -1;
    if (reset) {
        static const unsigned long long z[16] = {};
        if (cudaMemcpyToSymbol(rb::g_batch_prof, z, sizeof(z)) != cudaSuccess) return -1;
    }
    return 0;
}
