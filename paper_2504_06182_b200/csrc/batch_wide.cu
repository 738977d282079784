// Pipeline batching, wide phase: one CTA per instance while the ready set is
// larger than a warp (batching.cpp:95-157, the same literal semantics as
// batching.cu).
//
// Every grid solve starts with many independent column events (bird's column
// pass, red-rec's compactions), so its first few thousand batches each move
// hundreds of paths: C5 moves half of its 10.7 M moves in its first ~8.6 K
// batches with up to 1,024 ready paths.  One warp walks those batches 32
// candidates at a time through global memory; here a CTA holds the whole
// ready set and the occupancy bitmap in shared memory and runs one batch in a
// handful of barriers:
//   1. each ready entry computes its next move (from -> to); it is a candidate
//      when `to` is empty before the batch (batching.cpp:111).  Candidates
//      claim `to` in a shared hash table; a second claimer flags contention,
//      and only then (rare) the minimum id per destination is resolved through
//      a per-vertex global array (batching.cpp:112-113: the first candidate
//      in ascending id wins a shared destination).  column_direction accepts
//      the candidates compatible with the minimum-id candidate
//      (batching.cpp:114-120).
//   2. accepted moves are applied atomically: sources vacated, barrier,
//      destinations filled (batching.cpp:131-136); the batch index is stored
//      at the move's path-major slot.
//   3. finished paths release their successors (CSR, global blocker counts):
//      the successor lists of all finished paths are concatenated by a CTA
//      scan and spread over the threads, loads first, then decrements.
//   4. the next ready list = live entries + newly released paths (order is
//      irrelevant: every decision above is a min over ids).
// When the ready set drops to <= 32 (or outgrows shared memory), the CTA
// writes the ready set as id-sorted records, the bitmap and the counters to
// global memory and the warp kernel (batching.cu) continues from there.

#include <algorithm>
#include <climits>

#include "batching.cuh"
#include "common.cuh"

namespace rb {

// phase cycle counters of the wide kernel (experiments: -DRECON_BATCH_PROF)
__device__ unsigned long long g_wide_prof[8];

namespace {

constexpr int WT = 512;  // threads per CTA
constexpr int NW = WT / 32;
constexpr int G = 4;  // chunks of 32 successor ids per warp in flight
constexpr int32_t VMIN_EMPTY = 0x7f7f7f7f;  // memset(0x7f) of the per-vertex min array

__device__ __forceinline__ int vtx(int H, int k, int xs, int ys, int xt, int yt) {
    const int dx = abs(xt - xs);
    if (k <= dx) return (xs + (xt > xs ? k : -k)) * H + ys;
    const int m = k - dx;
    return xt * H + ys + (yt > ys ? m : -m);
}

__device__ __forceinline__ int move_dir_w(int H, int32_t a, int32_t b) {
    const int ay = a % H, by = b % H;
    if (by > ay) return 0;
    if (by < ay) return 1;
    if (b / H < a / H) return 2;
    return 3;
}

// ConstraintSet::compatible (batching.cpp:17-24)
__device__ __forceinline__ bool compatible_w(int preset, int H, int32_t af, int32_t at, int32_t bf, int32_t bt) {
    if (preset == 0) return true;
    const int da = move_dir_w(H, af, at), db = move_dir_w(H, bf, bt);
    if (da != db) return false;
    if (da <= 1) return af / H == bf / H;
    return af % H == bf % H;
}

__device__ __forceinline__ unsigned hslot(int v, int hbits) { return ((unsigned)v * 2654435761u) >> (32 - hbits); }

struct WideLayout {
    int64_t occ, hash, rec, base, q0, qn, eslot, fq0, fqn, flag, total;
};

__host__ __device__ inline int64_t al16w(int64_t x) { return (x + 15) / 16 * 16; }

__host__ __device__ inline WideLayout wide_layout(int64_t nwb, int rmax, int hsize) {
    WideLayout L;
    int64_t o = 0;
    L.occ = o;
    o = al16w(o + nwb * 4);
    L.hash = o;
    o = al16w(o + (int64_t)hsize * 4);
    L.rec = o;  // 2 buffers
    o = al16w(o + (int64_t)rmax * 16 * 2);
    L.base = o;
    o = al16w(o + (int64_t)rmax * 4 * 2);
    L.q0 = o;
    o = al16w(o + (int64_t)rmax * 4 * 2);
    L.qn = o;
    o = al16w(o + (int64_t)rmax * 4 * 2);
    L.eslot = o;  // int16 claim slot per entry (hsize <= 32768)
    o = al16w(o + (int64_t)rmax * 2);
    L.fq0 = o;
    o = al16w(o + (int64_t)rmax * 4);
    L.fqn = o;
    o = al16w(o + (int64_t)rmax * 4);
    L.flag = o;
    o = al16w(o + (int64_t)rmax);
    L.total = o;
    return L;
}

// entry flags
constexpr unsigned char F_CAND = 1, F_WON = 4;

struct WideBufs {
    int4 *rec;
    int *base, *q0, *qn;
};

// appends one ready entry to the next list (shared memory, or the global
// staging area past rmax: the hand-off then reads it from there)
__device__ __forceinline__ void wide_put(const WideBufs &B, int i, int rmax, int4 *stg, int32_t *stb, int4 r, int base,
                                         int q0, int qn, int *ovf) {
    if (i < rmax) {
        B.rec[i] = r;
        B.base[i] = base;
        B.q0[i] = q0;
        B.qn[i] = qn;
    } else {
        stg[i] = r;
        stb[i] = base;
        *ovf = 1;
    }
}

__global__ void __launch_bounds__(WT, 2) batch_wide_kernel(PipelineArgs a, int rmax, int hbits) {
    extern __shared__ __align__(16) unsigned char wsm[];
    // per-batch counters, double-buffered by batch parity: batch b uses [b & 1]
    // and resets [(b + 1) & 1] after its first barrier
    __shared__ int s_cnt[2], s_nacc[2], s_nf[2], s_contend[2], s_first[2];
    __shared__ int s_ovf, s_ff, s_ft;
    __shared__ unsigned long long s_left;
    const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
    const int W = a.W, H = a.H, hsize = 1 << hbits;
    const int64_t S = (int64_t)W * a.k, WH = (int64_t)W * H, nwb = (WH + 31) / 32;
    const WideLayout L = wide_layout(nwb, rmax, hsize);
    uint32_t *occ = (uint32_t *)(wsm + L.occ);
    uint32_t *hash = (uint32_t *)(wsm + L.hash);
    // buffer q of the two ready lists
    auto bufs = [&](int q) {
        return WideBufs{(int4 *)(wsm + L.rec) + q * rmax, (int *)(wsm + L.base) + q * rmax,
                        (int *)(wsm + L.q0) + q * rmax, (int *)(wsm + L.qn) + q * rmax};
    };
    int16_t *eslot = (int16_t *)(wsm + L.eslot);
    int *fq0 = (int *)(wsm + L.fq0), *fqn = (int *)(wsm + L.fqn);
    unsigned char *eflag = wsm + L.flag;
    for (int inst = blockIdx.x; inst < a.count; inst += gridDim.x) {
        int64_t *st = a.wstate + (int64_t)inst * 4;
        if (a.solve_status[inst] != 0) {
            if (tid == 0) st[0] = 0;  // the warp kernel reports the solve status
            continue;
        }
        const int64_t o = (int64_t)inst * S;
        const int P = a.path_count[inst];
        const int64_t *mbase = a.mbase + o, *soff = a.soff + o;
        const int64_t mb0 = mbase[0], e0 = soff[0];
        const int64_t moves = mbase[P] - mb0;
        if (moves > a.move_stride || moves >= INT_MAX) {
            if (tid == 0) st[0] = 0;  // the warp kernel reports the capacity status
            continue;
        }
        int32_t *blk = a.indeg + o;
        int32_t *mb = a.move_batch + (int64_t)inst * a.move_stride;
        const int4 *prec = a.prec + (int64_t)inst * (S + 1);  // path records (batching.cu prec_kernel)
        int4 *stg = a.rec2 + o;  // hand-off staging (and overflow past rmax)
        int32_t *stb = a.rb2 + o;
        const int32_t *succ = a.succ + e0;
        const int32_t *slen = a.slen ? a.slen + o : nullptr;  // list lengths (else up to the next list)
        // ---- ready set at batch 0 (read-only: on a bail-out the warp kernel
        // starts from scratch)
        if (tid == 0) {
            s_cnt[0] = s_cnt[1] = 0;
            s_nacc[0] = s_nacc[1] = 0;
            s_nf[0] = s_nf[1] = 0;
            s_contend[0] = s_contend[1] = 0;
            s_first[0] = s_first[1] = INT_MAX;
            s_ovf = 0;
            s_left = 0;
        }
        __syncthreads();
        long long myleft = 0;
        int zero_len = 0;
        for (int p = tid; p < P; p += WT) {
            const int4 r = prec[p];
            const int len = abs((r.y & 0xffff) - (r.x & 0xffff)) + abs((r.y >> 16) - (r.x >> 16));
            myleft += len;
            if (len == 0) {
                zero_len = 1;  // zero-length paths: the warp kernel's init releases them
            } else if (blk[p] == 0) {
                const int i = atomicAdd(&s_cnt[1], 1);  // [1]: batch 0 appends to [0]
                wide_put(bufs(0), i, rmax, stg, stb, make_int4(p, len << 16, r.x, r.y), r.z, r.w, slen ? slen[p] : prec[p + 1].w - r.w,
                         &s_ovf);
            }
        }
        if (zero_len) s_ovf = 1;
        myleft = warp_sum64(myleft);
        if (lane == 0) atomicAdd(&s_left, (unsigned long long)myleft);
        for (int64_t w = tid; w < nwb; w += WT) occ[w] = a.occ[(int64_t)inst * nwb + w];
        for (int h = tid; h < hsize; h += WT) hash[h] = 0u;
        __syncthreads();
        int R = s_cnt[1];
        long long left = (long long)s_left;
        if (s_ovf || R <= 32 || left == 0) {
            if (tid == 0) st[0] = 0;
            __syncthreads();
            continue;
        }
        int cur = 0, nb = 0, status = RECON_OK;
#ifdef RECON_BATCH_PROF
        long long wp[4] = {0, 0, 0, 0}, wt = clock64();
#define WPROF(i)                          \
    do {                                  \
        const long long t_ = clock64();   \
        wp[i] += t_ - wt;                 \
        wt = t_;                          \
    } while (0)
#else
#define WPROF(i) (void)0
#endif
        for (;;) {
            const int par = nb & 1;
            const WideBufs A = bufs(cur), B = bufs(cur ^ 1);
            // ---- 1. candidates and destination claims
            const bool none = a.preset == 0;
            for (int e = tid; e < R; e += WT) {
                const int4 r = A.rec[e];
                const int to = vtx(H, (r.y & 0xffff) + 1, r.z & 0xffff, r.z >> 16, r.w & 0xffff, r.w >> 16);
                unsigned char f = 0;
                int slot = -1;
                if (!((occ[to >> 5] >> (to & 31)) & 1u)) {
                    f = F_CAND;
                    if (!none) {  // column_direction: claims in the hash table
                        unsigned h = hslot(to, hbits);
                        for (int probes = 0;; ++probes) {
                            RB_CHECK(probes < hsize, "wide: claim table full");
                            const uint32_t old = atomicCAS(&hash[h], 0u, (uint32_t)to + 1u);
                            if (old == 0u) {
                                slot = (int)h;
                                break;
                            }
                            if (old == (uint32_t)to + 1u) {
                                s_contend[par] = 1;
                                break;
                            }
                            h = (h + 1) & (hsize - 1);
                        }
                        atomicMin(&s_first[par], r.x);
                    }
                }
                eslot[e] = (int16_t)slot;
                eflag[e] = f;
            }
            if (none) {
                // preset none: every candidate is accepted unless it shares its
                // destination, and the destination ends up occupied either way,
                // so candidates claim it in the occupancy bitmap itself (after
                // every candidate has read the pre-batch bitmap): a set bit seen
                // by a claim is a second claimer
                __syncthreads();
                for (int e = tid; e < R; e += WT) {
                    if (!(eflag[e] & F_CAND)) continue;
                    const int4 r = A.rec[e];
                    const int to = vtx(H, (r.y & 0xffff) + 1, r.z & 0xffff, r.z >> 16, r.w & 0xffff, r.w >> 16);
                    if (atomicOr(&occ[to >> 5], 1u << (to & 31)) & (1u << (to & 31))) s_contend[par] = 1;
                }
            }
            __syncthreads();
            WPROF(0);
            if (tid == 0) {  // next batch's counters (their last readers passed the barrier above)
                s_cnt[par ^ 1] = 0;
                s_nacc[par ^ 1] = 0;
                s_nf[par ^ 1] = 0;
                s_contend[par ^ 1] = 0;
                s_first[par ^ 1] = INT_MAX;
            }
            const bool contend = s_contend[par] != 0;
            if (contend) {
                // rare: minimum id per contended destination (batching.cpp:112-113)
                int32_t *vmin = a.vmin + (int64_t)inst * WH;
                auto dest = [&](int e) {
                    const int4 r = A.rec[e];
                    return vtx(H, (r.y & 0xffff) + 1, r.z & 0xffff, r.z >> 16, r.w & 0xffff, r.w >> 16);
                };
                for (int e = tid; e < R; e += WT)
                    if (eflag[e] & F_CAND) atomicMin(&vmin[dest(e)], A.rec[e].x);
                __threadfence_block();
                __syncthreads();
                for (int e = tid; e < R; e += WT)
                    if ((eflag[e] & F_CAND) && __ldcg(&vmin[dest(e)]) == A.rec[e].x) eflag[e] |= F_WON;
                __syncthreads();
                for (int e = tid; e < R; e += WT)
                    if (eflag[e] & F_CAND) vmin[dest(e)] = VMIN_EMPTY;
            }
            if (a.preset != 0) {
                const int first = s_first[par];
                for (int e = tid; e < R; e += WT)
                    if ((eflag[e] & F_CAND) && A.rec[e].x == first) {
                        const int4 r = A.rec[e];
                        s_ff = vtx(H, r.y & 0xffff, r.z & 0xffff, r.z >> 16, r.w & 0xffff, r.w >> 16);
                        s_ft = vtx(H, (r.y & 0xffff) + 1, r.z & 0xffff, r.z >> 16, r.w & 0xffff, r.w >> 16);
                    }
                __syncthreads();
            }
            // ---- 2. application (a move toggles its source bit, and its
            // destination bit unless the claim set it: the sets are disjoint,
            // so no ordering is needed), the move's
            // batch index, finished paths to the release list, live paths to
            // the next list
            int nacc = 0;
            for (int e0 = 0; e0 < R; e0 += WT) {  // (warp-uniform trip count: the appends are warp-aggregated)
                const int e = e0 + tid;
                const bool valid = e < R;
                const unsigned char f = valid ? eflag[e] : 0;
                int4 r = valid ? A.rec[e] : make_int4(0, 0, 0, 0);
                bool fin = false;
                if (f & F_CAND) {
                    if (eslot[e] >= 0) hash[eslot[e]] = 0u;
                    const int fr = vtx(H, r.y & 0xffff, r.z & 0xffff, r.z >> 16, r.w & 0xffff, r.w >> 16);
                    const int to = vtx(H, (r.y & 0xffff) + 1, r.z & 0xffff, r.z >> 16, r.w & 0xffff, r.w >> 16);
                    bool won = contend ? (f & F_WON) != 0 : true;
                    if (won && a.preset != 0) won = compatible_w(a.preset, H, fr, to, s_ff, s_ft);
                    if (won) {
                        atomicXor(&occ[fr >> 5], 1u << (fr & 31));
                        if (!none) atomicXor(&occ[to >> 5], 1u << (to & 31));  // (none: claimed already)
                        const int k = r.y & 0xffff, len = r.y >> 16;
                        __stcs(mb + A.base[e] + k, nb);
                        r.y = (k + 1) | (len << 16);
                        ++nacc;
                        fin = k + 1 == len;
                        // one move left: its successor list into L2 for the release
                        if (k + 2 == len) prefetch_l2(succ + A.q0[e], A.qn[e] * 4);
                    }
                }
                const bool live = valid && !fin;
                const unsigned lm = __ballot_sync(FULL, live), fm = __ballot_sync(FULL, fin);
                int lb = 0, fb = 0;
                if (lane == 0) {
                    if (lm) lb = atomicAdd(&s_cnt[par], __popc(lm));
                    if (fm) fb = atomicAdd(&s_nf[par], __popc(fm));
                }
                lb = __shfl_sync(FULL, lb, 0);
                fb = __shfl_sync(FULL, fb, 0);
                if (live) wide_put(B, lb + __popc(lm & lanemask_lt()), rmax, stg, stb, r, A.base[e], A.q0[e], A.qn[e], &s_ovf);
                if (fin) {
                    const int i = fb + __popc(fm & lanemask_lt());
                    RB_CHECK(i < rmax, "wide: finished list overflow");
                    fq0[i] = A.q0[e];
                    fqn[i] = A.qn[e];
                }
            }
            nacc = warp_sum(nacc);
            if (lane == 0 && nacc) atomicAdd(&s_nacc[par], nacc);
            __syncthreads();
            WPROF(1);
            const int nacc_all = s_nacc[par];
            if (nacc_all == 0) {
                status = RECON_ERR_INPUT;  // batching.cpp:127-128
                break;
            }
            left -= nacc_all;
            ++nb;
            // ---- 3. release (for the next batch): warp w takes finished paths
            // w, w + NW, ...; its lanes load 32 successor ids of one finished
            // path at a time into G register slots, then decrement them all;
            // a released path joins the next list from its path record
            const int nf = s_nf[par];
            {
                int sc[G];
                int nsl = 0;  // filled slots (warp-uniform)
                auto flush = [&]() {
                    bool rel[G];
                    int4 pr[G];
                    int qe[G];
                    int old[G];
#pragma unroll
                    for (int c = 0; c < G; ++c) {
                        const bool ok = c < nsl && sc[c] >= 0;
                        if (ok) {
                            pr[c] = __ldg(prec + sc[c]);
                            qe[c] = slen ? __ldg(slen + sc[c]) : __ldg(&prec[sc[c] + 1].w);
                        }
                        old[c] = (int)atom_add_if(ok, reinterpret_cast<uint32_t *>(blk + max(sc[c], 0)), 0xffffffffu);
                    }
#pragma unroll
                    for (int c = 0; c < G; ++c) rel[c] = c < nsl && sc[c] >= 0 && old[c] == 1;
#pragma unroll
                    for (int c = 0; c < G; ++c) {
                        if (!rel[c]) continue;
                        const int len = abs((pr[c].y & 0xffff) - (pr[c].x & 0xffff)) + abs((pr[c].y >> 16) - (pr[c].x >> 16));
                        const int i = atomicAdd(&s_cnt[par], 1);
                        wide_put(B, i, rmax, stg, stb,
                                 make_int4(sc[c], len << 16, pr[c].x, pr[c].y), pr[c].z, pr[c].w, slen ? qe[c] : qe[c] - pr[c].w, &s_ovf);
                    }
                    nsl = 0;
                };
                for (int f = warp; f < nf; f += NW) {
                    const int fq = fq0[f], fn = fqn[f];
                    for (int j0 = 0; j0 < fn; j0 += 32) {
                        const int v = j0 + lane < fn ? __ldg(succ + fq + j0 + lane) : -1;
#pragma unroll
                        for (int c = 0; c < G; ++c)
                            if (c == nsl) sc[c] = v;
                        if (++nsl == G) flush();
                    }
                }
                if (nsl) flush();
            }
            __syncthreads();
            WPROF(2);
            RB_CHECK(s_cnt[par] <= S, "wide: ready list larger than the path count");
            R = s_cnt[par];
            cur ^= 1;
            if (left == 0 || R <= 32 || s_ovf) break;
        }
#ifdef RECON_BATCH_PROF
        if (tid == 0) {
            for (int i = 0; i < 3; ++i) atomicAdd(&g_wide_prof[i], (unsigned long long)wp[i]);
            atomicAdd(&g_wide_prof[3], (unsigned long long)nb);
            atomicAdd(&g_wide_prof[4], 1ull);
        }
#endif
        // ---- hand-off to the warp kernel, or the instance's result
        if (status == RECON_OK && left > 0) {
            // the ready set as records ranked by id into the warp kernel's
            // records (entries past rmax are already in the staging area)
            const WideBufs A = bufs(cur);
            const int n = R;
            for (int i = tid; i < min(n, rmax); i += WT) {
                stg[i] = A.rec[i];
                stb[i] = A.base[i];
            }
            __threadfence();
            __syncthreads();
            for (int i = tid; i < n; i += WT) {
                const int4 x = __ldcg(&stg[i]);
                int rank = 0;
                for (int j = 0; j < n; ++j) rank += __ldcg(&stg[j].x) < x.x;
                a.rec[o + rank] = x;
                a.rb[o + rank] = __ldcg(&stb[i]);
            }
            for (int64_t w = tid; w < nwb; w += WT) a.occ[(int64_t)inst * nwb + w] = occ[w];
            if (tid == 0) {
                st[0] = 1;
                st[1] = nb;
                st[2] = left;
                st[3] = n;
            }
        } else if (tid == 0) {
            st[0] = 2;
            a.batch_count[inst] = status == RECON_OK ? nb : 0;
            a.status[inst] = status;
            if (a.detail) a.detail[inst] = status == RECON_OK ? 0 : RECON_D_BATCH_NO_PROGRESS;
        }
        __syncthreads();
    }
}

}  // namespace

// largest ready set the wide kernel holds in `smem_budget` bytes, and its hash bits
bool pipeline_wide_config(int W, int H, int64_t smem_budget, int *rmax, int *hbits, size_t *smem) {
    const int64_t nwb = ((int64_t)W * H + 31) / 32;
    for (int r = 4096; r >= 256; r -= 64) {
        int hb = 1;
        while ((1 << hb) < 2 * r) ++hb;
        if (hb > 15) continue;  // int16 claim slots
        const WideLayout L = wide_layout(nwb, r, 1 << hb);
        if (L.total <= smem_budget) {
            *rmax = r;
            *hbits = hb;
            *smem = (size_t)L.total;
            return true;
        }
    }
    return false;
}

cudaError_t launch_batch_wide(const PipelineArgs &a, int sms, int rmax, int hbits, size_t smem, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(batch_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, batch_wide_kernel, WT, smem);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<int64_t>(a.count, (int64_t)sms * std::max(1, per_sm));
    batch_wide_kernel<<<grid, WT, smem, st>>>(a, rmax, hbits);
    return cudaGetLastError();
}

}  // namespace rb

// experiments: the wide kernel's phase counters (zero unless built with -DRECON_BATCH_PROF)
extern "C" int recon_debug_wide_prof(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, rb::g_wide_prof, sizeof(rb::g_wide_prof)) != cudaSuccess) return -1;
    if (reset) {
        static const unsigned long long z[8] = {};
        if (cudaMemcpyToSymbol(rb::g_wide_prof, z, sizeof(z)) != cudaSuccess) return -1;
    }
    return 0;
}
