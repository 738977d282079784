// Pipeline batching, wide phase for preset none in windows of batches
// (batching.cpp:95-157, the same literal semantics as batch_wide.cu).
//
// Without stalls the schedule is the occupancy DAG's longest-path schedule:
// a ready path moves in every batch, so an entry with k of its len moves done
// finishes at offset len - k - 1, and a successor whose last blocker finishes
// at f becomes ready at f + 1.  On C5 the first ~8.6 K batches
// (up to 1,024 ready paths each) hold only ~30 stalls, so a CTA runs them L
// batches at a time:
//   1. plan: the entries that finish inside the window release their
//      successors in the blocker counts (global atomics, undone on a stall);
//      a released path starts at t_j = 1 + the latest finish among its
//      blockers in the window, found by a second pass over the finishers'
//      successor lists against a shared-memory hash of the released ids.
//      Released paths that also finish inside the window cascade in further
//      rounds.  A few parallel passes per window instead of one dependent
//      release per batch.
//   2. replay: the window's batches in shared memory, batch by batch, every
//      entry's state in registers: each entry active at t claims its next
//      vertex in the occupancy bitmap; a claim that finds the bit set (a token
//      there before the batch, or a second claimer) is a stall at t, which
//      ends the verified prefix.  Otherwise the batch is applied.  A verified
//      prefix is exactly the literal batches (an entry moves iff it is ready
//      and its next vertex is free and unclaimed, batching.cpp:109-136).
//   3. commit: finishes at or after the stall are undone (blocker counts +1),
//      releases at offsets past it are dropped, the live entries are
//      compacted; the stalled batch then runs literally (minimum id per
//      contended destination, batching.cpp:112-113) with an immediate release.
// When the ready set drops to <= 32 (or outgrows shared memory) the ready set
// goes to the warp kernel (batching.cu) exactly like batch_wide.cu's hand-off.

#include <algorithm>
#include <climits>

#include "batching.cuh"
#include "common.cuh"

namespace rb {

// counters of the window kernel (experiments: -DRECON_BATCH_PROF)
// [0] windows [1] stalled windows [2] overflowed plans [3] literal batches
// [4] batches [5] plan cycles [6] replay cycles [7] instances [8] finishers
// [9] plan rounds [10] other cycles (literal batches) [11] commit cycles
// [12] plan: finisher scan [13] pass 1 [14] pass 2 [15] pass 3 [16] pass 1's successor ranges
__device__ unsigned long long g_window_prof[20];

namespace {

constexpr int WT = 512;  // threads per CTA
constexpr int NW = WT / 32;
constexpr int EPT = 4;          // entries per thread in the replay: rmax <= EPT * WT
#ifndef RECON_WIN_PC
#define RECON_WIN_PC 8
#endif
constexpr int PC = RECON_WIN_PC;  // successors per piece (a thread's loads, then its decrements, in flight)
// release offsets through a per-path tag array raised (red.max) with each
// decrement, instead of a second pass against a shared hash of the released
// ids (measured equal; experiments: -DRECON_WIN_TMAX=1)
#ifndef RECON_WIN_TMAX
#define RECON_WIN_TMAX 0
#endif
constexpr bool TMAX = RECON_WIN_TMAX;
constexpr int LMAX = 128;       // window length cap (offsets fit a byte)
constexpr int LINIT = 16;
constexpr int32_t VMIN_EMPTY = 0x7f7f7f7f;

__device__ __forceinline__ int wvtx(int H, int k, int xs, int ys, int xt, int yt) {
    const int dx = abs(xt - xs);
    if (k <= dx) return (xs + (xt > xs ? k : -k)) * H + ys;
    const int m = k - dx;
    return xt * H + ys + (yt > ys ? m : -m);
}

__device__ __forceinline__ int rec_vtx(int H, const int4 &r, int k) {
    return wvtx(H, k, r.z & 0xffff, r.z >> 16, r.w & 0xffff, r.w >> 16);
}

__device__ __forceinline__ int rec_len(const int4 &p) {  // from a path record {src, tgt, ...}
    return abs((p.y & 0xffff) - (p.x & 0xffff)) + abs((p.y >> 16) - (p.x >> 16));
}

struct WinLayout {
    int64_t occ, rec, base, st, total;
};

__host__ __device__ inline int64_t al16(int64_t x) { return (x + 15) / 16 * 16; }

__host__ __device__ inline WinLayout win_layout(int64_t nwb, int rmax) {
    WinLayout L;
    int64_t o = 0;
    L.occ = o;
    o = al16(o + nwb * 4);
    L.rec = o;  // 2 buffers each
    o = al16(o + (int64_t)rmax * 16 * 2);
    L.base = o;
    o = al16(o + (int64_t)rmax * 4 * 2);
    L.st = o;
    o = al16(o + (int64_t)rmax * 2);
    L.total = o;
    return L;
}

// one ready list: records {pid, k | len << 16, src x|y<<16, tgt x|y<<16},
// move bases, start offsets inside the current window
struct WinBufs {
    int4 *rec;
    int *base;
    unsigned char *st;
};

__global__ void __launch_bounds__(WT, 2) batch_window_kernel(PipelineArgs a, int rmax) {
    extern __shared__ __align__(16) unsigned char wsm[];
    __shared__ int s_cnt, s_nf, s_ovf, s_nacc, s_contend, s_maxfin, s_nx;
    __shared__ unsigned long long s_left;
    const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
    const int W = a.W, H = a.H;
    const int64_t S = (int64_t)W * a.k, WH = (int64_t)W * H, nwb = (WH + 31) / 32;
    const WinLayout Lo = win_layout(nwb, rmax);
    uint32_t *occ = (uint32_t *)(wsm + Lo.occ);
    auto bufs = [&](int q) {
        return WinBufs{(int4 *)(wsm + Lo.rec) + q * rmax, (int *)(wsm + Lo.base) + q * rmax, wsm + Lo.st + q * rmax};
    };
    // instances taken one at a time from a counter: CTAs that drew short wide
    // phases take more, so the kernel's tail is one instance, not a wave
    __shared__ int s_inst;
    for (;;) {
        __syncthreads();  // (the previous instance's shared state is read no more)
        if (tid == 0) s_inst = atomicAdd(a.wnext, 1);
        __syncthreads();
        const int inst = s_inst;
        if (inst >= a.count) break;
        int64_t *wst = a.wstate + (int64_t)inst * 4;
        if (a.solve_status[inst] != 0) {
            if (tid == 0) wst[0] = 0;  // the warp kernel reports the solve status
            continue;
        }
        const int64_t o = (int64_t)inst * S;
        const int P = a.path_count[inst];
        const int64_t *mbase = a.mbase + o, *soff = a.soff + o;
        const int64_t moves_total = mbase[P] - mbase[0], e0 = soff[0];
        if (moves_total > a.move_stride || moves_total >= INT_MAX) {
            if (tid == 0) wst[0] = 0;  // the warp kernel reports the capacity status
            continue;
        }
        int32_t *blk = a.indeg + o;
        // the blocker counts as u16 pairs while the kernel runs (half the
        // random-access footprint: the counts of the ~300 instances in flight
        // then stay in L2); unpacked into blk for the warp kernel at the end
        uint32_t *b16 = (uint32_t *)(a.mto + o);
        uint32_t *tmax = (uint32_t *)(a.mem + o);  // TMAX: window id << 8 | latest blocker finish offset
        int32_t *mb = a.move_batch + (int64_t)inst * a.move_stride;
        const int4 *prec = a.prec + (int64_t)inst * (S + 1);  // path records (batching.cu prec_kernel)
        int4 *stg = a.rec2 + o;                               // hand-off staging (and overflow past rmax)
        int32_t *stb = a.rb2 + o;
        const int32_t *succ = a.succ + e0;
        const int32_t *slen = a.slen ? a.slen + o : nullptr;  // list lengths (else up to the next list)
        int32_t *vmin = a.vmin + (int64_t)inst * WH;

#ifdef RECON_BATCH_PROF
        unsigned long long wp[20] = {};
        long long wt = clock64();
#define WINPROF(i)                        \
    do {                                  \
        const long long t_ = clock64();   \
        wp[i] += t_ - wt;                 \
        wt = t_;                          \
    } while (0)
#define WINCOUNT(i, v) (wp[i] += (v))
#else
#define WINPROF(i) (void)0
#define WINCOUNT(i, v) (void)0
#endif
        // appends entry i of list X (shared memory, or the staging area past rmax)
        auto put = [&](const WinBufs &X, int i, int4 r, int base, int st) {
            if (i < rmax) {
                X.rec[i] = r;
                X.base[i] = base;
                X.st[i] = (unsigned char)st;
            } else {
                stg[i] = r;
                stb[i] = base;
                s_ovf = 1;
            }
        };

        // ---- ready set at batch 0 (read-only: on a bail-out the warp kernel
        // starts from scratch)
        if (tid == 0) {
            s_cnt = 0;
            s_ovf = 0;
            s_left = 0;
        }
        __syncthreads();
        {
            const WinBufs A0 = bufs(0);
            long long myleft = 0;
            int zero_len = 0;
            for (int p = tid; p < P; p += WT) {
                const int4 r = prec[p];
                const int len = rec_len(r);
                myleft += len;
                if (TMAX) tmax[p] = 0u;
                if (len == 0) {
                    zero_len = 1;  // zero-length paths: the warp kernel's init releases them
                } else if (blk[p] == 0) {
                    put(A0, atomicAdd(&s_cnt, 1), make_int4(p, len << 16, r.x, r.y), r.z, 0);
                }
            }
            for (int w = tid; w < (P + 1) / 2; w += WT) {
                const int lo = blk[2 * w], hi = 2 * w + 1 < P ? blk[2 * w + 1] : 0;
                if (lo > 0xffff || hi > 0xffff) zero_len = 1;  // (counts past u16: the warp kernel)
                b16[w] = (uint32_t)lo | (uint32_t)hi << 16;
            }
            if (zero_len) s_ovf = 1;
            if (TMAX) __threadfence();
            myleft = warp_sum64(myleft);
            if (lane == 0) atomicAdd(&s_left, (unsigned long long)myleft);
            for (int64_t w = tid; w < nwb; w += WT) occ[w] = a.occ[(int64_t)inst * nwb + w];
        }
        __syncthreads();
        int R = s_cnt;
        long long left = (long long)s_left;
        if (s_ovf || R <= 32 || left == 0) {
            if (tid == 0) wst[0] = 0;
            __syncthreads();
            continue;
        }
        // release hash of a plan (in B's move bases, free until the commit):
        // hk[hcap] = (pid + 1) << 8 | latest blocker finish offset, keyed by
        // the released ids, and a bit filter of them (pass 2 skips the
        // successors that were not released without probing)
        int hb = 4;
        while (3 * (2 << hb) / 2 <= rmax) ++hb;
        const int hbits = hb, hcap = 1 << hb, fmask = hcap * 16 - 1;
        uint32_t *hk = nullptr, *filt = nullptr;
        auto hslot = [&](int v) { return ((unsigned)v * 2654435761u) >> (32 - hbits); };
        auto fbit = [&](int v) { return ((unsigned)v * 0x85ebca6bu >> 7) & (unsigned)fmask; };
        auto hfind = [&](int v) -> int {
            for (unsigned h = hslot(v);; h = (h + 1) & (unsigned)(hcap - 1)) {
                const uint32_t x = hk[h];
                if (x == 0u) return -1;
                if ((x >> 8) == (uint32_t)v + 1) return (int)h;
            }
        };
        // Passes 1 and 2 run a thread per finisher over pieces of PC successors
        // (a warp per finisher spends most of its instructions gathering
        // chunks); the pieces past a finisher's first go to the list xl and
        // are taken by all threads after a barrier.
        //
        // pass 1 of a release round: the successors of finishers F[f0, f1)
        // {pid, finish offset, q0, qn} lose a blocker (global counts, issued
        // back to back); a path whose count reaches 0 is appended to A as a
        // placeholder {pid} (and in a plan, keyed into the release hash)
        auto dec_piece = [&](const WinBufs &A, int q0, int lo, int hi, bool plan, int pmax, uint32_t tag) {
            int v[PC], r[PC];
#pragma unroll
            for (int c = 0; c < PC; ++c) v[c] = lo + c < hi ? __ldg(succ + q0 + lo + c) : -1;
            if (TMAX && plan)
#pragma unroll
                for (int c = 0; c < PC; ++c)
                    if (v[c] >= 0) asm volatile("red.global.max.u32 [%0], %1;" ::"l"(tmax + v[c]), "r"(tag) : "memory");
#pragma unroll
            for (int c = 0; c < PC; ++c)
                r[c] = (int)atom_add_if(v[c] >= 0, &b16[max(v[c], 0) >> 1], (v[c] & 1) ? 0xffff0000u : 0xffffffffu);
#pragma unroll
            for (int c = 0; c < PC; ++c) {
                if (v[c] < 0 || ((unsigned)r[c] >> ((v[c] & 1) * 16) & 0xffffu) != 1u) continue;
                const int i = atomicAdd(&s_cnt, 1);
                if (i >= pmax) {
                    s_ovf = 1;
                } else if (i >= rmax) {  // (literal batch) past shared memory: the staging area
                    stg[i].x = v[c];
                    s_ovf = 1;
                } else {
                    A.rec[i].x = v[c];
                    if (plan && !TMAX) {
                        const unsigned fb = fbit(v[c]);
                        atomicOr(&filt[fb >> 5], 1u << (fb & 31));
                        unsigned h = hslot(v[c]);
                        while (atomicCAS(&hk[h], 0u, (uint32_t)(v[c] + 1) << 8) != 0u) h = (h + 1) & (unsigned)(hcap - 1);
                    }
                }
            }
        };
        // pass 2 piece: the released successors' latest blocker finish
        auto max_piece = [&](int q0, int lo, int hi, int fin) {
            int v[PC];
#pragma unroll
            for (int c = 0; c < PC; ++c) v[c] = lo + c < hi ? __ldg(succ + q0 + lo + c) : -1;
#pragma unroll
            for (int c = 0; c < PC; ++c) {
                if (v[c] < 0) continue;
                const unsigned fb = fbit(v[c]);
                if (!(filt[fb >> 5] >> (fb & 31) & 1u)) continue;
                const int h = hfind(v[c]);
                if (h >= 0) atomicMax(&hk[h], ((uint32_t)(v[c] + 1) << 8) | (uint32_t)fin);
            }
        };
        // runs op(f, q0, lo, hi) over the pieces of finishers F[f0, f1):
        // first pieces inline, the rest from xl[0, xcap) after a barrier
        // (or inline when xl is full)
        auto for_pieces = [&](int4 *F, int f0, int f1, uint32_t *xl, int xcap, bool ranges, auto op) {
            if (tid == 0) s_nx = 0;
            __syncthreads();
            for (int f = f0 + tid; f < f1; f += WT) {
#ifdef RECON_BATCH_PROF
                const long long pt0 = clock64();
#endif
                int q0, qn;
                if (ranges) {
                    const int pid = F[f].x;
                    q0 = __ldg(&prec[pid].w);
                    qn = slen ? __ldg(slen + pid) : __ldg(&prec[pid + 1].w) - q0;
                    F[f].z = q0;
                    F[f].w = qn;
                    if (qn > PC) prefetch_l2(succ + q0 + PC, (qn - PC) * 4);  // (the pieces taken after the barrier)
                } else {
                    q0 = F[f].z;
                    qn = F[f].w;
                }
#ifdef RECON_BATCH_PROF
                const long long pt1 = clock64();
#endif
                op(f, q0, 0, min(qn, PC));
#ifdef RECON_BATCH_PROF
                if (ranges && tid == 0) {
                    wp[17] += (unsigned long long)(pt1 - pt0);
                    wp[18] += (unsigned long long)(clock64() - pt1);
                    wp[19] += 1;
                }
#endif
                for (int pc = 1; pc * PC < qn; ++pc) {
                    const int x = atomicAdd(&s_nx, 1);
                    if (x < xcap && pc < 256)
                        xl[x] = (uint32_t)f << 8 | (uint32_t)pc;
                    else
                        op(f, q0, pc * PC, min(qn, (pc + 1) * PC));
                }
            }
            __syncthreads();
            const int nx = min(s_nx, xcap);
            for (int x = tid; x < nx; x += WT) {
                const int f = (int)(xl[x] >> 8), pc = (int)(xl[x] & 255u);
                const int q0 = F[f].z, qn = F[f].w;
                op(f, q0, pc * PC, min(qn, (pc + 1) * PC));
            }
        };
        auto release_pass1 = [&](const WinBufs &A, int4 *F, int f0, int f1, bool plan, int pmax, uint32_t *xl, int xcap,
                                 uint32_t wtag) {
            for_pieces(F, f0, f1, xl, xcap, true,
                       [&](int f, int q0, int lo, int hi) { dec_piece(A, q0, lo, hi, plan, pmax, wtag | (uint32_t)F[f].y); });
            if (TMAX && plan) __threadfence();  // the raises before pass 3 reads them (after a barrier)
        };
        // pass 2 (plan): over all finishers so far (a path released in this
        // round may have blockers from earlier rounds)
        auto release_pass2 = [&](int4 *F, int f1, uint32_t *xl, int xcap) {
            for_pieces(F, 0, f1, xl, xcap, false, [&](int f, int q0, int lo, int hi) { max_piece(q0, lo, hi, F[f].y); });
        };
        // pass 3: placeholders A[i0, i1) become entries; start offset = 1 +
        // latest blocker finish in the window (plan), or 1 (literal batch);
        // plan releases that finish inside [0, L) join F (the cascade)
        auto release_pass3 = [&](const WinBufs &A, int4 *F, int i0, int i1, bool plan, int L, uint32_t wtag) {
            for (int i = i0 + tid; i < i1; i += WT) {
                const int j = i < rmax ? A.rec[i].x : stg[i].x;
                const int4 pr = __ldg(prec + j);
                const int len = rec_len(pr);
                int tj = 1;
                if (plan && TMAX) {
                    const unsigned tm = __ldcg(tmax + j);
                    RB_CHECK((tm & ~0xffu) == wtag, "window: release tag of another window");
                    tj = (int)(tm & 0xffu) + 1;
                } else if (plan) {
                    const int h = hfind(j);
                    RB_CHECK(h >= 0, "window: released path missing from the hash");
                    tj = (int)(hk[h] & 0xffu) + 1;
                }
                RB_CHECK(tj <= L, "window: release past the window");
                if (i >= rmax) {
                    stg[i] = make_int4(j, len << 16, pr.x, pr.y);
                    stb[i] = pr.z;
                    continue;
                }
                A.rec[i] = make_int4(j, len << 16, pr.x, pr.y);
                A.base[i] = pr.z;
                A.st[i] = (unsigned char)tj;
                if (plan) {
                    atomicMax(&s_maxfin, tj + len - 1);
                    if (tj + len - 1 < L) {
                        const int fi = atomicAdd(&s_nf, 1);
                        if (fi < rmax)
                            F[fi] = make_int4(j, tj + len - 1, 0, 0);
                        else
                            s_ovf = 1;
                    }
                }
            }
        };
        // undoes the decrements of the processed finishers F[0, nf) with
        // finish offset >= from
        auto undo = [&](const int4 *F, int nf, int from) {
            for (int f = warp; f < nf; f += NW) {
                const int4 fr = F[f];
                if (fr.y < from) continue;
                for (int j = lane; j < fr.w; j += 32) {
                    const int v = __ldg(succ + fr.z + j);
                    if (v >= 0) atomicAdd(&b16[v >> 1], (v & 1) ? 0x10000u : 1u);
                }
            }
        };
        // the ready list A[0, n) (entries past rmax in the staging area) as
        // id-ranked records for the warp kernel, finished entries dropped
        auto handoff = [&](const WinBufs &A, int n) {
            __syncthreads();
            for (int i = tid; i < min(n, rmax); i += WT) {
                stg[i] = A.rec[i];
                stb[i] = A.base[i];
            }
            __threadfence();
            if (tid == 0) s_cnt = 0;
            __syncthreads();
            int kept = 0;
            for (int i = tid; i < n; i += WT) {
                const int4 x = __ldcg(&stg[i]);
                if ((x.y & 0xffff) >= (x.y >> 16)) continue;
                int rank = 0;
                for (int j = 0; j < n; ++j) {
                    const int4 y = __ldcg(&stg[j]);
                    rank += (y.y & 0xffff) < (y.y >> 16) && y.x < x.x;
                }
                a.rec[o + rank] = x;
                a.rb[o + rank] = __ldcg(&stb[i]);
                ++kept;
            }
            kept = warp_sum(kept);
            if (lane == 0 && kept) atomicAdd(&s_cnt, kept);
            for (int64_t w = tid; w < nwb; w += WT) a.occ[(int64_t)inst * nwb + w] = occ[w];
            __syncthreads();
        };

        int cur = 0, nb = 0, status = RECON_OK, L = LINIT;
        unsigned wid = 0;  // plan id (TMAX tags; < 2^24)
        bool hand = false;  // (uniform) hand the ready set to the warp kernel
        int hand_n = 0;
        for (;;) {
            WinBufs A = bufs(cur), B = bufs(cur ^ 1);
            int4 *F = B.rec;  // finisher list {pid, finish offset, q0, qn}
            // ---------------- 1. plan the window [0, L)
            WINPROF(10);
            const int R0 = R;
            if (tid == 0) {
                s_cnt = R;
                s_nf = 0;
                s_ovf = 0;
                s_nacc = 0;
                s_maxfin = -1;
            }
            __syncthreads();
            for (int b0 = 0; b0 < R; b0 += WT) {  // (warp-uniform trips: warp-aggregated appends)
                const int e = b0 + tid;
                bool f = false;
                int4 fr = make_int4(0, 0, 0, 0);
                if (e < R) {
                    const int4 r = A.rec[e];
                    fr.x = r.x;
                    fr.y = (int)A.st[e] + (r.y >> 16) - (r.y & 0xffff) - 1;
                    f = fr.y < L;
                }
                const unsigned fm = __ballot_sync(FULL, f);
                int fb = 0;
                if (lane == 0 && fm) fb = atomicAdd(&s_nf, __popc(fm));
                fb = __shfl_sync(FULL, fb, 0);
                if (f) F[fb + __popc(fm & lanemask_lt())] = fr;
                const int mf = __reduce_max_sync(FULL, e < R ? fr.y : -1);
                if (lane == 0) atomicMax(&s_maxfin, mf);
            }
            __syncthreads();
            int f0 = 0, f1 = s_nf, ovf = 0;
            __syncthreads();
            ++wid;
            const int pmax = TMAX ? rmax : min(rmax, R + hcap * 3 / 4);  // (hash load <= 3/4)
            hk = (uint32_t *)B.base;
            filt = hk + hcap;
            uint32_t *xl = TMAX ? hk : filt + hcap / 2;  // extra pieces (the rest of B's move bases)
            const int xcap = TMAX ? rmax : rmax - hcap - hcap / 2;
            if (!TMAX)
                for (int h = tid; h < hcap + hcap / 2; h += WT) hk[h] = 0u;
            __syncthreads();
            WINPROF(12);
            while (f0 < f1) {
                WINCOUNT(9, 1);
                const int i0 = s_cnt;
                release_pass1(A, F, f0, f1, true, pmax, xl, xcap, wid << 8);
                __syncthreads();
                WINPROF(13);
                const int i1 = min(s_cnt, pmax);
                if (s_ovf) {
                    ovf = 1;
                    f0 = f1;
                    break;
                }
                if (i1 > i0) {
                    if (!TMAX) {
                        release_pass2(F, f1, xl, xcap);
                        __syncthreads();
                    }
                    WINPROF(14);
                    release_pass3(A, F, i0, i1, true, L, wid << 8);
                    __syncthreads();
                    WINPROF(15);
                }
                f0 = f1;
                f1 = min(s_nf, rmax);
                ovf = s_ovf;
                __syncthreads();
                if (ovf) break;
            }
            const int Rw = s_cnt;
            const int Lrun = min(L, s_maxfin + 1);  // no entry is active from Lrun on
            WINPROF(5);
            WINCOUNT(8, f0);
            if (ovf) {
                // the releases outgrow the list: undo them all, halve the window
                undo(F, f0, 0);
                __syncthreads();
                WINCOUNT(2, 1);
                if (L == 1) {
                    hand = true;
                    hand_n = R;
                    break;
                }
                L = max(1, L / 2);
                continue;
            }
            // ---------------- 2. replay [0, L) in shared memory
            int t_exec = Lrun, moves = 0;  // (then: the window's moves)
            {
                // per entry: vertex, claimed vertex, and its batch times in
                // the window: start | end << 8 | turn << 16 | right << 24 | up << 25
                // (it moves in batches [start, end), horizontally before
                // `turn`); slots past the list are skipped a warp at a time
                int cur_v[EPT], to[EPT];
                unsigned pk[EPT];
                const int wb = tid & ~31;
                const int nsl = Rw > wb ? min(EPT, (Rw - wb + WT - 1) / WT) : 0;
#pragma unroll
                for (int i = 0; i < EPT; ++i) {
                    const int e = tid + i * WT;
                    cur_v[i] = to[i] = 0;
                    pk[i] = 0;  // start = end = 0: never active
                    if (e < Rw) {
                        const int4 r = A.rec[e];
                        const int xs = r.z & 0xffff, ys = r.z >> 16, xt = r.w & 0xffff, yt = r.w >> 16;
                        const int k = r.y & 0xffff, len = r.y >> 16, s0 = A.st[e];
                        const int en = min(s0 + len - k, 255), tt = min(s0 + max(abs(xt - xs) - k, 0), 255);
                        pk[i] = (unsigned)s0 | (unsigned)en << 8 | (unsigned)tt << 16 | (unsigned)(xt > xs) << 24 |
                                (unsigned)(yt > ys) << 25;
                        cur_v[i] = wvtx(H, k, xs, ys, xt, yt);
                    }
                }
                // One barrier per batch: batch t's vacated vertices are
                // released in the same phase as batch t+1's claims, so a claim
                // can find a vertex still held by an entry that left it in t
                // (an entry following another, rare: ~1e-4 of the moves).
                // Such failures get a second chance after the barrier, when
                // every release of t is done; only a claim that fails again
                // (occupied before the batch, or claimed twice) is a stall.
                unsigned pend = 0;  // entries that moved in the previous batch
                for (int t = 0; t < Lrun; ++t) {
                    bool fail = false;
                    unsigned claimed = 0, act = 0;
#pragma unroll
                    for (int i = 0; i < EPT; ++i)
                        if (pend >> i & 1u) {
                            atomicAnd(&occ[cur_v[i] >> 5], ~(1u << (cur_v[i] & 31)));
                            cur_v[i] = to[i];
                        }
#pragma unroll
                    for (int i = 0; i < EPT; ++i) {
                        if (i >= nsl) break;
                        if ((int)(pk[i] & 0xffu) <= t && t < (int)(pk[i] >> 8 & 0xffu)) {
                            act |= 1u << i;
                            const int step = t < (int)(pk[i] >> 16 & 0xffu) ? ((pk[i] >> 24 & 1u) ? H : -H)
                                                                             : ((pk[i] >> 25 & 1u) ? 1 : -1);
                            to[i] = cur_v[i] + step;
                            const uint32_t bit = 1u << (to[i] & 31);
                            if (atomicOr(&occ[to[i] >> 5], bit) & bit)
                                fail = true;
                            else
                                claimed |= 1u << i;
                        }
                    }
                    if (__syncthreads_or(fail)) {
                        fail = false;
#pragma unroll
                        for (int i = 0; i < EPT; ++i)
                            if ((act & ~claimed) >> i & 1u) {
                                const uint32_t bit = 1u << (to[i] & 31);
                                if (atomicOr(&occ[to[i] >> 5], bit) & bit)
                                    fail = true;
                                else
                                    claimed |= 1u << i;
                            }
                        if (__syncthreads_or(fail)) {
                            // a stall at t: t is not applied (its claims are undone)
#pragma unroll
                            for (int i = 0; i < EPT; ++i)
                                if (claimed >> i & 1u) atomicAnd(&occ[to[i] >> 5], ~(1u << (to[i] & 31)));
                            t_exec = t;
                            claimed = 0;
                        }
                    }
                    pend = claimed;
                    if (t_exec == t) break;
                }
#pragma unroll
                for (int i = 0; i < EPT; ++i)
                    if (pend >> i & 1u) atomicAnd(&occ[cur_v[i] >> 5], ~(1u << (cur_v[i] & 31)));
                // each entry moved in every batch of [start, min(end, t_exec));
                // the window's schedule: its moves are one run of consecutive
                // slots and batch indices, stored 16 bytes at a time where aligned
                int moved[EPT];
#pragma unroll
                for (int i = 0; i < EPT; ++i) {
                    const int e = tid + i * WT;
                    moved[i] = max(0, min(t_exec, (int)(pk[i] >> 8 & 0xffu)) - (int)(pk[i] & 0xffu));
                    moves += moved[i];
                    if (e >= Rw) continue;
                    const int klo = A.rec[e].y & 0xffff;
                    const int n = moved[i], b0 = nb + (int)(pk[i] & 0xffu);
                    int32_t *d = mb + A.base[e] + klo;
                    int j = 0;
                    for (; j < n && ((uintptr_t)(d + j) & 15u); ++j) __stcs(d + j, b0 + j);
                    for (; j + 4 <= n; j += 4)
                        __stcs(reinterpret_cast<int4 *>(d + j), make_int4(b0 + j, b0 + j + 1, b0 + j + 2, b0 + j + 3));
                    for (; j < n; ++j) __stcs(d + j, b0 + j);
                }
                moves = warp_sum(moves);
                if (lane == 0 && moves) atomicAdd(&s_nacc, moves);
                __syncthreads();
                moves = s_nacc;
                WINPROF(6);
                WINCOUNT(0, 1);
                if (t_exec < L) {
                    WINCOUNT(1, t_exec < Lrun);
                    undo(F, f1, t_exec);  // (past Lrun: nothing to undo)
                }
                if (tid == 0) s_cnt = 0;
                __syncthreads();
                // ---------------- 3. commit: live entries (releases at or
                // before t_exec) to the other list
#pragma unroll
                for (int i = 0; i < EPT; ++i) {
                    const int e = tid + i * WT;
                    int4 r = make_int4(0, 0, 0, 0);
                    if (e < Rw) {
                        r = A.rec[e];
                        r.y += moved[i];
                    }
                    const bool keep = e < Rw && (r.y & 0xffff) < (r.y >> 16) && (int)(pk[i] & 0xffu) <= t_exec;
                    const unsigned km = __ballot_sync(FULL, keep);
                    int kb = 0;
                    if (lane == 0 && km) kb = atomicAdd(&s_cnt, __popc(km));
                    kb = __shfl_sync(FULL, kb, 0);
                    if (keep) {
                        const int j = kb + __popc(km & lanemask_lt());
                        B.rec[j] = r;
                        B.base[j] = A.base[e];
                        B.st[j] = 0;
                        // a finisher of the next window (if L holds): its successor
                        // range's record into L2 for the plan's first load
                        if ((r.y >> 16) - (r.y & 0xffff) <= L) {
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(prec + r.x));
                            if (slen) asm volatile("prefetch.global.L2 [%0];" ::"l"(slen + r.x));
                        }
                    }
                }
            }
            __syncthreads();
            left -= moves;
            nb += t_exec;
            WINCOUNT(4, t_exec);
            WINPROF(11);
            R = s_cnt;
            cur ^= 1;
            if (left == 0) break;
            if (t_exec < Lrun) {
                // ---------------- the stalled batch, literally
                A = bufs(cur);
                B = bufs(cur ^ 1);
                F = B.rec;
                unsigned char *fl = B.st;  // 1 candidate, 2 winner of a contended destination
                if (tid == 0) {
                    s_contend = 0;
                    s_nf = 0;
                    s_nacc = 0;
                    s_cnt = R;
                    s_ovf = 0;
                }
                for (int e = tid; e < R; e += WT) {
                    const int4 r = A.rec[e];
                    const int to = rec_vtx(H, r, (r.y & 0xffff) + 1);
                    fl[e] = ((occ[to >> 5] >> (to & 31)) & 1u) ? 0 : 1;  // batching.cpp:111
                }
                __syncthreads();
                for (int e = tid; e < R; e += WT) {
                    if (!fl[e]) continue;
                    const int4 r = A.rec[e];
                    const int to = rec_vtx(H, r, (r.y & 0xffff) + 1);
                    if (atomicOr(&occ[to >> 5], 1u << (to & 31)) & (1u << (to & 31))) s_contend = 1;
                }
                __syncthreads();
                const bool contend = s_contend != 0;
                if (contend) {  // minimum id per contended destination (batching.cpp:112-113)
                    for (int e = tid; e < R; e += WT)
                        if (fl[e]) {
                            const int4 r = A.rec[e];
                            atomicMin(&vmin[rec_vtx(H, r, (r.y & 0xffff) + 1)], r.x);
                        }
                    __threadfence();
                    __syncthreads();
                    for (int e = tid; e < R; e += WT)
                        if (fl[e]) {
                            const int4 r = A.rec[e];
                            if (__ldcg(&vmin[rec_vtx(H, r, (r.y & 0xffff) + 1)]) == r.x) fl[e] = 2;
                        }
                    __syncthreads();
                    for (int e = tid; e < R; e += WT)
                        if (fl[e]) {
                            const int4 r = A.rec[e];
                            vmin[rec_vtx(H, r, (r.y & 0xffff) + 1)] = VMIN_EMPTY;
                        }
                }
                int nacc = 0;
                for (int b0 = 0; b0 < R; b0 += WT) {
                    const int e = b0 + tid;
                    bool fin = false;
                    int pid = 0;
                    if (e < R && fl[e] == (contend ? 2 : 1)) {
                        int4 r = A.rec[e];
                        const int k = r.y & 0xffff;
                        const int fr = rec_vtx(H, r, k);
                        atomicAnd(&occ[fr >> 5], ~(1u << (fr & 31)));
                        __stcs(mb + A.base[e] + k, nb);
                        A.rec[e].y = r.y + 1;
                        ++nacc;
                        fin = k + 1 == (r.y >> 16);
                        pid = r.x;
                    }
                    const unsigned fm = __ballot_sync(FULL, fin);
                    int fb = 0;
                    if (lane == 0 && fm) fb = atomicAdd(&s_nf, __popc(fm));
                    fb = __shfl_sync(FULL, fb, 0);
                    if (fin) F[fb + __popc(fm & lanemask_lt())] = make_int4(pid, 0, 0, 0);
                }
                nacc = warp_sum(nacc);
                if (lane == 0 && nacc) atomicAdd(&s_nacc, nacc);
                __syncthreads();
                const int nacc_all = s_nacc;
                WINCOUNT(3, 1);
                if (nacc_all == 0) {
                    status = RECON_ERR_INPUT;  // batching.cpp:127-128
                    break;
                }
                left -= nacc_all;
                ++nb;
                WINCOUNT(4, 1);
                {
                    const int i0 = s_cnt;
                    release_pass1(A, F, 0, s_nf, false, S, (uint32_t *)B.base, rmax, 0u);
                    __syncthreads();
                    release_pass3(A, F, i0, s_cnt, false, 1, 0u);
                    __syncthreads();
                }
                const int Rl = s_cnt, lovf = s_ovf;
                __syncthreads();
                if (lovf) {
                    hand = true;
                    hand_n = Rl;
                    break;
                }
                if (tid == 0) s_cnt = 0;
                __syncthreads();
                for (int b0 = 0; b0 < Rl; b0 += WT) {
                    const int e = b0 + tid;
                    int4 r = make_int4(0, 0, 0, 0);
                    if (e < Rl) r = A.rec[e];
                    const bool keep = e < Rl && (r.y & 0xffff) < (r.y >> 16);
                    const unsigned km = __ballot_sync(FULL, keep);
                    int kb = 0;
                    if (lane == 0 && km) kb = atomicAdd(&s_cnt, __popc(km));
                    kb = __shfl_sync(FULL, kb, 0);
                    if (keep) {
                        const int j = kb + __popc(km & lanemask_lt());
                        B.rec[j] = r;
                        B.base[j] = A.base[e];
                        B.st[j] = 0;
                    }
                }
                __syncthreads();
                R = s_cnt;
                cur ^= 1;
                if (left == 0) break;
            } else {
                // next window length: double while the releases leave room
                const int nrel = Rw - R0, relcap = TMAX ? rmax - rmax / 8 - R : min(rmax - rmax / 8 - R, hcap * 5 / 8);
                if (L < LMAX && 2 * nrel + 32 < relcap)
                    L = min(LMAX, 2 * L);
                else if (L > 1 && nrel > relcap)
                    L /= 2;
            }
            if (R <= 32) {
                hand = true;
                hand_n = R;
                break;
            }
        }
#ifdef RECON_BATCH_PROF
        if (tid == 0) {
            for (int i = 0; i < 20; ++i)
                if (i != 7) atomicAdd(&g_window_prof[i], wp[i]);
            atomicAdd(&g_window_prof[7], 1ull);
        }
#endif
        // ---- hand-off to the warp kernel, or the instance's result
        if (status == RECON_OK && left > 0) {
            RB_CHECK(hand, "window: unfinished instance without a hand-off");
            for (int p = tid; p < P; p += WT) blk[p] = (int)(b16[p >> 1] >> ((p & 1) * 16) & 0xffffu);
            handoff(bufs(cur), hand_n);
            if (tid == 0) {
                wst[0] = 1;
                wst[1] = nb;
                wst[2] = left;
                wst[3] = s_cnt;
            }
        } else if (tid == 0) {
            wst[0] = 2;
            a.batch_count[inst] = status == RECON_OK ? nb : 0;
            a.status[inst] = status;
            if (a.detail) a.detail[inst] = status == RECON_OK ? 0 : RECON_D_BATCH_NO_PROGRESS;
        }
        __syncthreads();
    }
}

}  // namespace

// largest ready list the window kernel holds in `smem_budget` bytes
bool pipeline_window_config(int W, int H, int64_t smem_budget, int *rmax, size_t *smem) {
    const int64_t nwb = ((int64_t)W * H + 31) / 32;
    for (int r = EPT * WT; r >= 256; r -= 64) {
        const WinLayout L = win_layout(nwb, r);
        if (L.total <= smem_budget) {
            *rmax = r;
            *smem = (size_t)L.total;
            return true;
        }
    }
    return false;
}

cudaError_t launch_batch_window(const PipelineArgs &a, int sms, int rmax, size_t smem, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(batch_window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, batch_window_kernel, WT, smem);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<int64_t>(a.count, (int64_t)sms * std::max(1, per_sm));
    batch_window_kernel<<<grid, WT, smem, st>>>(a, rmax);
    return cudaGetLastError();
}

}  // namespace rb

// experiments: the window kernel's counters (zero unless built with -DRECON_BATCH_PROF)
extern "C" int recon_debug_window_prof(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, rb::g_window_prof, sizeof(rb::g_window_prof)) != cudaSuccess) return -1;
    if (reset) {
        static const unsigned long long z[20] = {};
        if (cudaMemcpyToSymbol(rb::g_window_prof, z, sizeof(z)) != cudaSuccess) return -1;
    }
    return 0;
}
