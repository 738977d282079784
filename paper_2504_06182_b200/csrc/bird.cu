// bird on sm_100a: one CTA per instance.
//
// Reference: /root/reference/proj/src/bird.cpp:12-123.
//
// Column pass (bird.cpp:114-115): every column with surplus >= 0 compacts
// on its own; the events are independent, so warps take them in parallel
// (solve + count, scan, emit + update).  Row pass (bird.cpp:119-120): each
// remaining column, ascending, runs one pooled event whose optional pool is
// every reservoir token of every column at virtual position depth -+ dist
// (build_generalized_instance, bird.cpp:35-46); these events are strictly
// sequential and each is solved CTA-wide (pooled_event below).

#include "grid_common.cuh"

namespace rb {

// OWN events [e0, e1) of the plan, round-robin over warps [w0, nw): solve
// and record a / path count.
__device__ bool own_count_range(const Geo &g, Block &b, int e0, int e1, int w0, int *fail) {
    const int warp = warp_id(), nw = blockDim.x >> 5;
    int16_t *L = b.lists + (size_t)warp * 4 * g.LK;
    for (int e = e0 + (warp - w0); e < e1; e += nw - w0) {
        const int c = b.ev_col[e];
        OwnSolve s;
        if (!own_solve(g, b.dep + (size_t)c * g.wpd, L, -1, s)) {
            if (lane_id() == 0) *fail = 1;
            continue;
        }
        if (lane_id() == 0) {
            b.ev_a[e] = (int16_t)s.a;
            b.ev_count[e] = s.n_right + s.n_left;
        }
        __syncwarp();
    }
    return true;
}

// Re-materializes and emits OWN events [e0, e1) at their offsets; optionally
// applies the column update (bird) and returns parked counts into sigma.
__device__ void own_emit_range(const Geo &g, Block &b, int e0, int e1, int w0, PathOut o, int base_off,
                               bool update, unsigned long long *disp_acc) {
    const int warp = warp_id(), nw = blockDim.x >> 5;
    int16_t *L = b.lists + (size_t)warp * 4 * g.LK;
    long long disp = 0;
    for (int e = e0 + (warp - w0); e < e1; e += nw - w0) {
        const int c = b.ev_col[e];
        OwnSolve s;
        if (!own_solve(g, b.dep + (size_t)c * g.wpd, L, b.ev_a[e], s)) continue;
        disp += own_emit(g, c, s, L, o, base_off + b.ev_off[e], e);
        if (update) {
            const int parked = own_update(g, b.dep + (size_t)c * g.wpd, s, L);
            if (lane_id() == 0) {
                b.sigma[c] = parked;
                b.solved[c] = 1;
            }
        }
        __syncwarp();
    }
    if (lane_id() == 0 && disp) atomicAdd(disp_acc, (unsigned long long)disp);
}

// exclusive scan of ev_count[e0, e1) into ev_off (relative to e0); returns total (warp 0 only)
__device__ int scan_counts(Block &b, int e0, int e1) {
    int run = 0;
    for (int i0 = e0; i0 < e1; i0 += 32) {
        const int i = i0 + lane_id();
        const int v = i < e1 ? b.ev_count[i] : 0;
        int tot;
        const int ex = warp_excl_scan(v, &tot);
        if (i < e1) b.ev_off[i] = run + ex;
        run += tot;
    }
    return run;
}

// --------------------------------------------------------------------------
// CTA-level pooled event (bird row pass, bird.cpp:35-46, 64-100)
//
// The optional pool of column c is every reservoir token of every column; a
// token of column x at depth d sits at virtual level d - |x-c| (top side) or
// d + |x-c| (bottom side), virtual_line.cpp:65-68.  Levels are scanned in
// 64-level windows outward from the band.  Inside a window the 2*dist+1
// columns that can reach it are "slots" in group order (own column, then
// dist 1 left, dist 1 right, ...; virtual_line.cpp:112-118); 32 slots x 64
// levels form a bit block that one warp transposes with shuffles, giving per
// level the ballot of slots holding a token (-> per-level counts and each
// token's rank inside its level).  Top and bottom windows are scanned by two
// warp groups at once, and scanning stops as soon as the split a is pinned
// down (Delta(a) is known on a contiguous range that brackets the
// minimiser), instead of collecting `holes` tokens per side.
// --------------------------------------------------------------------------

__device__ __forceinline__ int slot_col(int c, int gslot, int W) {
    if (gslot == 0) return c;
    const int dl = (gslot + 1) >> 1;
    const int x = (gslot & 1) ? c - dl : c + dl;
    return (x >= 0 && x < W) ? x : -1;
}

struct PooledScratch {
    int16_t *otop, *obot;  // [LK] virtual levels of the k-th nearest optional token per side (1-based)
    int *lvl_t, *lvl_b;    // [LT], [LB]: count << 16 | tokens at nearer levels (saturating)
    uint32_t *bal;         // [2][nchunk][64] transposed slot words of the current window per side
    int *scal;             // scalars
};

// 32 slots x 64 levels: lane L receives the slot masks of levels L and L+32
__device__ __forceinline__ void transpose64(uint64_t word, uint32_t &t_lo, uint32_t &t_hi) {
    uint32_t a = (uint32_t)word, b = (uint32_t)(word >> 32);
    const int lane = lane_id();
#pragma unroll
    for (int j = 16; j >= 1; j >>= 1) {
        const uint32_t m = j == 16 ? 0x0000FFFFu : (j == 8 ? 0x00FF00FFu : (j == 4 ? 0x0F0F0F0Fu : (j == 2 ? 0x33333333u : 0x55555555u)));
        const uint32_t ya = __shfl_xor_sync(FULL, a, j), yb = __shfl_xor_sync(FULL, b, j);
        if (lane & j) {
            a = (a & ~m) | ((ya & ~m) >> j);
            b = (b & ~m) | ((yb & ~m) >> j);
        } else {
            a = (a & m) | ((ya & m) << j);
            b = (b & m) | ((yb & m) << j);
        }
    }
    t_lo = a;
    t_hi = b;
}

// token word of a slot: bit i = a reservoir token at virtual level V0 + i
__device__ __forceinline__ uint64_t slot_word(const Geo &g, const uint64_t *dep, int c, int gslot, int nslots,
                                              int V0, bool top, int *col_out, int *dist_out, uint64_t wmask) {
    *col_out = -1;
    *dist_out = 0;
    if (gslot >= nslots) return 0ull;
    const int x = slot_col(c, gslot, g.W);
    if (x < 0) return 0ull;
    const int dist = x > c ? x - c : c - x;
    *col_out = x;
    *dist_out = dist;
    const uint64_t *m = dep + (size_t)x * g.wpd;
    if (top) {  // depth = v + dist < lo
        const int start = V0 + dist;
        const uint64_t w = extract64(m, g.wpd, start);
        const int nvalid = g.lo - start;
        if (nvalid <= 0) return 0ull;
        return (nvalid >= 64 ? w : (w & ((1ull << nvalid) - 1ull))) & wmask;
    }
    const int start = V0 - dist;  // depth = v - dist > hi
    const uint64_t w = extract64(m, g.wpd, start);
    const int skip = g.hi + 1 - start;
    if (skip >= 64) return 0ull;
    return (skip <= 0 ? w : (w & ~((1ull << skip) - 1ull))) & wmask;
}


// Windows cover level indices [win_lo(w), win_hi(w)): the first BIRD_W0
// levels, then 64 at a time.
#ifndef BIRD_W0
#define BIRD_W0 64
#endif
__device__ __forceinline__ int win_hi(int w) { return BIRD_W0 + 64 * w; }
__device__ __forceinline__ int win_lo(int w) { return w == 0 ? 0 : win_hi(w - 1); }
__device__ __forceinline__ int win_of(int li) { return li < BIRD_W0 ? 0 : (li - BIRD_W0) / 64 + 1; }
__device__ __forceinline__ int win_V0(const Geo &g, bool top, int w) {
    return top ? g.lo - win_hi(w) : g.hi + 1 + win_lo(w);
}
// slots (columns in group order) that reach levels < lim: distance <= level
__device__ __forceinline__ int win_nslots(const Geo &g, int lim) { return 2 * min(g.W - 1, lim - 1) + 1; }
// window bit i -> level index (0 = nearest the band)
__device__ __forceinline__ int bit_li(bool top, int w, int i) { return top ? win_hi(w) - 1 - i : win_lo(w) + i; }

// bits of window w holding levels <= lim (all of them: lim >= win_hi - 1)
__device__ __forceinline__ uint64_t win_mask(bool top, int w, int lim) {
    const int lo = win_lo(w), n = min(win_hi(w), lim + 1) - lo;  // levels [lo, lo + n)
    if (n <= 0) return 0ull;
    const uint64_t low = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
    const int size = win_hi(w) - lo;
    return top ? low << (size - n) : low;  // top: bit i <-> level win_hi - 1 - i
}

// counts one window of one side with the warps [g0, g0 + gn) of the CTA and
// leaves its transposed slot words in T (as transpose_window would)
__device__ void count_window(const Geo &g, const uint64_t *dep, int c, bool top, int w, int *lvl, uint32_t *T,
                             int g0, int gn) {
    const int warp = warp_id(), lane = lane_id();
    if (warp < g0 || warp >= g0 + gn) return;
    const int V0 = win_V0(g, top, w), nslots = win_nslots(g, win_hi(w)), nch = (nslots + 31) / 32;
    const uint64_t wmask = win_mask(top, w, win_hi(w));
    int acc_lo = 0, acc_hi = 0;
    for (int ch = warp - g0; ch < nch; ch += gn) {
        int col, dist;
        const uint64_t word = slot_word(g, dep, c, ch * 32 + lane, nslots, V0, top, &col, &dist, wmask);
        uint32_t t_lo = 0u, t_hi = 0u;
        if (__any_sync(FULL, word != 0ull)) transpose64(word, t_lo, t_hi);
        T[ch * 64 + lane] = t_lo;
        T[ch * 64 + 32 + lane] = t_hi;
        acc_lo += __popc(t_lo);
        acc_hi += __popc(t_hi);
    }
    if (acc_lo) atomicAdd(&lvl[bit_li(top, w, lane)], acc_lo);  // bits past the window are 0
    if (acc_hi) atomicAdd(&lvl[bit_li(top, w, lane + 32)], acc_hi);
}

// (one warp) cumulative over a freshly counted window; materializes the
// 1-based token stream list[] (levels, nearest first) up to `cap` entries.
// Returns the running total.
__device__ int finish_window(const Geo &g, bool top, int w, int *lvl, int found, int16_t *list, int cap) {
    const int lane = lane_id();
    int run = found;
    for (int i0 = win_lo(w); i0 < win_hi(w); i0 += 32) {
        const int li = i0 + lane;
        const int cnt = li < win_hi(w) ? lvl[li] : 0;
        int tot;
        const int ex = warp_excl_scan(cnt, &tot);
        const int cb = run + ex;
        if (li < win_hi(w)) lvl[li] = (cnt << 16) | min(cb, 65535);
        const int v = top ? g.lo - 1 - li : g.hi + 1 + li;
        for (int q = cb + 1; q <= min(cb + cnt, cap); ++q) list[q] = (int16_t)v;
        run += tot;
    }
    return run;
}

// Emits (and clears from their columns) the used tokens of one side in one
// window; T = this side's transposed words of the window (all chunks).
__device__ long long emit_window(const Geo &g, uint64_t *dep, int *sigma, int c, bool top, int w, int used, int a,
                                 int R, int n_right, int n_left, const int *lvl, const uint32_t *T, int vstar_li,
                                 int r_star, PathOut o, int off, int evid, int g0, int gn) {
    const int warp = warp_id(), lane = lane_id();
    long long disp = 0;
    if (warp < g0 || warp >= g0 + gn) return 0;
    // only levels <= vstar are used; they reach no column farther than vstar
    const int lim = min(win_hi(w), vstar_li + 1);
    const int V0 = win_V0(g, top, w), nslots = win_nslots(g, lim), nch = (nslots + 31) / 32;
    const uint64_t wmask = win_mask(top, w, vstar_li);
    for (int ch = warp - g0; ch < nch; ch += gn) {
        int col, dist;
        const uint64_t word = slot_word(g, dep, c, ch * 32 + lane, nslots, V0, top, &col, &dist, wmask);
        uint64_t cleared = 0ull;
        for (uint64_t x = word; x; x &= x - 1) {
            const int i = __ffsll((long long)x) - 1;
            const int li = bit_li(top, w, i);
            int rank_lt = __popc(T[ch * 64 + i] & lanemask_lt());
            for (int q = 0; q < ch; ++q) rank_lt += __popc(T[q * 64 + i]);
            int jside;
            if (li == vstar_li) {
                if (rank_lt >= r_star) continue;
                jside = top ? rank_lt : used - r_star + rank_lt;
            } else {
                const int cb = lvl[li] & 0xffff, cnt = lvl[li] >> 16;
                jside = top ? used - (cb + cnt) + rank_lt : cb + rank_lt;
            }
            const int v = V0 + i;
            const int depth = top ? v + dist : v - dist;
            const int j = top ? jside : a + R + jside;
            const int t = g.lo + j;
            const int p = off + emit_slot(g, j, n_right, n_left);
            o.src[p] = col * g.H + (g.H - 1 - depth);
            o.dst[p] = c * g.H + (g.H - 1 - t);
            if (o.ev) o.ev[p] = evid;
            disp += top ? t - v : v - t;
            cleared |= 1ull << i;
        }
        if (cleared) {
            uint64_t *m = dep + (size_t)col * g.wpd;
            const int start = top ? V0 + dist : V0 - dist;
            // top and bottom windows run concurrently and may share a word / a
            // column: the window's bits (depths start + i, all >= 0) cover at
            // most two plane words, one atomic AND each
            if (start >= 0) {
                const int w0 = start >> 6, sh = start & 63;
                atomicAnd((unsigned long long *)&m[w0], ~(cleared << sh));
                if (sh && (cleared >> (64 - sh))) atomicAnd((unsigned long long *)&m[w0 + 1], ~(cleared >> (64 - sh)));
            } else {
                atomicAnd((unsigned long long *)&m[0], ~(cleared >> (-start)));
            }
            if (col != c) atomicSub(&sigma[col], __popcll(cleared));
        }
    }
    return disp;
}

// stores the transposed words of one window (all chunks) into T
__device__ void transpose_window(const Geo &g, const uint64_t *dep, int c, bool top, int w, int vstar_li, uint32_t *T,
                                 int g0, int gn) {
    const int warp = warp_id(), lane = lane_id();
    if (warp < g0 || warp >= g0 + gn) return;
    const int lim = min(win_hi(w), vstar_li + 1);
    const int V0 = win_V0(g, top, w), nslots = win_nslots(g, lim), nch = (nslots + 31) / 32;
    const uint64_t wmask = win_mask(top, w, vstar_li);
    for (int ch = warp - g0; ch < nch; ch += gn) {
        int col, dist;
        const uint64_t word = slot_word(g, dep, c, ch * 32 + lane, nslots, V0, top, &col, &dist, wmask);
        uint32_t t_lo, t_hi;
        transpose64(word, t_lo, t_hi);
        T[ch * 64 + lane] = t_lo;
        T[ch * 64 + 32 + lane] = t_hi;
    }
}

// Delta(a) = cost(a) - cost(a-1) (split rule, no mandatory reservoir tokens)
__device__ __forceinline__ int pooled_delta(const Geo &g, int a, int holes, int R, const int16_t *otop,
                                            const int16_t *obot, const int16_t *hole) {
    return (g.lo + a - 1) - otop[a] + 2 * (hole[a] - g.lo - a + 1) - R - obot[holes - a + 1] + g.hi - (holes - a);
}

// One bird row-pass event for column c (BirdRunner::solve_column(c, true)).
// Returns the path count (CTA-uniform) or -1 when infeasible.
__device__ int pooled_event(const Geo &g, uint64_t *dep, int *sigma, int c, int16_t *L0, PooledScratch ps,
                            PathOut o, int off, int evid, unsigned long long *disp_acc, long long *dbg) {
    const int lane = lane_id(), warp = warp_id(), nw = blockDim.x >> 5;
    int16_t *hole = L0 + 2 * g.LK, *res = L0 + 3 * g.LK;
    int *S = ps.scal;
    enum { sR, sHoles, sFoundT, sFoundB, sWT, sWB, sWantT, sWantB, sDone, sA, sFail };
    const int maxlev_t = g.lo + g.W - 1, maxlev_b = (g.H - 1 - g.hi) + g.W - 1;
    // A: own residents and holes (warp 0); level tables cleared
    for (int i = threadIdx.x; i < g.LT; i += blockDim.x) ps.lvl_t[i] = 0;
    for (int i = threadIdx.x; i < g.LB; i += blockDim.x) ps.lvl_b[i] = 0;
    if (warp == 0) {
        const int B = g.B, base = lane * B;
        const uint32_t ch = lane_chunk(dep + (size_t)c * g.wpd, g.wpd, lane, B);
        const uint32_t bandr = chunk_range(base, B, g.lo, g.hi + 1);
        const uint32_t resm = ch & bandr, holem = ~ch & bandr;
        int R, nh;
        int er = warp_excl_scan(__popc(resm), &R);
        int eh = warp_excl_scan(__popc(holem), &nh);
        for (uint32_t x = holem; x; x &= x - 1, ++eh) hole[eh + 1] = (int16_t)(base + __ffs(x) - 1);
        for (uint32_t x = resm; x; x &= x - 1, ++er) res[er] = (int16_t)(base + __ffs(x) - 1);
        if (lane == 0) {
            hole[0] = (int16_t)(g.lo - 1);
            hole[nh + 1] = (int16_t)(g.hi + 1);
            S[sR] = R;
            S[sHoles] = nh;
            S[sFoundT] = S[sFoundB] = 0;
            S[sWT] = S[sWB] = 0;
            S[sWantT] = S[sWantB] = nh > 0;
            S[sDone] = nh == 0;
            S[sA] = 0;
            S[sFail] = 0;
        }
    }
    __syncthreads();
    const int R = S[sR], holes = S[sHoles];
    // B: progressive two-sided scan until the split a is pinned down
    while (!S[sDone]) {
        const bool wt = S[sWantT], wb = S[sWantB];
        const int wtop = S[sWT], wbot = S[sWB];
        const int half = nw / 2;
        if (wt) count_window(g, dep, c, true, wtop, ps.lvl_t, ps.bal, 0, wb ? half : nw);
        if (wb) count_window(g, dep, c, false, wbot, ps.lvl_b, ps.bal + (size_t)g.nchunk * 64, wt ? half : 0,
                             wt ? nw - half : nw);
        __syncthreads();
        if (warp == 0 && wt) {
            const int f = finish_window(g, true, wtop, ps.lvl_t, S[sFoundT], ps.otop, holes);
            if (lane == 0) {
                S[sFoundT] = f;
                S[sWT] = wtop + 1;
            }
        }
        if (warp == (nw > 1 ? 1 : 0) && wb) {
            __syncwarp();
            const int f = finish_window(g, false, wbot, ps.lvl_b, S[sFoundB], ps.obot, holes);
            if (lane == 0) {
                S[sFoundB] = f;
                S[sWB] = wbot + 1;
            }
        }
        __syncthreads();
        if (warp == 0) {
            const int ft = S[sFoundT], fb = S[sFoundB];
            const bool exh_t = (S[sWT] ? win_hi(S[sWT] - 1) : 0) >= maxlev_t;
            const bool exh_b = (S[sWB] ? win_hi(S[sWB] - 1) : 0) >= maxlev_b;
            const int BIG = 1 << 28;
            const int n_ot = exh_t ? ft : BIG, n_ob = exh_b ? fb : BIG;
            const int amin = max(0, holes - n_ob), amax = min(n_ot, holes);
            bool need_t = false, need_b = false, done = false, fail = false;
            int astar = 0;
            if (amin > amax) {
                fail = true;
            } else {
                // Delta(a) is computable for a in [A_lo, A_hi]
                const int A_lo = max(amin + 1, holes + 1 - min(fb, holes)), A_hi = min(amax, min(ft, holes));
                if (amin == amax) {
                    astar = amin;
                    done = true;
                } else if (A_lo > A_hi) {
                    need_t = ft < holes && !exh_t;
                    need_b = fb < holes && !exh_b;
                } else {
                    const int d_lo = pooled_delta(g, A_lo, holes, R, ps.otop, ps.obot, hole);
                    const int d_hi = pooled_delta(g, A_hi, holes, R, ps.otop, ps.obot, hole);
                    need_b = d_lo > 0 && A_lo > amin + 1;
                    need_t = d_hi <= 0 && A_hi < amax;
                    if (!need_b && !need_t) {
                        int cnt = 0;
                        if (d_lo <= 0) {
                            for (int a0 = A_lo; a0 <= A_hi; a0 += 32) {
                                const int aa = a0 + lane;
                                const bool le = aa <= A_hi && pooled_delta(g, aa, holes, R, ps.otop, ps.obot, hole) <= 0;
                                cnt += __popc(__ballot_sync(FULL, le));
                            }
                            cnt += A_lo - (amin + 1);
                        }
                        astar = amin + cnt;
                        done = true;
                    }
                }
            }
            if (done) {
                // the emission needs the used tokens' levels on both sides
                if (ft < astar && !exh_t) need_t = true, done = false;
                if (fb < holes - astar && !exh_b) need_b = true, done = false;
            }
            if (lane == 0) {
                S[sWantT] = need_t;
                S[sWantB] = need_b;
                S[sDone] = done || fail;
                S[sFail] = fail;
                S[sA] = astar;
            }
        }
        __syncthreads();
    }
    if (S[sFail]) return -1;
    const int a = S[sA], b = holes - a;
    if (dbg && threadIdx.x == 0) {
        dbg[0] = holes;
        dbg[1] = S[sWT] ? win_hi(S[sWT] - 1) : 0;
        dbg[2] = S[sWB] ? win_hi(S[sWB] - 1) : 0;
        dbg[3] = S[sFoundT];
        dbg[4] = S[sFoundB];
        dbg[5] = a;
        dbg[6] = b;
    }
    const int cntE = hole[a] - g.lo - a + 1;
    const int nstat = hole[a + 1] - hole[a] - 1;
    const int n_right = a + cntE, n_left = (R - cntE - nstat) + b;
    // C: last used level per side and how many of its members (group order) are used
    int vt_li = -1, rt = 0, vb_li = -1, rb = 0;
    if (a >= 1) {
        vt_li = g.lo - 1 - ps.otop[a];
        rt = a - (ps.lvl_t[vt_li] & 0xffff);
    }
    if (b >= 1) {
        vb_li = ps.obot[b] - (g.hi + 1);
        rb = b - (ps.lvl_b[vb_li] & 0xffff);
    }
    // D: emission, top and bottom windows side by side
    long long disp = 0;
    const int last_t = vt_li >= 0 ? win_of(vt_li) : -1, last_b = vb_li >= 0 ? win_of(vb_li) : -1;
    uint32_t *Tt = ps.bal, *Tb = ps.bal + (size_t)g.nchunk * 64;
    // windows in reverse: each side's last counted window still has its
    // transposed words in T from the count (rows of levels <= v* are the same
    // with the emission's narrower mask: farther slots reach no such level);
    // windows hold disjoint levels, so the emission order does not matter
    bool cached_t = last_t >= 0 && last_t == S[sWT] - 1, cached_b = last_b >= 0 && last_b == S[sWB] - 1;
    for (int w = max(last_t, last_b); w >= 0; --w) {
        const bool dt = w <= last_t, db = w <= last_b;
        const bool tt = dt && !(cached_t && w == last_t), tb = db && !(cached_b && w == last_b);
        const int half = nw / 2;
        if (tt) transpose_window(g, dep, c, true, w, vt_li, Tt, 0, db ? half : nw);
        if (tb) transpose_window(g, dep, c, false, w, vb_li, Tb, dt ? half : 0, dt ? nw - half : nw);
        if (tt || tb) __syncthreads();
        if (dt)
            disp += emit_window(g, dep, sigma, c, true, w, a, a, R, n_right, n_left, ps.lvl_t, Tt, vt_li, rt, o, off,
                                evid, 0, db ? half : nw);
        if (db)
            disp += emit_window(g, dep, sigma, c, false, w, b, a, R, n_right, n_left, ps.lvl_b, Tb, vb_li, rb, o, off,
                                evid, dt ? half : 0, dt ? nw - half : nw);
        __syncthreads();
    }
    // E: residents
    if (warp == 0) {
        for (int i = lane; i < R; i += 32) {
            const int depth = res[i], j = a + i, t = g.lo + j;
            if (t == depth) continue;
            const int p = off + emit_slot(g, j, n_right, n_left);
            o.src[p] = c * g.H + (g.H - 1 - depth);
            o.dst[p] = c * g.H + (g.H - 1 - t);
            if (o.ev) o.ev[p] = evid;
            disp += t > depth ? t - depth : depth - t;
        }
    }
    disp = warp_sum64(disp);
    if (lane == 0 && disp) atomicAdd(disp_acc, (unsigned long long)disp);
    __syncthreads();
    // F: own column = band + unused own reservoir (bird.cpp:90-99)
    if (warp == 0) {
        int left = 0;
        for (int w = lane; w < g.wpd; w += 32) {
            uint64_t *m = dep + (size_t)c * g.wpd + w;
            const uint64_t band = word_range(64 * w, g.lo, g.hi + 1);
            left += __popcll(*m & ~band);
            *m |= band;
        }
        left = warp_sum(left);
        if (lane == 0) sigma[c] = left;
    }
    __syncthreads();
    return n_right + n_left;
}

// MODE 1 (lone instance): up to 16 warps (more chunks of a window in flight),
// up to 128 registers.  Batches: MODE 0 (up to 85 registers; the compiler
// keeps 64, best on small grids) or MODE 2 (up to 128; better from 128^2).
template <int MODE>
__global__ void __launch_bounds__(MODE == 1 ? 512 : 256, MODE == 0 ? 3 : (MODE == 1 ? 1 : 2)) bird_kernel(GridParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geo g = make_geo(p.shape);
    Block b = carve(p.shape, smem);
    const int warp = warp_id(), lane = lane_id();
    __shared__ long long s_tokens;
    __shared__ unsigned long long s_disp;
    __shared__ int s_status, s_detail, s_n1, s_off, s_fail;
    PooledScratch ps;
    ps.otop = b.plists;
    ps.obot = b.plists + g.LK;
    ps.lvl_t = b.lvl_t;
    ps.lvl_b = b.lvl_b;
    ps.bal = b.bal;
    ps.scal = b.scal;
    __shared__ int s_next;
    for (int inst = blockIdx.x; inst < p.count; inst = next_instance(p, inst, &s_next)) {
        const size_t pbase = (size_t)inst * g.W * g.k;
        PathOut o{p.path_src + pbase, p.path_dst + pbase, p.path_event ? p.path_event + pbase : nullptr};
        if (threadIdx.x == 0) {
            s_tokens = 0;
            s_disp = 0;
            s_status = RECON_OK;
            s_detail = 0;
            s_fail = 0;
        }
        __syncthreads();
        load_instance(g, p.occ + (size_t)inst * g.W * g.wpd, b, &s_tokens);
        __syncthreads();
        if (threadIdx.x == 0 && s_tokens < (long long)g.W * g.k) {
            s_status = RECON_ERR_INFEASIBLE;
            s_detail = RECON_D_FEWER_SOURCES;
        }
        // column pass plan: sigma >= 0 ascending, then the rest ascending (bird.cpp:114-120)
        if (warp == 0) {
            int nev = 0;
            for (int pass = 0; pass < 2; ++pass)
                for (int x0 = 0; x0 < g.W; x0 += 32) {
                    const int c = x0 + lane;
                    const bool take = c < g.W && ((b.sigma[c] >= 0) == (pass == 0));
                    const unsigned bt = __ballot_sync(FULL, take);
                    if (take) b.ev_col[nev + __popc(bt & lanemask_lt())] = (int16_t)c;
                    nev += __popc(bt);
                    if (pass == 0 && x0 + 32 >= g.W && lane == 0) s_n1 = nev;
                }
        }
        __syncthreads();
        if (s_status == RECON_OK) {
            const int n1 = s_n1;
            own_count_range(g, b, 0, n1, 0, &s_fail);
            __syncthreads();
            if (warp == 0) {
                const int t = scan_counts(b, 0, n1);
                if (lane == 0) s_off = t;
            }
            __syncthreads();
            own_emit_range(g, b, 0, n1, 0, o, 0, true, &s_disp);
            __syncthreads();
            // row pass: pooled events, strictly sequential.  An event's path
            // count is CTA-uniform (read from shared state after its last
            // barrier), so every thread keeps the running offset itself.
            int off = s_off;
            for (int e = n1; e < g.W; ++e) {
                const int c = b.ev_col[e];
                long long *dbg = (p.phase_clock && inst == 0) ? p.phase_clock + 8 + 8 * (e - n1) : nullptr;
                const int cnt = pooled_event(g, b.dep, b.sigma, c, b.lists, ps, o, off, e, &s_disp, dbg);
                if (cnt < 0) {
                    if (threadIdx.x == 0) s_fail = 1;
                    __syncthreads();
                    break;
                }
                off += cnt;
            }
            __syncthreads();
            if (threadIdx.x == 0) s_off = off;
            if (s_fail && threadIdx.x == 0) {
                s_status = RECON_ERR_INFEASIBLE;
                s_detail = RECON_D_GEN_NO_ASSIGNMENT;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const bool ok = s_status == RECON_OK;
            p.path_count[inst] = ok ? s_off : 0;
            p.total_displacement[inst] = ok ? (long long)s_disp : 0;
            p.status[inst] = s_status;
            if (p.detail) p.detail[inst] = s_detail;
        }
        if (p.events && s_status == RECON_OK)
            for (int e = threadIdx.x; e < g.W; e += blockDim.x) p.events[(size_t)inst * g.W + e] = b.ev_col[e];
        __syncthreads();
    }
}

template __global__ void bird_kernel<0>(GridParams);
template __global__ void bird_kernel<1>(GridParams);
template __global__ void bird_kernel<2>(GridParams);

}  // namespace rb
