// red-rec on sm_100a: one CTA per instance.
//
// Reference: /root/reference/proj/src/redrec.cpp:15-232.
//
// 1. Plan (warp 0).  red-rec's control flow depends only on the surplus
//    vector (the pairing loop reads sigma and `solved`, redrec.cpp:43-86,
//    205-232), so the whole event sequence is replayed first from sigma.
//    Per lane, a block of <= 32 columns is held as register bitmasks
//    (receivers, donors; unsolved = non-transit), so the nearest
//    non-transit column on either side of a receiver (scan_for_donor,
//    redrec.cpp:43-51) is a bit-scan plus a warp max/min scan instead of a
//    walk through shared memory.  The plan also assigns each pairing-loop
//    event a dependency level: 1 + the last level touching any column it
//    reads/writes or the mark set of its receiver.
// 2. Waves.  Loop events of one level touch disjoint state and run
//    concurrently, one warp per event.  Every event (phase 1, loop, phase 3)
//    writes its paths, in emission order, to its own k-slot region of a
//    per-CTA staging buffer (global, L2-resident in practice) right after
//    its solve, and records its path count.
// 3. Phase-3 compactions are solved in parallel on the final state.
// 4. One scan over all W events in canonical order gives every event's
//    output offset; the staged paths move there with coalesced copies.
// Marks (parked tokens of a donating compaction, redrec.cpp:155-160) stay in
// the marker's column plane and are never cleared: only their receiver's
// transfer reads them.

#include "grid_common.cuh"

namespace rb {

// --------------------------------------------------------------------------
// warp-level transfer event (Runner::flush + build_redistribution_instance,
// redrec.cpp:92-116, 169-191): receiver r's own tokens and the marks parked
// for it are mandatory, donor d's reservoir is the optional pool
// --------------------------------------------------------------------------

struct FlushSolve {
    int a, b, R, holes, m_top, m_bot, n_ot, n_ob, n_right, n_left, dd;
};

// Marks parked for receiver r form a list through the marker columns:
// mark_head[r], then mark_next[x] (-1 ends it); order is irrelevant.
__device__ bool flush_solve(const Geo &g, const uint64_t *mr, const uint64_t *md, int r, int d, const uint64_t *dep,
                            int mark_first, const int16_t *mark_next, int16_t *L, int forced_a, FlushSolve &f) {
    int16_t *otop = L, *obot = L + g.LK, *hole = L + 2 * g.LK, *res = L + 3 * g.LK;
    const int lane = lane_id(), B = g.B, base = lane * B;
    const int dd = d > r ? d - r : r - d;
    const uint32_t rtop = chunk_range(base, B, 0, g.lo), rband = chunk_range(base, B, g.lo, g.hi + 1),
                   rbot = chunk_range(base, B, g.hi + 1, g.H);
    const uint32_t chr = lane_chunk(mr, g.wpd, lane, B);
    const uint32_t resm = chr & rband, holem = ~chr & rband;
    int R, nh;
    int er = warp_excl_scan(__popc(resm), &R);
    int eh = warp_excl_scan(__popc(holem), &nh);
    const int holes = nh;
    for (uint32_t x = holem; x; x &= x - 1, ++eh) hole[eh + 1] = (int16_t)(base + __ffs(x) - 1);
    for (uint32_t x = resm; x; x &= x - 1, ++er) res[er] = (int16_t)(base + __ffs(x) - 1);
    int m_top = __popc(chr & rtop), m_bot = __popc(chr & rbot);
    for (int x = mark_first; x >= 0; x = mark_next[x]) {
        const uint32_t chx = lane_chunk(dep + (size_t)x * g.wpd, g.wpd, lane, B);
        m_top += __popc(chx & rtop);
        m_bot += __popc(chx & rbot);
    }
    m_top = warp_sum(m_top);
    m_bot = warp_sum(m_bot);
    const uint32_t chd = lane_chunk(md, g.wpd, lane, B);
    const uint32_t dtop = chd & rtop, dbot = chd & rbot;
    int n_ot, n_ob;
    int et = warp_excl_scan(__popc(dtop), &n_ot);
    int eb = warp_excl_scan(__popc(dbot), &n_ob);
    for (uint32_t x = dtop; x; x &= x - 1, ++et) {
        const int desc = n_ot - 1 - et;
        if (desc < holes) otop[desc + 1] = (int16_t)(base + __ffs(x) - 1 - dd);
    }
    for (uint32_t x = dbot; x; x &= x - 1, ++eb)
        if (eb < holes) obot[eb + 1] = (int16_t)(base + __ffs(x) - 1 + dd);
    if (lane == 0) {
        hole[0] = (int16_t)(g.lo - 1);
        hole[holes + 1] = (int16_t)(g.hi + 1);
    }
    __syncwarp();
    const int amin = max(m_top, holes - m_bot - n_ob), amax = min(m_top + n_ot, holes - m_bot);
    if (amin > amax) return false;
    int a = forced_a;
    if (a < 0) {
        int cnt = 0;
        for (int a0 = amin + 1; a0 <= amax; a0 += 32) {
            const int aa = a0 + lane;
            bool le = false;
            if (aa <= amax) {
                const int delta = (g.lo + aa - 1) - otop[aa - m_top] + 2 * (hole[aa] - g.lo - aa + 1) - R -
                                  obot[holes - aa + 1 - m_bot] + g.hi - (holes - aa);
                le = delta <= 0;
            }
            cnt += __popc(__ballot_sync(FULL, le));
        }
        a = amin + cnt;
    }
    f.a = a;
    f.b = holes - a;
    f.R = R;
    f.holes = holes;
    f.m_top = m_top;
    f.m_bot = m_bot;
    f.n_ot = n_ot;
    f.n_ob = n_ob;
    f.dd = dd;
    const int cntE = hole[a] - g.lo - a + 1;
    const int nstat = hole[a + 1] - hole[a] - 1;
    f.n_right = a + cntE;
    f.n_left = (R - cntE - nstat) + f.b;
    return true;
}

__device__ long long flush_emit(const Geo &g, const FlushSolve &f, const uint64_t *mr, const uint64_t *md, int r,
                                int d, const uint64_t *dep, int mark_first, const int16_t *mark_next,
                                const int16_t *L, uint32_t *keys, uint32_t *st) {
    const int16_t *res = L + 3 * g.LK;
    const int lane = lane_id(), B = g.B, base = lane * B;
    const uint32_t rtop = chunk_range(base, B, 0, g.lo), rbot = chunk_range(base, B, g.hi + 1, g.H);
    const int a = f.a, b = f.b, R = f.R, dd = f.dd;
    const int xa = a - f.m_top, xb = b - f.m_bot;
    uint32_t *ktop = keys, *kbot = keys + g.LK;
    // keys of the used tokens: own, each marker column's, the donor's
    {
        const uint32_t chr = lane_chunk(mr, g.wpd, lane, B);
        int tot;
        int e = warp_excl_scan(__popc(chr & rtop), &tot);
        for (uint32_t x = chr & rtop; x; x &= x - 1) ktop[e++] = tok_key(base + __ffs(x) - 1, 0, r);
        int pos_t = tot;
        e = warp_excl_scan(__popc(chr & rbot), &tot);
        for (uint32_t x = chr & rbot; x; x &= x - 1) kbot[e++] = tok_key(base + __ffs(x) - 1, 0, r);
        int pos_b = tot;
        for (int x = mark_first; x >= 0; x = mark_next[x]) {
            const int dx = x > r ? x - r : r - x;
            const uint32_t chx = lane_chunk(dep + (size_t)x * g.wpd, g.wpd, lane, B);
            e = warp_excl_scan(__popc(chx & rtop), &tot);
            for (uint32_t y = chx & rtop; y; y &= y - 1) ktop[pos_t + e++] = tok_key(base + __ffs(y) - 1 - dx, dx, x);
            pos_t += tot;
            e = warp_excl_scan(__popc(chx & rbot), &tot);
            for (uint32_t y = chx & rbot; y; y &= y - 1) kbot[pos_b + e++] = tok_key(base + __ffs(y) - 1 + dx, dx, x);
            pos_b += tot;
        }
        // donor: innermost xa top, innermost xb bottom
        const uint32_t chd = lane_chunk(md, g.wpd, lane, B);
        const uint32_t dtop = chd & rtop, dbot = chd & rbot;
        e = warp_excl_scan(__popc(dtop), &tot);
        for (uint32_t x = dtop; x; x &= x - 1, ++e) {
            const int desc = f.n_ot - 1 - e;
            if (desc < xa) ktop[pos_t + desc] = tok_key(base + __ffs(x) - 1 - dd, dd, d);
        }
        e = warp_excl_scan(__popc(dbot), &tot);
        for (uint32_t x = dbot; x; x &= x - 1, ++e)
            if (e < xb) kbot[pos_b + e] = tok_key(base + __ffs(x) - 1 + dd, dd, d);
    }
    __syncwarp();
    // a token's target index is its rank among the used keys (all distinct)
    long long disp = 0;
    for (int i = lane; i < a; i += 32) {
        const uint32_t key = ktop[i];
        int rank = 0;
        for (int q = 0; q < a; ++q) rank += ktop[q] < key;
        const int v = (int)(key >> 20) - 2048, dist = (key >> 10) & 1023, col = key & 1023;
        const int depth = v + dist, j = rank, t = g.lo + j;
        emit_put(st, g, emit_slot(g, j, f.n_right, f.n_left), col, depth, r, t, 0);
        disp += t - v;
    }
    for (int i = lane; i < b; i += 32) {
        const uint32_t key = kbot[i];
        int rank = 0;
        for (int q = 0; q < b; ++q) rank += kbot[q] < key;
        const int v = (int)(key >> 20) - 2048, dist = (key >> 10) & 1023, col = key & 1023;
        const int depth = v - dist, j = a + R + rank, t = g.lo + j;
        emit_put(st, g, emit_slot(g, j, f.n_right, f.n_left), col, depth, r, t, 0);
        disp += v - t;
    }
    for (int i = lane; i < R; i += 32) {
        const int depth = res[i], j = a + i, t = g.lo + j;
        if (t == depth) continue;
        emit_put(st, g, emit_slot(g, j, f.n_right, f.n_left), r, depth, r, t, 0);
        disp += t > depth ? t - depth : depth - t;
    }
    __syncwarp();
    return warp_sum64(disp);
}

// donor loses its drawn innermost reservoir tokens; receiver keeps band cells
__device__ void flush_update(const Geo &g, uint64_t *dep, int r, int d, const FlushSolve &f, const int16_t *L) {
    const int16_t *otop = L, *obot = L + g.LK;
    const int xa = f.a - f.m_top, xb = f.b - f.m_bot;
    const int thr_t = xa >= 1 ? otop[xa] + f.dd : g.lo;  // clear donor top depth >= thr_t
    const int thr_b = xb >= 1 ? obot[xb] - f.dd : g.hi;  // clear donor bottom depth <= thr_b
    __syncwarp();
    uint64_t *md = dep + (size_t)d * g.wpd;
    for (int w = lane_id(); w < g.wpd; w += 32) {
        md[w] &= ~(word_range(64 * w, thr_t, g.lo) | word_range(64 * w, g.hi + 1, thr_b + 1));
        dep[(size_t)r * g.wpd + w] = word_range(64 * w, g.lo, g.hi + 1);
    }
    __syncwarp();
}

// --------------------------------------------------------------------------
// plan: surplus-only replay of redrec.cpp:205-232 with dependency levels
// --------------------------------------------------------------------------

// link word of column c: NL (nearest unsolved column on the left, -1 if none)
// in the low half, NR (on the right, W if none) in the high half
__device__ __forceinline__ int link_l(int v) { return (int)(int16_t)(v & 0xffff); }
__device__ __forceinline__ int link_r(int v) { return v >> 16; }
__device__ __forceinline__ int make_link(int l, int r) { return (r << 16) | (l & 0xffff); }

// key of receiver q: best of its nearest unsolved neighbours that are donors,
// ranked (-exchange, |d-r|, deficit-exchange, r, d) (select_best_pair,
// redrec.cpp:55-86), packed as hi = (2047-ex)<<21 | dist<<11 | (deficit-ex)
// (|sigma| <= H <= 1024, so every field fits) and lo = q<<10 | d; ~0 when
// neither side has an admissible donor.  Transit columns have sigma 0, so
// `sig[d] > 0` alone admits a donor.
__device__ __forceinline__ unsigned long long receiver_key(int q, int W, int sq, int lk, const int *sig) {
    const int deficit = -sq;
    const int dl = link_l(lk), dr = link_r(lk);
    const int sl = dl >= 0 ? sig[dl] : 0, sr = dr < W ? sig[dr] : 0;
    auto key = [&](int d, int sd) {
        const int ex = min(sd, deficit);
        const unsigned hi = ((unsigned)(2047 - ex) << 21) | ((unsigned)(d > q ? d - q : q - d) << 11) |
                            (unsigned)(deficit - ex);
        return sd > 0 ? ((unsigned long long)hi << 32) | ((unsigned)q << 10) | (unsigned)d : ~0ull;
    };
    const unsigned long long kl = key(dl, sl), kr = key(dr, sr);
    return kl < kr ? kl : kr;
}

// Surplus-only replay of the pairing loop with incremental candidate keys.
// Columns are "unsolved" (non-transit, sigma != 0) or solved with zero
// surplus (transit, scan_for_donor redrec.cpp:43-51).  The unsolved columns
// form a doubly linked list, so a column turning transit is unlinked in O(1);
// links are only read at columns that were unsolved when the iteration began,
// and a neighbour unlinked in the same iteration is skipped with one more hop.
// An iteration changes only the donor d and the receiver r, so only r and the
// receivers adjacent to d and r need new keys.  Keys live in shared memory
// (lane L owns columns [L*per, L*per+per)); the global minimum is two
// redux.sync reductions over the lanes' minima.
template <class B>
__device__ int redrec_plan(const Geo &g, B &b, int *n1o, int *n2o, int *nlevo, long long *prof = nullptr) {
    const int lane = lane_id(), W = g.W;
    const int per = (W + 31) / 32, c0 = lane * per, c1 = min(W, c0 + per);
    int *sig = b.ev_count;                                    // scratch: plan-time surplus
    int *lnk = b.links;                                       // NL / NR pairs
    unsigned long long *rkey = (unsigned long long *)b.keys;  // 32*per + 8 entries
    int nrecv = 0;
    for (int c = c0; c < c1; ++c) {
        const int s = b.sigma[c];
        sig[c] = s;
        nrecv += s < 0;
        b.lastc[c] = 0;
        b.lastm[c] = 0;
    }
    nrecv = warp_sum(nrecv);
    int nev = 0;
    for (int x0 = 0; x0 < W; x0 += 32) {
        const int c = x0 + lane;
        const bool z = c < W && b.sigma[c] == 0;  // phase 1 (redrec.cpp:211-212)
        const unsigned bz = __ballot_sync(FULL, z);
        if (z) {
            const int slot = nev + __popc(bz & lanemask_lt());
            b.ev_type[slot] = EV_OWN;
            b.ev_col[slot] = (int16_t)c;
            b.ev_aux[slot] = -1;
        }
        nev += __popc(bz);
    }
    const int n1 = nev;
    // initial links: nearest unsolved (sigma != 0) column on each side
    {
        uint32_t ntm = 0;
        for (int c = c0; c < c1; ++c)
            if (b.sigma[c] != 0) ntm |= 1u << (c - c0);
        int exL = ntm ? c0 + 31 - __clz(ntm) : -1;
        int exR = ntm ? c0 + __ffs(ntm) - 1 : W;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, exL, o);
            if (lane >= o) exL = max(exL, y);
            const int z = __shfl_down_sync(FULL, exR, o);
            if (lane + o < 32) exR = min(exR, z);
        }
        int left = __shfl_up_sync(FULL, exL, 1);
        int right = __shfl_down_sync(FULL, exR, 1);
        if (lane == 0) left = -1;
        if (lane == 31) right = W;
        for (int c = c0; c < c1; ++c) {
            lnk[c] = left & 0xffff;
            if (b.sigma[c] != 0) left = c;
        }
        for (int c = c1 - 1; c >= c0; --c) {
            lnk[c] |= right << 16;
            if (b.sigma[c] != 0) right = c;
        }
    }
    __syncwarp();
    for (int i = lane; i < 32 * per + 8; i += 32) {
        const int sq = i < W ? sig[i] : 0;
        rkey[i] = sq < 0 ? receiver_key(i, W, sq, lnk[i], sig) : ~0ull;
    }
    __syncwarp();
    int nlev = 0;
    long long pt[3] = {0, 0, 0}, t0 = prof ? clock64() : 0;
    auto tick = [&](int i) {
        if (prof) {
            const long long t = clock64();
            pt[i] += t - t0;
            t0 = t;
        }
    };
    while (nrecv > 0) {
        // lane minimum over 8 keys at a time (the tail past the lane's own
        // columns reads its neighbour's keys, which cannot change the minimum)
        unsigned long long best = ~0ull;
        for (int i0 = 0; i0 < per; i0 += 8) {
            unsigned long long k[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) k[i] = rkey[c0 + i0 + i];
#pragma unroll
            for (int i = 0; i < 8; ++i) best = k[i] < best ? k[i] : best;
        }
        const unsigned hi = __reduce_min_sync(FULL, (unsigned)(best >> 32));
        const unsigned lo = __reduce_min_sync(FULL, (unsigned)(best >> 32) == hi ? (unsigned)best : ~0u);
        if (hi == ~0u) return RECON_D_NO_DONOR;
        const int d = (int)(lo & 1023), r = (int)((lo >> 10) & 1023);
        // exchange and deficit straight from the key: ex < deficit <=> OWN(d, r)
        const int ex = 2047 - (int)(hi >> 21), def = ex + (int)(hi & 2047);
        tick(0);
        int tr0, tr1 = -1;  // columns turning transit
        if (ex < def) {
            tr0 = d;  // OWN(d, r): d donates by marking (ds = ex)
            if (lane == 0) {
                const int lv = 1 + max((int)b.lastc[d], (int)b.lastm[r]);
                b.lastc[d] = b.lastm[r] = (int16_t)lv;
                nlev = max(nlev, lv);
                b.ev_type[nev] = EV_OWN;
                b.ev_col[nev] = (int16_t)d;
                b.ev_aux[nev] = (int16_t)r;
                b.ev_level[nev] = (int16_t)lv;
                sig[r] = ex - def;
                sig[d] = 0;
            }
            nev += 1;
        } else {
            // FLUSH(r, d), then OWN(d, -1) if the donor is exhausted exactly
            const int ds = sig[d];
            tr0 = r;
            if (ds == def) tr1 = d;
            nrecv -= 1;
            if (lane == 0) {
                int lv = 1 + max(max((int)b.lastc[r], (int)b.lastc[d]), (int)b.lastm[r]);
                b.lastc[r] = b.lastc[d] = b.lastm[r] = (int16_t)lv;
                b.ev_type[nev] = EV_FLUSH;
                b.ev_col[nev] = (int16_t)r;
                b.ev_aux[nev] = (int16_t)d;
                b.ev_level[nev] = (int16_t)lv;
                nlev = max(nlev, lv);
                sig[d] = ds - def;
                sig[r] = 0;
                rkey[r] = ~0ull;
                if (ds == def) {
                    lv += 1;
                    b.lastc[d] = (int16_t)lv;
                    b.ev_type[nev + 1] = EV_OWN;
                    b.ev_col[nev + 1] = (int16_t)d;
                    b.ev_aux[nev + 1] = -1;
                    b.ev_level[nev + 1] = (int16_t)lv;
                    nlev = max(nlev, lv);
                }
            }
            nev += ds == def ? 2 : 1;
        }
        // unlink the columns that turned transit (in order)
        if (lane == 0) {
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int x = t == 0 ? tr0 : tr1;
                if (x < 0) continue;
                const int v = lnk[x], L = link_l(v), R = link_r(v);
                if (L >= 0) lnk[L] = make_link(link_l(lnk[L]), R);
                if (R < W) lnk[R] = make_link(L, link_r(lnk[R]));
            }
        }
        __syncwarp();
        tick(1);
        // refresh r (lane 0) and the nearest unsolved receivers on both sides
        // of d (lanes 1, 2) and r (lanes 3, 4)
        if (lane < 5) {
            const int x = lane == 0 ? r : (lane <= 2 ? d : r);
            const bool left = (lane & 1) != 0;
            int q = x;
            if (lane > 0) {
                const int v = lnk[x];
                q = left ? link_l(v) : link_r(v);
            }
            const bool in = q >= 0 && q < W;
            int lq = in ? lnk[q] : 0, sq = in ? sig[q] : 1;
            if (lane > 0 && in && sq == 0) {  // unlinked this iteration: one more hop
                q = left ? link_l(lq) : link_r(lq);
                const bool in2 = q >= 0 && q < W;
                lq = in2 ? lnk[q] : 0;
                sq = in2 ? sig[q] : 1;
            }
            if (sq < 0) rkey[q] = receiver_key(q, W, sq, lq, sig);
        }
        __syncwarp();
        tick(2);
    }
    if (prof && lane == 0)
        for (int i = 0; i < 3; ++i) prof[i] = pt[i];
    const int n2 = nev - n1;
    // phase 3: remaining columns ascending (redrec.cpp:228-229)
    for (int x0 = 0; x0 < W; x0 += 32) {
        const int c = x0 + lane;
        const bool u = c < W && sig[c] != 0;
        const unsigned bu = __ballot_sync(FULL, u);
        if (u) {
            const int slot = nev + __popc(bu & lanemask_lt());
            b.ev_type[slot] = EV_OWN;
            b.ev_col[slot] = (int16_t)c;
            b.ev_aux[slot] = -1;
        }
        nev += __popc(bu);
    }
    // waves: counting sort of the loop events by level -> wave_list / wave_off
    nlev = __shfl_sync(FULL, nlev, 0);
    for (int i = lane; i <= nlev + 1; i += 32) b.wave_off[i] = 0;
    __syncwarp();
    for (int e = n1 + lane; e < n1 + n2; e += 32) atomicAdd(&b.wave_off[b.ev_level[e]], 1);
    __syncwarp();
    if (lane == 0) {
        int run = 0;
        for (int lv = 0; lv <= nlev + 1; ++lv) {
            const int c = b.wave_off[lv];
            b.wave_off[lv] = run;
            run += c;
        }
        for (int e = n1; e < n1 + n2; ++e) {
            const int lv = b.ev_level[e];
            b.wave_list[b.wave_off[lv]++] = (int16_t)e;
        }
        for (int lv = nlev + 1; lv >= 1; --lv) b.wave_off[lv] = b.wave_off[lv - 1];
        b.wave_off[0] = 0;
    }
    __syncwarp();
    *n1o = n1;
    *n2o = n2;
    *nlevo = nlev;
    return 0;
}

// --------------------------------------------------------------------------
// kernel
// --------------------------------------------------------------------------

// --------------------------------------------------------------------------
// planner kernel: one warp per instance, plans written to global memory
// --------------------------------------------------------------------------

// the planner warp's shared-memory view (same field names as Block)
struct PlanView {
    int *sigma, *ev_count, *wave_off;
    uint32_t *keys;
    uint8_t *ev_type;
    int *links;
    int16_t *ev_col, *ev_aux, *ev_level, *wave_list, *ev_a, *lastc, *lastm;
};

__host__ __device__ inline int64_t plan_warp_bytes(int W) {
    return align_up((align_up(W, 32) + 8) * 8, 16) + align_up((int64_t)W * 4, 16) * 3 + align_up((int64_t)(W + 2) * 4, 16) +
           align_up(W, 16) * 2 + align_up((int64_t)W * 2, 16) * 7;
}

__device__ PlanView carve_plan(unsigned char *base, int W) {
    PlanView v;
    int64_t off = 0;
    auto take = [&](int64_t bytes) {
        unsigned char *at = base + off;
        off += align_up(bytes, 16);
        return at;
    };
    v.keys = (uint32_t *)take(((int64_t)align_up(W, 32) + 8) * 8);
    v.links = (int *)take((int64_t)W * 4);
    v.sigma = (int *)take((int64_t)W * 4);
    v.ev_count = (int *)take((int64_t)W * 4);
    v.wave_off = (int *)take((int64_t)(W + 2) * 4);
    v.ev_type = (uint8_t *)take(W);
    v.ev_col = (int16_t *)take((int64_t)W * 2);
    v.ev_aux = (int16_t *)take((int64_t)W * 2);
    v.ev_level = (int16_t *)take((int64_t)W * 2);
    v.wave_list = (int16_t *)take((int64_t)W * 2);
    v.ev_a = (int16_t *)take((int64_t)W * 2);
    v.lastc = (int16_t *)take((int64_t)W * 2);
    v.lastm = (int16_t *)take((int64_t)W * 2);
    return v;
}

int64_t redrec_plan_smem(int W) { return plan_warp_bytes(W); }

__global__ void __launch_bounds__(128) redrec_plan_kernel(GridParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geo g = make_geo(p.shape);
    const int warp = warp_id(), lane = lane_id(), wpb = blockDim.x >> 5;
    PlanView v = carve_plan(smem + (size_t)warp * plan_warp_bytes(g.W), g.W);
    const RedrecPlans pg = p.plans;
    const uint64_t last_mask = (g.H & 63) ? ((1ull << (g.H & 63)) - 1ull) : ~0ull;
    // the executor (launched as a programmatic dependent) may start loading
    // its instances now; it waits for this grid before reading the plans
    asm volatile("griddepcontrol.launch_dependents;");
    for (int inst = blockIdx.x * wpb + warp; inst < p.count; inst += gridDim.x * wpb) {
        const uint64_t *occ = p.occ + (size_t)inst * g.W * g.wpd;
        long long tot = 0;
        for (int x = lane; x < g.W; x += 32) {
            int cnt = 0;
            for (int j = 0; j < g.wpd; ++j) cnt += __popcll(occ[(size_t)x * g.wpd + j] & (j == g.wpd - 1 ? last_mask : ~0ull));
            v.sigma[x] = cnt - g.k;
            tot += cnt;
        }
        tot = warp_sum64(tot);
        __syncwarp();
        int n1 = 0, n2 = 0, nlev = 0, st = RECON_OK, det = 0;
        if (tot < (long long)g.W * g.k) {  // Problem::check (problem.hpp:113-116)
            st = RECON_ERR_INFEASIBLE;
            det = RECON_D_FEWER_SOURCES;
        } else {
            const int rc = redrec_plan(g, v, &n1, &n2, &nlev, (p.phase_clock && inst == 0) ? p.phase_clock + 8 : nullptr);
            if (rc) {
                st = RECON_ERR_LOGIC;
                det = rc;
            }
        }
        __syncwarp();
        int *meta = pg.meta + (size_t)inst * 8;
        if (lane == 0) {
            meta[0] = n1;
            meta[1] = n2;
            meta[2] = nlev;
            meta[3] = st;
            meta[4] = det;
        }
        if (st == RECON_OK) {
            const size_t W = g.W;
            for (int e = lane; e < g.W; e += 32) {
                pg.ev_type[inst * W + e] = v.ev_type[e];
                pg.ev_col[inst * W + e] = v.ev_col[e];
                pg.ev_aux[inst * W + e] = v.ev_aux[e];
                pg.wave_list[inst * W + e] = v.wave_list[e];
            }
            for (int i = lane; i <= nlev + 1; i += 32) pg.wave_off[inst * (W + 2) + i] = v.wave_off[i];
        }
        __syncwarp();
    }
}

// MINB = 1: up to 32 warps for a lone instance (latency), 64 registers;
// otherwise 8-warp CTAs, MINB per SM (batches)
template <int MINB>
__global__ void __launch_bounds__(MINB == 1 ? 1024 : 256, MINB) redrec_kernel(GridParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geo g = make_geo(p.shape);
    Block b = carve(p.shape, smem);
    const int warp = warp_id(), lane = lane_id(), nw = blockDim.x >> 5;
    int16_t *L = b.lists + (size_t)warp * 4 * g.LK;
    uint32_t *keys = b.keys + (size_t)warp * 2 * g.LK;
    // event e's paths are staged (packed, emission order) at stage + ks*e,
    // ks = k rounded to a 128-byte line so consumed lines can be discarded
    const int ks = stage_stride(g.k);
    uint32_t *const stage = p.stage + (size_t)blockIdx.x * g.W * ks;
    __shared__ long long s_tokens;
    __shared__ unsigned long long s_disp;
    __shared__ int s_status, s_detail, s_n1, s_n2, s_nlev, s_total, s_fail;
    __shared__ int s_next;
    for (int inst = blockIdx.x; inst < p.count; inst = next_instance(p, inst, &s_next)) {
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
            s_status = RECON_ERR_INFEASIBLE;  // Problem::check (problem.hpp:113-116)
            s_detail = RECON_D_FEWER_SOURCES;
        }
        __syncthreads();
        if (p.phase_clock && inst == 0 && threadIdx.x == 0) p.phase_clock[0] = clock64();
        // the instance's plan (redrec_plan_kernel) -> shared memory; under
        // programmatic dependent launch, wait for the planner grid first
        // (returns at once when it has completed, or without the attribute)
        asm volatile("griddepcontrol.wait;" ::: "memory");
        {
            const RedrecPlans pg = p.plans;
            const int *meta = pg.meta + (size_t)inst * 8;
            const size_t W = g.W;
            if (threadIdx.x == 0) {
                s_n1 = meta[0];
                s_n2 = meta[1];
                s_nlev = meta[2];
                if (s_status == RECON_OK && meta[3] != RECON_OK) {
                    s_status = meta[3];
                    s_detail = meta[4];
                }
            }
            if (meta[3] == RECON_OK) {
                for (int e = threadIdx.x; e < g.W; e += blockDim.x) {
                    b.ev_type[e] = pg.ev_type[inst * W + e];
                    b.ev_col[e] = pg.ev_col[inst * W + e];
                    b.ev_aux[e] = pg.ev_aux[inst * W + e];
                    b.wave_list[e] = pg.wave_list[inst * W + e];
                }
                for (int i = threadIdx.x; i <= meta[2] + 1; i += blockDim.x) b.wave_off[i] = pg.wave_off[inst * (W + 2) + i];
            }
        }
        __syncthreads();
        if (s_status == RECON_OK) {
            const int n1 = s_n1, n2 = s_n2, nlev = s_nlev, W = g.W;
            long long disp = 0;
            if (p.phase_clock && inst == 0 && threadIdx.x == 0) p.phase_clock[1] = clock64();
            // phase 1 (sigma == 0 compactions): solve + stage
            for (int e = warp; e < n1; e += nw) {
                OwnSolve s;
                const int c = b.ev_col[e];
                if (!own_solve(g, b.dep + (size_t)c * g.wpd, L, -1, s)) {
                    if (lane == 0) s_fail = 1;
                    continue;
                }
                disp += own_emit(g, c, s, L, stage + (size_t)e * ks, 0, e);
                if (lane == 0) b.ev_count[e] = s.n_right + s.n_left;
                __syncwarp();
            }
            // pairing-loop events in dependency waves: solve, stage, update
            for (int lv = 1; lv <= nlev; ++lv) {
                for (int q = b.wave_off[lv] + warp; q < b.wave_off[lv + 1]; q += nw) {
                    const int e = b.wave_list[q];
                    const int col = b.ev_col[e], aux = b.ev_aux[e];
                    uint64_t *mc = b.dep + (size_t)col * g.wpd;
                    uint32_t *st = stage + (size_t)e * ks;
                    if (b.ev_type[e] == EV_OWN) {
                        OwnSolve s;
                        if (!own_solve(g, mc, L, -1, s)) {
                            if (lane == 0) s_fail = 1;
                            continue;
                        }
                        disp += own_emit(g, col, s, L, st, 0, e);
                        own_update(g, mc, s, L);
                        if (lane == 0) {
                            b.ev_count[e] = s.n_right + s.n_left;
                            if (aux >= 0) {  // parked -> marks for aux
                                b.mark_next[col] = b.mark_head[aux];
                                b.mark_head[aux] = (int16_t)col;
                            }
                        }
                    } else {
                        uint64_t *md = b.dep + (size_t)aux * g.wpd;
                        FlushSolve f;
                        const int mfirst = b.mark_head[col];
                        if (!flush_solve(g, mc, md, col, aux, b.dep, mfirst, b.mark_next, L, -1, f)) {
                            if (lane == 0) s_fail = 1;
                            continue;
                        }
                        disp += flush_emit(g, f, mc, md, col, aux, b.dep, mfirst, b.mark_next, L, keys, st);
                        flush_update(g, b.dep, col, aux, f, L);
                        if (lane == 0) b.ev_count[e] = f.n_right + f.n_left;
                    }
                    __syncwarp();
                }
                __syncthreads();
            }
            if (p.phase_clock && inst == 0 && threadIdx.x == 0) p.phase_clock[2] = clock64();
            // phase 3: remaining compactions on the final state
            for (int e = n1 + n2 + warp; e < W; e += nw) {
                OwnSolve s;
                const int c = b.ev_col[e];
                if (!own_solve(g, b.dep + (size_t)c * g.wpd, L, -1, s)) {
                    if (lane == 0) s_fail = 1;
                    continue;
                }
                disp += own_emit(g, c, s, L, stage + (size_t)e * ks, 0, e);
                if (lane == 0) b.ev_count[e] = s.n_right + s.n_left;
                __syncwarp();
            }
            if (lane == 0 && disp) atomicAdd(&s_disp, (unsigned long long)disp);
            __syncthreads();
            // canonical offsets (event order), then the staged paths move to
            // their offsets with coalesced copies
            if (warp == 0) {
                int run = 0;
                for (int i0 = 0; i0 < W; i0 += 32) {
                    const int i = i0 + lane;
                    const int v = i < W ? b.ev_count[i] : 0;
                    int tot;
                    const int ex = warp_excl_scan(v, &tot);
                    if (i < W) b.ev_off[i] = run + ex;
                    run += tot;
                }
                if (lane == 0) s_total = run;
            }
            __syncthreads();
            if (!s_fail) {
                const size_t pbase = (size_t)inst * g.W * g.k;
                int32_t *const osrc = p.path_src + pbase, *const odst = p.path_dst + pbase;
                int32_t *const oev = p.path_event ? p.path_event + pbase : nullptr;
                for (int e = warp; e < W; e += nw) {
                    const int n = b.ev_count[e], off = b.ev_off[e];
                    const int dbase = b.ev_col[e] * g.H + g.H - 1;
                    const uint32_t *st = stage + (size_t)e * ks;
                    for (int i0 = 0; i0 < n; i0 += 256) {  // 8 loads in flight per lane
                        uint32_t v[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int i = i0 + 32 * u + lane;
                            v[u] = i < n ? __ldlu(st + i) : 0u;  // last use
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int i = i0 + 32 * u + lane;
                            if (i < n) {
                                // streaming stores: the output must not evict the staging from L2
                                __stcs(osrc + off + i, (int)(v[u] >> 20) * g.H + g.H - 1 - (int)((v[u] >> 10) & 1023));
                                __stcs(odst + off + i, dbase - (int)(v[u] & 1023));
                                if (oev) __stcs(oev + off + i, e);
                            }
                        }
                    }
                    // the event's staged lines are dead: drop them from L2 without write-back
                    __syncwarp();
                    for (int l = lane; 32 * l < n; l += 32)
                        asm volatile("discard.global.L2 [%0], 128;" ::"l"(st + 32 * l) : "memory");
                }
            }
            __syncthreads();
            if (p.phase_clock && inst == 0 && threadIdx.x == 0) {
                p.phase_clock[3] = clock64();
                p.phase_clock[4] = n1;
                p.phase_clock[5] = n2 * 1000 + nlev;
            }
            if (s_fail && threadIdx.x == 0) {
                s_status = RECON_ERR_INFEASIBLE;
                s_detail = RECON_D_GEN_NO_ASSIGNMENT;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const bool ok = s_status == RECON_OK;
            p.path_count[inst] = ok ? s_total : 0;
            p.total_displacement[inst] = ok ? (long long)s_disp : 0;
            p.status[inst] = s_status;
            if (p.detail) p.detail[inst] = s_detail;
        }
        if (p.events && s_status == RECON_OK) {
            for (int e = threadIdx.x; e < g.W; e += blockDim.x) {
                int32_t *ev = p.events + ((size_t)inst * g.W + e) * 4;
                ev[0] = e;
                ev[1] = b.ev_col[e];
                ev[2] = b.ev_type[e] == EV_FLUSH ? b.ev_aux[e] : -1;
                ev[3] = b.ev_type[e] == EV_OWN ? b.ev_aux[e] : -1;
            }
        }
        __syncthreads();
    }
}

template __global__ void redrec_kernel<1>(GridParams);
template __global__ void redrec_kernel<3>(GridParams);
template __global__ void redrec_kernel<4>(GridParams);

}  // namespace rb
