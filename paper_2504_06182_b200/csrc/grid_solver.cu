// Grid solvers (red-rec and bird) on sm_100a: one CTA per instance.
//
// Reference: /root/reference/proj/src/redrec.cpp:124-232, bird.cpp:54-123,
// virtual_line.cpp:97-229, exact1d.cpp:155-207, 374-407, 494-515.
//
// Layout in shared memory: every column is a depth bit plane (bit d = row d
// counted from the top, geometry.hpp:105) of wpd = ceil(H/64) u64 words.  The
// band is depths [lo, hi]; "top" reservoir is depth < lo, "bottom" > hi.
//
// Every event fills the receiver's band (targets lo..hi, virtual_line.cpp:125)
// from residents (always used), top-side tokens (virtual pos < lo) and
// bottom-side tokens (virtual pos > hi).  The reference solves it with a
// windowed DP whose tie rule is "lex-min use vector read from the last source"
// (exact1d.cpp:155-207).  For band targets that optimum is the SPLIT RULE:
// with a = number of top tokens used (mandatory ones plus the a - m_top
// optional ones nearest the band) and b = holes - a bottom tokens, cost(a) is
// convex, and the reference's tie rule picks the LARGEST minimiser.  Convexity
// makes the minimiser a count: a = a_min + #{a in (a_min, a_max] : Delta(a) <= 0}.
// The used tokens, sorted by (virtual pos, dist, column), take targets
// lo, lo+1, ... (virtual_line.cpp:112-118, 195-225), which fixes every path
// and its emission slot: rights (target > pos) by descending target, then lefts
// by ascending target (order_1d_intervals, exact1d.cpp:494-515).  The CPU
// restatement of exactly this procedure is oracle/recon_oracle.c.
//
// Engines:
//   own_*   : warp-level compaction of one column (OWN events; red-rec
//             phases 1/3 and donating compactions, bird's column pass)
//   flush   : warp-level red-rec transfer (receiver + pending marks mandatory,
//             donor reservoir optional, redrec.cpp:92-116, 169-191)
//   pooled  : CTA-level bird row-pass event; optional tokens of every column
//             are counted per virtual position with 64-level ballot windows
//             over the diagonals depth - dist (bird.cpp:35-46).

#include <cstdint>
#include <cstdio>

#include "common.cuh"
#include "grid_solver.cuh"

namespace rb {

// --------------------------------------------------------------------------
// geometry + shared-memory carve-up
// --------------------------------------------------------------------------

__host__ __device__ inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline void grid_smem_layout(const GridShape &s, GridSmem &o) {
    int64_t off = 0;
    o.dep = off;
    off += (int64_t)s.W * s.wpd * 8;
    o.keys = off;
    off += (int64_t)2 * (s.k + 2) * 4;
    o.bal = off;
    off += (int64_t)s.nchunk * 64 * 4;
    o.sigma = off;
    off += (int64_t)s.W * 4;
    o.ev_count = off;
    off += (int64_t)s.W * 4;
    o.ev_off = off;
    off += (int64_t)(s.W + 1) * 4;
    o.lvl_t = off;
    off += (int64_t)s.LT * 4;
    o.lvl_b = off;
    off += (int64_t)s.LB * 4;
    o.scal = off;
    off += 32 * 8;
    o.lists = off;
    off += (int64_t)s.nwarps * 4 * s.LK * 2;
    o.plists = off;
    off += (int64_t)2 * s.LK * 2;
    o.mark_dest = off;
    off += (int64_t)s.W * 2;
    o.ev_col = off;
    off += (int64_t)s.W * 2;
    o.ev_aux = off;
    off += (int64_t)s.W * 2;
    o.ev_a = off;
    off += (int64_t)s.W * 2;
    o.ev_type = off;
    off += s.W;
    o.solved = off;
    off += s.W;
    o.total = align_up(off, 16);
}

struct Geo {
    int W, H, k, lo, hi, wpd, B, LK, LT, LB, nchunk;
};

__device__ __forceinline__ Geo make_geo(const GridShape &s) {
    Geo g;
    g.W = s.W;
    g.H = s.H;
    g.k = s.k;
    // centered band rows y in [(H-h')/2, +h'-1] (problem.hpp:78-79) -> depths
    const int ylo = (s.H - s.k) / 2, yhi = ylo + s.k - 1;
    g.lo = s.H - 1 - yhi;
    g.hi = s.H - 1 - ylo;
    g.wpd = s.wpd;
    g.B = s.B;
    g.LK = s.LK;
    g.LT = s.LT;
    g.LB = s.LB;
    g.nchunk = s.nchunk;
    return g;
}

enum : uint8_t { EV_OWN = 0, EV_FLUSH = 1 };

// --------------------------------------------------------------------------
// warp-level compaction of one column (OWN event)
// --------------------------------------------------------------------------

struct OwnSolve {
    int a, b, R, holes, nt, nb, n_right, n_left;
};

// Lists (per warp, LK int16 each): otop[1..] = top depths, innermost first;
// obot[1..] = bottom depths, innermost first; hole[0..holes+1] = empty band
// depths with sentinels lo-1 / hi+1; res[0..R) = resident depths.
__device__ bool own_solve(const Geo &g, const uint64_t *m, int16_t *L, int forced_a, OwnSolve &s) {
    int16_t *otop = L, *obot = L + g.LK, *hole = L + 2 * g.LK, *res = L + 3 * g.LK;
    const int lane = lane_id(), B = g.B, base = lane * B;
    const uint32_t ch = lane_chunk(m, g.wpd, lane, B);
    const uint32_t bandr = chunk_range(base, B, g.lo, g.hi + 1);
    const uint32_t topm = ch & chunk_range(base, B, 0, g.lo);
    const uint32_t resm = ch & bandr;
    const uint32_t holem = ~ch & bandr;
    const uint32_t botm = ch & chunk_range(base, B, g.hi + 1, g.H);
    int nt, R, nb, nh;
    int et = warp_excl_scan(__popc(topm), &nt);
    int er = warp_excl_scan(__popc(resm), &R);
    int eb = warp_excl_scan(__popc(botm), &nb);
    int eh = warp_excl_scan(__popc(holem), &nh);
    const int holes = nh;
    for (uint32_t x = topm; x; x &= x - 1, ++et) {
        const int desc = nt - 1 - et;
        if (desc < holes) otop[desc + 1] = (int16_t)(base + __ffs(x) - 1);
    }
    for (uint32_t x = botm; x; x &= x - 1, ++eb)
        if (eb < holes) obot[eb + 1] = (int16_t)(base + __ffs(x) - 1);
    for (uint32_t x = holem; x; x &= x - 1, ++eh) hole[eh + 1] = (int16_t)(base + __ffs(x) - 1);
    for (uint32_t x = resm; x; x &= x - 1, ++er) res[er] = (int16_t)(base + __ffs(x) - 1);
    if (lane == 0) {
        hole[0] = (int16_t)(g.lo - 1);
        hole[holes + 1] = (int16_t)(g.hi + 1);
    }
    __syncwarp();
    const int amin = max(0, holes - nb), amax = min(nt, holes);
    if (amin > amax) return false;
    int a = forced_a;
    if (a < 0) {
        int cnt = 0;
        for (int a0 = amin + 1; a0 <= amax; a0 += 32) {
            const int aa = a0 + lane;
            bool le = false;
            if (aa <= amax) {
                const int delta = (g.lo + aa - 1) - otop[aa] + 2 * (hole[aa] - g.lo - aa + 1) - R -
                                  obot[holes - aa + 1] + g.hi - (holes - aa);
                le = delta <= 0;
            }
            cnt += __popc(__ballot_sync(FULL, le));
        }
        a = amin + cnt;
    }
    s.a = a;
    s.b = holes - a;
    s.R = R;
    s.holes = holes;
    s.nt = nt;
    s.nb = nb;
    const int cntE = hole[a] - g.lo - a + 1;
    const int nstat = hole[a + 1] - hole[a] - 1;
    s.n_right = a + cntE;
    s.n_left = (R - cntE - nstat) + s.b;
    return true;
}

__device__ __forceinline__ int emit_slot(const Geo &g, int j, int n_right, int n_left) {
    return j < n_right ? n_right - 1 - j : n_right + j - (g.k - n_left);
}

struct PathOut {
    int32_t *src, *dst, *ev;
};

// Emits the paths of a solved OWN event at [off, off + count); returns the
// event's total displacement (warp-uniform).
__device__ long long own_emit(const Geo &g, int col, const OwnSolve &s, const int16_t *L, PathOut o,
                              int off, int evid) {
    const int16_t *otop = L, *obot = L + g.LK, *res = L + 3 * g.LK;
    long long disp = 0;
    for (int j = lane_id(); j < g.k; j += 32) {
        const bool right = j < s.n_right, left = j >= g.k - s.n_left;
        if (!right && !left) continue;
        const int depth = j < s.a ? otop[s.a - j] : (j < s.a + s.R ? res[j - s.a] : obot[j - s.a - s.R + 1]);
        const int t = g.lo + j;
        const int p = off + emit_slot(g, j, s.n_right, s.n_left);
        o.src[p] = col * g.H + (g.H - 1 - depth);
        o.dst[p] = col * g.H + (g.H - 1 - t);
        if (o.ev) o.ev[p] = evid;
        disp += t > depth ? t - depth : depth - t;
    }
    return warp_sum64(disp);
}

// Column after its OWN event: band full, used reservoir tokens gone, parked
// (unused) reservoir tokens stay (redrec.cpp:150-164, bird.cpp:90-99).
// Returns the parked count.
__device__ int own_update(const Geo &g, uint64_t *m, const OwnSolve &s, const int16_t *L) {
    const int16_t *otop = L, *obot = L + g.LK;
    const int thr_t = s.a >= 1 ? otop[s.a] : g.lo;
    const int thr_b = s.b >= 1 ? obot[s.b] : g.hi;
    __syncwarp();
    for (int w = lane_id(); w < g.wpd; w += 32) {
        const uint64_t keep = word_range(64 * w, 0, thr_t) | word_range(64 * w, thr_b + 1, g.H);
        m[w] = (m[w] & keep) | word_range(64 * w, g.lo, g.hi + 1);
    }
    __syncwarp();
    return (s.nt - s.a) + (s.nb - s.b);
}

// --------------------------------------------------------------------------
// warp-level red-rec transfer (FLUSH)
// --------------------------------------------------------------------------

__device__ __forceinline__ uint32_t tok_key(int v, int dist, int col) {
    return ((uint32_t)(v + 2048) << 20) | ((uint32_t)dist << 10) | (uint32_t)col;
}

// Receiver r's own tokens and the marks parked for it are mandatory; donor
// d's reservoir is the optional pool (build_redistribution_instance,
// redrec.cpp:92-116).  Emits at `off`, updates state (redrec.cpp:169-191).
// Returns the path count, or -1 on an infeasible instance.
__device__ int flush_event(const Geo &g, uint64_t *dep, int16_t *mark_dest, int r, int d, int16_t *L,
                           uint32_t *keys, PathOut o, int off, int evid, long long *disp_out) {
    int16_t *otop = L, *obot = L + g.LK, *hole = L + 2 * g.LK, *res = L + 3 * g.LK;
    const int lane = lane_id(), B = g.B, base = lane * B;
    const uint64_t *mr = dep + (size_t)r * g.wpd;
    uint64_t *md = dep + (size_t)d * g.wpd;
    const int dd = d > r ? d - r : r - d;
    const uint32_t rtop = chunk_range(base, B, 0, g.lo), rband = chunk_range(base, B, g.lo, g.hi + 1),
                   rbot = chunk_range(base, B, g.hi + 1, g.H);
    // receiver: residents, holes, mandatory reservoir
    const uint32_t chr = lane_chunk(mr, g.wpd, lane, B);
    const uint32_t resm = chr & rband, holem = ~chr & rband;
    int R, nh;
    int er = warp_excl_scan(__popc(resm), &R);
    int eh = warp_excl_scan(__popc(holem), &nh);
    const int holes = nh;
    for (uint32_t x = holem; x; x &= x - 1, ++eh) hole[eh + 1] = (int16_t)(base + __ffs(x) - 1);
    for (uint32_t x = resm; x; x &= x - 1, ++er) res[er] = (int16_t)(base + __ffs(x) - 1);
    int m_top = __popc(chr & rtop), m_bot = __popc(chr & rbot);
    long long s_top = 0, s_bot = 0;
    for (uint32_t x = chr & rtop; x; x &= x - 1) s_top += base + __ffs(x) - 1;
    for (uint32_t x = chr & rbot; x; x &= x - 1) s_bot += base + __ffs(x) - 1;
    // marks (pending parked tokens of donating columns, redrec.cpp:155-160)
    for (int x0 = 0; x0 < g.W; x0 += 32) {
        unsigned mk = __ballot_sync(FULL, x0 + lane < g.W && mark_dest[x0 + lane] == r);
        while (mk) {
            const int x = x0 + __ffs(mk) - 1;
            mk &= mk - 1;
            const int dx = x > r ? x - r : r - x;
            const uint32_t chx = lane_chunk(dep + (size_t)x * g.wpd, g.wpd, lane, B);
            for (uint32_t y = chx & rtop; y; y &= y - 1, ++m_top) s_top += base + __ffs(y) - 1 - dx;
            for (uint32_t y = chx & rbot; y; y &= y - 1, ++m_bot) s_bot += base + __ffs(y) - 1 + dx;
        }
    }
    m_top = warp_sum(m_top);
    m_bot = warp_sum(m_bot);
    s_top = warp_sum64(s_top);
    s_bot = warp_sum64(s_bot);
    (void)s_top;
    (void)s_bot;
    // donor reservoir: optional streams, innermost first
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
    if (amin > amax) return -1;
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
    const int a = amin + cnt, b = holes - a;
    const int xa = a - m_top, xb = b - m_bot;  // donor tokens drawn per side
    const int cntE = hole[a] - g.lo - a + 1;
    const int nstat = hole[a + 1] - hole[a] - 1;
    const int n_right = a + cntE, n_left = (R - cntE - nstat) + b;
    // gather used top / bottom keys (a and b of them)
    uint32_t *ktop = keys, *kbot = keys + g.LK;
    {
        int tot;
        int e = warp_excl_scan(__popc(chr & rtop), &tot);
        for (uint32_t x = chr & rtop; x; x &= x - 1) ktop[e++] = tok_key(base + __ffs(x) - 1, 0, r);
        int pos_t = tot;
        e = warp_excl_scan(__popc(chr & rbot), &tot);
        for (uint32_t x = chr & rbot; x; x &= x - 1) kbot[e++] = tok_key(base + __ffs(x) - 1, 0, r);
        int pos_b = tot;
        for (int x0 = 0; x0 < g.W; x0 += 32) {
            unsigned mk = __ballot_sync(FULL, x0 + lane < g.W && mark_dest[x0 + lane] == r);
            while (mk) {
                const int x = x0 + __ffs(mk) - 1;
                mk &= mk - 1;
                const int dx = x > r ? x - r : r - x;
                const uint32_t chx = lane_chunk(dep + (size_t)x * g.wpd, g.wpd, lane, B);
                e = warp_excl_scan(__popc(chx & rtop), &tot);
                for (uint32_t y = chx & rtop; y; y &= y - 1) ktop[pos_t + e++] = tok_key(base + __ffs(y) - 1 - dx, dx, x);
                pos_t += tot;
                e = warp_excl_scan(__popc(chx & rbot), &tot);
                for (uint32_t y = chx & rbot; y; y &= y - 1) kbot[pos_b + e++] = tok_key(base + __ffs(y) - 1 + dx, dx, x);
                pos_b += tot;
            }
        }
        // donor: innermost xa top (largest depth), innermost xb bottom
        e = warp_excl_scan(__popc(dtop), &tot);
        for (uint32_t x = dtop; x; x &= x - 1, ++e) {
            const int desc = n_ot - 1 - e;
            if (desc < xa) ktop[pos_t + desc] = tok_key(base + __ffs(x) - 1 - dd, dd, d);
        }
        e = warp_excl_scan(__popc(dbot), &tot);
        for (uint32_t x = dbot; x; x &= x - 1, ++e)
            if (e < xb) kbot[pos_b + e] = tok_key(base + __ffs(x) - 1 + dd, dd, d);
    }
    __syncwarp();
    long long disp = 0;
    // top used: sorted index by rank among keys (distinct)
    for (int i = lane; i < a; i += 32) {
        const uint32_t key = ktop[i];
        int rank = 0;
        for (int q = 0; q < a; ++q) rank += ktop[q] < key;
        const int v = (int)(key >> 20) - 2048, dist = (key >> 10) & 1023, col = key & 1023;
        const int depth = v + dist, j = rank, t = g.lo + j;
        const int p = off + emit_slot(g, j, n_right, n_left);
        o.src[p] = col * g.H + (g.H - 1 - depth);
        o.dst[p] = r * g.H + (g.H - 1 - t);
        if (o.ev) o.ev[p] = evid;
        disp += t - v;
    }
    for (int i = lane; i < b; i += 32) {
        const uint32_t key = kbot[i];
        int rank = 0;
        for (int q = 0; q < b; ++q) rank += kbot[q] < key;
        const int v = (int)(key >> 20) - 2048, dist = (key >> 10) & 1023, col = key & 1023;
        const int depth = v - dist, j = a + R + rank, t = g.lo + j;
        const int p = off + emit_slot(g, j, n_right, n_left);
        o.src[p] = col * g.H + (g.H - 1 - depth);
        o.dst[p] = r * g.H + (g.H - 1 - t);
        if (o.ev) o.ev[p] = evid;
        disp += v - t;
    }
    for (int i = lane; i < R; i += 32) {
        const int depth = res[i], j = a + i, t = g.lo + j;
        if (t == depth) continue;
        const int p = off + emit_slot(g, j, n_right, n_left);
        o.src[p] = r * g.H + (g.H - 1 - depth);
        o.dst[p] = r * g.H + (g.H - 1 - t);
        if (o.ev) o.ev[p] = evid;
        disp += t > depth ? t - depth : depth - t;
    }
    *disp_out = warp_sum64(disp);
    // state: donor loses its drawn innermost tokens; receiver and its markers
    // keep only band cells; marks cleared
    const int thr_t = xa >= 1 ? otop[xa] + dd : g.lo;     // clear donor top depth >= thr_t
    const int thr_b = xb >= 1 ? obot[xb] - dd : g.hi;     // clear donor bottom depth <= thr_b
    __syncwarp();
    for (int w = lane; w < g.wpd; w += 32) {
        const uint64_t band = word_range(64 * w, g.lo, g.hi + 1);
        md[w] &= ~(word_range(64 * w, thr_t, g.lo) | word_range(64 * w, g.hi + 1, thr_b + 1));
        dep[(size_t)r * g.wpd + w] = band;
    }
    for (int x0 = 0; x0 < g.W; x0 += 32) {
        const bool is = x0 + lane < g.W && mark_dest[x0 + lane] == r;
        unsigned mk = __ballot_sync(FULL, is);
        while (mk) {
            const int x = x0 + __ffs(mk) - 1;
            mk &= mk - 1;
            for (int w = lane; w < g.wpd; w += 32) dep[(size_t)x * g.wpd + w] = word_range(64 * w, g.lo, g.hi + 1);
        }
        __syncwarp();
        if (is) mark_dest[x0 + lane] = -1;
    }
    __syncwarp();
    return n_right + n_left;
}

// --------------------------------------------------------------------------
// red-rec control plane (surplus-only replay of redrec.cpp:205-232)
// --------------------------------------------------------------------------

// Emits the event plan: type, column, donor / mark destination.  Runs on one
// warp over W columns held in shared memory (sigma, solved are clobbered).
// Returns 0 or a LOGIC detail code.
__device__ int redrec_plan(const Geo &g, int *sig, uint8_t *solved, uint8_t *ev_type, int16_t *ev_col,
                           int16_t *ev_aux, int *n_phase1, int *n_loop) {
    const int lane = lane_id(), W = g.W;
    const int per = (W + 31) / 32, c0 = lane * per, c1 = min(W, c0 + per);
    int nev = 0;
    // phase 1: sigma == 0 columns ascending (redrec.cpp:211-212)
    for (int x0 = 0; x0 < W; x0 += 32) {
        const int c = x0 + lane;
        const bool z = c < W && sig[c] == 0;
        const unsigned bz = __ballot_sync(FULL, z);
        if (z) {
            const int slot = nev + __popc(bz & lanemask_lt());
            ev_type[slot] = EV_OWN;
            ev_col[slot] = (int16_t)c;
            ev_aux[slot] = -1;
            solved[c] = 1;
        }
        nev += __popc(bz);
    }
    *n_phase1 = nev;
    __syncwarp();
    // pairing loop (redrec.cpp:214-226)
    for (;;) {
        // nearest non-transit column to the left of each column (transit =
        // solved with zero surplus, scan_for_donor redrec.cpp:43-51)
        int lastL = -1;
        for (int c = c0; c < c1; ++c)
            if (!(solved[c] && sig[c] == 0)) lastL = c;
        int firstR = W;
        for (int c = c1 - 1; c >= c0; --c)
            if (!(solved[c] && sig[c] == 0)) firstR = c;
        // exclusive max-scan from the left, min-scan from the right
        int inL = lastL;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, inL, o);
            if (lane >= o) inL = max(inL, y);
        }
        int exL = __shfl_up_sync(FULL, inL, 1);
        if (lane == 0) exL = -1;
        int inR = firstR;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_down_sync(FULL, inR, o);
            if (lane + o < 32) inR = min(inR, y);
        }
        int exR = __shfl_down_sync(FULL, inR, 1);
        if (lane == 31) exR = W;
        // candidates, key (-exchange, |d-r|, deficit-exchange, r, d) packed
        unsigned long long best = ~0ull;
        bool any_recv = false;
        int left = exL;
        for (int r = c0; r < c1; ++r) {
            const bool transit = solved[r] && sig[r] == 0;
            if (!solved[r] && sig[r] < 0) {
                any_recv = true;
                int right = exR;
                for (int c = r + 1; c < c1; ++c)
                    if (!(solved[c] && sig[c] == 0)) {
                        right = c;
                        break;
                    }
                for (int side = 0; side < 2; ++side) {
                    const int d = side == 0 ? left : right;
                    if (d < 0 || d >= W || solved[d] || sig[d] <= 0) continue;
                    const int deficit = -sig[r];
                    const int ex = min(sig[d], deficit);
                    const unsigned long long key =
                        ((unsigned long long)(4095 - ex) << 42) | ((unsigned long long)(d > r ? d - r : r - d) << 32) |
                        ((unsigned long long)(deficit - ex) << 20) | ((unsigned long long)r << 10) | (unsigned long long)d;
                    best = key < best ? key : best;
                }
            }
            if (!transit) left = r;
        }
        any_recv = __any_sync(FULL, any_recv);
        if (!any_recv) break;
        best = warp_min_u64(best);
        if (best == ~0ull) return RECON_D_NO_DONOR;
        const int d = (int)(best & 1023), r = (int)((best >> 10) & 1023);
        const int ds = sig[d], def = -sig[r];
        __syncwarp();
        if (lane == 0) {
            if (ds < def) {
                ev_type[nev] = EV_OWN;
                ev_col[nev] = (int16_t)d;
                ev_aux[nev] = (int16_t)r;
                sig[r] += ds;
                sig[d] = 0;
                solved[d] = 1;
            } else {
                ev_type[nev] = EV_FLUSH;
                ev_col[nev] = (int16_t)r;
                ev_aux[nev] = (int16_t)d;
                sig[d] -= def;
                sig[r] = 0;
                solved[r] = 1;
                if (ds == def) {
                    ev_type[nev + 1] = EV_OWN;
                    ev_col[nev + 1] = (int16_t)d;
                    ev_aux[nev + 1] = -1;
                    solved[d] = 1;
                }
            }
        }
        nev += (ds < def) ? 1 : (ds == def ? 2 : 1);
        __syncwarp();
    }
    *n_loop = nev - *n_phase1;
    // phase 3: remaining columns ascending (redrec.cpp:228-229)
    for (int x0 = 0; x0 < W; x0 += 32) {
        const int c = x0 + lane;
        const bool u = c < W && !solved[c];
        const unsigned bu = __ballot_sync(FULL, u);
        if (u) {
            const int slot = nev + __popc(bu & lanemask_lt());
            ev_type[slot] = EV_OWN;
            ev_col[slot] = (int16_t)c;
            ev_aux[slot] = -1;
        }
        nev += __popc(bu);
    }
    __syncwarp();
    return 0;
}

// --------------------------------------------------------------------------
// CTA-level pooled event (bird row pass)
// --------------------------------------------------------------------------

__device__ __forceinline__ int slot_col(int c, int gslot, int W) {
    if (gslot == 0) return c;
    const int dl = (gslot + 1) >> 1;
    const int x = (gslot & 1) ? c - dl : c + dl;
    return (x >= 0 && x < W) ? x : -1;
}

struct PooledScratch {
    int16_t *otop, *obot;      // [LK]
    int *lvl_t, *lvl_b;        // [LT], [LB]: count << 16 | cum_before (cum < 65536)
    uint32_t *bal;             // [nchunk][64]
    int *scal;                 // scalars
};

// 64 ballots per warp: per-level token counts of the slots this warp holds
__device__ __forceinline__ void ballot_counts(uint64_t word, uint32_t *bal_row, int *cnt_lo, int *cnt_hi) {
    const int lane = lane_id();
#pragma unroll 8
    for (int i = 0; i < 64; ++i) {
        const uint32_t b = __ballot_sync(FULL, (word >> i) & 1ull);
        if (bal_row && lane == 0) bal_row[i] = b;
        if (i < 32) {
            if (lane == i) *cnt_lo = __popc(b);
        } else {
            if (lane == i - 32) *cnt_hi = __popc(b);
        }
    }
}

// token word of a slot: bit i = a reservoir token at virtual level V0 + i
__device__ __forceinline__ uint64_t slot_word(const Geo &g, const uint64_t *dep, int c, int gslot, int nslots,
                                              int V0, bool top, int *col_out, int *dist_out) {
    *col_out = -1;
    *dist_out = 0;
    if (gslot >= nslots) return 0ull;
    const int x = slot_col(c, gslot, g.W);
    if (x < 0) return 0ull;
    const int dist = x > c ? x - c : c - x;
    *col_out = x;
    *dist_out = dist;
    const uint64_t *m = dep + (size_t)x * g.wpd;
    if (top) {
        // depth = v + dist < lo
        const int start = V0 + dist;
        const uint64_t w = extract64(m, g.wpd, start);
        const int nvalid = g.lo - start;  // bits i < nvalid have depth < lo
        if (nvalid <= 0) return 0ull;
        return nvalid >= 64 ? w : (w & ((1ull << nvalid) - 1ull));
    } else {
        // depth = v - dist > hi
        const int start = V0 - dist;
        const uint64_t w = extract64(m, g.wpd, start);
        const int skip = g.hi + 1 - start;  // bits i < skip have depth <= hi
        if (skip >= 64) return 0ull;
        return skip <= 0 ? w : (w & ~((1ull << skip) - 1ull));
    }
}

// Scans 64-level windows outward from the band until `need` tokens are found
// or no token can exist further out.  Fills lvl[] (count << 16 | cum_before).
// Returns total found (scalars: found, nlevels) — CTA-uniform.
__device__ void pooled_scan(const Geo &g, const uint64_t *dep, int c, bool top, int need, int *lvl,
                            int *scal_found, int *scal_nlev) {
    const int lane = lane_id(), warp = warp_id(), nw = blockDim.x >> 5;
    const int maxlev = top ? (g.lo + g.W - 1) : ((g.H - 1 - g.hi) + g.W - 1);  // levels available
    int found = 0, nlev = 0;
    for (int w = 0; nlev < maxlev && found < need; ++w) {
        const int V0 = top ? g.lo - 64 * (w + 1) : g.hi + 1 + 64 * w;
        const int maxd = min(g.W - 1, 64 * (w + 1));
        const int nslots = 2 * maxd + 1;
        const int base_li = 64 * w;  // level index of the level nearest the band in this window
        for (int i = threadIdx.x; i < 64; i += blockDim.x) lvl[base_li + i] = 0;
        __syncthreads();
        for (int chn = warp; chn * 32 < nslots; chn += nw) {
            int col, dist;
            const uint64_t word = slot_word(g, dep, c, chn * 32 + lane, nslots, V0, top, &col, &dist);
            if (!__any_sync(FULL, word != 0ull)) continue;
            int clo = 0, chi = 0;
            ballot_counts(word, nullptr, &clo, &chi);
            // window bit i <-> level index: top li = 63 - i + base_li; bottom li = i + base_li
            if (clo) atomicAdd(&lvl[base_li + (top ? 63 - lane : lane)], clo);
            if (chi) atomicAdd(&lvl[base_li + (top ? 31 - lane : lane + 32)], chi);
        }
        __syncthreads();
        // cumulative (warp 0): li ascending = outward from the band
        if (warp == 0) {
            int run = found;
            for (int i0 = 0; i0 < 64; i0 += 32) {
                const int li = base_li + i0 + lane;
                const int cnt = lvl[li];
                int tot;
                const int ex = warp_excl_scan(cnt, &tot);
                lvl[li] = (cnt << 16) | min(run + ex, 65535);
                run += tot;
            }
            if (lane == 0) *scal_found = run;
        }
        __syncthreads();
        found = *scal_found;
        nlev = 64 * (w + 1);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *scal_found = found;
        *scal_nlev = nlev;
    }
    __syncthreads();
}

// Emits the used reservoir tokens of one side and clears them from their
// columns (drawn externals leave their reservoirs, bird.cpp:79-88).
__device__ long long pooled_emit_side(const Geo &g, uint64_t *dep, int *sigma, int c, bool top, int used,
                                      int a, int R, int n_right, int n_left, const int *lvl, uint32_t *bal,
                                      int vstar_li, int r_star, PathOut o, int off, int evid) {
    const int lane = lane_id(), warp = warp_id(), nw = blockDim.x >> 5;
    long long disp = 0;
    if (used <= 0) return 0;
    const int last_w = vstar_li / 64;
    for (int w = 0; w <= last_w; ++w) {
        const int V0 = top ? g.lo - 64 * (w + 1) : g.hi + 1 + 64 * w;
        const int maxd = min(g.W - 1, 64 * (w + 1));
        const int nslots = 2 * maxd + 1;
        const int nch = (nslots + 31) / 32;
        // pass 1: ballots per chunk (group-order prefix within a level)
        for (int chn = warp; chn < nch; chn += nw) {
            int col, dist;
            const uint64_t word = slot_word(g, dep, c, chn * 32 + lane, nslots, V0, top, &col, &dist);
            int clo, chi;
            ballot_counts(word, bal + chn * 64, &clo, &chi);
        }
        __syncthreads();
        // pass 2: emit
        for (int chn = warp; chn < nch; chn += nw) {
            int col, dist;
            const int gslot = chn * 32 + lane;
            uint64_t word = slot_word(g, dep, c, gslot, nslots, V0, top, &col, &dist);
            uint64_t cleared = 0ull;
            for (uint64_t x = word; x; x &= x - 1) {
                const int i = __ffsll((long long)x) - 1;
                const int li = top ? 64 * w + 63 - i : 64 * w + i;
                if (li > vstar_li) continue;  // beyond the last used level
                int rank_lt = __popc(bal[chn * 64 + i] & lanemask_lt());
                for (int q = 0; q < chn; ++q) rank_lt += __popc(bal[q * 64 + i]);
                int jside;
                if (li == vstar_li) {
                    if (rank_lt >= r_star) continue;
                    jside = top ? rank_lt : (used - 1 - (r_star - 1 - rank_lt));
                } else {
                    const int cb = lvl[li] & 0xffff, cnt = lvl[li] >> 16;
                    // top: ascending (pos, g) index = used - (#at levels nearer + this level) + rank
                    // bottom: ascending index = levels nearer + rank
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
                // clear bits depth = start + i
                for (uint64_t x = cleared; x; x &= x - 1) {
                    const int dpt = start + __ffsll((long long)x) - 1;
                    m[dpt >> 6] &= ~(1ull << (dpt & 63));
                }
                if (col != c) sigma[col] -= __popcll(cleared);
            }
        }
        __syncthreads();
    }
    return disp;
}

// One bird row-pass event for column c (BirdRunner::solve_column(c, true)).
// Returns the path count (CTA-uniform) or -1 when infeasible.
__device__ int pooled_event(const Geo &g, uint64_t *dep, int *sigma, int c, int16_t *L0, PooledScratch ps,
                            PathOut o, int off, int evid, unsigned long long *disp_acc) {
    const int lane = lane_id(), warp = warp_id();
    int16_t *hole = L0 + 2 * g.LK, *res = L0 + 3 * g.LK;
    int *S = ps.scal;
    // A: own residents and holes (warp 0)
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
            S[0] = R;
            S[1] = nh;
        }
    }
    __syncthreads();
    const int R = S[0], holes = S[1];
    // B/C: optional streams per side
    pooled_scan(g, dep, c, true, holes, ps.lvl_t, &S[2], &S[3]);
    pooled_scan(g, dep, c, false, holes, ps.lvl_b, &S[4], &S[5]);
    const int found_t = S[2], nlev_t = S[3], found_b = S[4], nlev_b = S[5];
    // D: materialize otop/obot (1-based, innermost first)
    for (int li = threadIdx.x; li < nlev_t; li += blockDim.x) {
        const int cnt = ps.lvl_t[li] >> 16, cb = ps.lvl_t[li] & 0xffff;
        for (int q = cb + 1; q <= min(cb + cnt, holes); ++q) ps.otop[q] = (int16_t)(g.lo - 1 - li);
    }
    for (int li = threadIdx.x; li < nlev_b; li += blockDim.x) {
        const int cnt = ps.lvl_b[li] >> 16, cb = ps.lvl_b[li] & 0xffff;
        for (int q = cb + 1; q <= min(cb + cnt, holes); ++q) ps.obot[q] = (int16_t)(g.hi + 1 + li);
    }
    if (threadIdx.x == 0) S[6] = 0;
    __syncthreads();
    const int n_ot = found_t, n_ob = found_b;  // exact when < holes, else >= holes
    const int amin = max(0, holes - n_ob), amax = min(n_ot, holes);
    if (amin > amax) return -1;
    // E: a = amin + #{Delta(a) <= 0}
    {
        int cnt = 0;
        for (int a0 = amin + 1 + warp * 32; a0 <= amax; a0 += blockDim.x) {
            const int aa = a0 + lane;
            bool le = false;
            if (aa <= amax) {
                const int delta = (g.lo + aa - 1) - ps.otop[aa] + 2 * (hole[aa] - g.lo - aa + 1) - R -
                                  ps.obot[holes - aa + 1] + g.hi - (holes - aa);
                le = delta <= 0;
            }
            cnt += __popc(__ballot_sync(FULL, le));
        }
        if (lane == 0 && cnt) atomicAdd(&S[6], cnt);
    }
    __syncthreads();
    const int a = amin + S[6], b = holes - a;
    const int cntE = hole[a] - g.lo - a + 1;
    const int nstat = hole[a + 1] - hole[a] - 1;
    const int n_right = a + cntE, n_left = (R - cntE - nstat) + b;
    // F: last used level and how many of its members (group order) are used
    int vt_li = -1, rt = 0, vb_li = -1, rb = 0;
    if (a >= 1) {
        vt_li = g.lo - 1 - ps.otop[a];
        rt = a - (ps.lvl_t[vt_li] & 0xffff);
    }
    if (b >= 1) {
        vb_li = ps.obot[b] - (g.hi + 1);
        rb = b - (ps.lvl_b[vb_li] & 0xffff);
    }
    __syncthreads();
    // G/H: emit + clear drawn tokens
    long long disp = 0;
    disp += pooled_emit_side(g, dep, sigma, c, true, a, a, R, n_right, n_left, ps.lvl_t, ps.bal, vt_li, rt, o, off,
                             evid);
    disp += pooled_emit_side(g, dep, sigma, c, false, b, a, R, n_right, n_left, ps.lvl_b, ps.bal, vb_li, rb, o,
                             off, evid);
    // I: residents
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
    // J: own column = band + unused own reservoir (bird.cpp:90-99)
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

// --------------------------------------------------------------------------
// the kernels
// --------------------------------------------------------------------------

struct Block {
    uint64_t *dep;
    uint32_t *keys, *bal;
    int *sigma, *ev_count, *ev_off, *lvl_t, *lvl_b, *scal;
    int16_t *lists, *plists, *mark_dest, *ev_col, *ev_aux, *ev_a;
    uint8_t *ev_type, *solved;
};

__device__ Block carve(const GridShape &s, unsigned char *smem) {
    GridSmem o;
    grid_smem_layout(s, o);
    Block b;
    b.dep = (uint64_t *)(smem + o.dep);
    b.keys = (uint32_t *)(smem + o.keys);
    b.bal = (uint32_t *)(smem + o.bal);
    b.sigma = (int *)(smem + o.sigma);
    b.ev_count = (int *)(smem + o.ev_count);
    b.ev_off = (int *)(smem + o.ev_off);
    b.lvl_t = (int *)(smem + o.lvl_t);
    b.lvl_b = (int *)(smem + o.lvl_b);
    b.scal = (int *)(smem + o.scal);
    b.lists = (int16_t *)(smem + o.lists);
    b.plists = (int16_t *)(smem + o.plists);
    b.mark_dest = (int16_t *)(smem + o.mark_dest);
    b.ev_col = (int16_t *)(smem + o.ev_col);
    b.ev_aux = (int16_t *)(smem + o.ev_aux);
    b.ev_a = (int16_t *)(smem + o.ev_a);
    b.ev_type = (uint8_t *)(smem + o.ev_type);
    b.solved = (uint8_t *)(smem + o.solved);
    return b;
}

// occ column (bit y from the bottom) -> depth plane (bit d = H-1-y); counts
__device__ void load_instance(const Geo &g, const uint64_t *occ, Block &b, long long *total_tokens) {
    const int wpc = g.wpd;  // same word count per column in both layouts
    const int shift = 64 * wpc - g.H;
    long long tot = 0;
    for (int x = threadIdx.x; x < g.W; x += blockDim.x) {
        const uint64_t *src = occ + (size_t)x * wpc;
        uint64_t *dst = b.dep + (size_t)x * g.wpd;
        int cnt = 0;
        const uint64_t last_mask = (g.H & 63) ? ((1ull << (g.H & 63)) - 1ull) : ~0ull;
        for (int j = 0; j < wpc; ++j) {
            // reversed word j = brev(src[wpc-1-j]); then shift right by `shift` across words
            const uint64_t lo = __brevll(src[wpc - 1 - j] & (j == 0 ? last_mask : ~0ull));
            const uint64_t hi = (j + 1 < wpc) ? __brevll(src[wpc - 2 - j] & (j + 1 == 0 ? last_mask : ~0ull)) : 0ull;
            const uint64_t v = shift == 0 ? lo : ((lo >> shift) | (hi << (64 - shift)));
            dst[j] = v;
            cnt += __popcll(v);
        }
        b.sigma[x] = cnt - g.k;
        b.solved[x] = 0;
        b.mark_dest[x] = -1;
        tot += cnt;
    }
    tot = warp_sum64(tot);
    if (lane_id() == 0 && tot) atomicAdd((unsigned long long *)total_tokens, (unsigned long long)tot);
}

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

__global__ void __launch_bounds__(256) redrec_kernel(GridParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geo g = make_geo(p.shape);
    Block b = carve(p.shape, smem);
    const int warp = warp_id(), lane = lane_id();
    __shared__ long long s_tokens;
    __shared__ unsigned long long s_disp;
    __shared__ int s_status, s_detail, s_n1, s_n2, s_base1, s_base2, s_fail;
    for (int inst = blockIdx.x; inst < p.count; inst += gridDim.x) {
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
            s_status = RECON_ERR_INFEASIBLE;  // Problem::check (problem.hpp:113-116)
            s_detail = RECON_D_FEWER_SOURCES;
        }
        __syncthreads();
        if (s_status == RECON_OK && warp == 0) {
            int n1 = 0, n2 = 0;
            // plan works on copies: sigma -> ev_count scratch, solved -> ev_type high bits? use ev_off
            int *sig = b.ev_off;  // W+1 ints of scratch
            uint8_t *sol = b.solved;
            for (int c = lane; c < g.W; c += 32) sig[c] = b.sigma[c];
            __syncwarp();
            const int rc = redrec_plan(g, sig, sol, b.ev_type, b.ev_col, b.ev_aux, &n1, &n2);
            if (lane == 0) {
                s_n1 = n1;
                s_n2 = n2;
                if (rc) {
                    s_status = RECON_ERR_LOGIC;
                    s_detail = rc;
                }
            }
        }
        __syncthreads();
        if (s_status == RECON_OK) {
            const int n1 = s_n1, n2 = s_n2, W = g.W;
            // phase 1: sigma==0 compactions (no state change matters afterwards)
            own_count_range(g, b, 0, n1, 0, &s_fail);
            __syncthreads();
            if (warp == 0) {
                const int t = scan_counts(b, 0, n1);
                if (lane == 0) s_base1 = t;
            }
            __syncthreads();
            if (warp == 0) {
                // pairing loop, sequential (redrec.cpp:214-226)
                int off = s_base1;
                long long disp = 0;
                int16_t *L = b.lists;
                for (int e = n1; e < n1 + n2; ++e) {
                    const int col = b.ev_col[e], aux = b.ev_aux[e];
                    if (b.ev_type[e] == EV_OWN) {
                        OwnSolve s;
                        if (!own_solve(g, b.dep + (size_t)col * g.wpd, L, -1, s)) {
                            if (lane == 0) s_fail = 1;
                            break;
                        }
                        disp += own_emit(g, col, s, L, o, off, e);
                        own_update(g, b.dep + (size_t)col * g.wpd, s, L);
                        if (aux >= 0 && lane == 0) b.mark_dest[col] = (int16_t)aux;  // parked -> marks
                        off += s.n_right + s.n_left;
                        __syncwarp();
                    } else {
                        long long dd = 0;
                        const int cnt = flush_event(g, b.dep, b.mark_dest, col, aux, L, b.keys, o, off, e, &dd);
                        if (cnt < 0) {
                            if (lane == 0) s_fail = 1;
                            break;
                        }
                        disp += dd;
                        off += cnt;
                    }
                }
                if (lane == 0) {
                    s_base2 = off;
                    if (disp) atomicAdd(&s_disp, (unsigned long long)disp);
                }
            } else {
                own_emit_range(g, b, 0, n1, 1, o, 0, false, &s_disp);
            }
            __syncthreads();
            // phase 3: remaining columns (current state)
            own_count_range(g, b, n1 + n2, W, 0, &s_fail);
            __syncthreads();
            if (warp == 0) {
                const int t = scan_counts(b, n1 + n2, W);
                if (lane == 0) s_base1 = s_base2 + t;  // total paths
            }
            __syncthreads();
            own_emit_range(g, b, n1 + n2, W, 0, o, s_base2, false, &s_disp);
            __syncthreads();
            if (s_fail && threadIdx.x == 0) {
                s_status = RECON_ERR_INFEASIBLE;
                s_detail = RECON_D_GEN_NO_ASSIGNMENT;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const bool ok = s_status == RECON_OK;
            p.path_count[inst] = ok ? s_base1 : 0;
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

__global__ void __launch_bounds__(256) bird_kernel(GridParams p) {
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
    for (int inst = blockIdx.x; inst < p.count; inst += gridDim.x) {
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
            // row pass: pooled events, strictly sequential
            for (int e = n1; e < g.W; ++e) {
                const int c = b.ev_col[e];
                const int cnt = pooled_event(g, b.dep, b.sigma, c, b.lists, ps, o, s_off, e, &s_disp);
                if (cnt < 0) {
                    if (threadIdx.x == 0) s_fail = 1;
                    __syncthreads();
                    break;
                }
                __syncthreads();
                if (threadIdx.x == 0) s_off += cnt;
                __syncthreads();
            }
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

// --------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------

bool grid_shape(int W, int H, int k, int nwarps, GridShape &s) {
    if (W <= 0 || H <= 0 || W > 1024 || H > 1024) return false;
    s.W = W;
    s.H = H;
    s.k = k;
    s.wpd = (H + 63) / 64;
    const int need = (H + 31) / 32;
    s.B = need <= 8 ? 8 : (need <= 16 ? 16 : 32);
    s.LK = k + 2;
    const int ylo = (H - k) / 2, yhi = ylo + k - 1;
    const int lo = H - 1 - yhi, hi = H - 1 - ylo;
    s.LT = (int)align_up(lo + W - 1 + 64, 64);
    s.LB = (int)align_up((H - 1 - hi) + W - 1 + 64, 64);
    s.nchunk = (2 * W - 1 + 31) / 32;
    s.nwarps = nwarps;
    GridSmem o;
    grid_smem_layout(s, o);
    s.smem_bytes = o.total;
    return s.smem_bytes <= 227 * 1024;
}

cudaError_t launch_grid_solver(int solver, const GridParams &p, int grid, cudaStream_t stream) {
    const int threads = 32 * p.shape.nwarps;
    void (*kern)(GridParams) = solver == 0 ? redrec_kernel : bird_kernel;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.shape.smem_bytes);
    if (e != cudaSuccess) return e;
    kern<<<grid, threads, p.shape.smem_bytes, stream>>>(p);
    return cudaGetLastError();
}

int grid_occupancy(int solver, const GridShape &s) {
    int nb = 0;
    void (*kern)(GridParams) = solver == 0 ? redrec_kernel : bird_kernel;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s.smem_bytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 32 * s.nwarps, s.smem_bytes);
    return nb;
}

}  // namespace rb
