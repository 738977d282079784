// Device building blocks shared by the red-rec and bird kernels.
//
// Reference: virtual_line.cpp:97-229 (events, realization, emission order),
// exact1d.cpp:155-207 (the DP tie rule the split rule reproduces).
//
// Every column is a depth bit plane in shared memory (bit d = row d from the
// top, geometry.hpp:105) of wpd = ceil(H/64) u64 words; the band is depths
// [lo, hi].  An event fills the receiver's band (targets lo..hi,
// virtual_line.cpp:125) from residents (always used), top-side tokens (virtual
// position < lo) and bottom-side tokens (> hi).  SPLIT RULE: with a = number
// of top tokens used (mandatory ones plus the a - m_top optional ones nearest
// the band) and b = holes - a, cost(a) is convex and the reference's tie rule
// (lex-min use vector read from the last source) is the LARGEST minimiser, so
// a = a_min + #{a in (a_min, a_max] : Delta(a) <= 0}.  Used tokens sorted by
// (virtual pos, dist, column) take targets lo, lo+1, ... (virtual_line.cpp:
// 112-118, 195-225); rights (target > pos) emit by descending target, then
// lefts by ascending target (order_1d_intervals, exact1d.cpp:494-515).
#pragma once

#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "grid_solver.cuh"

namespace rb {

__host__ __device__ inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline void grid_smem_layout(const GridShape &s, GridSmem &o) {
    int64_t off = 0;
    auto take = [&](int64_t bytes, int64_t align) {
        off = align_up(off, align);
        const int64_t at = off;
        off += bytes;
        return at;
    };
    // arrays only one executor touches get no space in the other's layout
    // (solver 0 = red-rec executor, 1 = bird, else both)
    const int64_t R = s.solver != 1, Bd = s.solver != 0;
    o.dep = take((int64_t)s.W * s.wpd * 8, 16);
    const int64_t keys_a = (int64_t)s.nwarps * 2 * s.LK * 4;
    o.keys = take(R * keys_a, 16);
    o.bal = take(Bd * 2 * s.nchunk * 64 * 4, 16);
    o.sigma = take((int64_t)s.W * 4, 16);
    o.ev_count = take((int64_t)s.W * 4, 16);
    o.ev_off = take((int64_t)(s.W + 1) * 4, 16);
    o.wave_off = take(R * (s.W + 2) * 4, 16);
    o.lvl_t = take(Bd * s.LT * 4, 16);
    o.lvl_b = take(Bd * s.LB * 4, 16);
    o.scal = take(32 * 8, 16);
    o.lists = take((int64_t)s.nwarps * 4 * s.LK * 2, 16);
    o.plists = take(Bd * 2 * s.LK * 2, 16);
    o.mark_next = take(R * s.W * 2, 16);
    o.mark_head = take((int64_t)s.W * 2, 16);
    o.ev_col = take((int64_t)s.W * 2, 16);
    o.ev_aux = take(R * s.W * 2, 16);
    o.ev_a = take(Bd * s.W * 2, 16);
    o.wave_list = take(R * s.W * 2, 16);
    o.ev_type = take(R * s.W, 16);
    o.solved = take(s.W, 16);
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
    g.lo = s.lo;
    g.hi = s.hi;
    g.wpd = s.wpd;
    g.B = s.B;
    g.LK = s.LK;
    g.LT = s.LT;
    g.LB = s.LB;
    g.nchunk = s.nchunk;
    return g;
}

enum : uint8_t { EV_OWN = 0, EV_FLUSH = 1 };

struct PathOut {
    int32_t *src, *dst, *ev;
};

__device__ __forceinline__ int emit_slot(const Geo &g, int j, int n_right, int n_left) {
    return j < n_right ? n_right - 1 - j : n_right + j - (g.k - n_left);
}

__device__ __forceinline__ uint32_t tok_key(int v, int dist, int col) {
    return ((uint32_t)(v + 2048) << 20) | ((uint32_t)dist << 10) | (uint32_t)col;
}

// --------------------------------------------------------------------------
// warp-level compaction of one column (OWN event)
// --------------------------------------------------------------------------

struct OwnSolve {
    int a, b, R, holes, nt, nb, n_right, n_left;
};

// Lists (per warp, LK int16 each): otop[1..] = top depths, innermost first;
// obot[1..] = bottom depths, innermost first; hole[0..holes+1] = empty band
// depths with sentinels lo-1 / hi+1; res[0..R) = resident depths.
__device__ __forceinline__ bool own_solve(const Geo &g, const uint64_t *m, int16_t *L, int forced_a, OwnSolve &s) {
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

// Path sinks: PathOut writes vertex ids (src/dst/event arrays); a packed
// stage (redrec) keeps one word per path, source column << 20 | source depth
// << 10 | target depth, the target column being the event's.
__device__ __forceinline__ void emit_put(const PathOut &o, const Geo &g, int p, int scol, int sdepth, int dcol, int t,
                                         int evid) {
    o.src[p] = scol * g.H + (g.H - 1 - sdepth);
    o.dst[p] = dcol * g.H + (g.H - 1 - t);
    if (o.ev) o.ev[p] = evid;
}
__device__ __forceinline__ void emit_put(uint32_t *st, const Geo &, int p, int scol, int sdepth, int, int t, int) {
    st[p] = ((uint32_t)scol << 20) | ((uint32_t)sdepth << 10) | (uint32_t)t;
}

// Emits a solved OWN event at [off, off + count); returns its displacement
// (warp-uniform).
template <class Out>
__device__ __forceinline__ long long own_emit(const Geo &g, int col, const OwnSolve &s, const int16_t *L, Out o,
                                              int off, int evid) {
    const int16_t *otop = L, *obot = L + g.LK, *res = L + 3 * g.LK;
    long long disp = 0;
#pragma unroll 2
    for (int j = lane_id(); j < g.k; j += 32) {
        const bool right = j < s.n_right, left = j >= g.k - s.n_left;
        if (!right && !left) continue;
        const int depth = j < s.a ? otop[s.a - j] : (j < s.a + s.R ? res[j - s.a] : obot[j - s.a - s.R + 1]);
        const int t = g.lo + j;
        emit_put(o, g, off + emit_slot(g, j, s.n_right, s.n_left), col, depth, col, t, evid);
        disp += t > depth ? t - depth : depth - t;
    }
    return warp_sum64(disp);
}

// Column after its OWN event: band full, used reservoir tokens gone, parked
// (unused) reservoir tokens stay (redrec.cpp:150-164, bird.cpp:90-99).
// Returns the parked count.
__device__ __forceinline__ int own_update(const Geo &g, uint64_t *m, const OwnSolve &s, const int16_t *L) {
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
// per-CTA shared state
// --------------------------------------------------------------------------

struct Block {
    uint64_t *dep;
    uint32_t *keys, *bal;
    int *sigma, *ev_count, *ev_off, *wave_off, *lvl_t, *lvl_b, *scal;
    int16_t *lists, *plists, *mark_next, *mark_head, *ev_col, *ev_aux, *ev_a, *wave_list;
    uint8_t *ev_type, *solved;
};

__device__ __forceinline__ Block carve(const GridShape &s, unsigned char *smem) {
    GridSmem o;
    grid_smem_layout(s, o);
    Block b;
    b.dep = (uint64_t *)(smem + o.dep);
    b.keys = (uint32_t *)(smem + o.keys);
    b.bal = (uint32_t *)(smem + o.bal);
    b.sigma = (int *)(smem + o.sigma);
    b.ev_count = (int *)(smem + o.ev_count);
    b.ev_off = (int *)(smem + o.ev_off);
    b.wave_off = (int *)(smem + o.wave_off);
    b.lvl_t = (int *)(smem + o.lvl_t);
    b.lvl_b = (int *)(smem + o.lvl_b);
    b.scal = (int *)(smem + o.scal);
    b.lists = (int16_t *)(smem + o.lists);
    b.plists = (int16_t *)(smem + o.plists);
    b.mark_next = (int16_t *)(smem + o.mark_next);
    b.mark_head = (int16_t *)(smem + o.mark_head);
    b.ev_col = (int16_t *)(smem + o.ev_col);
    b.ev_aux = (int16_t *)(smem + o.ev_aux);
    b.ev_a = (int16_t *)(smem + o.ev_a);
    b.wave_list = (int16_t *)(smem + o.wave_list);
    b.ev_type = (uint8_t *)(smem + o.ev_type);
    b.solved = (uint8_t *)(smem + o.solved);
    return b;
}

// occ column (bit y from the bottom) -> depth plane (bit d = H-1-y); counts
__device__ __forceinline__ void load_instance(const Geo &g, const uint64_t *occ, Block &b,
                                              long long *total_tokens) {
    const int wpc = g.wpd;
    const int shift = 64 * wpc - g.H;
    const uint64_t last_mask = (g.H & 63) ? ((1ull << (g.H & 63)) - 1ull) : ~0ull;
    long long tot = 0;
    for (int x = threadIdx.x; x < g.W; x += blockDim.x) {
        const uint64_t *src = occ + (size_t)x * wpc;
        uint64_t *dst = b.dep + (size_t)x * g.wpd;
        int cnt = 0;
        for (int j = 0; j < wpc; ++j) {
            // reversed word j = brev(src[wpc-1-j]); then shift right by `shift` across words
            const uint64_t lo = __brevll(src[wpc - 1 - j] & (j == 0 ? last_mask : ~0ull));
            const uint64_t hi = (j + 1 < wpc) ? __brevll(src[wpc - 2 - j]) : 0ull;
            const uint64_t v = shift == 0 ? lo : ((lo >> shift) | (hi << (64 - shift)));
            dst[j] = v;
            cnt += __popcll(v);
        }
        b.sigma[x] = cnt - g.k;
        b.solved[x] = 0;
        b.mark_head[x] = -1;
        tot += cnt;
    }
    tot = warp_sum64(tot);
    if (lane_id() == 0 && tot) atomicAdd((unsigned long long *)total_tokens, (unsigned long long)tot);
}

// next instance of a persistent CTA: the static stride, or (p.work) the next
// unclaimed instance of a global counter -- instance costs vary, and a static
// split leaves the last round's CTAs idle behind the slowest ones
__device__ __forceinline__ int next_instance(const GridParams &p, int inst, int *s_next) {
    if (!p.work) return inst + gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) *s_next = gridDim.x + atomicAdd(p.work, 1);
    __syncthreads();
    return *s_next;
}

// exclusive scan of vals[idx[i]] for i in [0, n) into out[idx[i]] (warp 0); returns the total
__device__ __forceinline__ int scan_indexed(const int *vals, const int16_t *idx, int n, int *out, int base) {
    int run = base;
    for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane_id();
        const int v = i < n ? vals[idx[i]] : 0;
        int tot;
        const int ex = warp_excl_scan(v, &tot);
        if (i < n) out[idx[i]] = run + ex;
        run += tot;
    }
    return run;
}

}  // namespace rb
