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

}  // namespace rb
